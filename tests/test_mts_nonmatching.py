"""Non-matching FE / PD meshes for the coupled MTS run (SURVEY.md 8(f) row 4,
an extension: the reference couples one conforming mesh, coupling.hpp:69-105).

The FE lattice (mesh.fe_spacing) covers the domain, the PD lattice (mesh.spacing,
which sets the horizon) the PD boxes' hull; the coupling row of each PD overlap
node interpolates the FE velocity with the shape functions of the FE element
containing it.  No oracle exists for it, so it is pinned two ways:
  * fe_spacing == spacing must rebuild the reference's conforming model exactly
    (host systems bitwise here; the device run bitwise in test_gpu_mts_nonmatching);
  * coarser FE lattices converge to the conforming analog (GPU test)."""
import copy

import numpy as np
import pytest

from conftest import load_golden
from paper_2403_03605_b200 import configs as cf
from paper_2403_03605_b200.mts import MtsSolver

SAME = ["fe_k_rowptr", "fe_k_col", "fe_k_val", "fe_mass", "fe_p_ext", "pd_mass", "pd_p_ext",
        "fe_bc_dofs", "fe_bc_vel", "pd_bc_dofs", "pd_bc_vel", "fe_dof", "pd_dof"]


def nonmatching(name: str, ratio: int) -> dict:
    sc = cf.get(name)
    sc["mesh"]["fe_spacing"] = sc["mesh"]["spacing"]
    sc["mesh"]["spacing"] = sc["mesh"]["spacing"] / ratio
    sc["region"]["overlap_width_factor"] = sc["region"]["overlap_width_factor"] * ratio
    return sc


@pytest.mark.parametrize("name", ["mts_mini", "mts_mini_implicit", "mts_bar3d"])
def test_unit_ratio_rebuilds_the_conforming_model(name):
    g = load_golden(name)
    sc = cf.get(g["meta"]["scenario"])
    sc["mesh"]["fe_spacing"] = sc["mesh"]["spacing"]
    s = MtsSolver(sc, device=-1).system()
    for k in SAME:  # == the reference's own assembled systems
        assert np.array_equal(s[k], g[k]), k
    assert np.all(s["cpl_fe_w"] == 1.0)
    assert np.array_equal(s["cpl_fe_col"], g["fe_dof"])
    assert np.array_equal(s["cpl_fe_rowptr"], np.arange(len(g["fe_dof"]) + 1))


@pytest.mark.parametrize("name,ratio", [("mts_mini", 2), ("mts_mini", 4), ("mts_bar3d", 2)])
def test_interpolation_rows(name, ratio):
    sc = nonmatching(name, ratio)
    s = MtsSolver(sc, device=-1).system()
    rp, w = s["cpl_fe_rowptr"], s["cpl_fe_w"]
    dim = int(sc["mesh"]["dim"])
    sums = np.add.reduceat(w, rp[:-1])
    assert np.array_equal(sums, np.ones_like(sums))  # partition of unity, exact on the lattice
    assert np.all(w > 0) and np.all(np.diff(rp) >= 1) and np.all(np.diff(rp) <= 2 ** dim)
    # a PD overlap node on an FE node is a plain (weight 1) row
    assert (np.diff(rp) == 1).sum() > 0
    # rows: the PD overlap nodes (x dim components, none constrained here)
    nodes = s["node_xyz"]
    nfe = s["fe_mesh_nodes"]
    pd_nodes = np.nonzero(s["pd_node_dof"] >= 0)[0]
    assert pd_nodes.min() >= nfe
    # the interpolated FE position of each row's node is the node itself
    fe_dof_node = {}
    for n in range(nfe):
        if s["fe_node_dof"][n] >= 0:
            fe_dof_node[int(s["fe_node_dof"][n])] = n
    pd_dof_node = {int(s["pd_node_dof"][n]): n for n in pd_nodes}
    for r in range(len(rp) - 1):
        c = int(s["pd_dof"][r]) % dim
        n = pd_dof_node[int(s["pd_dof"][r]) - c]
        x = sum(w[j] * nodes[fe_dof_node[int(s["cpl_fe_col"][j]) - c]] for j in range(rp[r], rp[r + 1]))
        assert np.allclose(x, nodes[n], rtol=0, atol=1e-15)


def test_rejects_unaligned_or_thin_overlap():
    sc = nonmatching("mts_mini", 2)
    sc["region"]["overlap_width_factor"] = 1.0  # 0.5 mm overlap < one FE element
    with pytest.raises(Exception):
        MtsSolver(sc, device=-1)
    sc = nonmatching("mts_mini", 2)
    sc["mesh"]["fe_spacing"] = 1.5e-3  # not a multiple of the PD spacing 0.5 mm? it is (3x)
    sc["mesh"]["fe_spacing"] = 1.25e-3
    with pytest.raises(Exception):
        MtsSolver(sc, device=-1)
