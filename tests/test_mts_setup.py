"""Coupled MTS setup: the product's host assembly
(pmts_mts_setup.cpp, built with device=-1 -- no GPU) against the reference's own
assembled systems (tests/golden/mts_*.npz, made by oracle/_ref/ref_mts_driver):
subdomain labels, blend weights, dof maps, the alpha-weighted FE stiffness in
CSR, lumped masses, surface loads, kinematic constraints and coupling rows --
all bitwise."""
import numpy as np
import pytest

from conftest import load_golden
from paper_2403_03605_b200 import configs as cf
from paper_2403_03605_b200.mts import MtsSolver

FIXTURES = ["mts_mini", "mts_mini_implicit", "mts_mini_frac", "mts_mini_mfree", "mts_bar3d"]
KEYS = ["labels", "alpha", "fe_node_dof", "pd_node_dof", "fe_k_rowptr", "fe_k_col", "fe_k_val",
        "fe_mass", "fe_p_ext", "pd_mass", "pd_p_ext", "fe_bc_dofs", "fe_bc_vel", "pd_bc_dofs",
        "pd_bc_vel", "fe_dof", "pd_dof"]


@pytest.mark.parametrize("name", FIXTURES)
def test_mts_setup_bitwise(name):
    g = load_golden(name)
    s = MtsSolver(cf.get(g["meta"]["scenario"]), device=-1)
    sy = s.system()
    for k in KEYS:
        assert np.array_equal(sy[k], g[k]), k
    assert s.n_lambda == int(g["meta"]["n_lambda"])
    assert s.dense == bool(g["meta"]["dense"])
    m = g["meta"]
    for k in ("delta", "c0", "l"):
        assert sy[k] == pytest.approx(m[k], rel=1e-15), k


def test_mts_setup_rejects_bad_region():
    sc = cf.get("mts_mini")
    sc["region"]["pd_box1"] = [0.0, 0.0, 0.03, 0.01]  # whole domain: no overlap band
    with pytest.raises(Exception):
        MtsSolver(sc, device=-1)
