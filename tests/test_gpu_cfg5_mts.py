"""BASELINE cfg5 as a coupled run (configs.py cfg5_mts: 3D plate, 0.25 mm PD core,
1 mm hex8 FE, m = 20, explicit FE) -- its small twin on the device: the coupled step
holds velocity continuity, stays finite, breaks bonds at the notch, and two PD shards
reproduce it bit for bit.  The at-size run is bench.py --workload
cfg5_mts (profiles/)."""
import copy

import numpy as np
import pytest

from paper_2403_03605_b200 import configs as cf
from paper_2403_03605_b200.mts import MtsSolver, ShardGroup

pytestmark = pytest.mark.gpu


def test_cfg5_twin_coupled_run():
    s = MtsSolver(cf.get("cfg5_mts_small"))
    s.initialize()
    reps = s.macro_step(20)
    assert max(r["continuity"] for r in reps) <= 1e-8
    for w in ("fe", "pd"):
        for x in s.state(w):
            assert np.isfinite(x).all()
    assert np.abs(s.state("pd")[0]).max() > 0


def test_cfg5_twin_shards_bitwise():
    c = copy.deepcopy(cf.get("cfg5_mts_small"))
    one = MtsSolver(c)
    one.initialize()
    grp = ShardGroup(c, 2)
    grp.initialize()
    r1, rg = one.macro_step(10), grp.macro_step(10)
    for a, b in zip(r1, rg):
        for f in ("newly_broken", "interface_iterations", "continuity", "lambda_fe", "lambda_pd"):
            assert a[f] == b[f], f
    assert np.array_equal(one.lam(), grp.lam())
    for w in ("fe", "pd"):
        for x, y in zip(one.state(w), grp.state(w)):
            assert np.array_equal(x, y)


def test_lattice_linear_force_matches_ell():
    """The homogeneous substeps' linear PD force on the lattice tile kernel (default on a
    3D box lattice, pd_mts_lat.cu) is the ELL form's operator -- the same coefficients in
    stencil order, xi = h o instead of centroid differences: the coupled run it drives
    equals the ELL-driven one to rounding (multipliers, states, broken counts)."""
    out = {}
    for form in ("lattice", "ell"):
        c = copy.deepcopy(cf.get("cfg5_mts_small"))
        c.setdefault("run", {})["pd_linear"] = form
        s = MtsSolver(c)
        assert bool(s.view.pd_linear_lattice) == (form == "lattice")
        s.initialize()
        reps = s.macro_step(12)
        out[form] = (reps, s.lam(), s.state("fe"), s.state("pd"))
    a, b = out["lattice"], out["ell"]
    assert [r["newly_broken"] for r in a[0]] == [r["newly_broken"] for r in b[0]]
    assert all(abs(x["interface_iterations"] - y["interface_iterations"]) <= 1
               for x, y in zip(a[0], b[0]))
    assert max(r["continuity"] for r in a[0]) <= 1e-8
    assert np.linalg.norm(a[1] - b[1]) <= 1e-7 * np.linalg.norm(b[1])
    for w in (2, 3):
        for x, y in zip(a[w], b[w]):
            assert np.linalg.norm(x - y) <= 1e-8 * max(np.linalg.norm(y), 1e-300)


def test_element_products_are_bitwise():
    """Free PD substeps with the per-element node products formed once per force call
    (the default from 2^18 PD elements on) instead of once per family entry: the same
    expressions, so reports, multipliers, states and bond states are bit for bit equal."""
    out = {}
    for form in ("on", "off"):
        c = copy.deepcopy(cf.get("cfg5_mts_small"))
        c.setdefault("run", {})["pd_elem_products"] = form
        s = MtsSolver(c)
        s.initialize()
        reps = s.macro_step(12)
        out[form] = (reps, s.lam(), s.state("fe"), s.state("pd"), s.intact())
    a, b = out["on"], out["off"]
    assert sum(r["newly_broken"] for r in a[0]) > 0
    for x, y in zip(a[0], b[0]):
        for f in ("newly_broken", "interface_iterations", "continuity", "lambda_fe", "lambda_pd"):
            assert x[f] == y[f], f
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[4], b[4])
    for w in (2, 3):
        for x, y in zip(a[w], b[w]):
            assert np.array_equal(x, y)
