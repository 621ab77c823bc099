"""Pin the CPU restatement (oracle/pd_oracle.c) against the reference's own outputs.

The goldens were produced by the unmodified reference loop (tests/golden/
make_golden.py).  PO_CSR replays the reference's arithmetic and must match
bit for bit; PO_MF (the order the CUDA deterministic kernel uses) must give the
identical broken-bond set and u/v/a within 1e-12 relative L2.
"""
import numpy as np
import pytest

from conftest import GOLDEN_SCENARIO, load_golden, oracle_sys
from oracle import pyoracle as po
from paper_2403_03605_b200 import configs as cf
from paper_2403_03605_b200.pd import Scenario

FAST = ["mini", "block3d", "cfg1_200"]


def _run(name, variant):
    g = load_golden(name)
    sc = Scenario(cf.get(GOLDEN_SCENARIO[name]))
    o = po.OraclePD(oracle_sys(g, sc), variant)
    o.init(g["scale"][0])
    steps = g["meta"]["steps"]
    br, st = o.step(g["scale"][1:steps + 1])
    return g, o, br, st


@pytest.mark.parametrize("name", FAST)
def test_csr_oracle_bitwise(name):
    g, o, br, st = _run(name, po.CSR)
    assert o.nnz() == g["meta"]["nnz"]
    u, v, a = o.state()
    assert np.array_equal(u, g["u"]) and np.array_equal(v, g["v"]) and np.array_equal(a, g["a"])
    assert np.array_equal(np.stack([st, br], 1), g["broken"])
    e, n = o.damage()
    assert np.array_equal(e, g["damage_elem"]) and np.array_equal(n, g["damage_node"])


@pytest.mark.parametrize("name", FAST)
def test_mf_oracle_matches_reference(name):
    g, o, br, st = _run(name, po.MF)
    assert np.array_equal(np.stack([st, br], 1), g["broken"])
    u, v, a = o.state()
    for x, ref in ((u, g["u"]), (v, g["v"]), (a, g["a"])):
        assert np.linalg.norm(x - ref) <= 1e-12 * np.linalg.norm(ref)
    e, n = o.damage()
    assert np.array_equal(e, g["damage_elem"]) and np.array_equal(n, g["damage_node"])


@pytest.mark.slow
def test_bp_coarse_2000_csr_bitwise():
    g, o, br, st = _run("bp_coarse_2000", po.CSR)
    u, v, a = o.state()
    assert np.array_equal(u, g["u"]) and np.array_equal(v, g["v"])
    assert np.array_equal(np.stack([st, br], 1), g["broken"])
    assert len(br) == 10  # first breaks appear before step 2000 in the reference too


@pytest.mark.parametrize("name", list(GOLDEN_SCENARIO))
def test_pair_search_matches_reference(name):
    g = load_golden(name)
    sc = Scenario(cf.get(GOLDEN_SCENARIO[name]))
    pairs = po.find_pairs(sc.dim, g["centroid"], g["volume"], g["meta"]["delta"], sc.notches())
    assert np.array_equal(pairs, g["pairs"])


@pytest.mark.parametrize("name", list(GOLDEN_SCENARIO))
def test_setup_matches_reference_bitwise(name):
    """The product's C++ setup (pmts_scenario_build) equals the reference's."""
    g = load_golden(name)
    sc = Scenario(cf.get(GOLDEN_SCENARIO[name]))
    assert np.array_equal(sc.centroid, g["centroid"])
    assert np.array_equal(sc.volume, g["volume"])
    assert np.array_equal(sc.mass, g["mass"])
    assert np.array_equal(sc.p_ext, g["p_ext"])
    m = g["meta"]
    assert sc.delta == m["delta"] and sc.l == m["l"] and sc.c0 == m["c0"]
    assert sc.char_length == m["char_length"]
    assert np.array_equal(sc.scales(0, len(g["scale"])), g["scale"])
