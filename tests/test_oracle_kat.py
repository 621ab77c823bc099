"""Known-answer tests of the reference (test_perifem.cpp, test_mesh.cpp) on the oracle."""
import numpy as np
import pytest

import kat_meshes as km
from oracle import pyoracle as po


def _u_move(mesh, elem, comp, val):
    u = np.zeros(2 * len(mesh["nodes"]))
    for n in mesh["conn"][elem]:
        u[2 * n + comp] = val
    return u


def test_stretch_elementary():  # test_perifem.cpp:126-145
    m = km.disjoint_quads()
    o = po.OraclePD(km.pd_sys(m, [[0, 1]]), po.MF)
    assert o.stretch(0, np.zeros(16)) == 0.0
    assert o.stretch(0, _u_move(m, 1, 0, 0.1)) == pytest.approx(0.1, rel=1e-12)
    assert o.stretch(0, _u_move(m, 1, 0, -1.0)) == -1.0


def test_stretch_vector_case():  # test_perifem.cpp:147-169
    m = km.manufactured_quads()
    o = po.OraclePD(km.pd_sys(m, [[0, 1]], delta=6.0, l=1.5), po.MF)
    u = _u_move(m, 1, 0, 0.6) + _u_move(m, 1, 1, 0.8)
    assert o.stretch(0, u) == pytest.approx(0.2, rel=1e-13)


def test_threshold_inclusive_and_irreversible():  # test_perifem.cpp:171-196
    m = km.disjoint_quads()
    s_crit = 0.1
    o = po.OraclePD(km.pd_sys(m, [[0, 1]], s_crit=s_crit), po.MF)
    assert len(o.update_bond_states(_u_move(m, 1, 0, s_crit - 1e-9))) == 0
    assert o.mu()[0] == 1
    assert list(o.update_bond_states(_u_move(m, 1, 0, s_crit))) == [0]
    assert o.mu()[0] == 0
    assert len(o.update_bond_states(_u_move(m, 1, 0, 2 * s_crit))) == 0
    assert o.mu()[0] == 0


def test_damage_limits():  # test_perifem.cpp:198-227
    m = km.grid(3, 1, 1.0)
    pairs = po.find_pairs(2, m["centroid"], m["volume"], 1.5)
    assert pairs.tolist() == [[0, 1], [1, 2]]
    o = po.OraclePD(km.pd_sys(m, pairs), po.MF)
    e, n = o.damage()
    assert (e == 0).all() and (n == 0).all()
    o.set_mu(np.array([0, 0], np.uint8))
    e, _ = o.damage()
    assert e == pytest.approx([1, 1, 1])
    o.set_mu(np.array([0, 1], np.uint8))
    e, _ = o.damage()
    assert e[1] == pytest.approx(0.5) and e[0] == pytest.approx(1.0) and e[2] == 0.0


def test_two_quads_pair_within_horizon():  # test_mesh.cpp:103-108
    m = km.grid(2, 1, 1.0)
    assert len(po.find_pairs(2, m["centroid"], m["volume"], 1.01)) == 1
    assert len(po.find_pairs(2, m["centroid"], m["volume"], 0.99)) == 0


def test_hash_equals_brute_force():  # test_mesh.cpp:110-120
    m = km.grid(40, 16, 1e-3)
    fast = po.find_pairs(2, m["centroid"], m["volume"], 3.03e-3)
    slow = km.brute_force_pairs(m["centroid"], 3.03e-3)
    assert np.array_equal(fast, slow)


def test_hash_equals_brute_force_with_notch():  # test_mesh.cpp:122-135
    m = km.grid(20, 10, 1e-3)
    notch = [10e-3, 10e-3, 0, 10e-3, 4e-3, 0]
    fast = po.find_pairs(2, m["centroid"], m["volume"], 3.03e-3, [notch])
    slow = km.brute_force_pairs(m["centroid"], 3.03e-3, [notch])
    assert np.array_equal(fast, slow)
    assert len(fast) < len(po.find_pairs(2, m["centroid"], m["volume"], 3.03e-3))


def test_notch_cases():  # test_mesh.cpp:137-153
    m = km.grid(2, 1, 1.0)
    cross = [1.0, -0.5, 0, 1.0, 1.5, 0]
    far = [1.0, 2.0, 0, 1.0, 3.0, 0]
    touch = [1.0, 0.5, 0, 1.0, 2.0, 0]
    assert len(po.find_pairs(2, m["centroid"], m["volume"], 1.01, [cross])) == 0
    assert len(po.find_pairs(2, m["centroid"], m["volume"], 1.01, [far])) == 1
    assert len(po.find_pairs(2, m["centroid"], m["volume"], 1.01, [touch])) == 0


def test_notch_monotone():  # test_mesh.cpp:155-173
    m = km.grid(12, 8, 1e-3)
    long_n = [6e-3, 8e-3, 0, 6e-3, 2e-3, 0]
    short_n = [6e-3, 8e-3, 0, 6e-3, 4e-3, 0]
    a = {tuple(p) for p in po.find_pairs(2, m["centroid"], m["volume"], 2.5e-3, [long_n])}
    b = {tuple(p) for p in po.find_pairs(2, m["centroid"], m["volume"], 2.5e-3, [short_n])}
    assert a <= b


def test_pairs_sorted_unique():  # test_mesh.cpp:248-257
    m = km.grid(10, 6, 1e-3)
    p = po.find_pairs(2, m["centroid"], m["volume"], 2.5e-3)
    assert (p[:, 0] < p[:, 1]).all()
    key = p[:, 0].astype(np.int64) * 10**6 + p[:, 1]
    assert (np.diff(key) > 0).all()


def test_bond_s_crit_factor_range():
    vals = np.array([po.bond_s_crit(1.0, 0.05, 1234, i, i + 7) for i in range(20000)])
    assert vals.min() >= 0.95 and vals.max() < 1.05
    assert abs(vals.mean() - 1.0) < 2e-3
    assert po.bond_s_crit(2e-4, 0.0, 1, 3, 4) == 2e-4
