"""The coupled-integrator hooks of the pure-PD handle: what a
reference CoupledIntegrator (mts.hpp:79-535) that keeps its own FE side calls for the
PD side -- the constraint load G_PD^T S_j of free_solve_pd (mts.hpp:160-162), the k_sync_
snapshot (mts.hpp:98, 252) and the homogeneous linear recursion of unit_pd_column /
apply_h_pd / recombine (mts.hpp:230-238, 398-420)."""
import numpy as np
import pytest

from paper_2403_03605_b200 import capi
from paper_2403_03605_b200 import configs as cf
from paper_2403_03605_b200.pd import PDSolver, Scenario

pytestmark = pytest.mark.gpu


def _handle(sc, p_ext=None, s_crit=None):
    over = {}
    if p_ext is not None:
        over["p_ext"] = p_ext
    if s_crit is not None:
        over["s_crit"] = s_crit
    return PDSolver.from_scenario(sc, mode=capi.DETERMINISTIC, **over).find_pe_pairs()


def test_constraint_load_is_an_external_load():
    """Stepping with a constraint load at some dofs is bitwise stepping with that load
    added to P (load scale 1: P * 1 + S == (P + S) * 1); clearing it restores P."""
    sc = Scenario(cf.get("mini"))
    rng = np.random.default_rng(3)
    dofs = np.array([10, 11, 200, 333, 501], dtype=np.int32)
    vals = rng.normal(size=len(dofs)) * 1e-3
    assert (sc.p_ext[dofs] == 0).all()
    a = _handle(sc)
    p2 = sc.p_ext.copy()
    p2[dofs] += vals
    b = _handle(sc, p_ext=p2)
    a.set_constraint_load(dofs, vals)
    a.initial_acceleration(1.0)
    b.initial_acceleration(1.0)
    na = a.step(np.ones(60))
    nb = b.step(np.ones(60))
    assert na == nb
    for x, y in zip(a.state(), b.state()):
        assert np.array_equal(x, y)
    assert np.array_equal(a.intact(), b.intact())


def test_homogeneous_recursion_equals_explicit_steps():
    """The m homogeneous linear substeps from rest under the ramped load w j/m at the
    rows equal m explicit steps of a fracture-free handle whose only load is w at those
    dofs with the load scales j/m (the recursion's centroid-form force against the step's
    per-entry form: within 1e-12)."""
    sc = Scenario(cf.get("mini"))
    m = 10
    rng = np.random.default_rng(5)
    dofs = np.array([40, 41, 95, 96, 700, 701], dtype=np.int32)
    w = rng.normal(size=len(dofs)) * 1e3
    a = _handle(sc, s_crit=0.0)
    a.snapshot_bonds()
    vel, (u, v, acc) = a.homogeneous_recursion(m, dofs, w, state=True)
    p = np.zeros(sc.n_dof)
    p[dofs] = w
    b = _handle(sc, p_ext=p, s_crit=0.0)
    b.initial_acceleration(0.0)
    assert np.all(vel[0] == 0.0)
    for j in range(1, m + 1):
        b.step([j / m])
        _, vb, _ = b.state()
        assert np.linalg.norm(vel[j] - vb[dofs]) <= 1e-12 * np.linalg.norm(vb[dofs])
    ub, vb, ab = b.state()
    for x, y in ((u, ub), (v, vb), (acc, ab)):
        assert np.linalg.norm(x - y) <= 1e-12 * np.linalg.norm(y)


def test_recursion_uses_the_snapshot():
    """Bonds broken after the snapshot do not change the recursion until the next
    snapshot (k_sync_ semantics, mts.hpp:249-260)."""
    sc = Scenario(cf.get("mini"))
    s = _handle(sc)
    s.snapshot_bonds()
    dofs = np.array([2 * (sc.n_nodes // 2), 2 * (sc.n_nodes // 2) + 1], dtype=np.int32)
    w = np.array([1e3, -2e3])
    r0 = s.homogeneous_recursion(5, dofs, w)
    s.initial_acceleration(sc.load_scale(0.0))
    assert s.step(sc.scales(1, 80)) > 0  # the mini plate cracks
    r1 = s.homogeneous_recursion(5, dofs, w)
    assert np.array_equal(r0, r1)
    s.snapshot_bonds()
    r2 = s.homogeneous_recursion(5, dofs, w)
    assert not np.array_equal(r0, r2)
