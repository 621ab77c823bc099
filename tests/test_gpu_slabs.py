"""Slab decomposition on the device: several rank handles on ONE GPU, stepped in
turn with a host-mediated halo exchange (pmts_pd_get_rows_layers / set_rows_layers)
-- no kernel ever waits on another rank -- must reproduce the single-domain run bit
for bit (owned u/v/a and bond states), in both modes.  2D plates are cut into
x-slabs, 3D blocks into z-x slabs (along y, one halo range per z node layer).  On
a multi-GPU box the same handles exchange with ncclSend/ncclRecv inside
pmts_pd_step instead (tests/test_gpu_nccl_slabs.py)."""
import numpy as np
import pytest

from paper_2403_03605_b200 import capi, slabs
from paper_2403_03605_b200 import configs as cf
from paper_2403_03605_b200.pd import PDSolver, Scenario

pytestmark = pytest.mark.gpu


def run_slabs(sc, nranks, mode, steps):
    hs = [slabs.solver_for_slab(sc, slabs.make_slab(sc.lattice, sc.dim, r, nranks), mode)
          for r in range(nranks)]
    v0 = sc.initial_velocity()
    for h in hs:
        h.find_pe_pairs()
        if v0.any():
            z = np.zeros(h.n_dof)
            h.set_state(z, v0[h.local_dofs], z)
        h.initial_acceleration(sc.load_scale(0.0))
    slabs.host_exchange(hs)
    nb = 0
    for i in range(1, steps + 1):
        for h in hs:
            nb += h.step([sc.load_scale(i * sc.dt)])
        slabs.host_exchange(hs)
    return hs, nb


def single_domain(sc, mode, steps):
    one = PDSolver.from_scenario(sc, mode=mode).find_pe_pairs()
    v0 = sc.initial_velocity()
    if v0.any():
        z = np.zeros(sc.n_dof)
        one.set_state(z, v0, z)
    one.initial_acceleration(sc.load_scale(0.0))
    nb = one.step([sc.load_scale(i * sc.dt) for i in range(1, steps + 1)])
    return one, nb


def assert_slabs_equal(sc, one, hs):
    """Owned u, v, a of every slab bitwise the single domain's; every owned bond's
    state equal; the owned nodes cover the mesh exactly once."""
    u, v, a = one.state()
    idx = {(int(i), int(j)): q for q, (i, j) in enumerate(one.pairs())}
    intact = one.intact()
    gu, gv, ga = slabs.gather_owned(hs, sc.n_dof, sc.dim)
    assert not np.isnan(gu).any()  # every node owned by some rank
    assert np.array_equal(gu, u) and np.array_equal(gv, v) and np.array_equal(ga, a)
    n_owned = 0
    for h in hs:
        s = h.slab
        n_owned += len(s.owned_nodes())
        lp, li = h.pairs(), h.intact()
        own = s.owns_elem(lp[:, 0])
        gi, gj = s.elem_global(lp[own, 0]), s.elem_global(lp[own, 1])
        q = np.array([idx[(int(i), int(j))] for i, j in zip(gi, gj)])
        assert np.array_equal(li[own], intact[q])
    assert n_owned == sc.n_nodes


@pytest.mark.parametrize("mode", [capi.DETERMINISTIC, capi.FAST])
@pytest.mark.parametrize("name,nranks,steps", [("mini", 3, 80), ("cfg1", 4, 120),
                                               ("cfg4_small", 2, 60), ("cfg5_core_small", 3, 120),
                                               ("block3d", 2, 100)])
def test_slabs_equal_single_domain(mode, name, nranks, steps):
    sc = Scenario(cf.get(name))
    one, nb1 = single_domain(sc, mode, steps)
    hs, nb = run_slabs(sc, nranks, mode, steps)
    assert nb == nb1
    if name != "cfg4_small":
        assert nb1 > 0
    assert_slabs_equal(sc, one, hs)


def test_slabs_3d_per_bond_spread_global_ids():
    """3D z-x slabs with the per-bond s0 factor: the hash keys of a slab's bonds are
    global ids through the layer map (slab_plane) -- bitwise the single domain."""
    c = cf.get("cfg5_core_small")
    c["ext"].update(s_crit_spread=0.05, seed=0x5eed5 + 5)
    sc = Scenario(c)
    for mode in (capi.DETERMINISTIC, capi.FAST):
        one, nb1 = single_domain(sc, mode, 120)
        hs, nb = run_slabs(sc, 3, mode, 120)
        assert nb == nb1 and nb1 > 0
        assert_slabs_equal(sc, one, hs)
