"""Slab decomposition on the device: several rank handles on ONE GPU, stepped in
turn with a host-mediated halo exchange (pmts_pd_get_rows / set_rows) -- no
kernel ever waits on another rank -- must reproduce the single-domain run bit
for bit (owned u/v/a and bond states), in both modes.  On a multi-GPU box the
same handles exchange with ncclSend/ncclRecv inside pmts_pd_step instead."""
import numpy as np
import pytest

from paper_2403_03605_b200 import capi, slabs
from paper_2403_03605_b200 import configs as cf
from paper_2403_03605_b200.pd import PDSolver, Scenario

pytestmark = pytest.mark.gpu


def _run_slabs(sc, nranks, mode, steps):
    hs = [slabs.solver_for_slab(sc, slabs.make_slab(sc.lattice, sc.dim, r, nranks), mode)
          for r in range(nranks)]
    v0 = sc.initial_velocity()
    d = sc.dim
    for h in hs:
        h.find_pe_pairs()
        if v0.any():
            n0, n1 = h.slab.node_first, h.slab.node_first + h.slab.n_nodes
            z = np.zeros(h.n_dof)
            h.set_state(z, v0[n0 * d:n1 * d], z)
        h.initial_acceleration(sc.load_scale(0.0))

    def exchange():
        msgs = []
        for r, h in enumerate(hs):
            plo, slo, rlo, nlo, phi, shi, rhi, nhi = h.slab.halo
            if plo >= 0:
                msgs.append((plo, hs[plo].slab.halo[6], nlo, h.get_rows(slo, nlo)))
            if phi >= 0:
                msgs.append((phi, hs[phi].slab.halo[2], nhi, h.get_rows(shi, nhi)))
        for dst, first, n, vals in msgs:
            hs[dst].set_rows(first, n, vals)

    exchange()
    nb = 0
    for i in range(1, steps + 1):
        for h in hs:
            nb += h.step([sc.load_scale(i * sc.dt)])
        exchange()
    return hs, nb


@pytest.mark.parametrize("mode", [capi.DETERMINISTIC, capi.FAST])
@pytest.mark.parametrize("name,nranks,steps", [("mini", 3, 80), ("cfg1", 4, 120),
                                               ("cfg4_small", 2, 60), ("cfg5_core_small", 2, 120)])
def test_slabs_equal_single_domain(mode, name, nranks, steps):
    sc = Scenario(cf.get(name))
    one = PDSolver.from_scenario(sc, mode=mode).find_pe_pairs()
    v0 = sc.initial_velocity()
    if v0.any():
        z = np.zeros(sc.n_dof)
        one.set_state(z, v0, z)
    one.initial_acceleration(sc.load_scale(0.0))
    nb1 = one.step([sc.load_scale(i * sc.dt) for i in range(1, steps + 1)])
    u, v, a = one.state()
    pairs = one.pairs()
    intact = one.intact()
    idx = {(int(i), int(j)): q for q, (i, j) in enumerate(pairs)}
    hs, nb = _run_slabs(sc, nranks, mode, steps)
    assert nb == nb1 and nb1 > 0
    d = sc.dim
    for h in hs:
        s = h.slab
        lu, lv, la = h.state()
        n0, n1 = s.own_nodes
        g0, g1 = s.global_nodes(n0, n1)
        assert np.array_equal(lu[n0 * d:n1 * d], u[g0 * d:g1 * d])
        assert np.array_equal(lv[n0 * d:n1 * d], v[g0 * d:g1 * d])
        assert np.array_equal(la[n0 * d:n1 * d], a[g0 * d:g1 * d])
        lp = h.pairs()
        li = h.intact()
        own = (lp[:, 0] >= s.own_elems[0]) & (lp[:, 0] < s.own_elems[1])
        for (i, j), m in zip(lp[own] + s.elem_first, li[own]):
            assert intact[idx[(int(i), int(j))]] == m
