"""Slab decomposition host logic, world_size 2 over gloo on CPU.

Each rank runs the matrix-free oracle (the order the device uses) on its slab
(`paper_2403_03605_b200.slabs`: the same partition, halo widths, ownership and
global-id mapping the GPU ranks use) and exchanges the halo node rows after
every step over torch.distributed; the owned u/v/a and bond states must equal
a single-domain run bit for bit.
"""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scenario(name, spread):
    from paper_2403_03605_b200 import configs as cf

    sc = cf.get(name)
    if spread:
        sc["ext"] = {"s_crit_spread": 0.05, "seed": 99}
    return sc


def _sysd(sc, la, pairs, slab=None):
    ext = sc.cfg.get("ext", {})
    d = dict(dim=sc.dim, n_nodes=len(la["nodes"]), conn=la["conn"], centroid=la["centroid"],
             volume=la["volume"], pairs=pairs, mass=la["mass"], p_ext=la["p_ext"],
             bc_dofs=la["bc_dofs"], bc_vel=la["bc_vel"], delta=sc.delta, l=sc.l, c0=sc.c0,
             s_crit=sc.s_crit, dt=sc.dt, gamma=sc.gamma, beta=sc.beta,
             global_id_offset=slab.elem_first if slab else 0)
    if ext.get("s_crit_spread"):
        d.update(s_crit_spread=ext["s_crit_spread"], seed=int(ext["seed"]))
    return d


def _worker(rank, world, port, name, steps, spread, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from oracle import pyoracle as po
    from paper_2403_03605_b200 import slabs
    from paper_2403_03605_b200.pd import Scenario

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    sc = Scenario(_scenario(name, spread))
    slab = slabs.make_slab(sc.lattice, sc.dim, rank, world)
    la = slabs.local_arrays(sc, slab)
    pairs = po.find_pairs(sc.dim, la["centroid"], la["volume"], sc.delta, sc.notches())
    o = po.OraclePD(_sysd(sc, la, pairs, slab), po.MF)
    o.init(sc.load_scale(0.0))
    d = sc.dim
    plo, slo, rlo, nlo, phi, shi, rhi, nhi = slab.halo
    for i in range(1, steps + 1):
        o.step([sc.load_scale(i * sc.dt)])
        st = list(o.state())
        reqs, bufs = [], []
        for peer, s0, r0, n in ((plo, slo, rlo, nlo), (phi, shi, rhi, nhi)):
            if peer < 0:
                continue
            send = torch.from_numpy(np.concatenate([x[s0 * d:(s0 + n) * d] for x in st]))
            recv = torch.empty_like(send)
            reqs += [dist.isend(send, peer), dist.irecv(recv, peer)]
            bufs.append((r0, n, recv))
        for q in reqs:
            q.wait()
        for r0, n, recv in bufs:
            v = recv.numpy().reshape(3, n * d)
            for x, part in zip(st, v):
                x[r0 * d:(r0 + n) * d] = part
        o.set_state(*st)
    u, v, a = o.state()
    n0, n1 = slab.own_nodes
    mu = o.mu()
    e0, e1 = slab.own_elems
    own_pairs = (pairs[:, 0] >= e0) & (pairs[:, 0] < e1)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), u=u[n0 * d:n1 * d], v=v[n0 * d:n1 * d],
             a=a[n0 * d:n1 * d], gnode=np.array(slab.global_nodes(n0, n1)),
             pairs=pairs[own_pairs] + slab.elem_first, mu=mu[own_pairs])
    dist.destroy_process_group()


@pytest.mark.parametrize("name,steps,spread", [("mini", 80, False), ("mini", 80, True)])
def test_two_rank_slabs_equal_single_domain(tmp_path, name, steps, spread):
    import torch.multiprocessing as mp

    from oracle import pyoracle as po
    from paper_2403_03605_b200.pd import Scenario

    port = _free_port()
    mp.spawn(_worker, args=(2, port, name, steps, spread, str(tmp_path)), nprocs=2, join=True)
    sc = Scenario(_scenario(name, spread))
    la = dict(nodes=sc.nodes, conn=sc.conn, centroid=sc.centroid, volume=sc.volume,
              mass=sc.mass, p_ext=sc.p_ext, bc_dofs=sc.bc_dofs, bc_vel=sc.bc_vel)
    pairs = po.find_pairs(sc.dim, sc.centroid, sc.volume, sc.delta, sc.notches())
    o = po.OraclePD(_sysd(sc, la, pairs), po.MF)
    o.init(sc.load_scale(0.0))
    o.step([sc.load_scale(i * sc.dt) for i in range(1, steps + 1)])
    u, v, a = o.state()
    mu = o.mu()
    idx = {(int(i), int(j)): q for q, (i, j) in enumerate(pairs)}
    d = sc.dim
    covered = 0
    n_broken = 0
    for r in range(2):
        z = np.load(tmp_path / f"r{r}.npz")
        g0, g1 = z["gnode"]
        assert np.array_equal(z["u"], u[g0 * d:g1 * d])
        assert np.array_equal(z["v"], v[g0 * d:g1 * d])
        assert np.array_equal(z["a"], a[g0 * d:g1 * d])
        for (i, j), m in zip(z["pairs"], z["mu"]):
            assert mu[idx[(int(i), int(j))]] == m
        covered += g1 - g0
        n_broken += int((z["mu"] == 0).sum())
    assert covered == sc.n_nodes
    assert n_broken == int((mu == 0).sum()) and n_broken > 0
