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
        sc["ext"] = dict(sc["ext"], s_crit_spread=0.05, seed=99)
    return sc


def _sysd(sc, la, pairs, slab=None):
    ext = sc.cfg.get("ext", {})
    d = dict(dim=sc.dim, n_nodes=len(la["nodes"]), conn=la["conn"], centroid=la["centroid"],
             volume=la["volume"], pairs=pairs, mass=la["mass"], p_ext=la["p_ext"],
             bc_dofs=la["bc_dofs"], bc_vel=la["bc_vel"], delta=sc.delta, l=sc.l, c0=sc.c0,
             s_crit=sc.s_crit, dt=sc.dt, gamma=sc.gamma, beta=sc.beta,
             global_id_offset=slab.elem_first if slab else 0,
             slab_plane=slab.plane if slab else (0, 0))
    if ext.get("micromodulus") == "constant":
        d.update(micromodulus=1, c_const=ext["c"], h=ext.get("h", 1.0))
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
    v0 = sc.initial_velocity()
    if v0.any():
        z = np.zeros(len(la["dofs"]))
        o.set_state(z, v0[la["dofs"]], z)
    o.init(sc.load_scale(0.0))
    d = sc.dim
    halo = slab.halo_nodes()  # (peer, send ids, recv ids), z layers expanded

    def dofs(ids):
        return (ids[:, None] * d + np.arange(d)).ravel()

    for i in range(1, steps + 1):
        o.step([sc.load_scale(i * sc.dt)])
        st = list(o.state())
        reqs, bufs = [], []
        for peer, snd, rcv in halo:
            send = torch.from_numpy(np.concatenate([x[dofs(snd)] for x in st]))
            recv = torch.empty_like(send)
            reqs += [dist.isend(send, peer), dist.irecv(recv, peer)]
            bufs.append((rcv, recv))
        for q in reqs:
            q.wait()
        for rcv, recv in bufs:
            v = recv.numpy().reshape(3, -1)
            for x, part in zip(st, v):
                x[dofs(rcv)] = part
        o.set_state(*st)
    u, v, a = o.state()
    own = slab.owned_nodes()
    mu = o.mu()
    own_pairs = slab.owns_elem(pairs[:, 0])
    gp = np.stack([slab.elem_global(pairs[own_pairs, 0]), slab.elem_global(pairs[own_pairs, 1])], 1)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), u=u[dofs(own)], v=v[dofs(own)],
             a=a[dofs(own)], gnode=slab.node_global(own), pairs=gp, mu=mu[own_pairs])
    dist.destroy_process_group()


@pytest.mark.parametrize("name,steps,spread", [("mini", 80, False), ("mini", 80, True),
                                               ("cfg4_small", 40, True),
                                               ("block3d", 100, True)])
def test_two_rank_slabs_equal_single_domain(tmp_path, name, steps, spread):
    """2D x-slabs and 3D z-x slabs (cut along y: strided halos, layer-mapped global
    ids for the per-bond hash) over gloo: owned fields and bond states bitwise."""
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
    v0 = sc.initial_velocity()
    if v0.any():
        z = np.zeros(sc.n_dof)
        o.set_state(z, v0, z)
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
        g = (z["gnode"][:, None] * d + np.arange(d)).ravel()
        assert np.array_equal(z["u"], u[g])
        assert np.array_equal(z["v"], v[g])
        assert np.array_equal(z["a"], a[g])
        for (i, j), m in zip(z["pairs"], z["mu"]):
            assert mu[idx[(int(i), int(j))]] == m
        covered += len(z["gnode"])
        n_broken += int((z["mu"] == 0).sum())
    assert covered == sc.n_nodes
    assert n_broken == int((mu == 0).sum())
    if name != "cfg4_small":
        assert n_broken > 0


def test_slab_partition_3d_is_zx():
    """3D blocks are cut along y (z-x slabs): every rank owns all x and z of its y
    rows; owned nodes partition the mesh; global ids round-trip."""
    from paper_2403_03605_b200 import slabs

    lat = (20, 24, 10)
    seen = np.zeros(21 * 25 * 11, dtype=int)
    for r in range(3):
        s = slabs.make_slab(lat, 3, r, 3)
        assert s.lattice[0] == 20 and s.lattice[2] == 10 and s.layers == 11
        seen[s.node_global(s.owned_nodes())] += 1
        ge = s.local_elems_global()
        assert len(np.unique(ge)) == s.n_elems
        # local order is the global order (gathers run in the single-domain order)
        assert np.all(np.diff(ge) > 0)
        assert np.all(np.diff(s.local_nodes_global()) > 0)
    assert (seen == 1).all()


def test_slab_redundancy_at_8_ranks():
    """per-rank bond work <= 1.1x its owned rows at 8 ranks on the two
    largest PD configurations (cfg4 200x200x50, cfg5 core 400x800x40)."""
    from paper_2403_03605_b200 import slabs

    for lat in ((200, 200, 50), (400, 800, 40)):
        r = slabs.redundancy(lat, 3, 8)
        assert r["bond"] <= 1.1, (lat, r)
