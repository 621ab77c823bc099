"""Slab decomposition over NCCL with real peers: one process per GPU, the halo
exchange is ncclSend/ncclRecv inside pmts_pd_step (2D x-slabs: contiguous rows;
3D z-x slabs: one range per z node layer, packed by the library).  Owned fields
and bond states must equal the single-domain run bit for bit.  Needs >= 2 GPUs
(skipped on the one-GPU boxes of this build; the host-mediated emulation in
test_gpu_slabs.py and the gloo test cover the same partition on one GPU / CPU)."""
import os
import socket

import numpy as np
import pytest

from conftest import gpu_available

pytestmark = pytest.mark.gpu
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _n_gpus():
    if not gpu_available():
        return 0
    import ctypes

    from paper_2403_03605_b200 import capi

    n = ctypes.c_int()
    capi.lib().pmts_device_count(ctypes.byref(n))
    return n.value


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, mode, steps, split, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from paper_2403_03605_b200 import capi
    from paper_2403_03605_b200 import configs as cf
    from paper_2403_03605_b200 import slabs
    from paper_2403_03605_b200.pd import PDSolver, Scenario

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    sc = Scenario(cf.get(name))
    slab = slabs.make_slab(sc.lattice, sc.dim, rank, world)
    h = slabs.solver_for_slab(sc, slab, mode, device=rank).find_pe_pairs()
    uid = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        uid[:] = torch.frombuffer(bytearray(PDSolver.nccl_unique_id()), dtype=torch.uint8)
    dist.broadcast(uid, 0)
    slabs.attach_nccl(h, bytes(uid.tolist()))
    if split:  # edge tile rows first, the NCCL halo on a second stream under the interior
        h.set_option(capi.OPT_HALO_OVERLAP, 1)
    v0 = sc.initial_velocity()
    if v0.any():
        z = np.zeros(h.n_dof)
        h.set_state(z, v0[h.local_dofs], z)
    h.initial_acceleration(sc.load_scale(0.0))
    # the initial halo: every rank computed its halo rows itself (same arithmetic)
    nb = h.step(sc.scales(1, steps))
    t = torch.tensor([nb], dtype=torch.int64)
    dist.all_reduce(t)
    own = slab.owned_nodes()
    d = sc.dim
    loc = (own[:, None] * d + np.arange(d)).ravel()
    u, v, a = h.state()
    lp, li = h.pairs(), h.intact()
    m = slab.owns_elem(lp[:, 0])
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), g=slab.node_global(own), u=u[loc], v=v[loc],
             a=a[loc], pi=slab.elem_global(lp[m, 0]), pj=slab.elem_global(lp[m, 1]),
             mu=li[m], nb=int(t.item()))
    del h
    dist.destroy_process_group()


@pytest.mark.skipif(_n_gpus() < 2, reason="needs >= 2 GPUs (NCCL peers)")
@pytest.mark.parametrize("name,steps,split", [("cfg1", 120, False), ("cfg1", 120, True),
                                              ("cfg5_core_small", 120, False)])
@pytest.mark.parametrize("mode", [0, 1])
def test_nccl_slabs_bitwise(tmp_path, name, steps, split, mode):
    import torch.multiprocessing as mp

    from paper_2403_03605_b200 import configs as cf
    from paper_2403_03605_b200.pd import PDSolver, Scenario

    world = 2
    mp.spawn(_worker, args=(world, _port(), name, mode, steps, split, str(tmp_path)),
             nprocs=world, join=True)
    sc = Scenario(cf.get(name))
    one = PDSolver.from_scenario(sc, mode=mode).find_pe_pairs()
    one.initial_acceleration(sc.load_scale(0.0))
    nb1 = one.step(sc.scales(1, steps))
    u, v, a = one.state()
    idx = {(int(i), int(j)): q for q, (i, j) in enumerate(one.pairs())}
    intact = one.intact()
    d = sc.dim
    covered = 0
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        g = (z["g"][:, None] * d + np.arange(d)).ravel()
        assert np.array_equal(z["u"], u[g]) and np.array_equal(z["v"], v[g])
        assert np.array_equal(z["a"], a[g])
        q = np.array([idx[(int(i), int(j))] for i, j in zip(z["pi"], z["pj"])])
        assert np.array_equal(z["mu"], intact[q])
        assert int(z["nb"]) == nb1
        covered += len(z["g"])
    assert covered == sc.n_nodes and nb1 > 0


@pytest.mark.parametrize("name", ["cfg4_small", "mini"])
def test_halo_nccl_loopback_one_gpu(name):
    """The NCCL halo path on one GPU: a handle in a clique of one whose lower and upper
    'neighbour' is itself.  exchange_halo runs ncclSend/ncclRecv to self in one group
    (the k-th send to a peer meets the k-th receive from it) -- in 3D around the pack /
    unpack kernels of the strided ranges (one 4-row range per z node layer), in 2D on
    the contiguous rows: afterwards each receive range holds the matching send range's
    predictor displacement, every other row is untouched."""
    if not gpu_available():
        pytest.skip("needs a GPU")
    from paper_2403_03605_b200 import configs as cf
    from paper_2403_03605_b200 import slabs
    from paper_2403_03605_b200.pd import PDSolver, Scenario

    sc = Scenario(cf.get(name))
    d = sc.dim
    slab = slabs.make_slab(sc.lattice, d, 0, 1)
    h = slabs.solver_for_slab(sc, slab, 1).find_pe_pairs()
    h.comm_init(PDSolver.nccl_unique_id(), 1, 0)
    nx, ny = sc.lattice[0], sc.lattice[1]
    layers = sc.lattice[2] + 1 if d == 3 else 1
    NX, NYL = nx + 1, ny + 1
    n = 4 * NX  # 4 node rows of one layer
    send_lo, recv_lo, send_hi, recv_hi = 0, 4 * NX, 8 * NX, 12 * NX
    h.set_halo(0, send_lo, recv_lo, n, 0, send_hi, recv_hi, n)
    if layers > 1:
        h.set_halo_layers(layers, NX * NYL)
    rng = np.random.default_rng(7)
    u = rng.normal(size=h.n_dof)
    z = np.zeros(h.n_dof)
    h.set_state(u, z, z)  # predictor = u exactly (v = a = 0), then the exchange
    rd = h.get_rows(0, NX * NYL, layers, NX * NYL).reshape(layers, NYL, NX, d)
    u4 = u.reshape(layers, NYL, NX, d)
    exp = u4.copy()
    exp[:, 4:8] = u4[:, 0:4]     # recv_lo <- send_lo (loopback: first send meets first receive)
    exp[:, 12:16] = u4[:, 8:12]  # recv_hi <- send_hi
    assert np.array_equal(rd, exp)
