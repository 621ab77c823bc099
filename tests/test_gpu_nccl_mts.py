"""Sharded coupled MTS over NCCL with real peers: one process per GPU,
shard r on GPU r, the ghost exchange as ncclSend/ncclRecv, the owner-sums as
ncclAllReduce and shard 0's FE results as ncclBroadcast, all on the handle's stream.
The states, multipliers, reports and bond states must equal the single-domain run bit
for bit.  Needs >= 2 GPUs (skipped on the one-GPU boxes of this build; the in-process
group of tests/test_gpu_mts_shards.py runs the same step code on one GPU)."""
import copy
import os

import numpy as np
import pytest

from test_gpu_nccl_slabs import ROOT, _n_gpus, _port

pytestmark = pytest.mark.gpu
FIELDS = ("newly_broken", "interface_iterations", "continuity", "lambda_fe", "lambda_pd")


def _cfg(name):
    from paper_2403_03605_b200 import configs as cf

    c = copy.deepcopy(cf.get(name))
    c["run"]["interface"] = "matrix_free"
    return c


def _worker(rank, world, port, name, steps, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from paper_2403_03605_b200.mts import MtsSolver
    from paper_2403_03605_b200.pd import PDSolver

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    s = MtsSolver(_cfg(name), device=rank, shard=(rank, world))
    uid = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        uid[:] = torch.frombuffer(bytearray(PDSolver.nccl_unique_id()), dtype=torch.uint8)
    dist.broadcast(uid, 0)
    s.comm_init(bytes(uid.tolist()))
    s.initialize()
    reps = s.macro_step(steps)
    own = np.repeat(s.shard["node_owned"], s.dim)
    u, v, a = s.state("pd")
    fe = s.state("fe") if rank == 0 else (np.zeros(0),) * 3
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), dofs=s.pd_local_dofs[own], u=u[own],
             v=v[own], a=a[own], fu=fe[0], fv=fe[1], fa=fe[2], lam=s.lam(),
             reps=np.array([[r[f] for f in FIELDS] for r in reps], dtype=np.float64))
    del s
    dist.destroy_process_group()


@pytest.mark.skipif(_n_gpus() < 2, reason="needs >= 2 GPUs (NCCL peers)")
@pytest.mark.parametrize("name,steps", [("mts_mini_frac", 60), ("cfg2_0p5", 200)])
def test_nccl_mts_shards_bitwise(tmp_path, name, steps):
    import torch.multiprocessing as mp

    from paper_2403_03605_b200.mts import MtsSolver

    world = 2
    mp.spawn(_worker, args=(world, _port(), name, steps, str(tmp_path)), nprocs=world, join=True)
    one = MtsSolver(_cfg(name))
    one.initialize()
    reps = one.macro_step(steps)
    ref = np.array([[r[f] for f in FIELDS] for r in reps], dtype=np.float64)
    u, v, a = one.state("pd")
    covered = 0
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        d = z["dofs"]
        assert np.array_equal(z["u"], u[d]) and np.array_equal(z["v"], v[d])
        assert np.array_equal(z["a"], a[d])
        assert np.array_equal(z["lam"], one.lam())
        assert np.array_equal(z["reps"][:, :2], ref[:, :2])  # broken counts, CG iterations
        if r == 0:
            assert np.array_equal(z["reps"], ref)
            for x, y in zip((z["fu"], z["fv"], z["fa"]), one.state("fe")):
                assert np.array_equal(x, y)
        covered += len(d)
    assert covered == one.pd_n_dof
