"""The shard plan of a sharded coupled run, on the CPU: host-only handles
(device = -1) of every shard expose their plan (pmts_mts_shard_view), which must
  * partition the PD-active nodes (ownership) and elements (owned ranges) exactly once,
  * hold, for every element incident to an owned node, that element's whole horizon
    family (partners within delta, brute force here) -- the exactness argument of the
    ghost exchange,
  * draw every ghost node from a neighbouring shard, with matching send / receive
    lists on both sides (same nodes, same order)."""
import copy

import numpy as np
import pytest

from paper_2403_03605_b200 import configs as cf
from paper_2403_03605_b200.capi import ConfigError
from paper_2403_03605_b200.mts import MtsSolver


def _cfg(name):
    c = copy.deepcopy(cf.get(name))
    c["run"]["interface"] = "matrix_free"
    return c


def _plans(name, world):
    return [MtsSolver(_cfg(name), device=-1, shard=(r, world)) for r in range(world)]


@pytest.mark.parametrize("name,world", [("mts_mini_frac", 2), ("mts_mini_frac", 3),
                                        ("cfg2_0p5", 2), ("cfg2_0p5", 4), ("cfg2_0p5", 8)])
def test_shard_plan_partition_and_closure(name, world):
    hs = _plans(name, world)
    sy = hs[0].system()
    pd_active = np.flatnonzero(sy["labels"] != 0)
    assert len(pd_active) == hs[0].view.n_pd_elems
    pd_nodes = np.unique(sy["elem_nodes"][pd_active])
    xyz, conn = sy["node_xyz"], sy["elem_nodes"]
    cen = xyz[conn].mean(axis=1)
    delta = sy["delta"]
    owner = {}
    own_elems = []
    for r, h in enumerate(hs):
        sh = h.shard
        assert sh["world"] == world and sh["rank"] == r
        ln = pd_nodes[sh["local_nodes"]]  # compact PD node -> global node
        for g in ln[sh["node_owned"]]:
            assert g not in owner
            owner[int(g)] = r
        lo, hi = sh["own_elems"]
        own_elems += list(pd_active[sh["local_elems"][lo:hi]])
    assert sorted(owner) == sorted(int(g) for g in pd_nodes)
    assert sorted(own_elems) == sorted(pd_active)
    for r, h in enumerate(hs):
        sh = h.shard
        le = set(int(e) for e in pd_active[sh["local_elems"]])
        ln = pd_nodes[sh["local_nodes"]]
        for g, o in zip(ln, sh["node_owned"]):
            if not o:
                assert abs(owner[int(g)] - r) == 1  # ghosts from the neighbours only
        owned = set(int(g) for g in ln[sh["node_owned"]])
        inc = [e for e in pd_active if owned.intersection(int(n) for n in conn[e])]
        for e in inc:
            assert int(e) in le
            d = np.linalg.norm(cen[pd_active] - cen[e], axis=1)
            for p in pd_active[d <= delta * (1 + 1e-9)]:
                assert int(p) in le, (r, int(e), int(p))


def test_shard_plan_redundancy_cfg2():
    """Local PD elements over owned ones (the ghost layers' redundant work) on the cfg2
    analog at 0.25 mm: <= 1.1 at 2 shards, <= 1.3 at 4 (80 element layers along y)."""
    for world, bound in ((2, 1.1), (4, 1.3)):
        hs = _plans("cfg2", world)
        loc = sum(len(h.shard["local_elems"]) for h in hs)
        assert loc / hs[0].view.n_pd_elems <= bound


def test_too_many_shards():
    with pytest.raises(ConfigError, match="layers per shard"):
        _plans("mts_mini_frac", 4)


def test_sharded_runs_need_the_matrix_free_interface():
    c = copy.deepcopy(cf.get("mts_mini_frac"))  # n_lambda <= 400: the dense interface
    with pytest.raises(ConfigError, match="matrix-free interface"):
        MtsSolver(c, device=-1, shard=(0, 2))
