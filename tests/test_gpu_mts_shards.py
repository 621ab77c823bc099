"""Sharded coupled MTS (north star item 5): the PD region cut into slabs
of element layers, one-horizon ghost layers exchanged every fine substep, shard 0
holding the FE side, the interface solve replicated on every shard.  Here the shards
run as one in-process group on one GPU (one host thread per shard, device copies at
host barriers -- no kernel ever waits on another shard); the multi-process NCCL
transport runs the same step code (tests/test_gpu_nccl_mts.py, >= 2 GPUs).

The bar is BITWISE equality with the single-domain integrator on the same config:
every report field the step computes, the multipliers, FE and PD states, every bond's
state and the damage field -- through crack growth, with the interface on the
precomputed H_PD and, after bonds break, on the distributed recursion."""
import copy

import numpy as np
import pytest

from paper_2403_03605_b200 import configs as cf
from paper_2403_03605_b200.mts import MtsSolver, ShardGroup

pytestmark = pytest.mark.gpu

FIELDS = ("newly_broken", "interface_iterations", "continuity", "quad_fe", "quad_pd",
          "lambda_fe", "lambda_pd")


def _cfg(name, h_pd="precompute"):
    c = copy.deepcopy(cf.get(name))
    c["run"]["interface"] = "matrix_free"
    c["run"]["interface_h_pd"] = h_pd
    return c


def _single_pairs(s):
    return {(int(i), int(j)): int(v) for (i, j), v in zip(s.system()["pairs"], s.intact())}


def _assert_same(one, grp, reps1, repsg):
    for a, b in zip(reps1, repsg):
        for f in FIELDS:
            assert a[f] == b[f], (f, a[f], b[f])
    assert np.array_equal(one.lam(), grp.lam())
    for w in ("fe", "pd"):
        for x, y in zip(one.state(w), grp.state(w)):
            assert np.array_equal(x, y), w
    assert _single_pairs(one) == grp.pairs_intact()
    e1, n1 = one.damage_field()
    eg, ng = grp.damage_field()
    assert np.array_equal(e1, eg) and np.array_equal(n1, ng)


@pytest.mark.parametrize("name,steps", [("mts_mini_frac", 60), ("mts_mini_mfree", 20),
                                        ("mts_bar3d_tall", 40)])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("h_pd", ["precompute", "recursion"])
def test_shards_bitwise_single_domain(name, steps, world, h_pd):
    if name == "mts_bar3d_tall" and world > 2:
        pytest.skip("8 element layers along z: at most 2 shards (D + 1 = 3 layers each)")
    c = _cfg(name, h_pd)
    one = MtsSolver(c)
    one.initialize()
    grp = ShardGroup(c, world)
    grp.initialize()
    for x, y in zip(one.state("pd"), grp.state("pd")):
        assert np.array_equal(x, y)
    r1, rg = [], []
    for k in (steps // 2, steps - steps // 2):
        r1 += one.macro_step(k)
        rg += grp.macro_step(k)
        _assert_same(one, grp, r1, rg)
    if name in ("mts_mini_frac", "mts_bar3d_tall"):
        assert sum(r["newly_broken"] for r in r1) > 0  # bond breaking covered


@pytest.mark.parametrize("world", [2, 4])
def test_shards_cfg2_analog_full_run(world):
    """BASELINE cfg2's conforming analog (0.5 mm twin: 100 x 40 mm plate, PD band
    100 x 20 mm, implicit FE, m = 10), its whole 200-macro-step run through crack
    growth, 2 and 4 shards: bitwise the single domain."""
    c = _cfg("cfg2_0p5")
    one = MtsSolver(c)
    one.initialize()
    grp = ShardGroup(c, world)
    grp.initialize()
    r1, rg = [], []
    for k in (100, 100):
        r1 += one.macro_step(k)
        rg += grp.macro_step(k)
        _assert_same(one, grp, r1, rg)
    assert sum(r["newly_broken"] for r in r1) > 0


def test_shards_cfg2_at_size_window():
    """BASELINE cfg2's analog at its own 0.25 mm (64,962 PD dofs, 14,436 multipliers),
    2 shards, 10 macro steps: bitwise the single domain."""
    c = _cfg("cfg2")
    one = MtsSolver(c)
    one.initialize()
    grp = ShardGroup(c, 2)
    grp.initialize()
    _assert_same(one, grp, one.macro_step(10), grp.macro_step(10))


def test_too_many_shards_is_a_config_error():
    from paper_2403_03605_b200.capi import ConfigError
    with pytest.raises(ConfigError, match="layers per shard"):
        ShardGroup(_cfg("mts_mini_frac"), 4)
