"""bench.py's launcher on CPU: --gpus N without torchrun's environment re-launches the
command under torch.distributed.run (one rank per GPU, 127.0.0.1 rendezvous); the
reference arm runs on rank 0 only and prints exactly one JSON line."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT
from oracle import pyoracle as po


@pytest.mark.skipif(not os.path.exists(po.REF_DRIVER), reason="oracle/_ref not built")
def test_gpus_two_spawns_ranks_reference_arm():
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl",
                        "reference", "--ref-workload", "cfg3_sample", "--steps", "1",
                        "--warmup", "3"], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    assert j["impl"] == "reference" and j["n_gpus"] == 2 and j["value"] > 0
    assert j["e2e"]["h2d_bytes_per_step"] == 0


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--steps", "1"], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode != 0 and "WORLD_SIZE 3" in (r.stderr + r.stdout)
