"""The reference-side drop-in, compiled and run: integration/b200_run
is the reference's own run_built pure-PD branch (driver_run.hpp:160-246) with the
fine step on the B200 through include/pmts_capi.h, built against the unmodified
reference headers.  Its artifacts are scored against the reference's own run by the
reference's compare_runs (driver.hpp:290-368): tracked-point error and the damage
agreement of every frame."""
import json
import os
import subprocess
import tempfile

import pytest

from conftest import ROOT
from oracle import pyoracle as po
from paper_2403_03605_b200 import configs as cf

SHIM = os.path.join(ROOT, "integration", "_build", "b200_run")
REF_ART = os.path.join(os.path.dirname(po.REF_DRIVER), "ref_artifacts")
need = pytest.mark.skipif(not (os.path.exists(SHIM) and os.path.exists(REF_ART)),
                          reason="integration/_build or oracle/_ref not built")


def _json(cmd):
    r = subprocess.run(cmd, check=True, capture_output=True, text=True)
    return json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])


def _cfg(name):
    c = cf.get(name)
    if name == "mts_mini_frac":
        c["output"].update(interval=6e-7, tracked1=[0.015, 0.005], tracked2=[0.029, 0.009])
        return c
    if name == "mts_bar3d":
        c["output"].update(interval=2e-7, tracked1=[0.006, 0.002, 0.002],
                           tracked2=[0.0115, 0.002, 0.002])
        return c
    if name == "mini":
        c["output"].update(interval=1e-6, tracked1=[0.02, 0.008], tracked2=[0.039, 0.015])
    else:  # the BASELINE cfg1 analog: 1000 steps, frames every 250
        c["output"].update(interval=6.25e-6, tracked1=[0.05, 0.02], tracked2=[0.099, 0.039])
    return c


@need
def test_shim_links_the_library():
    out = subprocess.run(["ldd", SHIM], capture_output=True, text=True).stdout
    assert "libpmts.so" in out


@pytest.mark.gpu
@need
@pytest.mark.parametrize("name,mode,fam", [("mini", "det", False), ("mini", "fast", True),
                                           ("cfg1", "det", False), ("cfg1", "fast", True)])
def test_shim_run_scored_by_reference_compare(name, mode, fam):
    with tempfile.TemporaryDirectory() as tmp:
        cfgp = os.path.join(tmp, "s.cfg")
        with open(cfgp, "w") as f:
            f.write(cf.render_cfg(_cfg(name)))
        ref = _json([REF_ART, "run", cfgp, os.path.join(tmp, "ref")])
        cmd = [SHIM, cfgp, os.path.join(tmp, "dev"), "--mode", mode]
        if fam:
            cmd.append("--device-families")
        mine = _json(cmd)
        assert mine["steps"] == ref["steps"] and mine["frames"] == ref["frames"]
        rep = _json([REF_ART, "compare", os.path.join(tmp, "dev"), os.path.join(tmp, "ref")])
    print(f"[shim {name} {mode}] broken {mine['broken']} vs ref {ref['broken']}; compare {rep}")
    assert rep["has_damage_frames"] and rep["frames_compared"] == ref["frames"]
    if mode == "det":  # bit-exact broken set: every frame's damage agrees exactly
        assert mine["broken"] == ref["broken"]
        assert rep["min_damage_agreement"] == 1.0
        assert max(rep["tracked_error_pct"]) <= 1e-8
    else:  # fast mode: north-star tolerances
        assert abs(mine["broken"] - ref["broken"]) <= 1e-3 * max(ref["broken"], 1)
        assert rep["min_damage_agreement"] >= 0.999
        assert max(rep["tracked_error_pct"]) <= 1e-4


@pytest.mark.gpu
@need
@pytest.mark.parametrize("name", ["mts_mini_frac", "mts_bar3d"])
def test_shim_coupled_run_scored_by_reference_compare(name):
    """run_built's coupled branch with the CoupledIntegrator on the device: scored by the
    reference's compare_runs against the reference's own coupled run."""
    with tempfile.TemporaryDirectory() as tmp:
        cfgp = os.path.join(tmp, "s.cfg")
        with open(cfgp, "w") as f:
            f.write(cf.render_cfg(_cfg(name)))
        ref = _json([REF_ART, "run", cfgp, os.path.join(tmp, "ref")])
        mine = _json([SHIM, cfgp, os.path.join(tmp, "dev")])
        assert (mine["steps"], mine["frames"]) == (ref["steps"], ref["frames"])
        rep = _json([REF_ART, "compare", os.path.join(tmp, "dev"), os.path.join(tmp, "ref")])
    print(f"[shim {name}] broken {mine['broken']} vs ref {ref['broken']}; compare {rep}")
    assert mine["broken"] == ref["broken"]
    assert rep["has_damage_frames"] and rep["frames_compared"] == ref["frames"]
    assert rep["min_damage_agreement"] == 1.0
    assert max(rep["tracked_error_pct"]) <= 1e-6  # percent
