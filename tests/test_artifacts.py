"""Run artifacts in the reference's format.

CPU: the mesh hash equals the reference's for the same mesh (the value
`compare` uses to refuse mismatched runs), and the writers produce files the
reference's readers accept (compared by the reference's own `compare` against
themselves).  GPU: device runs (pure PD and coupled MTS) scored against the
reference's own runs by the reference's `compare` -- tracked-point global error
and damage agreement of every frame."""
import json
import os
import subprocess
import tempfile

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2403_03605_b200 import artifacts as A
from paper_2403_03605_b200 import capi
from paper_2403_03605_b200 import configs as cf
from paper_2403_03605_b200.pd import Scenario

REF_ART = os.path.join(os.path.dirname(po.REF_DRIVER), "ref_artifacts")
need_ref = pytest.mark.skipif(not os.path.exists(REF_ART), reason="oracle/_ref not built")


def _pd_cfg():
    c = cf.get("mini")
    c["output"].update(interval=1e-6, tracked1=[0.02, 0.008], tracked2=[0.039, 0.015])
    return c


def _mts_cfg():
    c = cf.get("mts_mini_frac")
    c["output"].update(interval=6e-7, tracked1=[0.015, 0.005], tracked2=[0.029, 0.009])
    return c


def _ref(*args):
    r = subprocess.run([REF_ART, *args], check=True, capture_output=True, text=True)
    return json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])


@need_ref
def test_mesh_hash_matches_reference():
    with tempfile.TemporaryDirectory() as tmp:
        cfgp = os.path.join(tmp, "s.cfg")
        with open(cfgp, "w") as f:
            f.write(cf.render_cfg(_pd_cfg()))
        _ref("run", cfgp, os.path.join(tmp, "ref"))
        meta = open(os.path.join(tmp, "ref", "meta.txt")).read()
    sc = Scenario(_pd_cfg())
    assert f"mesh_hash = {A.mesh_hash(sc.dim, sc.nodes, sc.conn)}\n" in meta


@need_ref
def test_writers_read_back_by_reference():
    sc = Scenario(_pd_cfg())
    with tempfile.TemporaryDirectory() as tmp:
        d = os.path.join(tmp, "a")
        os.makedirs(d)
        n = sc.n_nodes
        rng = np.random.default_rng(0)
        A.write_vtk(os.path.join(d, "frame_00000.vtk"), 2, sc.nodes, sc.conn,
                    rng.normal(size=2 * n), rng.normal(size=2 * n), rng.random(n),
                    rng.random(sc.n_elems), np.ones(sc.n_elems), np.zeros(sc.n_elems))
        A.write_csv(["frame", "t"], [[0.0, 0.0]], os.path.join(d, "frames.csv"))
        A.write_csv(["t", "p0_ux", "p0_uy"], [[0.0, 1.0, 2.0], [1e-6, 1.5, 2.5]],
                    os.path.join(d, "tracked.csv"))
        A.write_csv(["step", "t_k", "t_u", "t_lambda", "t_y", "broken", "continuity"],
                    [[0.0, 1e-3, 0, 0, 0, 0, 0]], os.path.join(d, "timing.csv"))
        A.write_meta(os.path.join(d, "meta.txt"), A.mesh_hash(2, sc.nodes, sc.conn), 2, n,
                     sc.n_elems, 1, "pure_pd", 5e-8, 1, 4e-6, 1e-6)
        rep = _ref("compare", d, d)
    assert rep["tracked_error_pct"] == [0] and rep["has_damage_frames"]
    assert rep["min_damage_agreement"] == 1


@pytest.mark.gpu
@need_ref
@pytest.mark.parametrize("kind", ["pure_pd", "coupled"])
def test_device_artifacts_scored_by_reference_compare(kind):
    cfg = _pd_cfg() if kind == "pure_pd" else _mts_cfg()
    with tempfile.TemporaryDirectory() as tmp:
        cfgp = os.path.join(tmp, "s.cfg")
        with open(cfgp, "w") as f:
            f.write(cf.render_cfg(cfg))
        ref = _ref("run", cfgp, os.path.join(tmp, "ref"))
        dev_dir = os.path.join(tmp, "dev")
        if kind == "pure_pd":
            mine = A.run_pure_pd(cfg, dev_dir, mode=capi.DETERMINISTIC)
        else:
            mine = A.run_coupled(cfg, dev_dir)
        assert (mine["steps"], mine["broken"], mine["frames"]) == (ref["steps"], ref["broken"],
                                                                   ref["frames"])
        rep = _ref("compare", dev_dir, os.path.join(tmp, "ref"))
    assert rep["has_damage_frames"] and rep["frames_compared"] == ref["frames"]
    assert rep["min_damage_agreement"] == 1.0
    assert max(rep["tracked_error_pct"]) <= 1e-8  # percent
