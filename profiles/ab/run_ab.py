"""A/B timing of libpmts.so variants on one workload (one subprocess per library).

    python profiles/ab/run_ab.py [--workload cfg3] [--mode fast] [--steps 1000] [--warmup 20]
        [--reps 3] name=path/to/libpmts_x.so ...

Each variant: a fresh handle stepped through the warm-up, `reps` timed windows of `steps`
steps (CUDA events on the handle's stream), the best and all windows, and a hash of the
final state + broken-bond set so variants can be compared bit for bit.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def child(args):
    sys.path.insert(0, ROOT)
    import numpy as np

    from paper_2403_03605_b200 import capi
    from paper_2403_03605_b200 import configs as cf
    from paper_2403_03605_b200.pd import PDSolver, Scenario

    mode = {"fast": capi.FAST, "det": capi.DETERMINISTIC, "f32pos": capi.FAST_F32POS}[args.mode]
    sc = Scenario(cf.get(args.workload))
    s = PDSolver.from_scenario(sc, mode=mode, device=0).find_pe_pairs()
    v0 = sc.initial_velocity()
    if v0.any():
        z = np.zeros(s.n_dof)
        s.set_state(z, v0, z)
    for o in args.opt:
        k, v = o.split("=")
        s.set_option(int(k), int(v))
    s.initial_acceleration(sc.load_scale(0.0))
    s.step(sc.scales(1, args.warmup))
    step0 = args.warmup + 1
    times = []
    for r in range(args.reps):
        ms = s.step_timed(sc.scales(step0, args.steps))
        step0 += args.steps
        times.append(ms / args.steps * 1e3)
    u, v, a = s.state()
    intact = s.intact()
    h = hashlib.sha256()
    for x in (u, v, a, intact):
        h.update(np.ascontiguousarray(x).tobytes())
    print(json.dumps({"us_per_step": times, "first_window_us": times[0],
                      "broken": int((intact == 0).sum()), "sha": h.hexdigest()[:16],
                      "bonds": s.info()["n_bonds"]}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg3")
    ap.add_argument("--mode", default="fast")
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--opt", action="append", default=[], help="pmts_pd_set_option ID=VALUE")
    ap.add_argument("variants", nargs="*")
    args = ap.parse_args()
    if args.child:
        return child(args)
    for v in args.variants:
        name, path = v.split("=", 1)
        env = dict(os.environ, PMTS_LIB_PATH=os.path.abspath(path))
        cmd = [sys.executable, os.path.abspath(__file__), "--child", "--workload", args.workload,
               "--mode", args.mode, "--steps", str(args.steps), "--warmup", str(args.warmup),
               "--reps", str(args.reps)] + [x for o in args.opt for x in ("--opt", o)]
        p = subprocess.run(cmd, env=env, capture_output=True, text=True)
        line = p.stdout.strip().splitlines()[-1] if p.stdout.strip() else p.stderr[-400:]
        print(name, line, flush=True)


if __name__ == "__main__":
    main()
