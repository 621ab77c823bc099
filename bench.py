#!/usr/bin/env python
"""Benchmark of the PD fine-step hot path (BASELINE.json metric: PD bond-updates/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]

A "step" is one PD fine step (bond gather + break test + velocity-Verlet node
update) over the whole BASELINE cfg3 plate (2000 x 800 elements, 22,331,624
bonds, per-bond s0 factor, constant micromodulus), synthetic geometry with
the config's shapes.  value = unique bonds x K / device time of K steps
(CUDA events on the handle's stream), max over ranks.  e2e = the same metric
through the public C-ABI with host buffers: initial state H2D from pinned
memory, the load scales in and the broken counts + tracked displacements
out (the step kernel writes the tracked row to mapped pinned memory), final
state D2H, timed on the host clock.

--impl reference times the reference's own CPU loop (oracle/_ref/ref_driver,
compiled from the unmodified reference headers) on all host cores, on a
bounded sample of the same workload; rank 0 only under torchrun.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PD bond-updates/s (fp64)"
UNIT = "bond-updates/s"
REF_SAMPLE = "cfg3_sample"
REF_FINE_PER_STEP = 1  # reference fine steps per bench step (bounded CPU sample)
FP64_PEAK_TFLOPS = 37.0  # nominal B200 FP64 (vector); MEASURED_PEAKS.json has no fp64 figure
WORKLOADS = {
    "cfg3": "cfg3 (BASELINE configs[2]: 2000x800 plate, dx 0.05 mm, delta 3.015 dx, "
            "per-bond s0 x U[0.95,1.05], constant micromodulus)",
    "cfg1": "cfg1 analog (BASELINE configs[0]: 200x80 plate, dx 0.5 mm, reference-native "
            "exponential kernel l = delta)",
    "cfg4": "cfg4 (BASELINE configs[3]: 3D 200x200x50 hex8 block, dx 0.5 mm, delta 3.015 dx, "
            "constant micromodulus, 20 m/s +-5% impact patch)",
    "cfg5_core": "cfg5 PD core (BASELINE configs[4], the largest PD config) as a pure-PD run: "
                 "3D 400x800x40 hex8 at 0.25 mm, 755M bonds, 40 mm pre-notch, 12 MPa bands, "
                 "constant micromodulus, dt 4 ns",
}


def _env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


class Clocks:
    """nvidia-smi clock / throttle sampling during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu),
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if len(s) > 5 + k and s[5 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def _ncu_traffic(kernel: str, workload: str = ""):
    """dram bytes per launch of `kernel` (on `workload` when captured per workload)
    from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            t = json.load(f)
        e = t.get(f"{kernel}@{workload}") or t.get(kernel, {})
        return e.get("dram_bytes_per_launch")
    return None


REF_DESC = {
    "cfg3_sample": "500x200 sub-plate of cfg3 (dx 0.05 mm, delta 3.015 dx, E 72 GPa, 12 MPa "
                   "bands, exponential kernel l=delta, scalar s_crit)",
    "cfg3_native": "the full cfg3 plate, 2000x800 at dx 0.05 mm (delta 3.015 dx, E 72 GPa, 12 MPa "
                   "bands), in the reference's own arithmetic: exponential kernel l=delta, scalar "
                   "s_crit (it has no constant micromodulus or per-bond s0); setup outside the "
                   "timed loop",
}


def run_reference_cpu(steps: int, warmup: int, threads: int | None = None,
                      name: str = REF_SAMPLE) -> dict:
    """The reference's own loop (ref_driver) on a cfg3 plate (the bounded sample by default)."""
    from oracle import pyoracle as po
    from paper_2403_03605_b200 import configs as cf

    threads = threads or os.cpu_count() or 1
    env = dict(os.environ, PERIMTS_WORKERS=str(threads))
    sc = cf.get(name)
    with tempfile.TemporaryDirectory() as tmp:
        if os.path.exists(po.REF_DRIVER):
            r = po.run_ref(cf.render_cfg(sc), tmp, steps=steps + warmup, dump=False,
                           extra=["--time", "--warmup", str(warmup)], env=env)
            kind = "reference"
        else:  # the C restatement (single thread) when the reference could not be built
            import numpy as np

            from paper_2403_03605_b200.pd import Scenario

            S = Scenario(sc)
            pairs = po.find_pairs(2, S.centroid, S.volume, S.delta, S.notches())
            o = po.OraclePD(dict(dim=2, n_nodes=S.n_nodes, conn=S.conn, centroid=S.centroid,
                                 volume=S.volume, pairs=pairs, mass=S.mass, p_ext=S.p_ext,
                                 delta=S.delta, l=S.l, c0=S.c0, s_crit=S.s_crit, dt=S.dt),
                            po.CSR)
            o.init(0.0)
            o.step(S.scales(1, warmup))
            t = time.perf_counter()
            o.step(S.scales(1 + warmup, steps))
            dt = time.perf_counter() - t
            r = {"bond_updates_per_s": len(pairs) * steps / dt, "bonds": len(pairs),
                 "loop_s": dt, "workers": 1}
            kind, threads = "port", 1
    r["kind"] = kind
    r["threads"] = threads
    r["sample"] = (f"{name}: {REF_DESC[name]}, {steps} timed fine steps after {warmup}, "
                   f"{r['bonds']} bonds")
    return r


MTS_METRIC = "coupled MTS coarse steps/s"
MTS_UNIT = "coarse steps/s"


def run_reference_mts(name: str, steps: int, warmup: int, threads: int | None = None) -> dict:
    """The reference's own coupled loop (ref_mts_driver) on a bounded sample."""
    from oracle import pyoracle as po
    from paper_2403_03605_b200 import configs as cf

    threads = threads or os.cpu_count() or 1
    env = dict(os.environ, PERIMTS_WORKERS=str(threads))
    if not os.path.exists(po.REF_MTS_DRIVER):
        return {"unavailable": "oracle/_ref/ref_mts_driver not built"}
    with tempfile.TemporaryDirectory() as tmp:
        r = po.run_ref_mts(cf.render_cfg(cf.get(name)), tmp, steps=steps + warmup, dump=False,
                           extra=["--time", "--warmup", str(warmup)], env=env)
    r["threads"] = threads
    return r


def bench_mts(steps: int, warmup: int, with_cpu: bool) -> dict:
    """Coupled MTS on BASELINE cfg2's conforming analog: device
    time of K macro steps (CUDA events around the whole sequence, host-side
    orchestration and interface solves inside), plus the same at 0.5 mm next to
    the reference's own coupled loop on that sample."""
    from paper_2403_03605_b200 import configs as cf
    from paper_2403_03605_b200.mts import MtsSolver

    out = {"metric": MTS_METRIC, "unit": MTS_UNIT, "higher_is_better": True}
    res = {}
    # the interface CG Jacobi-preconditioned (run.interface_precond = jacobi, an addition;
    # DESIGN.md 9) on every workload, and cfg2's analog once more with the reference's
    # plain CG (the library default)
    for name, pc in (("cfg2", "jacobi"), ("cfg2_0p5", "jacobi"), ("cfg2_nm", "jacobi"),
                     ("cfg2", "none")):
        c = cf.get(name)
        c["run"]["interface_precond"] = pc
        key = name if pc == "jacobi" else name + "_plain_cg"
        t0 = time.perf_counter()
        s = MtsSolver(c)
        setup = time.perf_counter() - t0
        s.initialize()
        s.macro_step(warmup)
        ms = s.macro_step_timed(steps)
        reps = s.macro_step(1)
        res[key] = {"value": steps / (ms * 1e-3), "ms_per_step": ms / steps, "setup_s": setup,
                    "interface_precond": pc,
                     "n_lambda": s.n_lambda, "fe_dof": s.fe_n_dof, "pd_dof": s.pd_n_dof,
                     "dense_interface": s.dense,
                     "interface_iterations": reps[0]["interface_iterations"]}
        del s
    out.update(value=res["cfg2"]["value"], ms_per_step=res["cfg2"]["ms_per_step"],
               steps=steps, warmup=warmup,
               config={"workload": "cfg2 conforming analog (BASELINE configs[1]; SURVEY App. A): "
                                   "100x40 mm plate, PD band 100x20 mm, FE elsewhere, both "
                                   "0.25 mm, 2 mm linear gluing zones, implicit FE (PCG), "
                                   "explicit PD, m=10, dt_pd 10 ns",
                       **{k: v for k, v in res["cfg2"].items() if k not in ("value", "ms_per_step")}},
               at_0p5mm=res["cfg2_0p5"],
               reference_plain_cg=res["cfg2_plain_cg"],
               as_written={**res["cfg2_nm"],
                           "workload": "cfg2 as BASELINE writes it (non-matching meshes, an "
                                       "extension the reference cannot run): PD band at 0.25 mm, "
                                       "FE on a 1 mm lattice, explicit central-difference FE, "
                                       "2 mm linear gluing zones, interpolating coupling rows, "
                                       "m=10, dt_pd 10 ns (DESIGN.md 11)"})
    if with_cpu:
        r = run_reference_mts("cfg2_0p5", 3, 1)
        if "unavailable" in r:
            out["cpu_baseline"] = r
        else:
            out["cpu_baseline"] = {
                "value": r["macro_steps_per_s"], "unit": MTS_UNIT, "cores": r["threads"],
                "kind": "reference",
                "sample": "cfg2 analog at 0.5 mm (n_lambda 4020), 3 timed macro steps after 1 "
                          f"(setup {r['setup_s']:.1f} s); compare with at_0p5mm.value",
                "ratio_at_0p5mm": res["cfg2_0p5"]["value"] / r["macro_steps_per_s"]}
    out["reference_published"] = ("SURVEY.md 3.2/6: the reference at 0.25 mm takes 541.5 s of "
                                  "setup and ~8.8 s per macro step on 8 cores")
    return out


def bench_reference(args):
    rank, _, world = _env_rank()
    if rank != 0:
        return
    fine = args.steps * REF_FINE_PER_STEP
    r = run_reference_cpu(fine, max(args.warmup, 1) * REF_FINE_PER_STEP, name=args.ref_workload)
    v = r["bond_updates_per_s"]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * r["loop_s"] / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": ("cfg3 (BASELINE configs[2]) at full size in the reference's "
                                "arithmetic" if args.ref_workload == "cfg3_native" else
                                "cfg3 (BASELINE configs[2]) bounded CPU sample"),
                   "sample": r["sample"], "fine_steps_per_step": REF_FINE_PER_STEP},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": r["threads"], "kind": r["kind"],
                         "sample": r["sample"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


class Ctx:
    """One process per GPU: rank / local rank / world from torchrun's environment,
    the gloo control plane (NCCL clique ids, bond counts, max-over-ranks times)."""

    def __init__(self, force_slabs: bool):
        self.rank, self.local, self.world = _env_rank()
        self.dist = None
        self.slabbed = self.world > 1 or force_slabs
        if self.slabbed:
            import torch
            import torch.distributed as dist

            torch.cuda.set_device(self.local)
            if self.world == 1:  # --force-slabs: the slab + NCCL path with one rank
                os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
                os.environ.setdefault("MASTER_PORT", "29533")
                dist.init_process_group("gloo", rank=0, world_size=1)
            else:
                dist.init_process_group("gloo")
            self.dist = dist

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def reduce(self, x: float, op: str = "max") -> float:
        if not self.dist:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64)
        self.dist.all_reduce(t, op={"max": self.dist.ReduceOp.MAX,
                                    "sum": self.dist.ReduceOp.SUM}[op])
        return float(t.item())

    def uid(self) -> bytes:
        import torch

        from paper_2403_03605_b200.pd import PDSolver

        u = torch.zeros(128, dtype=torch.uint8)
        if self.rank == 0:
            u[:] = torch.frombuffer(bytearray(PDSolver.nccl_unique_id()), dtype=torch.uint8)
        self.dist.broadcast(u, 0)
        return bytes(u.tolist())


def measure_pd(args, ctx: Ctx, workload: str, scaling: str, K: int, W: int, mode,
               full: bool = True) -> dict:
    """Device time, roofline, (full:) fp32-position variant and e2e of K fine steps of
    `workload` after W warm-up steps, on ctx.world ranks (slabs: weak = one copy of
    the plate per rank stacked, strong = the plate cut into world slabs)."""
    import numpy as np

    from paper_2403_03605_b200 import capi
    from paper_2403_03605_b200 import configs as cf
    from paper_2403_03605_b200 import slabs
    from paper_2403_03605_b200.pd import PDSolver, Scenario

    rank, local, world = ctx.rank, ctx.local, ctx.world
    if ctx.slabbed:
        sc = Scenario(cf.stacked(workload, world) if scaling == "weak" else cf.get(workload))
        slab = slabs.make_slab(sc.lattice, sc.dim, rank, world)
    else:
        sc = Scenario(cf.get(workload))
        slab = None
    B = None

    def fresh():
        """A new handle stepped through the W warm-up steps: every measurement below
        (device time, roofline, end to end) covers the same steps W+1 .. W+K of the
        BASELINE run, so they time the same physics (cracks start late in cfg3)."""
        nonlocal B
        if slab is not None:
            s = slabs.solver_for_slab(sc, slab, mode, device=local).find_pe_pairs()
            slabs.attach_nccl(s, ctx.uid())
            if B is None:
                lp = s.pairs()
                B = int(ctx.reduce(float(slab.owns_elem(lp[:, 0]).sum()), "sum"))
        else:
            s = PDSolver.from_scenario(sc, mode=mode, device=local).find_pe_pairs()
            if B is None:
                B = s.info()["n_bonds"]
        v0 = sc.initial_velocity()  # cfg4's impact patch (extension); zero for the plates
        if v0.any():
            if slab is not None:  # this slab's nodes (halo included)
                v0 = v0[s.local_dofs]
            z = np.zeros(s.n_dof)
            s.set_state(z, v0, z)
        s.initial_acceleration(sc.load_scale(0.0))
        s.step(sc.scales(1, W))
        return s

    t0 = time.perf_counter()
    s = fresh()
    t_setup = time.perf_counter() - t0
    info = s.info()
    step0 = W + 1
    with Clocks(local) as clk:
        ctx.barrier()
        ms = s.step_timed(sc.scales(step0, K))  # synchronises the stream on both sides
        ctx.barrier()
    variant = None
    if full and slab is None and mode == capi.FAST and sc.dim == 2 and not args.no_variant:
        # BASELINE cfg3's fp32-position / fp64-accumulate variant over the same steps,
        # and how far it lands from the fp64 run at the end of the window
        u64, _, _ = s.state()
        b64 = s.intact() == 0
        del s
        sv = PDSolver.from_scenario(sc, mode=capi.FAST_F32POS, device=local).find_pe_pairs()
        sv.initial_acceleration(sc.load_scale(0.0))
        sv.step(sc.scales(1, W))
        ms_v = sv.step_timed(sc.scales(step0, K))
        u32, _, _ = sv.state()
        b32 = sv.intact() == 0
        variant = {"mode": "f32pos (PMTS_FAST_F32POS)", "dtype": "f32 positions / f64 accumulate",
                   "value": B * K / (ms_v * 1e-3), "unit": UNIT, "ms_per_step": ms_v / K,
                   "u_rel_l2_vs_fp64": float(np.linalg.norm(u32 - u64) / np.linalg.norm(u64)),
                   "broken_fp64": int(b64.sum()), "broken_f32pos": int(b32.sum()),
                   "broken_agreement": float(1.0 - np.logical_xor(b64, b32).sum()
                                             / max(int(b64.sum()), 1))}
        del sv
    else:
        del s
    s = fresh()
    bond_ms, tot_ms = s.profile(sc.scales(step0, K))
    ms = ctx.reduce(ms, "max")
    value = B * K / (ms * 1e-3)  # B = unique bonds of the whole job

    # roofline of the dominant (bond) kernel
    peak, peak_src = _peaks()
    bond_avg_s = bond_ms * 1e-3 / K
    timing = "each launch between its own pair of CUDA events (profile pass)"
    if info["kernels_per_step"] == 1 and not ctx.dist:
        # one kernel per step (the 2D tile kernel): the timed region's K back-to-back
        # launches between two events on the launching stream ARE the kernel's launches;
        # per-launch events would break programmatic dependent launch, which overlaps
        # each launch with the previous one's tail
        bond_avg_s = ms * 1e-3 / K
        timing = ("timed region: K back-to-back launches of the step's only kernel between two "
                  "CUDA events on its stream (programmatic dependent launch on)")
    achieved = info["bond_bytes_per_step"] / bond_avg_s / 1e9
    kname = {2: "k_tile9", 1: "k_lat3_bond" if info["stencil_size"] == 122 else "k_lat_bond"}.get(
        info["path"], "k_fast_bond" if mode == capi.FAST else "k_det_bond")
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": _ncu_traffic(kname, workload),
            "kernel": kname, "bytes_per_launch": info["bond_bytes_per_step"],
            "avg_launch_us": bond_avg_s * 1e6, "launch_timing": timing,
            "avg_launch_us_isolated": bond_ms * 1e3 / K,
            "bond_share_of_step": bond_ms / tot_ms if tot_ms else None, "peak_source": peak_src}
    if info["path"] == 2:
        # round 2 restated the model: 72 B per node (rd, rv in and out, {1/M | flags}) plus
        # 8 B per element only on the tiles that still stage and re-write their bond
        # states (clean tiles touch none); round 1 counted 81 B per element everywhere
        r1 = s.n_nodes * 73.0 + s.n_elems * 8.0
        roof["bytes_model"] = ("72 B/node + 8 B/element on tiles staging bond states "
                               "(info at the window's start)")
        roof["frac_round1_model"] = r1 / bond_avg_s / 1e9 / peak
    # the bond work is fp64-arithmetic heavy.  2D: 14 flops per directed entry in fast
    # mode (eta 2, xi.eta 3, force 4, |eta|^2 3, test 2) = 28 per unique bond; 3D (the
    # 122-offset kernel, break test screened off on cold tiles): eta 3, o.eta 3 (small-
    # integer multiplies as adds), scale 1, force 3 = 10 per directed entry, 20 per bond
    fpb = 28 if sc.dim == 2 else 20
    flops = fpb * (B / world) / bond_avg_s / 1e12
    roof_fp64 = {"bound": "fp64", "achieved": flops, "peak": FP64_PEAK_TFLOPS,
                 "unit": "TFLOP/s", "frac": flops / FP64_PEAK_TFLOPS,
                 "flops_per_bond": fpb, "peak_source": "nominal B200 FP64 (no measured fp64 peak)"}

    # end to end through the public C-ABI with host buffers
    e2e = None
    if full:
        try:
            import torch

            del s
            s = fresh()
            nd = s.n_dof
            hu = torch.empty(nd, dtype=torch.float64, pin_memory=True).numpy()
            hv = torch.empty(nd, dtype=torch.float64, pin_memory=True).numpy()
            ha = torch.empty(nd, dtype=torch.float64, pin_memory=True).numpy()
            u0, v0, a0 = s.state()
            hu[:], hv[:], ha[:] = u0, v0, a0
            tracked = np.array([sc.dim * (s.n_nodes // 2) + 1], dtype=np.int32)
            scales = sc.scales(step0, K)
            trk = torch.empty((K, len(tracked)), dtype=torch.float64, pin_memory=True).numpy()
            nbk = torch.empty(K, dtype=torch.int64, pin_memory=True).numpy()
            hsc = torch.empty(K, dtype=torch.float64, pin_memory=True).numpy()
            hsc[:] = scales
            ctx.barrier()
            t = time.perf_counter()
            s.set_state(hu, hv, ha)
            # one public call for the K steps; inside it, per step and asynchronously:
            # the step's scale H2D, the step, its tracked displacement + broken count D2H
            s.step_tracked(hsc, tracked, trk, nbk)
            s.get_state_into(hu, hv, ha)
            e2e_s = ctx.reduce(time.perf_counter() - t, "max")
            h2d = (3 * nd * 8 + K * 8) / K
            d2h = (3 * nd * 8 + K * (8 + 8 * len(tracked))) / K
            e2e = {"value": B * K / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * e2e_s / K,
                   "note": "per rank, one pmts_pd_step_tracked call for the K steps: state H2D "
                           "from pinned memory, the K load scales H2D in one copy, per step "
                           "(async on the stream) the step and its tracked displacement written "
                           "into mapped pinned memory (2D: by the step kernel; 3D lattice: by a "
                           "tiny launch reading the step's predictor); the K broken counts D2H "
                           "in one copy; final state D2H"}
        except Exception as ex:  # pragma: no cover - reported, never silent
            e2e = {"value": None, "unit": UNIT, "error": repr(ex)}
    # the late regime of the BASELINE run (cfg3: cracks start near step 700, so the
    # default window W+1..W+K is the cold-tile screen's best case): steps 1001..1000+K2
    # after fast-forwarding a fresh handle, with the fraction of tiles the screen let
    # through; and the end-to-end number over 1000 steps (state copies amortised)
    late = steady = None
    if full and slab is None and sc.dim == 2:
        try:
            import torch

            del s
            K2 = 200
            s = PDSolver.from_scenario(sc, mode=mode, device=local).find_pe_pairs()
            s.initial_acceleration(sc.load_scale(0.0))
            s.step(sc.scales(1, 1000))
            s.set_option(capi.OPT_COUNT_HOT, 1)
            ms_l = s.step_timed(sc.scales(1001, K2))
            inf = s.info()
            late = {"steps": f"1001..{1000 + K2}", "value": B * K2 / (ms_l * 1e-3), "unit": UNIT,
                    "ms_per_step": ms_l / K2, "broken_total": s.broken_total(),
                    "hot_tile_fraction": inf["hot_tiles"] / max(inf["tested_tiles"], 1),
                    "note": "fresh handle fast-forwarded through steps 1..1000; hot tiles = "
                            "tiles whose break test the cold-tile screen could not skip"}
            if K < 1000:
                del s
                s = fresh()
                nd = s.n_dof
                hu = torch.empty(nd, dtype=torch.float64, pin_memory=True).numpy()
                hv = torch.empty(nd, dtype=torch.float64, pin_memory=True).numpy()
                ha = torch.empty(nd, dtype=torch.float64, pin_memory=True).numpy()
                u0, v0, a0 = s.state()
                hu[:], hv[:], ha[:] = u0, v0, a0
                K3 = 1000
                tracked = np.array([sc.dim * (s.n_nodes // 2) + 1], dtype=np.int32)
                trk = torch.empty((K3, 1), dtype=torch.float64, pin_memory=True).numpy()
                nbk = torch.empty(K3, dtype=torch.int64, pin_memory=True).numpy()
                hsc = torch.empty(K3, dtype=torch.float64, pin_memory=True).numpy()
                hsc[:] = sc.scales(step0, K3)
                t = time.perf_counter()
                s.set_state(hu, hv, ha)
                s.step_tracked(hsc, tracked, trk, nbk)
                s.get_state_into(hu, hv, ha)
                e3 = time.perf_counter() - t
                steady = {"steps": K3, "value": B * K3 / e3, "unit": UNIT,
                          "ms_per_step": 1e3 * e3 / K3,
                          "h2d_bytes_per_step": (3 * nd * 8 + K3 * 8) / K3,
                          "d2h_bytes_per_step": (3 * nd * 8 + K3 * 16) / K3,
                          "note": "the e2e procedure over 1000 steps in one call: the state "
                                  "copies amortised as in a production run"}
        except Exception as ex:  # pragma: no cover - reported, never silent
            late = {"error": repr(ex)}
    del s
    ws = info["device_bytes"] / 1e6
    if world == 1:
        par = "single" if slab is None else "slabs1 (NCCL clique of one)"
    else:
        par = f"slabs{world} (z-x slabs, NCCL halo send/recv)" if sc.dim == 3 else \
            f"slabs{world} (x-slabs, NCCL halo send/recv)"
    desc = WORKLOADS.get(workload, workload)
    if world > 1:
        desc += (f"; weak scaling: {world} copies stacked, one slab per GPU" if scaling == "weak"
                 else f"; strong scaling: the same plate cut into {world} slabs")
    out = {"value": value, "unit": UNIT, "ms_per_step": ms / K, "steps": K, "warmup": W,
           "scaling": scaling, "bonds": B,
           "config": {"workload": desc, "mode": args.mode, "bonds": B, "elements": sc.n_elems,
                      "nodes": sc.n_nodes, "parallelism": par,
                      "l2": f"inputs larger than L2 (device working set {ws:.0f} MB per rank "
                            f"> 126 MB)", "setup_s": t_setup},
           "roofline": roof, "roofline_fp64": roof_fp64, "e2e": e2e,
           "gpu_launches": K * info["kernels_per_step"], "clocks": clk.summary()}
    if slab is not None and sc.dim == 3:
        out["config"]["redundancy"] = slabs.redundancy(sc.lattice, 3, world)
    if variant:
        out["f32pos_variant"] = variant
    if late:
        out["late_window"] = late
    if steady:
        out["e2e_1000_steps"] = steady
    return out


def bench_cfg5_mts(steps: int, warmup: int) -> dict:
    """BASELINE cfg5 (configs[4]) as the coupled run it describes (configs.py cfg5_mts:
    12.8M-hex PD core at 0.25 mm, 1 mm hex8 FE, m = 20, 1.77M multipliers) on one GPU:
    setup time, then K macro steps (CUDA events), the interface operator in its
    recursion form (the precomputed H_PD would be ~10^11 entries)."""
    import torch

    from paper_2403_03605_b200 import configs as cf
    from paper_2403_03605_b200.mts import MtsSolver

    c = cf.get("cfg5_mts")
    c["run"]["interface_precond"] = "jacobi"  # (as the cfg2 line; the plain CG: +~1x iters)
    t0 = time.perf_counter()
    s = MtsSolver(c)
    t1 = time.perf_counter()
    s.initialize()
    setup = time.perf_counter() - t0
    free_b, total_b = torch.cuda.mem_get_info(0)
    reps = s.macro_step(warmup)
    torch.cuda.profiler.start()  # (a range for `ncu --profile-from-start off`; no-op otherwise)
    ms = s.macro_step_timed(steps)
    torch.cuda.profiler.stop()
    last = s.macro_step(1)[0]
    u = s.state("pd")[0]
    return {"metric": MTS_METRIC, "unit": MTS_UNIT, "value": steps / (ms * 1e-3),
            "ms_per_step": ms / steps, "steps": steps, "warmup": warmup, "n_gpus": 1,
            "higher_is_better": True, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "BASELINE cfg5 coupled: 400x200x10 mm plate, PD core "
                                   "100x200x10 mm at 0.25 mm (12.8M hexes), FE hex8 1 mm "
                                   "(non-matching), 2 mm linear gluing zones, explicit FE, "
                                   "m=20, dt_pd 4 ns, 40 mm pre-notch, 12 MPa",
                       "n_lambda": s.n_lambda, "fe_dof": s.fe_n_dof, "pd_dof": s.pd_n_dof,
                       "pd_pairs": int(s.n_pairs), "create_s": t1 - t0, "setup_s": setup,
                       "interface_precond": "jacobi",
                       "device_mem_used_gb": (total_b - free_b) / 1e9},
            "interface_iterations": [r["interface_iterations"] for r in reps] +
                                    [last["interface_iterations"]],
            "continuity_max": max(r["continuity"] for r in reps + [last]),
            "newly_broken": [r["newly_broken"] for r in reps] + [last["newly_broken"]],
            "pd_u_max": float(abs(u).max())}


def bench_mts_sharded(args):
    """Coupled MTS with the PD band sharded across N GPUs (north star item 5; DESIGN.md
    9a): shard r on GPU r, ghost layers over NCCL every fine substep, FE on rank 0, the
    interface solve replicated (the reference's plain CG: the Jacobi option is single-
    domain only).  Device time of K macro steps per rank (CUDA events), max over ranks."""
    from paper_2403_03605_b200 import configs as cf
    from paper_2403_03605_b200.mts import MtsSolver

    ctx = Ctx(False)
    c = cf.get("cfg2")
    c["run"]["interface"] = "matrix_free"
    t0 = time.perf_counter()
    s = MtsSolver(c, device=ctx.local, shard=(ctx.rank, ctx.world))
    s.comm_init(ctx.uid())
    s.initialize()
    setup = ctx.reduce(time.perf_counter() - t0)
    s.macro_step(args.warmup)
    ctx.barrier()
    ms = ctx.reduce(s.macro_step_timed(args.steps))
    if ctx.rank == 0:
        v = args.steps / (ms * 1e-3)
        print(json.dumps({
            "metric": MTS_METRIC, "value": v, "unit": MTS_UNIT, "n_gpus": ctx.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "gpu_launches": None,
            "config": {"workload": "cfg2 conforming analog, PD band sharded in y slabs "
                                   "(DESIGN.md 9a), interface plain CG", "setup_s": setup,
                       "parallelism": f"pd_shards{ctx.world}",
                       "pd_local_elems": len(s.shard["local_elems"]),
                       "pd_layers": s.shard["n_layers"]}}), flush=True)
    del s


def bench_native(args):
    from paper_2403_03605_b200 import capi

    ctx = Ctx(args.force_slabs)
    if ctx.world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {ctx.world}")
    mode = {"fast": capi.FAST, "det": capi.DETERMINISTIC, "f32pos": capi.FAST_F32POS}[args.mode]
    K, W = args.steps, args.warmup
    scaling = args.scaling or ("weak" if args.workload == "cfg3" else "strong")
    r = measure_pd(args, ctx, args.workload, scaling, K, W, mode)
    # the 3D configurations (BASELINE cfg4, and cfg5's PD core -- the north star's
    # scaling target, cut into ctx.world z-x slabs): shorter windows, same metric
    workloads = {}
    if not args.no_workloads and args.workload == "cfg3":
        for name, k in (("cfg4", args.w3d_steps), ("cfg5_core", max(args.w3d_steps // 2, 10))):
            try:
                wmode = capi.FAST if mode == capi.FAST_F32POS else mode  # fp32 pos.: 2D only
                w = measure_pd(args, ctx, name, "strong", k, W, wmode, full=False)
                workloads[name] = {key: w[key] for key in
                                   ("value", "unit", "ms_per_step", "steps", "warmup", "scaling",
                                    "config", "roofline", "roofline_fp64", "gpu_launches")}
            except Exception as ex:  # pragma: no cover - reported, never silent
                workloads[name] = {"error": repr(ex)}
    cpu = None
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu_baseline:
        c = run_reference_cpu(args.cpu_steps, 4)
        cpu = {"value": c["bond_updates_per_s"], "unit": UNIT, "cores": c["threads"],
               "kind": c["kind"], "sample": c["sample"]}
    if ctx.rank == 0:
        line = {
            "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": ctx.world, "steps": K,
            "warmup": W, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
            "scaling": r["scaling"], "vs_baseline": None,
            "dtype": "f32 positions / f64 accumulate" if mode == capi.FAST_F32POS else "f64",
            "data": "synthetic",
            "config": r["config"],
            "roofline": r["roofline"],
            "roofline_fp64": r["roofline_fp64"],
            "cpu_baseline": cpu,
            "e2e": r["e2e"],
            "gpu_launches": r["gpu_launches"],
            "clocks": r["clocks"],
        }
        for key in ("f32pos_variant", "late_window", "e2e_1000_steps"):
            if key in r:
                line[key] = r[key]
        if workloads:
            line["workloads"] = workloads
        if ctx.world == 1 and not args.no_mts:
            try:
                line["coupled_mts"] = bench_mts(args.mts_steps, 3, not args.no_cpu_baseline)
            except Exception as ex:  # pragma: no cover - reported, never silent
                line["coupled_mts"] = {"metric": MTS_METRIC, "error": repr(ex)}
        print(json.dumps(line), flush=True)
    if ctx.dist:
        ctx.dist.destroy_process_group()


def _spawn_ranks(args) -> int:
    """--gpus N without torchrun's environment: re-launch this command under
    torch.distributed.run, one rank per GPU (127.0.0.1 rendezvous)."""
    import socket

    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--workload", default="cfg3")
    ap.add_argument("--mode", default="fast", choices=["fast", "det", "f32pos"])
    ap.add_argument("--cpu-steps", type=int, default=200)
    ap.add_argument("--ref-workload", default="cfg3_native", choices=["cfg3_native", "cfg3_sample"],
                    help="--impl reference: the full cfg3 plate (default) or the 500x200 sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-variant", action="store_true",
                    help="skip the fp32-position variant line of the default run")
    ap.add_argument("--no-mts", action="store_true",
                    help="skip the coupled MTS (cfg2) section of the line")
    ap.add_argument("--mts-steps", type=int, default=20)
    ap.add_argument("--force-slabs", action="store_true",
                    help="run the multi-GPU slab path (NCCL clique) even with one rank")
    ap.add_argument("--scaling", choices=["weak", "strong"], default=None,
                    help="N > 1: weak = one copy of the plate per GPU (cfg3 default), strong = "
                         "the plate cut into N slabs (3D default)")
    ap.add_argument("--no-workloads", action="store_true",
                    help="skip the cfg4 / cfg5_core section of the default line")
    ap.add_argument("--w3d-steps", type=int, default=200,
                    help="timed fine steps of the cfg4 workload (cfg5_core: half)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(_spawn_ranks(args))
    if "WORLD_SIZE" in os.environ and _env_rank()[2] != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {_env_rank()[2]}")
    if args.workload == "cfg2" and args.impl != "reference" and _env_rank()[2] > 1:
        bench_mts_sharded(args)  # the PD band sharded across the ranks
        return
    if args.workload == "cfg5_mts":  # BASELINE cfg5 as a coupled run, at size
        if _env_rank()[0] == 0:
            print(json.dumps(bench_cfg5_mts(args.steps, args.warmup)), flush=True)
        return
    if args.workload == "cfg2":  # the coupled MTS metric as its own line
        rank, _, _ = _env_rank()
        if rank != 0:
            return
        if args.impl == "reference":
            r = run_reference_mts("cfg2_0p5", args.steps, args.warmup)
            v = r.get("macro_steps_per_s")
            line = {"impl": "reference", "metric": MTS_METRIC, "value": v, "unit": MTS_UNIT,
                    "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                    "ms_per_step": 1e3 / v if v else None, "higher_is_better": True,
                    "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                    "config": {"workload": "cfg2 analog at 0.5 mm (bounded CPU sample; the "
                                           "0.25 mm setup alone takes ~9 min on the CPU)"},
                    "cpu_baseline": {"value": v, "unit": MTS_UNIT, "cores": r.get("threads"),
                                     "kind": "reference", "sample": "cfg2 analog at 0.5 mm"},
                    "e2e": {"value": v, "unit": MTS_UNIT, "h2d_bytes_per_step": 0,
                            "d2h_bytes_per_step": 0}}
        else:
            out = bench_mts(args.steps, args.warmup, not args.no_cpu_baseline)
            line = {"n_gpus": 1, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                    "data": "synthetic", "gpu_launches": None, **out}
        print(json.dumps(line), flush=True)
        return
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_native(args)


if __name__ == "__main__":
    main()
