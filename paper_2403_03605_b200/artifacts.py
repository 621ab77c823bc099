"""Run artifacts in the reference's on-disk format, so the
reference's own `compare` (driver.hpp:290-334) can score device runs against
reference runs: meta.txt, tracked.csv, timing.csv, energy.csv (coupled), frames.csv
and legacy-VTK frames with damage cell data -- the files `finalize_outputs` and
`FrameWriter` write (driver_run.hpp:58-113, driver.hpp:234-262, io.hpp:28-94,
185-199).  The runs are the device paths: `run_pure_pd` drives a `PDSolver`,
`run_coupled` an `MtsSolver`.
"""
from __future__ import annotations

import os
import time

import numpy as np

from . import capi


# ---- formats ----------------------------------------------------------------
def mesh_hash(dim: int, nodes: np.ndarray, conn: np.ndarray) -> int:
    """io.hpp:224-247: FNV-1a over dim, counts, coordinate bits, kinds, node ids."""
    h = 1469598103934665603
    mask = (1 << 64) - 1

    def mix(v: int):
        nonlocal h
        for b in range(8):
            h ^= (v >> (8 * b)) & 0xFF
            h = (h * 1099511628211) & mask

    mix(dim)
    mix(len(nodes))
    mix(len(conn))
    for bits in np.ascontiguousarray(nodes[:, :dim]).view(np.uint64).ravel():
        mix(int(bits))
    kind = 0 if dim == 2 else 1  # ElemKind::quad4 / hex8
    for row in conn:
        mix(kind)
        for a in row:
            mix(int(a))
    return h


def write_csv(header, rows, path):
    """io.hpp:185-199 -- '%.16e' values."""
    with open(path, "w") as f:
        f.write(",".join(header) + "\n")
        for row in rows:
            f.write(",".join("%.16e" % v for v in row) + "\n")


def write_vtk(path, dim, nodes, conn, disp, vel, damage_avg, damage, labels, alpha):
    """io.hpp:28-94 (ASCII legacy unstructured grid)."""
    nn, ne = len(nodes), len(conn)
    out = ["# vtk DataFile Version 3.0", "perimts fields", "ASCII", "DATASET UNSTRUCTURED_GRID",
           f"POINTS {nn} double"]
    out += ["%.17g %.17g %.17g" % tuple(p) for p in nodes]
    k = conn.shape[1]
    out.append(f"CELLS {ne} {ne * (1 + k)}")
    out += [f"{k} " + " ".join(str(int(a)) for a in row) for row in conn]
    out.append(f"CELL_TYPES {ne}")
    out += [("9" if dim == 2 else "12")] * ne
    out.append(f"POINT_DATA {nn}")

    def vec(name, v):
        v = np.asarray(v).reshape(nn, dim)
        out.append(f"VECTORS {name} double")
        for r in v:
            out.append("%.17g %.17g %.17g" % (r[0], r[1], r[2] if dim == 3 else 0.0))

    vec("displacement", disp)
    vec("velocity", vel)
    out.append("SCALARS damage_avg double 1")
    out.append("LOOKUP_TABLE default")
    out += ["%.17g" % x for x in damage_avg]
    out.append(f"CELL_DATA {ne}")
    out.append("SCALARS damage double 1")
    out.append("LOOKUP_TABLE default")
    out += ["%.17g" % x for x in damage]
    out.append("SCALARS subdomain_label int 1")
    out.append("LOOKUP_TABLE default")
    out += [str(int(x)) for x in labels]
    out.append("SCALARS alpha double 1")
    out.append("LOOKUP_TABLE default")
    out += ["%.17g" % x for x in alpha]
    with open(path, "w") as f:
        f.write("\n".join(out) + "\n")


def write_meta(path, mhash, dim, n_nodes, n_elems, n_tracked, mode, dt_pd, m, total_time,
               interval):
    """driver_run.hpp:62-80 (ostream default formatting: %g)."""
    with open(path, "w") as f:
        f.write("[run]\n")
        f.write(f"mesh_hash = {mhash}\n")
        f.write(f"dim = {dim}\nnodes = {n_nodes}\nelements = {n_elems}\n")
        f.write(f"tracked = {n_tracked}\nmode = {mode}\n")
        f.write("dt_pd = %g\nm = %d\ntotal_time = %g\ninterval = %g\n" % (dt_pd, m, total_time,
                                                                        interval))


def tracked_nodes(sc: dict, nodes: np.ndarray) -> list[int]:
    """detail::nearest_node for every output.tracked<k> point (driver.hpp:58-71)."""
    dim = int(sc["mesh"]["dim"])
    out = []
    for k, v in sorted(sc.get("output", {}).items()):
        if not k.startswith("tracked"):
            continue
        p = np.zeros(3)
        p[:dim] = v[:dim]
        d = np.sqrt(((nodes - p) ** 2).sum(axis=1))
        out.append(int(np.argmin(d)))  # first minimum, as the reference's strict <
    return out


class _Frames:
    """FrameWriter.due (driver.hpp:244-248)."""

    def __init__(self, interval, dt_pd):
        self.interval = interval
        self.tol = 1e-9 * max(dt_pd, 1e-300)
        self.next = 0
        self.index = []

    def due(self, t):
        return self.interval > 0.0 and t + self.tol >= self.next * self.interval


# ---- runs -------------------------------------------------------------------
def run_pure_pd(cfg: dict, out_dir: str, mode=capi.DETERMINISTIC, steps=None) -> dict:
    """run_built's pure-PD branch (driver_run.hpp:160-246) on the device, with its
    artifacts."""
    from .pd import PDSolver, Scenario

    os.makedirs(out_dir, exist_ok=True)
    sc = Scenario(cfg)
    s = PDSolver.from_scenario(sc, mode=mode).find_pe_pairs()
    dim, nodes, conn = sc.dim, sc.nodes, sc.conn
    tn = tracked_nodes(cfg, nodes)
    dofs = np.array([n * dim + c for n in tn for c in range(dim)], dtype=np.int32)
    n_steps = sc.n_steps if steps is None else steps
    out = cfg.get("output", {})
    interval = float(out.get("interval", 0.0))
    frames = _Frames(interval, sc.dt)
    ne = sc.n_elems
    labels, alpha = np.ones(ne, dtype=np.int32), np.zeros(ne)

    def emit(t):
        u, v, _ = s.state()
        de, dn = s.damage_field()
        write_vtk(os.path.join(out_dir, "frame_%05d.vtk" % frames.next), dim, nodes, conn, u, v,
                  dn, de, labels, alpha)
        frames.index.append([float(frames.next), t])
        frames.next += 1

    s.initial_acceleration(sc.load_scale(0.0))
    u0, _, _ = s.state()
    t_rows = [[0.0] + list(u0[dofs])]
    timing = []
    if frames.due(0.0):
        emit(0.0)
    i = 1
    while i <= n_steps:
        # run to the next frame (or the end) in one tracked batch
        j = i
        while j < n_steps and not frames.due(j * sc.dt):
            j += 1
        tick = time.perf_counter()
        trk, nb = s.step_tracked(sc.scales(i, j - i + 1), dofs)
        per = (time.perf_counter() - tick) / (j - i + 1)
        for k in range(j - i + 1):
            t = (i + k) * sc.dt
            t_rows.append([t] + list(trk[k]))
            timing.append([float(i + k - 1), per, 0.0, 0.0, 0.0, float(nb[k]), 0.0])
        if frames.due(j * sc.dt):
            emit(j * sc.dt)
        i = j + 1
    header = ["t"] + [f"p{p}_u{'xyz'[c]}" for p in range(len(tn)) for c in range(dim)]
    write_csv(header, t_rows, os.path.join(out_dir, "tracked.csv"))
    write_csv(["step", "t_k", "t_u", "t_lambda", "t_y", "broken", "continuity"], timing,
              os.path.join(out_dir, "timing.csv"))
    if frames.index:
        write_csv(["frame", "t"], frames.index, os.path.join(out_dir, "frames.csv"))
    tm = cfg["time"]
    write_meta(os.path.join(out_dir, "meta.txt"), mesh_hash(dim, nodes, conn), dim, len(nodes),
               ne, len(tn), "pure_pd", tm["dt_pd"], int(tm.get("m", 1)), tm["total_time"],
               interval)
    return {"steps": n_steps, "broken": int(sum(r[5] for r in timing)), "frames": len(frames.index)}


def run_coupled(cfg: dict, out_dir: str, steps=None) -> dict:
    """run_built's coupled branch (driver_run.hpp:247-295) on the device, with its
    artifacts (nodal values alpha-blended as NodalFieldSampler, :16-56)."""
    from .mts import MtsSolver

    os.makedirs(out_dir, exist_ok=True)
    ms = MtsSolver(cfg)
    sy = ms.system()
    dim, nodes, conn = ms.dim, sy["node_xyz"], sy["elem_nodes"]
    fnd, pnd, nal = sy["fe_node_dof"], sy["pd_node_dof"], sy["node_alpha"]
    tn = tracked_nodes(cfg, nodes)
    n_macro = ms.n_macro if steps is None else steps
    out = cfg.get("output", {})
    interval = float(out.get("interval", 0.0))
    frames = _Frames(interval, ms.dt_pd)

    def blend(fe_x, pd_x, node, c):
        in_fe, in_pd = fnd[node] >= 0, pnd[node] >= 0
        if in_fe and in_pd:
            a = nal[node]
            return a * fe_x[fnd[node] + c] + (1.0 - a) * pd_x[pnd[node] + c]
        if in_fe:
            return fe_x[fnd[node] + c]
        if in_pd:
            return pd_x[pnd[node] + c]
        return 0.0

    def sample():
        fu, fv, _ = ms.state("fe")
        pu, pv, _ = ms.state("pd")
        return fu, fv, pu, pv

    def emit(t):
        fu, fv, pu, pv = sample()
        nn = len(nodes)
        disp = np.array([blend(fu, pu, n, c) for n in range(nn) for c in range(dim)])
        vel = np.array([blend(fv, pv, n, c) for n in range(nn) for c in range(dim)])
        de, dn = ms.damage_field()
        write_vtk(os.path.join(out_dir, "frame_%05d.vtk" % frames.next), dim, nodes, conn, disp,
                  vel, dn, de, sy["labels"], sy["alpha"])
        frames.index.append([float(frames.next), t])
        frames.next += 1

    def row(t):
        fu, _, pu, _ = sample()
        return [t] + [blend(fu, pu, n, c) for n in tn for c in range(dim)]

    ms.initialize()
    t_rows = [row(0.0)]
    if frames.due(0.0):
        emit(0.0)
    timing, energy = [], []
    for i in range(1, n_macro + 1):
        rep = ms.macro_step(1)[0]
        t = i * ms.dt_fe
        timing.append([float(i - 1), rep["t_kinematic"], rep["t_update"], rep["t_lambda"],
                       rep["t_unit"], float(rep["newly_broken"]), rep["continuity"]])
        e = [rep["quad_fe"], rep["quad_pd"], rep["lambda_fe"], rep["lambda_pd"]]
        energy.append([float(i - 1)] + e + [sum(e)])
        t_rows.append(row(t))
        if frames.due(t):
            emit(t)
    header = ["t"] + [f"p{p}_u{'xyz'[c]}" for p in range(len(tn)) for c in range(dim)]
    write_csv(header, t_rows, os.path.join(out_dir, "tracked.csv"))
    write_csv(["step", "t_k", "t_u", "t_lambda", "t_y", "broken", "continuity"], timing,
              os.path.join(out_dir, "timing.csv"))
    write_csv(["step", "quad_fe", "quad_pd", "lambda_fe", "lambda_pd", "total"], energy,
              os.path.join(out_dir, "energy.csv"))
    if frames.index:
        write_csv(["frame", "t"], frames.index, os.path.join(out_dir, "frames.csv"))
    tm = cfg["time"]
    write_meta(os.path.join(out_dir, "meta.txt"), mesh_hash(dim, nodes, conn), dim, len(nodes),
               len(conn), len(tn), "coupled_mts", tm["dt_pd"], int(tm.get("m", 1)),
               tm["total_time"], interval)
    return {"steps": n_macro, "broken": int(sum(r[5] for r in timing)),
            "frames": len(frames.index)}
