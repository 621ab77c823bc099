"""Coupled multi-time-step (Arlequin PD + FE) integrator -- the Python side of
pmts_mts_* (include/pmts_capi.h), SURVEY.md 8(f) row 1.

Mirrors the reference's coupled run (driver_run.hpp:247-295 ->
CoupledIntegrator, mts.hpp:79-535): build the scenario, initialize the
accelerations, then macro steps of one FE step and m PD substeps glued by
Lagrange multipliers on the overlap.  The integrator runs on the device;
device=-1 builds only the host-assembled systems (for setup parity checks).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import capi
from .capi import check, lib, ptr
from .pd import scenario_desc

WEIGHT_KIND = {"constant": 0, "linear": 1, "cubic": 2}
INTERFACE = {"auto": 0, "dense": 1, "matrix_free": 2}


def _arr(p, ctype, n, shape=None):
    if n == 0 or not p:
        return np.zeros(0 if shape is None else shape, dtype=np.dtype(ctype))
    a = np.ctypeslib.as_array(C.cast(p, C.POINTER(ctype)), shape=(n,)).copy()
    return a.reshape(shape) if shape else a


class MtsSolver:
    """One coupled run (reference config vocabulary: [region], time.m, gamma_fe,
    beta_fe, run.interface, ...)."""

    def __init__(self, sc: dict, device: int = 0, shard: tuple[int, int] | None = None):
        """shard = (rank, world): PD shard `rank` of a sharded run; join the
        shards with ShardGroup (one process) or comm_init (NCCL, one process per GPU)."""
        self.cfg = sc
        self._keep = []
        sd = scenario_desc(sc, self._keep)
        self._sd = sd
        reg, tm, run = sc["region"], sc["time"], sc.get("run", {})
        dim = int(sc["mesh"]["dim"])
        boxes = []
        for k, v in sorted(reg.items()):
            if k.startswith("pd_box"):
                lo = [v[i] if i < dim else 0.0 for i in range(3)]
                hi = [v[dim + i] if i < dim else 0.0 for i in range(3)]
                boxes.append(lo + hi)
        self._boxes = np.array(boxes or [[0.0] * 6], dtype=np.float64)
        d = capi.MtsDesc()
        d.scenario = C.pointer(sd)
        d.n_pd_box, d.pd_boxes = len(boxes), ptr(self._boxes)
        d.overlap_width_factor = reg.get("overlap_width_factor", 3.0)
        d.weight_kind = WEIGHT_KIND[reg.get("weight_kind", "cubic")]
        d.gamma_fe, d.beta_fe = tm.get("gamma_fe", 0.5), tm.get("beta_fe", 0.25)
        d.interface_mode = INTERFACE[run.get("interface", "auto")]
        d.enforce_continuity = 1 if run.get("enforce_continuity", True) else 0
        d.track_energy = 1 if sc.get("output", {}).get("energy", True) else 0
        d.device = device
        # extension: non-matching FE lattice (mesh.fe_spacing), DESIGN.md section 11
        d.fe_spacing = float(sc["mesh"].get("fe_spacing") or 0.0)
        # extension: Jacobi-preconditioned interface CG (run.interface_precond = jacobi);
        # the default is the reference's plain CG
        d.interface_precond = 1 if run.get("interface_precond", "none") == "jacobi" else 0
        # run.interface_h_pd = precompute (default) | recursion
        d.interface_recursion = 1 if run.get("interface_h_pd", "precompute") == "recursion" else 0
        # run.interface_h_fe = sparse (default) | unit_columns (explicit FE side)
        d.interface_h_fe = 1 if run.get("interface_h_fe", "sparse") == "unit_columns" else 0
        # run.pd_linear = lattice (default: where the PD elements are a 3D box lattice) | ell
        d.pd_linear = 1 if run.get("pd_linear", "lattice") == "ell" else 0
        # run.pd_elem_products = auto (default) | on | off
        d.pd_elem_products = {"auto": 0, "on": 1, "off": 2}[run.get("pd_elem_products", "auto")]
        if shard is not None:
            d.shard_rank, d.shard_world = int(shard[0]), int(shard[1])
        h = C.c_void_p()
        check(lib().pmts_mts_create(C.byref(d), C.byref(h)))
        self.h = h
        v = capi.MtsView()
        check(lib().pmts_mts_view_get(h, C.byref(v)))
        self.view = v
        self.dim, self.n_nodes, self.n_elems = v.dim, v.n_nodes, v.n_elems
        self.fe_n_dof, self.pd_n_dof, self.n_lambda = v.fe_n_dof, v.pd_n_dof, v.n_lambda
        self.dense, self.m, self.n_macro = bool(v.dense), v.m, v.n_macro
        self.dt_pd = v.dt_pd
        self.dt_fe = v.m * v.dt_pd
        self.n_pairs = v.n_pairs
        sv = capi.MtsShardView()
        check(lib().pmts_mts_shard_view_get(h, C.byref(sv)))
        self.shard = {
            "world": sv.world, "rank": sv.rank, "axis": sv.axis, "reach_layers": sv.reach_layers,
            "n_layers": sv.n_layers, "own_elems": (sv.own_elem_lo, sv.own_elem_hi),
            "local_nodes": _arr(sv.local_nodes, C.c_int32, sv.n_local_nodes),
            "local_elems": _arr(sv.local_elems, C.c_int32, sv.n_local_elems),
            "node_owned": _arr(sv.node_owned, C.c_uint8, sv.n_local_nodes).astype(bool),
            "layer_bounds": _arr(sv.layer_bounds, C.c_int32, sv.world + 1),
        }
        self.pd_local_dofs = (self.shard["local_nodes"][:, None] * self.dim
                              + np.arange(self.dim)[None, :]).reshape(-1)

    def comm_init(self, uid: bytes):
        """Join the NCCL clique of a sharded run (uid: pmts_nccl_unique_id of shard 0)."""
        buf = C.create_string_buffer(uid, 128)
        check(lib().pmts_mts_comm_init(self.h, buf))

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            lib().pmts_mts_destroy(h)
            self.h = None

    # -- assembled systems (host) -------------------------------------------
    def system(self) -> dict:
        v, i32, f64 = self.view, C.c_int32, C.c_double
        nf, npd, E, N = v.fe_n_dof, v.pd_n_dof, v.n_elems, v.n_nodes
        return {
            "labels": _arr(v.labels, i32, E), "alpha": _arr(v.alpha, f64, E),
            "fe_node_dof": _arr(v.fe_node_dof, i32, N), "pd_node_dof": _arr(v.pd_node_dof, i32, N),
            "fe_k_rowptr": _arr(v.fe_k_rowptr, i32, nf + 1), "fe_k_col": _arr(v.fe_k_col, i32, v.fe_nnz),
            "fe_k_val": _arr(v.fe_k_val, f64, v.fe_nnz),
            "fe_mass": _arr(v.fe_mass, f64, nf), "fe_p_ext": _arr(v.fe_p_ext, f64, nf),
            "pd_mass": _arr(v.pd_mass, f64, npd), "pd_p_ext": _arr(v.pd_p_ext, f64, npd),
            "fe_bc_dofs": _arr(v.fe_bc_dofs, i32, v.fe_n_bc), "fe_bc_vel": _arr(v.fe_bc_vel, f64, v.fe_n_bc),
            "pd_bc_dofs": _arr(v.pd_bc_dofs, i32, v.pd_n_bc), "pd_bc_vel": _arr(v.pd_bc_vel, f64, v.pd_n_bc),
            "fe_dof": _arr(v.cpl_fe_dof, i32, v.n_lambda), "pd_dof": _arr(v.cpl_pd_dof, i32, v.n_lambda),
            "pairs": _arr(v.pairs, i32, 2 * v.n_pairs, (v.n_pairs, 2)),
            "pe_weight": _arr(v.pe_weight, f64, v.n_pairs),
            "delta": v.delta, "c0": v.c0, "l": v.l, "char_length": v.char_length,
            "load_ramp": v.load_ramp,
            "node_xyz": _arr(v.node_xyz, f64, 3 * N, (N, 3)),
            "elem_nodes": _arr(v.elem_nodes, i32, E * (4 if v.dim == 2 else 8),
                               (E, 4 if v.dim == 2 else 8)),
            "node_alpha": _arr(v.node_alpha, f64, N),
            "cpl_fe_rowptr": _arr(v.cpl_fe_rowptr, i32, v.n_lambda + 1),
            "cpl_fe_col": _arr(v.cpl_fe_col, i32, v.cpl_fe_nnz),
            "cpl_fe_w": _arr(v.cpl_fe_w, f64, v.cpl_fe_nnz),
            "fe_mesh_elems": v.fe_mesh_elems, "fe_mesh_nodes": v.fe_mesh_nodes,
            "pd_linear_lattice": bool(v.pd_linear_lattice),
        }

    # -- integration --------------------------------------------------------
    def initialize(self):
        check(lib().pmts_mts_init(self.h))

    def macro_step(self, n: int = 1) -> list[dict]:
        reps = (capi.MtsReport * max(n, 1))()
        check(lib().pmts_mts_macro_step(self.h, n, reps))
        return [{f: getattr(r, f) for f, _ in capi.MtsReport._fields_} for r in reps[:n]]

    def macro_step_timed(self, n: int) -> float:
        ms = C.c_float()
        check(lib().pmts_mts_macro_step_timed(self.h, n, C.byref(ms)))
        return ms.value

    def state(self, which: str):
        """(u, v, a) of the FE or PD subdomain; a PD shard returns its local dofs
        (self.pd_local_dofs order)."""
        n = self.fe_n_dof if which == "fe" else len(self.pd_local_dofs)
        u, v, a = np.empty(n), np.empty(n), np.empty(n)
        check(lib().pmts_mts_get_state(self.h, 0 if which == "fe" else 1, ptr(u), ptr(v), ptr(a)))
        return u, v, a

    def lam(self):
        out = np.empty(self.n_lambda)
        check(lib().pmts_mts_get_lambda(self.h, ptr(out)))
        return out

    def intact(self):
        out = np.empty(self.n_pairs, dtype=np.uint8)
        check(lib().pmts_mts_get_intact(self.h, ptr(out)))
        return out

    def damage_field(self):
        """damage_field over the whole mesh (element, node)."""
        e = np.empty(self.n_elems)
        n = np.empty(self.n_nodes)
        check(lib().pmts_mts_damage(self.h, ptr(e), ptr(n)))
        return e, n



class ShardGroup:
    """The PD shards of one coupled run driven from one process: one
    handle per shard on `devices` (all on one GPU by default -- the shards exchange
    through device copies at host barriers, no kernel waits on another), stepped
    together; the assembled outputs compare one-to-one with a single-domain MtsSolver."""

    def __init__(self, sc: dict, world: int, devices=None):
        devices = list(devices or [0] * world)
        self.world = world
        self.shards = [MtsSolver(sc, device=devices[r], shard=(r, world)) for r in range(world)]
        self._arr = (C.c_void_p * world)(*[s.h.value for s in self.shards])
        check(lib().pmts_mts_group_join(self._arr, world))
        r0 = self.shards[0]
        self.dim, self.fe_n_dof, self.pd_n_dof = r0.dim, r0.fe_n_dof, r0.pd_n_dof
        self.n_lambda, self.n_elems, self.n_nodes = r0.n_lambda, r0.n_elems, r0.n_nodes

    def initialize(self):
        check(lib().pmts_mts_group_init(self._arr, self.world))

    def macro_step(self, n: int = 1) -> list[dict]:
        reps = (capi.MtsReport * max(n, 1))()
        check(lib().pmts_mts_group_macro_step(self._arr, self.world, n, reps))
        return [{f: getattr(r, f) for f, _ in capi.MtsReport._fields_} for r in reps[:n]]

    def state(self, which: str):
        if which == "fe":
            return self.shards[0].state("fe")
        out = [np.full(self.pd_n_dof, np.nan) for _ in range(3)]
        for s in self.shards:
            own = np.repeat(s.shard["node_owned"], self.dim)
            dofs = s.pd_local_dofs[own]
            for o, x in zip(out, s.state("pd")):
                o[dofs] = x[own]
        return tuple(out)

    def lam(self):
        return self.shards[0].lam()

    def pairs_intact(self):
        """{(i, j): intact} over every bond, each taken from the shard owning i."""
        out = {}
        for s in self.shards:
            sy = s.system()
            lo, hi = s.shard["own_elems"]
            le = s.shard["local_elems"]
            # local element index of each pair's first element (global ids -> PD-active)
            pa = np.flatnonzero(sy["labels"] != 0)  # PD-active elements, ascending
            g2l = {int(pa[e]): k for k, e in enumerate(le)}
            it = s.intact()
            for (i, j), v in zip(sy["pairs"], it):
                k = g2l[int(i)]
                if lo <= k < hi:
                    out[(int(i), int(j))] = int(v)
        return out

    def damage_field(self):
        e = np.zeros(self.n_elems)
        n = np.zeros(self.n_nodes)
        for s in self.shards:
            de, dn = s.damage_field()
            e += de
            n += dn
        return e, n
