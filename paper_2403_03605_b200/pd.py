"""Host-side mirror of the reference's pure-PD interface, over the C ABI.

Reference call sites this stands in for (
/root/reference/proj/include/perimts/):
  build_scenario            driver.hpp:170-231       -> Scenario
  find_pe_pairs             mesh.hpp:416-495         -> PDSolver.find_pe_pairs
  initial_acceleration      newmark.hpp:110-116      -> PDSolver.initial_acceleration
  advance_dynamic_step +
  update_bond_states +
  incremental_stiffness_update (driver_run.hpp:216-236) -> PDSolver.step
  damage_field              perifem.hpp:202-231      -> PDSolver.damage_field
  run_built (pure-PD loop)  driver_run.hpp:160-246   -> PDSolver.run
Every call runs on the GPU through libpmts.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import capi
from .capi import check, lib, ptr

_FORMULATION = {"plane_stress": 0, "plane_strain": 1, "three_d": 2, "3d": 2}


def _boxes(values, n_per):
    a = np.ascontiguousarray(np.array(values, dtype=np.float64).reshape(-1, n_per))
    return a


def _box3(v, dim, nvals):
    """config box (lo per axis, hi per axis, then nvals values) -> lo[3] hi[3] vals."""
    lo = list(v[:dim]) + [0.0] * (3 - dim)
    hi = list(v[dim:2 * dim]) + [0.0] * (3 - dim)
    vals = list(v[2 * dim:2 * dim + nvals])
    if dim == 2:  # z extent of a 2D box is irrelevant (BoundsBox::contains loops k < dim)
        lo[2], hi[2] = 0.0, 0.0
    return lo + hi, vals


def _splitmix64(x: int) -> int:
    m = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & m
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & m
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & m
    return x ^ (x >> 31)


def _hash_factor(i: int, j: int, seed: int, spread: float) -> float:
    """U[1 - spread, 1 + spread] from the counter hash of (i, j, seed) -- the same
    construction as the per-bond s0 factor (pd_common.cuh bond_s_crit)."""
    if spread == 0.0:
        return 1.0
    key = ((i & 0xFFFFFFFF) << 32) | (j & 0xFFFFFFFF)
    h = _splitmix64(seed ^ _splitmix64(key))
    u = (h >> 11) * 2.0 ** -53
    return (1.0 - spread) + (2.0 * spread) * u


def scenario_desc(sc: dict, keep: list) -> "capi.ScenarioDesc":
    """pmts_scenario_desc of a scenario dict (reference config vocabulary); the
    arrays it points into are appended to keep (the caller holds them)."""
    m, mat, pdc, load, tm = sc["mesh"], sc["material"], sc["pd"], sc.get("load", {}), sc["time"]
    dim = int(m["dim"])
    d = capi.ScenarioDesc()
    d.dim = dim
    b = m["bounds"]
    for k in range(3):
        d.lo[k] = b[k] if k < dim else 0.0
        d.hi[k] = b[dim + k] if k < dim else 0.0
    d.spacing = m["spacing"]
    d.E, d.nu, d.rho = mat["E"], mat["nu"], mat["rho"]
    d.formulation = _FORMULATION[mat["formulation"]]
    d.delta_factor, d.l_factor = pdc["delta_factor"], pdc["l_factor"]
    d.s_crit = pdc.get("s_crit", 0.0)
    notches = [v for k, v in sorted(m.items()) if k.startswith("notch") and v]
    npts, pts = [], []
    for v in notches:
        if len(v) == 4:
            npts.append(2)
            pts += [v[0], v[1], 0.0, v[2], v[3], 0.0]
        else:
            npts.append(len(v) // 3)
            pts += list(v)
    notch_npts = np.array(npts or [0], dtype=np.int32)
    notch_pts = np.array(pts or [0.0], dtype=np.float64)
    d.n_notch = len(npts)
    d.notch_npts, d.notch_pts = ptr(notch_npts), ptr(notch_pts)
    trac, bodyp, vel, fixed = [], [], [], []
    for k, v in sorted(load.items()):
        if k.startswith("traction"):
            bx, val = _box3(v, dim, dim)
            trac.append(bx + val + [0.0] * (3 - dim))
        elif k.startswith("body_patch"):
            bx, val = _box3(v, dim, dim)
            bodyp.append(bx + val + [0.0] * (3 - dim))
        elif k.startswith("velocity_bc"):
            bx, val = _box3(v, dim, 2)
            vel.append(bx + val)
        elif k.startswith("fixed"):
            bx, _ = _box3(v, dim, 0)
            fixed.append(bx)
    trac_a = np.array(trac or [[0.0] * 9], dtype=np.float64)
    bodyp_a = np.array(bodyp or [[0.0] * 9], dtype=np.float64)
    vel_a = np.array(vel or [[0.0] * 8], dtype=np.float64)
    fixed_a = np.array(fixed or [[0.0] * 6], dtype=np.float64)
    d.n_traction, d.traction = len(trac), ptr(trac_a)
    d.n_body_patch, d.body_patch = len(bodyp), ptr(bodyp_a)
    bf = load.get("body_force", [0.0] * dim)
    for k in range(3):
        d.body_force[k] = bf[k] if k < dim else 0.0
    d.n_velocity_bc, d.velocity_bc = len(vel), ptr(vel_a)
    d.n_fixed, d.fixed = len(fixed), ptr(fixed_a)
    d.dt_pd, d.m, d.total_time = tm["dt_pd"], int(tm.get("m", 1)), tm["total_time"]
    ramp = load.get("load_ramp", "auto")
    d.load_ramp = -1.0 if ramp in (None, "auto") else float(ramp)
    d.gamma, d.beta = tm.get("gamma_pd", 0.5), tm.get("beta_pd", 0.0)
    keep += [notch_npts, notch_pts, trac_a, bodyp_a, vel_a, fixed_a]
    return d


class Scenario:
    """build_scenario for a generated pure-PD run (host C++ setup in libpmts)."""

    def __init__(self, sc: dict, host_setup: bool = False):
        self.cfg = sc
        self._keep = []
        d = scenario_desc(sc, self._keep)
        d.host_setup = 1 if host_setup else 0
        self.notch_npts, self.notch_pts = self._keep[0], self._keep[1]
        h = C.c_void_p()
        check(lib().pmts_scenario_build(C.byref(d), C.byref(h)))
        self.h = h
        v = capi.ScenarioView()
        check(lib().pmts_scenario_get(h, C.byref(v)))
        self.view = v
        self.dim, self.n_nodes, self.n_elems = v.dim, v.n_nodes, v.n_elems
        self.n_dof, self.n_steps = v.n_dof, v.n_steps
        self.lattice = tuple(v.lattice)
        self.delta, self.l, self.c0 = v.delta, v.l, v.c0
        self.char_length, self.dt, self.gamma, self.beta = v.char_length, v.dt, v.gamma, v.beta
        self.s_crit, self.load_ramp = v.s_crit, v.load_ramp
        nn = 4 if self.dim == 2 else 8

        def view(p, ctype, n, shape=None):
            if n == 0:
                return np.zeros(0, dtype=np.dtype(ctype))
            a = np.ctypeslib.as_array(C.cast(p, C.POINTER(ctype)), shape=(n,)).copy()
            return a.reshape(shape) if shape else a

        self.nodes = view(v.node_xyz, C.c_double, 3 * self.n_nodes, (-1, 3))
        self.conn = view(v.elem_nodes, C.c_int32, nn * self.n_elems, (-1, nn))
        self.centroid = view(v.centroid, C.c_double, 3 * self.n_elems, (-1, 3))
        self.volume = view(v.volume, C.c_double, self.n_elems)
        self.mass = view(v.mass, C.c_double, self.n_dof)
        self.p_ext = view(v.p_ext, C.c_double, self.n_dof)
        self.bc_dofs = view(v.bc_dofs, C.c_int32, v.n_bc)
        self.bc_vel = view(v.bc_vel, C.c_double, v.n_bc)

    def __del__(self):
        if getattr(self, "h", None):
            lib().pmts_scenario_destroy(self.h)
            self.h = None

    def load_scale(self, t: float) -> float:
        return lib().pmts_scenario_load_scale(self.h, t)

    def scales(self, first_step: int, n: int) -> np.ndarray:
        """load_scale(i dt) for i = first_step .. first_step + n - 1 (driver_run.hpp:220)."""
        return np.array([self.load_scale(i * self.dt) for i in range(first_step, first_step + n)])

    def initial_velocity(self) -> np.ndarray:
        """BASELINE cfg4 extension: seeded velocity on a face patch (the reference has no
        initial-velocity hook; its velocity BCs are re-imposed every step).  Per node in
        the box: value * U[1 - spread, 1 + spread] from the same counter hash as the
        per-bond s0 factor, keyed by (node id, component, seed)."""
        v = np.zeros(self.n_dof)
        iv = self.cfg.get("ext", {}).get("initial_velocity")
        if not iv:
            return v
        lo, hi = np.array(iv["lo"]), np.array(iv["hi"])
        d = self.dim
        inside = np.all((self.nodes[:, :d] >= lo[:d]) & (self.nodes[:, :d] <= hi[:d]), axis=1)
        ids = np.nonzero(inside)[0]
        spread, seed = float(iv.get("spread", 0.0)), int(iv.get("seed", 0))
        fac = np.array([_hash_factor(int(n), int(iv["comp"]), seed, spread) for n in ids])
        v[ids * d + int(iv["comp"])] = float(iv["value"]) * fac
        return v

    def notches(self):
        out, k = [], 0
        for n in self.notch_npts[: len(self.notch_npts) if self.notch_npts[0] else 0]:
            out.append(list(self.notch_pts[3 * k:3 * (k + n)]))
            k += n
        return out


class PDSolver:
    """One device-resident PD fine-step handle (pmts_pd)."""

    def __init__(self, *, dim, nodes, conn, mass, p_ext, delta, dt, bc_dofs=None, bc_vel=None,
                 micromodulus=capi.MICRO_EXP, c0=0.0, l=1.0, c_const=0.0, h=1.0, s_crit=0.0,
                 s_crit_spread=0.0, seed=0, gamma=0.5, beta=0.0, mode=capi.DETERMINISTIC,
                 device=0, notch_npts=None, notch_pts=None, lattice=(0, 0, 0),
                 global_id_offset=0, owned_elems=(0, 0), lattice_h=0.0, lattice_vol=0.0,
                 slab_plane=(0, 0), node_rows=(0, 0)):
        self.dim = dim
        self._nodes = np.ascontiguousarray(nodes, dtype=np.float64).reshape(-1, 3)
        self._conn = np.ascontiguousarray(conn, dtype=np.int32)
        self._mass = np.ascontiguousarray(mass, dtype=np.float64)
        self._p = np.ascontiguousarray(p_ext, dtype=np.float64)
        self._bcd = np.ascontiguousarray(bc_dofs if bc_dofs is not None else [], dtype=np.int32)
        self._bcv = np.ascontiguousarray(bc_vel if bc_vel is not None else [], dtype=np.float64)
        self._npts = np.ascontiguousarray(notch_npts if notch_npts is not None else [0],
                                          dtype=np.int32)
        self._pts = np.ascontiguousarray(notch_pts if notch_pts is not None else [0.0],
                                         dtype=np.float64)
        n_notch = 0 if notch_npts is None else len(notch_npts)
        d = capi.PDDesc()
        d.dim = dim
        d.n_nodes = len(self._nodes)
        d.n_elems = len(self._conn)
        d.node_xyz, d.elem_nodes = ptr(self._nodes), ptr(self._conn)
        d.mass, d.p_ext = ptr(self._mass), ptr(self._p)
        d.n_bc, d.bc_dofs, d.bc_vel = len(self._bcd), ptr(self._bcd), ptr(self._bcv)
        d.delta, d.micromodulus, d.c0, d.l = delta, micromodulus, c0, l
        d.c_const, d.h = c_const, h
        d.s_crit, d.s_crit_spread, d.seed = s_crit, s_crit_spread, seed
        d.gamma, d.beta, d.dt = gamma, beta, dt
        d.mode, d.device = mode, device
        d.n_notch, d.notch_npts, d.notch_pts = n_notch, ptr(self._npts), ptr(self._pts)
        for k in range(3):
            d.lattice[k] = lattice[k]
        d.global_id_offset = int(global_id_offset)
        d.owned_elems[0], d.owned_elems[1] = int(owned_elems[0]), int(owned_elems[1])
        d.lattice_h, d.lattice_vol = float(lattice_h), float(lattice_vol)
        d.slab_plane[0], d.slab_plane[1] = int(slab_plane[0]), int(slab_plane[1])
        d.node_rows[0], d.node_rows[1] = int(node_rows[0]), int(node_rows[1])
        self.n_nodes, self.n_elems = d.n_nodes, d.n_elems
        self.n_dof = self.n_nodes * dim
        self.mode = mode
        hh = C.c_void_p()
        check(lib().pmts_pd_create(C.byref(d), C.byref(hh)))
        self.h = hh

    @classmethod
    def from_scenario(cls, sc: Scenario, mode=capi.DETERMINISTIC, device=0, **over):
        ext = sc.cfg.get("ext", {})
        kw = dict(dim=sc.dim, nodes=sc.nodes, conn=sc.conn, mass=sc.mass, p_ext=sc.p_ext,
                  delta=sc.delta, dt=sc.dt, bc_dofs=sc.bc_dofs, bc_vel=sc.bc_vel,
                  c0=sc.c0, l=sc.l, s_crit=sc.s_crit, gamma=sc.gamma, beta=sc.beta,
                  mode=mode, device=device, lattice=sc.lattice)
        if sc.notch_npts[0] if len(sc.notch_npts) else 0:
            kw["notch_npts"] = sc.notch_npts
            kw["notch_pts"] = sc.notch_pts
        if ext.get("micromodulus") == "constant":
            kw.update(micromodulus=capi.MICRO_CONST, c_const=ext["c"], h=ext.get("h", 1.0))
        if ext.get("s_crit_spread"):
            kw.update(s_crit_spread=ext["s_crit_spread"], seed=int(ext.get("seed", 0)))
        if any(sc.lattice):  # nominal stencil constants: same table as any slab run
            kw.update(lattice_h=float(sc.nodes[1, 0] - sc.nodes[0, 0]),
                      lattice_vol=float(sc.volume[0]))
        kw.update(over)
        s = cls(**kw)
        s.scenario = sc
        return s

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib().pmts_nccl_unique_id(buf))
        return buf.raw

    def __del__(self):
        if getattr(self, "h", None):
            lib().pmts_pd_destroy(self.h)
            self.h = None

    # -- families ---------------------------------------------------------
    def find_pe_pairs(self):
        check(lib().pmts_pd_build_families(self.h))
        return self

    def set_pairs(self, pairs):
        p = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 2)
        check(lib().pmts_pd_set_pairs(self.h, len(p), ptr(p)))
        return self

    def pairs(self) -> np.ndarray:
        n = C.c_int64()
        check(lib().pmts_pd_get_pairs(self.h, None, 0, C.byref(n)))
        out = np.zeros((max(n.value, 1), 2), dtype=np.int32)
        check(lib().pmts_pd_get_pairs(self.h, ptr(out), n.value, C.byref(n)))
        return out[: n.value]

    def info(self) -> dict:
        i = capi.PDInfo()
        check(lib().pmts_pd_info_get(self.h, C.byref(i)))
        return {f: getattr(i, f) for f, _ in i._fields_}

    # -- stepping ---------------------------------------------------------
    def initial_acceleration(self, scale0: float):
        check(lib().pmts_pd_init(self.h, float(scale0)))

    def step(self, scales) -> int:
        s = np.ascontiguousarray(scales, dtype=np.float64)
        nb = C.c_int64()
        check(lib().pmts_pd_step(self.h, len(s), ptr(s), C.byref(nb)))
        return nb.value

    def step_tracked(self, scales, dofs, out=None, broken=None):
        """Steps + per-step tracked displacements and broken counts (one sync)."""
        s = np.ascontiguousarray(scales, dtype=np.float64)
        d = np.ascontiguousarray(dofs, dtype=np.int32)
        if out is None:
            out = np.zeros((len(s), len(d)))
        if broken is None:
            broken = np.zeros(len(s), dtype=np.int64)
        check(lib().pmts_pd_step_tracked(self.h, len(s), ptr(s), len(d), ptr(d), ptr(out),
                                         ptr(broken)))
        return out, broken

    def step_timed(self, scales) -> float:
        s = np.ascontiguousarray(scales, dtype=np.float64)
        ms = C.c_float()
        check(lib().pmts_pd_step_timed(self.h, len(s), ptr(s), C.byref(ms)))
        return ms.value

    def profile(self, scales):
        s = np.ascontiguousarray(scales, dtype=np.float64)
        b, t = C.c_float(), C.c_float()
        check(lib().pmts_pd_profile(self.h, len(s), ptr(s), C.byref(b), C.byref(t)))
        return b.value, t.value

    # -- state ------------------------------------------------------------
    def state(self):
        u, v, a = (np.zeros(self.n_dof) for _ in range(3))
        check(lib().pmts_pd_get_state(self.h, ptr(u), ptr(v), ptr(a)))
        return u, v, a

    def get_state_into(self, u, v, a):
        """get_state into caller-owned (e.g. pinned) float64 buffers."""
        check(lib().pmts_pd_get_state(self.h, ptr(u), ptr(v), ptr(a)))

    def set_state(self, u=None, v=None, a=None):
        arrs = [None if x is None else np.ascontiguousarray(x, dtype=np.float64) for x in (u, v, a)]
        check(lib().pmts_pd_set_state(self.h, *(ptr(x) for x in arrs)))

    def intact(self) -> np.ndarray:
        n = C.c_int64()
        check(lib().pmts_pd_get_pairs(self.h, None, 0, C.byref(n)))
        out = np.zeros(max(n.value, 1), dtype=np.uint8)
        check(lib().pmts_pd_get_intact(self.h, ptr(out), n.value))
        return out[: n.value]

    def break_log(self, cap: int) -> np.ndarray:
        out = np.zeros((max(cap, 1), 3), dtype=np.int32)
        n = C.c_int64()
        check(lib().pmts_pd_take_break_log(self.h, ptr(out), cap, C.byref(n)))
        if n.value > cap:
            raise capi.PmtsError(f"break log holds {n.value} rows > cap {cap}")
        return out[: n.value]

    def broken_total(self) -> int:
        return lib().pmts_pd_broken_total(self.h)

    def damage_field(self):
        e = np.zeros(self.n_elems)
        n = np.zeros(self.n_nodes)
        check(lib().pmts_pd_damage(self.h, ptr(e), ptr(n)))
        return e, n

    def gather_disp(self, dofs) -> np.ndarray:
        d = np.ascontiguousarray(dofs, dtype=np.int32)
        out = np.zeros(len(d))
        check(lib().pmts_pd_gather_disp(self.h, len(d), ptr(d), ptr(out)))
        return out

    # -- slab decomposition ---------------------------------------------------
    def get_rows(self, first, n, layers=1, stride=0) -> np.ndarray:
        out = np.zeros(n * self.dim * layers)
        check(lib().pmts_pd_get_rows_layers(self.h, first, n, layers, stride, ptr(out)))
        return out

    def set_rows(self, first, n, vals, layers=1, stride=0):
        v = np.ascontiguousarray(vals, dtype=np.float64)
        assert v.size == n * self.dim * layers
        check(lib().pmts_pd_set_rows_layers(self.h, first, n, layers, stride, ptr(v)))

    def set_option(self, option: int, value: int):
        """pmts_pd_set_option (capi.OPT_*): results are bitwise unchanged."""
        check(lib().pmts_pd_set_option(self.h, int(option), int(value)))
        return self

    # -- coupled-integrator hooks (deterministic mode) ------------------------
    def set_constraint_load(self, dofs, vals):
        """G_PD^T S_j (mts.hpp:160-162): added to P * load_scale until replaced."""
        d = np.ascontiguousarray(dofs, dtype=np.int32)
        v = np.ascontiguousarray(vals, dtype=np.float64)
        check(lib().pmts_pd_set_constraint_load(self.h, len(d), ptr(d), ptr(v)))

    def snapshot_bonds(self):
        check(lib().pmts_pd_snapshot_bonds(self.h))

    def homogeneous_recursion(self, m, dofs, w, state=False):
        """The m homogeneous linear substeps from rest on the bond snapshot
        (mts.hpp:230-238, 398-420): velocities at dofs after each substep, (m+1) x n."""
        d = np.ascontiguousarray(dofs, dtype=np.int32)
        w = np.ascontiguousarray(w, dtype=np.float64)
        vel = np.zeros((m + 1, len(d)))
        u, v, a = (np.zeros(self.n_dof) for _ in range(3)) if state else (None, None, None)
        check(lib().pmts_pd_homogeneous_recursion(self.h, m, len(d), ptr(d), ptr(w), ptr(vel),
                                                  ptr(u), ptr(v), ptr(a)))
        return (vel, (u, v, a)) if state else vel

    def set_halo_layers(self, layers, stride):
        check(lib().pmts_pd_set_halo_layers(self.h, layers, stride))

    def comm_init(self, uid: bytes, nranks: int, rank: int):
        buf = C.create_string_buffer(uid, 128)
        check(lib().pmts_pd_comm_init(self.h, buf, nranks, rank))

    def set_halo(self, peer_lo, send_lo, recv_lo, n_lo, peer_hi, send_hi, recv_hi, n_hi):
        check(lib().pmts_pd_set_halo(self.h, peer_lo, send_lo, recv_lo, n_lo, peer_hi,
                                     send_hi, recv_hi, n_hi))

    def allreduce_sum(self, v: int) -> int:
        x = C.c_int64(v)
        check(lib().pmts_pd_allreduce_sum(self.h, C.byref(x)))
        return x.value

    # -- run_built's pure-PD loop ------------------------------------------
    def run(self, n_steps=None, batch=100):
        """driver_run.hpp:199-245 (minus file output): returns per-step broken counts."""
        sc = self.scenario
        n_steps = sc.n_steps if n_steps is None else n_steps
        v0 = sc.initial_velocity()
        if v0.any():
            z = np.zeros(self.n_dof)
            self.set_state(z, v0, z)
        self.initial_acceleration(sc.load_scale(0.0))
        broken = []
        i = 1
        while i <= n_steps:
            k = min(batch, n_steps - i + 1)
            broken.append(self.step(sc.scales(i, k)))
            i += k
        return broken
