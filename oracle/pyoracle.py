"""ORACLE / TEST INFRASTRUCTURE ONLY -- ctypes view of oracle/_build/libpd_oracle.so.

Imported only by tests/, bench.py's cpu_baseline leg and __graft_entry__.smoke(),
always as the checker.  The product path (paper_2403_03605_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libpd_oracle.so")
REF_DRIVER = os.path.join(HERE, "_ref", "ref_driver")

CSR, MF = 0, 1
MICRO_EXP, MICRO_CONST = 0, 1

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE, "restatement"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        p = C.c_void_p
        L.po_find_pairs.restype = C.c_int64
        L.po_find_pairs.argtypes = [C.c_int, C.c_int, p, p, C.c_double, C.c_int, p, p, p,
                                    C.c_int64]
        L.po_pd_create.restype = p
        L.po_pd_create.argtypes = [C.c_int, C.c_int, C.c_int, p, p, p, C.c_int64, p, p, p,
                                   C.c_int, p, p, p, p]
        L.po_pd_destroy.argtypes = [p]
        L.po_pd_init.argtypes = [p, C.c_double]
        L.po_pd_step.restype = C.c_int64
        L.po_pd_step.argtypes = [p, C.c_int, p, p, p, C.c_int64]
        L.po_pd_get_state.argtypes = [p, p, p, p]
        L.po_pd_set_state.argtypes = [p, p, p, p]
        L.po_pd_get_mu.argtypes = [p, p]
        L.po_pd_damage.argtypes = [p, p, p]
        L.po_micromodulus.restype = C.c_double
        L.po_micromodulus.argtypes = [p, C.c_double]
        L.po_bond_s_crit.restype = C.c_double
        L.po_bond_s_crit.argtypes = [C.c_double, C.c_double, C.c_uint64, C.c_int32, C.c_int32]
        L.po_bond_stretch.restype = C.c_double
        L.po_bond_stretch.argtypes = [p, C.c_int64, p]
        L.po_pd_nnz.restype = C.c_int64
        L.po_pd_nnz.argtypes = [p]
        L.po_pd_update_bond_states.restype = C.c_int64
        L.po_pd_update_bond_states.argtypes = [p, p, p, C.c_int64]
        L.po_pd_set_mu.argtypes = [p, p]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _notch_arrays(notches):
    npts = np.array([len(n) // 3 for n in notches] or [0], dtype=np.int32)
    pts = np.array([x for n in notches for x in n] or [0.0], dtype=np.float64)
    return npts, pts


def find_pairs(dim, centroid, volume, delta, notches=()):
    """notches: list of flat xyz point lists (2 points in 2D, >=3 in 3D)."""
    cen = np.ascontiguousarray(centroid, dtype=np.float64).reshape(-1, 3)
    vol = np.ascontiguousarray(volume, dtype=np.float64)
    npts, pts = _notch_arrays(notches)
    L = lib()
    n = L.po_find_pairs(dim, len(vol), _p(cen), _p(vol), delta, len(notches), _p(npts),
                        _p(pts), None, 0)
    out = np.zeros((max(n, 1), 2), dtype=np.int32)
    L.po_find_pairs(dim, len(vol), _p(cen), _p(vol), delta, len(notches), _p(npts), _p(pts),
                    _p(out), n)
    return out[:n]


def bond_s_crit(s_crit, spread, seed, i, j):
    return lib().po_bond_s_crit(s_crit, spread, seed, i, j)


class OraclePD:
    """Step loop of driver_run.hpp:216-236 on the CPU restatement."""

    def __init__(self, sysd: dict, variant=CSR):
        self.d = sysd
        dim = int(sysd["dim"])
        self.dim = dim
        self._keep = []

        def arr(name, dt):
            a = np.ascontiguousarray(sysd[name], dtype=dt)
            self._keep.append(a)
            return a

        conn = arr("conn", np.int32)
        cen = arr("centroid", np.float64)
        vol = arr("volume", np.float64)
        pairs = arr("pairs", np.int32)
        M = arr("mass", np.float64)
        P = arr("p_ext", np.float64)
        bcd = np.ascontiguousarray(sysd.get("bc_dofs", np.zeros(0)), dtype=np.int32)
        bcv = np.ascontiguousarray(sysd.get("bc_vel", np.zeros(0)), dtype=np.float64)
        self._keep += [bcd, bcv]
        prm = np.array([sysd["delta"], sysd.get("l", 1.0), sysd.get("c0", 0.0),
                        sysd.get("c_const", 0.0), sysd.get("h", 1.0), sysd.get("s_crit", 0.0),
                        sysd.get("s_crit_spread", 0.0), sysd.get("gamma", 0.5),
                        sysd.get("beta", 0.0), sysd["dt"]], dtype=np.float64)
        iprm = np.array([sysd.get("micromodulus", MICRO_EXP), sysd.get("seed", 0), variant,
                         sysd.get("global_id_offset", 0), *sysd.get("slab_plane", (0, 0))],
                        dtype=np.int64)
        self._keep += [prm, iprm]
        self.n_nodes = int(sysd["n_nodes"])
        self.n_elems = len(vol)
        self.n_pairs = len(pairs)
        self.n_dof = self.n_nodes * dim
        self.h = lib().po_pd_create(dim, self.n_nodes, self.n_elems, _p(conn), _p(cen), _p(vol),
                                    self.n_pairs, _p(pairs), _p(M), _p(P), len(bcd), _p(bcd),
                                    _p(bcv), _p(prm), _p(iprm))

    def __del__(self):
        if getattr(self, "h", None):
            lib().po_pd_destroy(self.h)
            self.h = None

    def init(self, scale0):
        lib().po_pd_init(self.h, float(scale0))

    def step(self, scales, cap=None):
        sc = np.ascontiguousarray(scales, dtype=np.float64)
        cap = self.n_pairs if cap is None else cap
        out = np.zeros(max(cap, 1), dtype=np.int32)
        st = np.zeros(max(cap, 1), dtype=np.int32)
        n = lib().po_pd_step(self.h, len(sc), _p(sc), _p(out), _p(st), cap)
        return out[:min(n, cap)].copy(), st[:min(n, cap)].copy()

    def state(self):
        u = np.zeros(self.n_dof)
        v = np.zeros(self.n_dof)
        a = np.zeros(self.n_dof)
        lib().po_pd_get_state(self.h, _p(u), _p(v), _p(a))
        return u, v, a

    def set_state(self, u, v, a):
        u, v, a = (np.ascontiguousarray(x, dtype=np.float64) for x in (u, v, a))
        lib().po_pd_set_state(self.h, _p(u), _p(v), _p(a))

    def mu(self):
        m = np.zeros(max(self.n_pairs, 1), dtype=np.uint8)
        lib().po_pd_get_mu(self.h, _p(m))
        return m[:self.n_pairs]

    def damage(self):
        e = np.zeros(self.n_elems)
        n = np.zeros(self.n_nodes)
        lib().po_pd_damage(self.h, _p(e), _p(n))
        return e, n

    def stretch(self, pair, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        return lib().po_bond_stretch(self.h, int(pair), _p(u))

    def nnz(self):
        return lib().po_pd_nnz(self.h)

    def update_bond_states(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.zeros(max(self.n_pairs, 1), dtype=np.int32)
        n = lib().po_pd_update_bond_states(self.h, _p(u), _p(out), self.n_pairs)
        return out[:n].copy()

    def set_mu(self, mu):
        m = np.ascontiguousarray(mu, dtype=np.uint8)
        lib().po_pd_set_mu(self.h, _p(m))


def load_ref_dump(d: str) -> dict:
    """Read a ref_driver --dump directory into a dict of numpy arrays."""
    meta = {}
    with open(os.path.join(d, "meta.txt")) as f:
        for line in f:
            k, v = line.split()
            meta[k] = float(v)
    out = dict(meta)
    dim = int(meta["dim"])
    out["dim"] = dim
    out["n_nodes"] = int(meta["n_nodes"])

    def rd(name, dt, shape=None):
        p = os.path.join(d, name)
        if not os.path.exists(p):
            return None
        a = np.fromfile(p, dtype=dt)
        return a.reshape(shape) if shape else a

    nn = 4 if dim == 2 else 8
    out["nodes"] = rd("nodes.f64", np.float64, (-1, 3))
    out["conn"] = rd("conn.i32", np.int32, (-1, nn))
    out["centroid"] = rd("centroid.f64", np.float64, (-1, 3))
    out["volume"] = rd("volume.f64", np.float64)
    out["pairs"] = rd("pairs.i32", np.int32, (-1, 2))
    out["xi_norm"] = rd("xi_norm.f64", np.float64)
    out["weight"] = rd("weight.f64", np.float64)
    out["mass"] = rd("mass.f64", np.float64)
    out["p_ext"] = rd("p_ext.f64", np.float64)
    out["bc_dofs"] = rd("bc_dofs.i32", np.int32)
    out["bc_vel"] = rd("bc_vel.f64", np.float64)
    out["a0"] = rd("a0.f64", np.float64)
    out["scale"] = rd("scale.f64", np.float64)
    for k in ("u", "v", "a", "damage_elem", "damage_node"):
        out[k] = rd(k + ".f64", np.float64)
    b = rd("broken.i32", np.int32)
    out["broken"] = b.reshape(-1, 2) if b is not None else None
    for name in os.listdir(d):
        if name.startswith(("u_", "v_", "a_")) and name.endswith(".f64"):
            out[name[:-4]] = rd(name, np.float64)
    return out


def run_ref(cfg_text: str, workdir: str, steps=None, dump=True, checkpoints=(), extra=(),
            env=None) -> dict:
    """Run oracle/_ref/ref_driver (the reference's own loop) on a config text."""
    import json
    os.makedirs(workdir, exist_ok=True)
    cfg = os.path.join(workdir, "scenario.cfg")
    with open(cfg, "w") as f:
        f.write(cfg_text)
    cmd = [REF_DRIVER, cfg]
    if steps is not None:
        cmd += ["--steps", str(steps)]
    if dump:
        cmd += ["--dump", workdir]
    if checkpoints:
        cmd += ["--checkpoints", ",".join(str(c) for c in checkpoints)]
    cmd += list(extra)
    r = subprocess.run(cmd, check=True, capture_output=True, text=True, env=env)
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    return json.loads(line)


REF_MTS_DRIVER = os.path.join(os.path.dirname(REF_DRIVER), "ref_mts_driver")

_MTS_FILES = {
    "labels": np.int32, "alpha": np.float64, "fe_node_dof": np.int32, "pd_node_dof": np.int32,
    "fe_k_rowptr": np.int32, "fe_k_col": np.int32, "fe_k_val": np.float64,
    "fe_mass": np.float64, "fe_p_ext": np.float64, "pd_k_rowptr": np.int32,
    "pd_k_col": np.int32, "pd_k_val": np.float64, "pd_mass": np.float64, "pd_p_ext": np.float64,
    "pairs": np.int32, "pe_weight": np.float64, "fe_bc_dofs": np.int32, "fe_bc_vel": np.float64,
    "pd_bc_dofs": np.int32, "pd_bc_vel": np.float64, "fe_dof": np.int32, "pd_dof": np.int32,
    "scale": np.float64, "lambda": np.float64, "broken": np.int32, "continuity": np.float64,
    "energy": np.float64, "iterations": np.int32,
}


def run_ref_mts(cfg_text: str, workdir: str, steps=None, dump=True, checkpoints=(), extra=(),
                env=None) -> dict:
    """Run oracle/_ref/ref_mts_driver (the reference's own coupled loop)."""
    import json
    os.makedirs(workdir, exist_ok=True)
    cfg = os.path.join(workdir, "scenario.cfg")
    with open(cfg, "w") as f:
        f.write(cfg_text)
    cmd = [REF_MTS_DRIVER, cfg]
    if steps is not None:
        cmd += ["--steps", str(steps)]
    if dump:
        cmd += ["--dump", workdir]
    if checkpoints:
        cmd += ["--checkpoints", ",".join(str(c) for c in checkpoints)]
    cmd += list(extra)
    r = subprocess.run(cmd, check=True, capture_output=True, text=True, env=env)
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    return json.loads(line)


def load_ref_mts_dump(d: str) -> dict:
    """Arrays written by ref_mts_driver --dump (see oracle/ref_mts_driver.cpp)."""
    out = {}
    for name, dt in _MTS_FILES.items():
        p = os.path.join(d, name + (".i32" if dt == np.int32 else ".f64"))
        if os.path.exists(p):
            out[name] = np.fromfile(p, dtype=dt)
    out["pairs"] = out["pairs"].reshape(-1, 2)
    out["broken"] = out["broken"].reshape(-1, 2)
    out["energy"] = out["energy"].reshape(-1, 4)
    for f in os.listdir(d):
        if f.endswith(".f64") and f.split("_")[0] in ("fe", "pd", "fe0", "pd0", "lambda"):
            key = f[:-4]
            if key not in out:
                out[key] = np.fromfile(os.path.join(d, f), dtype=np.float64)
    with open(os.path.join(d, "meta.txt")) as fh:
        for line in fh:
            k, v = line.split()
            out[k] = float(v) if "." in v or "e" in v else int(v)
    return out

