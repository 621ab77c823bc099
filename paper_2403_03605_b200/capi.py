"""ctypes binding of include/pmts_capi.h (libpmts.so, built in-tree for sm_100a).

This is the Python side of the C-ABI boundary: the structs mirror the header
field for field, every call returns the header's status code and a failed call
raises the exception class the reference would have thrown (errors.hpp:8-21).
There is no fallback: if the library is missing, importing this module fails.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PMTS_LIB_PATH") or os.path.join(HERE, "lib", "libpmts.so")

PMTS_OK, PMTS_ERR_INTERNAL, PMTS_ERR_CONFIG, PMTS_ERR_SOLVER = 0, 1, 2, 3
DETERMINISTIC, FAST, FAST_F32POS = 0, 1, 2
MICRO_EXP, MICRO_CONST = 0, 1
OPT_BREAK_SCREEN, OPT_HALO_OVERLAP, OPT_COUNT_HOT, OPT_CLEAN_TILES = 1, 2, 3, 4


class PmtsError(RuntimeError):
    """InternalError / CUDA failure (status 1)."""


class ConfigError(PmtsError):
    """ConfigError (status 2)."""


class SolverError(PmtsError):
    """SolverError (status 3)."""


_P = C.c_void_p
_D = C.c_double
_I = C.c_int32


class ScenarioDesc(C.Structure):
    _fields_ = [("dim", _I), ("lo", _D * 3), ("hi", _D * 3), ("spacing", _D), ("E", _D),
                ("nu", _D), ("rho", _D), ("formulation", _I), ("delta_factor", _D),
                ("l_factor", _D), ("s_crit", _D), ("n_notch", _I), ("notch_npts", _P),
                ("notch_pts", _P), ("n_traction", _I), ("traction", _P),
                ("n_body_patch", _I), ("body_patch", _P), ("body_force", _D * 3),
                ("n_velocity_bc", _I), ("velocity_bc", _P), ("n_fixed", _I), ("fixed", _P),
                ("dt_pd", _D), ("m", _I), ("total_time", _D), ("load_ramp", _D),
                ("gamma", _D), ("beta", _D), ("host_setup", _I)]


class ScenarioView(C.Structure):
    _fields_ = [("dim", _I), ("n_nodes", _I), ("n_elems", _I), ("n_dof", _I), ("n_bc", _I),
                ("n_steps", _I), ("lattice", _I * 3), ("delta", _D), ("l", _D), ("c0", _D),
                ("char_length", _D), ("dt", _D), ("gamma", _D), ("beta", _D), ("s_crit", _D),
                ("load_ramp", _D), ("node_xyz", _P), ("elem_nodes", _P), ("centroid", _P),
                ("volume", _P), ("mass", _P), ("p_ext", _P), ("bc_dofs", _P), ("bc_vel", _P)]


class PDDesc(C.Structure):
    _fields_ = [("dim", _I), ("n_nodes", _I), ("n_elems", _I), ("node_xyz", _P),
                ("elem_nodes", _P), ("mass", _P), ("p_ext", _P), ("n_bc", _I),
                ("bc_dofs", _P), ("bc_vel", _P), ("delta", _D), ("micromodulus", _I),
                ("c0", _D), ("l", _D), ("c_const", _D), ("h", _D), ("s_crit", _D),
                ("s_crit_spread", _D), ("seed", C.c_uint64), ("gamma", _D), ("beta", _D),
                ("dt", _D), ("mode", _I), ("device", _I), ("n_notch", _I),
                ("notch_npts", _P), ("notch_pts", _P), ("lattice", _I * 3),
                ("global_id_offset", C.c_int64), ("owned_elems", _I * 2),
                ("lattice_h", _D), ("lattice_vol", _D), ("slab_plane", _I * 2),
                ("node_rows", _I * 2)]


class PDInfo(C.Structure):
    _fields_ = [("n_bonds", C.c_int64), ("n_entries", C.c_int64), ("max_family", _I),
                ("path", _I), ("kernels_per_step", _I), ("stencil_size", _I),
                ("bytes_per_step", _D), ("bond_bytes_per_step", _D),
                ("device_bytes", _D), ("hot_tiles", C.c_int64), ("tested_tiles", C.c_int64)]


# exported symbols, with ctypes signatures: the CPU test checks the library
# exports every one of them (and the header declares the same set).
class MtsDesc(C.Structure):
    _fields_ = [("scenario", C.POINTER(ScenarioDesc)), ("n_pd_box", _I), ("pd_boxes", _P),
                ("overlap_width_factor", _D), ("weight_kind", _I), ("gamma_fe", _D),
                ("beta_fe", _D), ("interface_mode", _I), ("enforce_continuity", _I),
                ("track_energy", _I), ("device", _I), ("fe_spacing", _D),
                ("interface_precond", _I), ("interface_recursion", _I), ("shard_world", _I),
                ("shard_rank", _I), ("interface_h_fe", _I), ("pd_linear", _I), ("pd_elem_products", _I)]


class MtsShardView(C.Structure):
    _fields_ = [("world", _I), ("rank", _I), ("axis", _I), ("reach_layers", _I),
                ("n_layers", _I), ("n_local_nodes", _I), ("n_local_elems", _I),
                ("own_elem_lo", _I), ("own_elem_hi", _I), ("local_nodes", _P),
                ("local_elems", _P), ("node_owned", _P), ("layer_bounds", _P)]


class MtsView(C.Structure):
    _fields_ = [("dim", _I), ("n_nodes", _I), ("n_elems", _I), ("fe_n_dof", _I),
                ("pd_n_dof", _I), ("n_lambda", _I), ("dense", _I), ("m", _I), ("n_macro", _I),
                ("fe_nnz", _I), ("fe_n_bc", _I), ("pd_n_bc", _I), ("n_pd_elems", _I),
                ("n_pairs", C.c_int64), ("dt_pd", _D), ("delta", _D), ("c0", _D), ("l", _D),
                ("char_length", _D), ("load_ramp", _D), ("labels", _P), ("alpha", _P),
                ("fe_node_dof", _P), ("pd_node_dof", _P), ("fe_k_rowptr", _P), ("fe_k_col", _P),
                ("fe_k_val", _P), ("fe_mass", _P), ("fe_p_ext", _P), ("pd_mass", _P),
                ("pd_p_ext", _P), ("fe_bc_dofs", _P), ("fe_bc_vel", _P), ("pd_bc_dofs", _P),
                ("pd_bc_vel", _P), ("cpl_fe_dof", _P), ("cpl_pd_dof", _P), ("pairs", _P),
                ("pe_weight", _P), ("node_xyz", _P), ("elem_nodes", _P), ("node_alpha", _P),
                ("cpl_fe_nnz", C.c_int64), ("cpl_fe_rowptr", _P), ("cpl_fe_col", _P),
                ("cpl_fe_w", _P), ("fe_mesh_elems", _I), ("fe_mesh_nodes", _I),
                ("pd_linear_lattice", _I)]


class MtsReport(C.Structure):
    _fields_ = [("t_kinematic", _D), ("t_update", _D), ("t_lambda", _D), ("t_unit", _D),
                ("quad_fe", _D), ("quad_pd", _D), ("lambda_fe", _D), ("lambda_pd", _D),
                ("continuity", _D), ("newly_broken", _I), ("interface_iterations", _I)]


SIGNATURES = {
    "pmts_last_error": (C.c_char_p, []),
    "pmts_abi_version": (C.c_int, []),
    "pmts_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "pmts_scenario_build": (C.c_int, [C.POINTER(ScenarioDesc), C.POINTER(_P)]),
    "pmts_scenario_get": (C.c_int, [_P, C.POINTER(ScenarioView)]),
    "pmts_scenario_load_scale": (_D, [_P, _D]),
    "pmts_scenario_destroy": (None, [_P]),
    "pmts_pd_create": (C.c_int, [C.POINTER(PDDesc), C.POINTER(_P)]),
    "pmts_pd_destroy": (None, [_P]),
    "pmts_pd_build_families": (C.c_int, [_P]),
    "pmts_pd_set_pairs": (C.c_int, [_P, C.c_int64, _P]),
    "pmts_pd_get_pairs": (C.c_int, [_P, _P, C.c_int64, C.POINTER(C.c_int64)]),
    "pmts_pd_info_get": (C.c_int, [_P, C.POINTER(PDInfo)]),
    "pmts_pd_init": (C.c_int, [_P, _D]),
    "pmts_pd_step": (C.c_int, [_P, _I, _P, C.POINTER(C.c_int64)]),
    "pmts_pd_step_timed": (C.c_int, [_P, _I, _P, C.POINTER(C.c_float)]),
    "pmts_pd_step_tracked": (C.c_int, [_P, _I, _P, _I, _P, _P, _P]),
    "pmts_pd_profile": (C.c_int, [_P, _I, _P, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    "pmts_pd_get_state": (C.c_int, [_P, _P, _P, _P]),
    "pmts_pd_set_state": (C.c_int, [_P, _P, _P, _P]),
    "pmts_pd_get_intact": (C.c_int, [_P, _P, C.c_int64]),
    "pmts_pd_take_break_log": (C.c_int, [_P, _P, C.c_int64, C.POINTER(C.c_int64)]),
    "pmts_pd_broken_total": (C.c_int64, [_P]),
    "pmts_pd_damage": (C.c_int, [_P, _P, _P]),
    "pmts_pd_gather_disp": (C.c_int, [_P, _I, _P, _P]),
    "pmts_pd_stream": (_P, [_P]),
    "pmts_pd_get_rows": (C.c_int, [_P, _I, _I, _P]),
    "pmts_pd_get_rows_layers": (C.c_int, [_P, _I, _I, _I, _I, _P]),
    "pmts_pd_set_rows_layers": (C.c_int, [_P, _I, _I, _I, _I, _P]),
    "pmts_pd_set_halo_layers": (C.c_int, [_P, _I, _I]),
    "pmts_pd_set_option": (C.c_int, [_P, _I, _I]),
    "pmts_pd_set_constraint_load": (C.c_int, [_P, _I, _P, _P]),
    "pmts_pd_snapshot_bonds": (C.c_int, [_P]),
    "pmts_pd_homogeneous_recursion": (C.c_int, [_P, _I, _I, _P, _P, _P, _P, _P, _P]),
    "pmts_pd_set_rows": (C.c_int, [_P, _I, _I, _P]),
    "pmts_nccl_unique_id": (C.c_int, [_P]),
    "pmts_pd_comm_init": (C.c_int, [_P, _P, _I, _I]),
    "pmts_pd_set_halo": (C.c_int, [_P, _I, _I, _I, _I, _I, _I, _I, _I]),
    "pmts_pd_allreduce_sum": (C.c_int, [_P, C.POINTER(C.c_int64)]),
    "pmts_mts_create": (C.c_int, [C.POINTER(MtsDesc), C.POINTER(_P)]),
    "pmts_mts_view_get": (C.c_int, [_P, C.POINTER(MtsView)]),
    "pmts_mts_init": (C.c_int, [_P]),
    "pmts_mts_macro_step": (C.c_int, [_P, _I, _P]),
    "pmts_mts_macro_step_timed": (C.c_int, [_P, _I, C.POINTER(C.c_float)]),
    "pmts_mts_get_state": (C.c_int, [_P, _I, _P, _P, _P]),
    "pmts_mts_get_lambda": (C.c_int, [_P, _P]),
    "pmts_mts_get_intact": (C.c_int, [_P, _P]),
    "pmts_mts_damage": (C.c_int, [_P, _P, _P]),
    "pmts_mts_destroy": (None, [_P]),
    "pmts_mts_shard_view_get": (C.c_int, [_P, C.POINTER(MtsShardView)]),
    "pmts_mts_group_join": (C.c_int, [_P, _I]),
    "pmts_mts_group_init": (C.c_int, [_P, _I]),
    "pmts_mts_group_macro_step": (C.c_int, [_P, _I, _I, _P]),
    "pmts_mts_comm_init": (C.c_int, [_P, _P]),
}

ABI_VERSION = 2  # include/pmts_capi.h PMTS_ABI_VERSION
_lib = None


def lib():
    """Load libpmts.so (in-tree).  Raises if it is missing -- no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        if L.pmts_abi_version() != ABI_VERSION:  # the structs below mirror that header
            raise ImportError(f"{LIB_PATH}: ABI {L.pmts_abi_version()}, this binding is for "
                              f"{ABI_VERSION}: rebuild (__graft_entry__.build())")
        _lib = L
    return _lib


def check(status: int):
    if status == PMTS_OK:
        return
    msg = lib().pmts_last_error().decode(errors="replace")
    cls = {PMTS_ERR_CONFIG: ConfigError, PMTS_ERR_SOLVER: SolverError}.get(status, PmtsError)
    raise cls(msg or f"pmts status {status}")


def ptr(a):
    """numpy array -> void* (None passes NULL)."""
    return None if a is None else a.ctypes.data_as(_P)
