"""ctypes binding of the C-ABI in include/axb_b200.h (libaxb_b200.so).

The shared library is built in-tree by ``build.py`` (``__graft_entry__.build()``).
Importing this module never falls back to anything: if the library is missing
or a symbol is absent, it raises.
"""
from __future__ import annotations

import ctypes as C
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# AXB_LIB_VARIANT=checked: the build with device bounds checks (build.py --checked)
LIB_PATH = os.path.join(PKG_DIR, "libaxb_b200_checked.so" if os.environ.get("AXB_LIB_VARIANT") == "checked"
                        else "libaxb_b200.so")

_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)


class AxbConfig(C.Structure):
    """axb_config — SolveConfig (solver.hpp:100-109)."""

    _fields_ = [
        ("method", C.c_int32),
        ("has_theta", C.c_int32),
        ("theta", C.c_double),
        ("alpha_rule", C.c_int32),
        ("stop_kind", C.c_int32),
        ("alpha_value", C.c_double),
        ("tol", C.c_double),
        ("reference", C.c_void_p),
        ("max_iter", C.c_uint64),
        ("seed", C.c_uint64),
        ("record_trace", C.c_int32),
        ("_pad", C.c_int32),
        ("refresh_interval", C.c_uint64),
    ]


class AxbReport(C.Structure):
    """axb_report — SolveReport (solver.hpp:120-133) minus the owned vectors."""

    _fields_ = [
        ("iterations", C.c_uint64),
        ("wall_seconds", C.c_double),
        ("final_rrn", C.c_double),
        ("final_residual_rel", C.c_double),
        ("terminated_by", C.c_int32),
        ("alpha_outside_bound", C.c_int32),
        ("alpha", C.c_double),
        ("seed", C.c_uint64),
        ("skipped_zero_rows", C.c_uint64),
        ("trace_len", C.c_uint64),
        ("diverged_iteration", C.c_uint64),
        ("diverged_residual", C.c_double),
    ]


class AxbOptions(C.Structure):
    """axb_options — B200 placement / execution options."""

    _fields_ = [
        ("device", C.c_int32),
        ("inputs_on_device", C.c_int32),
        ("cache_gram", C.c_int32),
        ("spectral_on_device", C.c_int32),
        ("graph_iters", C.c_int32),
        ("tie_guard", C.c_int32),
        ("spectral_max_iter", C.c_uint64),
        ("alpha_override", C.c_double),
        ("nccl_comm", C.c_void_p),
        ("world_size", C.c_int32),
        ("rank", C.c_int32),
        ("m_global", C.c_uint64),
        ("row_offset", C.c_uint64),
        ("sm_share", C.c_int32),
        ("_pad0", C.c_int32),
    ]


class AxbMatrix(C.Structure):
    """axb_matrix — the reference's axb::Matrix variant (dense or CSR)."""

    _fields_ = [
        ("kind", C.c_int32),
        ("_pad", C.c_int32),
        ("rows", C.c_uint64),
        ("cols", C.c_uint64),
        ("nnz", C.c_uint64),
        ("dense", C.c_void_p),
        ("row_ptr", C.c_void_p),
        ("col_idx", C.c_void_p),
        ("values", C.c_void_p),
    ]


# (name, restype, argtypes) for every symbol include/axb_b200.h declares
_H = C.c_void_p
SIGNATURES = [
    ("axb_options_default", None, [C.POINTER(AxbOptions)]),
    ("axb_abi_version", C.c_int, []),
    ("axb_checked_build", C.c_int, []),
    ("axb_nccl_unique_id", C.c_int, [C.c_char_p]),
    ("axb_nccl_comm_create", C.c_int, [C.c_int, C.c_char_p, C.c_int, C.c_int,
                                       C.POINTER(C.c_void_p)]),
    ("axb_nccl_comm_destroy", C.c_int, [C.c_void_p]),
    ("axb_nccl_emulated_group", C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    ("axb_device_available", C.c_int, []),
    ("axb_solver_create", C.c_int,
     [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p,
      C.c_void_p, C.POINTER(AxbConfig), C.POINTER(AxbOptions), C.POINTER(_H)]),
    ("axb_solver_create_ex", C.c_int,
     [C.POINTER(AxbMatrix), C.POINTER(AxbMatrix), C.c_void_p, C.c_void_p, C.POINTER(AxbConfig),
      C.POINTER(AxbOptions), C.POINTER(_H)]),
    ("axb_solver_destroy", None, [_H]),
    ("axb_solver_last_error", C.c_char_p, [_H]),
    ("axb_last_create_error", C.c_char_p, []),
    ("axb_solver_last_error_info", C.c_int, [_H, _u64p, _dp]),
    ("axb_solver_step", C.c_int, [_H, _u64p]),
    ("axb_solver_steps", C.c_int, [_H, C.c_uint64, _u64p, C.c_int32]),
    ("axb_solver_replay", C.c_int, [_H, C.c_uint64, _u64p, C.c_int32]),
    ("axb_solver_update_row", C.c_int, [_H, C.c_uint64]),
    ("axb_solver_run", C.c_int,
     [_H, C.POINTER(AxbReport), _u64p, _dp, _dp, _u64p, C.c_uint64, _dp]),
    ("axb_solver_select_cyclic", C.c_int, [_H, _u64p]),
    ("axb_solver_select_rbk", C.c_int, [_H, _u64p]),
    ("axb_solver_select_greedy", C.c_int, [_H, C.c_double, _u64p]),
    ("axb_solver_select_mwrbk", C.c_int, [_H, _u64p]),
    ("axb_solver_greedy_threshold", C.c_int, [_H, C.c_double, _dp]),
    ("axb_solver_rgrbk_threshold", C.c_int, [_H, C.c_double, _dp]),
    ("axb_solver_greedy_index_set", C.c_int, [_H, C.c_double, _u64p, _u64p]),
    ("axb_solver_max_residual_ratio", C.c_int, [_H, _u64p, _dp]),
    ("axb_solver_current_metric", C.c_int, [_H, _dp]),
    ("axb_solver_current_residual_rel", C.c_int, [_H, _dp]),
    ("axb_solver_exact_metric", C.c_int, [_H, _dp]),
    ("axb_solver_exact_residual_rel", C.c_int, [_H, _dp]),
    ("axb_solver_residual_drift", C.c_int, [_H, _dp]),
    ("axb_solver_checkpoint", C.c_int, [_H]),
    ("axb_solver_iteration", C.c_uint64, [_H]),
    ("axb_solver_alpha", C.c_double, [_H]),
    ("axb_solver_spectral_norm_b", C.c_double, [_H]),
    ("axb_solver_alpha_outside_bound", C.c_int, [_H]),
    ("axb_solver_gram_cached", C.c_int, [_H]),
    ("axb_solver_a_fro_sq", C.c_double, [_H]),
    ("axb_solver_residual_fro_sq", C.c_int, [_H, _dp]),
    ("axb_solver_get_X", C.c_int, [_H, _dp]),
    ("axb_solver_get_R", C.c_int, [_H, _dp]),
    ("axb_solver_get_r_sq", C.c_int, [_H, _dp]),
    ("axb_solver_get_a_sq", C.c_int, [_H, _dp]),
    ("axb_solver_dims", C.c_int, [_H, _u64p]),
    ("axb_solver_last_timing", C.c_int, [_H, _dp, _dp, _u64p, _u64p]),
    ("axb_solver_kernel_times", C.c_int, [_H, _dp]),
    ("axb_solver_collective_times", C.c_int, [_H, _dp]),
    ("axb_solver_debug_state", C.c_int, [_H, _u64p]),
    ("axb_solver_set_profiling", C.c_int, [_H, C.c_int32]),
    ("axb_debug_timeline", C.c_int, [_u64p, C.c_int32]),
    ("axb_debug_dgemm", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64,
                                  C.c_uint64, C.c_uint64, C.c_int32, C.c_int32, _dp]),
    ("axb_solvers_run", C.c_int,
     [C.POINTER(_H), C.c_uint32, C.POINTER(AxbReport), C.POINTER(_dp), C.POINTER(C.c_int32)]),
    # reference solutions
    ("axb_svd", C.c_int, [_dp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int32, _dp, _dp, _dp,
                          _u64p]),
    ("axb_pseudoinverse", C.c_int, [_dp, C.c_uint64, C.c_uint64, C.c_double, C.c_int32, _dp]),
    ("axb_reference_solution", C.c_int,
     [C.POINTER(AxbMatrix), C.POINTER(AxbMatrix), _dp, C.c_double, C.c_int32, _dp,
      C.POINTER(C.c_int32), _dp]),
    ("axb_bk_limit", C.c_int,
     [C.POINTER(AxbMatrix), C.POINTER(AxbMatrix), _dp, _dp, C.c_int32, _dp]),
    ("axb_rrn", C.c_int, [_dp, _dp, C.c_uint64, C.c_int32, _dp]),
    ("axb_analysis_stats", C.c_int, [_u64p, _dp]),
]

_lib = None


def load():
    """Load libaxb_b200.so (raises if it was not built — there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (the B200 solver has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)  # AttributeError if the export is missing
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def device_available() -> bool:
    return bool(load().axb_device_available())
