"""ctypes declarations of include/pgmres.h (the C ABI of libpgmres.so)."""
from __future__ import annotations

import ctypes as C
import os

from .build import LIB

PGM_OK, PGM_EINVAL, PGM_ENONFINITE, PGM_ESINGULAR, PGM_ECUDA, PGM_ENCCL, PGM_ENOMEM, \
    PGM_ESTATE = range(8)
PGM_DEVICE_PTRS = 1


class ContextConfig(C.Structure):
    _fields_ = [("device", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32),
                ("nccl_id", C.c_void_p), ("loopback", C.c_void_p), ("n_axis", C.c_uint32),
                ("n_global", C.c_uint32), ("deterministic", C.c_int32)]


class Partition(C.Structure):
    _fields_ = [("row_begin", C.c_uint32), ("row_end", C.c_uint32), ("halo_lo", C.c_uint32),
                ("halo_hi", C.c_uint32)]


class CsrView(C.Structure):
    _fields_ = [("n", C.c_uint32), ("nnz", C.c_uint64), ("row_ptr", C.c_void_p),
                ("col_idx", C.c_void_p), ("values", C.c_void_p)]


class GmresConfigC(C.Structure):
    _fields_ = [("m", C.c_uint32), ("max_restarts", C.c_uint32), ("rel_tol", C.c_double),
                ("fixed_iterations", C.c_int32), ("breakdown_scale", C.c_double)]


class DeflationConfigC(C.Structure):
    _fields_ = [("r_max", C.c_uint32), ("drop", C.c_uint32), ("accept_tol", C.c_double),
                ("inv_power_maxit", C.c_uint32), ("inv_power_tol", C.c_double),
                ("power_maxit", C.c_uint32)]


class ReportC(C.Structure):
    _fields_ = [("beta0", C.c_double), ("restarts", C.c_uint32), ("total_inner", C.c_uint64),
                ("converged", C.c_int32), ("breakdown", C.c_int32),
                ("final_relative", C.c_double), ("n_inner", C.c_uint32),
                ("inner_restart", C.POINTER(C.c_uint32)), ("inner_step", C.POINTER(C.c_uint32)),
                ("inner_monitored", C.POINTER(C.c_double)),
                ("explicit_residual", C.POINTER(C.c_double)), ("solve_seconds", C.c_double)]


class DeflationRecordC(C.Structure):
    _fields_ = [("restart", C.c_uint32), ("r", C.c_uint32), ("mu", C.c_double),
                ("smallest_ritz", C.c_double)]


class NewtonConfigC(C.Structure):
    _fields_ = [("max_iters", C.c_uint32), ("update_tol", C.c_double),
                ("gmres", GmresConfigC), ("deflation", DeflationConfigC),
                ("use_deflation", C.c_int32), ("continuation", C.c_int32),
                ("continuation_steps", C.c_uint32)]


class NewtonRecordC(C.Structure):
    _fields_ = [("iter", C.c_uint32), ("lam", C.c_double), ("update_inf", C.c_double),
                ("residual_norm", C.c_double), ("gmres_restarts", C.c_uint32),
                ("gmres_inner", C.c_uint64)]


class NewtonReportC(C.Structure):
    _fields_ = [("iters", C.POINTER(NewtonRecordC)), ("n_iters", C.c_uint32),
                ("converged", C.c_int32), ("final_residual", C.c_double),
                ("final_update", C.c_double), ("total_inner", C.c_uint64),
                ("seconds", C.c_double)]


# Every symbol the header declares (tests check the .so exports all of them).
EXPORTS = [
    "pgm_context_create", "pgm_context_destroy", "pgm_last_error", "pgm_context_partition",
    "pgm_partition_rows", "pgm_context_stream", "pgm_matrix_upload", "pgm_matrix_update_values",
    "pgm_matrix_destroy", "pgm_matrix_info", "pgm_spmv", "pgm_deflator_create",
    "pgm_deflator_destroy", "pgm_deflator_reset", "pgm_deflator_info", "pgm_deflator_history",
    "pgm_deflator_basis", "pgm_deflator_push", "pgm_deflator_truncate",
    "pgm_deflator_observe_ritz", "pgm_deflator_apply", "pgm_solve", "pgm_report_free",
    "pgm_context_launch_count", "pgm_context_set_profiling", "pgm_context_profile",
    "pgm_bratu_nnz", "pgm_bratu_assemble", "pgm_nccl_unique_id", "pgm_loopback_create",
    "pgm_loopback_destroy", "pgm_newton_solve", "pgm_newton_report_free", "pgm_peer_export",
    "pgm_peer_import", "pgm_set_restart_observer", "pgm_restart_basis",
    "pgm_restart_hessenberg",
]

# pgm_restart_observer: int32 (*)(void* user, uint32 restart, uint32 steps)
RestartObserver = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_uint32, C.c_uint32)

_lib = None


def lib():
    """Load libpgmres.so; fails loudly when the CUDA library was not built."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("PGMRES_LIB", LIB)  # variant builds for tuning studies
    if not os.path.exists(path):
        raise ImportError(f"libpgmres.so not built at {path}; run __graft_entry__.build() "
                          "(there is no CPU fallback)")
    L = C.CDLL(path)
    vp, u32, i32, dbl = C.c_void_p, C.c_uint32, C.c_int32, C.c_double
    sig = {
        "pgm_context_create": ([C.POINTER(ContextConfig), C.POINTER(vp)], C.c_int),
        "pgm_context_destroy": ([vp], None),
        "pgm_last_error": ([vp], C.c_char_p),
        "pgm_context_partition": ([vp, C.POINTER(Partition)], C.c_int),
        "pgm_partition_rows": ([u32, u32, u32, C.POINTER(Partition)], C.c_int),
        "pgm_context_stream": ([vp], vp),
        "pgm_context_launch_count": ([vp], C.c_uint64),
        "pgm_matrix_upload": ([vp, C.POINTER(CsrView), i32, C.POINTER(vp)], C.c_int),
        "pgm_matrix_update_values": ([vp, vp, i32], C.c_int),
        "pgm_matrix_destroy": ([vp], None),
        "pgm_matrix_info": ([vp, C.POINTER(u32), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                             C.POINTER(C.c_uint64)], C.c_int),
        "pgm_spmv": ([vp, vp, vp, i32], C.c_int),
        "pgm_deflator_create": ([vp, C.POINTER(DeflationConfigC), C.POINTER(vp)], C.c_int),
        "pgm_deflator_destroy": ([vp], None),
        "pgm_deflator_reset": ([vp], C.c_int),
        "pgm_deflator_info": ([vp, C.POINTER(u32), C.POINTER(dbl), C.POINTER(u32),
                               C.POINTER(u32)], C.c_int),
        "pgm_deflator_history": ([vp, C.POINTER(DeflationRecordC), u32], C.c_int),
        "pgm_deflator_basis": ([vp, vp, vp], C.c_int),
        "pgm_deflator_push": ([vp, vp, vp, i32, C.POINTER(i32)], C.c_int),
        "pgm_deflator_truncate": ([vp], C.c_int),
        "pgm_deflator_observe_ritz": ([vp, dbl], C.c_int),
        "pgm_deflator_apply": ([vp, vp, vp, i32], C.c_int),
        "pgm_solve": ([vp, vp, vp, vp, vp, C.POINTER(GmresConfigC), i32, C.POINTER(ReportC)],
                      C.c_int),
        "pgm_report_free": ([C.POINTER(ReportC)], None),
        "pgm_context_set_profiling": ([vp, i32], C.c_int),
        "pgm_context_profile": ([vp, vp, vp, vp, vp, u32], u32),
        "pgm_bratu_nnz": ([vp, u32, C.POINTER(C.c_uint64)], C.c_int),
        "pgm_bratu_assemble": ([vp, u32, dbl, vp, i32, vp, vp, vp, vp], C.c_int),
        "pgm_nccl_unique_id": ([vp], C.c_int),
        "pgm_loopback_create": ([i32, C.POINTER(vp)], C.c_int),
        "pgm_loopback_destroy": ([vp], None),
        "pgm_newton_solve": ([vp, u32, dbl, vp, i32, C.POINTER(NewtonConfigC),
                              C.POINTER(NewtonReportC)], C.c_int),
        "pgm_newton_report_free": ([C.POINTER(NewtonReportC)], None),
        "pgm_peer_export": ([vp, vp], C.c_int),
        "pgm_peer_import": ([vp, vp], C.c_int),
        "pgm_set_restart_observer": ([vp, RestartObserver, vp], C.c_int),
        "pgm_restart_basis": ([vp, u32, vp], C.c_int),
        "pgm_restart_hessenberg": ([vp, vp], C.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L
