"""ctypes binding of libl1g.so (include/l1g.h).  No fallback: a missing or unloadable
extension raises immediately."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libl1g.so")

OK, EINVAL, ERUNTIME, ECANCELED = 0, 1, 2, 3
REASONS = {0: "stationary", 1: "max_iterations", 2: "max_matvecs", 3: "max_seconds",
           4: "objective_tol"}
RED_DOT, RED_SQ, RED_ABS, RED_MAX = 0, 1, 2, 3


class GpConfigC(C.Structure):
    _fields_ = [("beta", C.c_double), ("theta", C.c_double), ("memory", C.c_int32),
                ("alpha2_memory", C.c_int32), ("alpha_min", C.c_double),
                ("alpha_max", C.c_double), ("tau1", C.c_double)]


class StopRuleC(C.Structure):
    _fields_ = [("max_iterations", C.c_int64), ("max_matvecs", C.c_int64),
                ("max_seconds", C.c_double), ("stationarity_tol", C.c_double),
                ("objective_tol", C.c_double)]


class IterRecordC(C.Structure):
    _fields_ = [("k", C.c_int64), ("f", C.c_double), ("stationarity", C.c_double),
                ("alpha", C.c_double), ("step", C.c_double), ("matvecs", C.c_int64),
                ("elapsed_seconds", C.c_double), ("bb_active", C.c_int32),
                ("halvings", C.c_int32), ("bb1_raw", C.c_double), ("bb2_raw", C.c_double),
                ("tau_before", C.c_double), ("tau_after", C.c_double), ("f_max", C.c_double),
                ("dir_derivative", C.c_double), ("theta", C.c_double), ("support", C.c_int64)]


class ResultC(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("matvecs", C.c_int64), ("objective", C.c_double),
                ("stationarity", C.c_double), ("elapsed_seconds", C.c_double),
                ("reason", C.c_int32), ("status", C.c_int32),
                ("f_history", C.c_double * 64), ("f_history_len", C.c_int32)]


class SlStateC(C.Structure):
    _fields_ = [("tau", C.c_double), ("hist", C.c_double * 66), ("hist_len", C.c_int32)]


class SlChoiceC(C.Structure):
    _fields_ = [("alpha", C.c_double), ("bb_active", C.c_int32), ("bb1_raw", C.c_double),
                ("bb2_raw", C.c_double), ("tau_before", C.c_double), ("tau_after", C.c_double)]


class GpStateC(C.Structure):  # l1g_gp_state
    _fields_ = [("f", C.c_double), ("k", C.c_int64), ("alpha0", C.c_double),
                ("stationary", C.c_int32), ("has_prev", C.c_int32),
                ("f_history_len", C.c_int32), ("f_history", C.c_double * 64),
                ("tau", C.c_double), ("alpha2_len", C.c_int32),
                ("alpha2_history", C.c_double * 66), ("choice", SlChoiceC)]


class RefOptionsC(C.Structure):  # l1g_ref_options
    _fields_ = [("oracle_tol", C.c_double), ("max_iterations", C.c_int64),
                ("check_interval", C.c_int64), ("nnz_threshold", C.c_double)]


class RefSolutionC(C.Structure):  # l1g_ref_solution
    _fields_ = [("lambda_", C.c_double), ("rho", C.c_double), ("oracle_tol", C.c_double),
                ("certificate", C.c_double), ("nnz", C.c_int64), ("iterations", C.c_int64),
                ("matvecs", C.c_int64)]


RECORD_FIELDS = [f for f, _ in IterRecordC._fields_]
ITER_CB = C.CFUNCTYPE(C.c_int, C.POINTER(IterRecordC), C.POINTER(C.c_double), C.c_int64,
                      C.c_void_p)

ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int64,
                           C.c_void_p)
_dp = C.POINTER(C.c_double)
_vp = C.c_void_p
_i64 = C.c_int64
_SIGS = {
    "l1g_last_error": (C.c_char_p, []),
    "l1g_version": (C.c_char_p, []),
    "l1g_ctx_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "l1g_ctx_destroy": (None, [_vp]),
    "l1g_ctx_info": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(_i64)]),
    "l1g_op_create_dense": (C.c_int, [_vp, _vp, _i64, _i64, C.c_int, C.POINTER(_vp)]),
    "l1g_op_generate_gaussian": (C.c_int, [_vp, _i64, _i64, C.c_uint64, _i64, _i64,
                                           C.POINTER(_vp)]),
    "l1g_op_generate_blur": (C.c_int, [_vp, _i64, _vp, C.c_int, C.POINTER(_vp)]),
    "l1g_op_scale": (C.c_int, [_vp, C.c_double]),
    "l1g_op_dims": (C.c_int, [_vp, C.POINTER(_i64), C.POINTER(_i64)]),
    "l1g_op_download": (C.c_int, [_vp, _vp]),
    "l1g_op_destroy": (None, [_vp]),
    "l1g_op_apply": (C.c_int, [_vp, _vp, _vp]),
    "l1g_op_apply_adjoint": (C.c_int, [_vp, _vp, _vp]),
    "l1g_op_apply_dev": (C.c_int, [_vp, _vp, _vp, _vp]),
    "l1g_op_apply_adjoint_dev": (C.c_int, [_vp, _vp, _vp, _vp]),
    "l1g_op_apply_batched": (C.c_int, [_vp, C.c_int, _vp, _vp]),
    "l1g_op_apply_adjoint_batched": (C.c_int, [_vp, C.c_int, _vp, _vp]),
    "l1g_op_spectral_norm": (C.c_int, [_vp, C.c_int, C.c_double, _dp, C.POINTER(_i64)]),
    "l1g_project_l1": (C.c_int, [_vp, _vp, _i64, C.c_double, _vp, _dp, C.POINTER(_i64)]),
    "l1g_soft_threshold": (C.c_int, [_vp, _vp, _i64, C.c_double, _vp]),
    "l1g_reduce": (C.c_int, [_vp, _vp, _vp, _i64, C.c_int, _dp]),
    "l1g_config_validate": (C.c_int, [C.POINTER(GpConfigC)]),
    "l1g_stop_validate": (C.c_int, [C.POINTER(StopRuleC)]),
    "l1g_steplength_init": (None, [C.POINTER(SlStateC), C.POINTER(GpConfigC)]),
    "l1g_steplength_select": (C.c_int, [_vp, C.POINTER(SlStateC), _vp, _vp, _i64,
                                        C.POINTER(GpConfigC), _i64, C.POINTER(SlChoiceC)]),
    "l1g_backtrack": (C.c_int, [_vp, C.c_double, C.c_double, C.c_double, C.c_double,
                                C.c_double, C.POINTER(GpConfigC), _dp, _dp,
                                C.POINTER(C.c_int32)]),
    "l1g_alpha0_from_gradient": (C.c_int, [_vp, C.c_double, _vp, _vp, _i64,
                                           C.POINTER(GpConfigC), _dp]),
    "l1g_solver_create": (C.c_int, [_vp, _vp, C.c_double, C.POINTER(GpConfigC),
                                    C.POINTER(_vp)]),
    "l1g_solver_create_group": (C.c_int, [C.POINTER(_vp), C.c_int, _vp, C.c_double,
                                          C.POINTER(GpConfigC), C.POINTER(_vp)]),
    "l1g_comm_unique_id": (C.c_int, [_vp]),
    "l1g_comm_create": (C.c_int, [_vp, C.c_int, C.c_int, _vp, C.POINTER(_vp)]),
    "l1g_comm_destroy": (None, [_vp]),
    "l1g_comm_create_host": (C.c_int, [_vp, C.c_int, C.c_int, ALLGATHER_FN, _vp,
                                       C.POINTER(_vp)]),
    "l1g_solver_create_sharded": (C.c_int, [_vp, _vp, _vp, C.c_double, C.POINTER(GpConfigC),
                                            C.POINTER(_vp)]),
    "l1g_batch_create": (C.c_int, [_vp, C.c_int, _vp, _vp, C.POINTER(GpConfigC), C.POINTER(_vp)]),
    "l1g_batch_init": (C.c_int, [_vp, _vp]),
    "l1g_batch_run": (C.c_int, [_vp, C.POINTER(StopRuleC), _vp]),
    "l1g_batch_get_x": (C.c_int, [_vp, _vp]),
    "l1g_batch_resume": (C.c_int, [_vp, C.POINTER(StopRuleC), _vp]),
    "l1g_batch_stream": (C.c_int, [_vp, C.POINTER(_vp)]),
    "l1g_batch_launches": (C.c_int, [_vp, C.POINTER(_i64), C.c_int]),
    "l1g_batch_destroy": (None, [_vp]),
    "l1g_batch_time_products": (C.c_int, [_vp, C.c_int, _dp, _dp]),
    "l1g_gpss_solve_batched": (C.c_int, [_vp, C.c_int, _vp, _vp, C.POINTER(GpConfigC),
                                         C.POINTER(StopRuleC), _vp, _vp]),
    "l1g_solver_time_exchange": (C.c_int, [_vp, C.c_int, _dp, _dp]),
    "l1g_solver_set_y": (C.c_int, [_vp, _vp]),
    "l1g_solver_set_y_dev": (C.c_int, [_vp, _vp]),
    "l1g_solver_init": (C.c_int, [_vp, _vp]),
    "l1g_solver_iterate": (C.c_int, [_vp, C.c_double, C.POINTER(IterRecordC),
                                     C.POINTER(C.c_int32)]),
    "l1g_solver_run": (C.c_int, [_vp, C.POINTER(StopRuleC), C.POINTER(ResultC), _vp, _i64]),
    "l1g_solver_run_cb": (C.c_int, [_vp, C.POINTER(StopRuleC), C.POINTER(ResultC), ITER_CB,
                                    _vp]),
    "l1g_solver_get": (C.c_int, [_vp, _vp, _vp, _vp, _dp, C.POINTER(_i64), _dp,
                                 C.POINTER(_i64)]),
    "l1g_solver_x_dev": (C.c_int, [_vp, C.POINTER(_vp)]),
    "l1g_solver_get_state": (C.c_int, [_vp, C.POINTER(GpStateC), _vp, _vp, _vp, _vp, _vp]),
    "l1g_solver_set_state": (C.c_int, [_vp, C.POINTER(GpStateC), _vp, _vp, _vp, _vp, _vp]),
    "l1g_solver_set_problem": (C.c_int, [_vp, C.POINTER(GpConfigC), C.c_double]),
    "l1g_solver_stream": (C.c_int, [_vp, C.POINTER(_vp)]),
    "l1g_solver_destroy": (None, [_vp]),
    "l1g_solver_set_timing": (C.c_int, [_vp, C.c_int]),
    "l1g_solver_set_forward": (C.c_int, [_vp, C.c_int]),
    "l1g_solver_small_path": (C.c_int, [_vp, C.POINTER(C.c_int)]),
    "l1g_solver_proj_profile": (C.c_int, [_vp, _dp]),
    "l1g_solver_timing": (C.c_int, [_vp, _dp, _dp, _dp, C.POINTER(_i64), C.POINTER(_i64),
                                    C.c_int]),
    "l1g_gpss_solve": (C.c_int, [_vp, _vp, C.c_double, C.POINTER(GpConfigC),
                                 C.POINTER(StopRuleC), _vp, _vp, C.POINTER(ResultC), _vp, _i64]),
    "l1g_rng_fill": (C.c_int, [_vp, C.c_int, C.c_uint64, C.c_uint32, C.c_uint64, _i64, _vp]),
    "l1g_psd_solve": (C.c_int, [_vp, _vp, C.c_double, C.POINTER(StopRuleC), _vp,
                                C.POINTER(ResultC), _vp, _i64, ITER_CB, _vp]),
    "l1g_shrinkage_solve": (C.c_int, [_vp, _vp, C.c_double, C.c_int, C.POINTER(StopRuleC), _vp,
                                      C.POINTER(ResultC), _vp, _i64, ITER_CB, _vp]),
    "l1g_problem_info": (C.c_int, [C.c_char_p, C.POINTER(_i64), C.POINTER(_i64),
                                   C.POINTER(C.c_uint64), _dp]),
    "l1g_problem_load": (C.c_int, [_vp, C.c_char_p, _vp, _vp, C.POINTER(C.c_uint64), _dp,
                                   C.POINTER(_vp)]),
    "l1g_problem_save": (C.c_int, [C.c_char_p, _vp, _vp, _vp, C.c_uint64, C.c_double]),
    "l1g_problem_hash": (C.c_int, [_vp, _vp, _vp, C.c_uint64, C.c_double,
                                   C.POINTER(C.c_uint64)]),
    "l1g_reference_minimizer": (C.c_int, [_vp, _vp, C.c_double, C.POINTER(RefOptionsC), _vp,
                                          C.POINTER(RefSolutionC)]),
    "l1g_penalized_fixed_point_residual": (C.c_int, [_vp, _vp, _vp, C.c_double, _dp]),
    "l1g_host_alloc": (C.c_int, [_i64, C.POINTER(_vp)]),
    "l1g_host_free": (None, [_vp]),
}

EXPORTED = sorted(_SIGS)
_lib = None


def load(path: str | None = None):
    """Load libl1g.so; raises if it is missing (no CPU fallback exists)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or os.environ.get("L1G_LIB_PATH", LIB_PATH)  # L1G_LIB_PATH: debug builds
    if not os.path.exists(p):
        raise ImportError(f"{p} is missing: build the CUDA extension first "
                          "(python -c 'import __graft_entry__ as g; g.build()')")
    L = C.CDLL(p)
    for name, (res, args) in _SIGS.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = L
    return L


def check(rc: int, what: str = ""):
    if rc == OK:
        return
    msg = (load().l1g_last_error() or b"").decode()
    if rc == EINVAL:
        raise ValueError(f"{what}: {msg}" if what else msg)
    raise RuntimeError(f"{what}: {msg}" if what else msg)


def ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None
