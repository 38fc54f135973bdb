"""ctypes front end of oracle/_ref (TEST INFRASTRUCTURE ONLY).

oracle/_ref/libref_{canon,fast}.so are the reference's own gpss.cpp / prox.cpp /
linear_operator.cpp / objective.cpp compiled by oracle/build_ref.sh against the Eigen
stand-in in oracle/eigen_shim (Eigen is absent from this image).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_libs = {}


def path(kind="canon"):
    return os.path.join(HERE, "_ref", f"libref_{kind}.so")


def available(kind="canon"):
    return os.path.exists(path(kind))


def lib(kind="canon"):
    if kind not in _libs:
        L = C.CDLL(path(kind))
        L.ref_op_create.restype = C.c_void_p
        L.ref_op_create.argtypes = [_dp, C.c_long, C.c_long]
        L.ref_op_free.argtypes = [C.c_void_p]
        L.ref_project_l1.restype = C.c_int
        L.ref_project_l1.argtypes = [_dp, C.c_long, C.c_double, _dp, C.POINTER(C.c_double)]
        L.ref_apply.restype = C.c_int
        L.ref_apply.argtypes = [C.c_void_p, _dp, _dp, C.c_int]
        L.ref_spectral_norm.restype = C.c_int
        L.ref_spectral_norm.argtypes = [C.c_void_p, C.c_int, C.c_double, C.POINTER(C.c_double)]
        L.ref_gpss_solve.restype = C.c_int
        L.ref_gpss_solve.argtypes = [C.c_void_p, _dp, C.c_double, C.POINTER(O.GpConfig),
                                     C.POINTER(O.StopRule), C.c_void_p, _dp,
                                     C.POINTER(O.Result), C.c_void_p, C.c_long]
        L.ref_psd_solve.restype = C.c_int
        L.ref_psd_solve.argtypes = [C.c_void_p, _dp, C.c_double, C.POINTER(O.StopRule), _dp,
                                    C.POINTER(O.Result), C.c_void_p, C.c_long]
        L.ref_shrinkage_solve.restype = C.c_int
        L.ref_shrinkage_solve.argtypes = [C.c_void_p, _dp, C.c_double, C.c_int,
                                          C.POINTER(O.StopRule), _dp, C.POINTER(O.Result),
                                          C.c_void_p, C.c_long]
        L.ref_problem_save.restype = C.c_int
        L.ref_problem_save.argtypes = [C.c_char_p, _dp, C.c_long, C.c_long, _dp, _dp,
                                       C.c_uint64, C.c_double]
        L.ref_problem_load.restype = C.c_int
        L.ref_problem_load.argtypes = [C.c_char_p, C.c_long, C.c_long, _dp, _dp, _dp,
                                       C.POINTER(C.c_uint64), C.POINTER(C.c_double)]
        L.ref_reference_minimizer.restype = C.c_int
        L.ref_reference_minimizer.argtypes = [C.c_void_p, _dp, C.c_double, C.c_double, C.c_long,
                                              C.c_long, _dp, C.POINTER(C.c_double),
                                              C.POINTER(C.c_double), C.POINTER(C.c_long)]
        L.ref_problem_hash.restype = C.c_int
        L.ref_problem_hash.argtypes = [_dp, C.c_long, C.c_long, _dp, _dp, C.c_uint64,
                                       C.c_double, C.POINTER(C.c_uint64)]
        _libs[kind] = L
    return _libs[kind]


class RefOperator:
    def __init__(self, K, kind="canon"):
        self.L = lib(kind)
        K = np.ascontiguousarray(K, dtype=np.float64)
        self.n, self.p = K.shape
        self.h = self.L.ref_op_create(K, self.n, self.p)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_op_free(self.h)
            self.h = None

    def apply(self, x, adjoint=False):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty(self.p if adjoint else self.n)
        O._check(self.L.ref_apply(self.h, x, out, int(adjoint)), "apply")
        return out

    def reference_minimizer(self, y, lam, oracle_tol=1e-12, max_iterations=500000,
                            check_interval=50):
        """reference.cpp:38-82 (the reference's own source). Returns (x, certificate, rho, nnz)."""
        y = np.ascontiguousarray(y, dtype=np.float64)
        x = np.zeros(self.p)
        cert, rho, nnz = C.c_double(), C.c_double(), C.c_long()
        O._check(self.L.ref_reference_minimizer(self.h, y, lam, oracle_tol, max_iterations,
                                                check_interval, x, C.byref(cert), C.byref(rho),
                                                C.byref(nnz)), "reference_minimizer")
        return x, cert.value, rho.value, nnz.value

    def spectral_norm(self, max_iters=1000, tol=1e-8):
        s = C.c_double()
        O._check(self.L.ref_spectral_norm(self.h, max_iters, tol, C.byref(s)), "spectral")
        return s.value

    def gpss_solve(self, y, rho, cfg=None, stop=None, x0=None, trace=True):
        cfg = cfg or O.GpConfig()
        stop = stop or O.StopRule()
        y = np.ascontiguousarray(y, dtype=np.float64)
        x = np.zeros(self.p)
        res = O.Result()
        cap = int(stop.max_iterations) if (trace and stop.max_iterations > 0) else 0
        recs = (O.IterRecord * max(cap, 1))()
        x0a = np.ascontiguousarray(x0, dtype=np.float64) if x0 is not None else None
        rc = self.L.ref_gpss_solve(self.h, y, rho, C.byref(cfg), C.byref(stop),
                                   x0a.ctypes.data if x0a is not None else None, x,
                                   C.byref(res), C.addressof(recs) if cap else None, cap)
        O._check(rc, "gpss_solve")
        out = {f: getattr(res, f) for f, _ in O.Result._fields_ if f != "f_history"}
        out["f_history"] = [res.f_history[i] for i in range(res.f_history_len)]
        out["reason_name"] = O.REASONS[res.reason]
        rec = O.records_to_dicts(recs, min(cap, res.iterations)) if cap else []
        return x, out, rec


def _solve_other(op, fn, args, stop, trace):
    cap = int(stop.max_iterations) if (trace and stop.max_iterations > 0) else 0
    recs = (O.IterRecord * max(cap, 1))()
    x, res = np.zeros(op.p), O.Result()
    O._check(fn(op.h, *args, C.byref(stop), x, C.byref(res), C.addressof(recs) if cap else None,
                cap), "solve")
    return x, O._result_dict(res), (O.records_to_dicts(recs, min(cap, res.iterations)) if cap else [])


def psd_solve(op: "RefOperator", y, rho, stop=None, trace=True):
    stop = stop or O.StopRule()
    return _solve_other(op, op.L.ref_psd_solve, (np.ascontiguousarray(y, dtype=np.float64), rho),
                        stop, trace)


def shrinkage_solve(op: "RefOperator", y, lam, accelerated, stop=None, trace=True):
    stop = stop or O.StopRule()
    return _solve_other(op, op.L.ref_shrinkage_solve,
                        (np.ascontiguousarray(y, dtype=np.float64), lam, int(accelerated)),
                        stop, trace)


def project_l1(x, rho, kind="canon"):
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    th = C.c_double()
    O._check(lib(kind).ref_project_l1(x, x.size, rho, out, C.byref(th)), "project_l1_ball")
    return out, th.value


def problem_save(path, K, y, x_true, seed, noise):
    K = np.ascontiguousarray(K, dtype=np.float64)
    n, p = K.shape
    O._check(lib().ref_problem_save(str(path).encode(), K, n, p, np.ascontiguousarray(y, dtype=np.float64),
                                    np.ascontiguousarray(x_true, dtype=np.float64), seed, noise),
             "save_problem")


def problem_load(path, n, p):
    K, y, x = np.empty((n, p)), np.empty(n), np.empty(p)
    seed, noise = C.c_uint64(), C.c_double()
    O._check(lib().ref_problem_load(str(path).encode(), n, p, K, y, x, C.byref(seed),
                                    C.byref(noise)), "load_problem")
    return dict(K=K, y=y, x_true=x, seed=seed.value, noise_level=noise.value)


def problem_hash(K, y, x_true, seed, noise):
    K = np.ascontiguousarray(K, dtype=np.float64)
    n, p = K.shape
    h = C.c_uint64()
    O._check(lib().ref_problem_hash(K, n, p, np.ascontiguousarray(y, dtype=np.float64),
                                    np.ascontiguousarray(x_true, dtype=np.float64), seed, noise,
                                    C.byref(h)), "problem_hash")
    return h.value
