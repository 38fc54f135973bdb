"""ctypes front end of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference``
legs import this module.  The product package (paper_0902_4424_b200) never does.

It wraps oracle/liboracle.so (l1oracle.c, a C restatement of the reference
proj/core/src/{gpss,prox,linear_operator,objective}.cpp) and adds the harness problem
builder used by both sides of every parity test.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

CANONICAL, LITERAL = 0, 1
REASONS = {0: "stationary", 1: "max_iterations", 2: "max_matvecs", 3: "max_seconds",
           4: "objective_tol"}

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


class GpConfig(C.Structure):
    """gpss.hpp:14-24 defaults."""
    _fields_ = [("beta", C.c_double), ("theta", C.c_double), ("memory", C.c_int32),
                ("alpha2_memory", C.c_int32), ("alpha_min", C.c_double),
                ("alpha_max", C.c_double), ("tau1", C.c_double)]

    def __init__(self, beta=1e-4, theta=0.5, memory=1, alpha_min=1e-10, alpha_max=1e10,
                 tau1=0.5, alpha2_memory=2):
        super().__init__(beta, theta, memory, alpha2_memory, alpha_min, alpha_max, tau1)


class StopRule(C.Structure):
    """solver.hpp:52-60 defaults."""
    _fields_ = [("max_iterations", C.c_int64), ("max_matvecs", C.c_int64),
                ("max_seconds", C.c_double), ("stationarity_tol", C.c_double),
                ("objective_tol", C.c_double)]

    def __init__(self, max_iterations=100000, max_matvecs=0, max_seconds=0.0,
                 stationarity_tol=1e-9, objective_tol=0.0):
        super().__init__(max_iterations, max_matvecs, max_seconds, stationarity_tol,
                         objective_tol)


class IterRecord(C.Structure):
    _fields_ = [("k", C.c_int64), ("f", C.c_double), ("stationarity", C.c_double),
                ("alpha", C.c_double), ("step", C.c_double), ("matvecs", C.c_int64),
                ("elapsed_seconds", C.c_double), ("bb_active", C.c_int32),
                ("halvings", C.c_int32), ("bb1_raw", C.c_double), ("bb2_raw", C.c_double),
                ("tau_before", C.c_double), ("tau_after", C.c_double), ("f_max", C.c_double),
                ("dir_derivative", C.c_double), ("theta", C.c_double), ("support", C.c_int64)]


class Result(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("matvecs", C.c_int64), ("objective", C.c_double),
                ("stationarity", C.c_double), ("elapsed_seconds", C.c_double),
                ("reason", C.c_int32), ("status", C.c_int32),
                ("f_history", C.c_double * 64), ("f_history_len", C.c_int32)]


class SlState(C.Structure):
    _fields_ = [("tau", C.c_double), ("hist", C.c_double * 66), ("hist_len", C.c_int32)]


class SlChoice(C.Structure):
    _fields_ = [("alpha", C.c_double), ("bb_active", C.c_int32), ("bb1_raw", C.c_double),
                ("bb2_raw", C.c_double), ("tau_before", C.c_double), ("tau_after", C.c_double)]


RECORD_FIELDS = [f for f, _ in IterRecord._fields_]


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        i64, dbl, i32 = C.c_int64, C.c_double, C.c_int
        sig = {
            "orc_set_mode": (None, [i32]),
            "orc_get_mode": (i32, []),
            "orc_pairwise_sum": (dbl, [_dp, i64]),
            "orc_dot": (dbl, [_dp, _dp, i64]),
            "orc_sqnorm": (dbl, [_dp, i64]),
            "orc_l1norm": (dbl, [_dp, i64]),
            "orc_linf": (dbl, [_dp, i64]),
            "orc_apply": (None, [_dp, i64, i64, _dp, _dp]),
            "orc_apply_adjoint": (None, [_dp, i64, i64, _dp, _dp]),
            "orc_spectral_norm": (i32, [_dp, i64, i64, i32, dbl, C.POINTER(dbl),
                                        C.POINTER(i64)]),
            "orc_soft_threshold": (i32, [_dp, i64, dbl, _dp]),
            "orc_project_l1": (i32, [_dp, i64, dbl, _dp, C.POINTER(dbl), C.POINTER(i64)]),
            "orc_config_validate": (i32, [C.POINTER(GpConfig)]),
            "orc_stop_validate": (i32, [C.POINTER(StopRule)]),
            "orc_clamp_step": (dbl, [dbl, C.POINTER(GpConfig)]),
            "orc_backtrack_quadratic": (i32, [dbl, dbl, dbl, dbl, dbl, C.POINTER(GpConfig),
                                              C.POINTER(dbl), C.POINTER(dbl), C.POINTER(i32)]),
            "orc_steplength_init": (None, [C.POINTER(SlState), C.POINTER(GpConfig)]),
            "orc_steplength_select": (i32, [C.POINTER(SlState), _dp, _dp, i64,
                                            C.POINTER(GpConfig), i64, C.POINTER(SlChoice)]),
            "orc_alpha0_from_gradient": (dbl, [dbl, _dp, _dp, i64, C.POINTER(GpConfig)]),
            "orc_gpss_solve": (i32, [_dp, i64, i64, _dp, dbl, C.POINTER(GpConfig),
                                     C.POINTER(StopRule), C.c_void_p, _dp, C.POINTER(Result),
                                     C.c_void_p, i64, C.c_void_p]),
            "orc_psd_solve": (i32, [_dp, i64, i64, _dp, dbl, C.POINTER(StopRule), _dp,
                                    C.POINTER(Result), C.c_void_p, i64]),
            "orc_shrinkage_solve": (i32, [_dp, i64, i64, _dp, dbl, i32, C.POINTER(StopRule), _dp,
                                          C.POINTER(Result), C.c_void_p, i64]),
            "orc_fnv1a": (C.c_uint64, [C.c_void_p, i64, C.c_uint64]),
            "orc_penalized_fpr": (dbl, [_dp, i64, i64, _dp, _dp, dbl]),
            "orc_reference_minimizer": (i32, [_dp, i64, i64, _dp, dbl, dbl, i64, i64, _dp,
                                              C.POINTER(dbl), C.POINTER(i64)]),
            "orc_gp_init": (i32, [_dp, i64, i64, _dp, dbl, C.POINTER(GpConfig), C.c_void_p,
                                  C.POINTER(C.c_void_p)]),
            "orc_gp_iterate": (i32, [C.c_void_p, dbl, C.POINTER(IterRecord),
                                     C.POINTER(C.c_int32)]),
            "orc_gp_get": (None, [C.c_void_p, _dp, _dp, _dp, C.POINTER(dbl), C.POINTER(i64),
                                  C.POINTER(dbl), C.POINTER(i64)]),
            "orc_gp_free": (None, [C.c_void_p]),
            "orc_gp_set": (i32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, dbl, i64,
                                 _dp, i32, C.POINTER(GpConfig), dbl]),
            "orc_det_log": (dbl, [dbl]),
            "orc_det_sincos2pi": (None, [dbl, C.POINTER(dbl), C.POINTER(dbl)]),
            "orc_normal": (dbl, [C.c_uint64, C.c_uint32, C.c_uint64]),
            "orc_uniform": (dbl, [C.c_uint64, C.c_uint32, C.c_uint64]),
            "orc_fill_normal": (None, [C.c_uint64, C.c_uint32, C.c_uint64, i64, _dp]),
            "orc_gaussian_matrix": (None, [C.c_uint64, i64, i64, _dp]),
            "orc_blur_matrix": (None, [i64, _dp, i32, _dp]),
            "orc_scale": (None, [_dp, i64, dbl]),
            "orc_sample_support": (i32, [C.c_uint64, C.c_uint32, i64, i64, _ip]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(rc, what):
    if rc == 1:
        raise ValueError(f"{what}: invalid argument")
    if rc == 2:
        raise RuntimeError(f"{what}: computation failed")


@contextlib.contextmanager
def mode(m):
    L = lib()
    old = L.orc_get_mode()
    L.orc_set_mode(m)
    try:
        yield
    finally:
        L.orc_set_mode(old)


def _a(x):
    return np.ascontiguousarray(x, dtype=np.float64)


# ---------------------------------------------------------------- reductions / operator
def pairwise_sum(t):
    t = _a(t)
    return lib().orc_pairwise_sum(t, t.size)


def dot(a, b):
    a, b = _a(a), _a(b)
    return lib().orc_dot(a, b, a.size)


def sqnorm(a):
    a = _a(a)
    return lib().orc_sqnorm(a, a.size)


def l1norm(a):
    a = _a(a)
    return lib().orc_l1norm(a, a.size)


def linf(a):
    a = _a(a)
    return lib().orc_linf(a, a.size)


def apply(K, x):
    K, x = _a(K), _a(x)
    n, p = K.shape
    if x.size != p:
        raise ValueError("apply: dimension mismatch")
    out = np.empty(n)
    lib().orc_apply(K, n, p, x, out)
    return out


def apply_adjoint(K, r):
    K, r = _a(K), _a(r)
    n, p = K.shape
    if r.size != n:
        raise ValueError("apply_adjoint: dimension mismatch")
    out = np.empty(p)
    lib().orc_apply_adjoint(K, n, p, r, out)
    return out


def spectral_norm(K, max_iters=1000, tol=1e-8):
    K = _a(K)
    s, mv = C.c_double(), C.c_int64()
    _check(lib().orc_spectral_norm(K, K.shape[0], K.shape[1], max_iters, tol, C.byref(s),
                                   C.byref(mv)), "spectral_norm_estimate")
    return s.value, mv.value


# ---------------------------------------------------------------- prox
def soft_threshold(x, t):
    x = _a(x)
    out = np.empty_like(x)
    _check(lib().orc_soft_threshold(x, x.size, t, out), "soft_threshold")
    return out


def project_l1(x, rho):
    """Returns (point, theta, support) -- prox.cpp:38-73."""
    x = _a(x)
    out = np.empty_like(x)
    th, sup = C.c_double(), C.c_int64()
    _check(lib().orc_project_l1(x, x.size, rho, out, C.byref(th), C.byref(sup)),
           "project_l1_ball")
    return out, th.value, sup.value


# ---------------------------------------------------------------- gpss pieces
def config_valid(cfg):
    return lib().orc_config_validate(C.byref(cfg)) == 0


def clamp_step(a, cfg):
    return lib().orc_clamp_step(a, C.byref(cfg))


def backtrack_quadratic(f0, a, b, f_max, gd, cfg):
    step, fn, h = C.c_double(), C.c_double(), C.c_int32()
    _check(lib().orc_backtrack_quadratic(f0, a, b, f_max, gd, C.byref(cfg), C.byref(step),
                                         C.byref(fn), C.byref(h)), "backtracking_search")
    return step.value, fn.value, h.value


class Steplength:
    def __init__(self, cfg):
        self.cfg = cfg
        self.st = SlState()
        lib().orc_steplength_init(C.byref(self.st), C.byref(cfg))

    @property
    def tau(self):
        return self.st.tau

    @property
    def history(self):
        return [self.st.hist[i] for i in range(self.st.hist_len)]

    def select(self, s, z, k):
        s, z = _a(s), _a(z)
        c = SlChoice()
        _check(lib().orc_steplength_select(C.byref(self.st), s, z, s.size, C.byref(self.cfg),
                                           k, C.byref(c)), "steplength_select")
        return {f: getattr(c, f) for f, _ in SlChoice._fields_}


def alpha0_from_gradient(rho, x0, grad, cfg):
    x0, grad = _a(x0), _a(grad)
    return lib().orc_alpha0_from_gradient(rho, x0, grad, x0.size, C.byref(cfg))


def records_to_dicts(arr, count):
    return [{f: getattr(arr[i], f) for f in RECORD_FIELDS} for i in range(count)]


def gpss_solve(K, y, rho, cfg=None, stop=None, x0=None, trace=True, x_trace=False):
    """gpss.cpp:221-292.  Returns (x, result-dict, records, x_history-or-None)."""
    cfg = cfg or GpConfig()
    stop = stop or StopRule()
    K, y = _a(K), _a(y)
    n, p = K.shape
    x = np.zeros(p)
    res = Result()
    cap = int(stop.max_iterations) if (trace and stop.max_iterations > 0) else 0
    recs = (IterRecord * max(cap, 1))()
    xs = np.zeros((max(cap, 1), p)) if (x_trace and cap) else None
    x0a = _a(x0) if x0 is not None else None
    rc = lib().orc_gpss_solve(K, n, p, y, rho, C.byref(cfg), C.byref(stop),
                              x0a.ctypes.data if x0a is not None else None, x, C.byref(res),
                              C.addressof(recs) if cap else None, cap,
                              xs.ctypes.data if xs is not None else None)
    _check(rc, "gpss_solve")
    out = {f: getattr(res, f) for f, _ in Result._fields_ if f not in ("f_history",)}
    out["f_history"] = [res.f_history[i] for i in range(res.f_history_len)]
    out["reason_name"] = REASONS[res.reason]
    rec = records_to_dicts(recs, min(cap, res.iterations)) if cap else []
    xh = xs[: res.iterations] if xs is not None else None
    return x, out, rec, xh


def _result_dict(res):
    out = {f: getattr(res, f) for f, _ in Result._fields_ if f not in ("f_history",)}
    out["f_history"] = [res.f_history[i] for i in range(res.f_history_len)]
    out["reason_name"] = REASONS[res.reason]
    return out


def penalized_fixed_point_residual(K, y, x, lam):
    """reference.cpp:9-13."""
    K = _a(K)
    return lib().orc_penalized_fpr(K, K.shape[0], K.shape[1], _a(y), _a(x), lam)


def reference_minimizer(K, y, lam, oracle_tol=1e-12, max_iterations=500000, check_interval=50,
                        nnz_threshold=1e-10):
    """reference.cpp:38-82.  Returns dict(x, lambda, rho, nnz, certificate, iterations)."""
    K, y = _a(K), _a(y)
    n, p = K.shape
    x = np.zeros(p)
    cert, its = C.c_double(), C.c_int64()
    rc = lib().orc_reference_minimizer(K, n, p, y, lam, oracle_tol, max_iterations,
                                       check_interval, x, C.byref(cert), C.byref(its))
    if rc == 2:
        raise RuntimeError(f"reference_minimizer: certificate {cert.value} did not reach "
                           f"tolerance {oracle_tol} within {max_iterations} iterations")
    _check(rc, "reference_minimizer")
    return dict(x=x, **{"lambda": lam}, rho=l1norm(x), nnz=int(np.sum(np.abs(x) > nnz_threshold)),
                certificate=cert.value, iterations=its.value, oracle_tol=oracle_tol)


def psd_solve(K, y, rho, stop=None, trace=True):
    """psd.cpp:14-93.  Returns (x, result-dict, records)."""
    stop = stop or StopRule()
    K, y = _a(K), _a(y)
    n, p = K.shape
    x, res = np.zeros(p), Result()
    cap = int(stop.max_iterations) if (trace and stop.max_iterations > 0) else 0
    recs = (IterRecord * max(cap, 1))()
    _check(lib().orc_psd_solve(K, n, p, y, rho, C.byref(stop), x, C.byref(res),
                               C.addressof(recs) if cap else None, cap), "psd_solve")
    return x, _result_dict(res), (records_to_dicts(recs, min(cap, res.iterations)) if cap else [])


def shrinkage_solve(K, y, lam, accelerated, stop=None, trace=True):
    """ista_solve / fista_solve, shrinkage.cpp:41-118.  Returns (x, result-dict, records)."""
    stop = stop or StopRule()
    K, y = _a(K), _a(y)
    n, p = K.shape
    x, res = np.zeros(p), Result()
    cap = int(stop.max_iterations) if (trace and stop.max_iterations > 0) else 0
    recs = (IterRecord * max(cap, 1))()
    _check(lib().orc_shrinkage_solve(K, n, p, y, lam, int(accelerated), C.byref(stop), x,
                                     C.byref(res), C.addressof(recs) if cap else None, cap),
           "fista_solve" if accelerated else "ista_solve")
    return x, _result_dict(res), (records_to_dicts(recs, min(cap, res.iterations)) if cap else [])


class GpState:
    """gp_init / gp_iterate (gpss.cpp:117-219) over the oracle."""

    def __init__(self, K, y, rho, cfg=None, x0=None):
        self.K, self.y = _a(K), _a(y)
        self.n, self.p = self.K.shape
        self.cfg = cfg or GpConfig()
        self.rho = rho
        self._x0 = _a(x0) if x0 is not None else None
        h = C.c_void_p()
        _check(lib().orc_gp_init(self.K, self.n, self.p, self.y, rho, C.byref(self.cfg),
                                 self._x0.ctypes.data if self._x0 is not None else None,
                                 C.byref(h)), "gp_init")
        self.h = h

    def iterate(self, tol=0.0):
        rec, st = IterRecord(), C.c_int32()
        _check(lib().orc_gp_iterate(self.h, tol, C.byref(rec), C.byref(st)), "gp_iterate")
        return {f: getattr(rec, f) for f in RECORD_FIELDS}, bool(st.value)

    def set(self, x, r, g, f, k, f_history, cfg=None, rho=None):
        """Write the public GpIterationState fields (and gp_iterate's cfg / ball)."""
        if cfg is not None:
            self.cfg = cfg
        if rho is not None:
            self.rho = rho
        arrs = [_a(v) if v is not None else None for v in (x, r, g)]
        ptrs = [a.ctypes.data if a is not None else None for a in arrs]
        _check(lib().orc_gp_set(self.h, *ptrs, f, k, _a(f_history), len(f_history),
                                C.byref(self.cfg), self.rho), "gp_set")

    def get(self):
        x, r, g = np.empty(self.p), np.empty(self.n), np.empty(self.p)
        f, k, a0, mv = C.c_double(), C.c_int64(), C.c_double(), C.c_int64()
        lib().orc_gp_get(self.h, x, r, g, C.byref(f), C.byref(k), C.byref(a0), C.byref(mv))
        return dict(x=x, kx_minus_y=r, grad=g, f=f.value, k=k.value, alpha0=a0.value,
                    matvecs=mv.value)

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            lib().orc_gp_free(h)
            self.h = None


# ---------------------------------------------------------------- generators
def normal(seed, stream, index):
    return lib().orc_normal(seed, stream, index)


def uniform(seed, stream, index):
    return lib().orc_uniform(seed, stream, index)


def fill_normal(seed, stream, first, count):
    out = np.empty(count)
    lib().orc_fill_normal(seed, stream, first, count, out)
    return out


def gaussian_matrix(seed, n, p):
    K = np.empty((n, p))
    lib().orc_gaussian_matrix(seed, n, p, K)
    return K


BLUR_SIGMA, BLUR_RADIUS = 4.0, 12


def blur_taps(sigma=BLUR_SIGMA, radius=BLUR_RADIUS):
    """Unit-sum Gaussian taps w(k), |k| <= radius (libm exp; sequential sum)."""
    w = [math.exp(-(k * k) / (2.0 * sigma * sigma)) for k in range(-radius, radius + 1)]
    s = 0.0
    for v in w:
        s += v
    return np.array([v / s for v in w])


def blur_matrix(n, taps=None, radius=BLUR_RADIUS):
    taps = blur_taps() if taps is None else _a(taps)
    K = np.empty((n, n))
    lib().orc_blur_matrix(n, taps, radius, K)
    return K


def sample_support(seed, stream, p, k):
    idx = np.empty(max(k, 1), dtype=np.int64)
    _check(lib().orc_sample_support(seed, stream, p, k, idx), "sample_support")
    return idx[:k]


@dataclass
class ProblemSpec:
    """Seeded synthetic problem."""
    kind: str          # "gaussian" | "blur"
    n: int
    p: int
    nnz: int
    seed: int
    values: str        # "sign" | "normal" | "usign"
    noise: float
    noise_mode: str    # "abs" | "rel"
    rho_factor: float = 1.0
    norm_target: float = 0.9
    power_iters: int = 1000
    power_tol: float = 1e-8
    sigma_hat: float | None = None   # fixed spectral-norm estimate (skips power iteration)
    name: str = field(default="")


def x_true_values(spec, count):
    s, st = spec.seed, 3
    if spec.values == "sign":
        return np.array([1.0 if uniform(s, st, t) < 0.5 else -1.0 for t in range(count)])
    if spec.values == "normal":
        return np.array([normal(s, st, t) for t in range(count)])
    if spec.values == "usign":
        out = []
        for t in range(count):
            mag = 0.5 + 1.5 * uniform(s, st, 2 * t)
            out.append(mag if uniform(s, st, 2 * t + 1) < 0.5 else -mag)
        return np.array(out)
    raise ValueError(spec.values)


def build_problem(spec: ProblemSpec):
    """Returns dict(K, y, x_true, rho, sigma_hat, scale) built with canonical reductions."""
    with mode(CANONICAL):
        if spec.kind == "gaussian":
            K = gaussian_matrix(spec.seed, spec.n, spec.p)
            if spec.sigma_hat is None:
                sigma_hat, _ = spectral_norm(K, spec.power_iters, spec.power_tol)
            else:
                sigma_hat = spec.sigma_hat
            scale = spec.norm_target / sigma_hat
            lib().orc_scale(K, K.size, scale)
        elif spec.kind == "blur":
            if spec.n != spec.p:
                raise ValueError("blur operator is square")
            K = blur_matrix(spec.n)
            sigma_hat, scale = float("nan"), 1.0
        else:
            raise ValueError(spec.kind)
        x_true = np.zeros(spec.p)
        sup = sample_support(spec.seed, 1, spec.p, spec.nnz)
        x_true[sup] = x_true_values(spec, spec.nnz)
        clean = apply(K, x_true)
        e = fill_normal(spec.seed, 2, 0, spec.n)
        if spec.noise_mode == "abs":
            sig = spec.noise
        else:
            sig = spec.noise * math.sqrt(sqnorm(clean)) / math.sqrt(spec.n)
        y = clean + sig * e
        rho = spec.rho_factor * l1norm(x_true)
    return dict(K=K, y=y, x_true=x_true, rho=rho, sigma_hat=sigma_hat, scale=scale,
                noise_sigma=sig, support=sup)


# ------------------------------------------------------------------ L1PROBv1 (problem_io.cpp)
L1PROB_MAGIC = b"L1PROBv1"
FNV_BASIS = 1469598103934665603


def problem_bytes(K, y, x_true, seed, noise):
    """The serialized L1PROBv1 bytes (problem_io.cpp:43-60, docs/problem_format.md)."""
    K = np.ascontiguousarray(K, dtype="<f8")
    n, p = K.shape
    head = L1PROB_MAGIC + np.array([n, p, seed], dtype="<u8").tobytes() + \
        np.array([noise], dtype="<f8").tobytes()
    return head + K.tobytes() + np.ascontiguousarray(y, dtype="<f8").tobytes() + \
        np.ascontiguousarray(x_true, dtype="<f8").tobytes()


def save_problem(path, K, y, x_true, seed, noise):
    with open(path, "wb") as f:
        f.write(problem_bytes(K, y, x_true, seed, noise))


def load_problem(path):
    raw = open(path, "rb").read()
    if raw[:8] != L1PROB_MAGIC:
        raise RuntimeError(f"not an L1PROBv1 problem file: {path}")
    n, p, seed = (int(v) for v in np.frombuffer(raw, dtype="<u8", count=3, offset=8))
    noise = float(np.frombuffer(raw, dtype="<f8", count=1, offset=32)[0])
    if n < 1 or p < 1 or len(raw) < 40 + 8 * (n * p + n + p):
        raise RuntimeError(f"corrupt or truncated problem file: {path}")
    K = np.frombuffer(raw, dtype="<f8", count=n * p, offset=40).reshape(n, p).copy()
    y = np.frombuffer(raw, dtype="<f8", count=n, offset=40 + 8 * n * p).copy()
    x = np.frombuffer(raw, dtype="<f8", count=p, offset=40 + 8 * (n * p + n)).copy()
    return dict(K=K, y=y, x_true=x, seed=seed, noise_level=noise)


def problem_hash(K, y, x_true, seed, noise):
    b = problem_bytes(K, y, x_true, seed, noise)
    buf = C.create_string_buffer(b, len(b))
    return int(lib().orc_fnv1a(C.addressof(buf), len(b), FNV_BASIS))
