"""Python mirror of the reference l1solve solver API (proj/core/include/l1solve), backed by
the B200 engine through its C-ABI (include/l1g.h).

Names, argument meaning and error behaviour follow the reference headers:
  linear_operator.hpp (LinearOperator, DenseOperator, spectral_norm_estimate),
  prox.hpp (L1Ball, soft_threshold, project_l1_ball[_with_threshold], lambda_max, ...),
  solver.hpp (Objective, StopReason, StopRule, IterationRecord, SolverState),
  gpss.hpp (GpConfig, SteplengthState, steplength_*, alpha0_*, backtracking_search,
            GpIterationState, gp_init, gp_iterate, gpss_solve).
std::invalid_argument maps to ValueError and std::runtime_error to RuntimeError.  Vectors are
float64 numpy arrays; all arithmetic runs on the GPU.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _lib as L
from ._lib import check, ptr


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64).ravel())


# ------------------------------------------------------------------------------ context
class Context:
    """One CUDA device (l1g_ctx).  One process per GPU."""

    def __init__(self, device: int = 0):
        self._lib = L.load()
        h = C.c_void_p()
        check(self._lib.l1g_ctx_create(device, C.byref(h)), "l1g_ctx_create")
        self.h = h
        self.device = device

    def info(self):
        sm, fr = C.c_int(), C.c_int64()
        check(self._lib.l1g_ctx_info(self.h, C.byref(sm), C.byref(fr)))
        return {"sm_count": sm.value, "free_bytes": fr.value}

    def close(self):
        if getattr(self, "h", None):
            self._lib.l1g_ctx_destroy(self.h)
            self.h = None


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# ------------------------------------------------------------------------------ types
@dataclass
class MatvecCounter:  # types.hpp:15-17
    count: int = 0


class StopReason(enum.IntEnum):  # solver.hpp:38-44
    Stationary = 0
    MaxIterations = 1
    MaxMatvecs = 2
    MaxSeconds = 3
    ObjectiveTol = 4


def to_string(r: StopReason) -> str:
    return L.REASONS[int(r)]


@dataclass
class GpConfig:  # gpss.hpp:14-24
    beta: float = 1e-4
    theta: float = 0.5
    memory: int = 1
    alpha_min: float = 1e-10
    alpha_max: float = 1e10
    tau1: float = 0.5
    alpha2_memory: int = 2

    def _c(self) -> L.GpConfigC:
        return L.GpConfigC(self.beta, self.theta, self.memory, self.alpha2_memory,
                           self.alpha_min, self.alpha_max, self.tau1)

    def validate(self):  # gpss.cpp:41-50
        c = self._c()
        check(L.load().l1g_config_validate(C.byref(c)), "GpConfig")


@dataclass
class StopRule:  # solver.hpp:52-60
    max_iterations: int = 100000
    max_matvecs: int = 0
    max_seconds: float = 0.0
    stationarity_tol: float = 1e-9
    objective_tol: float = 0.0

    def _c(self) -> L.StopRuleC:
        return L.StopRuleC(self.max_iterations, self.max_matvecs, self.max_seconds,
                           self.stationarity_tol, self.objective_tol)

    def validate(self):  # objective.cpp:42-48
        c = self._c()
        check(L.load().l1g_stop_validate(C.byref(c)), "StopRule")


@dataclass
class IterationRecord:  # solver.hpp:68-84 (+ halvings, theta, support)
    k: int = 0
    f: float = math.nan
    stationarity: float = math.nan
    alpha: float = math.nan
    step: float = math.nan
    matvecs: int = 0
    elapsed_seconds: float = 0.0
    bb_active: bool = False
    halvings: int = 0
    bb1_raw: float = math.nan
    bb2_raw: float = math.nan
    tau_before: float = math.nan
    tau_after: float = math.nan
    f_max: float = math.nan
    dir_derivative: float = math.nan
    theta: float = math.nan
    support: int = 0

    @staticmethod
    def from_c(r: L.IterRecordC) -> "IterationRecord":
        d = {f: getattr(r, f) for f in L.RECORD_FIELDS}
        d["bb_active"] = bool(d["bb_active"])
        return IterationRecord(**d)

    def as_dict(self):
        return dict(self.__dict__)


IterationCallback = Callable[[IterationRecord, np.ndarray], None]


@dataclass
class SolverState:  # solver.hpp:91-100
    x: np.ndarray
    iterations: int = 0
    matvecs: MatvecCounter = field(default_factory=MatvecCounter)
    f_history: list = field(default_factory=list)
    objective: float = math.nan
    stationarity: float = math.inf
    elapsed_seconds: float = 0.0
    reason: StopReason = StopReason.MaxIterations


# ------------------------------------------------------------------------------ operators
class LinearOperator:
    """linear_operator.hpp:15-33: counted apply/apply_adjoint with dimension checks."""

    def rows(self) -> int:
        raise NotImplementedError

    def cols(self) -> int:
        raise NotImplementedError

    def apply(self, x, mv: Optional[MatvecCounter] = None) -> np.ndarray:
        x = _f64(x)
        if x.size != self.cols():
            raise ValueError(f"apply: vector has length {x.size}, operator expects {self.cols()}")
        out = self._do_apply(x)
        if mv is not None:
            mv.count += 1
        return out

    def apply_adjoint(self, r, mv: Optional[MatvecCounter] = None) -> np.ndarray:
        r = _f64(r)
        if r.size != self.rows():
            raise ValueError(
                f"apply_adjoint: vector has length {r.size}, operator expects {self.rows()}")
        out = self._do_apply_adjoint(r)
        if mv is not None:
            mv.count += 1
        return out

    def _do_apply(self, x):
        raise NotImplementedError

    def _do_apply_adjoint(self, r):
        raise NotImplementedError


class DenseOperator(LinearOperator):
    """linear_operator.hpp:36-52.  K lives on the GPU in the tiled layout."""

    def __init__(self, K=None, ctx: Optional[Context] = None, _handle=None, _dims=None):
        self.ctx = ctx or default_context()
        self._lib = L.load()
        if _handle is not None:
            self.h = _handle
            self._n, self._p = _dims
            return
        K = np.ascontiguousarray(np.asarray(K, dtype=np.float64))
        if K.ndim != 2:
            raise ValueError("DenseOperator: K must be a 2-D array")
        self._n, self._p = K.shape
        h = C.c_void_p()
        check(self._lib.l1g_op_create_dense(self.ctx.h, ptr(K), self._n, self._p, 1,
                                            C.byref(h)), "DenseOperator")
        self.h = h

    @classmethod
    def generate_gaussian(cls, n, p, seed, ctx=None, col_offset=0, p_total=0):
        """Harness: raw K_ij = N(0,1) from the Philox stream (synthetic data)."""
        ctx = ctx or default_context()
        h = C.c_void_p()
        check(L.load().l1g_op_generate_gaussian(ctx.h, n, p, seed, col_offset, p_total,
                                                C.byref(h)), "generate_gaussian")
        return cls(ctx=ctx, _handle=h, _dims=(n, p))

    @classmethod
    def generate_blur(cls, n, taps, radius, ctx=None):
        ctx = ctx or default_context()
        taps = _f64(taps)
        h = C.c_void_p()
        check(L.load().l1g_op_generate_blur(ctx.h, n, ptr(taps), radius, C.byref(h)),
              "generate_blur")
        return cls(ctx=ctx, _handle=h, _dims=(n, n))

    def rows(self):
        return self._n

    def cols(self):
        return self._p

    def scale(self, c: float):
        check(self._lib.l1g_op_scale(self.h, c), "scale")

    def matrix(self) -> np.ndarray:
        K = np.empty((self._n, self._p))
        check(self._lib.l1g_op_download(self.h, ptr(K)), "matrix")
        return K

    def _do_apply(self, x):
        out = np.empty(self._n)
        check(self._lib.l1g_op_apply(self.h, ptr(x), ptr(out)), "apply")
        return out

    def _do_apply_adjoint(self, r):
        out = np.empty(self._p)
        check(self._lib.l1g_op_apply_adjoint(self.h, ptr(r), ptr(out)), "apply_adjoint")
        return out

    def close(self):
        if getattr(self, "h", None):
            self._lib.l1g_op_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def spectral_norm_estimate(op: DenseOperator, max_iters: int = 1000, tol: float = 1e-8,
                           mv: Optional[MatvecCounter] = None) -> float:
    """linear_operator.cpp:43-60 on the device."""
    s, m = C.c_double(), C.c_int64()
    check(L.load().l1g_op_spectral_norm(op.h, max_iters, tol, C.byref(s), C.byref(m)),
          "spectral_norm_estimate")
    if mv is not None:
        mv.count += m.value
    return s.value


# ------------------------------------------------------------------------------ prox
class L1Ball:  # prox.hpp:9-17
    def __init__(self, rho: float):
        if not (rho >= 0.0):
            raise ValueError("L1Ball: radius must be >= 0")
        self._rho = float(rho)

    def radius(self) -> float:
        return self._rho

    def contains(self, x, tol: float = 1e-12) -> bool:
        return l1_norm(x) <= self._rho + tol


class PenaltyWeight:  # prox.hpp:19-27
    def __init__(self, lam: float):
        if not (lam >= 0.0):
            raise ValueError("PenaltyWeight: lambda must be >= 0")
        self._lam = float(lam)

    def value(self):
        return self._lam


def _reduce(a, b, op, ctx=None) -> float:
    ctx = ctx or default_context()
    a = _f64(a)
    b = _f64(b) if b is not None else None
    out = C.c_double()
    check(L.load().l1g_reduce(ctx.h, ptr(a), ptr(b), a.size, op, C.byref(out)), "reduce")
    return out.value


def dot(a, b, ctx=None) -> float:
    return _reduce(a, b, L.RED_DOT, ctx)


def squared_norm(a, ctx=None) -> float:
    return _reduce(a, None, L.RED_SQ, ctx)


def l1_norm(a, ctx=None) -> float:
    return _reduce(a, None, L.RED_ABS, ctx)


def linf_norm(a, ctx=None) -> float:
    return _reduce(a, None, L.RED_MAX, ctx)


def soft_threshold(x, t, ctx=None) -> np.ndarray:  # prox.cpp:23-36
    if isinstance(t, PenaltyWeight):
        t = t.value()
    ctx = ctx or default_context()
    x = _f64(x)
    out = np.empty_like(x)
    check(L.load().l1g_soft_threshold(ctx.h, ptr(x), x.size, float(t), ptr(out)),
          "soft_threshold")
    return out


@dataclass
class L1Projection:  # prox.hpp:29-32
    point: np.ndarray
    threshold: float
    support: int = 0


def project_l1_ball_with_threshold(x, ball: L1Ball, ctx=None) -> L1Projection:
    """prox.cpp:38-73, computed by the cluster projection kernel."""
    ctx = ctx or default_context()
    x = _f64(x)
    out = np.empty_like(x)
    th, sup = C.c_double(), C.c_int64()
    check(L.load().l1g_project_l1(ctx.h, ptr(x), x.size, ball.radius(), ptr(out), C.byref(th),
                                  C.byref(sup)), "project_l1_ball")
    return L1Projection(out, th.value, sup.value)


def project_l1_ball(x, ball: L1Ball, ctx=None) -> np.ndarray:
    return project_l1_ball_with_threshold(x, ball, ctx).point


def lambda_max(op: LinearOperator, y, mv: Optional[MatvecCounter] = None) -> float:
    return linf_norm(op.apply_adjoint(y, mv))  # prox.cpp:79-81


def lambda_from_rho(op: LinearOperator, y, x_rho, mv: Optional[MatvecCounter] = None) -> float:
    misfit = _f64(y) - op.apply(x_rho, mv)  # prox.cpp:88-92 (elementwise, exact)
    return linf_norm(op.apply_adjoint(misfit, mv))


def rho_from_lambda(x_lambda) -> float:
    return l1_norm(x_lambda)


# ------------------------------------------------------------------------------ objective
class Objective:  # solver.hpp:20-36, objective.cpp:5-40
    def __init__(self, op: LinearOperator, y):
        y = _f64(y).copy()
        if y.size != op.rows():
            raise ValueError("Objective: data vector length does not match operator rows")
        self._op, self._y = op, y

    def op(self):
        return self._op

    def y(self):
        return self._y

    def dim(self):
        return self._op.cols()

    def value(self, x, mv=None):
        return squared_norm(self._op.apply(x, mv) - self._y)

    def residual(self, x, mv=None):
        return self._op.apply_adjoint(self._y - self._op.apply(x, mv), mv)

    def gradient(self, x, mv=None):
        return -2.0 * self.residual(x, mv)

    def value_and_gradient(self, x, mv=None):
        misfit = self._op.apply(x, mv) - self._y
        return squared_norm(misfit), 2.0 * self._op.apply_adjoint(misfit, mv)


# ------------------------------------------------------------------------------ gpss
class SteplengthState:  # gpss.hpp:31-36
    def __init__(self, cfg: GpConfig):
        self._c = L.SlStateC()
        c = cfg._c()
        L.load().l1g_steplength_init(C.byref(self._c), C.byref(c))
        self.prev_x = None     # x and grad of the previous iterate (set by gp_iterate)
        self.prev_grad = None

    @property
    def tau(self):
        return self._c.tau

    @tau.setter
    def tau(self, v):
        self._c.tau = float(v)

    @property
    def alpha2_history(self):
        return [self._c.hist[i] for i in range(self._c.hist_len)]


@dataclass
class SteplengthChoice:  # gpss.hpp:43-50
    alpha: float = 0.0
    bb_active: bool = False
    bb1_raw: float = math.nan
    bb2_raw: float = math.nan
    tau_before: float = math.nan
    tau_after: float = math.nan


def steplength_init(cfg: GpConfig) -> SteplengthState:  # gpss.cpp:52-57
    cfg.validate()
    return SteplengthState(cfg)


def steplength_select(st: SteplengthState, s, z, cfg: GpConfig, k: int,
                      ctx=None) -> SteplengthChoice:  # gpss.cpp:59-91
    ctx = ctx or default_context()
    s, z = _f64(s), _f64(z)
    if s.size != z.size:
        raise ValueError("steplength_select: size mismatch")
    out = L.SlChoiceC()
    c = cfg._c()
    check(L.load().l1g_steplength_select(ctx.h, C.byref(st._c), ptr(s), ptr(z), s.size,
                                         C.byref(c), k, C.byref(out)), "steplength_select")
    return SteplengthChoice(out.alpha, bool(out.bb_active), out.bb1_raw, out.bb2_raw,
                            out.tau_before, out.tau_after)


def alpha0_from_gradient(ball: L1Ball, x0, grad, cfg: GpConfig, ctx=None) -> float:
    ctx = ctx or default_context()
    x0, grad = _f64(x0), _f64(grad)
    out = C.c_double()
    c = cfg._c()
    check(L.load().l1g_alpha0_from_gradient(ctx.h, ball.radius(), ptr(x0), ptr(grad), x0.size,
                                            C.byref(c), C.byref(out)), "alpha0_from_gradient")
    return out.value


def alpha0_init(prob: Objective, ball: L1Ball, x0, cfg: GpConfig,
                mv: MatvecCounter) -> float:  # gpss.cpp:100-104
    cfg.validate()
    return alpha0_from_gradient(ball, x0, prob.gradient(x0, mv), cfg)


@dataclass
class BacktrackResult:  # gpss.hpp:71-75
    step: float = 1.0
    f_new: float = 0.0
    halvings: int = 0


def backtracking_search(prob: Objective, x, d, f_max: float, dir_derivative: float,
                        cfg: GpConfig, mv: MatvecCounter, ctx=None) -> BacktrackResult:
    """gpss.cpp:106-115: 2 matvecs, then the quadratic backtracking on the device."""
    if not dir_derivative < 0.0:
        raise ValueError("backtracking_search: d must be a descent direction")
    ctx = ctx or default_context()
    misfit = prob.op().apply(x, mv) - prob.y()
    kd = prob.op().apply(d, mv)
    step, fn, h = C.c_double(), C.c_double(), C.c_int32()
    c = cfg._c()
    check(L.load().l1g_backtrack(ctx.h, squared_norm(misfit), dot(misfit, kd),
                                 squared_norm(kd), f_max, dir_derivative, C.byref(c),
                                 C.byref(step), C.byref(fn), C.byref(h)), "backtracking_search")
    return BacktrackResult(step.value, fn.value, h.value)


def _require_dense(prob: Objective) -> DenseOperator:
    op = prob.op()
    if not isinstance(op, DenseOperator):
        raise TypeError("the device-resident GPSS loop needs a DenseOperator")
    return op


class GpIterationState:
    """gpss.hpp:89-98: x, kx_minus_y, grad, f, k, f_history, alpha0, stationary are plain
    attributes, refreshed from the device (an l1g_solver) after gp_init / gp_iterate;
    attributes a caller changes are written back before the next step."""

    def __init__(self, prob: Objective, ball: L1Ball, x0, cfg: GpConfig):
        op = _require_dense(prob)
        self._lib = L.load()
        self._op = op
        self._y = prob.y()
        h = C.c_void_p()
        c = cfg._c()
        check(self._lib.l1g_solver_create(op.h, ptr(self._y), ball.radius(), C.byref(c),
                                          C.byref(h)), "gp_init")
        self.h = h
        x0a = _f64(x0) if x0 is not None and np.size(x0) else None
        if x0a is not None and x0a.size != prob.dim():
            self.close()
            raise ValueError("gp_init: starting point has wrong dimension")
        rc = self._lib.l1g_solver_init(self.h, ptr(x0a))
        if rc:
            self.close()
        check(rc, "gp_init")
        self._cfg = (c.beta, c.theta, c.memory, c.alpha2_memory, c.alpha_min, c.alpha_max,
                     c.tau1)
        self._rho = ball.radius()
        self._pull(None)

    # device -> attributes (and the copy changes are detected against)
    def _pull(self, sls):
        n, p = self._op.rows(), self._op.cols()
        g = L.GpStateC()
        x, r, gr, xp, gp = np.empty(p), np.empty(n), np.empty(p), np.empty(p), np.empty(p)
        check(self._lib.l1g_solver_get_state(self.h, C.byref(g), ptr(x), ptr(r), ptr(gr),
                                             ptr(xp), ptr(gp)), "gp state")
        self.x, self.kx_minus_y, self.grad = x, r, gr
        self.f, self.k, self.alpha0 = g.f, g.k, g.alpha0
        self.stationary = bool(g.stationary)
        self.f_history = [g.f_history[i] for i in range(g.f_history_len)]
        self._m = dict(x=x.copy(), r=r.copy(), g=gr.copy(), f=g.f, k=g.k, a0=g.alpha0,
                       st=bool(g.stationary), fh=list(self.f_history), tau=g.tau,
                       a2=[g.alpha2_history[i] for i in range(g.alpha2_len)],
                       xp=xp.copy() if g.has_prev else None, gp=gp.copy() if g.has_prev else None)
        if sls is not None:
            sls._c.tau = g.tau
            sls._c.hist_len = g.alpha2_len
            for i in range(g.alpha2_len):
                sls._c.hist[i] = g.alpha2_history[i]
            if g.has_prev:
                sls.prev_x, sls.prev_grad = xp, gp
        return g

    # attributes / steplength state / cfg / ball -> device, where they changed
    def _push(self, sls, cfg: GpConfig, ball: L1Ball):
        c = cfg._c()
        key = (c.beta, c.theta, c.memory, c.alpha2_memory, c.alpha_min, c.alpha_max, c.tau1)
        if key != self._cfg or ball.radius() != self._rho:
            check(self._lib.l1g_solver_set_problem(self.h, C.byref(c), ball.radius()),
                  "gp_iterate")
            self._cfg, self._rho = key, ball.radius()
        m = self._m
        neq = lambda a, b: not (np.shape(a) == np.shape(b) and
                                np.array_equal(np.asarray(a).view(np.int64),
                                               np.asarray(b).view(np.int64)))
        x = _f64(self.x) if neq(_f64(self.x), m["x"]) else None
        r = _f64(self.kx_minus_y) if neq(_f64(self.kx_minus_y), m["r"]) else None
        g = _f64(self.grad) if neq(_f64(self.grad), m["g"]) else None
        xp = gp = None
        tau, a2 = m["tau"], m["a2"]
        if sls is not None:
            tau, a2 = sls.tau, sls.alpha2_history
            px, pg = getattr(sls, "prev_x", None), getattr(sls, "prev_grad", None)
            if self.k > 0 and px is not None and pg is not None:
                if m["xp"] is None or neq(_f64(px), m["xp"]):
                    xp = _f64(px)
                if m["gp"] is None or neq(_f64(pg), m["gp"]):
                    gp = _f64(pg)
        scal = (self.f != m["f"] or self.k != m["k"] or list(self.f_history) != m["fh"] or
                self.alpha0 != m["a0"] or bool(self.stationary) != m["st"] or tau != m["tau"] or
                list(a2) != m["a2"])
        if not (scal or any(v is not None for v in (x, r, g, xp, gp))):
            return
        st = L.GpStateC()
        st.f, st.k, st.alpha0, st.stationary = self.f, self.k, self.alpha0, int(self.stationary)
        st.f_history_len = len(self.f_history)
        for i, v in enumerate(self.f_history):
            st.f_history[i] = v
        st.tau, st.alpha2_len = tau, len(a2)
        for i, v in enumerate(a2):
            st.alpha2_history[i] = v
        check(self._lib.l1g_solver_set_state(self.h, C.byref(st), ptr(x), ptr(r), ptr(g),
                                             ptr(xp), ptr(gp)), "gp_iterate")
        self._pull(None)

    def close(self):
        if getattr(self, "h", None):
            self._lib.l1g_solver_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class GpStepInfo:  # gpss.hpp:105-115
    stationary: bool = False
    alpha: float = math.nan
    step: float = math.nan
    f_after: float = math.nan
    stationarity: float = math.nan
    f_max: float = math.nan
    dir_derivative: float = math.nan
    steplength: SteplengthChoice = field(default_factory=SteplengthChoice)
    halvings: int = 0
    theta: float = math.nan
    support: int = 0


def gp_init(prob: Objective, ball: L1Ball, x0, cfg: GpConfig,
            mv: MatvecCounter) -> GpIterationState:  # gpss.cpp:117-134
    cfg.validate()
    st = GpIterationState(prob, ball, x0, cfg)
    mv.count += 2
    return st


def gp_iterate(prob: Objective, ball: L1Ball, cfg: GpConfig, state: GpIterationState,
               sls: Optional[SteplengthState], mv: MatvecCounter,
               stationarity_tol: float = 0.0) -> GpStepInfo:  # gpss.cpp:136-219
    """One step on the device; `state` (and `sls`, when given) are read and updated like the
    reference's (changed attributes, GpConfig and ball are written back first)."""
    state._push(sls, cfg, ball)
    if state.stationary:  # gpss.cpp:139-143
        return GpStepInfo(stationary=True, stationarity=0.0)
    rec, st = L.IterRecordC(), C.c_int32()
    mv0 = C.c_int64()
    lib = state._lib
    check(lib.l1g_solver_get(state.h, None, None, None, None, None, None, C.byref(mv0)))
    check(lib.l1g_solver_iterate(state.h, stationarity_tol, C.byref(rec), C.byref(st)),
          "gp_iterate")
    mv1 = C.c_int64()
    check(lib.l1g_solver_get(state.h, None, None, None, None, None, None, C.byref(mv1)))
    mv.count += mv1.value - mv0.value
    g = state._pull(sls)
    r = IterationRecord.from_c(rec)
    ch = g.choice  # the steplength choice before any escalation (gpss.cpp:148-153)
    info = GpStepInfo(stationary=bool(st.value), alpha=r.alpha, f_after=state.f,
                      stationarity=r.stationarity,
                      steplength=SteplengthChoice(ch.alpha, bool(ch.bb_active), ch.bb1_raw,
                                                  ch.bb2_raw, ch.tau_before, ch.tau_after),
                      theta=r.theta, support=r.support)
    if not info.stationary:
        info.step, info.f_max, info.dir_derivative = r.step, r.f_max, r.dir_derivative
        info.halvings = r.halvings
    elif not math.isnan(r.dir_derivative):
        info.dir_derivative = r.dir_derivative
    return info


def _state_from(res: L.ResultC, x) -> SolverState:
    return SolverState(x=x, iterations=res.iterations, matvecs=MatvecCounter(res.matvecs),
                       f_history=[res.f_history[i] for i in range(res.f_history_len)],
                       objective=res.objective, stationarity=res.stationarity,
                       elapsed_seconds=res.elapsed_seconds, reason=StopReason(res.reason))


def gpss_solve(prob: Objective, ball: L1Ball, cfg: GpConfig, stop: StopRule,
               cb: Optional[IterationCallback] = None, x0=None,
               trace: Optional[list] = None) -> SolverState:
    """gpss.cpp:221-292.  Without a callback the whole loop runs on the device (CUDA graphs
    of the projection / forward / adjoint kernels); with one, each iteration is followed by
    a synchronisation so cb(record, x) sees every step in order.  `trace`, if given, receives
    every IterationRecord (device ring buffer, copied once at the end)."""
    stop.validate()
    cfg.validate()
    op = _require_dense(prob)
    lib = L.load()
    y = prob.y()
    x0a = _f64(x0) if x0 is not None and np.size(x0) else None
    if x0a is not None and x0a.size != prob.dim():
        raise ValueError("gp_init: starting point has wrong dimension")
    res = L.ResultC()
    c, s = cfg._c(), stop._c()
    x = np.empty(op.cols())
    if cb is None:
        cap = stop.max_iterations if (trace is not None and stop.max_iterations > 0) else 0
        recs = (L.IterRecordC * max(cap, 1))()
        check(lib.l1g_gpss_solve(op.h, ptr(y), ball.radius(), C.byref(c), C.byref(s), ptr(x0a),
                                 ptr(x), C.byref(res), C.addressof(recs) if cap else None, cap),
              "gpss_solve")
        if trace is not None:
            trace.extend(IterationRecord.from_c(recs[i]) for i in range(min(cap, res.iterations)))
        return _state_from(res, x)
    h = C.c_void_p()
    check(lib.l1g_solver_create(op.h, ptr(y), ball.radius(), C.byref(c), C.byref(h)),
          "gpss_solve")
    err = []

    def _cb(rec_p, x_p, p, user):
        try:
            rec = IterationRecord.from_c(rec_p.contents)
            xv = np.ctypeslib.as_array(x_p, shape=(p,)).copy()
            if trace is not None:
                trace.append(rec)
            cb(rec, xv)
            return 0
        except BaseException as e:  # stops the run now; re-raised below
            err.append(e)
            return 1

    cfun = L.ITER_CB(_cb)
    try:
        check(lib.l1g_solver_init(h, ptr(x0a)), "gp_init")
        rc = lib.l1g_solver_run_cb(h, C.byref(s), C.byref(res), cfun, None)
        if err:
            raise err[0]
        check(rc, "gpss_solve")
        check(lib.l1g_solver_get(h, ptr(x), None, None, None, None, None, None))
    finally:
        lib.l1g_solver_destroy(h)
    return _state_from(res, x)


# ------------------------------------------------------------------ PSD, ISTA, FISTA
def _other_solve(prob: Objective, param: float, kind: int, stop: StopRule,
                 cb: Optional[IterationCallback], trace: Optional[list]) -> SolverState:
    stop.validate()
    op = _require_dense(prob)
    lib = L.load()
    y = prob.y()
    res = L.ResultC()
    s = stop._c()
    x = np.empty(op.cols())
    cap = stop.max_iterations if (trace is not None and stop.max_iterations > 0) else 0
    recs = (L.IterRecordC * max(cap, 1))()
    err = []

    def _cb(rec_p, x_p, p, user):
        try:
            cb(IterationRecord.from_c(rec_p.contents),
               np.ctypeslib.as_array(x_p, shape=(p,)).copy())
            return 0
        except BaseException as e:  # stops the run now; re-raised below
            err.append(e)
            return 1

    cfun = L.ITER_CB(_cb) if cb is not None else L.ITER_CB()
    if kind == 0:
        rc = lib.l1g_psd_solve(op.h, ptr(y), param, C.byref(s), ptr(x), C.byref(res),
                               C.addressof(recs) if cap else None, cap, cfun, None)
    else:
        rc = lib.l1g_shrinkage_solve(op.h, ptr(y), param, int(kind == 2), C.byref(s), ptr(x),
                                     C.byref(res), C.addressof(recs) if cap else None, cap,
                                     cfun, None)
    if err:
        raise err[0]
    check(rc, ["psd_solve", "ista_solve", "fista_solve"][kind])
    if trace is not None:
        trace.extend(IterationRecord.from_c(recs[i]) for i in range(min(cap, res.iterations)))
    return _state_from(res, x)


def psd_solve(prob: Objective, ball: L1Ball, stop: StopRule,
              cb: Optional[IterationCallback] = None,
              trace: Optional[list] = None) -> SolverState:
    """Projected steepest descent, psd.cpp:14-93 (3 matvecs per iteration)."""
    return _other_solve(prob, ball.radius(), 0, stop, cb, trace)


def ista_solve(prob: Objective, lam: PenaltyWeight, stop: StopRule,
               cb: Optional[IterationCallback] = None,
               trace: Optional[list] = None) -> SolverState:
    """Iterative soft thresholding, shrinkage.cpp:41-112 (c = 0.999 rescaling)."""
    return _other_solve(prob, lam.value(), 1, stop, cb, trace)


def fista_solve(prob: Objective, lam: PenaltyWeight, stop: StopRule,
                cb: Optional[IterationCallback] = None,
                trace: Optional[list] = None) -> SolverState:
    """Accelerated soft thresholding, shrinkage.cpp:41-118."""
    return _other_solve(prob, lam.value(), 2, stop, cb, trace)


# ------------------------------------------------------------------ reference minimizer
@dataclass
class ReferenceOptions:  # reference.hpp:19-24
    oracle_tol: float = 1e-12
    max_iterations: int = 500000
    check_interval: int = 50
    nnz_threshold: float = 1e-10


@dataclass
class ReferenceSolution:  # reference.hpp:9-17
    lambda_: float = 0.0
    rho: float = 0.0
    x: Optional[np.ndarray] = None
    nnz: int = 0
    oracle_tol: float = 0.0
    certificate: float = 0.0
    iterations: int = 0
    matvecs: int = 0


def reference_minimizer(prob: Objective, lam: float,
                        opt: Optional[ReferenceOptions] = None) -> ReferenceSolution:
    """reference.cpp:38-82 on the device FISTA kernels: the penalized minimizer x(lambda),
    driven until ||x - S_lambda(x + K^T(y - Kx))||_inf <= oracle_tol.  RuntimeError if the
    certificate is not reached within max_iterations (as the reference throws)."""
    opt = opt or ReferenceOptions()
    op = _require_dense(prob)
    o = L.RefOptionsC(opt.oracle_tol, opt.max_iterations, opt.check_interval, opt.nnz_threshold)
    out = L.RefSolutionC()
    x = np.empty(op.cols())
    check(L.load().l1g_reference_minimizer(op.h, ptr(prob.y()), float(lam), C.byref(o), ptr(x),
                                           C.byref(out)), "reference_minimizer")
    return ReferenceSolution(out.lambda_, out.rho, x, out.nnz, out.oracle_tol, out.certificate,
                             out.iterations, out.matvecs)


def penalized_fixed_point_residual(prob: Objective, x, lam: float) -> float:
    """reference.cpp:9-13 (2 matvecs on the device)."""
    op = _require_dense(prob)
    out = C.c_double()
    check(L.load().l1g_penalized_fixed_point_residual(op.h, ptr(prob.y()), ptr(_f64(x)),
                                                      float(lam), C.byref(out)),
          "penalized_fixed_point_residual")
    return out.value


# ------------------------------------------------------------------ L1PROBv1 problem files
@dataclass
class GeneratedProblem:  # generators.hpp:14-20
    op: DenseOperator
    y: np.ndarray
    x_true: np.ndarray
    noise_level: float = 0.0
    seed: int = 0


def load_problem(path, ctx: Optional[Context] = None) -> GeneratedProblem:
    """problem_io.cpp load_problem: K goes straight into the device tiled layout."""
    ctx = ctx or default_context()
    lib = L.load()
    n, p = C.c_int64(), C.c_int64()
    check(lib.l1g_problem_info(str(path).encode(), C.byref(n), C.byref(p), None, None),
          "load_problem")
    y, x = np.empty(n.value), np.empty(p.value)
    seed, noise, h = C.c_uint64(), C.c_double(), C.c_void_p()
    check(lib.l1g_problem_load(ctx.h, str(path).encode(), ptr(y), ptr(x), C.byref(seed),
                               C.byref(noise), C.byref(h)), "load_problem")
    op = DenseOperator(ctx=ctx, _handle=h.value, _dims=(n.value, p.value))
    return GeneratedProblem(op, y, x, noise.value, seed.value)


def save_problem(prob: GeneratedProblem, path):
    """problem_io.cpp save_problem (K read back from the device)."""
    y, x = _f64(prob.y), _f64(prob.x_true)
    if y.size != prob.op.rows() or x.size != prob.op.cols():
        raise ValueError("save_problem: inconsistent problem dimensions")
    check(L.load().l1g_problem_save(str(path).encode(), prob.op.h, ptr(y), ptr(x),
                                    int(prob.seed), float(prob.noise_level)), "save_problem")


def problem_hash(prob: GeneratedProblem) -> int:
    """problem_io.cpp problem_hash: FNV-1a 64 of the serialized L1PROBv1 bytes."""
    h = C.c_uint64()
    check(L.load().l1g_problem_hash(prob.op.h, ptr(_f64(prob.y)), ptr(_f64(prob.x_true)),
                                    int(prob.seed), float(prob.noise_level), C.byref(h)),
          "problem_hash")
    return h.value
