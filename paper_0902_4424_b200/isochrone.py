"""Approximation isochrones over a lambda grid (isochrone.hpp / isochrone.cpp:35-196), with
the constrained GPSS runs of every grid point solved in lockstep on the batched engine.

The reference runs each (solver, grid point) trajectory alone, samples it at a ladder of
matvec budgets (the last iterate whose matvec count fits the budget) and records the
relative error to the grid point's reference minimizer.  Here the GPSS runs of all grid
points share K, so they are one batched solve (B = grid points, rho_i = ||x(lambda_i)||_1,
products on the FP64 tensor cores): the batch runs to the smallest budget, every iterate is
read, and the same trajectories resume to the next budget (l1g_batch_resume) -- the
samples are the reference's, the products agree with the per-point solve to rounding
(DESIGN.md section 9).  ISTA / FISTA / PSD (and GPSS under wall-clock budgets) run per grid
point through the device drivers with the reference's callback sampling.
"""
from __future__ import annotations

import ctypes as C
import enum
import io
import json
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib as L
from . import api
from ._lib import check, ptr


class SolverId(enum.IntEnum):  # isochrone.hpp:13
    Ista = 0
    Fista = 1
    Psd = 2
    Gpss = 3


_NAMES = {SolverId.Ista: "ista", SolverId.Fista: "fista", SolverId.Psd: "psd",
          SolverId.Gpss: "gpss"}


def to_string(sid: SolverId) -> str:
    return _NAMES.get(SolverId(sid), "unknown")


def solver_from_string(name: str) -> SolverId:  # isochrone.cpp:28-33
    for k, v in _NAMES.items():
        if v == name:
            return k
    raise ValueError(f"unknown solver '{name}'; expected one of {{ista, fista, psd, gpss}}")


@dataclass
class LambdaGrid:  # isochrone.hpp:19-27
    lambda_max: float = 0.0
    exponents: List[float] = field(default_factory=list)
    lambdas: List[float] = field(default_factory=list)

    def size(self) -> int:
        return len(self.lambdas)


def build_grid(op, y, count: int = 50, min_exp: float = 0.5, max_exp: float = 16.0) -> LambdaGrid:
    """isochrone.cpp:35-52: lambda_i = lambda_max * 2^-e_i, e_i equally spaced."""
    if count < 2:
        raise ValueError("build_grid: count must be >= 2")
    if not max_exp > min_exp:
        raise ValueError("build_grid: need max_exp > min_exp")
    lmax = api.lambda_max(op, y)
    if lmax == 0.0:
        raise ValueError("build_grid: lambda_max is zero (zero data)")
    step = (max_exp - min_exp) / float(count - 1)
    ex = [min_exp + step * i for i in range(count)]
    return LambdaGrid(lmax, ex, [lmax * math.pow(2.0, -e) for e in ex])


@dataclass
class IsochroneRecord:  # isochrone.hpp:31-44
    solver: SolverId = SolverId.Ista
    lambda_index: int = 0
    exponent: float = 0.0
    lambda_: float = 0.0
    rho: float = 0.0
    nnz: int = 0
    budget_matvecs: int = 0
    budget_seconds: float = 0.0
    rel_error: float = 0.0
    matvecs_used: int = 0
    seconds_used: float = 0.0


@dataclass
class IsochroneOptions:  # isochrone.hpp:46-53
    budget_matvecs: List[int] = field(default_factory=list)
    budget_seconds: List[float] = field(default_factory=list)
    gp: api.GpConfig = field(default_factory=api.GpConfig)
    stationarity_tol: float = 1e-14
    jobs: int = 1
    record_wall_time: bool = True
    batched_gpss: bool = True   # B200: GPSS grid points in lockstep on the batched engine


def reference_solutions(prob: api.Objective, grid: LambdaGrid,
                        opt: Optional[api.ReferenceOptions] = None) -> List[api.ReferenceSolution]:
    """reference_minimizer at every grid point (the references run_isochrones needs)."""
    return [api.reference_minimizer(prob, lam, opt) for lam in grid.lambdas]


def _rel(x, x_ref, ref_norm):
    return float(np.linalg.norm(np.asarray(x) - x_ref) / ref_norm)


def _trace_run(sid, prob, lam, rho, x_ref, opt, mv_cap, s_cap):
    """isochrone.cpp:64-90: the zero start, then one sample per completed iteration."""
    ref_norm = float(np.linalg.norm(x_ref))
    samples = [(0, _rel(np.zeros_like(x_ref), x_ref, ref_norm), 0.0)]

    def cb(rec, x):
        samples.append((rec.matvecs, _rel(x, x_ref, ref_norm),
                        rec.elapsed_seconds if opt.record_wall_time else 0.0))

    stop = api.StopRule(max_iterations=0, max_matvecs=mv_cap, max_seconds=s_cap,
                        stationarity_tol=opt.stationarity_tol)
    if sid == SolverId.Ista:
        api.ista_solve(prob, api.PenaltyWeight(lam), stop, cb)
    elif sid == SolverId.Fista:
        api.fista_solve(prob, api.PenaltyWeight(lam), stop, cb)
    elif sid == SolverId.Psd:
        api.psd_solve(prob, api.L1Ball(rho), stop, cb)
    else:
        api.gpss_solve(prob, api.L1Ball(rho), opt.gp, stop, cb)
    return samples


def _at_budget(samples, budget, idx):  # isochrone.cpp:92-108
    best = samples[0]
    for s in samples:
        if s[idx] <= budget:
            best = s
        else:
            break
    return best


def _gpss_batched(prob, grid, refs, points, budgets_mv, opt):
    """The GPSS trajectories of `points` in lockstep: one batched solve per budget rung,
    resumed in place.  Returns {grid index: [(matvecs, rel_error, seconds) per budget]}."""
    op = api._require_dense(prob)
    lib = L.load()
    n, p = op.rows(), op.cols()
    B = len(points)
    Y = np.ascontiguousarray(np.tile(prob.y(), (B, 1)))
    rho = np.ascontiguousarray([refs[i].rho for i in points], dtype=np.float64)
    h = C.c_void_p()
    check(lib.l1g_batch_create(op.h, B, ptr(Y), ptr(rho), C.byref(opt.gp._c()), C.byref(h)),
          "isochrone batch")
    out = {i: [] for i in points}
    try:
        check(lib.l1g_batch_init(h, None), "isochrone batch init")
        res = (L.ResultC * B)()
        X = np.empty((B, p))
        xr = [refs[i].x for i in points]
        norms = [float(np.linalg.norm(v)) for v in xr]
        started = False
        for b in budgets_mv:
            if b < 4:  # no completed iteration fits: the zero start (isochrone.cpp:70)
                for j, i in enumerate(points):
                    out[i].append((0, _rel(np.zeros(p), xr[j], norms[j]), 0.0))
                continue
            # the last iterate with at most b matvecs has 2 * floor(b / 2): stop at the
            # first loop top whose count reaches 2 * floor(b / 2) - 1 (gpss.cpp:238)
            stop = api.StopRule(max_iterations=0, max_matvecs=2 * (b // 2) - 1,
                                stationarity_tol=opt.stationarity_tol)
            fn = lib.l1g_batch_resume if started else lib.l1g_batch_run
            check(fn(h, C.byref(stop._c()), res), "isochrone batch run")
            started = True
            check(lib.l1g_batch_get_x(h, ptr(X)), "isochrone batch x")
            for j, i in enumerate(points):
                used = res[j].matvecs if res[j].iterations > 0 else 0
                x = X[j] if res[j].iterations > 0 else np.zeros(p)
                out[i].append((used, _rel(x, xr[j], norms[j]),
                               res[j].elapsed_seconds if opt.record_wall_time else 0.0))
    finally:
        lib.l1g_batch_destroy(h)
    return out


def run_isochrones(prob: api.Objective, grid: LambdaGrid, solvers: Sequence[SolverId],
                   refs: Sequence[api.ReferenceSolution],
                   opt: IsochroneOptions) -> List[IsochroneRecord]:
    """isochrone.cpp:110-196: every (solver, grid point, budget) cell, ordered by (solver,
    grid point, budget); grid points with a zero reference are skipped."""
    if len(refs) != grid.size():
        raise ValueError(f"run_isochrones: need one reference per grid point (got {len(refs)} "
                         f"for {grid.size()} points)")
    if not opt.budget_matvecs and not opt.budget_seconds:
        raise ValueError("run_isochrones: no budgets given")
    bmv = sorted(opt.budget_matvecs)
    bs = sorted(opt.budget_seconds)
    mv_cap = bmv[-1] if bmv else 0
    s_cap = bs[-1] if bs else 0.0
    points = [i for i in range(grid.size()) if refs[i].rho != 0.0]
    batched = None
    if SolverId.Gpss in solvers and opt.batched_gpss and not bs and points:
        batched = _gpss_batched(prob, grid, refs, points, bmv, opt)
    records = []
    for sid in solvers:
        for i in points:
            base = dict(solver=SolverId(sid), lambda_index=i, exponent=grid.exponents[i],
                        lambda_=grid.lambdas[i], rho=refs[i].rho, nnz=refs[i].nnz)
            if sid == SolverId.Gpss and batched is not None:
                for b, (used, err, sec) in zip(bmv, batched[i]):
                    records.append(IsochroneRecord(**base, budget_matvecs=b, rel_error=err,
                                                   matvecs_used=used, seconds_used=sec))
                continue
            samples = _trace_run(sid, prob, grid.lambdas[i], refs[i].rho, refs[i].x, opt,
                                 mv_cap, s_cap)
            for b in bmv:
                s = _at_budget(samples, b, 0)
                records.append(IsochroneRecord(**base, budget_matvecs=b, rel_error=s[1],
                                               matvecs_used=s[0], seconds_used=s[2]))
            for b in bs:
                s = _at_budget(samples, b, 2)
                records.append(IsochroneRecord(**base, budget_seconds=b, rel_error=s[1],
                                               matvecs_used=s[0], seconds_used=s[2]))
    return records


def _fmt17(v: float) -> str:
    return "%.17g" % v


def emit_isochrone_table(records: Sequence[IsochroneRecord], fmt: str = "csv",
                         out=None) -> str:
    """isochrone.cpp:209-246: the fixed header, floats with 17 significant digits."""
    if not records:
        raise ValueError("emit_isochrone_table: no records")
    buf = io.StringIO()
    if fmt == "csv":
        buf.write("solver,exponent,lambda,rho,nnz,budget_matvecs,budget_seconds,rel_error,"
                  "matvecs,seconds\n")
        for r in records:
            buf.write(",".join([to_string(r.solver), _fmt17(r.exponent), _fmt17(r.lambda_),
                                _fmt17(r.rho), str(r.nnz), str(r.budget_matvecs),
                                _fmt17(r.budget_seconds), _fmt17(r.rel_error),
                                str(r.matvecs_used), _fmt17(r.seconds_used)]) + "\n")
    elif fmt == "json":
        rows = [{"solver": to_string(r.solver), "exponent": r.exponent, "lambda": r.lambda_,
                 "rho": r.rho, "nnz": r.nnz, "budget_matvecs": r.budget_matvecs,
                 "budget_seconds": r.budget_seconds, "rel_error": r.rel_error,
                 "matvecs": r.matvecs_used, "seconds": r.seconds_used} for r in records]
        buf.write(json.dumps(rows, indent=2) + "\n")
    else:
        raise ValueError("emit_isochrone_table: format is csv or json")
    text = buf.getvalue()
    if out is not None:
        if isinstance(out, str):
            with open(out, "w") as f:
                f.write(text)
        else:
            out.write(text)
    return text
