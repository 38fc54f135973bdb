"""Seeded synthetic problems built on the device (BASELINE.json configs).

Mirror of oracle.oracle.build_problem: the same Philox streams, the same canonical
reductions, so the operator, y, x_true and rho are bit-identical to the oracle's
(tests/test_gpu_harness.py).  K is generated directly into the tiled HBM layout, which is
how the 68.7 GB config C4 is built without a host copy.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib as L
from . import api
from ._lib import check, ptr

BLUR_SIGMA, BLUR_RADIUS = 4.0, 12


@dataclass
class ProblemSpec:
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
    sigma_hat: Optional[float] = None
    name: str = field(default="")


CONFIGS = {
    "C1": ProblemSpec("gaussian", 256, 1024, 20, 1, "sign", 1e-3, "abs", name="C1"),
    "C2": ProblemSpec("gaussian", 8192, 32768, 400, 2, "normal", 1e-2, "rel", name="C2"),
    "C3": ProblemSpec("blur", 16384, 16384, 300, 3, "usign", 1e-3, "abs", rho_factor=0.8,
                      name="C3"),
    "C4": ProblemSpec("gaussian", 32768, 262144, 4000, 4, "normal", 1e-2, "rel", name="C4"),
}
ITERATIONS = {"C1": 500, "C2": 300, "C3": 2000, "C4": 200, "C5": 300}

# C5: one Gaussian K shared by B problems (BASELINE.json configs[4])
C5 = dict(n=4096, p=16384, batch=128, nnz=150, seed=5, noise=1e-3)


def rng(ctx, kind, seed, stream, first, count) -> np.ndarray:
    out = np.empty(max(count, 1))
    check(L.load().l1g_rng_fill(ctx.h, kind, seed, stream, first, count, ptr(out)), "rng_fill")
    return out[:count]


def blur_taps(sigma=BLUR_SIGMA, radius=BLUR_RADIUS) -> np.ndarray:
    w = [math.exp(-(k * k) / (2.0 * sigma * sigma)) for k in range(-radius, radius + 1)]
    s = 0.0
    for v in w:
        s += v
    return np.array([v / s for v in w])


def sample_support(ctx, seed, stream, p, k) -> np.ndarray:
    """Partial Fisher-Yates on the uniform stream (same as orc_sample_support)."""
    if k < 0 or k > p:
        raise ValueError("sample_support: k must lie in [0, p]")
    u = rng(ctx, 1, seed, stream, 0, k)
    pool = np.arange(p, dtype=np.int64)
    for t in range(k):
        j = t + int(math.floor(u[t] * float(p - t)))
        if j >= p:
            j = p - 1
        pool[t], pool[j] = pool[j], pool[t]
    return pool[:k].copy()


def x_true_values(ctx, spec: ProblemSpec, count: int) -> np.ndarray:
    s, st = spec.seed, 3
    if spec.values == "sign":
        u = rng(ctx, 1, s, st, 0, count)
        return np.where(u < 0.5, 1.0, -1.0)
    if spec.values == "normal":
        return rng(ctx, 0, s, st, 0, count)
    if spec.values == "usign":
        u = rng(ctx, 1, s, st, 0, 2 * count)
        out = []
        for t in range(count):
            mag = 0.5 + 1.5 * float(u[2 * t])
            out.append(mag if u[2 * t + 1] < 0.5 else -mag)
        return np.array(out)
    raise ValueError(spec.values)


def build_operator(spec: ProblemSpec, ctx=None, col_offset: int = 0, p_local: int = 0):
    """Returns (op, sigma_hat, scale).  With p_local > 0 only columns
    [col_offset, col_offset + p_local) are materialised (one rank's shard); the spectral
    norm must then come from spec.sigma_hat."""
    ctx = ctx or api.default_context()
    if spec.kind == "gaussian":
        pl = p_local or spec.p
        op = api.DenseOperator.generate_gaussian(spec.n, pl, spec.seed, ctx=ctx,
                                                 col_offset=col_offset, p_total=spec.p)
        if spec.sigma_hat is not None:
            sigma_hat = spec.sigma_hat
        else:
            if p_local and p_local != spec.p:
                raise ValueError("sharded operator needs spec.sigma_hat")
            sigma_hat = api.spectral_norm_estimate(op, spec.power_iters, spec.power_tol)
        scale = spec.norm_target / sigma_hat
        op.scale(scale)
        return op, sigma_hat, scale
    if spec.kind == "blur":
        if spec.n != spec.p or p_local:
            raise ValueError("blur operator is square and unsharded")
        return api.DenseOperator.generate_blur(spec.n, blur_taps(), BLUR_RADIUS, ctx=ctx), \
            math.nan, 1.0
    raise ValueError(spec.kind)


def build_vectors(spec: ProblemSpec, op, ctx=None):
    """x_true, y, rho for an operator covering all columns."""
    ctx = ctx or api.default_context()
    x_true = np.zeros(spec.p)
    sup = sample_support(ctx, spec.seed, 1, spec.p, spec.nnz)
    x_true[sup] = x_true_values(ctx, spec, spec.nnz)
    clean = op.apply(x_true)
    e = rng(ctx, 0, spec.seed, 2, 0, spec.n)
    if spec.noise_mode == "abs":
        sig = spec.noise
    else:
        sig = spec.noise * math.sqrt(api.squared_norm(clean, ctx)) / math.sqrt(spec.n)
    y = clean + sig * e
    rho = spec.rho_factor * api.l1_norm(x_true, ctx)
    return dict(x_true=x_true, y=y, rho=rho, noise_sigma=sig, support=sup)


def build_problem(spec: ProblemSpec, ctx=None):
    op, sigma_hat, scale = build_operator(spec, ctx)
    d = build_vectors(spec, op, ctx)
    d.update(op=op, sigma_hat=sigma_hat, scale=scale)
    return d


def build_batch_problem(n, p, batch, nnz, seed, noise, ctx=None, sigma_hat=None,
                        power_iters=1000, power_tol=1e-8):
    """BASELINE C5 recipe: K iid N(0,1) (Philox stream 0 of `seed`) scaled to ||K||_2 = 0.9;
    problem j has its own x_true (nnz N(0,1) values at positions sampled from seed
    1000*seed + j), y_j = K x_true_j + noise * e_j, rho_j = (0.2 + 0.8 j/(B-1)) ||x_true_j||_1.
    Returns dict(op, Y (B x n), rho (B,), X_true (B x p), sigma_hat)."""
    ctx = ctx or api.default_context()
    spec = ProblemSpec("gaussian", n, p, nnz, seed, "normal", noise, "abs",
                       sigma_hat=sigma_hat, power_iters=power_iters, power_tol=power_tol)
    op, sig, _ = build_operator(spec, ctx)
    Y = np.empty((batch, n))
    X = np.zeros((batch, p))
    rho = np.empty(batch)
    for j in range(batch):
        sj = 1000 * seed + j
        sub = ProblemSpec("gaussian", n, p, nnz, sj, "normal", noise, "abs")
        sup = sample_support(ctx, sj, 1, p, nnz)
        X[j, sup] = x_true_values(ctx, sub, nnz)
        clean = op.apply(X[j])
        Y[j] = clean + noise * rng(ctx, 0, sj, 2, 0, n)
        rho[j] = (0.2 + 0.8 * j / max(batch - 1, 1)) * api.l1_norm(X[j], ctx)
    return dict(op=op, Y=Y, rho=rho, X_true=X, sigma_hat=sig)
