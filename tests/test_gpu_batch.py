"""Batched-RHS products on the FP64 tensor cores (dmma.cu, BASELINE config C5).

DMMA accumulates with fused multiply-adds in its own order, so these are compared with the
canonical single-RHS products (oracle) to a tolerance written here: |error| <= 1e-13 times
the sum of |K_ij x_j| (a rounding-error bound with a safety margin).
"""
import ctypes as C

import numpy as np
import pytest

import paper_0902_4424_b200 as l1
from oracle import oracle as O
from paper_0902_4424_b200 import _lib as L

pytestmark = pytest.mark.gpu
TOL = 1e-13


def batched(op, X, adjoint=False):
    lib = L.load()
    B = X.shape[0]
    n, p = op.rows(), op.cols()
    out = np.empty((B, p if adjoint else n))
    X = np.ascontiguousarray(X, dtype=np.float64)
    fn = lib.l1g_op_apply_adjoint_batched if adjoint else lib.l1g_op_apply_batched
    L.check(fn(op.h, B, L.ptr(X), L.ptr(out)), "batched")
    return out


@pytest.mark.parametrize("n,p,B", [(300, 1000, 1), (300, 1000, 5), (512, 2048, 128),
                                   (96, 4096, 130), (1024, 512, 33)])
def test_batched_products(n, p, B):
    rng = np.random.default_rng(n + p + B)
    K = rng.normal(size=(n, p))
    op = l1.DenseOperator(K)
    X = rng.normal(size=(B, p)) * (rng.random((B, p)) < 0.2)
    R = rng.normal(size=(B, n))
    Y = batched(op, X)
    G = batched(op, R, adjoint=True)
    for b in range(B):
        ref = O.apply(K, X[b])
        bound = np.abs(K) @ np.abs(X[b])
        assert np.all(np.abs(Y[b] - ref) <= TOL * bound + 1e-300), b
        refg = O.apply_adjoint(K, R[b])
        boundg = np.abs(K).T @ np.abs(R[b])
        assert np.all(np.abs(G[b] - refg) <= TOL * boundg + 1e-300), b


def batch_problems(n, p, B, seed):
    """B problems on one Gaussian K: distinct sparse x_true, y = K x_true + noise, rho_b
    spaced from 0.2 to 1.0 of ||x_true_b||_1 (the C5 recipe at a small size)."""
    K = O.gaussian_matrix(seed, n, p)
    sig, _ = O.spectral_norm(K, 200, 1e-10)
    K *= 0.9 / sig
    rng = np.random.default_rng(seed)
    Y, rho, xt = [], [], []
    for b in range(B):
        x = np.zeros(p)
        idx = rng.choice(p, size=max(3, p // 60), replace=False)
        x[idx] = rng.normal(size=idx.size)
        y = O.apply(K, x) + 1e-3 * rng.normal(size=n)
        Y.append(y)
        rho.append((0.2 + 0.8 * b / max(B - 1, 1)) * float(np.abs(x).sum()))
        xt.append(x)
    return K, np.array(Y), np.array(rho)


@pytest.mark.parametrize("n,p,B,iters,strict", [
    (256, 1024, 6, 15, True), (200, 2048, 130, 15, True), (1024, 4096, 16, 20, True),
    (512, 2048, 16, 80, False), (256, 1024, 6, 60, False)])
def test_batched_solve_matches_single(n, p, B, iters, strict):
    """Every problem of the batch against its own canonical solve.  Away from the arithmetic
    floor the iterates agree to ~1e-15 (tolerance 1e-9, equal steps); once a run reaches the
    floor (gpss.cpp:180-189: no descent left at rounding level) the stop iteration may differ
    by a few steps and the iterates agree to the floor's own resolution (1e-7 here), the
    objective to 1e-9."""
    K, Y, rho = batch_problems(n, p, B, 31 + B)
    op = l1.DenseOperator(K)
    lib = L.load()
    cfg = l1.GpConfig()._c()
    stop = l1.StopRule(max_iterations=iters, stationarity_tol=0.0)._c()
    X = np.empty((B, p))
    res = (L.ResultC * B)()
    L.check(lib.l1g_gpss_solve_batched(op.h, B, L.ptr(np.ascontiguousarray(Y)), L.ptr(rho),
                                       C.byref(cfg), C.byref(stop), L.ptr(X), res), "batched")
    for b in range(0, B, max(1, B // 8)):
        sol = l1.gpss_solve(l1.Objective(op, Y[b]), l1.L1Ball(rho[b]), l1.GpConfig(),
                            l1.StopRule(max_iterations=iters, stationarity_tol=0.0))
        scale = max(1.0, np.abs(sol.x).max())
        if strict:
            assert res[b].iterations == sol.iterations == iters, b
            assert res[b].reason == int(sol.reason), b
            assert res[b].matvecs == sol.matvecs.count, b
            assert np.abs(X[b] - sol.x).max() <= 1e-9 * scale, (b, np.abs(X[b] - sol.x).max())
        else:
            assert np.abs(X[b] - sol.x).max() <= 1e-7 * scale, (b, np.abs(X[b] - sol.x).max())
        assert abs(res[b].objective - sol.objective) <= 1e-9 * abs(sol.objective), b
        assert np.abs(X[b]).sum() <= rho[b] * (1 + 1e-12) + 1e-12


_COMPACT_SNIPPET = r"""
import ctypes as C, sys, numpy as np
sys.path.insert(0, {root!r})
import paper_0902_4424_b200 as l1
from paper_0902_4424_b200 import _lib as L
from tests.test_gpu_batch import batch_problems
K, Y, rho = batch_problems(256, 2048, 140, 77)
op = l1.DenseOperator(K)
lib = L.load()
cfg = l1.GpConfig()._c()
stop = l1.StopRule(max_iterations=400, stationarity_tol=0.0)._c()
B = Y.shape[0]
X = np.empty((B, 2048))
res = (L.ResultC * B)()
L.check(lib.l1g_gpss_solve_batched(op.h, B, L.ptr(np.ascontiguousarray(Y)), L.ptr(rho),
                                   C.byref(cfg), C.byref(stop), L.ptr(X), res), "batched")
np.savez({out!r}, X=X, its=np.array([res[b].iterations for b in range(B)]),
         f=np.array([res[b].objective for b in range(B)]),
         reason=np.array([res[b].reason for b in range(B)]))
"""


def test_compaction_bit_identical(tmp_path):
    """Products on the compacted live problems (dead blocks, warp groups and tiles skipped,
    either projection plan) give every problem the bits of the in-place full-width products:
    a 140-problem batch (two problem blocks) run to every problem's stop, with problems
    stopping at different iterations, in three processes (the switches are read once)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for name, env in [("plain", {"L1G_BATCH_COMPACT": "0"}),
                      ("compact", {"L1G_BATCH_COMPACT": "1", "L1G_BATCH_PROJ_TWO": "0"}),
                      ("compact2", {"L1G_BATCH_COMPACT": "1", "L1G_BATCH_PROJ_TWO": "1"})]:
        out = str(tmp_path / f"{name}.npz")
        e = dict(os.environ, **env)
        r = subprocess.run([sys.executable, "-c", _COMPACT_SNIPPET.format(root=root, out=out)],
                           env=e, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(out))
    a = outs[0]
    assert len(set(a["its"].tolist())) > 3  # the problems do stop at different iterations
    for b in outs[1:]:
        assert np.array_equal(a["its"], b["its"]) and np.array_equal(a["reason"], b["reason"])
        assert np.array_equal(a["f"], b["f"])
        assert np.array_equal(a["X"], b["X"])
