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
