"""Time the FP64 tensor-core batched products at the C5 shape (n=4096, p=16384, B=128)."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_0902_4424_b200 as l1  # noqa: E402
from paper_0902_4424_b200 import _lib as L  # noqa: E402

n, p, B = 4096, 16384, 128
op = l1.DenseOperator.generate_gaussian(n, p, 5)
lib = L.load()
X = np.random.default_rng(0).normal(size=(B, p))
R = np.random.default_rng(1).normal(size=(B, n))
Y = np.empty((B, n))
G = np.empty((B, p))
for _ in range(3):
    L.check(lib.l1g_op_apply_batched(op.h, B, L.ptr(X), L.ptr(Y)))
    L.check(lib.l1g_op_apply_adjoint_batched(op.h, B, L.ptr(R), L.ptr(G)))
print("ok")
