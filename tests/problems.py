"""Seeded synthetic problems for parity tests (BASELINE.json configs and reduced sizes).

Sizes here are chosen so the CPU oracle finishes in seconds; the full BASELINE sizes are
exercised on the GPU through size-independent properties (see tests/test_gpu_*.py).
"""
from oracle import oracle as O

# BASELINE.json configs[0..4] (C4/C5 full sizes are GPU-only)
C1 = O.ProblemSpec("gaussian", 256, 1024, 20, 1, "sign", 1e-3, "abs", name="C1")
C2 = O.ProblemSpec("gaussian", 8192, 32768, 400, 2, "normal", 1e-2, "rel", name="C2")
C3 = O.ProblemSpec("blur", 16384, 16384, 300, 3, "usign", 1e-3, "abs", rho_factor=0.8, name="C3")
C4 = O.ProblemSpec("gaussian", 32768, 262144, 4000, 4, "normal", 1e-2, "rel", name="C4")
C5_K = dict(n=4096, p=16384, batch=128, nnz=150, seed=5, noise=1e-3)

ITERS = {"C1": 500, "C2": 300, "C3": 2000, "C4": 200, "C5": 300}

# reduced-size stand-ins with the same distributions (oracle-checkable in seconds)
C2_MINI = O.ProblemSpec("gaussian", 512, 2048, 25, 12, "normal", 1e-2, "rel", name="C2mini")
C3_MINI = O.ProblemSpec("blur", 512, 512, 10, 13, "usign", 1e-3, "abs", rho_factor=0.8,
                        name="C3mini")
C4_MINI = O.ProblemSpec("gaussian", 384, 3000, 40, 14, "normal", 1e-2, "rel", name="C4mini")
RAGGED = O.ProblemSpec("gaussian", 77, 301, 9, 15, "sign", 1e-3, "abs", name="ragged")
TINY = O.ProblemSpec("gaussian", 3, 5, 2, 16, "sign", 1e-3, "abs", name="tiny")
