"""The forward product's density switch (gemv.cu fwd_sparse_kernel -> fwd_dense_body): when d
has at least L1G_FWD_DENSE_FRAC * p nonzeros the iteration's K d runs as the dense TMA stream
instead of the support gather, decided on the device from the projection's nonzero count.
All three forward modes must give the oracle's bits (linear_operator.hpp:45, gpss.cpp:194):
0 = dense stream, 1 = sparse with the switch (default), 2 = sparse only."""
import ctypes as C

import numpy as np
import pytest

import paper_0902_4424_b200 as l1
from oracle import oracle as O
from paper_0902_4424_b200 import _lib as L
from paper_0902_4424_b200 import shard as S

pytestmark = pytest.mark.gpu

# rho well above ||x_true||_1: the ball constraint is inactive for the first steps, so h = v
# and d are dense; it becomes active (and d sparse) as the iterate grows -- both sides of the
# switch in one run
DENSE = O.ProblemSpec("gaussian", 256, 2048, 30, 21, "normal", 1e-2, "rel", rho_factor=6.0,
                      name="dense-d")
SPARSE = O.ProblemSpec("gaussian", 512, 2048, 25, 12, "normal", 1e-2, "rel", name="C2mini")


def run(P, mode, iters):
    lib = L.load()
    op = l1.DenseOperator(P["K"])
    h = C.c_void_p()
    cfg = l1.GpConfig()._c()
    y = np.ascontiguousarray(P["y"])
    L.check(lib.l1g_solver_create(op.h, L.ptr(y), P["rho"], C.byref(cfg), C.byref(h)))
    try:
        L.check(lib.l1g_solver_set_forward(h, mode))
        res, recs = S.solve(h, l1.StopRule(max_iterations=iters, stationarity_tol=0.0),
                            trace_cap=iters)
        x = S.solver_x(h, P["K"].shape[1])
        prof = (C.c_double * 32)()
        L.check(lib.l1g_solver_proj_profile(h, prof))
        return res, recs, x, prof[23]
    finally:
        lib.l1g_solver_destroy(h)


@pytest.mark.parametrize("spec", [DENSE, SPARSE], ids=lambda s: s.name)
def test_forward_modes_bit_identical(spec):
    P = O.build_problem(spec)
    iters = 60
    xo, ro, reco, _ = O.gpss_solve(P["K"], P["y"], P["rho"], O.GpConfig(),
                                   O.StopRule(iters, 0, 0, 0.0))
    dense_calls = {}
    for mode in (0, 1, 2):
        res, recs, x, nd = run(P, mode, iters)
        assert res.iterations == ro["iterations"], (mode, res.iterations, ro["iterations"])
        assert np.array_equal(x, xo), (mode, float(np.abs(x - xo).max()))
        assert [r.f for r in recs] == [r["f"] for r in reco]
        assert [r.support for r in recs] == [r["support"] for r in reco]
        dense_calls[mode] = nd
    assert dense_calls[2] == 0 and dense_calls[0] == 0  # the switch only acts in mode 1
    if spec is DENSE:
        assert dense_calls[1] > 0  # d was dense: the switch took the dense stream
    else:
        assert dense_calls[1] == 0  # d sparse throughout
