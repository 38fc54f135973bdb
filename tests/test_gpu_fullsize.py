"""BASELINE.json sizes on the device, through size-independent properties (the CPU oracle
cannot run these in test time): feasibility, monotone objective (memory 1), matvec
accounting, and equalities between execution strategies that must not change a bit --
dense vs support-sparse forward product, unsharded vs column-sharded."""
import ctypes as C
import json
import os

import numpy as np
import pytest

import paper_0902_4424_b200 as l1
from paper_0902_4424_b200 import _lib as L
from paper_0902_4424_b200 import harness as H
from paper_0902_4424_b200 import shard as S

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SIGMA = json.load(open(os.path.join(ROOT, "tests", "golden", "sigma_hat.json")))


def solve(h, iters):
    res, recs = S.solve(h, l1.StopRule(max_iterations=iters, stationarity_tol=0.0),
                        trace_cap=iters)
    return res, recs


def check_properties(res, recs, rho, x):
    assert np.abs(x).sum() <= rho * (1 + 1e-12) + 1e-12
    assert res.matvecs == 2 + 2 * res.iterations
    f = [r.f for r in recs]
    assert all(b <= a * (1 + 1e-12) for a, b in zip(f, f[1:]))


@pytest.fixture(scope="module")
def c2():
    spec = H.CONFIGS["C2"]
    spec.sigma_hat = SIGMA["C2"]
    return H.build_problem(spec)


def test_c2_dense_sparse_sharded_identical(c2):
    lib = L.load()
    cfg = l1.GpConfig()
    out = []
    for mode in ("sparse", "dense"):
        h = C.c_void_p()
        L.check(lib.l1g_solver_create(c2["op"].h, L.ptr(c2["y"]), c2["rho"], C.byref(cfg._c()),
                                      C.byref(h)))
        L.check(lib.l1g_solver_set_forward(h, int(mode == "sparse")))
        res, recs = solve(h, 300)
        out.append((res, recs, S.solver_x(h, 32768)))
        lib.l1g_solver_destroy(h)
    (ra, reca, xa), (rb, recb, xb) = out
    assert ra.iterations == rb.iterations and np.array_equal(xa, xb)
    assert [r.f for r in reca] == [r.f for r in recb]
    check_properties(ra, reca, c2["rho"], xa)
    # the same problem as 4 column shards of 8192 columns in one process
    spec = H.CONFIGS["C2"]
    ops = [H.build_operator(spec, col_offset=sh.col0, p_local=sh.p_local)[0]
           for sh in S.shard_plan(spec.p, 4)]
    hg = S.create_group_solver(ops, c2["y"], c2["rho"], cfg)
    try:
        rg, recg = solve(hg, 300)
        xg = S.solver_x(hg, spec.p)
    finally:
        lib.l1g_solver_destroy(hg)
    assert rg.iterations == ra.iterations and np.array_equal(xg, xa)
    assert [r.f for r in recg] == [r.f for r in reca]


def test_c5_batch_matches_single_solves():
    c = dict(H.C5)
    P = H.build_batch_problem(**c, sigma_hat=SIGMA["C5"])
    B, p = c["batch"], c["p"]
    iters = 12  # before any problem reaches its arithmetic floor
    X = np.empty((B, p))
    res = (L.ResultC * B)()
    L.check(L.load().l1g_gpss_solve_batched(
        P["op"].h, B, L.ptr(np.ascontiguousarray(P["Y"])), L.ptr(P["rho"]),
        C.byref(l1.GpConfig()._c()),
        C.byref(l1.StopRule(max_iterations=iters, stationarity_tol=0.0)._c()), L.ptr(X), res))
    for b in (0, 37, 127):
        sol = l1.gpss_solve(l1.Objective(P["op"], P["Y"][b]), l1.L1Ball(P["rho"][b]),
                            l1.GpConfig(), l1.StopRule(max_iterations=iters, stationarity_tol=0.0))
        assert res[b].iterations == sol.iterations == iters
        assert np.abs(X[b] - sol.x).max() <= 1e-9 * max(1.0, np.abs(sol.x).max())
        assert abs(res[b].objective - sol.objective) <= 1e-9 * abs(sol.objective)
        assert np.abs(X[b]).sum() <= P["rho"][b] * (1 + 1e-12) + 1e-12


def test_c4_full_size_steps():
    """68.7 GB operator on one B200: a few iterations, dense vs sparse forward identical."""
    spec = H.CONFIGS["C4"]
    spec.sigma_hat = SIGMA["C4"]
    P = H.build_problem(spec)
    lib = L.load()
    xs, fs = [], []
    for sparse in (1, 0):
        h = C.c_void_p()
        L.check(lib.l1g_solver_create(P["op"].h, L.ptr(P["y"]), P["rho"],
                                      C.byref(l1.GpConfig()._c()), C.byref(h)))
        L.check(lib.l1g_solver_set_forward(h, sparse))
        res, recs = solve(h, 6)
        xs.append(S.solver_x(h, spec.p))
        fs.append([r.f for r in recs])
        check_properties(res, recs, P["rho"], xs[-1])
        lib.l1g_solver_destroy(h)
    assert np.array_equal(xs[0], xs[1]) and fs[0] == fs[1]
    P["op"].close()
