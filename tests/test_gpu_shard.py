"""Column-sharded solver on one GPU.

The in-process shard group runs R shards in lockstep with device copies as the exchange;
the NCCL transport is exercised with a one-rank communicator.  With p/R a power of two the
sharded trajectory must equal the unsharded one (and the oracle's) bit for bit.
"""
import numpy as np
import pytest

import paper_0902_4424_b200 as l1
from oracle import oracle as O
from paper_0902_4424_b200 import _lib as L
from paper_0902_4424_b200 import shard as S

pytestmark = pytest.mark.gpu

SPEC = O.ProblemSpec("gaussian", 512, 4096, 30, 21, "normal", 1e-2, "rel", name="shard4096")
FIELDS = ["k", "f", "stationarity", "alpha", "step", "matvecs", "bb_active", "halvings",
          "theta", "support", "f_max", "dir_derivative"]


@pytest.fixture(scope="module")
def problem():
    P = O.build_problem(SPEC)
    op = l1.DenseOperator(P["K"])
    trace = []
    sol = l1.gpss_solve(l1.Objective(op, P["y"]), l1.L1Ball(P["rho"]), l1.GpConfig(),
                        l1.StopRule(max_iterations=150, stationarity_tol=0.0), trace=trace)
    return P, sol, trace


def shard_ops(K, nranks):
    return [l1.DenseOperator(np.ascontiguousarray(K[:, sh.cols]))
            for sh in S.shard_plan(K.shape[1], nranks)]


def check_same(res, recs, x, sol, trace):
    assert res.iterations == sol.iterations
    assert res.reason == int(sol.reason)
    assert np.array_equal(x, sol.x), np.abs(x - sol.x).max()
    assert res.objective == sol.objective
    assert len(recs) == len(trace)
    for a, b in zip(recs, trace):
        for f in FIELDS:
            va, vb = getattr(a, f), getattr(b, f)
            assert va == vb or (np.isnan(va) and np.isnan(vb)), (b.k, f, va, vb)


@pytest.mark.parametrize("nranks", [1, 2, 4, 8])
@pytest.mark.parametrize("sparse", [1, 0])
def test_group_bit_identical(problem, nranks, sparse):
    P, sol, trace = problem
    ops = shard_ops(P["K"], nranks)
    h = S.create_group_solver(ops, P["y"], P["rho"], l1.GpConfig())
    try:
        L.check(L.load().l1g_solver_set_forward(h, sparse))
        res, recs = S.solve(h, l1.StopRule(max_iterations=150, stationarity_tol=0.0), trace_cap=200)
        x = S.solver_x(h, SPEC.p)
    finally:
        L.load().l1g_solver_destroy(h)
    check_same(res, recs, x, sol, trace)


def test_group_x0_and_repeat(problem):
    P, _, _ = problem
    x0 = np.zeros(SPEC.p)
    x0[::97] = 0.5 * P["rho"] / len(x0[::97])
    op = l1.DenseOperator(P["K"])
    trace = []
    ref = l1.gpss_solve(l1.Objective(op, P["y"]), l1.L1Ball(P["rho"]), l1.GpConfig(memory=3),
                        l1.StopRule(max_iterations=60, stationarity_tol=0.0), x0=x0, trace=trace)
    ops = shard_ops(P["K"], 4)
    h = S.create_group_solver(ops, P["y"], P["rho"], l1.GpConfig(memory=3))
    try:
        for _ in range(2):  # a second solve on the same workspace gives the same bits
            res, recs = S.solve(h, l1.StopRule(max_iterations=60, stationarity_tol=0.0), x0=x0,
                                trace_cap=100)
            check_same(res, recs, S.solver_x(h, SPEC.p), ref, trace)
    finally:
        L.load().l1g_solver_destroy(h)


def test_group_unaligned_shards_close(problem):
    """p/R not a power of two: a different (deterministic) column tree, same solution."""
    spec = O.ProblemSpec("gaussian", 256, 1536, 12, 22, "normal", 1e-2, "rel", name="s1536")
    P = O.build_problem(spec)
    op = l1.DenseOperator(P["K"])
    ref = l1.gpss_solve(l1.Objective(op, P["y"]), l1.L1Ball(P["rho"]), l1.GpConfig(),
                        l1.StopRule(max_iterations=40, stationarity_tol=0.0))
    xs = []
    for _ in range(2):
        ops = shard_ops(P["K"], 2)  # 768 columns per shard
        h = S.create_group_solver(ops, P["y"], P["rho"], l1.GpConfig())
        try:
            res, _ = S.solve(h, l1.StopRule(max_iterations=40, stationarity_tol=0.0))
            xs.append(S.solver_x(h, spec.p))
        finally:
            L.load().l1g_solver_destroy(h)
    assert np.array_equal(xs[0], xs[1])
    assert np.abs(xs[0] - ref.x).max() <= 1e-9 * max(1.0, np.abs(ref.x).max())


def test_group_rejects_bad_shards(problem):
    P, _, _ = problem
    a = l1.DenseOperator(np.ascontiguousarray(P["K"][:, :300]))
    b = l1.DenseOperator(np.ascontiguousarray(P["K"][:, 300:600]))
    with pytest.raises(ValueError):
        S.create_group_solver([a, b], P["y"], P["rho"], l1.GpConfig())  # 300 % 256 != 0
    c = l1.DenseOperator(np.ascontiguousarray(P["K"][:, :512]))
    d = l1.DenseOperator(np.ascontiguousarray(P["K"][:, :1024]))
    with pytest.raises(ValueError):
        S.create_group_solver([c, d], P["y"], P["rho"], l1.GpConfig())  # unequal shards


def test_nccl_single_rank(problem):
    """The NCCL transport (runtime-loaded libnccl, allgather captured in the graph)."""
    P, sol, trace = problem
    ctx = l1.default_context()
    uid = (np.zeros(128, dtype=np.uint8))
    L.check(L.load().l1g_comm_unique_id(uid.ctypes.data), "unique_id")
    comm = S.Comm(ctx, 0, 1, uid.tobytes())
    op = l1.DenseOperator(P["K"])
    h = S.create_sharded_solver(op, comm, P["y"], P["rho"], l1.GpConfig())
    try:
        res, recs = S.solve(h, l1.StopRule(max_iterations=150, stationarity_tol=0.0), trace_cap=200)
        x = S.solver_x(h, SPEC.p)
    finally:
        L.load().l1g_solver_destroy(h)
        comm.close()
    check_same(res, recs, x, sol, trace)
