"""The run graph is an execution detail: a whole run as one WHILE-loop graph (conditional node,
abi.cu make_while_graph), with one iteration per loop body, or the host-polled chunked graphs
(L1G_LOOP_GRAPH=0, what profiled runs use) must give bit-identical runs."""
import ctypes as C

import numpy as np
import pytest

import paper_0902_4424_b200 as l1
from oracle import oracle as O
from paper_0902_4424_b200 import _lib as L
from tests import problems as PB
from tests.test_gpu_batch import batch_problems
from tests.test_gpu_parity import FIELDS, same

pytestmark = pytest.mark.gpu

# chunked graphs; the WHILE loop; one iteration per loop body; a profiler's injection
# environment (ncu sets NV_COMPUTE_PROFILER_PERFWORKS_DIR): chunked graphs again
MODES = [{"L1G_LOOP_GRAPH": "0"}, {}, {"L1G_LOOP_US": "1"},
         {"NV_COMPUTE_PROFILER_PERFWORKS_DIR": "/nonexistent"}]


def _set_mode(monkeypatch, env):
    for k in ("L1G_LOOP_GRAPH", "L1G_LOOP_US", "NV_COMPUTE_PROFILER_PERFWORKS_DIR"):
        monkeypatch.delenv(k, raising=False)
    for k, v in env.items():
        monkeypatch.setenv(k, v)


@pytest.mark.parametrize("spec,iters,tol", [(PB.C2_MINI, 300, 0.0), (PB.RAGGED, 200, 0.0),
                                            (PB.C1, 120, 1e-6)],
                         ids=lambda v: getattr(v, "name", str(v)))
def test_single_run_graph_modes(spec, iters, tol, monkeypatch):
    P = O.build_problem(spec)
    runs = []
    for env in MODES:
        _set_mode(monkeypatch, env)
        op = l1.DenseOperator(P["K"])  # a fresh operator: its cached solver builds new graphs
        trace = []
        sol = l1.gpss_solve(l1.Objective(op, P["y"]), l1.L1Ball(P["rho"]), l1.GpConfig(),
                            l1.StopRule(max_iterations=iters, stationarity_tol=tol), trace=trace)
        runs.append((sol, trace))
    s0, t0 = runs[0]
    for sol, trace in runs[1:]:
        assert sol.iterations == s0.iterations
        assert int(sol.reason) == int(s0.reason)
        assert sol.matvecs.count == s0.matvecs.count
        assert np.array_equal(sol.x, s0.x)
        assert sol.objective == s0.objective
        assert len(trace) == len(t0)
        for a, b in zip(trace, t0):
            for f in FIELDS:
                assert same(getattr(a, f), getattr(b, f)), (b.k, f)


def test_batched_run_graph_modes(monkeypatch):
    n, p, B, iters = 256, 1024, 6, 40
    K, Y, rho = batch_problems(n, p, B, 77)
    lib = L.load()
    cfg = l1.GpConfig()._c()
    stop = l1.StopRule(max_iterations=iters, stationarity_tol=0.0)._c()
    outs = []
    for env in MODES[:2]:
        _set_mode(monkeypatch, env)
        op = l1.DenseOperator(K)
        X = np.empty((B, p))
        res = (L.ResultC * B)()
        L.check(lib.l1g_gpss_solve_batched(op.h, B, L.ptr(np.ascontiguousarray(Y)), L.ptr(rho),
                                           C.byref(cfg), C.byref(stop), L.ptr(X), res), "batched")
        outs.append((X, [(res[b].iterations, res[b].reason, res[b].objective) for b in range(B)]))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert outs[0][1] == outs[1][1]
