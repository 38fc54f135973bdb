"""The product's multi-rank sharded solver in separate processes.

Two processes, one column shard each, run libl1g's sharded solver end to end: rank-owned x
and g slices, the K d and [x | g | scalars] exchanges inside the iteration graphs.  The pool
gives one GPU, and NCCL refuses two ranks on one device, so the transport here is the
engine's host transport (pinned staging + a gloo allgather run as graph host nodes); the
device code and the graphs are the ones NCCL runs use.  No kernel ever waits on another
process: the host nodes do the waiting.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SPEC = dict(kind="gaussian", n=384, p=4096, nnz=30, seed=31, values="normal", noise=1e-2,
            noise_mode="rel")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_0902_4424_b200 as l1
    from oracle import oracle as O
    from paper_0902_4424_b200 import _lib as L
    from paper_0902_4424_b200 import shard as S
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    res = {}
    try:
        P = O.build_problem(O.ProblemSpec(**SPEC, name="mp"))
        sh = S.shard_plan(SPEC["p"], world)[rank]
        ctx = l1.Context(0)
        op = l1.DenseOperator(np.ascontiguousarray(P["K"][:, sh.cols]), ctx=ctx)
        comm = S.HostComm(ctx, rank, world, pg=dist)
        h = S.create_sharded_solver(op, comm, P["y"], P["rho"], l1.GpConfig())
        lib = L.load()
        try:
            r1, recs = S.solve(h, l1.StopRule(max_iterations=120, stationarity_tol=0.0),
                               trace_cap=120)
            res["x"] = S.solver_x(h, SPEC["p"])
            res["it"], res["reason"] = r1.iterations, r1.reason
            res["f"] = [rc.f for rc in recs]
            # a time budget: every rank must stop on the same iteration
            r2, _ = S.solve(h, l1.StopRule(max_iterations=100000, max_seconds=0.01,
                                           stationarity_tol=0.0))
            res["t_it"], res["t_reason"] = r2.iterations, r2.reason
            res["t_x"] = S.solver_x(h, SPEC["p"])
            res["errors"] = [repr(e) for e in comm.errors]
        finally:
            lib.l1g_solver_destroy(h)
            comm.close()
        dist.barrier()
    finally:
        dist.destroy_process_group()
    out.put((rank, res))


def test_two_process_sharded_solve_matches_single_gpu():
    import multiprocessing as mp

    import paper_0902_4424_b200 as l1
    from oracle import oracle as O
    P = O.build_problem(O.ProblemSpec(**SPEC, name="mp"))
    trace = []
    ref = l1.gpss_solve(l1.Objective(l1.DenseOperator(P["K"]), P["y"]), l1.L1Ball(P["rho"]),
                        l1.GpConfig(), l1.StopRule(max_iterations=120, stationarity_tol=0.0),
                        trace=trace)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = dict(q.get(timeout=600) for _ in procs)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    for rank in (0, 1):
        r = out[rank]
        assert not r["errors"], r["errors"]
        assert r["it"] == ref.iterations and r["reason"] == int(ref.reason)
        assert np.array_equal(r["x"], ref.x), np.abs(r["x"] - ref.x).max()
        assert r["f"] == [t.f for t in trace]
    # the time budget: the same stop iteration and iterate on both ranks
    assert out[0]["t_reason"] == out[1]["t_reason"] == 3  # StopReason::MaxSeconds
    assert out[0]["t_it"] == out[1]["t_it"]
    assert np.array_equal(out[0]["t_x"], out[1]["t_x"])
