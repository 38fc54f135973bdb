"""Randomised differential run: the CUDA path against the CPU oracle, bit for bit.

Draws problem shapes, radii, configurations and starting points at random (seeded) and
compares whole GPSS runs (iterate, every record field, stop) and single projections with the
oracle.  Shapes are biased towards the boundaries of the kernels' plans: the one-cluster step
kernel (n_pad <= 384, p_pad <= 1024), one-CTA and cluster projections, tile and group
multiples +- 1.  Test infrastructure: the oracle is the checker, never the thing measured.

  python tools/fuzz_parity.py --seconds 120 --seed 1 [--out gpurun_out/fuzz.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import paper_0902_4424_b200 as l1  # noqa: E402
from oracle import oracle as O  # noqa: E402

FIELDS = ["k", "f", "stationarity", "alpha", "step", "matvecs", "bb_active", "halvings",
          "bb1_raw", "bb2_raw", "tau_before", "tau_after", "f_max", "dir_derivative", "theta",
          "support"]
EDGES_N = [1, 2, 31, 32, 33, 63, 64, 65, 127, 128, 129, 255, 256, 257, 383, 384, 385, 511, 513]
EDGES_P = [1, 2, 31, 33, 63, 64, 65, 255, 256, 257, 511, 512, 513, 1023, 1024, 1025, 2047, 2049,
           4095, 4096, 4097, 8191, 8193]


def same(a, b):
    return a == b or (isinstance(a, float) and np.isnan(a) and np.isnan(b))


def draw_dim(rng, edges, hi):
    if rng.random() < 0.45:
        return int(rng.choice(edges))
    return int(rng.integers(1, hi + 1))


def one_solve(rng, case):
    n = draw_dim(rng, EDGES_N, 600)
    p = draw_dim(rng, EDGES_P, 6000 if n <= 256 else 3000)
    K = rng.normal(size=(n, p)) * (10.0 ** rng.uniform(-2, 1)) / np.sqrt(max(n, p))
    if rng.random() < 0.15:  # sparse operator: exact zeros in products and sums
        K *= rng.random(size=K.shape) < 0.3
    nnz = int(rng.integers(0, max(1, min(p, 60)) + 1))
    xt = np.zeros(p)
    if nnz:
        xt[rng.choice(p, size=nnz, replace=False)] = rng.normal(size=nnz)
    y = K @ xt + rng.normal(size=n) * 10.0 ** rng.uniform(-4, -1)
    base = float(np.abs(xt).sum()) or 1.0
    rho = base * float(rng.choice([0.0, 1e-3, 0.2, 0.8, 1.0, 1.0, 1.0, 1.5, 4.0, 50.0]))
    cfg_kw = {}
    if rng.random() < 0.4:
        cfg_kw = dict(memory=int(rng.choice([1, 2, 5, 10])), tau1=float(rng.choice([0.2, 0.5, 0.9])),
                      alpha2_memory=int(rng.choice([1, 2, 4])),
                      alpha_min=float(rng.choice([1e-10, 1e-3])),
                      alpha_max=float(rng.choice([1e10, 1e2, 5.0])),
                      beta=float(rng.choice([1e-4, 1e-2])), theta=float(rng.choice([0.5, 0.25])))
    iters = int(rng.choice([1, 3, 40, 120]))
    tol = float(rng.choice([0.0, 0.0, 1e-9, 1e-4]))
    x0 = None
    kind = rng.random()
    if kind < 0.25:  # dense feasible start
        x0 = rng.normal(size=p)
        s = float(np.abs(x0).sum())
        x0 = x0 * (0.7 * rho / s) if (s > 0 and rho > 0) else np.zeros(p)
    elif kind < 0.30:  # infeasible start: rejected by both sides (L1Ball::contains, gpss.cpp:121)
        x0 = rng.normal(size=p) + 1.0
        x0 *= (2.0 * rho + 1.0) / float(np.abs(x0).sum())
    desc = dict(case=case, kind="solve", n=n, p=p, rho=rho, iters=iters, tol=tol, cfg=cfg_kw,
                x0=None if x0 is None else ("feasible" if kind < 0.25 else "free"))
    desc["iterations"] = 0
    if desc["x0"] == "free":
        errs = []
        for fn in (lambda: O.gpss_solve(K, y, rho, O.GpConfig(**cfg_kw),
                                        O.StopRule(iters, 0, 0, tol), x0=x0),
                   lambda: l1.gpss_solve(l1.Objective(l1.DenseOperator(K), y), l1.L1Ball(rho),
                                         l1.GpConfig(**cfg_kw),
                                         l1.StopRule(max_iterations=iters, stationarity_tol=tol),
                                         x0=x0)):
            try:
                fn()
                errs.append(None)
            except ValueError as e:
                errs.append(str(e))
        return desc, ([] if all(errs) else [("infeasible x0 accepted", errs)])
    xo, ro, reco, _ = O.gpss_solve(K, y, rho, O.GpConfig(**cfg_kw), O.StopRule(iters, 0, 0, tol),
                                   x0=x0)
    trace = []
    sol = l1.gpss_solve(l1.Objective(l1.DenseOperator(K), y), l1.L1Ball(rho), l1.GpConfig(**cfg_kw),
                        l1.StopRule(max_iterations=iters, stationarity_tol=tol), x0=x0, trace=trace)
    bad = []
    if sol.iterations != ro["iterations"]:
        bad.append(("iterations", sol.iterations, ro["iterations"]))
    if int(sol.reason) != ro["reason"]:
        bad.append(("reason", int(sol.reason), ro["reason"]))
    if sol.matvecs.count != ro["matvecs"]:
        bad.append(("matvecs", sol.matvecs.count, ro["matvecs"]))
    if not np.array_equal(sol.x, xo):
        bad.append(("x", float(np.abs(sol.x - xo).max())))
    if not same(sol.objective, ro["objective"]):
        bad.append(("objective", sol.objective, ro["objective"]))
    for a, b in zip(trace, reco):
        for f in FIELDS:
            if not same(getattr(a, f), b[f]):
                bad.append((f"rec[{b['k']}].{f}", getattr(a, f), b[f]))
                break
        if bad:
            break
    desc["iterations"] = ro["iterations"]
    return desc, bad


def one_projection(rng, case):
    big = rng.random() < 0.2
    p = int(rng.integers(1, 300000)) if big else draw_dim(rng, EDGES_P, 20000)
    style = rng.integers(0, 5)
    if style == 0:
        x = rng.normal(size=p) * (10.0 ** rng.uniform(-6, 6))
    elif style == 1:  # wide dynamic range
        x = rng.normal(size=p) * 10.0 ** rng.uniform(-12, 12, size=p)
    elif style == 2:  # few distinct magnitudes: ties in the sort, whole bins collide
        x = rng.choice([-1.0, 1.0, 0.5, -0.25, 2.0, 0.0], size=p)
    elif style == 3:  # coarse grid: rounding ties in the cumulative sum
        x = rng.integers(-4096, 4097, size=p).astype(np.float64) * 2.0 ** int(rng.integers(-30, 30))
    else:  # sparse
        x = rng.normal(size=p) * (rng.random(size=p) < 0.05)
    l1n = float(np.abs(x).sum())
    rho = l1n * float(rng.choice([0.0, 1e-6, 0.01, 0.3, 0.9, 0.999999, 1.0, 1.2]))
    desc = dict(case=case, kind="projection", p=p, style=int(style), rho=rho)
    u, th, sup = O.project_l1(x, rho)
    pr = l1.project_l1_ball_with_threshold(x, l1.L1Ball(rho))
    bad = []
    if pr.threshold != th:
        bad.append(("theta", pr.threshold, th))
    if pr.support != sup:
        bad.append(("support", pr.support, sup))
    if not np.array_equal(pr.point, u):
        bad.append(("point", float(np.abs(pr.point - u).max())))
    return desc, bad


def one_shard(rng, case):
    """Column-sharded in-process group (R shards in lockstep on one GPU, power-of-two shard
    widths) against the one-GPU solve: bit-identical trajectories."""
    from paper_0902_4424_b200 import _lib as L
    from paper_0902_4424_b200 import shard as S
    R = int(rng.choice([2, 4, 8]))
    w = int(rng.choice([256, 512, 1024]))
    p = R * w
    n = draw_dim(rng, EDGES_N, 400)
    K = rng.normal(size=(n, p)) / np.sqrt(max(n, p))
    nnz = int(rng.integers(1, 40))
    xt = np.zeros(p)
    xt[rng.choice(p, size=nnz, replace=False)] = rng.normal(size=nnz)
    y = K @ xt + rng.normal(size=n) * 1e-2
    rho = float(np.abs(xt).sum()) * float(rng.choice([0.0, 0.3, 1.0, 1.0, 3.0]))
    cfg = l1.GpConfig(memory=int(rng.choice([1, 3, 10])))
    iters = int(rng.choice([1, 2, 30, 90]))
    tol = float(rng.choice([0.0, 0.0, 1e-6]))
    fwd_mode = int(rng.choice([0, 1, 2]))
    x0 = None
    if rng.random() < 0.3 and rho > 0:
        x0 = rng.normal(size=p)
        x0 *= 0.5 * rho / float(np.abs(x0).sum())
    desc = dict(case=case, kind="shard", n=n, p=p, R=R, rho=rho, iters=iters, tol=tol,
                memory=cfg.memory, fwd=fwd_mode, x0=x0 is not None)
    stop = l1.StopRule(max_iterations=iters, stationarity_tol=tol)
    trace = []
    sol = l1.gpss_solve(l1.Objective(l1.DenseOperator(K), y), l1.L1Ball(rho), cfg, stop, x0=x0,
                        trace=trace)
    ops = [l1.DenseOperator(np.ascontiguousarray(K[:, sh.cols])) for sh in S.shard_plan(p, R)]
    h = S.create_group_solver(ops, y, rho, cfg)
    try:
        L.check(L.load().l1g_solver_set_forward(h, fwd_mode))
        res, recs = S.solve(h, stop, x0=x0, trace_cap=iters + 1)
        x = S.solver_x(h, p)
    finally:
        L.load().l1g_solver_destroy(h)
    bad = []
    if res.iterations != sol.iterations:
        bad.append(("iterations", res.iterations, sol.iterations))
    if res.reason != int(sol.reason):
        bad.append(("reason", res.reason, int(sol.reason)))
    if not np.array_equal(x, sol.x):
        bad.append(("x", float(np.abs(x - sol.x).max())))
    if not same(res.objective, sol.objective):
        bad.append(("objective", res.objective, sol.objective))
    for a, b in zip(recs, trace):
        for f in ["k", "f", "stationarity", "alpha", "step", "matvecs", "bb_active", "halvings",
                  "theta", "support", "f_max", "dir_derivative"]:
            if not same(getattr(a, f), getattr(b, f)):
                bad.append((f"rec[{b.k}].{f}", getattr(a, f), getattr(b, f)))
                break
        if bad:
            break
    return desc, bad


def one_other(rng, case):
    """psd / ista / fista device drivers against the oracle, bit for bit."""
    n = draw_dim(rng, EDGES_N, 400)
    p = draw_dim(rng, EDGES_P, 3000)
    K = rng.normal(size=(n, p)) / np.sqrt(max(n, p))
    nnz = int(rng.integers(0, min(p, 30) + 1))
    xt = np.zeros(p)
    if nnz:
        xt[rng.choice(p, size=nnz, replace=False)] = rng.normal(size=nnz)
    y = K @ xt + rng.normal(size=n) * 1e-2
    solver = str(rng.choice(["psd", "ista", "fista"]))
    iters = int(rng.choice([1, 5, 60]))
    tol = float(rng.choice([0.0, 1e-7]))
    ostop = O.StopRule(iters, 0, 0, tol, 1e-12 if tol else 0.0)
    stop = l1.StopRule(max_iterations=iters, stationarity_tol=tol,
                       objective_tol=1e-12 if tol else 0.0)
    obj = l1.Objective(l1.DenseOperator(K), y)
    trace = []
    desc = dict(case=case, kind="other", solver=solver, n=n, p=p, iters=iters, tol=tol)
    if solver == "psd":
        rho = (float(np.abs(xt).sum()) or 1.0) * float(rng.choice([0.0, 0.5, 1.0, 2.0]))
        desc["rho"] = rho
        xo, ro, reco = O.psd_solve(K, y, rho, ostop)
        sol = l1.psd_solve(obj, l1.L1Ball(rho), stop, trace=trace)
    else:
        lam = float(rng.choice([0.01, 0.05, 0.5, 1.5])) * float(np.abs(O.apply_adjoint(K, y)).max())
        desc["lam"] = lam
        xo, ro, reco = O.shrinkage_solve(K, y, lam, solver == "fista", ostop)
        fn = l1.fista_solve if solver == "fista" else l1.ista_solve
        sol = fn(obj, l1.PenaltyWeight(lam), stop, trace=trace)
    bad = []
    if sol.iterations != ro["iterations"] or int(sol.reason) != ro["reason"]:
        bad.append(("stop", sol.iterations, ro["iterations"], int(sol.reason), ro["reason"]))
    if not np.array_equal(sol.x, xo):
        bad.append(("x", float(np.abs(sol.x - xo).max())))
    if not same(sol.objective, ro["objective"]):
        bad.append(("objective", sol.objective, ro["objective"]))
    for a, b in zip(trace, reco):
        for f in ["k", "f", "stationarity", "alpha", "step", "matvecs"]:
            if not same(getattr(a, f), b[f]):
                bad.append((f"rec[{b['k']}].{f}", getattr(a, f), b[f]))
                break
        if bad:
            break
    return desc, bad


KINDS = {"solve": one_solve, "projection": one_projection, "shard": one_shard, "other": one_other}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kinds", default="solve,projection",
                    help="comma list of solve, projection, shard, other")
    ap.add_argument("--seconds", type=float, default=60.0)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    rng = np.random.default_rng(args.seed)
    t0 = time.time()
    kinds = args.kinds.split(",")
    cases, failures, counts = 0, [], {k: 0 for k in kinds}
    while time.time() - t0 < args.seconds:
        fn = KINDS[kinds[int(rng.integers(0, len(kinds)))]]
        desc, bad = fn(rng, cases)
        counts[desc["kind"]] += 1
        cases += 1
        if bad:
            failures.append(dict(desc=desc, bad=[[str(v) for v in b] for b in bad]))
            print("MISMATCH", json.dumps(failures[-1]), flush=True)
    summary = dict(seed=args.seed, seconds=round(time.time() - t0, 1), cases=cases, counts=counts,
                   failures=failures)
    print(json.dumps(dict(summary, failures=len(failures))))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(summary, f, indent=1)
    sys.exit(1 if failures else 0)


if __name__ == "__main__":
    main()
