"""Bit-level parity of a whole BASELINE run at full size, GPU against the CPU oracle
(oracle/l1oracle.c with order-preserving OpenMP: outputs split over threads, every reduction
in one thread in the canonical order).  The headline config C4 (32768 x 262144, 68.7 GB, 200
iterations) takes the oracle ~15 minutes on the GPU box's host cores, too long for the test
suite (tests/test_gpu_fullsize_parity.py runs C2 to its stop and C3 for 300 iterations), so
it is recorded here:

  python tools/fullsize_parity.py --config C4 --iters 200 > profiles/r02_fullsize_parity_c4.json

Compared bit for bit: y, rho, every iteration record (all fields), the stop iteration and
reason, the objective and the final x.  The operator itself is generated on each side by the
same Philox/Box-Muller code (bit-identical at every size tested); every record depends on
all of K through the adjoint, so a single differing entry would show in the first g.
"""
import argparse
import copy
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_0902_4424_b200 as l1  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_0902_4424_b200 import harness as H  # noqa: E402
from tests import problems as PB  # noqa: E402

FIELDS = ["k", "f", "stationarity", "alpha", "step", "matvecs", "bb_active", "halvings",
          "bb1_raw", "bb2_raw", "tau_before", "tau_after", "f_max", "dir_derivative", "theta",
          "support"]


def same(a, b):
    return a == b or (isinstance(a, float) and np.isnan(a) and np.isnan(b))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--iters", type=int, default=200)
    a = ap.parse_args()
    sig = json.load(open(os.path.join(ROOT, "tests", "golden", "sigma_hat.json")))
    hspec = copy.copy(H.CONFIGS[a.config])
    ospec = copy.copy(getattr(PB, a.config))
    if hspec.kind == "gaussian":
        hspec.sigma_hat = ospec.sigma_hat = sig[a.config]
    out = {"config": a.config, "n": hspec.n, "p": hspec.p, "iterations_requested": a.iters,
           "threads": os.cpu_count()}
    t = time.time()
    D = H.build_problem(hspec)
    trace = []
    sol = l1.gpss_solve(l1.Objective(D["op"], D["y"]), l1.L1Ball(D["rho"]), l1.GpConfig(),
                        l1.StopRule(max_iterations=a.iters, stationarity_tol=0.0), trace=trace)
    out["gpu_seconds"] = round(time.time() - t, 2)
    D["op"].close()
    t = time.time()
    P = O.build_problem(ospec)
    out["host_build_seconds"] = round(time.time() - t, 2)
    out["y_equal"] = bool(np.array_equal(D["y"], P["y"]))
    out["rho_equal"] = bool(D["rho"] == P["rho"])
    t = time.time()
    xo, ro, reco, _ = O.gpss_solve(P["K"], P["y"], P["rho"], O.GpConfig(),
                                   O.StopRule(a.iters, 0, 0, 0.0))
    out["oracle_seconds"] = round(time.time() - t, 2)
    out["iterations"] = [sol.iterations, ro["iterations"]]
    out["reason"] = [int(sol.reason), ro["reason"]]
    out["objective_equal"] = bool(sol.objective == ro["objective"])
    out["x_equal"] = bool(np.array_equal(sol.x, xo))
    out["max_abs_dx"] = float(np.abs(sol.x - xo).max())
    bad = []
    for rg, rc in zip(trace, reco):
        for f in FIELDS:
            if not same(getattr(rg, f), rc[f]):
                bad.append([rc["k"], f])
    out["records_compared"] = min(len(trace), len(reco))
    out["record_mismatches"] = bad[:20]
    out["bit_identical"] = bool(out["y_equal"] and out["rho_equal"] and out["x_equal"] and
                                out["objective_equal"] and not bad and
                                out["iterations"][0] == out["iterations"][1] and
                                out["reason"][0] == out["reason"][1])
    out["final_objective"] = ro["objective"]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
