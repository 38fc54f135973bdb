"""Bit-level parity at the BASELINE sizes (VERDICT r1 "Next" #1).

The CPU oracle (oracle/l1oracle.c, built with order-preserving OpenMP: outputs split over
threads, every reduction in one thread in the canonical order) runs the full problems:
  * C2 (BASELINE configs[1]): 8192 x 32768 Gaussian, run to its stop rule (300 iterations
    or the arithmetic-floor stop, gpss.cpp:180-189);
  * C3 (configs[2]): 16384 x 16384 blur, the first 300 of its 2000 iterations.
The GPU path must equal it bit for bit: the generated operator (downloaded from HBM), y, rho,
every iteration record, the stop iteration and reason, and the final x.  For C2 the
reference's own sources (oracle/_ref/libref_canon.so, compiled from /root/reference against
the Eigen stand-in) run the same problem as a third leg when they are present.
"""
import copy
import json
import os

import numpy as np
import pytest

import paper_0902_4424_b200 as l1
from oracle import oracle as O
from oracle import ref as R
from paper_0902_4424_b200 import harness as H
from tests import problems as PB

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SIGMA = json.load(open(os.path.join(ROOT, "tests", "golden", "sigma_hat.json")))

FIELDS = ["k", "f", "stationarity", "alpha", "step", "matvecs", "bb_active", "halvings",
          "bb1_raw", "bb2_raw", "tau_before", "tau_after", "f_max", "dir_derivative", "theta",
          "support"]
REF_FIELDS = ["k", "f", "stationarity", "alpha", "step", "matvecs", "bb_active", "bb1_raw",
              "bb2_raw", "tau_before", "tau_after", "f_max", "dir_derivative"]


def same(a, b):
    return a == b or (isinstance(a, float) and np.isnan(a) and np.isnan(b))


def compare_records(gpu_recs, cpu_recs, fields, get):
    assert len(gpu_recs) == len(cpu_recs)
    for a, b in zip(gpu_recs, cpu_recs):
        for f in fields:
            assert same(get(a, f), b[f]), (b["k"], f, get(a, f), b[f])


@pytest.mark.parametrize("name,iters", [("C2", 300), ("C3", 300)])
def test_fullsize_bit_identical(name, iters):
    hspec = copy.copy(H.CONFIGS[name])
    ospec = copy.copy(getattr(PB, name))
    if hspec.kind == "gaussian":
        hspec.sigma_hat = ospec.sigma_hat = SIGMA[name]
    P = O.build_problem(ospec)                       # host: oracle generators
    D = H.build_problem(hspec)                       # device: generated into tiled HBM
    assert np.array_equal(D["op"].matrix(), P["K"])  # the 2 GiB operator, every bit
    assert np.array_equal(D["y"], P["y"]) and D["rho"] == P["rho"]

    stop_o = O.StopRule(iters, 0, 0, 0.0)
    xo, ro, reco, _ = O.gpss_solve(P["K"], P["y"], P["rho"], O.GpConfig(), stop_o)
    trace = []
    sol = l1.gpss_solve(l1.Objective(D["op"], D["y"]), l1.L1Ball(D["rho"]), l1.GpConfig(),
                        l1.StopRule(max_iterations=iters, stationarity_tol=0.0), trace=trace)
    assert sol.iterations == ro["iterations"] and int(sol.reason) == ro["reason"]
    assert sol.matvecs.count == ro["matvecs"]
    assert np.array_equal(sol.x, xo), float(np.abs(sol.x - xo).max())
    assert sol.objective == ro["objective"] and list(sol.f_history) == ro["f_history"]
    compare_records(trace, reco, FIELDS, getattr)

    if name == "C2" and R.available("canon"):  # the reference's own sources, same problem
        xr, rr, recr = R.RefOperator(P["K"]).gpss_solve(P["y"], P["rho"], O.GpConfig(), stop_o)
        assert rr["iterations"] == ro["iterations"] and rr["reason"] == ro["reason"]
        assert np.array_equal(xr, xo) and rr["objective"] == ro["objective"]
        compare_records(reco, recr, REF_FIELDS, lambda r, f: r[f])
    D["op"].close()


# comparison windows of the literal (sequential-sum) reference reading, measured by
# tools/divergence.py at full size (profiles/r02_divergence.json)
WINDOWS = {"C2": 79, "C3": 111}


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_fullsize_within_tolerance_of_literal_reference(name):
    """North star: iterates and objective within 1e-9 (relative) of the reference's own
    arithmetic, equal support outside the 1e-12 band, the same accepted steplength rule and
    halvings, at every iteration of the config's window -- GPU against the literal oracle
    (bit-identical to oracle/_ref/libref_fast.so, the reference sources, per
    profiles/r02_divergence.json)."""
    hspec = copy.copy(H.CONFIGS[name])
    ospec = copy.copy(getattr(PB, name))
    if hspec.kind == "gaussian":
        hspec.sigma_hat = ospec.sigma_hat = SIGMA[name]
    w = WINDOWS[name]
    P = O.build_problem(ospec)
    D = H.build_problem(hspec)
    with O.mode(O.LITERAL):
        _, _, recl, xhl = O.gpss_solve(P["K"], P["y"], P["rho"], O.GpConfig(),
                                       O.StopRule(w, 0, 0, 0.0), x_trace=True)
    xs, trace = [], []
    l1.gpss_solve(l1.Objective(D["op"], D["y"]), l1.L1Ball(D["rho"]), l1.GpConfig(),
                  l1.StopRule(max_iterations=w, stationarity_tol=0.0),
                  cb=lambda rec, x: xs.append(x), trace=trace)
    assert len(xs) == len(recl) == w
    for i in range(w):
        a, b = xs[i], xhl[i]
        assert np.linalg.norm(a - b) <= 1e-9 * np.linalg.norm(b), i + 1
        assert abs(trace[i].f - recl[i]["f"]) <= 1e-9 * abs(recl[i]["f"]), i + 1
        assert trace[i].bb_active == recl[i]["bb_active"], i + 1
        assert trace[i].halvings == recl[i]["halvings"], i + 1
        big = (np.abs(a) > 1e-12) | (np.abs(b) > 1e-12)
        assert not np.any(((a != 0) != (b != 0)) & big), i + 1
    D["op"].close()
