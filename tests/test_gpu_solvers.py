"""PSD, ISTA and FISTA on the device kernels against the oracle, bit for bit.

The oracle's restatements of psd.cpp / shrinkage.cpp are pinned to the reference sources in
tests/test_oracle_ref.py; the device drivers use the canonical GEMVs, the exact projection
and element-wise kernels with rounded products, so every record must match exactly.
"""
import numpy as np
import pytest

import paper_0902_4424_b200 as l1
from oracle import oracle as O
from tests import problems as PB

pytestmark = pytest.mark.gpu
FIELDS = ["k", "f", "stationarity", "alpha", "step", "matvecs"]


@pytest.mark.parametrize("spec,iters", [(PB.C1, 150), (PB.C2_MINI, 80), (PB.RAGGED, 80),
                                        (PB.C3_MINI, 60)], ids=lambda v: getattr(v, "name", str(v)))
@pytest.mark.parametrize("solver", ["psd", "ista", "fista"])
def test_solver_bit_identical(spec, iters, solver):
    P = O.build_problem(spec)
    obj = l1.Objective(l1.DenseOperator(P["K"]), P["y"])
    for tol in (0.0, 1e-7):
        ostop = O.StopRule(iters, 0, 0, tol, 1e-12 if tol else 0.0)
        stop = l1.StopRule(max_iterations=iters, stationarity_tol=tol,
                           objective_tol=1e-12 if tol else 0.0)
        trace, seen = [], []
        cb = lambda rec, x: seen.append((rec.k, x))  # noqa: E731
        if solver == "psd":
            xo, ro, reco = O.psd_solve(P["K"], P["y"], P["rho"], ostop)
            sol = l1.psd_solve(obj, l1.L1Ball(P["rho"]), stop, cb=cb, trace=trace)
        else:
            lam = 0.05 * float(np.abs(O.apply_adjoint(P["K"], P["y"])).max())
            xo, ro, reco = O.shrinkage_solve(P["K"], P["y"], lam, solver == "fista", ostop)
            fn = l1.fista_solve if solver == "fista" else l1.ista_solve
            sol = fn(obj, l1.PenaltyWeight(lam), stop, cb=cb, trace=trace)
        assert sol.iterations == ro["iterations"] and int(sol.reason) == ro["reason"]
        assert sol.matvecs.count == ro["matvecs"]
        assert np.array_equal(sol.x, xo), np.abs(sol.x - xo).max()
        assert sol.objective == ro["objective"] and list(sol.f_history) == ro["f_history"]
        assert sol.stationarity == ro["stationarity"]
        assert len(trace) == len(reco) == len(seen)
        for a, b in zip(trace, reco):
            for f in FIELDS:
                assert getattr(a, f) == b[f], (b["k"], f, getattr(a, f), b[f])
        if seen:
            assert np.array_equal(seen[-1][1], sol.x)
