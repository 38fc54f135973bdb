"""North-star tolerance against the reference's literal arithmetic, inside each config's
comparison window (profiles/r02_divergence.json).

The GPU reproduces the canonical oracle bit for bit (tests/test_gpu_*parity.py).  The
reference itself sums sequentially (oracle/_ref/libref_fast.so, the reference's own sources:
bit-identical to the oracle's LITERAL mode, checked below).  Two legal summation orders
drift apart at a rate set by the problem's conditioning, so the north star's bar -- relative
iterate and objective error <= 1e-9, equal support where the margin exceeds 1e-12, the same
accepted steplength rule every iteration -- holds over a finite window per config, measured
by tools/divergence.py.  Inside the window every iteration must meet the bar.
"""
import numpy as np
import pytest

from oracle import oracle as O
from oracle import ref as R
from tests import problems as PB

TOL, BAND = 1e-9, 1e-12
# windows measured by tools/divergence.py (profiles/r02_divergence.json, "window")
WINDOWS = {"C1": 94, "C2mini": 81, "C3mini": 105, "C4mini": 200}
SPECS = {"C1": PB.C1, "C2mini": PB.C2_MINI, "C3mini": PB.C3_MINI, "C4mini": PB.C4_MINI}


def support_agrees(a, b):
    big = (np.abs(a) > BAND) | (np.abs(b) > BAND)
    return not np.any(((a != 0) != (b != 0)) & big)


def check_window(xhc, recc, xhl, recl, window):
    assert len(recc) >= window and len(recl) >= window
    for i in range(window):
        a, b = xhc[i], xhl[i]
        assert np.linalg.norm(a - b) <= TOL * np.linalg.norm(a), i + 1
        assert abs(recc[i]["f"] - recl[i]["f"]) <= TOL * abs(recc[i]["f"]), i + 1
        assert recc[i]["bb_active"] == recl[i]["bb_active"], i + 1
        assert recc[i]["halvings"] == recl[i]["halvings"], i + 1
        assert support_agrees(a, b), i + 1


@pytest.mark.parametrize("name", sorted(WINDOWS))
def test_canonical_vs_literal_inside_window(name):
    P = O.build_problem(SPECS[name])
    stop = O.StopRule(WINDOWS[name], 0, 0, 0.0)
    with O.mode(O.CANONICAL):
        _, _, recc, xhc = O.gpss_solve(P["K"], P["y"], P["rho"], O.GpConfig(), stop, x_trace=True)
    with O.mode(O.LITERAL):
        xl, rl, recl, xhl = O.gpss_solve(P["K"], P["y"], P["rho"], O.GpConfig(), stop,
                                         x_trace=True)
    check_window(xhc, recc, xhl, recl, WINDOWS[name])
    if R.available("fast"):  # LITERAL mode is the reference sources' own arithmetic
        xf, rf, recf = R.RefOperator(P["K"], "fast").gpss_solve(P["y"], P["rho"], O.GpConfig(),
                                                                stop)
        assert np.array_equal(xf, xl) and rf["objective"] == rl["objective"]
        assert [r["f"] for r in recf] == [r["f"] for r in recl]
