"""The reference minimizer on the device (reference.cpp:38-82) and the
constrained/penalized cross checks the reference's tests make with it.

* the device driver equals the oracle restatement bit for bit (the oracle is pinned to the
  reference's own source in tests/test_oracle_ref.py);
* test_gpss.cpp:377-391: GPSS at rho = ||x(lambda)||_1 reproduces the penalized minimizer to
  1e-6 and is projected-gradient stationary to 1e-7;
* acceptance_main.cpp:180-264 (criteria 4, 5, 6) on this harness's seeded Gaussian
  problems: every cell matches, lambda is recovered through the rho link, the telemetry
  invariants hold on every record, and FISTA beats ISTA at 500 matvecs.
"""
import math

import numpy as np
import pytest

import paper_0902_4424_b200 as l1
from oracle import oracle as O
from tests import problems as PB

pytestmark = pytest.mark.gpu


def gauss(seed, n=60, p=256, nnz=10, noise=0.02):
    """gen_gaussian_problem(n, p, nnz, noise, seed) shape (generators.cpp:99-117): ||K|| = 1,
    +-1 spikes, relative noise -- with this harness's Philox streams."""
    spec = O.ProblemSpec("gaussian", n, p, nnz, seed, "sign", noise, "rel", norm_target=1.0,
                         name=f"g{seed}")
    return O.build_problem(spec)


def test_device_reference_minimizer_bit_identical():
    P = O.build_problem(PB.C1)
    K, y = P["K"], P["y"]
    obj = l1.Objective(l1.DenseOperator(K), y)
    lmax = l1.lambda_max(obj.op(), y)
    assert lmax == float(np.abs(O.apply_adjoint(K, y)).max())
    for frac in (0.25, 1.0 / 64.0, 2.0):
        lam = lmax * frac
        ro = O.reference_minimizer(K, y, lam)
        rd = l1.reference_minimizer(obj, lam)
        assert np.array_equal(rd.x, ro["x"]) and rd.certificate == ro["certificate"]
        assert rd.rho == ro["rho"] and rd.nnz == ro["nnz"] and rd.iterations == ro["iterations"]
        assert rd.certificate <= 1e-12
        assert l1.penalized_fixed_point_residual(obj, rd.x, lam) == \
            O.penalized_fixed_point_residual(K, y, rd.x, lam)
    with pytest.raises(ValueError):
        l1.reference_minimizer(obj, -1.0)
    with pytest.raises(RuntimeError):  # not converged: the reference throws runtime_error
        l1.reference_minimizer(obj, lmax / 64.0, l1.ReferenceOptions(max_iterations=3))


def test_gpss_matches_penalized_reference_through_rho():
    """test_gpss.cpp:377-391."""
    P = gauss(73)
    obj = l1.Objective(l1.DenseOperator(P["K"]), P["y"])
    lam = l1.lambda_max(obj.op(), P["y"]) / 256.0
    ref = l1.reference_minimizer(obj, lam)
    assert ref.rho > 0.0
    sol = l1.gpss_solve(obj, l1.L1Ball(ref.rho), l1.GpConfig(),
                        l1.StopRule(max_iterations=20000, stationarity_tol=1e-12))
    assert np.linalg.norm(sol.x - ref.x) / np.linalg.norm(ref.x) <= 1e-6
    grad = obj.gradient(sol.x, l1.MatvecCounter())
    pg = l1.project_l1_ball(sol.x - grad, l1.L1Ball(ref.rho)) - sol.x
    assert np.abs(pg).max() <= 1e-7


def test_acceptance_criteria_4_5_6():
    """acceptance_main.cpp:180-264 over 10 seeds x 5 exponents."""
    agree = lam_ok = cells = wins = 0
    violations = 0
    for seed in range(1, 11):
        P = gauss(seed)
        op = l1.DenseOperator(P["K"])
        obj = l1.Objective(op, P["y"])
        lmax = l1.lambda_max(op, P["y"])
        for e in (2.0, 4.0, 6.0, 8.0, 10.0):
            lam = lmax * math.pow(2.0, -e)
            cells += 1
            ref = l1.reference_minimizer(obj, lam)
            recs = []
            sol = l1.gpss_solve(obj, l1.L1Ball(ref.rho), l1.GpConfig(),
                                l1.StopRule(max_iterations=40000, stationarity_tol=1e-12),
                                cb=lambda r, x: recs.append(r))
            if np.linalg.norm(sol.x - ref.x) / np.linalg.norm(ref.x) <= 1e-6:
                agree += 1
            if abs(l1.lambda_from_rho(op, P["y"], sol.x) - lam) / lam <= 1e-3:
                lam_ok += 1
            f_prev = math.inf
            for r in recs:  # criterion 5
                ok = 1e-10 <= r.alpha <= 1e10
                if math.isfinite(f_prev):
                    ok = ok and r.f <= f_prev + 1e-12 * max(1.0, f_prev)
                if r.bb_active:
                    ok = ok and r.bb2_raw <= r.bb1_raw * (1.0 + 1e-12)
                    ratio = r.tau_after / r.tau_before
                    ok = ok and (abs(ratio - 0.9) < 1e-12 or abs(ratio - 1.1) < 1e-12)
                violations += not ok
                f_prev = r.f
            race = l1.StopRule(max_iterations=0, max_matvecs=500, stationarity_tol=0.0)
            xi = l1.ista_solve(obj, l1.PenaltyWeight(lam), race)
            xf = l1.fista_solve(obj, l1.PenaltyWeight(lam), race)
            mv = l1.MatvecCounter()
            fi = obj.value(xi.x, mv) + 2.0 * lam * np.abs(xi.x).sum()
            ff = obj.value(xf.x, mv) + 2.0 * lam * np.abs(xf.x).sum()
            wins += ff <= fi
    assert agree == cells and lam_ok == cells
    assert violations == 0
    assert wins / cells >= 0.95
