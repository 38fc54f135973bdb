"""Approximation isochrones over a lambda grid (isochrone.cpp:35-246).

The GPSS cells of every grid point run in lockstep on the batched engine, resumed along the
budget ladder.  They must sample the same trajectories as the reference's per-point runs:
the per-point path (device drivers with callbacks, bit-identical to the oracle) gives the
exact samples, and the batched cells agree with them -- matvec counts exactly, relative
errors to the rounding of the tensor-core products.  The table format is the reference's
(fixed header, 17 significant digits, exact round trip).
"""
import io
import json

import numpy as np
import pytest

import paper_0902_4424_b200 as l1
from oracle import oracle as O
from paper_0902_4424_b200 import isochrone as I

pytestmark = pytest.mark.gpu
BUDGETS = [0, 3, 4, 9, 20, 50, 200, 1000]


@pytest.fixture(scope="module")
def campaign():
    spec = O.ProblemSpec("gaussian", 64, 256, 10, 91, "sign", 0.02, "rel", norm_target=1.0,
                         name="iso")
    P = O.build_problem(spec)
    op = l1.DenseOperator(P["K"])
    obj = l1.Objective(op, P["y"])
    grid = I.build_grid(op, P["y"], count=6, min_exp=0.5, max_exp=8.0)
    refs = I.reference_solutions(obj, grid)
    return P, obj, grid, refs


def test_grid(campaign):
    P, obj, grid, refs = campaign
    lmax = float(np.abs(O.apply_adjoint(P["K"], P["y"])).max())
    assert grid.lambda_max == lmax and grid.size() == 6
    assert all(a > b for a, b in zip(grid.lambdas, grid.lambdas[1:]))
    assert grid.lambdas[0] == lmax * 2.0 ** -0.5
    with pytest.raises(ValueError):
        I.build_grid(obj.op(), P["y"], count=1)
    with pytest.raises(ValueError):
        I.build_grid(obj.op(), np.zeros(64))


def test_batched_gpss_cells_follow_the_per_point_trajectories(campaign):
    P, obj, grid, refs = campaign
    opt = I.IsochroneOptions(budget_matvecs=BUDGETS, record_wall_time=False)
    batched = I.run_isochrones(obj, grid, [I.SolverId.Gpss], refs, opt)
    opt.batched_gpss = False
    single = I.run_isochrones(obj, grid, [I.SolverId.Gpss], refs, opt)
    assert len(batched) == len(single) == grid.size() * len(BUDGETS)
    for a, b in zip(batched, single):
        assert (a.lambda_index, a.budget_matvecs) == (b.lambda_index, b.budget_matvecs)
        assert a.matvecs_used <= a.budget_matvecs
        full = 0 if b.budget_matvecs < 4 else 2 * (b.budget_matvecs // 2)
        if b.matvecs_used == full and a.matvecs_used == full:
            assert abs(a.rel_error - b.rel_error) <= 1e-7 + 1e-6 * b.rel_error
        else:
            # a run that reached its arithmetic floor (stationary stop) may stop a few steps
            # apart under the tensor-core rounding; both sit at the floor
            assert a.matvecs_used < full and b.matvecs_used < full
            assert abs(a.rel_error - b.rel_error) <= 1e-6 + 1e-2 * b.rel_error
    # the per-point samples are the oracle's trajectory (bit-identical iterates)
    i = 3
    rho, xr = refs[i].rho, refs[i].x
    x_o, r_o, _, xs = O.gpss_solve(P["K"], P["y"], rho, O.GpConfig(),
                                   O.StopRule(600, 1000, 0, 1e-14), x_trace=True)
    for rec in (r for r in single if r.lambda_index == i and r.matvecs_used >= 4):
        k = (rec.matvecs_used - 2) // 2
        assert rec.rel_error == float(np.linalg.norm(xs[k - 1] - xr) / np.linalg.norm(xr))
    # budgets 0 and 3 fit no completed iteration: the zero start, error exactly 1
    assert [r.rel_error for r in batched if r.lambda_index == i][:2] == [1.0, 1.0]


def test_other_solvers_and_table(campaign):
    P, obj, grid, refs = campaign
    opt = I.IsochroneOptions(budget_matvecs=[10, 100], record_wall_time=False)
    recs = I.run_isochrones(obj, grid, [I.SolverId.Fista, I.SolverId.Psd, I.SolverId.Gpss],
                            refs, opt)
    assert [r.solver for r in recs[:2]] == [I.SolverId.Fista] * 2
    assert recs[-1].solver == I.SolverId.Gpss
    # one trajectory per cell, sampled at growing budgets
    for j in range(0, len(recs), 2):
        assert recs[j].matvecs_used <= recs[j + 1].matvecs_used <= 100
    csv = I.emit_isochrone_table(recs, "csv")
    lines = csv.strip().split("\n")
    assert lines[0] == ("solver,exponent,lambda,rho,nnz,budget_matvecs,budget_seconds,"
                        "rel_error,matvecs,seconds")
    row = lines[1].split(",")
    assert row[0] == "fista" and float(row[2]) == recs[0].lambda_ and float(row[7]) == recs[0].rel_error
    js = json.loads(I.emit_isochrone_table(recs, "json"))
    assert js[0]["solver"] == "fista" and js[0]["lambda"] == recs[0].lambda_
    out = io.StringIO()
    I.emit_isochrone_table(recs, "csv", out)
    assert out.getvalue() == csv
    with pytest.raises(ValueError):
        I.run_isochrones(obj, grid, [I.SolverId.Gpss], refs[:2], opt)
    with pytest.raises(ValueError):
        I.solver_from_string("adam")
    assert I.solver_from_string("gpss") == I.SolverId.Gpss
