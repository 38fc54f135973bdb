"""The oracle restatement against the reference's own sources (oracle/_ref, CPU only).

oracle/_ref/libref_canon.so is /root/reference/proj/core/src/{gpss,prox,linear_operator,
objective}.cpp compiled unmodified against the Eigen stand-in (oracle/build_ref.sh).  With
the same reduction order the two must agree bit for bit, which pins every control-flow
decision and scalar formula of the restatement to the reference code itself.
"""
import numpy as np
import pytest

from oracle import oracle as O
from oracle import ref as R
from tests import problems as PB

pytestmark = pytest.mark.skipif(not R.available("canon"), reason="oracle/_ref not built")

FIELDS = ["k", "f", "stationarity", "alpha", "step", "matvecs", "bb_active", "bb1_raw",
          "bb2_raw", "tau_before", "tau_after", "f_max", "dir_derivative"]


def same(a, b):
    return a == b or (np.isnan(a) and np.isnan(b))


@pytest.mark.parametrize("spec,iters,memory", [
    (PB.C1, 500, 1), (PB.C2_MINI, 300, 1), (PB.C3_MINI, 400, 1), (PB.RAGGED, 200, 5),
    (PB.TINY, 50, 1), (PB.C4_MINI, 200, 3)], ids=lambda v: getattr(v, "name", str(v)))
def test_trajectory_bit_identical(spec, iters, memory):
    P = O.build_problem(spec)
    cfg, stop = O.GpConfig(memory=memory), O.StopRule(iters, 0, 0, 0.0)
    xo, ro, reco, _ = O.gpss_solve(P["K"], P["y"], P["rho"], cfg, stop)
    xr, rr, recr = R.RefOperator(P["K"]).gpss_solve(P["y"], P["rho"], cfg, stop)
    assert ro["iterations"] == rr["iterations"] and ro["reason"] == rr["reason"]
    assert ro["matvecs"] == rr["matvecs"]
    assert np.array_equal(xo, xr)
    assert ro["objective"] == rr["objective"] and ro["f_history"] == rr["f_history"]
    assert len(reco) == len(recr)
    for a, b in zip(reco, recr):
        for f in FIELDS:
            assert same(a[f], b[f]), (a["k"], f, a[f], b[f])


def test_projection_bit_identical():
    rng = np.random.default_rng(5)
    for rep in range(300):
        p = int(rng.integers(1, 400))
        x = rng.normal(size=p) * (10.0 ** rng.uniform(-3, 3))
        if rep % 7 == 0:
            x[rng.integers(0, p, size=max(1, p // 3))] = 0.0
        rho = float(rng.uniform(0.0, 1.2)) * float(np.abs(x).sum())
        u, th, _ = O.project_l1(x, rho)
        ur, thr = R.project_l1(x, rho)
        assert np.array_equal(u, ur) and th == thr


def test_operator_and_power_iteration():
    K = O.gaussian_matrix(9, 70, 230)
    op = R.RefOperator(K)
    rng = np.random.default_rng(2)
    for _ in range(5):
        x, r = rng.normal(size=230), rng.normal(size=70)
        assert np.array_equal(op.apply(x), O.apply(K, x))
        assert np.array_equal(op.apply(r, adjoint=True), O.apply_adjoint(K, r))
    assert op.spectral_norm() == O.spectral_norm(K)[0]


def test_literal_mode_within_tolerance():
    """Plain sequential reductions stay within the north-star tolerance of canonical ones
    on a trajectory that does not reach the arithmetic floor."""
    P = O.build_problem(PB.C2_MINI)
    cfg, stop = O.GpConfig(), O.StopRule(40, 0, 0, 0.0)
    xc, rc, recc, _ = O.gpss_solve(P["K"], P["y"], P["rho"], cfg, stop)
    with O.mode(O.LITERAL):
        xl, rl, recl, _ = O.gpss_solve(P["K"], P["y"], P["rho"], cfg, stop)
    assert np.linalg.norm(xc - xl) <= 1e-9 * np.linalg.norm(xc)
    assert abs(rc["objective"] - rl["objective"]) <= 1e-9 * abs(rc["objective"])


OTHER_FIELDS = ["k", "f", "stationarity", "alpha", "step", "matvecs"]


@pytest.mark.parametrize("spec,iters", [(PB.C1, 120), (PB.C2_MINI, 60), (PB.RAGGED, 80),
                                        (PB.TINY, 30)], ids=lambda v: getattr(v, "name", str(v)))
@pytest.mark.parametrize("solver", ["psd", "ista", "fista"])
def test_psd_ista_fista_bit_identical(spec, iters, solver):
    """psd.cpp / shrinkage.cpp: the restatement against the reference sources."""
    P = O.build_problem(spec)
    op = R.RefOperator(P["K"])
    for tol in (0.0, 1e-7):
        stop = O.StopRule(iters, 0, 0, tol, 1e-12 if tol else 0.0)
        if solver == "psd":
            xo, ro, reco = O.psd_solve(P["K"], P["y"], P["rho"], stop)
            xr, rr, recr = R.psd_solve(op, P["y"], P["rho"], stop)
        else:
            lam = 0.05 * float(np.abs(O.apply_adjoint(P["K"], P["y"])).max())
            acc = solver == "fista"
            xo, ro, reco = O.shrinkage_solve(P["K"], P["y"], lam, acc, stop)
            xr, rr, recr = R.shrinkage_solve(op, P["y"], lam, acc, stop)
        assert ro["iterations"] == rr["iterations"] and ro["reason"] == rr["reason"]
        assert ro["matvecs"] == rr["matvecs"]
        assert np.array_equal(xo, xr)
        assert ro["objective"] == rr["objective"] and ro["f_history"] == rr["f_history"]
        assert ro["stationarity"] == rr["stationarity"]
        for a, b in zip(reco, recr):
            for f in OTHER_FIELDS:
                assert same(a[f], b[f]), (a["k"], f, a[f], b[f])


def test_l1prob_format_matches_reference(tmp_path):
    """problem_io.cpp: the oracle's L1PROBv1 writer / reader / FNV-1a hash against the
    reference's own save_problem / load_problem / problem_hash."""
    rng = np.random.default_rng(9)
    for (n, p) in [(3, 4), (9, 21), (77, 301)]:
        K, y, x = rng.normal(size=(n, p)), rng.normal(size=n), rng.normal(size=p)
        seed, noise = int(rng.integers(0, 2**63)), float(rng.random())
        a, b = tmp_path / "a.l1prob", tmp_path / "b.l1prob"
        O.save_problem(a, K, y, x, seed, noise)
        R.problem_save(b, K, y, x, seed, noise)
        assert a.read_bytes() == b.read_bytes()
        assert len(a.read_bytes()) == 40 + 8 * (n * p + n + p)
        back = R.problem_load(a, n, p)
        assert np.array_equal(back["K"], K) and np.array_equal(back["y"], y)
        assert np.array_equal(back["x_true"], x)
        assert back["seed"] == seed and back["noise_level"] == noise
        mine = O.load_problem(b)
        assert np.array_equal(mine["K"], K) and mine["seed"] == seed
        assert O.problem_hash(K, y, x, seed, noise) == R.problem_hash(K, y, x, seed, noise)
    # documented offsets (test_operator.cpp:176-200): K(0,1) at byte 48
    K = np.arange(12.0).reshape(3, 4)
    O.save_problem(tmp_path / "c.l1prob", K, np.zeros(3), np.zeros(4), 123, 0.0)
    raw = (tmp_path / "c.l1prob").read_bytes()
    assert raw[:8] == b"L1PROBv1" and np.frombuffer(raw, "<f8", 1, 48)[0] == K[0, 1]


def test_reference_minimizer_bit_identical():
    """reference.cpp:38-82 restated (oracle) == the reference's own source (oracle/_ref)."""
    P = O.build_problem(PB.C1)
    K, y = P["K"], P["y"]
    lmax = float(np.abs(O.apply_adjoint(K, y)).max())
    op = R.RefOperator(K)
    for frac in (1.0 / 4.0, 1.0 / 64.0, 2.0):  # the last: lambda >= lambda_max -> zero
        lam = lmax * frac
        ro = O.reference_minimizer(K, y, lam)
        xr, cert, rho, nnz = op.reference_minimizer(y, lam)
        assert np.array_equal(ro["x"], xr) and ro["certificate"] == cert
        assert ro["rho"] == rho and ro["nnz"] == nnz
        assert ro["certificate"] <= 1e-12
    with pytest.raises(ValueError):
        O.reference_minimizer(K, y, 0.0)
