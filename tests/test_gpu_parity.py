"""Bit-level parity of the B200 path with the CPU oracle on seeded problems.

The oracle (oracle/l1oracle.c) is itself checked bit-for-bit against the reference's own
sources (tests/test_oracle_ref.py).  With the canonical reduction order the GPU
must reproduce every iterate, every telemetry field and the stop iteration exactly; values
are compared with ==, so +0.0 and -0.0 count as equal.
"""
import numpy as np
import pytest

import paper_0902_4424_b200 as l1
from oracle import oracle as O
from tests import problems as PB

pytestmark = pytest.mark.gpu

FIELDS = ["k", "f", "stationarity", "alpha", "step", "matvecs", "bb_active", "halvings",
          "bb1_raw", "bb2_raw", "tau_before", "tau_after", "f_max", "dir_derivative", "theta",
          "support"]


def same(a, b):
    return a == b or (isinstance(a, float) and np.isnan(a) and np.isnan(b))


def run_both(spec, iters, memory=1, tol=0.0):
    P = O.build_problem(spec)
    xo, ro, reco, _ = O.gpss_solve(P["K"], P["y"], P["rho"], O.GpConfig(memory=memory),
                                   O.StopRule(iters, 0, 0, tol))
    op = l1.DenseOperator(P["K"])
    trace = []
    sol = l1.gpss_solve(l1.Objective(op, P["y"]), l1.L1Ball(P["rho"]), l1.GpConfig(memory=memory),
                        l1.StopRule(max_iterations=iters, stationarity_tol=tol), trace=trace)
    return P, (xo, ro, reco), (sol, trace)


@pytest.mark.parametrize("spec,iters,memory", [
    (PB.TINY, 50, 1), (PB.RAGGED, 200, 5), (PB.C1, 500, 1), (PB.C2_MINI, 300, 1),
    (PB.C3_MINI, 400, 1), (PB.C4_MINI, 200, 3)], ids=lambda v: getattr(v, "name", str(v)))
def test_trajectory_bit_identical(spec, iters, memory):
    P, (xo, ro, reco), (sol, trace) = run_both(spec, iters, memory)
    assert sol.iterations == ro["iterations"]
    assert int(sol.reason) == ro["reason"]
    assert sol.matvecs.count == ro["matvecs"]
    assert np.array_equal(sol.x, xo), np.abs(sol.x - xo).max()
    assert sol.objective == ro["objective"]
    assert list(sol.f_history) == ro["f_history"]
    assert len(trace) == len(reco)
    for a, b in zip(trace, reco):
        for f in FIELDS:
            assert same(getattr(a, f), b[f]), (b["k"], f, getattr(a, f), b[f])


def test_operator_bit_identical():
    rng = np.random.default_rng(3)
    for (n, p) in [(1, 1), (5, 8), (77, 301), (256, 1024), (129, 257), (700, 2100)]:
        K = rng.normal(size=(n, p))
        op = l1.DenseOperator(K)
        x, r = rng.normal(size=p), rng.normal(size=n)
        assert np.array_equal(op.apply(x), O.apply(K, x))
        assert np.array_equal(op.apply_adjoint(r), O.apply_adjoint(K, r))
        assert np.array_equal(op.matrix(), K)


def test_projection_bit_identical():
    rng = np.random.default_rng(5)
    for rep in range(200):
        p = int(rng.integers(1, 3000))
        x = rng.normal(size=p) * (10.0 ** rng.uniform(-3, 3))
        if rep % 7 == 0:
            x[rng.integers(0, p, size=max(1, p // 3))] = 0.0
        rho = float(rng.uniform(0.0, 1.2)) * float(np.abs(x).sum())
        u, th, sup = O.project_l1(x, rho)
        pr = l1.project_l1_ball_with_threshold(x, l1.L1Ball(rho))
        assert np.array_equal(pr.point, u) and pr.threshold == th and pr.support == sup


@pytest.mark.parametrize("p", [40000, 131072, 262144])
def test_projection_large(p):
    """Cluster path (cs > 1) and the global-memory sort for large candidate sets."""
    rng = np.random.default_rng(p)
    vectors = [rng.normal(size=p),
               # few distinct magnitudes: whole key bins collide (unbalanced bucket ranges)
               rng.choice([-1.0, 1.0, 0.5, -0.25, 2.0], size=p) * (rng.random(p) < 0.7)]
    for x in vectors:
        for frac in (0.9, 0.3, 0.01):
            rho = frac * float(np.abs(x).sum())
            u, th, sup = O.project_l1(x, rho)
            pr = l1.project_l1_ball_with_threshold(x, l1.L1Ball(rho))
            assert pr.threshold == th and pr.support == sup
            assert np.array_equal(pr.point, u)


@pytest.mark.parametrize("p", [400000, 1048576, 3000000])
def test_projection_beyond_shared_memory(p):
    """p > 262 144: the cluster keeps v in the L2-resident global scratch (M = 64 .. 512)."""
    rng = np.random.default_rng(p)
    x = rng.normal(size=p)
    for frac in (0.5, 0.02):
        rho = frac * float(np.abs(x).sum())
        u, th, sup = O.project_l1(x, rho)
        pr = l1.project_l1_ball_with_threshold(x, l1.L1Ball(rho))
        assert pr.threshold == th and pr.support == sup
        assert np.array_equal(pr.point, u)


def test_trajectory_beyond_shared_memory():
    """A whole solve with p = 600 000 (projection with v in global scratch) equals the oracle."""
    spec = O.ProblemSpec("gaussian", 64, 600000, 40, 31, "normal", 1e-2, "rel",
                         sigma_hat=800.0, name="wide")
    P = O.build_problem(spec)
    iters = 25
    xo, ro, reco, _ = O.gpss_solve(P["K"], P["y"], P["rho"], O.GpConfig(),
                                   O.StopRule(iters, 0, 0, 0.0))
    trace = []
    sol = l1.gpss_solve(l1.Objective(l1.DenseOperator(P["K"]), P["y"]), l1.L1Ball(P["rho"]),
                        l1.GpConfig(), l1.StopRule(max_iterations=iters, stationarity_tol=0.0),
                        trace=trace)
    assert sol.iterations == ro["iterations"]
    assert np.array_equal(sol.x, xo), float(np.abs(sol.x - xo).max())
    assert [r.f for r in trace] == [r["f"] for r in reco]
    assert [r.support for r in trace] == [r["support"] for r in reco]


@pytest.mark.parametrize("p", [65536, 262144])
def test_projection_cluster_prefix_ties(p):
    """The cluster-wide exact prefix (> 8192 candidates, project.cu prefix_break_cluster) on
    values from a coarse grid: many equal magnitudes (rank-sort ties) and running sums whose
    next addend is an odd multiple of half a grid step (rounding ties resolved by parity
    segments composed across CTAs)."""
    rng = np.random.default_rng(p + 3)
    for grid_bits, frac in ((12, 0.95), (20, 0.6), (8, 0.8)):
        x = rng.integers(1, 1 << grid_bits, size=p) * 2.0 ** -grid_bits
        x *= rng.choice([-1.0, 1.0], size=p)
        rho = frac * float(np.abs(x).sum())
        u, th, sup = O.project_l1(x, rho)
        pr = l1.project_l1_ball_with_threshold(x, l1.L1Ball(rho))
        assert pr.threshold == th and pr.support == sup, (grid_bits, frac)
        assert np.array_equal(pr.point, u)


def test_generators_bit_identical():
    K = O.gaussian_matrix(11, 130, 333)
    op = l1.DenseOperator.generate_gaussian(130, 333, 11)
    assert np.array_equal(op.matrix(), K)
    taps = O.blur_taps()
    opb = l1.DenseOperator.generate_blur(200, taps, O.BLUR_RADIUS)
    assert np.array_equal(opb.matrix(), O.blur_matrix(200, taps))
    # column shard of a larger matrix (multi-GPU layout)
    sh = l1.DenseOperator.generate_gaussian(130, 100, 11, col_offset=200, p_total=333)
    assert np.array_equal(sh.matrix(), K[:, 200:300])


def test_spectral_norm_bit_identical():
    K = O.gaussian_matrix(21, 150, 420)
    op = l1.DenseOperator.generate_gaussian(150, 420, 21)
    mv = l1.MatvecCounter()
    s = l1.spectral_norm_estimate(op, 1000, 1e-8, mv)
    so, mvo = O.spectral_norm(K, 1000, 1e-8)
    assert s == so and mv.count == mvo


def test_gp_iterate_steps_match_solve():
    P = O.build_problem(PB.C2_MINI)
    st = O.GpState(P["K"], P["y"], P["rho"])
    obj = l1.Objective(l1.DenseOperator(P["K"]), P["y"])
    ball, cfg, mv = l1.L1Ball(P["rho"]), l1.GpConfig(), l1.MatvecCounter()
    gs = l1.gp_init(obj, ball, None, cfg, mv)
    assert gs.alpha0 == st.get()["alpha0"] and gs.f == st.get()["f"]
    for _ in range(25):
        info_o, so = st.iterate(0.0)
        info_g = l1.gp_iterate(obj, ball, cfg, gs, None, mv, 0.0)
        assert info_g.stationary == so
        assert info_g.alpha == info_o["alpha"] and info_g.step == info_o["step"]
        assert np.array_equal(gs.x, st.get()["x"])
    assert mv.count == st.get()["matvecs"]


def test_callback_path_matches_graph_path():
    P = O.build_problem(PB.C2_MINI)
    obj = l1.Objective(l1.DenseOperator(P["K"]), P["y"])
    ball, cfg = l1.L1Ball(P["rho"]), l1.GpConfig()
    stop = l1.StopRule(max_iterations=80, stationarity_tol=0.0)
    recs, xs = [], []
    a = l1.gpss_solve(obj, ball, cfg, stop, cb=lambda r, x: (recs.append(r), xs.append(x)))
    t = []
    b = l1.gpss_solve(obj, ball, cfg, stop, trace=t)
    assert np.array_equal(a.x, b.x) and a.iterations == b.iterations == len(recs)
    assert [r.f for r in recs] == [r.f for r in t]
    assert np.array_equal(xs[-1], a.x)


def test_budgets_and_objective_tol():
    P = O.build_problem(PB.C2_MINI)
    op = l1.DenseOperator(P["K"])
    obj, ball, cfg = l1.Objective(op, P["y"]), l1.L1Ball(P["rho"]), l1.GpConfig()
    for stop in [O.StopRule(0, 41, 0, 0.0), O.StopRule(300, 0, 0, 0.0, 1e-6),
                 O.StopRule(7, 0, 0, 0.0), O.StopRule(300, 0, 0, 1e-9)]:
        xo, ro, _, _ = O.gpss_solve(P["K"], P["y"], P["rho"], O.GpConfig(), stop)
        sol = l1.gpss_solve(obj, ball, cfg, l1.StopRule(stop.max_iterations, stop.max_matvecs,
                                                        stop.max_seconds, stop.stationarity_tol,
                                                        stop.objective_tol))
        assert sol.iterations == ro["iterations"] and int(sol.reason) == ro["reason"]
        assert sol.matvecs.count == ro["matvecs"] and np.array_equal(sol.x, xo)


@pytest.mark.parametrize("spec,iters,kind", [(PB.C2_MINI, 150, "feasible"), (PB.RAGGED, 120, "feasible"),
                                             (PB.C2_MINI, 150, "zeros")],
                         ids=lambda v: getattr(v, "name", str(v)))
def test_trajectory_from_x0(spec, iters, kind):
    """gp_init from a given x0 (gpss.cpp:117-134): a feasible nonzero start, and an explicit
    all-zero x0, which takes the full forward pass over K where x0 = None skips it
    (launch_fwd_init_zero) -- both bit-identical to the oracle."""
    P = O.build_problem(spec)
    rng = np.random.default_rng(11)
    if kind == "zeros":
        x0 = np.zeros(spec.p)
    else:
        x0 = O.project_l1(rng.normal(size=spec.p), 0.5 * P["rho"])[0]
    xo, ro, reco, _ = O.gpss_solve(P["K"], P["y"], P["rho"], O.GpConfig(),
                                   O.StopRule(iters, 0, 0, 0.0), x0=x0)
    op = l1.DenseOperator(P["K"])
    trace = []
    sol = l1.gpss_solve(l1.Objective(op, P["y"]), l1.L1Ball(P["rho"]), l1.GpConfig(),
                        l1.StopRule(max_iterations=iters, stationarity_tol=0.0), x0=x0,
                        trace=trace)
    assert sol.iterations == ro["iterations"]
    assert sol.matvecs.count == ro["matvecs"]
    assert np.array_equal(sol.x, xo), np.abs(sol.x - xo).max()
    assert sol.objective == ro["objective"]
    for a, b in zip(trace, reco):
        for f in FIELDS:
            assert same(getattr(a, f), b[f]), (b["k"], f, getattr(a, f), b[f])


@pytest.mark.parametrize("params", [
    dict(beta=1e-2, theta=0.3, memory=4, alpha_min=1e-6, alpha_max=1e3, tau1=0.9,
         alpha2_memory=5),
    dict(beta=0.25, theta=0.7, memory=2, alpha_min=1e-3, alpha_max=50.0, tau1=0.1,
         alpha2_memory=1),
], ids=["nonmonotone_wide_tau", "tight_alpha_clamps"])
def test_trajectory_config_variants(params):
    """Every GpConfig field (gpss.hpp:14-24) reaches the device steplength, clamps, history
    and backtracking rule: non-default configurations stay bit-identical to the oracle."""
    spec = PB.C2_MINI
    P = O.build_problem(spec)
    iters = 150
    xo, ro, reco, _ = O.gpss_solve(P["K"], P["y"], P["rho"], O.GpConfig(**params),
                                   O.StopRule(iters, 0, 0, 0.0))
    op = l1.DenseOperator(P["K"])
    trace = []
    sol = l1.gpss_solve(l1.Objective(op, P["y"]), l1.L1Ball(P["rho"]), l1.GpConfig(**params),
                        l1.StopRule(max_iterations=iters, stationarity_tol=0.0), trace=trace)
    assert sol.iterations == ro["iterations"]
    assert int(sol.reason) == ro["reason"]
    assert np.array_equal(sol.x, xo), np.abs(sol.x - xo).max()
    assert sol.objective == ro["objective"]
    assert list(sol.f_history) == ro["f_history"]
    for a, b in zip(trace, reco):
        for f in FIELDS:
            assert same(getattr(a, f), b[f]), (b["k"], f, getattr(a, f), b[f])


def test_max_seconds_stop():
    """The wall-clock budget (gpss.cpp:242-245) is checked on the device (%globaltimer) at the
    top of every iteration, inside the one-launch run graph: the run stops with MaxSeconds
    and its iterate is the oracle's after the same number of iterations."""
    spec = PB.C3_MINI
    P = O.build_problem(spec)
    op = l1.DenseOperator(P["K"])
    obj, ball = l1.Objective(op, P["y"]), l1.L1Ball(P["rho"])
    # (the clock starts with gp_init, as gpss.cpp:224 does: a first solve also pays for
    # building the run graph, so the budget is applied to the second one)
    l1.gpss_solve(obj, ball, l1.GpConfig(), l1.StopRule(max_iterations=5, stationarity_tol=0.0))
    sol = l1.gpss_solve(obj, ball, l1.GpConfig(),
                        l1.StopRule(max_iterations=0, max_seconds=3e-3, stationarity_tol=0.0))
    assert sol.reason == l1.StopReason.MaxSeconds, sol.reason
    assert sol.iterations >= 1
    xo, ro, _, _ = O.gpss_solve(P["K"], P["y"], P["rho"], O.GpConfig(),
                                O.StopRule(sol.iterations, 0, 0, 0.0))
    assert ro["iterations"] == sol.iterations
    assert np.array_equal(sol.x, xo)
    assert sol.objective == ro["objective"]


@pytest.mark.parametrize("scale", ["tiny", "subnormal", "huge", "wide", "outlier"])
def test_projection_extreme_magnitudes(scale):
    """Edge magnitudes through the exact sort-and-scan: sums near the bottom of the normal
    range (the prefix's plain-step path), subnormal entries, sums near the overflow limit,
    vectors spanning hundreds of binades (many epochs) and one dominant entry."""
    rng = np.random.default_rng(["tiny", "subnormal", "huge", "wide", "outlier"].index(scale) + 90)
    for rep in range(12):
        p = int(rng.integers(2, 6000)) if rep % 3 else int(rng.integers(2, 300))
        z = rng.normal(size=p)
        if scale == "tiny":
            x = z * 1e-300
        elif scale == "subnormal":
            x = z * 1e-300
            x[::3] = rng.choice([5e-324, -1e-320, 2.5e-315], size=x[::3].size)
        elif scale == "huge":
            x = z * 1e300 / max(p, 1)
        elif scale == "wide":
            x = z * 10.0 ** rng.uniform(-200, 200, size=p)
        else:
            x = z * 1e-3
            x[int(rng.integers(0, p))] = 1e6
        for frac in (0.95, 0.5, 0.05):
            rho = frac * float(np.abs(x).sum())
            if not np.isfinite(rho):
                continue
            u, th, sup = O.project_l1(x, rho)
            pr = l1.project_l1_ball_with_threshold(x, l1.L1Ball(rho))
            assert pr.threshold == th and pr.support == sup, (scale, rep, frac)
            assert np.array_equal(pr.point, u), (scale, rep, frac)


def test_operator_extreme_magnitudes():
    """K x and K^T r bit for bit when the products are subnormal (fp64 on the device keeps
    denormals; every product and sum is one IEEE operation on both sides), near the overflow
    limit, and spread over many binades."""
    rng = np.random.default_rng(21)
    for (n, p) in [(77, 301), (256, 1024), (129, 2100)]:
        base = rng.normal(size=(n, p))
        for kscale, vscale in [(1e-160, 1e-160), (1e-300, 1.0), (1e150, 1e150 / 4096),
                               (None, None)]:
            if kscale is None:
                K = base * 10.0 ** rng.uniform(-100, 100, size=(n, p))
                x, r = rng.normal(size=p) * 1e-50, rng.normal(size=n) * 1e50
            else:
                K = base * kscale
                x, r = rng.normal(size=p) * vscale, rng.normal(size=n) * vscale
            op = l1.DenseOperator(K)
            assert np.array_equal(op.apply(x), O.apply(K, x)), (n, p, kscale)
            assert np.array_equal(op.apply_adjoint(r), O.apply_adjoint(K, r)), (n, p, kscale)


@pytest.mark.parametrize("n,p", [(3, 0), (0, 4), (1, 1)])
def test_empty_and_degenerate_shapes(n, p):
    """Empty operators and vectors (prox.cpp:38-73 on an empty x; gp_init / gp_iterate with no
    columns or no rows): the reference stops stationary at k = 0 (oracle and reference sources
    agree); the drop-in does the same with the same x and objective."""
    rng = np.random.default_rng(n * 10 + p)
    K = rng.normal(size=(n, p))
    y = rng.normal(size=n)
    xo, ro, _, _ = O.gpss_solve(K, y, 1.0, O.GpConfig(), O.StopRule(10, 0, 0, 0.0))
    sol = l1.gpss_solve(l1.Objective(l1.DenseOperator(K), y), l1.L1Ball(1.0), l1.GpConfig(),
                        l1.StopRule(max_iterations=10, stationarity_tol=0.0))
    assert sol.iterations == ro["iterations"] and int(sol.reason) == ro["reason"]
    assert np.array_equal(sol.x, xo) and sol.objective == ro["objective"]
    u, th, sup = O.project_l1(np.zeros(p), 1.0)
    pr = l1.project_l1_ball_with_threshold(np.zeros(p), l1.L1Ball(1.0))
    assert np.array_equal(pr.point, u) and pr.threshold == th and pr.support == sup


def test_small_step_kernel_and_large_path_identical(monkeypatch):
    """C1-sized problems run the step after the projection as one cluster kernel (small.cu);
    the five-kernel large path (L1G_SMALL=0) must give the same bits, both equal to the oracle."""
    P = O.build_problem(PB.C1)
    iters = 60
    xo, ro, reco, _ = O.gpss_solve(P["K"], P["y"], P["rho"], O.GpConfig(),
                                   O.StopRule(iters, 0, 0, 0.0))
    out = []
    for small in ("1", "0"):
        monkeypatch.setenv("L1G_SMALL", small)
        trace = []
        sol = l1.gpss_solve(l1.Objective(l1.DenseOperator(P["K"]), P["y"]), l1.L1Ball(P["rho"]),
                            l1.GpConfig(), l1.StopRule(max_iterations=iters, stationarity_tol=0.0),
                            trace=trace)
        assert sol.iterations == ro["iterations"]
        assert np.array_equal(sol.x, xo)
        assert [r.f for r in trace] == [r["f"] for r in reco]
        out.append(sol)
    assert np.array_equal(out[0].x, out[1].x)
