"""Known-answer and property cases restated from the reference's own tests.

Each ``case_*`` function takes a backend (the CPU oracle, the reference sources compiled
against the Eigen stand-in, or the B200 product through its C-ABI) and asserts the value
the reference test pins.  Sources (relative to /root/reference/proj/tests):
test_gpss.cpp, test_prox.cpp, test_operator.cpp, acceptance/acceptance_main.cpp.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import oracle as O


def approx(v, target, eps):
    """doctest::Approx(target).epsilon(eps)"""
    return abs(v - target) <= eps * (1.0 + max(abs(v), abs(target)))


# ------------------------------------------------------------------ test_gpss.cpp
def case_config_validation(B):  # test_gpss.cpp:28-46
    assert B.config_valid(O.GpConfig())
    for kw in [dict(beta=0.0), dict(theta=1.0), dict(alpha_min=1.0, alpha_max=0.5),
               dict(memory=0), dict(tau1=1.0)]:
        assert not B.config_valid(O.GpConfig(**kw))


def case_steplength_nonpositive(B):  # test_gpss.cpp:48-61
    cfg = O.GpConfig()
    st = B.steplength(cfg)
    c1 = st.select([1.0, 0.0], [-1.0, 0.0], 1)
    assert c1["alpha"] == cfg.alpha_max and not c1["bb_active"]
    assert st.tau == cfg.tau1 and st.history == []
    c2 = st.select([0.0, 0.0], [1.0, 1.0], 2)
    assert c2["alpha"] == cfg.alpha_max and not c2["bb_active"]


def case_steplength_worked(B):  # test_gpss.cpp:63-74
    cfg = O.GpConfig()
    st = B.steplength(cfg)
    c = st.select([1.0, 1.0], [1.0, 3.0], 1)
    assert c["bb_active"]
    assert approx(c["bb1_raw"], 0.5, 1e-15) and approx(c["bb2_raw"], 0.4, 1e-15)
    assert approx(c["alpha"], 0.5, 1e-15) and approx(c["tau_after"], 0.55, 1e-15)
    assert len(st.history) == 1


def case_steplength_collinear(B):  # test_gpss.cpp:76-86
    cfg = O.GpConfig()
    st = B.steplength(cfg)
    s = np.array([0.3, -0.7, 0.1])
    c = st.select(s, 2.0 * s, 1)
    assert approx(c["bb1_raw"], 0.5, 1e-14) and approx(c["bb2_raw"], 0.5, 1e-14)
    assert approx(c["alpha"], 0.5, 1e-14) and approx(c["tau_after"], 1.1 * cfg.tau1, 1e-15)


def case_steplength_bb2_branch(B):  # test_gpss.cpp:88-102
    cfg = O.GpConfig(tau1=0.9)
    st = B.steplength(cfg)
    st.select([1.0, 1.0], [1.0, 3.0], 1)
    c = st.select([2.0, 2.0], [1.0, 3.0], 2)
    assert c["bb_active"] and approx(c["bb2_raw"], 0.8, 1e-15)
    assert approx(c["alpha"], 0.4, 1e-15)
    assert approx(c["tau_after"], 0.9 * c["tau_before"], 1e-15)
    assert len(st.history) == 2


def case_steplength_secant_oracle(B):  # test_gpss.cpp:104-153 (grid-scan oracle)
    rng = np.random.default_rng(97)
    cfg = O.GpConfig()
    for _ in range(20):
        p = 3 + int(rng.integers(0, 6))
        s, z = rng.normal(size=p), rng.normal(size=p)
        if s @ z <= 0:
            z = -z
        if s @ z <= 0:
            continue
        c = B.steplength(cfg).select(s, z, 1)
        assert c["bb_active"]

        def scan(obj, lo, hi):
            best = lo
            for _ in range(3):
                a = np.linspace(lo, hi, 20001)
                v = obj(a)
                i = int(np.argmin(v))
                best = a[i]
                step = (hi - lo) / 20000
                lo, hi = max(lo, best - step), best + step
            return best

        sz = s @ z
        hi1 = 4.0 * (s @ s) / sz
        hi2 = 2.0 * np.linalg.norm(s) / np.linalg.norm(z)
        bb1 = scan(lambda a: ((s[None, :] / a[:, None] - z[None, :]) ** 2).sum(1), hi1 / 1e5, hi1)
        bb2 = scan(lambda a: ((s[None, :] - a[:, None] * z[None, :]) ** 2).sum(1), 0.0, hi2)
        assert approx(c["bb1_raw"], bb1, 1e-4) and approx(c["bb2_raw"], bb2, 1e-4)


def case_steplength_history_cap(B):  # test_gpss.cpp:155-162
    cfg = O.GpConfig(alpha2_memory=2)
    st = B.steplength(cfg)
    for k in range(1, 6):
        st.select([1.0, 1.0], [1.0, 3.0], k)
    assert len(st.history) == 3


def case_steplength_clamped(B):  # test_gpss.cpp:164-173
    cfg = O.GpConfig(alpha_min=0.45, alpha_max=0.48)
    c = B.steplength(cfg).select([1.0, 1.0], [1.0, 3.0], 1)
    assert cfg.alpha_min <= c["alpha"] <= cfg.alpha_max


def case_alpha0(B):  # test_gpss.cpp:175-193
    cfg = O.GpConfig()
    a0, mv = B.alpha0_init(np.eye(2), [1.0, 0.5], 10.0, [0.0, 0.0], cfg)
    assert approx(a0, 0.5, 1e-15) and mv == 2
    assert B.alpha0_from_gradient(10.0, [0.0, 0.0], [-1e-20, 0.0], cfg) == cfg.alpha_max
    assert B.alpha0_from_gradient(1e30, [0.0, 0.0], [-1e20, 0.0], cfg) == cfg.alpha_min
    assert B.alpha0_from_gradient(10.0, [0.0, 0.0], [0.0, 0.0], cfg) == cfg.alpha_max


def case_backtracking_hand_trace(B):  # test_gpss.cpp:195-207
    cfg = O.GpConfig()
    step, f_new, h = B.backtracking_search(np.ones((1, 1)), [0.0], [1.0], [-2.0], 1.0, -4.0, cfg)
    assert approx(step, 0.5, 1e-15) and approx(f_new, 0.0, 1e-15) and h == 1


def case_backtracking_errors(B):  # test_gpss.cpp:209-222
    cfg = O.GpConfig()
    with pytest.raises(ValueError):
        B.backtracking_search(np.ones((1, 1)), [0.0], [1.0], [2.0], 1.0, 4.0, cfg)
    with pytest.raises(RuntimeError):
        B.backtracking_search(np.ones((1, 1)), [0.0], [1.0], [-2.0], -1e10, -4.0, cfg)


def case_backtracking_nonmonotone(B):  # test_gpss.cpp:224-241
    cfg = O.GpConfig()
    mono = B.backtracking_search(np.ones((1, 1)), [0.0], [1.0], [-2.0], 1.0, -4.0, cfg)
    assert approx(mono[0], 0.5, 1e-12)
    relaxed = B.backtracking_search(np.ones((1, 1)), [0.0], [1.0], [-2.0], 4.0, -4.0, cfg)
    assert relaxed[0] == 1.0 and approx(relaxed[1], 1.0, 1e-12)


def case_gp_iterate_fixed_point(B):  # test_gpss.cpp:243-256
    y = np.array([0.25, -0.25])
    st = B.gp_state(np.eye(2), y, 1.0, O.GpConfig(), x0=y)
    info, stationary = st.iterate(0.0)
    assert stationary
    assert np.array_equal(st.get()["x"], y)


def case_gp_iterate_single_step(B):  # test_gpss.cpp:258-272
    st = B.gp_state(np.eye(2), [3.0, 1.0], 1.0, O.GpConfig(), x0=[0.0, 0.0])
    f0 = st.get()["f"]
    info, stationary = st.iterate(0.0)
    assert not stationary
    s = st.get()
    assert np.abs(s["x"]).sum() <= 1.0 + 1e-12 and s["f"] < f0


def case_gp_iterate_descent(B):  # test_gpss.cpp:274-296, with this harness's generator
    rng = np.random.default_rng(61)
    checked = 0
    for rep in range(100):
        P = O.build_problem(O.ProblemSpec("gaussian", 8, 20, 3, 1000 + rep, "sign", 0.02, "rel",
                                          norm_target=1.0))
        rho = 0.1 + 2.0 * rng.uniform()
        x0, _, _ = O.project_l1(rng.normal(size=20), rho)
        st = B.gp_state(P["K"], P["y"], rho, O.GpConfig(), x0=x0)
        info, stationary = st.iterate(0.0)
        if stationary:
            continue
        assert info["dir_derivative"] < 0.0
        checked += 1
    assert checked >= 90


def case_identity_projection(B):  # test_gpss.cpp:298-307
    y = np.array([3.0, 0.0])
    x, res, recs = B.gpss_solve(np.eye(2), y, 1.0, O.GpConfig(), O.StopRule(50, 0, 0, 1e-10))
    u, _, _ = O.project_l1(y, 1.0)
    assert np.abs(x - u).max() <= 1e-10
    assert res["iterations"] <= 3 and res["reason_name"] == "stationary"


def case_infeasible_start(B):  # test_gpss.cpp:309-315
    with pytest.raises(ValueError):
        B.gpss_solve(np.eye(2), [1.0, 1.0], 0.5, O.GpConfig(), O.StopRule(20000, 0, 0, 1e-12),
                     x0=[1.0, 1.0])


def case_feasible_monotone(B):  # test_gpss.cpp:317-343
    P = O.build_problem(O.ProblemSpec("gaussian", 30, 100, 6, 67, "sign", 0.02, "rel",
                                      norm_target=1.0))
    rho = O.l1norm(P["x_true"])
    for memory in (1, 5):
        cfg = O.GpConfig(memory=memory)
        x, res, recs = B.gpss_solve(P["K"], P["y"], rho, cfg, O.StopRule(500, 0, 0, 1e-13),
                                    x_trace=True)
        assert len(recs) > 5
        for r, xk in zip(recs, res["x_trace"]):
            assert np.abs(xk).sum() <= rho + 1e-10
        for i in range(1, len(recs)):
            a, b = recs[i - 1], recs[i]
            if memory == 1:
                assert b["f"] <= a["f"] + 1e-12 * max(1.0, a["f"])
            assert b["f"] <= b["f_max"] + cfg.beta * b["step"] * b["dir_derivative"] + \
                1e-12 * max(1.0, b["f_max"])


def case_bb_telemetry(B):  # test_gpss.cpp:345-364
    P = O.build_problem(O.ProblemSpec("gaussian", 30, 100, 6, 71, "sign", 0.02, "rel",
                                      norm_target=1.0))
    cfg = O.GpConfig()
    x, res, recs = B.gpss_solve(P["K"], P["y"], O.l1norm(P["x_true"]), cfg,
                                O.StopRule(500, 0, 0, 1e-13))
    assert len(recs) > 10
    for r in recs:
        assert cfg.alpha_min <= r["alpha"] <= cfg.alpha_max
        if r["bb_active"]:
            assert r["bb2_raw"] <= r["bb1_raw"] * (1.0 + 1e-12)
            ratio = r["tau_after"] / r["tau_before"]
            assert abs(ratio - 0.9) < 1e-12 or abs(ratio - 1.1) < 1e-12
        elif r["k"] > 0:
            assert r["tau_after"] == r["tau_before"]


def case_matvec_accounting(B):  # test_gpss.cpp:366-375
    P = O.build_problem(O.ProblemSpec("gaussian", 10, 20, 3, 79, "sign", 0.02, "rel",
                                      norm_target=1.0))
    x, res, recs = B.gpss_solve(P["K"], P["y"], 1.0, O.GpConfig(), O.StopRule(4, 0, 0, 0.0))
    assert res["iterations"] == 4 and res["matvecs"] == 2 + 2 * 4


def case_zero_radius(B):  # test_gpss.cpp:393-404
    P = O.build_problem(O.ProblemSpec("gaussian", 8, 16, 3, 83, "sign", 0.02, "rel",
                                      norm_target=1.0))
    x, res, recs = B.gpss_solve(P["K"], P["y"], 0.0, O.GpConfig(), O.StopRule(50, 0, 0, 1e-12))
    assert np.abs(x).sum() == 0.0 and res["reason_name"] == "stationary"
    assert res["iterations"] == 0


def case_one_dimensional(B):  # test_gpss.cpp:406-416
    x, res, recs = B.gpss_solve(np.array([[0.7]]), [2.0], 1.0, O.GpConfig(),
                                O.StopRule(100, 0, 0, 1e-12))
    assert approx(x[0], 1.0, 1e-10)


# ------------------------------------------------------------------ test_prox.cpp
def case_soft_threshold(B):  # test_prox.cpp:51-56
    x = np.array([2.0, -0.5, 1.5])
    assert np.array_equal(B.soft_threshold(x, 1.0), [1.0, 0.0, 0.5])
    assert np.array_equal(B.soft_threshold(x, 0.0), x)
    with pytest.raises(ValueError):
        B.soft_threshold(x, -0.1)


def case_projection_kats(B):  # test_prox.cpp:83-98
    u, th = B.project_l1([3.0, 0.0], 1.0)
    assert np.array_equal(u, [1.0, 0.0])
    f = np.array([1.0, -0.5])
    assert np.array_equal(B.project_l1(f, 2.0)[0], f)
    u, th = B.project_l1([0.9, 0.5], 1.0)
    assert approx(th, 0.2, 1e-12) and np.abs(u - [0.7, 0.3]).max() < 1e-12
    assert np.abs(B.project_l1([1.0, -2.0], 0.0)[0]).sum() == 0.0
    with pytest.raises(ValueError):
        B.project_l1([1.0], -0.5)


def _bisection(x, rho):  # test_prox.cpp:36-47
    if np.abs(x).sum() <= rho:
        return x
    lo, hi = 0.0, float(np.abs(x).max())
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if O.l1norm(O.soft_threshold(x, mid)) > rho:
            lo = mid
        else:
            hi = mid
    return O.soft_threshold(x, hi)


def case_projection_bisection(B):  # test_prox.cpp:100-110 and acceptance criterion 1
    rng = np.random.default_rng(31)
    for _ in range(200):
        p = 2 + int(rng.integers(0, 11))
        x = 2.5 * rng.normal(size=p)
        rho = 0.05 + 2.0 * rng.uniform()
        assert np.abs(B.project_l1(x, rho)[0] - _bisection(x, rho)).max() <= 1e-8


def case_projection_idempotent(B):  # test_prox.cpp:112-121
    rng = np.random.default_rng(37)
    for _ in range(100):
        x = 4.0 * rng.normal(size=24)
        rho = 0.2 + 2.0 * rng.uniform()
        once = B.project_l1(x, rho)[0]
        assert O.l1norm(once) <= rho + 1e-12
        assert np.array_equal(B.project_l1(once, rho)[0], once)


def case_projection_nonexpansive(B):  # test_prox.cpp:123-132
    rng = np.random.default_rng(41)
    for _ in range(100):
        x = 3.0 * rng.normal(size=16)
        x2 = x + rng.normal(size=16)
        rho = 0.5 + rng.uniform()
        d = np.linalg.norm(B.project_l1(x, rho)[0] - B.project_l1(x2, rho)[0])
        assert d <= np.linalg.norm(x - x2) * (1.0 + 1e-12)


def case_projection_equals_threshold(B):  # test_prox.cpp:134-143
    rng = np.random.default_rng(43)
    for _ in range(50):
        x = 3.0 * rng.normal(size=10)
        rho = 0.3 * O.l1norm(x)
        u, th = B.project_l1(x, rho)
        assert np.array_equal(u, O.soft_threshold(x, th)) and th >= 0.0


# ------------------------------------------------------------------ test_operator.cpp
def case_operator_arithmetic(B):  # test_operator.cpp:32-54
    assert np.array_equal(B.apply(np.eye(2), [3.0, -1.0]), [3.0, -1.0])
    K = np.array([[1.0, 2.0], [0.0, 1.0]])
    assert np.array_equal(B.apply(K, [1.0, 1.0]), [3.0, 1.0])
    assert np.array_equal(B.apply_adjoint(np.eye(2), [1.0, 2.0]), [1.0, 2.0])
    assert np.array_equal(B.apply_adjoint(K, [1.0, 0.0]), [1.0, 2.0])
    with pytest.raises(ValueError):
        B.apply(np.zeros((3, 5)), np.zeros(3))
    with pytest.raises(ValueError):
        B.apply_adjoint(np.zeros((3, 5)), np.zeros(5))


def case_operator_adjoint_identity(B):  # test_operator.cpp:56-70
    rng = np.random.default_rng(11)
    K = rng.normal(size=(5, 8))
    for _ in range(100):
        u, v = rng.normal(size=8), rng.normal(size=5)
        lhs = B.apply(K, u) @ v
        rhs = u @ B.apply_adjoint(K, v)
        assert abs(lhs - rhs) <= 1e-10 * max(abs(lhs), abs(rhs), 1.0)
        assert np.abs(B.apply_adjoint(K, v) - K.T @ v).max() < 1e-14


def case_spectral_norm(B):  # test_operator.cpp:86-102
    assert approx(B.spectral_norm(3.0 * np.eye(4))[0], 3.0, 1e-10)
    assert approx(B.spectral_norm(np.diag([1.0, 5.0]))[0], 5.0, 1e-10)
    m = np.random.default_rng(17).normal(size=(20, 50))
    svd = np.linalg.svd(m, compute_uv=False)[0]
    est = B.spectral_norm(m, 5000, 1e-12)[0]
    assert approx(est, svd, 1e-6) and est <= svd * (1.0 + 1e-12)


def case_identity_closed_form(B):  # acceptance_main.cpp:137-170 (GPSS part)
    rng = np.random.default_rng(303)
    y = 2.0 * rng.normal(size=6)
    rho = 0.4 * O.l1norm(y)
    star = O.project_l1(y, rho)[0]
    x, res, recs = B.gpss_solve(np.eye(6), y, rho, O.GpConfig(), O.StopRule(50, 0, 0, 1e-13))
    assert np.linalg.norm(x - star) / np.linalg.norm(star) <= 1e-9 and res["iterations"] <= 50


ALL_CASES = [v for k, v in sorted(globals().items()) if k.startswith("case_")]
