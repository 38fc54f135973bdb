"""Drop-in fidelity of gp_init / gp_iterate (gpss.cpp:117-219; VERDICT r1 "Next" #7).

GpIterationState exposes the reference's public fields (gpss.hpp:89-98).  A caller may read
them after any step, edit them between steps (the reference's gp_iterate is a function of
the struct it is handed) and pass a different GpConfig / L1Ball per call: the device must
follow exactly what the reference's gp_iterate would do, here the oracle's GpState with the
same edits.  Also: GpStepInfo.steplength.alpha is the choice before any escalation, and a
throwing callback stops the device loop at once.
"""
import numpy as np
import pytest

import paper_0902_4424_b200 as l1
from oracle import oracle as O
from tests import problems as PB

pytestmark = pytest.mark.gpu


def test_edited_state_and_config_follow_the_reference():
    P = O.build_problem(PB.C2_MINI)
    K, y, rho = P["K"], P["y"], P["rho"]
    ora = O.GpState(K, y, rho)
    obj = l1.Objective(l1.DenseOperator(K), y)
    ball, cfg, mv = l1.L1Ball(rho), l1.GpConfig(), l1.MatvecCounter()
    gs = l1.gp_init(obj, ball, None, cfg, mv)
    sls = l1.steplength_init(cfg)
    for _ in range(5):
        info_o, _ = ora.iterate(0.0)
        info_g = l1.gp_iterate(obj, ball, cfg, gs, sls, mv, 0.0)
        assert info_g.alpha == info_o["alpha"]
    o = ora.get()
    assert np.array_equal(gs.x, o["x"]) and np.array_equal(gs.grad, o["grad"])
    assert np.array_equal(gs.kx_minus_y, o["kx_minus_y"]) and gs.f == o["f"] and gs.k == 5
    assert len(gs.f_history) == 1 and gs.f_history[0] == gs.f
    assert sls.prev_x is not None and sls.tau > 0  # read back from the device
    # the caller's edits: a shrunken iterate with its caches, memory 3, a larger ball
    with O.mode(O.CANONICAL):
        x = o["x"] * 0.5
        r = O.apply(K, x) - y
        g = 2.0 * O.apply_adjoint(K, r)
        f = O.sqnorm(r)
    cfg3, ball2 = l1.GpConfig(memory=3), l1.L1Ball(rho * 1.25)
    ora.set(x, r, g, f, 5, [f], cfg=O.GpConfig(memory=3), rho=rho * 1.25)
    gs.x, gs.kx_minus_y, gs.grad, gs.f, gs.f_history = x, r, g, f, [f]
    for _ in range(12):
        info_o, so = ora.iterate(0.0)
        info_g = l1.gp_iterate(obj, ball2, cfg3, gs, sls, mv, 0.0)
        assert info_g.stationary == so
        assert info_g.alpha == info_o["alpha"] and info_g.step == info_o["step"]
        assert info_g.f_after == info_o["f"]
    o = ora.get()
    assert np.array_equal(gs.x, o["x"]) and gs.f == o["f"] and gs.k == o["k"]
    assert len(gs.f_history) == 3


def test_steplength_alpha_is_before_escalation():
    """gpss.cpp:148-153 vs :192: info.steplength.alpha is the BB choice, info.alpha the
    escalated one; on a run to the floor the escalation happens at least once."""
    P = O.build_problem(PB.C1)
    obj = l1.Objective(l1.DenseOperator(P["K"]), P["y"])
    ball, cfg, mv = l1.L1Ball(P["rho"]), l1.GpConfig(), l1.MatvecCounter()
    gs = l1.gp_init(obj, ball, None, cfg, mv)
    sls = l1.steplength_init(cfg)
    ora = O.GpState(P["K"], P["y"], P["rho"])
    for _ in range(500):
        info_o, so = ora.iterate(0.0)
        info = l1.gp_iterate(obj, ball, cfg, gs, sls, mv, 0.0)
        assert info.stationary == so and info.alpha == info_o["alpha"]
        if gs.k > 1 and not so:
            assert info.steplength.alpha <= info.alpha
            assert info.steplength.bb1_raw == info_o["bb1_raw"]
        if so:
            break


def test_throwing_callback_stops_at_once():
    P = O.build_problem(PB.C2_MINI)
    obj = l1.Objective(l1.DenseOperator(P["K"]), P["y"])
    calls = []

    def cb(rec, x):
        calls.append(rec.k)
        if len(calls) == 3:
            raise KeyError("stop")

    with pytest.raises(KeyError):
        l1.gpss_solve(obj, l1.L1Ball(P["rho"]), l1.GpConfig(),
                      l1.StopRule(max_iterations=200, stationarity_tol=0.0), cb=cb)
    assert len(calls) == 3
