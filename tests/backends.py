"""Backends the shared KAT cases (tests/kat_cases.py) run against."""
from __future__ import annotations

import numpy as np

from oracle import oracle as O


class OracleBackend:
    """The CPU restatement (oracle/l1oracle.c), canonical reduction order."""
    name = "oracle"

    def config_valid(self, cfg):
        return O.config_valid(cfg)

    def steplength(self, cfg):
        return O.Steplength(cfg)

    def alpha0_init(self, K, y, rho, x0, cfg):
        K, y, x0 = np.asarray(K, float), np.asarray(y, float), np.asarray(x0, float)
        g = 2.0 * O.apply_adjoint(K, O.apply(K, x0) - y)
        return O.alpha0_from_gradient(rho, x0, g, cfg), 2

    def alpha0_from_gradient(self, rho, x0, grad, cfg):
        return O.alpha0_from_gradient(rho, x0, grad, cfg)

    def backtracking_search(self, K, y, x, d, f_max, gd, cfg):
        if not gd < 0.0:
            raise ValueError("backtracking_search: d must be a descent direction")
        K = np.asarray(K, float)
        misfit = O.apply(K, x) - np.asarray(y, float)
        kd = O.apply(K, d)
        return O.backtrack_quadratic(O.sqnorm(misfit), O.dot(misfit, kd), O.sqnorm(kd), f_max,
                                     gd, cfg)

    def gp_state(self, K, y, rho, cfg, x0=None):
        return O.GpState(K, y, rho, cfg, x0)

    def gpss_solve(self, K, y, rho, cfg, stop, x0=None, x_trace=False):
        x, res, recs, xh = O.gpss_solve(K, y, rho, cfg, stop, x0, trace=True, x_trace=x_trace)
        if x_trace:
            res["x_trace"] = list(xh)
        return x, res, recs

    def soft_threshold(self, x, t):
        return O.soft_threshold(x, t)

    def project_l1(self, x, rho):
        u, th, _ = O.project_l1(x, rho)
        return u, th

    def apply(self, K, x):
        return O.apply(K, x)

    def apply_adjoint(self, K, r):
        return O.apply_adjoint(K, r)

    def spectral_norm(self, K, iters=1000, tol=1e-8):
        return O.spectral_norm(K, iters, tol)


class GpuBackend:
    """The B200 product, through its C-ABI (paper_0902_4424_b200.api -> libl1g.so)."""
    name = "gpu"

    def __init__(self):
        import paper_0902_4424_b200 as l1
        self.l1 = l1

    def _cfg(self, cfg):
        return self.l1.GpConfig(beta=cfg.beta, theta=cfg.theta, memory=cfg.memory,
                                alpha_min=cfg.alpha_min, alpha_max=cfg.alpha_max,
                                tau1=cfg.tau1, alpha2_memory=cfg.alpha2_memory)

    def _stop(self, s):
        return self.l1.StopRule(s.max_iterations, s.max_matvecs, s.max_seconds,
                                s.stationarity_tol, s.objective_tol)

    def config_valid(self, cfg):
        try:
            self._cfg(cfg).validate()
            return True
        except ValueError:
            return False

    def steplength(self, cfg):
        l1, c = self.l1, self._cfg(cfg)

        class _S:
            def __init__(s):
                s.st = l1.steplength_init(c)

            @property
            def tau(s):
                return s.st.tau

            @property
            def history(s):
                return s.st.alpha2_history

            def select(s, a, b, k):
                ch = l1.steplength_select(s.st, a, b, c, k)
                return {"alpha": ch.alpha, "bb_active": int(ch.bb_active),
                        "bb1_raw": ch.bb1_raw, "bb2_raw": ch.bb2_raw,
                        "tau_before": ch.tau_before, "tau_after": ch.tau_after}
        return _S()

    def alpha0_init(self, K, y, rho, x0, cfg):
        l1 = self.l1
        mv = l1.MatvecCounter()
        obj = l1.Objective(l1.DenseOperator(np.asarray(K, float)), y)
        return l1.alpha0_init(obj, l1.L1Ball(rho), x0, self._cfg(cfg), mv), mv.count

    def alpha0_from_gradient(self, rho, x0, grad, cfg):
        return self.l1.alpha0_from_gradient(self.l1.L1Ball(rho), x0, grad, self._cfg(cfg))

    def backtracking_search(self, K, y, x, d, f_max, gd, cfg):
        l1 = self.l1
        obj = l1.Objective(l1.DenseOperator(np.asarray(K, float)), y)
        r = l1.backtracking_search(obj, x, d, f_max, gd, self._cfg(cfg), l1.MatvecCounter())
        return r.step, r.f_new, r.halvings

    def gp_state(self, K, y, rho, cfg, x0=None):
        l1, be = self.l1, self
        obj = l1.Objective(l1.DenseOperator(np.asarray(K, float)), y)
        ball, c = l1.L1Ball(rho), self._cfg(cfg)

        class _G:
            def __init__(s):
                s.mv = l1.MatvecCounter()
                s.st = l1.gp_init(obj, ball, x0, c, s.mv)

            def iterate(s, tol=0.0):
                info = l1.gp_iterate(obj, ball, c, s.st, None, s.mv, tol)
                return {"dir_derivative": info.dir_derivative, "alpha": info.alpha,
                        "stationarity": info.stationarity, "f": info.f_after}, info.stationary

            def get(s):
                st = s.st
                return dict(x=st.x, kx_minus_y=st.kx_minus_y, grad=st.grad, f=st.f, k=st.k,
                            alpha0=st.alpha0, matvecs=s.mv.count)
        return _G()

    def gpss_solve(self, K, y, rho, cfg, stop, x0=None, x_trace=False):
        l1 = self.l1
        obj = l1.Objective(l1.DenseOperator(np.asarray(K, float)), y)
        trace, xs = [], []
        cb = (lambda rec, x: xs.append(x)) if x_trace else None
        sol = l1.gpss_solve(obj, l1.L1Ball(rho), self._cfg(cfg), self._stop(stop), cb=cb,
                            x0=x0, trace=trace)
        res = {"iterations": sol.iterations, "matvecs": sol.matvecs.count,
               "objective": sol.objective, "stationarity": sol.stationarity,
               "reason": int(sol.reason), "reason_name": l1.to_string(sol.reason),
               "f_history": list(sol.f_history)}
        if x_trace:
            res["x_trace"] = xs
        return sol.x, res, [r.as_dict() for r in trace]

    def soft_threshold(self, x, t):
        return self.l1.soft_threshold(x, t)

    def project_l1(self, x, rho):
        pr = self.l1.project_l1_ball_with_threshold(x, self.l1.L1Ball(rho))
        return pr.point, pr.threshold

    def apply(self, K, x):
        return self.l1.DenseOperator(np.asarray(K, float)).apply(x)

    def apply_adjoint(self, K, r):
        return self.l1.DenseOperator(np.asarray(K, float)).apply_adjoint(r)

    def spectral_norm(self, K, iters=1000, tol=1e-8):
        mv = self.l1.MatvecCounter()
        return self.l1.spectral_norm_estimate(self.l1.DenseOperator(np.asarray(K, float)),
                                              iters, tol, mv), mv.count
