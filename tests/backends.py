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
