"""B200-native GPSS engine: the gradient-projection iteration loop of arXiv 0902.4424
(l1solve's gpss_solve) on sm_100a.  See DESIGN.md."""
from ._lib import load as _load_lib  # noqa: F401
from .api import (  # noqa: F401
    BacktrackResult, Context, DenseOperator, GpConfig, GpIterationState, GpStepInfo,
    IterationRecord, L1Ball, L1Projection, LinearOperator, MatvecCounter, Objective,
    PenaltyWeight, SolverState, SteplengthChoice, SteplengthState, StopReason, StopRule,
    GeneratedProblem, alpha0_from_gradient, alpha0_init, backtracking_search, default_context, dot, fista_solve,
    gp_init, gp_iterate, gpss_solve, ista_solve, load_problem, problem_hash, psd_solve,
    save_problem, l1_norm, lambda_from_rho, lambda_max, linf_norm,
    project_l1_ball, project_l1_ball_with_threshold, rho_from_lambda, soft_threshold,
    spectral_norm_estimate, squared_norm, steplength_init, steplength_select, to_string,
    ReferenceOptions, ReferenceSolution, reference_minimizer, penalized_fixed_point_residual)
from . import isochrone  # noqa: F401

__version__ = "0.1.0"
