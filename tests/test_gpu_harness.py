"""The device problem builder (paper_0902_4424_b200.harness) against the oracle's."""
import numpy as np
import pytest

import paper_0902_4424_b200 as l1
from oracle import oracle as O
from paper_0902_4424_b200 import harness as H
from tests import problems as PB

pytestmark = pytest.mark.gpu


def as_product(spec):
    return H.ProblemSpec(spec.kind, spec.n, spec.p, spec.nnz, spec.seed, spec.values,
                         spec.noise, spec.noise_mode, spec.rho_factor, spec.norm_target,
                         spec.power_iters, spec.power_tol, spec.sigma_hat, spec.name)


@pytest.mark.parametrize("spec", [PB.C1, PB.C2_MINI, PB.C3_MINI, PB.RAGGED],
                         ids=lambda s: s.name)
def test_problem_bit_identical(spec):
    Po = O.build_problem(spec)
    Pg = H.build_problem(as_product(spec))
    assert np.array_equal(Pg["op"].matrix(), Po["K"])
    assert np.array_equal(Pg["x_true"], Po["x_true"])
    assert np.array_equal(Pg["y"], Po["y"])
    assert Pg["rho"] == Po["rho"]
    if spec.kind == "gaussian":
        assert Pg["sigma_hat"] == Po["sigma_hat"]
    assert np.array_equal(H.blur_taps(), O.blur_taps())
