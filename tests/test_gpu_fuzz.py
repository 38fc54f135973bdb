"""A short seeded run of tools/fuzz_parity.py: random shapes, radii, configurations and starts,
the CUDA path against the CPU oracle bit for bit (the long runs are in profiles/)."""
import numpy as np
import pytest

from tools import fuzz_parity as F

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [11, 12])
def test_random_cases_bit_identical(seed):
    rng = np.random.default_rng(seed)
    for case in range(150):
        fn = F.one_solve if rng.random() < 0.6 else F.one_projection
        desc, bad = fn(rng, case)
        assert not bad, (desc, bad)
