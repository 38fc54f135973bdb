"""The B200 product against every known answer the reference's own tests pin."""
import pytest

from tests import kat_cases
from tests.backends import GpuBackend

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    return GpuBackend()


@pytest.mark.parametrize("case", kat_cases.ALL_CASES, ids=lambda c: c.__name__[5:])
def test_gpu_kat(case, gpu):
    case(gpu)
