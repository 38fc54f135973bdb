"""The CPU oracle against every known answer the reference's own tests pin (CPU only)."""
import pytest

from tests import kat_cases
from tests.backends import OracleBackend


@pytest.mark.parametrize("case", kat_cases.ALL_CASES, ids=lambda c: c.__name__[5:])
def test_oracle_kat(case):
    case(OracleBackend())
