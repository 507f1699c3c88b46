"""Reports the reference test modules this suite does not collect, and why."""

import pytest

from ref_conformance.conftest import NOT_COLLECTED


@pytest.mark.parametrize("module", sorted(NOT_COLLECTED))
def test_not_collected(module):
    pytest.skip(f"{module}: {NOT_COLLECTED[module]}")
