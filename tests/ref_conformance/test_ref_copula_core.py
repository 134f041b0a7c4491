"""ref tests/test_copula_core.py through the drop-in (see conftest.py)."""

import pytest

from test_copula_core import *  # noqa: F401,F403

pytestmark = pytest.mark.gpu
