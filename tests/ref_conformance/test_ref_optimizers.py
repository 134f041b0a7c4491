"""ref tests/test_optimizers.py through the drop-in (see conftest.py)."""

import pytest

from test_optimizers import *  # noqa: F401,F403

pytestmark = pytest.mark.gpu
