"""ref tests/test_measures.py through the drop-in (see conftest.py)."""

import pytest

from test_measures import *  # noqa: F401,F403

pytestmark = pytest.mark.gpu
