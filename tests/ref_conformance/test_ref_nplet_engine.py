"""ref tests/test_nplet_engine.py through the drop-in (see conftest.py)."""

import pytest

from test_nplet_engine import *  # noqa: F401,F403

pytestmark = pytest.mark.gpu
