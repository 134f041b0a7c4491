"""ref tests/test_scanner.py through the drop-in (see conftest.py)."""

import pytest

from test_scanner import *  # noqa: F401,F403

pytestmark = pytest.mark.gpu
