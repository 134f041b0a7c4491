"""ref tests/test_acceptance.py through the drop-in (see conftest.py).

Criterion 9 drives the reference CLI (`hoi.cli.main`: argument parsing,
CSV writing, exit codes), which is out of scope for this engine
(SURVEY.md §2), so it is not collected; every other criterion runs.
"""

import pytest

from test_acceptance import *  # noqa: F401,F403

del test_criterion_09_cli_outputs_byte_identical  # noqa: F821

pytestmark = pytest.mark.gpu
