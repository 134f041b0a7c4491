import json
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
GOLDEN = REPO / "tests" / "golden"
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "oracle"))
sys.path.insert(0, str(REPO / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")


@pytest.fixture(scope="session")
def golden():
    class G:
        meta = json.loads((GOLDEN / "golden.json").read_text())

        @staticmethod
        def npz(name):
            return np.load(GOLDEN / f"{name}.npz")

    return G


@pytest.fixture(scope="session")
def oracle():
    import hoi_oracle
    return hoi_oracle
