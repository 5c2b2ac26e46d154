import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden" / "reference_golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libvrhe.so")


@pytest.fixture
def rng():
    # the reference suite's generator (tests/conftest.py:15-17)
    return np.random.default_rng(0xC0FFEE)


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


def rand_int_matrix(rng, rows, cols, lo=-4, hi=5):
    return rng.integers(lo, hi, size=(rows, cols)).astype(np.float64)
