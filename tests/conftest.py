import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running (large configs)")


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


def rel_err(actual, expected):
    """max |a - e| / max |e|  -- the reference's tolerance metric (conftest.py:25-28)."""
    scale = max(1e-6, float(np.max(np.abs(expected))))
    return float(np.max(np.abs(np.asarray(actual, np.float64) - np.asarray(expected, np.float64)))) / scale


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
