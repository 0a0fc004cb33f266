import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture
def rng():
    return np.random.default_rng(20240917)


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def unpack_cores(z, prefix):
    n = int(z[f"{prefix}_n"])
    return [np.array(z[f"{prefix}_{k}"]) for k in range(n)]
