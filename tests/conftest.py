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


@pytest.fixture
def rng():
    # the reference suite's fixed seed (pkg/tests/conftest.py:7-9)
    return np.random.default_rng(20240817)


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


def random_model_arrays(n, rng, sigma_range=(0.05, 0.6)):
    """The reference's ``random_model`` draws (pkg/tests/conftest.py:12-20)."""
    return (
        rng.normal(0.0, 2.0, n),
        rng.normal(0.0, 2.0, n),
        rng.uniform(*sigma_range, n),
        rng.uniform(*sigma_range, n),
    )
