import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 and the built libhelmsolve_b200.so")


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


def complex_noise(rng, shape, scale=1.0):
    return scale * (rng.standard_normal(shape) + 1j * rng.standard_normal(shape))


def relerr(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def history_dev(h, ref):
    """max over common entries of |h - ref| / ref (the north-star per-iteration bar)."""
    n = min(len(h), len(ref))
    h, ref = np.asarray(h[:n]), np.asarray(ref[:n])
    return float(np.max(np.abs(h - ref) / np.abs(ref)))
