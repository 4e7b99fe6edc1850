import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


GOLDEN = os.path.join(ROOT, "tests", "golden")


def rel_err(x, ref):
    """SURVEY.md §8(c) parity metric: per cell max|y - y_ref| / max|y_ref|,
    max over cells."""
    import numpy as np

    x = np.asarray(x, dtype=float).reshape(ref.shape[0], -1)
    ref = np.asarray(ref, dtype=float).reshape(ref.shape[0], -1)
    den = np.abs(ref).max(axis=1)
    den = np.where(den == 0, 1.0, den)
    return float((np.abs(x - ref).max(axis=1) / den).max())


@pytest.fixture(scope="session")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch
