import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def rel_err(got, want):
    """proj/tests/support/oracles.hpp:55-58 — scale max(|a|,|b|,1), elementwise, max over entries."""
    import numpy as np

    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    scale = np.maximum(np.maximum(np.abs(got), np.abs(want)), 1.0)
    return float(np.max(np.abs(got - want) / scale)) if got.size else 0.0


def norm_rel_err(got, want):
    """Norm-wise relative error ||a-b|| / max(||b||, tiny)."""
    import numpy as np

    got = np.asarray(got, dtype=np.float64).ravel()
    want = np.asarray(want, dtype=np.float64).ravel()
    den = max(np.linalg.norm(want), 1e-300)
    return float(np.linalg.norm(got - want) / den)


@pytest.fixture(scope="session")
def orc():
    import oracle

    oracle.lib()
    return oracle
