import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the CUDA extension")
    config.addinivalue_line("markers", "slow: long-running")


def tol_ok(got, ref, rel=1e-4, abs_=1e-6):
    """North-star bar (BASELINE.json): max|err| <= 1e-4 * max|ref| + 1e-6,
    applied per output tensor per instance."""
    import numpy as np
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (got.shape, ref.shape)
    if ref.size == 0:
        return True, 0.0, 0.0
    err = float(np.max(np.abs(got - ref)))
    bound = rel * float(np.max(np.abs(ref))) + abs_
    return err <= bound, err, bound
