import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(ROOT, "tests", "golden", "zk_golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


def rel_err(got, ref):
    """max over columns of |got-ref| / max(1, max|ref|) (the reference's
    convention, tests/test_acceptance.py:117-118)."""
    got = np.asarray(got)
    ref = np.asarray(ref)
    if ref.size == 0:
        return 0.0
    scale = np.maximum(1.0, np.abs(ref).max(axis=0))
    return float((np.abs(got - ref).max(axis=0) / scale).max())


def within_tolerance(got, ref):
    """north_star bar: |gpu - ref| <= 1e-13 + 1e-12 * max(1, max_col|ref|) per column."""
    got = np.asarray(got)
    ref = np.asarray(ref)
    if ref.size == 0:
        return True
    scale = np.maximum(1.0, np.abs(ref).max(axis=0))
    return bool((np.abs(got - ref) <= 1e-13 + 1e-12 * scale).all())
