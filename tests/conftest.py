"""Shared test plumbing.

Markers: `gpu` = needs a B200 (run with `-m gpu` on the GPU box); everything
else runs on CPU here.  The oracle (oracle/fpm_oracle.py) is test
infrastructure and is imported only from tests.
"""

import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")


def golden_cases():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "c*.npz"))
                  + glob.glob(os.path.join(GOLDEN, "mix_*.npz")))


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def bits_equal(a, b):
    """Bitwise equality of float/complex arrays (NaN == NaN, -0.0 != +0.0)."""
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    if np.iscomplexobj(a):
        a = a.view(np.float64)
        b = b.view(np.float64)
    na, nb = np.isnan(a), np.isnan(b)
    return bool(np.array_equal(na, nb) and np.array_equal(a[~na].view(np.uint64), b[~nb].view(np.uint64)))


@pytest.fixture
def oracle():
    import fpm_oracle
    return fpm_oracle
