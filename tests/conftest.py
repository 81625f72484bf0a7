"""Shared test plumbing.

Markers: `gpu` = needs a B200 (run with `-m gpu` on the GPU box); everything
else runs on CPU here.  The oracle (oracle/fpm_oracle.py) is test
infrastructure and is imported only from tests.
"""

import glob
import os
import subprocess
import sys
import tempfile

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


# The library reads its FPM_* planner knobs ONCE, when it loads (no per-call
# getenv).  Tests that force another kernel path (FPM_NO_WS, FPM_NO_CGW,
# FPM_FORCE_GENERIC, FPM_CGW_TMEM) therefore run that half in a fresh
# interpreter: the parent calls run_knob_child(nodeid, knobs), the child test
# (decorated @knob_child) runs only there and may hand arrays back through
# save_child_out(**arrays).
IN_CHILD = os.environ.get("FPM_TEST_CHILD") == "1"
knob_child = pytest.mark.skipif(not IN_CHILD, reason="child half of a knob test (runs in a fresh process)")


def run_knob_child(nodeid: str, knobs: dict, timeout: int = 900) -> dict:
    env = dict(os.environ)
    env.update(knobs)
    env["FPM_TEST_CHILD"] = "1"
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "out.npz")
        env["FPM_TEST_CHILD_OUT"] = out
        r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", nodeid],
                           cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
        assert r.returncode == 0 and " passed" in r.stdout, (nodeid, knobs, r.stdout[-4000:], r.stderr[-2000:])
        if not os.path.exists(out):
            return {}
        with np.load(out, allow_pickle=False) as z:
            return {k: z[k] for k in z.files}


def save_child_out(**arrays) -> None:
    np.savez(os.environ["FPM_TEST_CHILD_OUT"], **arrays)
