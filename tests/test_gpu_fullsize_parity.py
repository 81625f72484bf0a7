"""Full-size parity on the default fused path (on-chip block inverses) at
every BASELINE.json config's stated batch size, against the oracle on the
same inputs (tests/fullsize.py).  Each case
writes its record to gpurun_out/parity/ (committed summary:
profiles/r02_parity.json, re-checked by test_parity_record.py)."""

import os

import pytest

import fullsize
from conftest import ROOT

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2504_09820_b200 import build
    build.build()


@pytest.mark.parametrize("name", list(fullsize.CASES))
def test_fullsize_counts_identical_to_oracle(name):
    scale = float(os.environ.get("FPM_PARITY_SCALE", "1.0"))
    rec = fullsize.run_case(name, scale)
    fullsize.write(rec, os.path.join(ROOT, "gpurun_out", "parity"))
    bad = fullsize.check(rec)
    assert not bad, bad[:10]
