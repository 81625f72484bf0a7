"""bench.py's multi-GPU launcher and rank logic, dry-run on CPU (gloo): the
driver's `python bench.py --gpus N` must spawn N ranks itself when no torchrun
environment exists, split the global c5 batch (2^20) into contiguous shards
and all-reduce the counters inside every step."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT


def _run(*args):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       env=env, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout   # rank 0 alone prints
    return lines[0]


@pytest.mark.parametrize("gpus", [1, 2, 4])
def test_bench_spawns_ranks_and_splits_global_batch(gpus):
    T = 1 << 20
    out = _run("--gpus", str(gpus), "--dry-run", "--T", str(T), "--steps", "3")
    assert out["n_gpus"] == gpus and out["global_batch"] == T and out["scaling"] == "strong"
    sh = out["shards"]
    assert sh[0][0] == 0 and sh[-1][1] == T and all(sh[i][1] == sh[i + 1][0] for i in range(gpus - 1))
    assert max(b - a for a, b in sh) - min(b - a for a, b in sh) <= 1
    assert out["counters"]["trials"] == 3 * T   # all-reduced inside each of the 3 steps


def test_bench_uneven_global_batch():
    out = _run("--gpus", "2", "--dry-run", "--T", "1001", "--steps", "1")
    assert out["shards"] == [[0, 501], [501, 1001]] and out["counters"]["trials"] == 1001
