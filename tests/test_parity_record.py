"""CPU re-check of the committed full-size parity record
(profiles/r02_parity.json, written by tests/test_gpu_fullsize_parity.py on a
B200): every BASELINE config was run at its stated size and met the bars."""

import json
import os

import fullsize
from conftest import ROOT

WANT = {  # config: (realizations per point, points, variants) -- VERDICT r01 next-round #1
    "c1": (4096, 1, {"cg_fp64"}),
    "c2": (8192, 11, {"fp_cg_fp16", "fp_cg_bf16"}),
    "c3": (16384, 1, {"bj4_fp16"}),
    "c4": (8192, 1, {"bj8_fp16", "bj8_fp16_gram32"}),
    "c5": (65536, 1, {"bj4_fp16", "bj4_fp64"}),
}


def test_committed_parity_record_covers_every_config_and_passes():
    with open(os.path.join(ROOT, "profiles", "r02_parity.json")) as f:
        rec = json.load(f)
    by = {r["config"]: r for r in rec["records"]}
    assert set(by) == set(WANT)
    for name, (T, npts, variants) in WANT.items():
        r = by[name]
        assert r["T_per_point"] >= T, name
        assert {p["variant"] for p in r["points"]} == variants, name
        assert len({p["snr_db"] for p in r["points"]}) == npts, name
        assert all(p["T"] >= T for p in r["points"]), name
        assert fullsize.check(r) == [], (name, fullsize.check(r)[:3])
        for p in r["points"]:
            assert p["counts_equal"] and p["bits_equal"] and p["flags_equal"] and p["x_within_tol"]
