#!/usr/bin/env python
"""Merge the per-config full-size parity records written by
tests/test_gpu_fullsize_parity.py (gpurun_out/parity/parity_<cfg>.json) into
the committed summary profiles/r02_parity.json (re-checked on CPU by
tests/test_parity_record.py).   python tools/merge_parity.py"""
import glob
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = os.path.join(ROOT, "profiles", "r02_parity.json")
prev = json.load(open(out))
recs = {}
for p in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "parity", "parity_*.json"))):
    r = json.load(open(p))
    recs[r["config"]] = r
keep = {r["config"]: r for r in prev["records"]}
keep.update(recs)
prev["records"] = [keep[k] for k in sorted(keep)]
json.dump(prev, open(out, "w"), indent=1)
print("merged", sorted(recs), "->", out)
