#!/usr/bin/env python
"""Stall samples at every mbarrier wait site of an ncu report's SASS page
(dev tool; the barrier operand tells the sites apart):
    python tools/ncu_waits.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
hdr, body = rows[hi], rows[hi + 1:]
si, ei = hdr.index("# Samples"), hdr.index("Instructions Executed")
tot = sum(int(r[si]) for r in body if r[si].isdigit())
print("total samples", tot)
for k, r in enumerate(body):
    if "TRYWAIT" in r[1]:
        s = sum(int(body[q][si]) for q in range(k, min(len(body), k + 2)))
        if s or int(r[ei]):
            print(f"{k:6d} {r[1].strip()[:64]:64s} samples(+branch) {s:7d} {100*s/tot:5.1f}%  exec {r[ei]}")
