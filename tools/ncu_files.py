#!/usr/bin/env python
"""Executed warp instructions and stall samples of an ncu report, summed per
source file and listed per line (dev tool):
    python tools/ncu_files.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f = None
hdr = None
rows = []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        s, ex = int(r[hdr.index("# Samples")]), int(r[hdr.index("Instructions Executed")])
    except (ValueError, IndexError):
        continue
    if not r[0].isdigit():
        continue
    rows.append((ex, s, f, int(r[0]), r[1][:100]))
if hdr:
    print("columns:", hdr[:12])
tot_ex = sum(r[0] for r in rows)
tot_s = sum(r[1] for r in rows)
by = collections.defaultdict(lambda: [0, 0])
for ex, s, f, ln, src in rows:
    by[f][0] += ex
    by[f][1] += s
print(f"total exec {tot_ex} samples {tot_s}")
for f, (ex, s) in sorted(by.items(), key=lambda kv: -kv[1][0]):
    print(f"{f:28s} exec {ex:12d} {100*ex/max(tot_ex,1):5.1f}%  samples {s:8d} {100*s/max(tot_s,1):5.1f}%")
rows.sort(reverse=True)
for ex, s, f, ln, src in rows[:top]:
    print(f"exec={ex:11d} {100*ex/max(tot_ex,1):5.1f}% samp={s:7d} {f}:{ln} {src}")
