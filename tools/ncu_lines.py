#!/usr/bin/env python
"""Top source lines by warp-stall samples from an ncu report (dev tool):
    python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f = None
hdr = None
rows = []
tot = 0
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
        s, ni, ex = int(r[4]), int(r[5]), int(r[7])
    except (ValueError, IndexError):
        continue
    tot += s
    rows.append((s, ni, ex, f, r[0], r[1][:90]))
rows.sort(reverse=True)
print(f"total samples {tot}")
for s, ni, ex, f, ln, src in rows[:top]:
    print(f"{s:7d} {100*s/max(tot,1):5.1f}% ni={ni:6d} exec={ex:10d} {f}:{ln} {src}")
