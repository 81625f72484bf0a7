#!/usr/bin/env python
"""Where the warps of fpm_detect_ws_kernel spend their time, from an ncu
report's source page (dev tool): stall samples per code region of
fpm_detect_ws.cuh (Gram row loops, stage / group overheads, hand-off, CG) and
the top lines outside the row loops.
    python tools/ncu_roles.py report.ncu-rep [top]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f = hdr = None
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
    if hdr is None or not r[0].isdigit():
        continue
    try:
        rows.append((f, int(r[0]), int(r[hdr.index("# Samples")]), int(r[hdr.index("Instructions Executed")]), r[1][:100]))
    except ValueError:
        continue
tot = sum(r[2] for r in rows)
# region markers in fpm_detect_ws.cuh found by text, so the tool follows edits
src = open(__file__.replace("tools/ncu_roles.py", "paper_2504_09820_b200/csrc/fpm_detect_ws.cuh")).read().split("\n")
def find(pat, start=0):
    for i in range(start, len(src)):
        if re.search(pat, src[i]):
            return i + 1
    return len(src)
g0 = find(r"=+ Gram warps =+")
stage = find(r"for \(int c = 0; c < nch; \+\+c\)", g0)
circ = find(r"software-pipelined: row mm\+1", stage)
half = find(r"half-pair job, software-pipelined", circ)
idle = find(r"idle job slot", half)
send = find(r"diag_jitter\(args.debug, 3", idle)
hand = find(r"hand-off: wait until the CG side", send)
puts = find(r"unsigned char\* sp = slots \+ slot", hand)
prod = find(r"=+ producer warp =+", puts)
cg = find(r"=+ CG warps =+", prod)
regions = [(g0, stage, "Gram: group prologue"), (stage, circ, "Gram: stage top"), (circ, half, "Gram: circulant loop"),
           (half, idle, "Gram: half-pair loop"), (idle, send, "Gram: idle/chains"), (send, hand, "Gram: stage end / gram-only"),
           (hand, puts, "Gram: slot wait"), (puts, prod, "Gram: hand-off stores"), (prod, cg, "producer / converter"),
           (cg, len(src) + 1, "CG role (ws)")]
agg = collections.Counter()
other = collections.Counter()
for fn, ln, s, ex, text in rows:
    if fn == "fpm_detect_ws.cuh":
        for a, b, n in regions:
            if a <= ln < b:
                agg[n] += s
                break
        else:
            agg["ws: setup"] += s
    else:
        other[fn] += s
print(f"total samples {tot}")
for a, b, n in regions:
    print(f"  {n:32s} lines {a:4d}-{b-1:4d}  {agg[n]:7d}  {100*agg[n]/tot:5.1f}%")
print(f"  {'ws: setup':32s} {'':15s} {agg['ws: setup']:7d}  {100*agg['ws: setup']/tot:5.1f}%")
for fn, s in other.most_common():
    print(f"  {fn:32s} {'':15s} {s:7d}  {100*s/tot:5.1f}%")
loops = set(range(circ, idle))
rest = [r for r in rows if not (r[0] == "fpm_detect_ws.cuh" and r[1] in loops) and not (r[0] == "fpm_gram.cuh" and 85 <= r[1] <= 97)]
rest.sort(key=lambda r: -r[2])
print("top lines outside the row loops:")
for fn, ln, s, ex, text in rest[:top]:
    print(f"  samp={s:6d} exec={ex:10d} {fn}:{ln} {text}")
