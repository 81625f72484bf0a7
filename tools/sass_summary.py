#!/usr/bin/env python
"""profiles/r02_sass_summary.txt: per-kernel counts of the SASS instructions
that show which hardware paths the product library uses (cuobjdump -sass of
every unit's object under paper_2504_09820_b200/_obj).  python tools/sass_summary.py > profiles/r02_sass_summary.txt"""
import glob
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["UTMALDG", "UBLKCP", "UBLKPF", "SYNCS", "USETMAXREG", "LDTM", "STTM", "DMUL", "DADD", "DFMA", "HFMA2", "HMUL2",
        "HADD2", "FMUL2", "FFMA2", "LDS.128", "STS.128", "LDL", "STL"]
print("# SASS summary of the product library (cuobjdump -sass of each unit's object, sm_100a), round 2")
print("# counts of the instructions that show which hardware paths the kernels use")
print("# (DFMA: inside the correctly rounded __ddiv_rn / __dsqrt_rn / __drcp_rn sequences only -- the Gram, CG sums and "
      "updates are -fmad=false DMUL / DADD)")
for obj in sorted(glob.glob(os.path.join(ROOT, "paper_2504_09820_b200", "_obj", "*.o"))):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    fn = None
    cnt = {}
    def flush():
        if fn and any(cnt.values()):
            print(f"{os.path.basename(obj):22s} {fn}")
            print("    " + ", ".join(f"{k} {cnt[k]}" for k in KEYS if cnt.get(k)))
    for line in out.split("\n"):
        m = re.search(r"Function : (\S+)", line)
        if m:
            flush()
            fn, cnt = m.group(1), {}
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_.]+)", line)
        if m:
            op = m.group(1)
            for k in KEYS:
                if op == k or op.startswith(k + ".") or (k in ("LDS.128", "STS.128") and op.startswith(k)):
                    cnt[k] = cnt.get(k, 0) + 1
    flush()
