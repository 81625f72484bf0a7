"""Build libfpmimo_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2504_09820_b200.build [--force]

Each format kind's kernels are a separate translation unit
(csrc/fpm_inst_<kind>.cu) compiled in parallel, then linked with the host
unit (csrc/fpm_host.cu).  Flags: -fmad=false (no FMA contraction: the
reference's arithmetic is separately rounded), no -use_fast_math / -ftz
(subnormals are part of the contract), -lineinfo for ncu source views.
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# FPM_BUILD_OUT / FPM_BUILD_OBJ: alternate output (development variants built
# with different FPM_NVCC_EXTRA macros, loaded through FPM_LIB)
OBJ = os.environ.get("FPM_BUILD_OBJ", os.path.join(HERE, "_obj"))
OUT = os.environ.get("FPM_BUILD_OUT", os.path.join(HERE, "libfpmimo_b200.so"))
HEADER = os.path.join(os.path.dirname(HERE), "include", "fpmimo_b200.h")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC"] + \
    os.environ.get("FPM_NVCC_EXTRA", "").split()


def _units():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [HEADER]


def _stamp() -> str:
    """Content hash of everything the library is built from: the compiler
    command line (nvcc path, FLAGS incl. FPM_NVCC_EXTRA), this script and every
    source / header.  Written next to the .so; a mismatch forces a rebuild (a
    pushed prebuilt library built from other sources or flags is never reused:
    bit-exactness depends on -fmad=false)."""
    h = hashlib.sha256()
    h.update(repr((NVCC, FLAGS, ARCH)).encode())
    for f in [os.path.abspath(__file__)] + _units() + _headers():
        h.update(os.path.basename(f).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()


def _stamp_path() -> str:
    return OUT + ".stamp"


def needs_build() -> bool:
    if not os.path.exists(OUT) or not os.path.exists(_stamp_path()):
        return True
    with open(_stamp_path()) as fh:
        return fh.read().strip() != _stamp()


def _compile(src: str, verbose: bool) -> tuple[str, str]:
    obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
    cmd = [NVCC, *FLAGS, "-c", src, "-o", obj] + (["-Xptxas", "-v"] if verbose else [])
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    if not (force or needs_build()):
        return OUT
    os.makedirs(OBJ, exist_ok=True)
    units = _units()
    with cf.ThreadPoolExecutor(max_workers=min(len(units), os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose), units))
    if verbose:
        for _, log in results:
            sys.stderr.write(log)
    cmd = [NVCC, *ARCH, "-shared", "-o", OUT + ".tmp"] + [o for o, _ in results]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}{r.stderr}")
    os.replace(OUT + ".tmp", OUT)
    with open(_stamp_path(), "w") as fh:
        fh.write(_stamp() + "\n")
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
