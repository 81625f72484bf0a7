#!/usr/bin/env python
"""Fused-detector throughput on every BASELINE.json config shape (dev tool):
det/s and fraction of the measured FP64 rate (Gram ops), inputs from the
library generator.  python tools/cfgbench.py [--T 65536]"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_09820_b200 import _lib, channel  # noqa: E402
from paper_2504_09820_b200.detect import DetectorSpec  # noqa: E402
from paper_2504_09820_b200.solvers import _stream  # noqa: E402

CFGS = {  # name: (M, N, zeta, snr, qam, detector kwargs)
    "c1": (128, 16, 0.0, 10.0, 16, dict(algorithm="cg", iters=8)),
    "c2_fp16": (128, 32, 0.5, 10.0, 16, dict(algorithm="fp_cg", iters=10, matvec="fp16", inner="fp16")),
    "c2_bf16": (128, 32, 0.5, 10.0, 16, dict(algorithm="fp_cg", iters=10, matvec="bfloat16", inner="bfloat16")),
    "c3": (256, 64, 0.7, 20.0, 64, dict(algorithm="fp_bj_cg", iters=6, L=4, matvec="fp16", inner="fp16")),
    "c4": (512, 128, 0.8, 25.0, 64, dict(algorithm="fp_bj_cg", iters=8, L=8, matvec="fp16", inner="fp16")),
    "c4_gram32": (512, 128, 0.8, 25.0, 64, dict(algorithm="fp_bj_cg", iters=8, L=8, matvec="fp16", inner="fp16",
                                                 gram="fp32")),
    "c5_fp16": (128, 64, 0.5, 15.0, 16, dict(algorithm="fp_bj_cg", iters=8, L=4, matvec="fp16", inner="fp16")),
    "c5_bf16": (128, 64, 0.5, 15.0, 16, dict(algorithm="fp_bj_cg", iters=8, L=4, matvec="bfloat16", inner="bfloat16")),
    "c5_fp64": (128, 64, 0.5, 15.0, 16, dict(algorithm="fp_bj_cg", iters=8, L=4)),
    "c5_lmmse": (128, 64, 0.5, 15.0, 16, dict(algorithm="lmmse")),
}


def measure(name, T_req, lib, peak, dev, reps=3):
    """det/s and FP64 fraction of the fused detector on config `name`."""
    M, N, zeta, snr, qam, kw = CFGS[name]
    T = max(1024, min(T_req, (8 << 30) // (M * N * 16)))
    b = channel.simulate_batch(M, N, zeta, zeta, snr, 0, T, 20261020, qam=qam, device=dev)
    det = DetectorSpec(**kw)
    x = torch.empty((T, N), dtype=torch.complex128, device=dev)
    brk = torch.empty((T,), dtype=torch.int32, device=dev)
    div = torch.empty((T,), dtype=torch.int32, device=dev)
    cnt = torch.zeros((8,), dtype=torch.int64, device=dev)
    ps = _lib.precision_struct(det.precision())
    L = det.L or 1

    def run():
        alg = _lib.FPM_ALG[det.algorithm] | (_lib.FPM_FLAG_GRAM_FP32 if det.gram == "fp32" else 0)
        _lib.check(lib.fpm_detect(b["H_est"].data_ptr(), b["y"].data_ptr(), b["bits"].data_ptr(), T, M, N,
                                  b["sigma_n2"], alg, L, det.iters, ps, 0, qam, None,
                                  x.data_ptr(), brk.data_ptr(), div.data_ptr(), None, cnt.data_ptr(), _stream()), name)
    run()
    torch.cuda.synchronize()
    cnt.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    bps = 4 if qam == 16 else 6
    fg = 4 * M * N * (N + 1) + 8 * M * N
    out = {"T": T, "ms": round(ms, 3), "det_s": round(T / ms * 1e3), "kernel": lib.fpm_last_kernel().decode(),
           "ber": round(int(cnt[0]) / (reps * T * bps * N), 5)}
    if det.gram == "fp32":
        # binary32 Gram: against the packed non-fused FP32 ceiling (FMUL2 / FFMA2
        # with an exact +-1 multiplier: 128 ops/clk/SM = 2x the measured
        # non-fused fp64 DMUL/DADD rate of 64 ops/clk/SM)
        out["fp32x2_frac"] = round(fg * T / (ms / 1e3) / (2 * peak), 3)
        out["peak"] = "2 x fpm_probe_fp64 (packed binary32 non-fused ceiling)"
    else:
        out["fp64_frac"] = round(fg * T / (ms / 1e3) / peak, 3)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=65536)
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    lib = _lib.load()
    pk = ctypes.c_double()
    _lib.check(lib.fpm_probe_fp64(200000, ctypes.byref(pk)), "probe")
    dev = torch.device("cuda", 0)
    out = {}
    for name in CFGS:
        if a.only and a.only != name:
            continue
        out[name] = measure(name, a.T, lib, pk.value, dev)
        print(name, json.dumps(out[name]), flush=True)


if __name__ == "__main__":
    main()
