#!/usr/bin/env python
"""Smoke-sized launches of every hand-written kernel, for compute-sanitizer
(racecheck / synccheck / memcheck; one tool per run):

    compute-sanitizer --tool racecheck --target-processes all \
        python tools/sanitize_cases.py [--tmem]

Covers the persistent warp-specialised detector (fp16 and fp64 hand-off
slots, several groups per CTA and a partial last group, on-chip and injected
block inverses, N = 16 / 32 / 64), the fallback fused kernel, the warp CG
(run_batch boundary, with and without histories; --tmem: the FPM_CGW_TMEM
variant -- the knob is read when the library loads, so pass it in the
environment), the lockstep CG, the FP32-Gram kernel, the LMMSE kernel, the
slicer and the generator.  Exits non-zero if a result disagrees with the
plain run's invariants (trial counts)."""

from __future__ import annotations

import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2504_09820_b200 import _lib, channel
    from paper_2504_09820_b200.detect import DetectorSpec, detect, gram_mf
    from paper_2504_09820_b200.solvers import build_blocks_batch, run_batch

    dev = torch.device("cuda", 0)
    lib = _lib.load()
    ran = []

    def batch(M, N, T, qam=16, zeta=0.5, snr=15.0):
        return channel.simulate_batch(M, N, zeta, zeta, snr, 0, T, 7, qam=qam, device=dev)

    # persistent WS kernel: 148 CTAs x (2 groups) + partial group at N = 64
    # (R = 2); fp16 slot and fp64 slot; on-chip inverses
    T = 148 * 2 * 2 + 1
    b = batch(128, 64, T)
    for mv in ("fp16", "fp64"):
        det = DetectorSpec("fp_bj_cg", iters=8, L=4, matvec=mv, inner=mv)
        r = detect(det, b["H_est"], b["y"], b["sigma_n2"], b["bits"])
        assert r.counters["trials"] == T
        ran.append(lib.fpm_last_kernel().decode())
    # injected inverses + textbook rho
    A, bb = gram_mf(b["H_est"], b["y"], b["sigma_n2"])
    ran.append("fpm_gram (WS Gram-only mode)")
    bl = build_blocks_batch(A, 4)
    ran.append("fpm_bj_kernel")
    det = DetectorSpec("fp_bj_cg", iters=4, L=4, matvec="fp16", inner="fp16", rho_update="textbook")
    r = detect(det, b["H_est"], b["y"], b["sigma_n2"], b["bits"], minv=bl.packed)
    ran.append(lib.fpm_last_kernel().decode())
    # small N: c1 / c2 shapes (large R per group), partial group
    for (M, N, alg, mv) in ((128, 16, "cg", "fp64"), (128, 32, "fp_cg", "fp16"), (128, 32, "fp_cg", "bfloat16")):
        bs = batch(M, N, 300)
        det = DetectorSpec(alg, iters=6, **({} if alg == "cg" else dict(matvec=mv, inner=mv)))
        r = detect(det, bs["H_est"], bs["y"], bs["sigma_n2"], bs["bits"])
        assert r.counters["trials"] == 300
        ran.append(lib.fpm_last_kernel().decode())
    # N = 128 (c4 shape), 64-QAM, fp16 and the FP32-Gram extension
    b4 = batch(512, 128, 40, qam=64, zeta=0.8, snr=25.0)
    for gram in ("fp64", "fp32"):
        det = DetectorSpec("fp_bj_cg", iters=3, L=8, matvec="fp16", inner="fp16", gram=gram)
        r = detect(det, b4["H_est"], b4["y"], b4["sigma_n2"], b4["bits"], qam=64)
        assert r.counters["trials"] == 40
        ran.append(lib.fpm_last_kernel().decode())
    # run_batch boundary: warp CG (histories on / off), lockstep CG (generic format)
    from paper_2504_09820_b200.formats import make_format
    Ah, bh = A[:300], bb[:300]
    for mv in ("fp16", "bfloat16", "fp32", "fp64"):
        from paper_2504_09820_b200.solvers import PrecisionConfig
        from paper_2504_09820_b200.formats import get_format
        pc = PrecisionConfig(matvec=get_format(mv), inner=get_format(mv))
        res = run_batch(Ah, bh, 5, pc, build_blocks_batch(Ah, 4))
        ran.append(f"run_batch[{mv}] histories")
        x = torch.empty_like(bh)
        brk = torch.empty(300, dtype=torch.int32, device=dev)
        div = torch.empty(300, dtype=torch.int32, device=dev)
        ps = _lib.precision_struct(pc)
        _lib.check(lib.fpm_cg(Ah.data_ptr(), bh.data_ptr(), bl.packed[:300].data_ptr(), 300, 64, 4, 5, ps, 0,
                              x.data_ptr(), brk.data_ptr(), div.data_ptr(), None), "fpm_cg")
        ran.append(lib.fpm_last_kernel().decode())
    pc = PrecisionConfig(matvec=make_format(9, 5), inner=make_format(9, 5))
    run_batch(Ah[:20], bh[:20], 4, pc, None)
    ran.append("run_batch[p9e5] (lockstep, generic)")
    # LMMSE comparator, slicer, generator
    r = detect(DetectorSpec("lmmse"), b["H_est"][:100], b["y"][:100], b["sigma_n2"], b["bits"][:100])
    ran.append(lib.fpm_last_kernel().decode())
    torch.cuda.synchronize()
    print("sanitize cases ran:", *ran, sep="\n  ")


if __name__ == "__main__":
    main()
