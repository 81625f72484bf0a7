#!/usr/bin/env python
"""Smoke-sized launches of every hand-written kernel, with our own race /
bounds / deadlock checks (compute-sanitizer is closed on this GPU pool):

    python tools/sanitize_cases.py [--dump out.npz]
    python tools/sanitize_cases.py --racecheck [--seeds 6]

Cases: the persistent warp-specialised detector (fp16 and fp64 hand-off
slots, several groups per CTA and a partial last group, on-chip and injected
block inverses, N = 16 / 32 / 64, 64-QAM), the fallback fused kernel (N =
128), the composed FP32-Gram path, the warp CG at the run_batch boundary
(with and without histories, every native kind), the lockstep CG (generic
format), the LMMSE comparator, the fused generator.

Checks:
  * guard bands: every output of the C-ABI calls sits between canary
    regions that must be untouched afterwards (out-of-bounds global writes);
  * --racecheck: the cases are re-run in fresh processes on the CHECKED
    diagnostic library (libfpmimo_b200_checked.so: -DFPM_DIAG -DFPM_CHECKED,
    built by tools/build_checked.sh) with schedule perturbation seeds
    (FPM_DEBUG bits 16..31: warps sleep pseudo-random 0..4 us at every
    mbarrier / named-barrier synchronisation site) -- a missing barrier or a
    wrong mbarrier phase changes the bits of some seed's results; every run
    must be bit-identical to the product library's.  The checked build also
    traps on an mbarrier wait that exceeds ~10 s (deadlock) and on a
    shared-memory layout outside the launch's dynamic allocation.
"""

from __future__ import annotations

import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CANARY = 0x5A
GUARD = 4096  # bytes on each side


def _guarded(torch, shape, dtype, dev):
    """Tensor view inside a canary-filled allocation."""
    n = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
    raw = torch.full((n + 2 * GUARD,), CANARY, dtype=torch.uint8, device=dev)
    view = raw[GUARD:GUARD + n].view(dtype).view(shape)
    return raw, view


def _guards_ok(raw):
    h = raw.cpu().numpy()
    return bool((h[:GUARD] == CANARY).all() and (h[-GUARD:] == CANARY).all())


def run_cases():
    import torch
    from paper_2504_09820_b200 import _lib, channel
    from paper_2504_09820_b200.detect import DetectorSpec, detect
    from paper_2504_09820_b200.formats import get_format, make_format
    from paper_2504_09820_b200.solvers import PrecisionConfig, _stream, build_blocks_batch, run_batch

    dev = torch.device("cuda", 0)
    lib = _lib.load()
    out = {}
    guards = []

    def batch(M, N, T, qam=16, zeta=0.5, snr=15.0):
        return channel.simulate_batch(M, N, zeta, zeta, snr, 0, T, 7, qam=qam, device=dev)

    def fused(tag, det, b, T, M, N, qam=16, minv=None):
        """fpm_detect through the C ABI with guarded outputs."""
        bps = 4 if qam == 16 else 6
        rx_raw, x = _guarded(torch, (T, N), torch.complex128, dev)
        rb_raw, brk = _guarded(torch, (T,), torch.int32, dev)
        rd_raw, div = _guarded(torch, (T,), torch.int32, dev)
        rr_raw, rx = _guarded(torch, (T, bps * N), torch.uint8, dev)
        rc_raw, cnt = _guarded(torch, (_lib.NCOUNTERS,), torch.int64, dev)
        cnt.zero_()
        L = det.L or 1
        alg = _lib.FPM_ALG[det.algorithm] | (_lib.FPM_FLAG_GRAM_FP32 if det.gram == "fp32" else 0)
        _lib.check(lib.fpm_detect(b["H_est"].data_ptr(), b["y"].data_ptr(), b["bits"].data_ptr(), T, M, N,
                                  b["sigma_n2"], alg, L, det.iters, _lib.precision_struct(det.precision()),
                                  _lib.FPM_RHO[det.rho_update], qam, None if minv is None else minv.data_ptr(),
                                  x.data_ptr(), brk.data_ptr(), div.data_ptr(), rx.data_ptr(), cnt.data_ptr(),
                                  _stream()), tag)
        torch.cuda.synchronize()
        guards.extend((tag, r) for r in (rx_raw, rb_raw, rd_raw, rr_raw, rc_raw))
        out[tag + ".x"] = x.cpu().numpy()
        out[tag + ".flags"] = np.stack([brk.cpu().numpy(), div.cpu().numpy()])
        out[tag + ".rx"] = rx.cpu().numpy()
        out[tag + ".cnt"] = cnt.cpu().numpy()
        out[tag + ".kernel"] = np.array(lib.fpm_last_kernel().decode())
        assert int(cnt[4]) == T, (tag, cnt)

    # persistent WS kernel at N = 64 (R = 2): 148 CTAs x 2 groups + a partial
    # group; fp16 slot and fp64 slot; on-chip block inverses
    T = 148 * 2 * 2 + 1
    b = batch(128, 64, T)
    for mv in ("fp16", "fp64"):
        fused(f"ws_n64_{mv}", DetectorSpec("fp_bj_cg", iters=8, L=4, matvec=mv, inner=mv), b, T, 128, 64)
    # injected inverses + textbook rho
    from paper_2504_09820_b200.detect import gram_mf
    A, bb = gram_mf(b["H_est"], b["y"], b["sigma_n2"])
    bl = build_blocks_batch(A, 4)
    fused("ws_n64_injected_textbook", DetectorSpec("fp_bj_cg", iters=4, L=4, matvec="fp16", inner="fp16",
                                                   rho_update="textbook"), b, T, 128, 64, minv=bl.packed)
    out["gram.A"] = A.cpu().numpy()
    out["gram.b"] = bb.cpu().numpy()
    # small N (large R per group), partial group; 64-QAM at N = 64 (c3 shape)
    for (M, N, alg, mv) in ((128, 16, "cg", "fp64"), (128, 32, "fp_cg", "fp16"), (128, 32, "fp_cg", "bfloat16")):
        bs = batch(M, N, 300)
        det = DetectorSpec(alg, iters=6, **({} if alg == "cg" else dict(matvec=mv, inner=mv)))
        fused(f"ws_n{N}_{mv}", det, bs, 300, M, N)
    b3 = batch(256, 64, 301, qam=64, zeta=0.7, snr=20.0)
    fused("ws_c3_64qam", DetectorSpec("fp_bj_cg", iters=6, L=4, matvec="fp16", inner="fp16"), b3, 301, 256, 64, qam=64)
    # N = 128 (c4 shape), 64-QAM: fused fallback kernel and the FP32-Gram path
    b4 = batch(512, 128, 40, qam=64, zeta=0.8, snr=25.0)
    for gram in ("fp64", "fp32"):
        fused(f"c4_{gram}", DetectorSpec("fp_bj_cg", iters=3, L=8, matvec="fp16", inner="fp16", gram=gram),
              b4, 40, 512, 128, qam=64)
    # run_batch boundary: warp CG (guarded outputs; histories on), lockstep CG (generic format)
    Ah, bh, mh = A[:300].contiguous(), bb[:300].contiguous(), bl.packed[:300].contiguous()
    for mv in ("fp16", "bfloat16", "fp32", "fp64"):
        pc = PrecisionConfig(matvec=get_format(mv), inner=get_format(mv))
        res = run_batch(Ah, bh, 5, pc, build_blocks_batch(Ah, 4))
        out[f"run_batch_{mv}.x"] = res.x.cpu().numpy()
        out[f"run_batch_{mv}.res"] = res.residual_norms.cpu().numpy()
        rx_raw, x = _guarded(torch, (300, 64), torch.complex128, dev)
        rb_raw, brk = _guarded(torch, (300,), torch.int32, dev)
        rd_raw, div = _guarded(torch, (300,), torch.int32, dev)
        _lib.check(lib.fpm_cg(Ah.data_ptr(), bh.data_ptr(), mh.data_ptr(), 300, 64, 4, 5, _lib.precision_struct(pc),
                              0, x.data_ptr(), brk.data_ptr(), div.data_ptr(), _stream()), "fpm_cg")
        torch.cuda.synchronize()
        guards.extend((f"fpm_cg_{mv}", r) for r in (rx_raw, rb_raw, rd_raw))
        out[f"fpm_cg_{mv}.x"] = x.cpu().numpy()
        out[f"fpm_cg_{mv}.kernel"] = np.array(lib.fpm_last_kernel().decode())
    pc = PrecisionConfig(matvec=make_format(9, 5), inner=make_format(9, 5))
    out["run_batch_p9e5.x"] = run_batch(Ah[:20], bh[:20], 4, pc, None).x.cpu().numpy()
    # LMMSE comparator
    fused("lmmse", DetectorSpec("lmmse"), b, 100, 128, 64)
    # fused generator with guarded outputs
    M, N, Tg = 24, 40, 33
    rh, H = _guarded(torch, (Tg, M, N), torch.complex128, dev)
    re, He = _guarded(torch, (Tg, M, N), torch.complex128, dev)
    ry, y = _guarded(torch, (Tg, M), torch.complex128, dev)
    rbits, bits = _guarded(torch, (Tg, 6 * N), torch.uint8, dev)
    rs, s = _guarded(torch, (Tg, N), torch.complex128, dev)
    _lib.check(lib.fpm_simulate(5, 2, 1, 3, Tg, M, N, 0.6, 0.7, 1, 0, 64, 0.01, 0.002, H.data_ptr(), He.data_ptr(),
                                y.data_ptr(), bits.data_ptr(), s.data_ptr(), _stream()), "simulate")
    torch.cuda.synchronize()
    guards.extend(("fpm_simulate", r) for r in (rh, re, ry, rbits, rs))
    out["sim.H"] = H.cpu().numpy()
    out["sim.y"] = y.cpu().numpy()
    bad = [tag for tag, r in guards if not _guards_ok(r)]
    return out, bad


def _compare(a, b):
    diff = []
    for k in sorted(set(a) | set(b)):
        if k not in a or k not in b:
            diff.append(f"{k}: missing")
            continue
        x, y = a[k], b[k]
        if x.dtype.kind in "fc":
            same = x.shape == y.shape and np.array_equal(np.ascontiguousarray(x).view(np.uint8),
                                                         np.ascontiguousarray(y).view(np.uint8))
        else:
            same = np.array_equal(x, y)
        if not same:
            diff.append(k)
    return diff


def racecheck(seeds: int) -> int:
    import tempfile
    lib_chk = os.path.join(ROOT, "paper_2504_09820_b200", "libfpmimo_b200_checked.so")
    if not os.path.exists(lib_chk):
        print("no checked library: run tools/build_checked.sh first")
        return 2
    rc = 0
    with tempfile.TemporaryDirectory() as d:
        runs = [("product", {}, 0)] + [(f"checked seed {k}", {"FPM_LIB": lib_chk, "FPM_DEBUG": str(k << 16)}, k)
                                       for k in range(seeds)]
        ref = None
        for name, env, _ in runs:
            p = os.path.join(d, "o.npz")
            e = dict(os.environ)
            e.update(env)
            import time
            t0 = time.time()
            r = subprocess.run([sys.executable, os.path.abspath(__file__), "--dump", p], env=e, capture_output=True,
                               text=True, timeout=1200)
            wall = time.time() - t0
            if r.returncode != 0:
                print(f"{name}: FAILED rc={r.returncode}\n{r.stdout[-3000:]}\n{r.stderr[-3000:]}")
                rc = 1
                continue
            with np.load(p) as z:
                o = {k: z[k] for k in z.files}
            guard_line = [ln for ln in r.stdout.splitlines() if ln.startswith("guards")]
            if ref is None:
                ref = o
                print(f"{name}: {len(o)} outputs; {guard_line[0] if guard_line else ''}; {wall:.1f} s")
                continue
            diff = _compare(ref, o)
            print(f"{name}: {'bit-identical to the product run' if not diff else 'DIFFERS: ' + ', '.join(diff[:10])}; "
                  f"{guard_line[0] if guard_line else ''}; {wall:.1f} s")
            rc |= bool(diff)
    print("racecheck:", "PASS" if rc == 0 else "FAIL")
    return rc


def main():
    if "--racecheck" in sys.argv:
        seeds = int(sys.argv[sys.argv.index("--seeds") + 1]) if "--seeds" in sys.argv else 6
        sys.exit(racecheck(seeds))
    out, bad = run_cases()
    print(f"guards: {'all intact' if not bad else 'CORRUPTED: ' + ', '.join(bad)}")
    kern = sorted({str(v) for k, v in out.items() if k.endswith(".kernel")})
    print("kernels:", *kern, sep="\n  ")
    if "--dump" in sys.argv:
        np.savez(sys.argv[sys.argv.index("--dump") + 1], **{k: v for k, v in out.items() if not k.endswith(".kernel")})
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
