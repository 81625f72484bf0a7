#!/usr/bin/env python
"""Per-kernel timing on the c5 shape (development tool, not the bench).

    python tools/kbench.py [--T 65536] [--reps 5] [--only detect|gram|cg]

Times fpm_gram, fpm_cg (A from HBM) and the fused fpm_detect with CUDA events
on the launching stream; prints ms per launch, detections/s and the fp64 /
HBM rooflines of each.
"""

import argparse
import ctypes
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2504_09820_b200 import _lib  # noqa: E402
from paper_2504_09820_b200.detect import DetectorSpec  # noqa: E402
from paper_2504_09820_b200.solvers import _stream  # noqa: E402


def timeit(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=65536)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--only", default="")
    ap.add_argument("--precision", default="fp16")
    ap.add_argument("--M", type=int, default=bench.M)
    ap.add_argument("--N", type=int, default=bench.N)
    ap.add_argument("--L", type=int, default=bench.L)
    ap.add_argument("--trace", action="store_true")
    ap.add_argument("--wstrace", action="store_true")
    ap.add_argument("--cgtrace", action="store_true")
    ap.add_argument("--cgwtrace", action="store_true")
    ap.add_argument("--alg", default="fp_bj_cg", choices=list(_lib.FPM_ALG))
    ap.add_argument("--iters", type=int, default=bench.ITERS)
    ap.add_argument("--gram32", action="store_true", help="FP32-Gram extension (FPM_FLAG_GRAM_FP32)")
    a = ap.parse_args()
    bench.ITERS = a.iters
    bench.M, bench.N, bench.L = a.M, a.N, a.L
    M, N, L, T = a.M, a.N, a.L, a.T
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    H, y, bits = bench.gen_inputs(T, 0, dev)
    det = DetectorSpec("fp_bj_cg", iters=bench.ITERS, L=L, matvec=a.precision, inner=a.precision)
    ps = _lib.precision_struct(det.precision())
    A = torch.empty((T, N, N), dtype=torch.complex128, device=dev)
    b = torch.empty((T, N), dtype=torch.complex128, device=dev)
    x = torch.empty((T, N), dtype=torch.complex128, device=dev)
    mv = torch.zeros((T, N * L), dtype=torch.complex128, device=dev)
    brk = torch.empty((T,), dtype=torch.int32, device=dev)
    div = torch.empty((T,), dtype=torch.int32, device=dev)
    cnt = torch.zeros((8,), dtype=torch.int64, device=dev)
    st = _stream()
    out = {}
    fg = 4 * M * N * (N + 1) + 8 * M * N
    pk = ctypes.c_double()
    _lib.check(lib.fpm_probe_fp64(200000, ctypes.byref(pk)), "probe")
    out["fp64_peak_tops"] = pk.value / 1e12

    def gram():
        _lib.check(lib.fpm_gram(H.data_ptr(), y.data_ptr(), T, M, N, bench.SIGMA2, A.data_ptr(), b.data_ptr(), st),
                   "gram")

    def bj():
        _lib.check(lib.fpm_bj_setup(A.data_ptr(), T, N, L, 0, mv.data_ptr(), None, st), "bj")

    def cg():
        _lib.check(lib.fpm_cg(A.data_ptr(), b.data_ptr(), mv.data_ptr(), T, N, L, bench.ITERS, ps, 0, x.data_ptr(),
                              brk.data_ptr(), div.data_ptr(), st), "cg")

    def cgx():  # run_batch boundary with the histories the Python mirror always requests
        _lib.check(lib.fpm_cg_ex(A.data_ptr(), b.data_ptr(), mv.data_ptr(), T, N, L, bench.ITERS, ps, 0,
                                 x.data_ptr(), brk.data_ptr(), div.data_ptr(), ctypes.byref(hist), st), "cg_ex")

    hres = torch.empty((bench.ITERS + 1, T), dtype=torch.float64, device=dev)
    hxn = torch.empty_like(hres)
    hal = torch.empty((bench.ITERS, T), dtype=torch.complex128, device=dev)
    hbe = torch.empty_like(hal)
    hconv = torch.empty((T,), dtype=torch.int32, device=dev)
    hist = _lib.CgHistory(hres.data_ptr(), hxn.data_ptr(), hal.data_ptr(), hbe.data_ptr(), hconv.data_ptr(),
                          1e-6, None, None)

    def fused():
        _lib.check(lib.fpm_detect(H.data_ptr(), y.data_ptr(), bits.data_ptr(), T, M, N, bench.SIGMA2, _lib.FPM_ALG[a.alg] | (_lib.FPM_FLAG_GRAM_FP32 if a.gram32 else 0), L,
                                  bench.ITERS, ps, 0, 16, None, x.data_ptr(), brk.data_ptr(), div.data_ptr(), None,
                                  cnt.data_ptr(), st), "detect")

    if a.only in ("", "gram"):
        ms = timeit(gram, a.reps)
        out["gram"] = {"ms": ms, "det_s": T / ms * 1e3, "fp64_frac": fg * T / (ms / 1e3) / pk.value}
    if a.only in ("", "cg"):
        gram()
        bj()
        ms = timeit(cg, a.reps)
        byts = 16 * N * N + 16 * N * (2 + L) + 8
        out["cg"] = {"ms": ms, "det_s": T / ms * 1e3, "hbm_gbs": byts * T / (ms / 1e3) / 1e9,
                     "hbm_frac": byts * T / (ms / 1e3) / 6554.9e9}
    if a.only == "cgx":
        gram()
        bj()
        ms = timeit(cgx, a.reps)
        out["cg_hist"] = {"ms": ms, "det_s": T / ms * 1e3, "kernel": lib.fpm_last_kernel().decode()}
    if a.cgtrace:  # standalone CG kernel, CTA 0 phase stamps (one wave: 1 CTA per SM)
        gram()
        bj()
        tr = torch.zeros(160, dtype=torch.int64, device=dev)
        lib.fpm_debug_set_trace(tr.data_ptr())
        cg()
        torch.cuda.synchronize()
        lib.fpm_debug_set_trace(None)
        c = tr.cpu().tolist()
        ph = ["A:matvec", "B:phi/alpha", "C:axpy+z", "E:rho1/beta", "-", "F:commit+p"]
        o = {"init": c[0] - c[60]}
        prev = c[0]
        for it in range(8):
            for k in range(6):
                v = c[1 + it * 6 + k]
                if v:
                    o.setdefault(ph[k], []).append(v - prev)
                    prev = v
        o["total"] = prev - c[60]
        o["A_detail_it2"] = [c[75] - c[1 + 6 + 5 - 6 + 0] if False else c[75] - c[6], c[76] - c[75], c[77] - c[76], c[1 + 6] - c[77]]
        o["B_detail_it2"] = [c[78] - c[1 + 6], c[79] - c[78], c[80] - c[79], c[1 + 6 + 1] - c[80]]
        o["C_detail_it2"] = [c[71] - c[70], c[72] - c[71], c[73] - c[72], c[74] - c[73], c[1 + 6 + 2] - c[74]]
        out["cg_trace"] = o
    if a.cgwtrace:  # warp CG: per-realization load / compute clocks and SM residency
        gram()
        bj()
        tr = torch.zeros(T * 4 + 256, dtype=torch.int64, device=dev)
        lib.fpm_debug_set_trace(tr.data_ptr())
        cg()
        torch.cuda.synchronize()
        lib.fpm_debug_set_trace(None)
        ph = tr[T * 4:].cpu().tolist()
        t4 = tr[:T * 4].view(T, 4).cpu()
        load = (t4[:, 1] - t4[:, 0]).double()
        comp = (t4[:, 2] - t4[:, 1]).double()
        res = []
        for sm in range(148):
            sel = t4[:, 3] == sm
            if sel.any():
                span = (t4[sel, 2].max() - t4[sel, 0].min()).item()
                res.append(((t4[sel, 2] - t4[sel, 0]).double().sum() / span).item())
        out["cgw_trace"] = {"load_cyc": load.mean().item(), "compute_cyc": comp.mean().item(),
                            "resident_per_sm": sum(res) / len(res), "compute_per_sweep": comp.mean().item() / bench.ITERS}
        names = ["matvec", "rho0", "phi", "alpha", "x,r", "z", "rho1", "beta", "p"]
        sweeps = []
        for it in range(1, bench.ITERS):  # sweep it+1 relative to the end of sweep it
            prev = ph[(it - 1) * 10 + 8]
            row = {}
            for k, nm in enumerate(names):
                v = ph[it * 10 + k]
                row[nm] = v - prev
                prev = v
            sweeps.append(row)
        out["cgw_phases_r0"] = sweeps[:3]
    if a.wstrace:
        tr = torch.zeros(160, dtype=torch.int64, device=dev)
        lib.fpm_debug_set_trace(tr.data_ptr())
        fused()
        torch.cuda.synchronize()
        lib.fpm_debug_set_trace(None)
        t = tr.cpu().tolist()
        t0 = t[0]
        out["ws_timeline"] = [{"gram_start": t[j*8]-t0, "gram_loop": t[j*8+1]-t[j*8], "slot_wait": t[j*8+2]-t[j*8+1],
                               "handoff": t[j*8+3]-t[j*8+2], "cg_start": t[j*8+4]-t0, "cg_bj_cg": t[j*8+5]-t[j*8+4],
                               "w0_empty_wait": t[j*8+6], "w0_full_wait": t[j*8+7], "w1_full_wait": t[64+j]}
                              for j in range(8)]
        out["ws_warp_loopend_g2"] = [t[72 + w] - t[2*8+0] for w in range(12)]
        c = t[96:160]
        if c[60]:
            ph = ["A:matvec", "B:phi/alpha", "C:axpy+z", "E:rho1/beta", "-", "F:commit+p"]
            out["ws_cg_g2"] = {"bj": c[60] - t[2*8+4], "init": c[0] - c[60]}
            prev = c[0]
            for it in range(8):
                for k in range(6):
                    v = c[1 + it * 6 + k]
                    if v:
                        out["ws_cg_g2"].setdefault(ph[k], []).append(v - prev)
                        prev = v
    if a.trace:
        tr = torch.zeros(64, dtype=torch.int64, device=dev)
        lib.fpm_debug_set_trace(tr.data_ptr())
        fused()
        torch.cuda.synchronize()
        lib.fpm_debug_set_trace(None)
        t = tr.cpu().tolist()
        names = {1: "gram", 2: "bj", 3: "A:init+matvec", 4: "B:phi/alpha", 5: "C:axpy", 6: "D:commit/z",
                 7: "E:rho1/beta", 8: "F:p", 9: "cg_rest(it>=2)", 10: "cg_tail", 15: "slice+writeback"}
        prev = t[0]
        out["trace_cycles"] = {}
        for i in sorted(names):
            if t[i] == 0:
                continue
            out["trace_cycles"][names[i]] = t[i] - prev
            prev = t[i]
        out["trace_cycles"]["total"] = t[15] - t[0]
        out["trace_cycles"]["gram.mainloop"] = t[16] - t[0]
        out["trace_cycles"]["gram.epilogue"] = t[1] - t[16]
        out["trace_cycles"]["gram.producer_empty_wait"] = t[16 + 5]
        out["trace_cycles"]["gram.w0_full_wait"] = t[16 + 6]
        out["trace_cycles"]["gram.w1_full_wait"] = t[16 + 7]
        out["trace_cycles"]["gram.warp_finish"] = [t[16 + 8 + w] - t[0] for w in range(16)]
    if a.only in ("", "detect"):
        ms = timeit(fused, a.reps)
        out["detect"] = {"ms": ms, "det_s": T / ms * 1e3, "fp64_frac": fg * T / (ms / 1e3) / pk.value}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
