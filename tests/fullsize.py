"""Full-size parity at the BASELINE.json configs (VERDICT r01 "next round" #1).

For each config at its stated batch size, the DEFAULT fused GPU path
(on-chip block inverses, the path bench.py times) and the oracle (the CPU
restatement of the reference path: einsum Gram detect.py:215-218, LAPACK
block inverses solvers.py:232-253, run_batch solvers.py:262-393, slicer
detect.py:70-84, error sum :261) run on identical inputs; the oracle runs in
`workers` spawned processes over shared memory.  The chunk loop of
run_ber_sweep (detect.py:255-263) accumulates the counters the same way on
both sides.

Inputs: the library's GPU generator (channel.simulate_batch; keyed Philox),
copied to host for the oracle -- parity here is about the detector, the
inputs only have to be identical on both sides.

Bars (BASELINE.json north_star):
  * sliced bits identical per realization, hence bit-error, symbol-error,
    divergence and breakdown counts identical per (config, SNR, precision);
  * plain CG / FP-CG (no block inverses): x_hat bit-identical;
  * FP-BJ-CG (GPU fp64 Cholesky inverses vs LAPACK zgesv): per-realization
    normwise relative x_hat difference <= 1e-12 (fp64 matvec) or
    2^-(p-2) (p stored fraction bits of the matvec format).

This module is test infrastructure: it imports the oracle as the checker.
"""

from __future__ import annotations

import json
import math
import multiprocessing as mp
import os
import time
from multiprocessing import shared_memory

import numpy as np

SEED = 20261020
FRAC_BITS = {"fp64": 52, "fp32": 23, "fp16": 10, "bfloat16": 7}

# name: (M, N, zeta, snr list, qam, T, variants); variant = (label, algorithm, L, iters, fmt, gram)
CASES = {
    "c1": (128, 16, 0.0, [10.0], 16, 4096, [("cg_fp64", "cg", None, 8, "fp64", "fp64")]),
    "c2": (128, 32, 0.5, [float(s) for s in range(0, 21, 2)], 16, 8192,
           [("fp_cg_fp16", "fp_cg", None, 10, "fp16", "fp64"), ("fp_cg_bf16", "fp_cg", None, 10, "bfloat16", "fp64")]),
    "c3": (256, 64, 0.7, [20.0], 64, 16384, [("bj4_fp16", "fp_bj_cg", 4, 6, "fp16", "fp64")]),
    "c4": (512, 128, 0.8, [25.0], 64, 8192,
           [("bj8_fp16", "fp_bj_cg", 8, 8, "fp16", "fp64"), ("bj8_fp16_gram32", "fp_bj_cg", 8, 8, "fp16", "fp32")]),
    "c5": (128, 64, 0.5, [15.0], 16, 1 << 16,
           [("bj4_fp16", "fp_bj_cg", 4, 8, "fp16", "fp64"), ("bj4_fp64", "fp_bj_cg", 4, 8, "fp64", "fp64")]),
}


def scaled(name: str, scale: float):
    M, N, z, snrs, qam, T, vs = CASES[name]
    return M, N, z, snrs, qam, max(1, int(T * scale)), vs


# ---------------------------------------------------------------------------
# oracle side (spawned workers; shared-memory inputs)
# ---------------------------------------------------------------------------

def _attach(spec):
    shm = shared_memory.SharedMemory(name=spec[0])
    return shm, np.ndarray(spec[1], dtype=np.dtype(spec[2]), buffer=shm.buf)


def _oracle_task(task):
    os.environ["OMP_NUM_THREADS"] = "1"
    import fpm_oracle as O
    (hs, ys), lo, hi, sigma2, qam, variants = task
    shm_h, H = _attach(hs)
    shm_y, y = _attach(ys)
    try:
        Hc = np.array(H[lo:hi])
        yc = np.array(y[lo:hi])
    finally:
        shm_h.close()
        shm_y.close()
    fm = {"fp64": O.FP64, "fp32": O.FP32, "fp16": O.FP16, "bfloat16": O.BF16}
    grams = {}
    out = []
    for label, alg, L, iters, fmt, gram in variants:
        if gram not in grams:
            grams[gram] = O.gram_mf_fp32(Hc, yc, sigma2) if gram == "fp32" else O.gram_mf_einsum(Hc, yc, sigma2)
        A, b = grams[gram]
        mats = O.bj_inverses(A, L) if alg == "fp_bj_cg" else None
        f = O.FP64 if alg == "cg" else fm[fmt]
        r = O.cg_batch(A, b, iters, O.FP64, f, f, mats)
        rx = O.demod16(r.x) if qam == 16 else O.demod64(r.x)
        out.append((label, r.x, rx, r.breakdown_at, r.diverged_at))
    return lo, hi, out


def oracle_run(H, y, sigma2, qam, variants, workers, chunk=256):
    """Oracle outputs for every variant over the whole batch."""
    T = H.shape[0]
    shms = []
    specs = []
    try:
        for a in (H, y):
            shm = shared_memory.SharedMemory(create=True, size=max(1, a.nbytes))
            np.ndarray(a.shape, a.dtype, buffer=shm.buf)[...] = a
            shms.append(shm)
            specs.append((shm.name, a.shape, a.dtype.str))
        tasks = [(tuple(specs), lo, min(T, lo + chunk), sigma2, qam, variants) for lo in range(0, T, chunk)]
        ctx = mp.get_context("spawn")
        env_keep = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")}
        for k in env_keep:
            os.environ[k] = "1"
        try:
            with ctx.Pool(workers) as pool:
                parts = pool.map(_oracle_task, tasks, chunksize=1)
        finally:
            for k, v in env_keep.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
    finally:
        for shm in shms:
            shm.close()
            shm.unlink()
    res = {}
    N = None
    for lo, hi, outs in sorted(parts, key=lambda p: p[0]):
        for label, x, rx, brk, div in outs:
            N = x.shape[1]
            d = res.setdefault(label, {"x": [], "rx": [], "brk": [], "div": []})
            d["x"].append(x)
            d["rx"].append(rx)
            d["brk"].append(brk)
            d["div"].append(div)
    return {k: {kk: np.concatenate(vv) for kk, vv in v.items()} for k, v in res.items()}


# ---------------------------------------------------------------------------
# GPU side and comparison
# ---------------------------------------------------------------------------

def counts(rx, tx, brk, div, bps):
    diff = np.asarray(rx) != np.asarray(tx)
    T = diff.shape[0]
    return {"bit_errors": int(diff.sum()),
            "symbol_errors": int(diff.reshape(T, -1, bps).any(-1).sum()),
            "diverged": int((np.asarray(div) >= 0).sum()),
            "breakdown": int((np.asarray(brk) >= 0).sum())}


def run_case(name: str, scale: float = 1.0, workers: int | None = None, gpu_chunk: int = 4096) -> dict:
    import torch
    from paper_2504_09820_b200 import channel
    from paper_2504_09820_b200.detect import DetectorSpec, detect

    M, N, zeta, snrs, qam, T, variants = scaled(name, scale)
    bps = 4 if qam == 16 else 6
    workers = workers or min(64, os.cpu_count() or 1)
    dev = torch.device("cuda", 0)
    record = {"config": name, "M": M, "N": N, "zeta": zeta, "qam": qam, "T_per_point": T, "points": []}
    for pi, snr in enumerate(snrs):
        t0 = time.time()
        batch = channel.simulate_batch(M, N, zeta, zeta, snr, 0, T, SEED, point=pi, qam=qam, device=dev)
        sigma2 = float(batch["sigma_n2"])
        gpu = {}
        for label, alg, L, iters, fmt, gram in variants:
            det = DetectorSpec(alg, iters=iters, L=L, matvec=fmt, inner=fmt, gram=gram)
            xs, rxs, bks, dvs = [], [], [], []
            cnt = {}
            # run_ber_sweep's chunk loop (detect.py:255-263): counters accumulate per chunk
            for c0 in range(0, T, gpu_chunk):
                c1 = min(T, c0 + gpu_chunk)
                r = detect(det, batch["H_est"][c0:c1], batch["y"][c0:c1], sigma2, batch["bits"][c0:c1], qam=qam,
                           want_bits=True)
                torch.cuda.synchronize()
                xs.append(r.x.cpu().numpy())
                rxs.append(r.bits.cpu().numpy())
                bks.append(r.breakdown_at.cpu().numpy())
                dvs.append(r.diverged_at.cpu().numpy())
                for k, v in r.counters.items():
                    cnt[k] = cnt.get(k, 0) + v
            from paper_2504_09820_b200 import _lib
            gpu[label] = {"x": np.concatenate(xs), "rx": np.concatenate(rxs), "brk": np.concatenate(bks),
                          "div": np.concatenate(dvs), "counters": cnt,
                          "kernel": _lib.load().fpm_last_kernel().decode()}
        t_gpu = time.time() - t0
        H = batch["H_est"].cpu().numpy()
        y = batch["y"].cpu().numpy()
        tx = batch["bits"].cpu().numpy()
        del batch
        torch.cuda.empty_cache()
        t1 = time.time()
        ora = oracle_run(H, y, sigma2, qam, variants, workers)
        t_cpu = time.time() - t1
        del H, y
        for label, alg, L, iters, fmt, gram in variants:
            g, o = gpu[label], ora[label]
            gc = g["counters"]
            oc = counts(o["rx"], tx, o["brk"], o["div"], bps)
            gcounts = {k: gc[k] for k in oc}
            num = np.linalg.norm(g["x"] - o["x"], axis=1)
            den = np.linalg.norm(o["x"], axis=1)
            rel = np.where(den > 0, num / np.where(den > 0, den, 1.0), num)
            rel = np.where(np.isfinite(rel), rel, np.inf)
            tol = 1e-12 if (alg == "cg" or fmt == "fp64") else 2.0 ** -(FRAC_BITS[fmt] - 2)
            xb = np.ascontiguousarray(g["x"]).view(np.uint64)
            ob = np.ascontiguousarray(o["x"]).view(np.uint64)
            rec = {"snr_db": snr, "variant": label, "algorithm": alg, "L": L, "iters": iters, "matvec_inner": fmt,
                   "gram": gram, "T": T, "kernel": g["kernel"],
                   "gpu_counts": gcounts, "oracle_counts": oc, "counts_equal": gcounts == oc,
                   "bits_equal": bool(np.array_equal(g["rx"], o["rx"])),
                   "flags_equal": bool(np.array_equal(g["brk"], o["brk"]) and np.array_equal(g["div"], o["div"])),
                   "gpu_trials": int(gc["trials"]), "nonpd": int(gc["nonpd"]),
                   "x_bit_identical_frac": float(np.mean(np.all(xb == ob, axis=1))),
                   "x_max_rel_err": float(rel.max()) if rel.size else 0.0, "x_tol": tol,
                   "x_within_tol": bool(rel.size == 0 or rel.max() <= tol),
                   "must_be_bit_exact": alg != "fp_bj_cg",
                   "gpu_s": round(t_gpu, 2), "oracle_s": round(t_cpu, 2), "oracle_workers": workers}
            record["points"].append(rec)
    return record


def check(record: dict) -> list:
    """Failures of one record against the bars (empty list = pass)."""
    bad = []
    for p in record["points"]:
        tag = f"{record['config']} {p['variant']} snr={p['snr_db']}"
        if not p["counts_equal"]:
            bad.append(f"{tag}: counts {p['gpu_counts']} != {p['oracle_counts']}")
        if not p["bits_equal"]:
            bad.append(f"{tag}: sliced bits differ")
        if not p["flags_equal"]:
            bad.append(f"{tag}: breakdown/diverged flags differ")
        if p["gpu_trials"] != p["T"]:
            bad.append(f"{tag}: trials {p['gpu_trials']} != {p['T']}")
        if not p["x_within_tol"]:
            bad.append(f"{tag}: x rel err {p['x_max_rel_err']:.3g} > {p['x_tol']:.3g}")
        if p["must_be_bit_exact"] and p["x_bit_identical_frac"] != 1.0:
            bad.append(f"{tag}: x not bit-identical ({p['x_bit_identical_frac']})")
    return bad


def write(record: dict, out_dir: str) -> str:
    os.makedirs(out_dir, exist_ok=True)
    p = os.path.join(out_dir, f"parity_{record['config']}.json")
    with open(p, "w") as f:
        json.dump(record, f, indent=1)
    return p


if __name__ == "__main__":  # python tests/fullsize.py [c1 c2 ...] [--scale s]
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [os.path.dirname(here), os.path.join(os.path.dirname(here), "oracle")]
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    scale = float(sys.argv[sys.argv.index("--scale") + 1]) if "--scale" in sys.argv else 1.0
    for name in [a for a in args if a in CASES] or list(CASES):
        rec = run_case(name, scale)
        path = write(rec, os.path.join(os.path.dirname(here), "gpurun_out", "parity"))
        print(name, "FAIL" if check(rec) else "ok", path, check(rec)[:5], flush=True)
