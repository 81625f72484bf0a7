"""Multi-GPU sharding of the detector.

Realizations are independent (solvers.py:270-272) and the reference's sweep
is invariant to chunking (detect.py:240-245, tests/test_detect.py:133-140),
so the path shards by trial range: one process per GPU, each rank detects a
contiguous slice of every chunk, no data-path collective.  The only exchange
is one int64 all-reduce of the error counters per SNR point (all detectors
in one tensor) -- NCCL on GPUs, gloo in the CPU tests.

    sharded_ber_sweep(cfg, simulate)   <- run_ber_sweep, detect.py:240-270
    shard_range(T, rank, world)        contiguous, balanced trial slices
    allreduce_counters(cnt)            the one collective
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ContractViolation

__all__ = ["shard_range", "dist_info", "init", "allreduce_counters", "sharded_detect", "sharded_ber_sweep",
           "BERPoint", "BERCurve", "wilson_interval"]


def shard_range(T: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of the T realizations owned by `rank`: contiguous, sizes
    differ by at most one, union is [0, T)."""
    if world < 1 or not 0 <= rank < world or T < 0:
        raise ContractViolation("bad shard request")
    q, r = divmod(T, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def dist_info():
    """(rank, world, group initialised) without requiring torch.distributed."""
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist.get_rank(), dist.get_world_size(), True
    except ImportError:  # pragma: no cover
        pass
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), False


def init(backend: str | None = None):
    """One process per GPU from the torchrun environment (RANK, WORLD_SIZE,
    LOCAL_RANK, MASTER_ADDR/PORT).  Returns (rank, world, device)."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    backend = backend or ("nccl" if torch.cuda.is_available() else "gloo")
    dev = torch.device("cuda", local) if backend == "nccl" else torch.device("cpu")
    if dev.type == "cuda":  # bind the rank's GPU before NCCL initialises
        torch.cuda.set_device(dev)
    if world > 1 and not dist.is_initialized():
        if dev.type == "cuda":
            dist.init_process_group(backend, device_id=dev)
        else:
            dist.init_process_group(backend)
    rank = dist.get_rank() if dist.is_initialized() else 0
    return rank, world, dev


def allreduce_counters(cnt):
    """Sum an int64 counter tensor over ranks in place (no-op single-process)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(cnt, op=dist.ReduceOp.SUM)
    return cnt


def _gpu_counts(det, batch, cnt):
    """Default per-rank detector: the fused GPU kernel accumulating into the
    device counter row `cnt` (no host sync)."""
    from .detect import detect
    H = batch.get("H_est", batch.get("H"))
    detect(det, H, batch["y"], float(batch["sigma_n2"]), batch["bits"], counters=cnt)


def sharded_detect(det, H, y, sigma2, tx_bits, *, counts_fn=None, device=None) -> dict:
    """Detect this rank's shard of a full batch and return the GLOBAL
    counters (bit_errors, symbol_errors, diverged, breakdown, trials, ...)."""
    import torch
    rank, world, _ = dist_info()
    T = len(H)
    lo, hi = shard_range(T, rank, world)
    batch = {"H": H[lo:hi], "H_est": H[lo:hi], "y": y[lo:hi], "bits": tx_bits[lo:hi], "sigma_n2": sigma2}
    dev = device or (torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu"))
    cnt = torch.zeros((_lib.NCOUNTERS,), dtype=torch.int64, device=dev)
    if hi > lo:
        (counts_fn or _gpu_counts)(det, batch, cnt)
    allreduce_counters(cnt)
    out = {k: int(v) for k, v in zip(_lib.COUNTERS, cnt.cpu().tolist())}
    _raise_on_nonpd(np.asarray([out[k] for k in _lib.COUNTERS]))
    return out


def _raise_on_nonpd(c) -> None:
    """build_blocks_batch raises ContractViolation on a non-PD diagonal block
    (solvers.py:246-249).  Callers that pass their own counter rows (every
    sharded path) see the 'nonpd' counter only here, after the all-reduce, so
    every rank raises together instead of counting frozen x = 0 lanes as
    ordinary bit errors."""
    c = np.asarray(c)
    nonpd = c[..., _lib.COUNTERS.index("nonpd")]
    if int(np.sum(nonpd)):
        raise ContractViolation(f"non-PD diagonal block in {int(np.sum(nonpd))} block(s)")


def wilson_interval(errors: int, n: int, z: float = 1.96) -> tuple[float, float]:
    """detect.py:177-186."""
    if n == 0:
        return 0.0, 1.0
    phat = errors / n
    denom = 1.0 + z * z / n
    center = (phat + z * z / (2 * n)) / denom
    half = z * math.sqrt(phat * (1 - phat) / n + z * z / (4 * n * n)) / denom
    return max(center - half, 0.0), min(center + half, 1.0)


@dataclass
class BERPoint:
    """detect.py:145-153."""
    snr_db: float
    trials: int
    bit_errors: int
    ber: float
    ci_low: float
    ci_high: float
    divergence_rate: float


@dataclass
class BERCurve:
    """detect.py:156-161."""
    detector: object
    zeta: float
    iters: int
    points: list = field(default_factory=list)


def sharded_ber_sweep(cfg, simulate, *, counts_fn=None, device=None) -> list:
    """run_ber_sweep (detect.py:240-270) with every chunk split over ranks.

    `cfg` is the reference's BERConfig (or anything with .channel.N,
    .channel.zeta_t, .detectors, .snr_grid, .trials, .chunk); `simulate(cfg,
    snr_idx, trial_ids) -> batch dict` is the reference's simulate_trials
    (its randomness depends only on the trial id, rng.py:19-39, so a rank can
    draw just its own slice).  `counts_fn(det, batch, cnt)` accumulates the
    8 counters of one detector on one batch into the int64 tensor row `cnt`
    (default: the fused GPU kernel).  Returns one BERCurve per detector,
    identical on every rank and equal to the single-process sweep."""
    import torch
    if cfg.trials < 1:
        raise ContractViolation("trials must be positive")
    rank, world, _ = dist_info()
    dev = device or (torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu"))
    counts_fn = counts_fn or _gpu_counts
    dets = list(cfg.detectors)
    curves = [BERCurve(detector=d, zeta=cfg.channel.zeta_t, iters=d.iters) for d in dets]
    bits_per_trial = 4 * cfg.channel.N
    for snr_idx in range(len(cfg.snr_grid)):
        cnt = torch.zeros((len(dets), _lib.NCOUNTERS), dtype=torch.int64, device=dev)
        done = 0
        while done < cfg.trials:
            n = min(cfg.chunk, cfg.trials - done)
            lo, hi = shard_range(n, rank, world)
            if hi > lo:
                batch = simulate(cfg, snr_idx, range(done + lo, done + hi))
                for di, det in enumerate(dets):
                    counts_fn(det, batch, cnt[di])
            done += n
        allreduce_counters(cnt)
        c = cnt.cpu().numpy()
        _raise_on_nonpd(c)
        be, dv = _lib.COUNTERS.index("bit_errors"), _lib.COUNTERS.index("diverged")
        total_bits = cfg.trials * bits_per_trial
        for di, curve in enumerate(curves):
            errs = int(c[di, be])
            lo_ci, hi_ci = wilson_interval(errs, total_bits)
            # NumPy scalars like the reference's (detect.py:264-268), so the
            # artefact writer formats them identically
            curve.points.append(BERPoint(snr_db=float(cfg.snr_grid[snr_idx]), trials=cfg.trials, bit_errors=errs,
                                         ber=np.int64(errs) / total_bits, ci_low=lo_ci, ci_high=hi_ci,
                                         divergence_rate=np.int64(c[di, dv]) / cfg.trials))
    return curves


def counters_from_arrays(rx_bits, tx_bits, diverged, breakdown, bits_per_symbol: int = 4) -> np.ndarray:
    """Host helper for custom `counts_fn`s: the counter row the fused kernel
    produces (bit errors, symbol errors, diverged, breakdown, trials)."""
    rx = np.asarray(rx_bits)
    tx = np.asarray(tx_bits)
    T = rx.shape[0]
    out = np.zeros(_lib.NCOUNTERS, np.int64)
    diff = rx != tx
    out[_lib.COUNTERS.index("bit_errors")] = int(diff.sum())
    sym = diff.reshape(T, diff.shape[-1] // bits_per_symbol, bits_per_symbol)
    out[_lib.COUNTERS.index("symbol_errors")] = int(sym.any(-1).sum())
    out[_lib.COUNTERS.index("diverged")] = int((np.asarray(diverged) >= 0).sum())
    out[_lib.COUNTERS.index("breakdown")] = int((np.asarray(breakdown) >= 0).sum())
    out[_lib.COUNTERS.index("trials")] = T
    return out
