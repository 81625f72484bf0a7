"""Multi-process sharding (paper_2504_09820_b200/parallel.py) on CPU with the
gloo backend, world_size 2.  The per-rank detector here is the oracle (test
infrastructure); on GPUs the same host logic drives the fused kernel and the
counters are all-reduced over NCCL."""

import os
import socket
import tempfile
from types import SimpleNamespace

import numpy as np
import pytest

import fpm_oracle as O
from paper_2504_09820_b200 import parallel as P
from paper_2504_09820_b200.detect import DetectorSpec

FMT = {"fp64": O.FP64, "fp32": O.FP32, "fp16": O.FP16, "bfloat16": O.BF16}
M, N = 16, 8


def _cfg(trials=23, chunk=10):
    dets = (DetectorSpec("fp_cg", iters=4, matvec="fp16", inner="fp16"),
            DetectorSpec("fp_bj_cg", iters=4, L=2, matvec="fp16", inner="fp16"),
            DetectorSpec("cg", iters=3))
    return SimpleNamespace(channel=SimpleNamespace(M=M, N=N, zeta_r=0.5, zeta_t=0.5), detectors=dets,
                           snr_grid=(0.0, 8.0), trials=trials, chunk=chunk, seed=11)


def _simulate(cfg, snr_idx, ids):
    H, y, bits, s2 = O.simulate(M, N, 0.5, cfg.snr_grid[snr_idx], ids, cfg.seed, point=snr_idx)
    return {"H": H, "H_est": H, "y": y, "bits": bits, "sigma_n2": s2}


def _oracle_counts(det, batch, cnt):
    import torch
    mv = FMT.get(det.matvec, O.FP64)
    ip = FMT.get(det.inner, O.FP64)
    _, _, _, out = O.detect(batch["H_est"], batch["y"], batch["sigma_n2"], det.algorithm, det.iters, det.L,
                            O.FP64, mv, ip)
    row = P.counters_from_arrays(O.demod16(out.x), batch["bits"], out.diverged_at, out.breakdown_at)
    cnt += torch.from_numpy(row)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir, trials, chunk):
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        cfg = _cfg(trials, chunk)
        curves = P.sharded_ber_sweep(cfg, _simulate, counts_fn=_oracle_counts, device=torch.device("cpu"))
        res = [[(p.bit_errors, p.divergence_rate, p.ci_low, p.ci_high) for p in c.points] for c in curves]
        # one more collective: sum of ranks through the counter path
        c = torch.full((8,), rank + 1, dtype=torch.int64)
        P.allreduce_counters(c)
        H, y, bits, s2 = O.simulate(M, N, 0.5, 4.0, range(9), 3)
        glob = P.sharded_detect(cfg.detectors[1], H, y, s2, bits, counts_fn=_oracle_counts,
                                device=torch.device("cpu"))
        np.save(os.path.join(out_dir, f"r{rank}.npy"),
                np.array([res, c.tolist(), glob], dtype=object), allow_pickle=True)
    finally:
        dist.destroy_process_group()


def _run_world(world, trials, chunk):
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(world, _free_port(), d, trials, chunk), nprocs=world, join=True,
                           start_method="spawn")
        return [np.load(os.path.join(d, f"r{r}.npy"), allow_pickle=True) for r in range(world)]


def test_shard_range_partitions():
    for T in (0, 1, 7, 64, 1000, 1 << 20):
        for world in (1, 2, 3, 8):
            spans = [P.shard_range(T, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == T
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def test_shard_range_rejects_bad_args():
    with pytest.raises(Exception):
        P.shard_range(10, 2, 2)
    with pytest.raises(Exception):
        P.shard_range(10, 0, 0)


def test_wilson_matches_reference_formula():
    lo, hi = P.wilson_interval(0, 100)
    assert lo == 0.0 and 0.03 < hi < 0.04
    assert P.wilson_interval(0, 0) == (0.0, 1.0)


def test_single_process_sweep_equals_direct_oracle():
    import torch
    cfg = _cfg()
    curves = P.sharded_ber_sweep(cfg, _simulate, counts_fn=_oracle_counts, device=torch.device("cpu"))
    for si, snr in enumerate(cfg.snr_grid):
        b = _simulate(cfg, si, range(cfg.trials))
        for di, det in enumerate(cfg.detectors):
            cnt = torch.zeros(8, dtype=torch.int64)
            _oracle_counts(det, b, cnt)
            assert curves[di].points[si].bit_errors == int(cnt[0])
            assert curves[di].points[si].divergence_rate == int(cnt[2]) / cfg.trials


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_sweep_equals_single_process(world):
    """SURVEY.md 8(e) invariance: the sharded sweep's counts equal the
    single-process sweep's at every world size (ragged chunks included)."""
    import torch
    trials, chunk = 23, 10   # ragged: chunks of 10, 10, 3
    outs = _run_world(world, trials, chunk)
    single = P.sharded_ber_sweep(_cfg(trials, chunk), _simulate, counts_fn=_oracle_counts,
                                 device=torch.device("cpu"))
    ref = [[(p.bit_errors, p.divergence_rate, p.ci_low, p.ci_high) for p in c.points] for c in single]
    for o in outs:
        assert o[0] == ref                      # every rank holds the global result
        assert o[1] == [world * (world + 1) // 2] * 8   # sum of rank + 1 over ranks
    assert outs[0][2] == outs[1][2]
    assert outs[0][2]["trials"] == 9


def test_gloo_world2_chunk_smaller_than_world():
    import torch
    outs = _run_world(2, 5, 1)                  # every chunk has one trial: rank 1 idles
    single = P.sharded_ber_sweep(_cfg(5, 1), _simulate, counts_fn=_oracle_counts, device=torch.device("cpu"))
    ref = [[(p.bit_errors, p.divergence_rate, p.ci_low, p.ci_high) for p in c.points] for c in single]
    assert outs[0][0] == ref and outs[1][0] == ref


@pytest.mark.gpu
def test_gpu_sweep_counters_equal_oracle():
    """The default per-rank detector (fused kernel, device counters) gives the
    oracle's bit-error and divergence counts for every (SNR, detector)."""
    import torch
    cfg = _cfg(trials=40, chunk=16)
    gpu = P.sharded_ber_sweep(cfg, _simulate, device=torch.device("cuda"))
    ref = P.sharded_ber_sweep(cfg, _simulate, counts_fn=_oracle_counts, device=torch.device("cpu"))
    for cg, cr in zip(gpu, ref):
        for pg, pr in zip(cg.points, cr.points):
            assert (pg.bit_errors, pg.divergence_rate) == (pr.bit_errors, pr.divergence_rate)


@pytest.mark.gpu
def test_gpu_generated_sweep_is_chunk_invariant():
    """With the keyed per-trial generator (channel.simulate_trials) the sweep's
    counts do not depend on the chunking -- the property that makes them
    independent of the GPU count (each rank draws only its own trials)."""
    import torch
    from paper_2504_09820_b200 import channel
    cfg = _cfg(trials=48, chunk=16)
    cfg.context = 2
    a = P.sharded_ber_sweep(cfg, channel.simulate_trials, device=torch.device("cuda"))
    cfg2 = _cfg(trials=48, chunk=40)
    cfg2.context = 2
    b = P.sharded_ber_sweep(cfg2, channel.simulate_trials, device=torch.device("cuda"))
    for ca, cb in zip(a, b):
        for pa, pb in zip(ca.points, cb.points):
            assert (pa.bit_errors, pa.divergence_rate) == (pb.bit_errors, pb.divergence_rate)


def test_sharded_sweep_raises_on_nonpd_block():
    """A non-PD diagonal block surfaces as ContractViolation on the sharded
    path too (build_blocks_batch, solvers.py:246-249), not as bit errors of
    frozen lanes: the check runs on the all-reduced counters."""
    import torch
    from paper_2504_09820_b200 import _lib
    from paper_2504_09820_b200.errors import ContractViolation

    def bad_counts(det, batch, cnt):
        _oracle_counts(det, batch, cnt)
        if det.algorithm == "fp_bj_cg":
            cnt[_lib.COUNTERS.index("nonpd")] += 1

    with pytest.raises(ContractViolation):
        P.sharded_ber_sweep(_cfg(5, 5), _simulate, counts_fn=bad_counts, device=torch.device("cpu"))
    H, y, bits, s2 = O.simulate(M, N, 0.5, 4.0, range(3), 3)
    with pytest.raises(ContractViolation):
        P.sharded_detect(_cfg().detectors[1], H, y, s2, bits, counts_fn=bad_counts, device=torch.device("cpu"))
