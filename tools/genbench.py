#!/usr/bin/env python
"""Input-generation and LMMSE throughput (dev tool): fpm_gen_trials draws
and the fused channel.simulate_batch kernel, per realization, c5 shape."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_09820_b200 import channel  # noqa: E402
from paper_2504_09820_b200.solvers import solve_direct_batch  # noqa: E402
from paper_2504_09820_b200.detect import gram_mf  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


M, N, T = 128, 64, 32768
ms = timed(lambda: channel.gen_trials(1, 0, 0, T, M, N))
print(f"fpm_gen_trials: {T / ms * 1e3 / 1e6:.2f} M realizations/s ({T * M * N * 16 * 2 / (ms / 1e3) / 1e9:.0f} GB/s written)")
ms = timed(lambda: channel.simulate_batch(M, N, 0.5, 0.5, 15.0, 0, T, 1))
print(f"simulate_batch (fpm_simulate: draws + AR(1) colouring + QAM + y, one kernel): {T / ms * 1e3 / 1e6:.2f} M "
      f"realizations/s ({T * (M * N * 16 + M * 16 + N * 16 + 4 * N) / (ms / 1e3) / 1e9:.0f} GB/s written)")
b = channel.simulate_batch(M, N, 0.5, 0.5, 15.0, 0, T, 1)
A, bb = gram_mf(b["H"], b["y"], b["sigma_n2"])
ms = timed(lambda: solve_direct_batch(A, bb))
print(f"fpm_lmmse (Cholesky solve, N={N}): {T / ms * 1e3 / 1e6:.2f} M systems/s")
