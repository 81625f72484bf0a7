import sys, time, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import bench
from paper_2504_09820_b200.detect import DetectorSpec, detect_host
dev = torch.device("cuda", 0)
Te = 32768
H, y, bits = bench.gen_inputs(Te, 0, dev)
Hh = torch.empty((Te, bench.M, bench.N), dtype=torch.complex128, pin_memory=True); Hh.copy_(H)
yh = torch.empty((Te, bench.M), dtype=torch.complex128, pin_memory=True); yh.copy_(y)
bh = torch.empty((Te, 4 * bench.N), dtype=torch.uint8, pin_memory=True); bh.copy_(bits)
det = DetectorSpec("fp_bj_cg", iters=8, L=4, matvec="fp16", inner="fp16")
t = torch.empty(1 << 28, dtype=torch.uint8, pin_memory=True)
d = torch.empty(1 << 28, dtype=torch.uint8, device=dev)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(5): d.copy_(t, non_blocking=True)
torch.cuda.synchronize(); print("raw H2D GB/s", 5 * (1 << 28) / (time.perf_counter() - t0) / 1e9)
for chunk in (0, 1024, 2048, 8192, 16384):
    detect_host(det, Hh.numpy(), yh.numpy(), bench.SIGMA2, bh.numpy(), chunk=chunk)
    t0 = time.perf_counter()
    for _ in range(3): detect_host(det, Hh.numpy(), yh.numpy(), bench.SIGMA2, bh.numpy(), chunk=chunk)
    el = time.perf_counter() - t0
    print("chunk", chunk, "det/s", 3 * Te / el, "GB/s", 3 * Te * 133376 / el / 1e9)
