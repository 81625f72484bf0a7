#!/usr/bin/env python
"""Pinned host -> device copy rate with 1 / 2 / 4 concurrent streams (dev tool)."""
import torch

n = 1 << 30
src = torch.empty(n, dtype=torch.uint8, pin_memory=True)
src.fill_(1)
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
for ns in (1, 2, 4):
    sts = [torch.cuda.Stream() for _ in range(ns)]
    part = n // ns
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k, s in enumerate(sts):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                for _ in range(4):
                    dst[k * part:(k + 1) * part].copy_(src[k * part:(k + 1) * part], non_blocking=True)
        for s in sts:
            e1.wait_stream(s) if hasattr(e1, "wait_stream") else torch.cuda.current_stream().wait_stream(s)
        torch.cuda.current_stream().wait_stream(sts[-1])
        for s in sts:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        e1.synchronize()
    print(f"{ns} streams: {4 * n / (e0.elapsed_time(e1) / 1e3) / 1e9:.2f} GB/s")
