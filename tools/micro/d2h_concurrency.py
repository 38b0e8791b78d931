"""Aggregate D2H bandwidth of W concurrent streams, each copying one cfg2-sized network
(49 MB) into its own page-locked buffer, repeated R times; with and without a
concurrent compute kernel -- the situation of the batch executor's workers."""
import sys
import time

import torch

MB = 49_000_000
R = 8
srcs = [torch.empty(MB // 8, dtype=torch.int64, device="cuda") for _ in range(8)]
dsts = [torch.empty(MB // 8, dtype=torch.int64, pin_memory=True) for _ in range(8)]
streams = [torch.cuda.Stream() for _ in range(8)]
busy = torch.empty(1 << 28, dtype=torch.float32, device="cuda")


def run(w, compute):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if compute:
        with torch.cuda.stream(streams[7]):
            for _ in range(40):
                busy.mul_(1.0000001)
    for r in range(R):
        for i in range(w):
            with torch.cuda.stream(streams[i]):
                dsts[i].copy_(srcs[i], non_blocking=True)
    for i in range(w):
        streams[i].synchronize()
    el = time.perf_counter() - t0
    torch.cuda.synchronize()
    return w * R * MB / el / 1e9


for compute in (False, True):
    for w in (1, 2, 4, 6):
        best = max(run(w, compute) for _ in range(3))
        print(f"streams={w} compute={compute}: {best:.1f} GB/s", flush=True)
