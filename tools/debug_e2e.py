import sys, time, ctypes
import numpy as np
sys.path.insert(0, '.')
import paper_2110_14734_b200 as w1g
from paper_2110_14734_b200 import _lib, synth, pipeline, network
a, b = synth.gaussian_cluster_pair(100000, 100000, seed=0)
params = w1g.ApproxParams(s=1.0, best_effort=True, delta=0.01)
ctx = _lib.context()
T = time.perf_counter
for it in range(6):
    t0 = T(); info = pipeline._front_end(ctx, a, b, params); t1 = T()
    net = network.fetch_network(ctx, int(info.node_count), int(info.n_arcs)); t2 = T()
    print(f"front_end {1e3*(t1-t0):.2f} ms (device total {info.stage_ms[7]:.2f}) fetch {1e3*(t2-t1):.2f} ms")
# raw D2H bandwidth pinned vs pageable
import torch
x = torch.empty(47_000_000, dtype=torch.uint8, device='cuda')
hp = torch.empty(47_000_000, dtype=torch.uint8, pin_memory=True)
hn = torch.empty(47_000_000, dtype=torch.uint8)
for name, h in (("pinned", hp), ("pageable", hn)):
    for _ in range(3):
        torch.cuda.synchronize(); t0 = T(); h.copy_(x); torch.cuda.synchronize(); t1 = T()
    print(name, f"{47/(t1-t0)/1e3:.1f} GB/s")
