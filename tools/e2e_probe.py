# e2e probe: sparsify (pinned inputs, network copied out inside the call) vs the
# device-timed front end (_front_end, pageable inputs, no copy-out) at one size
import sys, time; sys.path.insert(0, '.')
import numpy as np
import paper_2110_14734_b200 as w1g
from paper_2110_14734_b200 import _lib, synth
from paper_2110_14734_b200.pipeline import _front_end
n = int(sys.argv[1]); mode = sys.argv[2] if len(sys.argv) > 2 else "e2e"
a, b = synth.gaussian_cluster_pair(n, n, seed=0)
params = w1g.ApproxParams(s=1.0, best_effort=True, delta=0.01)
ap, bp = w1g.pinned_points(a), w1g.pinned_points(b)
ts, dev = [], []
for it in range(6):
    t0 = time.perf_counter()
    if mode == "e2e":
        net, d = w1g.sparsify(ap, bp, params); del net
        dev.append(d.stage_ms.get("total")); st = list(d.stage_ms.values())
    elif mode == "e2e_pageable":
        net, d = w1g.sparsify(a, b, params); del net
        dev.append(d.stage_ms.get("total"))
    else:
        info = _front_end(_lib.context(), ap if mode == "dev_pinned" else a, bp if mode == "dev_pinned" else b, params)
        dev.append(info.stage_ms[7]); st = list(info.stage_ms)
    ts.append(1e3 * (time.perf_counter() - t0))
print(mode, "wall ms", round(float(np.median(ts[1:])), 3), "dev total", round(float(np.median(dev[1:])), 3),
      "last stages", [round(x, 3) for x in st])
