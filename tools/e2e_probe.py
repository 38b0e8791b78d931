"""Where the end-to-end batch time goes: sparsify_batch over the cfg2 batch with
pageable vs page-locked inputs, several stream counts, with and without keeping
the networks, against the device-only batch and the host link's D2H bound.

    python tools/e2e_probe.py [PAIRS] [STREAMS,..] [DISTINCT]
"""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2110_14734_b200 as w1g  # noqa: E402
from paper_2110_14734_b200 import synth  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 32
D = int(sys.argv[3]) if len(sys.argv) > 3 else P  # distinct pairs (generating them dominates the run)
diags = []
for p in range(D):
    a, b = synth.gaussian_cluster_pair(100_000, 100_000, seed=p)
    diags += [a, b]
pinned = [w1g.pinned_points(d) for d in diags]
pairs = [(2 * (p % D), 2 * (p % D) + 1) for p in range(P)]
params = w1g.ApproxParams(s=1.0, best_effort=True, delta=0.01)


def run(ds, streams, reps=3):
    nbytes = [0]

    def keep(i, j, net, d):
        nbytes[0] += sum(getattr(net, f).nbytes for f in ("supplies", "tails", "heads", "costs", "row_offsets"))

    w1g.sparsify_batch(ds, params, pairs=pairs, streams_per_device=streams, on_network=keep)
    ts = []
    for _ in range(reps):
        nbytes[0] = 0
        t0 = time.perf_counter()
        w1g.sparsify_batch(ds, params, pairs=pairs, streams_per_device=streams, on_network=keep)
        ts.append(time.perf_counter() - t0)
    t = min(ts)
    return {"streams": streams, "ms": 1e3 * t, "pairs_per_s": P / t, "d2h_gb": nbytes[0] / 1e9,
            "d2h_gbs_if_link_bound": nbytes[0] / t / 1e9}


streams = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2, 4, 6, 8]
for inputs, ds in (("pageable", diags), ("pinned", pinned)):
    for st in streams:
        print(json.dumps({"inputs": inputs, **run(ds, st)}), flush=True)
