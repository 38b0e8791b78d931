"""Device-only cfg2 batches (w1g_front_end_batch, 64 distinct pairs) at several child-context
counts: the batch `value` as a function of the streams per GPU (best of 4 repetitions).

    python tools/micro/batch_streams.py [STREAMS,..]
"""
import ctypes
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2110_14734_b200 import _lib, synth  # noqa: E402
from paper_2110_14734_b200.lower_bound import load_corpus  # noqa: E402

streams = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [4, 5, 6, 7, 8, 10]
ctx = _lib.context(0)
P = 64
diags = []
for p in range(P):
    a, b = synth.gaussian_cluster_pair(100_000, 100_000, seed=p)
    diags += [a, b]
load_corpus(diags, 0)
pairs = np.array([(2 * p, 2 * p + 1) for p in range(P)], dtype=np.int32)
infos = (_lib.FrontEndInfo * P)()
for st in streams:
    best = []
    for rep in range(5):
        ms = ctypes.c_float(0)
        _lib.check(ctx.lib.w1g_front_end_batch(ctx.handle, pairs.ctypes.data, P, 1.0, 1, 1, 0.01, 0.99,
                                               ctypes.c_uint64(0), st, infos, ctypes.byref(ms)))
        if rep:
            best.append(P / (ms.value * 1e-3))
    print(json.dumps({"streams": st, "pairs_per_s": round(max(best), 1), "median": round(float(np.median(best)), 1)}),
          flush=True)
