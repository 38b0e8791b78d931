"""Is the batch executor bound by the host (kernel launches and round trips) or by
the device?  Device-only batches (w1g_front_end_batch) of 64 pairs at three sizes
and 1..8 child contexts: at 1k points the device work is negligible, so the pairs/s
there is the host's issue rate.

    python tools/launch_rate.py
"""
import ctypes
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2110_14734_b200 import _lib, synth  # noqa: E402
from paper_2110_14734_b200.lower_bound import load_corpus  # noqa: E402

ctx = _lib.context(0)
for n in (1000, 20000, 100000):
    diags = []
    P = 64 if n < 100000 else 32
    for p in range(P):
        a, b = synth.gaussian_cluster_pair(n, n, seed=p)
        diags += [a, b]
    load_corpus(diags, 0)
    pairs = np.array([(2 * p, 2 * p + 1) for p in range(P)], dtype=np.int32)
    infos = (_lib.FrontEndInfo * P)()
    for st in (1, 2, 4, 8):
        ms = ctypes.c_float(0)
        for rep in range(4):
            l0 = _lib.launch_count()
            t0 = time.perf_counter()
            _lib.check(ctx.lib.w1g_front_end_batch(ctx.handle, pairs.ctypes.data, P, 1.0, 1, 1, 0.01, 0.99,
                                                   ctypes.c_uint64(0), st, infos, ctypes.byref(ms)))
            wall = time.perf_counter() - t0
            launches = (_lib.launch_count() - l0) / P
        dev = float(np.median([infos[i].stage_ms[7] for i in range(P)]))
        print(json.dumps({"n": n, "streams": st, "pairs_per_s_device_makespan": P / (ms.value * 1e-3),
                          "pairs_per_s_wall": P / wall, "launches_per_pair": launches,
                          "median_single_front_end_ms": dev}), flush=True)
