"""Where a worker's time goes in the end-to-end batch: sparsify_batch over 64 cfg2
pairs (4 distinct, repeated) with W1G_BATCH_TRACE=1 (per-worker block wait, front
end and hand-off time), pageable and page-locked inputs.

    W1G_BATCH_TRACE=1 python tools/micro/e2e_trace.py
"""
import sys
import time

sys.path.insert(0, ".")
import paper_2110_14734_b200 as w1g  # noqa: E402
from paper_2110_14734_b200 import synth  # noqa: E402

D, P = 4, 64
diags = []
for p in range(D):
    a, b = synth.gaussian_cluster_pair(100_000, 100_000, seed=p)
    diags += [a, b]
pairs = [(2 * (p % D), 2 * (p % D) + 1) for p in range(P)]
params = w1g.ApproxParams(s=1.0, best_effort=True, delta=0.01)
import numpy as np  # noqa: E402

for name, ds in (("pageable", diags), ("pinned", [w1g.pinned_points(d) for d in diags])):
    for rep in range(3):
        st = []
        t = time.perf_counter()
        w1g.sparsify_batch(ds, params, pairs=pairs, streams_per_device=4,
                           on_network=lambda i, j, n, d: st.append(d.stage_ms))
        print(name, rep, round(1e3 * (time.perf_counter() - t), 2), "ms", file=sys.stderr, flush=True)
    # per-stage device time (events on the front end's stream), median over the last batch
    print(name, "stage ms", {k: round(float(np.median([x[k] for x in st])), 3) for k in st[0]}, file=sys.stderr)

# the same front ends without delivering the networks: host inputs (each worker uploads
# its pair), networks left on the device -- the input side alone
import ctypes  # noqa: E402

from paper_2110_14734_b200 import _lib  # noqa: E402

ctx = _lib.context(0)
for name, ds in (("pageable", diags), ("pinned", [w1g.pinned_points(d) for d in diags])):
    ptrs = (ctypes.c_void_p * len(ds))(*[_lib.addr(p) for p in ds])
    sizes = np.array([p.shape[0] for p in ds], dtype=np.int64)
    ctx.call("w1g_corpus_set_host", ptrs, _lib.i64p(sizes), len(ds))
    pa = np.array(pairs, dtype=np.int32)
    infos = (_lib.FrontEndInfo * P)()
    for rep in range(3):
        ms = ctypes.c_float(0)
        t = time.perf_counter()
        _lib.check(ctx.lib.w1g_front_end_batch(ctx.handle, pa.ctypes.data, P, 1.0, 1, 1, 0.01, 0.99,
                                               ctypes.c_uint64(0), 4, infos, ctypes.byref(ms)))
        print("no-delivery", name, rep, round(1e3 * (time.perf_counter() - t), 2), "ms wall,", round(ms.value, 2),
              "ms device", file=sys.stderr, flush=True)
    print("no-delivery", name, "stage ms", {nm: round(float(np.median([infos[q].stage_ms[i] for q in range(P)])), 3)
                                            for i, nm in enumerate(_lib.STAGES)}, file=sys.stderr)
