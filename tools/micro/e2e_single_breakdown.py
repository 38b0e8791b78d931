"""Where the single-pair end-to-end time goes: sparsify() wall time vs the device
makespan of its front end, and the cost of the Python wrapper around the C call.

    python tools/micro/e2e_single_breakdown.py [pageable]
"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2110_14734_b200 as w1g  # noqa: E402
from paper_2110_14734_b200 import _lib, synth  # noqa: E402
from paper_2110_14734_b200.pipeline import _front_end  # noqa: E402

a, b = synth.gaussian_cluster_pair(100_000, 100_000, seed=0)
if "pageable" not in sys.argv:
    a, b = w1g.pinned_points(a), w1g.pinned_points(b)
p = w1g.ApproxParams(s=1.0, best_effort=True, delta=0.01)
for _ in range(5):
    w1g.sparsify(a, b, p)
ts, dev = [], []
for _ in range(30):
    t = time.perf_counter()
    net, d = w1g.sparsify(a, b, p)
    ts.append(time.perf_counter() - t)
    dev.append(d.stage_ms["total"])
ctx = _lib.context()
tc = []
for _ in range(30):
    t = time.perf_counter()
    _front_end(ctx, a, b, p)
    tc.append(time.perf_counter() - t)
print({"sparsify_ms": round(1e3 * float(np.median(ts)), 3), "device_ms": round(float(np.median(dev)), 3),
       "front_end_call_no_copy_ms": round(1e3 * float(np.median(tc)), 3)})

# the Python pieces alone
import timeit  # noqa: E402

from paper_2110_14734_b200.pipeline import _diagnostics  # noqa: E402

ncap, mcap = ctx.net_hint
_info = _front_end(ctx, a, b, p)
specs = [((ncap,), np.int64), ((mcap,), np.int64), ((mcap,), np.int64), ((mcap,), np.float64), ((ncap + 1,), np.int64)]
pieces = {
    "points_of x2": lambda: (w1g.diagram.points_of(a), w1g.diagram.points_of(b)),
    "pinned_arrays": lambda: _lib.pinned_arrays(specs),
    "diagnostics": lambda: _diagnostics(_info),
    "context()": lambda: _lib.context(),
}
out = _lib.pinned_arrays(specs)
pieces["set_network_out"] = lambda: ctx.call("w1g_set_network_out", _lib.addr(out[0]), _lib.addr(out[1]),
                                             _lib.addr(out[2]), _lib.addr(out[3]), _lib.addr(out[4]), ncap, mcap)
for k, f in pieces.items():
    n = 2000
    print(k, round(1e6 * timeit.timeit(f, number=n) / n, 2), "us")
