import sys, time; sys.path.insert(0, '.')
import numpy as np
import paper_2110_14734_b200 as w1g
from paper_2110_14734_b200 import _lib, synth
from paper_2110_14734_b200.pipeline import _front_end, _diagnostics, points_of
from paper_2110_14734_b200.network import TransshipmentNetwork
a, b = synth.gaussian_cluster_pair(100000, 100000, seed=0)
p = w1g.ApproxParams(s=1.0, best_effort=True, delta=0.01)
ap, bp = w1g.pinned_points(a), w1g.pinned_points(b)
for _ in range(3): net, d = w1g.sparsify(ap, bp, p); del net
ctx = _lib.context()
T = {}
def t(k, t0): T.setdefault(k, []).append(1e6 * (time.perf_counter() - t0))
for _ in range(20):
    t00 = time.perf_counter()
    t0 = time.perf_counter(); a1, b1 = points_of(ap), points_of(bp); t("points_of", t0)
    t0 = time.perf_counter(); ctx = _lib.context(None); t("context", t0)
    ncap, mcap = ctx.net_hint
    t0 = time.perf_counter()
    out = _lib.pinned_arrays([((ncap,), np.int64), ((mcap,), np.int64), ((mcap,), np.int64), ((mcap,), np.float64), ((ncap + 1,), np.int64)])
    t("pinned_arrays", t0)
    t0 = time.perf_counter()
    ctx.call("w1g_set_network_out", _lib.addr(out[0]), _lib.addr(out[1]), _lib.addr(out[2]), _lib.addr(out[3]), _lib.addr(out[4]), ncap, mcap)
    t("set_out", t0)
    t0 = time.perf_counter(); info = _front_end(ctx, a1, b1, p); t("front_end_call", t0)
    t0 = time.perf_counter(); diag = _diagnostics(info); t("diagnostics", t0)
    n, m = int(info.node_count), int(info.n_arcs)
    t0 = time.perf_counter(); sup, tails, heads, costs, ro = out; net = TransshipmentNetwork(n, sup[:n], tails[:m], heads[:m], costs[:m], ro[:n + 1]); t("network", t0)
    t("total", t00)
    T.setdefault("dev_total_us", []).append(1e3 * info.stage_ms[7])
    del net, out, sup, tails, heads, costs, ro
for k, v in T.items(): print(f"{k:16s} median {np.median(v[2:]):9.1f} us")
