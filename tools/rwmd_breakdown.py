"""The RWMD stage alone (w1g_rwmd on a zero-condensed pair) at a size, with the
sub-stage timings of W1G_TIMING=1 on stderr: its preparation (member compaction,
Morton keys and sort) against the tile / refine / summation work that row
sharding divides (DESIGN.md section 8's estimate).

    W1G_TIMING=1 python tools/rwmd_breakdown.py N
"""
import sys
import time

sys.path.insert(0, ".")
import paper_2110_14734_b200 as w1g  # noqa: E402
from paper_2110_14734_b200 import lower_bound, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
a, b = synth.gaussian_cluster_pair(n, n, seed=0)
n0 = w1g.zero_condense(a, b)
for _ in range(3):
    t0 = time.perf_counter()
    L = lower_bound.rwmd_sides(n0)
    print(f"n={n}: L={L[0]!r} host {1e3 * (time.perf_counter() - t0):.2f} ms (incl. node upload)", flush=True)
