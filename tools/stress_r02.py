"""Repetition stress of the concurrent kernels (the depth-first WSPD's work queue and
termination, the batch executor's workers / expanders / pool): many front ends at
several sizes and batches of pairs, every result compared with the first one.

    python tools/stress_r02.py [REPS]
"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2110_14734_b200 as w1g  # noqa: E402
from paper_2110_14734_b200 import synth  # noqa: E402

REPS = int(sys.argv[1]) if len(sys.argv) > 1 else 50
FIELDS = ("supplies", "tails", "heads", "costs", "row_offsets")
t0 = time.time()
for n, s, d in ((100000, 1.0, 0.01), (100000, 16.0, 0.001), (20000, 4.0, 0.001), (3000, 40.0, 0.0)):
    a, b = synth.gaussian_cluster_pair(n, n, seed=7)
    p = w1g.ApproxParams(s=s, best_effort=True, delta=d if d > 0 else None, use_condensation=d > 0)
    ref, _ = w1g.sparsify(a, b, p)
    for r in range(REPS if n < 100000 or s < 8 else max(3, REPS // 10)):
        net, _ = w1g.sparsify(a, b, p)
        for f in FIELDS:
            if not np.array_equal(getattr(net, f), getattr(ref, f)):
                raise SystemExit(f"MISMATCH n={n} s={s} rep={r} field={f}")
    print(f"n={n} s={s} delta={d}: ok", flush=True)
diags = synth.shared_centre_batch(24, 5000, seed=1)
params = w1g.ApproxParams(s=2.0, best_effort=True, delta=0.01)
first = {}
w1g.sparsify_batch(diags, params, streams_per_device=4, on_network=lambda i, j, net, d: first.__setitem__(
    (i, j), net.costs.copy()))
for r in range(max(3, REPS // 5)):
    got = {}
    w1g.sparsify_batch(diags, params, streams_per_device=4 + (r % 3),
                       on_network=lambda i, j, net, d: got.__setitem__((i, j), net.costs.copy()))
    assert sorted(got) == sorted(first)
    for k in got:
        if not np.array_equal(got[k], first[k]):
            raise SystemExit(f"BATCH MISMATCH rep={r} pair={k}")
print(f"batches ok; {time.time() - t0:.1f} s", flush=True)
