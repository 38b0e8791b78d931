"""Large-input check against the C oracle (exercises the multi-kernel tree fallback
beyond the cooperative kernel's tile cap): python tools/big_check.py N"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np

import paper_2110_14734_b200 as w1g
from oracle import w1oracle as O
from paper_2110_14734_b200 import synth

n = int(sys.argv[1])
a, b = synth.gaussian_cluster_pair(n, n, seed=5)
params = w1g.ApproxParams(s=1.0, best_effort=True, delta=0.01)
t0 = time.perf_counter()
net, diag = w1g.sparsify(a, b, params)
t1 = time.perf_counter()
fe = O.front_end(a, b, 1.0, delta=0.01)
t2 = time.perf_counter()
same = all(getattr(net, f).tobytes() == getattr(fe.network, f).tobytes()
           for f in ("supplies", "tails", "heads", "costs", "row_offsets"))
print({"n": n, "gpu_s": t1 - t0, "oracle_s": t2 - t1, "L": diag.lower_bound, "L_oracle": fe.lower_bound,
       "arcs": int(net.arc_count), "tree_depth": diag.tree_depth, "network_bit_exact": same,
       "stage_ms": diag.stage_ms})
