# one warm cfg2 front end for launch-list profiling (ncu -s skips the warm-up)
import sys; sys.path.insert(0, '.')
import paper_2110_14734_b200 as w1g
from paper_2110_14734_b200 import _lib, synth
from paper_2110_14734_b200.pipeline import _front_end
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
a, b = synth.gaussian_cluster_pair(n, n, seed=0)
p = w1g.ApproxParams(s=1.0, best_effort=True, delta=0.01)
ctx = _lib.context()
c0 = _lib.launch_count(); _front_end(ctx, a, b, p); c1 = _lib.launch_count()
info = _front_end(ctx, a, b, p)
print("launches per front end", c1 - c0, "total ms", info.stage_ms[7])
print("tree_depth", info.tree_depth, "wspd_levels", info.n_levels_wspd, "n_points", info.n_points, "pairs", info.n_pairs)
