import sys; sys.path.insert(0, '.')
import paper_2110_14734_b200 as w1g
from paper_2110_14734_b200 import _lib, synth
from paper_2110_14734_b200.pipeline import _front_end
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
a, b = synth.gaussian_cluster_pair(n, n, seed=0)
p = w1g.ApproxParams(s=1.0, best_effort=True, delta=0.01)
ctx = _lib.context()
for _ in range(3):
    info = _front_end(ctx, a, b, p)
print("tree global levels", info.tree_depth, "wspd levels", info.n_levels_wspd, "stage ms", [round(x, 3) for x in info.stage_ms])
