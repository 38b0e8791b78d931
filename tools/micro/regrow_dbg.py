import os, sys
sys.path.insert(0, ".")
import numpy as np
import paper_2110_14734_b200 as w1g
from paper_2110_14734_b200 import synth
which = sys.argv[1]
a, b = synth.gaussian_cluster_pair(20_000, 20_000, seed=3)
params = w1g.ApproxParams(s=4.0, best_effort=True, delta=0.001)
ref, _ = w1g.sparsify(a, b, params)
nodes = w1g.zero_condense(a, b)
tree = w1g.build_split_tree(nodes.points)
ref_pairs = w1g.build_wspd(tree, 4.0)
os.environ["W1G_WSPD_TINY_CAPS"] = "1"
for r in range(5):
    if which == "fused":
        got, _ = w1g.sparsify(a, b, params)
        assert np.array_equal(got.heads, ref.heads)
    else:
        gp = w1g.build_wspd(tree, 4.0)
        assert np.array_equal(gp.node_pairs, ref_pairs.node_pairs)
print(which, "ok")
