import os, sys
sys.path.insert(0, '.')
import numpy as np
import paper_2110_14734_b200 as w1g
from paper_2110_14734_b200 import lower_bound, synth
from oracle import w1oracle as O
n = int(sys.argv[1])
a, b = synth.gaussian_cluster_pair(n, n, seed=0)
n0 = w1g.zero_condense(a, b)
on = O.zero_condense(a, b)
r = lower_bound.rwmd_best(n0, 'a')
best = O.rwmd_best(on, 'a')
pts = on.points[on.a_mass > 0]
diag = np.abs(pts[:, 1] - pts[:, 0]) / np.sqrt(2)
ratio = r / np.maximum(best, 1e-300)
print(n, "radius/best percentiles 50/90/99/99.9/max:", np.percentile(ratio, [50, 90, 99, 99.9, 100]).round(3))
print("best==diag fraction", np.mean(best == diag).round(4), "median best", np.median(best), "median r", np.median(r))
