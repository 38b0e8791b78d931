"""Dump the refine search radius (W1G_DEBUG_RADIUS=1) and the exact best of both RWMD sides
for offline candidate-count simulation: python tools/dump_radius.py N out.npz"""
import os
import sys

sys.path.insert(0, ".")
import numpy as np

import paper_2110_14734_b200 as w1g
from paper_2110_14734_b200 import lower_bound, synth

n = int(sys.argv[1])
a, b = synth.gaussian_cluster_pair(n, n, seed=0)
n0 = w1g.zero_condense(a, b)
out = {}
for s in "ab":
    out["r_" + s] = lower_bound.rwmd_best(n0, s)
np.savez(sys.argv[2], **out)
