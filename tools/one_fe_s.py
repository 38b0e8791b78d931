# one warm front end at (n, s, delta) with the stage timers (W1G_TIMING=1) and the row-length profile
import sys; sys.path.insert(0, '.')
import numpy as np
import paper_2110_14734_b200 as w1g
from paper_2110_14734_b200 import _lib, synth
from paper_2110_14734_b200.pipeline import _front_end
n = int(sys.argv[1]); s = float(sys.argv[2]); delta = float(sys.argv[3])
a, b = synth.gaussian_cluster_pair(n, n, seed=0)
p = w1g.ApproxParams(s=s, best_effort=True, delta=delta)
ctx = _lib.context()
_front_end(ctx, a, b, p)
info = _front_end(ctx, a, b, p)
print("total ms", info.stage_ms[7], "stages", [round(x, 3) for x in info.stage_ms[:7]])
net, _ = w1g.sparsify(a, b, p)
L = np.diff(net.row_offsets)
print("rows", len(L), "avg", L.mean(), "max", L.max(), "hist", [(t, int((L > t).sum())) for t in (16, 32, 256, 1024, 4096)])
