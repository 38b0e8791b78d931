for ps in 1 2 4; do
  W1G_COOP_PER_SM=$ps python - <<'PY'
import sys, os; sys.path.insert(0, '.')
import paper_2110_14734_b200 as w1g
from paper_2110_14734_b200 import _lib, synth
from paper_2110_14734_b200.pipeline import _front_end
a, b = synth.gaussian_cluster_pair(100000, 100000, seed=0)
p = w1g.ApproxParams(s=1.0, best_effort=True, delta=0.01)
ctx = _lib.context()
rs = [_front_end(ctx, a, b, p) for _ in range(5)]
import numpy as np
print(os.environ['W1G_COOP_PER_SM'], 'tree', round(min(r.stage_ms[3] for r in rs),3), 'wspd', round(min(r.stage_ms[4] for r in rs),3), 'total', round(min(r.stage_ms[7] for r in rs),3), flush=True)
PY
done
