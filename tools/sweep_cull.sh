for cs in 3 5 9 17 33; do
  W1G_CULL_STEPS=$cs python - <<'PY'
import sys, os; sys.path.insert(0, '.')
import paper_2110_14734_b200 as w1g
from paper_2110_14734_b200 import _lib, synth
from paper_2110_14734_b200.pipeline import _front_end
for n in (100000, 1000000):
    a, b = synth.gaussian_cluster_pair(n, n, seed=0)
    p = w1g.ApproxParams(s=1.0, best_effort=True, delta=0.01)
    ctx = _lib.context()
    r = [ _front_end(ctx, a, b, p).stage_ms[1] for _ in range(3) ]
    print(os.environ['W1G_CULL_STEPS'], n, 'rwmd_ms', round(min(r), 3), flush=True)
PY
done
