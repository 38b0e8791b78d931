import faulthandler, sys, time
sys.path.insert(0, ".")
faulthandler.dump_traceback_later(90, exit=True)
import paper_2110_14734_b200 as w1g
from paper_2110_14734_b200 import synth
diags = []
for p in range(2):
    a, b = synth.gaussian_cluster_pair(100_000, 100_000, seed=p)
    diags += [a, b]
pairs = [(2 * (p % 2), 2 * (p % 2) + 1) for p in range(16)]
params = w1g.ApproxParams(s=1.0, best_effort=True, delta=0.01)
for st in (4, 4, 6, 6, 2):
    t = time.perf_counter()
    n = w1g.sparsify_batch(diags, params, pairs=pairs, streams_per_device=st, on_network=lambda i, j, net, d: None)
    print(st, n, round(time.perf_counter() - t, 3), flush=True)
