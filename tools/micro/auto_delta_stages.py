"""Stage breakdown of the cfg2 front end with the reference's automatic delta (delta=None:
delta from the RWMD bound, the sequential schedule) next to the fixed delta=0.01 run.

    python tools/micro/auto_delta_stages.py [REPS]
"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2110_14734_b200 as w1g  # noqa: E402
from paper_2110_14734_b200 import _lib, synth  # noqa: E402
from paper_2110_14734_b200.pipeline import _front_end  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 15
a, b = synth.gaussian_cluster_pair(100_000, 100_000, seed=0)
ctx = _lib.context()
for delta in (None, 0.01):
    p = w1g.ApproxParams(s=1.0, best_effort=True, delta=delta)
    _front_end(ctx, a, b, p)
    rows = []
    for _ in range(reps):
        info = _front_end(ctx, a, b, p)
        rows.append([float(info.stage_ms[i]) for i in range(len(_lib.STAGES))])
    med = np.median(np.array(rows), axis=0)
    print(f"delta={delta} (used {info.delta:.6g}):", {nm: round(float(med[i]), 4) for i, nm in enumerate(_lib.STAGES)})
