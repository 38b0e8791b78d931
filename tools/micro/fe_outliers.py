"""Repeat the cfg2 fused front end and report the stage breakdown of the slow calls
(tail latency: which stage a 3-4x outlier spends its time in).

    python tools/micro/fe_outliers.py [REPS]
"""
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2110_14734_b200 as w1g  # noqa: E402
from paper_2110_14734_b200 import _lib, synth  # noqa: E402
from paper_2110_14734_b200.pipeline import _front_end  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
a, b = synth.gaussian_cluster_pair(100_000, 100_000, seed=0)
p = w1g.ApproxParams(s=1.0, best_effort=True, delta=0.01)
ctx = _lib.context()
_front_end(ctx, a, b, p)
rows = []
for _ in range(reps):
    info = _front_end(ctx, a, b, p)
    rows.append({nm: round(float(info.stage_ms[i]), 4) for i, nm in enumerate(_lib.STAGES)})
tot = np.array([r["total"] for r in rows])
med = float(np.median(tot))
print(json.dumps({"reps": reps, "median": med, "p90": float(np.percentile(tot, 90)), "p99": float(np.percentile(tot, 99)),
                  "max": float(tot.max()), "n_over_2x": int((tot > 2 * med).sum())}))
med_stage = {k: float(np.median([r[k] for r in rows])) for k in rows[0]}
print(json.dumps({"median_stages": med_stage}))
for i in np.argsort(-tot)[:5]:
    print(json.dumps({"rank": int(i), **rows[i]}))
