"""The brute-force FP32 all-pairs tile kernel (culling off) at N + N points:
event-timed launch, evaluations and TFLOP/s (bench.py's north_star_kernel).

    python tools/micro/brute_tile.py [N]
"""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2110_14734_b200 as w1g  # noqa: E402
from paper_2110_14734_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
r = bench.north_star_kernel(_lib.context(), w1g, n)
print(json.dumps({k: r[k] for k in ("config", "achieved", "frac", "ms_per_launch", "evals_per_launch")}))
