"""k_refine per launch (CUDA events, w1g_profile_rwmd) and the RWMD value, for the
threads-per-source variant chosen by W1G_RF_TPQ (read once per process).

    W1G_RF_TPQ=4 python tools/micro/refine_tpq.py [N]
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, ".")
import paper_2110_14734_b200 as w1g  # noqa: E402
from paper_2110_14734_b200 import _lib, synth  # noqa: E402
from paper_2110_14734_b200.diagram import load_nodes  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
a, b = synth.gaussian_cluster_pair(n, n, seed=0)
ctx = _lib.context()
n0 = w1g.zero_condense(a, b)
load_nodes(ctx, _lib.NODES0, n0)
ms = (ctypes.c_float * 4)()
ev = (ctypes.c_int64 * 4)()
directed = ctypes.c_int64(0)
ctx.call("w1g_profile_rwmd", 1, ms, ev, ctypes.byref(directed))
ctx.call("w1g_profile_rwmd", 9, ms, ev, ctypes.byref(directed))
from paper_2110_14734_b200.lower_bound import rwmd_best, rwmd_sides  # noqa: E402
import hashlib  # noqa: E402
L = rwmd_sides(n0)
bh = hashlib.sha1(rwmd_best(n0, 'a').tobytes() + rwmd_best(n0, 'b').tobytes()).hexdigest()[:16]
print(json.dumps({"tpq": os.environ.get("W1G_RF_TPQ", "2"), "n": n, "ms": [round(x, 4) for x in ms],
                  "evals": list(ev), "L": [float(x).hex() for x in L], "best_sha": bh}))
