"""The FP32 all-pairs RWMD tile kernel in full brute-force mode, once per direction
(for ncu: sm__pipe_fma_cycles_active at n = 1M, BASELINE.json's north-star figure).

    python tools/brute_once.py N
"""
import ctypes
import sys

sys.path.insert(0, ".")
import paper_2110_14734_b200 as w1g  # noqa: E402
from paper_2110_14734_b200 import _lib, synth  # noqa: E402
from paper_2110_14734_b200.diagram import load_nodes  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
a, b = synth.gaussian_cluster_pair(n, n, seed=0)
ctx = _lib.context()
n0 = w1g.zero_condense(a, b)
load_nodes(ctx, _lib.NODES0, n0)
ctx.call("w1g_set_rwmd_culling", 0)
ms = ctypes.c_float(0)
ev = ctypes.c_int64(0)
ctx.call("w1g_profile_rwmd_tile", 1, ctypes.byref(ms), ctypes.byref(ev))
print(f"brute force n={n}: {ms.value:.3f} ms per launch, {ev.value} evaluations, "
      f"{5 * ev.value / (ms.value * 1e-3) / 1e12:.2f} TFLOP/s")
