import sys, time, ctypes
import numpy as np
sys.path.insert(0, '.')
import paper_2110_14734_b200 as w1g
from paper_2110_14734_b200 import _lib, lower_bound, synth
from oracle import w1oracle as O
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
a, b = synth.gaussian_cluster_pair(n, n, seed=0)
n0 = w1g.zero_condense(a, b)
on = O.zero_condense(a, b)
ctx = _lib.context()
ref = {s: O.rwmd_best(on, s) for s in 'ab'}
for cull in (0, 1):
    ctx.call("w1g_set_rwmd_culling", cull)
    for side in 'ab':
        t0 = time.perf_counter(); got = lower_bound.rwmd_best(n0, side); t1 = time.perf_counter()
        bad = np.flatnonzero(got != ref[side])
        print(f"cull={cull} side={side} time={1e3*(t1-t0):.1f}ms mismatches={bad.size}", flush=True)
        if bad.size:
            print("  idx", bad[:5], "got", got[bad[:5]], "ref", ref[side][bad[:5]])
    ms = ctypes.c_float(); ev = ctypes.c_int64()
    ctx.call("w1g_profile_rwmd_tile", 2, ctypes.byref(ms), ctypes.byref(ev))
    print(f"cull={cull} tile kernel {ms.value:.3f} ms/launch evals={ev.value}", flush=True)
keys = np.random.default_rng(0).integers(0, 2**34, (1, 1750000), dtype=np.uint64)
perm = np.empty(keys.shape[1], np.uint32)
for _ in range(3):
    t0 = time.perf_counter(); ctx.call("w1g_debug_radix_sort", keys.ctypes.data, 1, keys.shape[1], perm.ctypes.data); t1 = time.perf_counter()
print(f"sort 1.75M x 34-bit: {1e3*(t1-t0):.2f} ms ok={np.array_equal(perm, np.argsort(keys[0], kind='stable'))}")
