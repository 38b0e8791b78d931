"""Which way of moving networks to the host slows the concurrent front ends least?
The device-only cfg2 batch (w1g_front_end_batch, 32 pairs, 4 child contexts) alone,
next to a stream of 49 MB copy-engine D2H copies, next to the same bytes written by
SM stores into page-locked host memory (zero copy, tools/micro/zc_write.cu) with
8 / 32 CTAs, and next to copy-engine D2H in chunks (mode ce_<bytes>).  Reports the batch time
and the side stream's achieved GB/s.

    nvcc -O3 -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC \\
        tools/micro/zc_write.cu -o tools/micro/libzc_write.so
    python tools/micro/d2h_interference2.py
"""
import ctypes
import json
import sys
import threading
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2110_14734_b200 import _lib, synth  # noqa: E402
from paper_2110_14734_b200.lower_bound import load_corpus  # noqa: E402

ctx = _lib.context(0)
zc = ctypes.CDLL("tools/micro/libzc_write.so")
zc.zc_copy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p]
diags = []
P = 32
for p in range(P):
    a, b = synth.gaussian_cluster_pair(100_000, 100_000, seed=p)
    diags += [a, b]
load_corpus(diags, 0)
pairs = np.array([(2 * p, 2 * p + 1) for p in range(P)], dtype=np.int32)
infos = (_lib.FrontEndInfo * P)()


def batch():
    ms = ctypes.c_float(0)
    _lib.check(ctx.lib.w1g_front_end_batch(ctx.handle, pairs.ctypes.data, P, 1.0, 1, 1, 0.01, 0.99,
                                           ctypes.c_uint64(0), 4, infos, ctypes.byref(ms)))
    return ms.value


NB = 49_000_000
src = torch.empty(NB // 8, dtype=torch.int64, device="cuda")
dst = torch.empty(NB // 8, dtype=torch.int64, pin_memory=True)
side = torch.cuda.Stream()
side2 = torch.cuda.Stream()


def run(mode):
    stop = threading.Event()
    moved = [0]

    def loop():
        while not stop.is_set():
            with torch.cuda.stream(side):
                for _ in range(4):
                    if mode == "ce":
                        dst.copy_(src, non_blocking=True)
                    elif mode.startswith("ce2_"):  # chunks alternating over two streams
                        ch = int(mode[4:]) // 8
                        for k, o in enumerate(range(0, NB // 8, ch)):
                            with torch.cuda.stream(side2 if k & 1 else side):
                                dst[o:o + ch].copy_(src[o:o + ch], non_blocking=True)
                    elif mode.startswith("ce_"):
                        ch = int(mode[3:]) // 8
                        for o in range(0, NB // 8, ch):
                            dst[o:o + ch].copy_(src[o:o + ch], non_blocking=True)
                    else:
                        zc.zc_copy(dst.data_ptr(), src.data_ptr(), NB, int(mode[2:]), side.cuda_stream)
                    moved[0] += NB
            side.synchronize()
            side2.synchronize()

    th = threading.Thread(target=loop)
    t0 = time.perf_counter()
    th.start()
    time.sleep(0.05)
    busy = min(batch() for _ in range(5))
    stop.set()
    th.join()
    return {"mode": mode, "batch_ms": busy, "side_gbs": moved[0] / (time.perf_counter() - t0) / 1e9}


for _ in range(3):
    batch()
print(json.dumps({"mode": "alone", "batch_ms": min(batch() for _ in range(5))}), flush=True)
for mode in sys.argv[1].split(",") if len(sys.argv) > 1 else ("ce", "ce_4000000", "zc32"):
    print(json.dumps(run(mode)), flush=True)
