"""Does a concurrent D2H stream slow the front ends?  The device-only cfg2 batch
(w1g_front_end_batch, 32 pairs, 4 child contexts) alone and while another stream
keeps the host link busy with 49 MB D2H copies (the e2e batch's situation)."""
import ctypes
import sys
import threading
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2110_14734_b200 import _lib, synth  # noqa: E402
from paper_2110_14734_b200.lower_bound import load_corpus  # noqa: E402

ctx = _lib.context(0)
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


src = torch.empty(49_000_000 // 8, dtype=torch.int64, device="cuda")
dst = torch.empty(49_000_000 // 8, dtype=torch.int64, pin_memory=True)
side = torch.cuda.Stream()
stop = threading.Event()


def d2h_loop():
    while not stop.is_set():
        with torch.cuda.stream(side):
            for _ in range(4):
                dst.copy_(src, non_blocking=True)
        side.synchronize()


for _ in range(3):
    batch()
alone = min(batch() for _ in range(5))
th = threading.Thread(target=d2h_loop)
th.start()
time.sleep(0.05)
busy = min(batch() for _ in range(5))
stop.set()
th.join()
print({"batch_ms_alone": alone, "batch_ms_with_d2h_stream": busy})
