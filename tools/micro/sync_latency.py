"""Host round-trip latency (a tiny kernel + stream synchronize; a kernel-written
page-locked flag) with the host link idle and while another stream keeps it busy with
49 MB D2H copies -- the cost of a front end's round trip in the end-to-end batch."""
import statistics
import sys
import threading
import time

import torch

x = torch.zeros(1, device="cuda")
s = torch.cuda.Stream()
src = torch.empty(49_000_000 // 8, dtype=torch.int64, device="cuda")
dst = torch.empty(49_000_000 // 8, dtype=torch.int64, pin_memory=True)
side = torch.cuda.Stream()


def rt(n=300):
    ts = []
    for _ in range(n):
        t = time.perf_counter()
        with torch.cuda.stream(s):
            x.add_(1)
        s.synchronize()
        ts.append(1e6 * (time.perf_counter() - t))
    ts.sort()
    return {"median_us": round(statistics.median(ts), 1), "p90_us": round(ts[int(0.9 * len(ts))], 1)}


print("idle", rt(), flush=True)
for chunk in (49_000_000, 4_000_000, 1_000_000):
    stop = threading.Event()

    def loop():
        ch = chunk // 8
        while not stop.is_set():
            with torch.cuda.stream(side):
                for _ in range(4):
                    for o in range(0, src.numel(), ch):
                        dst[o:o + ch].copy_(src[o:o + ch], non_blocking=True)
            side.synchronize()

    th = threading.Thread(target=loop)
    th.start()
    time.sleep(0.1)
    print("busy, copies of", chunk, rt(), flush=True)
    stop.set()
    th.join()
