"""What does host-link traffic do to a stream of small kernels?  87 back-to-back tiny
kernels (a front end's launch count) then one synchronize, and the same work captured
in a CUDA graph, with the link idle and while another stream keeps it busy with 49 MB
D2H copies."""
import statistics
import threading
import time

import torch

x = torch.zeros(1024, device="cuda")
s = torch.cuda.Stream()
src = torch.empty(49_000_000 // 8, dtype=torch.int64, device="cuda")
dst = torch.empty(49_000_000 // 8, dtype=torch.int64, pin_memory=True)
side = torch.cuda.Stream()
N = 87
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    for _ in range(3):
        x.add_(1)
    s.synchronize()
    with torch.cuda.graph(g, stream=s):
        for _ in range(N):
            x.add_(1)


def burst(graph):
    ts = []
    for _ in range(200):
        t = time.perf_counter()
        with torch.cuda.stream(s):
            if graph:
                g.replay()
            else:
                for _ in range(N):
                    x.add_(1)
        s.synchronize()
        ts.append(1e6 * (time.perf_counter() - t))
    return round(statistics.median(ts), 1)


print({"idle_launches_us": burst(False), "idle_graph_us": burst(True)}, flush=True)
stop = threading.Event()


def loop():
    while not stop.is_set():
        with torch.cuda.stream(side):
            for _ in range(4):
                dst.copy_(src, non_blocking=True)
        side.synchronize()


th = threading.Thread(target=loop)
th.start()
time.sleep(0.1)
print({"busy_launches_us": burst(False), "busy_graph_us": burst(True)}, flush=True)
stop.set()
th.join()
