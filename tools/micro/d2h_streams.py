import torch, time
n = 47_000_000 // 8
srcs = [torch.empty(n // 3, dtype=torch.int64, device="cuda") for _ in range(3)]
dsts = [torch.empty(n // 3, dtype=torch.int64, pin_memory=True) for _ in range(3)]
ss = [torch.cuda.Stream() for _ in range(3)]
def run(k):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for i in range(3):
        s = ss[i % k]
        with torch.cuda.stream(s):
            dsts[i].copy_(srcs[i], non_blocking=True)
    torch.cuda.synchronize(); return time.perf_counter() - t0
for k in (1, 3, 1, 3):
    ts = [run(k) for _ in range(10)]
    print(k, "streams", round(min(ts) * 1e3, 3), "ms", round(47e6 / min(ts) / 1e9, 1), "GB/s")
