"""Phase times of distributed.sparsify_sharded at world size 1 (NCCL group of one):
where the sharded one-pair path spends its time on a single GPU."""
import os
import socket
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2110_14734_b200 as w1g  # noqa: E402
from paper_2110_14734_b200 import distributed as D, synth  # noqa: E402

s = socket.socket()
s.bind(("127.0.0.1", 0))
port = s.getsockname()[1]
s.close()
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
a, b = synth.gaussian_cluster_pair(n, n, seed=0)
params = w1g.ApproxParams(s=1.0, best_effort=True, delta=0.01)

# wrap the library calls the sharded path makes, timing each (device synchronised)
lib = w1g._lib
orig_call = lib.Context.call
acc = {}


def timed_call(self, name, *args):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = orig_call(self, name, *args)
    torch.cuda.synchronize()
    acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0
    return r


for rep in range(3):
    acc.clear()
    lib.Context.call = timed_call
    t0 = time.perf_counter()
    net, d = D.sparsify_sharded(a, b, params, 0, 1)
    torch.cuda.synchronize()
    total = time.perf_counter() - t0
    lib.Context.call = orig_call
    print(f"total {1e3 * total:.2f} ms; " + ", ".join(f"{k} {1e3 * v:.2f}" for k, v in sorted(acc.items(),
                                                                                       key=lambda kv: -kv[1])))
dist.destroy_process_group()
