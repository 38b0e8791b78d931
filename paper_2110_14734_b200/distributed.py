"""Multi-GPU plumbing (one process per GPU, torch.distributed for the plumbing).

Two workloads of the north star shard naturally:

* batched pairwise W1 (cfg4): the i<j pairs are dealt round-robin to ranks;
  every rank sparsifies its pairs on its own B200 and solves them with the
  reference's host simplex; the (i, j, W1) triples are all-gathered.  There
  is no collective on the data path.
* one huge pair (cfg3): the RWMD rows are sharded.  numpy's np.sum is a
  fixed pairwise tree (loops_utils.h.src), so each rank takes whole
  subtrees of that tree (`pairwise_plan`), computes their exact sums on its
  device (w1g_rwmd_range), and the G partial sums are all-gathered and
  recombined in tree order (`pairwise_combine`) -- bit-identical to the
  single-device value.  An all-reduce is not used: its summation order is
  implementation-defined.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .diagram import SuppliedNodes, load_nodes
from .pipeline import ApproxParams, approx_w1, pair_shard

LEAF = 128  # numpy PW_BLOCKSIZE: segments of <= 128 terms are not split


def _split(n: int) -> int:
    n2 = n // 2
    return n2 - n2 % 8


def pairwise_plan(n: int, pieces: int) -> list[tuple[int, int]]:
    """Subtrees [begin, end) of numpy's summation tree over n terms: the tree
    is cut ceil(log2(pieces)) levels below the root (segments of <= 128 terms
    are leaves and stay whole), leaves in order."""
    depth = max(0, int(np.ceil(np.log2(max(pieces, 1)))))
    out: list[tuple[int, int]] = []

    def rec(b: int, ln: int, d: int):
        if d == depth or ln <= LEAF:
            out.append((b, b + ln))
            return
        n2 = _split(ln)
        rec(b, n2, d + 1)
        rec(b + n2, ln - n2, d + 1)

    rec(0, n, 0)
    return out


def pairwise_combine(n: int, pieces: int, partials) -> float:
    """Recombine the per-subtree sums of `pairwise_plan(n, pieces)` in the
    tree's own order (left + right at every internal node)."""
    depth = max(0, int(np.ceil(np.log2(max(pieces, 1)))))
    it = iter(float(p) for p in partials)

    def rec(ln: int, d: int) -> float:
        if d == depth or ln <= LEAF:
            return next(it)
        n2 = _split(ln)
        left = rec(n2, d + 1)
        right = rec(ln - n2, d + 1)
        return left + right

    return rec(n, 0) if n > 0 else 0.0


def _all_gather_f64(values: np.ndarray, group=None, device=None) -> np.ndarray:
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", device if device is not None else torch.cuda.current_device()) \
        if backend == "nccl" else torch.device("cpu")
    t = torch.from_numpy(np.ascontiguousarray(values, dtype=np.float64)).to(dev)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t, group=group)
    return np.stack([o.cpu().numpy() for o in outs])


def _device_partial(nodes: SuppliedNodes, side: int, begin: int, end: int, device=None) -> float:
    ctx = _lib.context(device)
    load_nodes(ctx, _lib.NODES0, nodes)
    out = ctypes.c_double(0.0)
    nm = ctypes.c_int64(0)
    ctx.call("w1g_rwmd_range", side, int(begin), int(end), ctypes.byref(out), ctypes.byref(nm))
    return out.value


def rwmd_rows(nodes: SuppliedNodes, rank: int, world: int, group=None, device=None,
              partial_fn=None) -> tuple[float, float, float]:
    """Row-sharded RWMD (lower_bound.py:61-75) over `world` ranks -> (L, L_A, L_B),
    identical on every rank and bit-identical to the single-device value.
    `partial_fn(side, begin, end)` overrides the device computation (tests)."""
    fn = partial_fn or (lambda side, b, e: _device_partial(nodes, side, b, e, device))
    sides = []
    for side, mass in enumerate((nodes.a_mass, nodes.b_mass)):
        n = int(np.count_nonzero(np.asarray(mass) > 0))
        plan = pairwise_plan(n, world)
        mine = np.zeros(len(plan))
        for i, (b, e) in enumerate(plan):
            if i % world == rank:
                mine[i] = fn(side, b, e)
        gathered = _all_gather_f64(mine, group, device)
        partials = [gathered[i % world, i] for i in range(len(plan))]
        sides.append(pairwise_combine(n, world, partials))
    la, lb = sides
    return (lb if lb > la else la), la, lb


def pairwise_w1_ranks(diagrams, params: ApproxParams, rank: int, world: int, group=None,
                      device=None, compute=None) -> np.ndarray:
    """Batched W1 matrix with the pairs dealt round-robin over ranks (no data
    collective); the (i, j, W1) results are all-gathered so every rank returns
    the full symmetric matrix.  `compute(i, j)` overrides the device path."""
    import torch.distributed as dist

    n = len(diagrams)
    mine = pair_shard(n, rank, world)
    if compute is None:
        def compute(i, j):
            return approx_w1(diagrams[i], diagrams[j], params, device=device)[0]
    results = [(i, j, float(compute(i, j))) for i, j in mine]
    gathered = [None] * world
    dist.all_gather_object(gathered, results, group=group)
    out = np.zeros((n, n))
    for part in gathered:
        for i, j, v in part:
            out[i, j] = out[j, i] = v
    return out
