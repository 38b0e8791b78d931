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
    counts = [int(np.count_nonzero(np.asarray(m) > 0)) for m in (nodes.a_mass, nodes.b_mass)]
    return rwmd_rows_counts(counts, rank, world, fn, group, device)


def _dist_on() -> bool:
    """A torch.distributed process group is up (even of one rank: its collectives run)."""
    try:
        import torch.distributed as dist

        return dist.is_available() and dist.is_initialized()
    except ImportError:
        return False


class _DeviceArray:
    """A library device buffer seen by torch without a copy (__cuda_array_interface__)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (int(ptr or 0), False),
                                         "version": 3, "strides": None}


def gather_arcs(tails, heads, costs, rank: int, world: int, group=None):
    """Rank 0 receives every rank's arc slice: gather_slices of (tails, heads, costs)."""
    return gather_slices((tails, heads, costs), rank, world, group)


def gather_slices(arrays, rank: int, world: int, group=None):
    """Rank 0 receives every rank's slices of the equally long 1-D `arrays`
    (grouped point-to-point: one send per array per rank, posted together --
    NCCL groups them into one ncclGroupStart/End over NVLink).  Arguments and
    results are torch tensors on the rank's device (NCCL) or on the CPU (gloo).
    Returns the concatenations on rank 0 (slices in rank order), None elsewhere."""
    import torch
    import torch.distributed as dist

    tails = arrays[0]
    dev = tails.device
    m = torch.tensor([tails.shape[0]], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(m) for _ in range(world)]
    dist.all_gather(counts, m, group=group)
    counts = [int(c.item()) for c in counts]
    ops = []
    out = None
    if rank == 0:
        total = sum(counts)
        out = tuple(torch.empty(total, dtype=x.dtype, device=dev) for x in arrays)
        for o, x in zip(out, arrays):
            o[:counts[0]].copy_(x)
        off = counts[0]
        for r in range(1, world):
            if counts[r]:
                for buf in out:
                    ops.append(dist.P2POp(dist.irecv, buf[off:off + counts[r]], r, group))
            off += counts[r]
    elif counts[rank]:
        for t in arrays:
            ops.append(dist.P2POp(dist.isend, t.contiguous(), 0, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    return out


def sparsify_sharded(a, b, params: ApproxParams, rank: int, world: int, group=None, device=None):
    """The sparsify front end of ONE pair over `world` ranks:

    * zero_condense, delta_condense and the split tree are replicated on every
      rank (cheap, and their sorts are global);
    * RWMD rows are sharded along numpy's summation tree (rwmd_rows): the G
      partial sums are all-gathered (8 bytes each) and combined in tree order;
    * the WSPD owner loop (spanner.py:206-241) is sharded: rank r runs the
      recursions of the internal nodes w with w % world == r;
    * the arc list is gathered on rank 0 in its compact form -- the shards' node
      pairs, 8 bytes per pair instead of two 24-byte arcs (grouped send/recv over
      NCCL) -- and rank 0, which holds the same nodes and tree, emits the arcs
      fused into its CSR build (the front end's network builder).

    Rank 0 returns (network, diagnostics); the other ranks (None, diagnostics).
    The network is bit-identical to the single-GPU front end's: the CSR is a
    function of the arc set alone, and the shards partition the WSPD."""
    import torch

    from .diagram import points_of
    from .network import fetch_network
    from .condensation import compute_delta
    from .pipeline import ApproxDiagnostics, condensation_epsilon

    ctx = _lib.context(device)
    diag = ApproxDiagnostics()
    ap, bp = points_of(a), points_of(b)
    k0 = ctypes.c_int64(0)
    bal = ctypes.c_int32(0)
    ctx.call("w1g_zero_condense", _lib.f64p(ap), ap.shape[0], _lib.f64p(bp), bp.shape[0], ctypes.byref(k0),
             ctypes.byref(bal))
    if k0.value == 0 or bal.value:
        diag.short_circuit = True
        return None, diag
    # RWMD rows over the ranks, on the resident nodes0 (no reload per range)
    def partial(side, b_, e_):
        out = ctypes.c_double(0.0)
        nm = ctypes.c_int64(0)
        ctx.call("w1g_rwmd_range", side, int(b_), int(e_), ctypes.byref(out), ctypes.byref(nm))
        return out.value

    na_, nb_ = ctypes.c_int64(0), ctypes.c_int64(0)
    ctx.call("w1g_member_counts", ctypes.byref(na_), ctypes.byref(nb_))
    counts = [int(na_.value), int(nb_.value)]
    L, la, lb = rwmd_rows_counts(counts, rank, world, partial, group, device)
    eps = condensation_epsilon(params.s)
    d = 0.0
    fixed = getattr(params, "delta", None)
    if params.use_condensation and L > 0.0:
        d = compute_delta(eps, L, ap.shape[0] + bp.shape[0]) if fixed is None else float(fixed)
    k = float(getattr(params, "k", 0.99))
    kk = ctypes.c_int64(0)
    ctx.call("w1g_delta_condense", d, k * d, (1.0 - k) * d / 2.0,
             ctypes.c_uint64(int(params.seed) & 0xFFFFFFFFFFFFFFFF), ctypes.byref(kk))
    nn = ctypes.c_int64(0)
    depth = ctypes.c_int32(0)
    ctx.call("w1g_split_tree", _lib.NODES, ctypes.byref(nn), ctypes.byref(depth))
    P = ctypes.c_int64(0)
    ctx.call("w1g_wspd_shard", float(params.s), int(rank), int(world), ctypes.byref(P))
    diag.lower_bound, diag.delta, diag.epsilon_condense = L, d, eps
    diag.n_pairs = int(P.value)
    gathered = None
    if _dist_on():
        # the shard's node pairs (int2, 8 bytes each) travel, not its arcs (two 24-byte arcs
        # per pair): every rank holds the same tree, so rank 0 emits the arcs itself, fused
        # into its CSR build
        up = ctypes.c_void_p()
        ctx.call("w1g_pairs_device", ctypes.byref(up), ctypes.byref(P))
        uv = torch.as_tensor(_DeviceArray(up.value, 2 * int(P.value), "<i4"), device=torch.device("cuda", ctx.device))
        gathered = gather_slices((uv,), rank, world, group)
    if rank != 0:
        return None, diag
    if gathered is not None:
        torch.cuda.synchronize(ctx.device)  # the received slices are complete before the library reads them
        (guv,) = gathered
        ctx.call("w1g_load_pairs_device", guv.data_ptr(), guv.shape[0] // 2)
    ncount, narcs = ctypes.c_int64(0), ctypes.c_int64(0)
    ctx.call("w1g_network_from_pairs", ctypes.byref(ncount), ctypes.byref(narcs))
    net = fetch_network(ctx, int(ncount.value), int(narcs.value))
    diag.n_nodes, diag.n_arcs = int(ncount.value), int(narcs.value)
    diag.n_pairs = int(guv.shape[0] // 2) if gathered is not None else diag.n_pairs
    return net, diag


def rwmd_rows_counts(counts, rank: int, world: int, partial_fn, group=None, device=None):
    """rwmd_rows given the per-side member counts and a partial_fn(side, begin, end):
    both sides' subtree sums of this rank travel in ONE all-gather."""
    plans = [pairwise_plan(n, world) for n in counts]
    mine = np.zeros(len(plans[0]) + len(plans[1]))
    for side, plan in enumerate(plans):
        base = 0 if side == 0 else len(plans[0])
        for i, (b_, e_) in enumerate(plan):
            if i % world == rank:
                mine[base + i] = partial_fn(side, b_, e_)
    gathered = _all_gather_f64(mine, group, device) if _dist_on() else mine[None, :]
    sides = []
    for side, (n, plan) in enumerate(zip(counts, plans)):
        base = 0 if side == 0 else len(plans[0])
        partials = [gathered[i % world, base + i] for i in range(len(plan))]
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
