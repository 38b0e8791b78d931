"""Top-level approximate W1 (reference: w1flow/pipeline.py:28-142).

`approx_w1` is the reference's entry point with the sparsify front end
(pipeline.py:105-130: zero_condense -> rwmd -> compute_delta ->
delta_condense -> build_split_tree -> build_wspd -> emit_arcs -> assemble)
fused into one device-resident call (w1g_front_end), followed by the
reference's own host network simplex.  Additions required by the north
star: an optional fixed `delta` in ApproxParams, `sparsify` (front end
only) and `pairwise_w1` (batched matrix, pairs sharded over devices).
"""

from __future__ import annotations

import ctypes
import math
import os
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

from . import _lib, solver
from .diagram import points_of
from .network import TransshipmentNetwork, fetch_network

GUARANTEE_MIN_S = 2.0


@dataclass(frozen=True)
class ApproxParams:
    """Knobs for one approximate distance computation (pipeline.py:28-50).

    `delta` (new): None derives the lattice pitch from the RWMD bound as the
    reference does (pipeline.py:116-122); a float fixes it.  `k` is the
    lattice fraction of CondensationParams (condensation.py:42)."""

    s: float
    use_condensation: bool = True
    seed: int = 0
    best_effort: bool = False
    block_size: int | None = None
    stop_c: float = 4.0
    stop_b: float = 1e5
    threads: int = 1
    delta: float | None = None
    k: float = 0.99

    def __post_init__(self):
        if self.s <= 0:
            raise ValueError("s must be positive")
        if self.s <= GUARANTEE_MIN_S and not self.best_effort:
            raise ValueError(
                "s <= 2 has no approximation guarantee; pass best_effort=True to acknowledge"
            )
        if self.threads < 1:
            raise ValueError("threads must be >= 1")
        if self.delta is not None and self.delta < 0:
            raise ValueError("delta must be nonnegative")
        if not (0.5 <= self.k < 1.0):
            raise ValueError("k must lie in [0.5, 1)")


@dataclass
class ApproxDiagnostics:
    """pipeline.py:53-64, plus device-side detail of the front end."""

    n_nodes: int = 0
    n_arcs: int = 0
    lower_bound: float = 0.0
    epsilon_condense: float = 0.0
    delta: float = 0.0
    node_drop_pct: float = 0.0
    pivots: int = 0
    blocks_searched: int = 0
    status: str = solver.OPTIMAL
    short_circuit: bool = False
    # additions
    n_pairs: int = 0
    tree_depth: int = 0
    stage_ms: dict = field(default_factory=dict)


def condensation_epsilon(s: float) -> float:
    """pipeline.py:67-69."""
    return 8.0 / (s - 4.0) if s >= 12 else 1.0


def total_error_factor(s: float) -> float:
    """pipeline.py:72-76."""
    if s <= 4:
        raise ValueError("the error expression requires s > 4")
    return (1.0 + 4.0 / s + 4.0 / (s - 2.0)) * (1.0 + 8.0 / (s - 4.0)) - 1.0


def s_from_error(eps_target: float) -> int:
    """pipeline.py:79-95."""
    if eps_target <= 0:
        raise ValueError("target error must be positive")
    lo = 12
    if total_error_factor(lo) <= eps_target:
        return lo
    hi = lo
    while total_error_factor(hi) > eps_target:
        hi *= 2
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if total_error_factor(mid) <= eps_target:
            hi = mid
        else:
            lo = mid
    return hi


def _front_end(ctx, ap: np.ndarray, bp: np.ndarray, params: ApproxParams) -> _lib.FrontEndInfo:
    info = _lib.FrontEndInfo()
    # the reference's own ApproxParams (no delta / k fields) works too
    delta = getattr(params, "delta", None)
    fixed = delta is not None
    ctx.call("w1g_front_end", _lib.f64p(ap), ap.shape[0], _lib.f64p(bp), bp.shape[0], float(params.s),
             1 if params.use_condensation else 0, 1 if fixed else 0,
             float(delta) if fixed else 0.0, float(getattr(params, "k", 0.99)),
             ctypes.c_uint64(int(params.seed) & 0xFFFFFFFFFFFFFFFF), ctypes.byref(info))
    return info


def _diagnostics(info: _lib.FrontEndInfo) -> ApproxDiagnostics:
    d = ApproxDiagnostics()
    if info.short_circuit:
        d.short_circuit = True
        return d
    d.lower_bound = info.lower_bound
    d.epsilon_condense = info.epsilon_condense
    d.delta = info.delta
    d.node_drop_pct = 100.0 * (1.0 - info.n_points / info.n_points0)
    d.n_nodes = int(info.node_count)
    d.n_arcs = int(info.n_arcs)
    d.n_pairs = int(info.n_pairs)
    d.tree_depth = int(info.tree_depth)
    d.stage_ms = {name: float(info.stage_ms[i]) for i, name in enumerate(_lib.STAGES)}
    return d


def sparsify(a, b, params: ApproxParams, device: int | None = None
             ) -> tuple[TransshipmentNetwork | None, ApproxDiagnostics]:
    """The sparsify front end alone (pipeline.py:105-130): the network that
    approx_w1 hands to the solver, or None when the distance short-circuits."""
    ap, bp = points_of(a), points_of(b)
    ctx = _lib.context(device)
    # arm a page-locked output block sized from the previous network of this
    # context: the front end then copies the network out inside the call,
    # overlapping the device work still running (the RWMD stream)
    out = None
    hint = getattr(ctx, "net_hint", None)
    if hint is not None:
        ncap, mcap = hint
        out = _lib.pinned_arrays([((ncap,), np.int64), ((mcap,), np.int64), ((mcap,), np.int64),
                                  ((mcap,), np.float64), ((ncap + 1,), np.int64)])
        ctx.call("w1g_set_network_out", _lib.addr(out[0]), _lib.addr(out[1]), _lib.addr(out[2]),
                 _lib.addr(out[3]), _lib.addr(out[4]), ncap, mcap)
    info = _front_end(ctx, ap, bp, params)
    diag = _diagnostics(info)
    if info.short_circuit:
        return None, diag
    n, m = int(info.node_count), int(info.n_arcs)
    ctx.net_hint = (n + n // 8 + 64, m + m // 8 + 1024)
    if info.network_copied:
        sup, tails, heads, costs, ro = out
        return TransshipmentNetwork(n, sup[:n], tails[:m], heads[:m], costs[:m], ro[:n + 1]), diag
    return fetch_network(ctx, n, m), diag


def solve_network(network: TransshipmentNetwork, params: ApproxParams, diag: ApproxDiagnostics) -> float:
    """Run the reference's host simplex on a device-built network (pipeline.py:133-142)."""
    result = solver.solve(network, block_size=params.block_size, stop_c=params.stop_c, stop_b=params.stop_b)
    diag.pivots = result.pivots
    diag.blocks_searched = result.blocks_searched
    diag.status = result.status
    return result.objective


def approx_w1(a, b, params: ApproxParams, device: int | None = None) -> tuple[float, ApproxDiagnostics]:
    """Approximate W1(a, b) with sparsity parameter params.s (pipeline.py:98-142)."""
    network, diag = sparsify(a, b, params, device)
    if network is None:
        return 0.0, diag
    return solve_network(network, params, diag), diag


def _devices(devices):
    if devices is None:
        n = _lib.device_count()
        return list(range(max(n, 1)))
    return list(devices)


def pair_shard(n_diagrams: int, rank: int, world: int) -> list[tuple[int, int]]:
    """Static round-robin of the unordered pairs i<j over `world` workers."""
    pairs = [(i, j) for i in range(n_diagrams) for j in range(i + 1, n_diagrams)]
    return pairs[rank::world]


def _device_pairs(pts, share, params, dev: int, streams: int, on_network) -> None:
    """One device's share of a pair list through the native batch executor
    (batch.cu): the diagrams are uploaded once, `streams` library worker threads
    run the front ends on child contexts, and this thread receives each network
    (zero-copy, page-locked) as it completes -- no Python in the per-pair loop
    on the device side."""
    from .network import TransshipmentNetwork

    if not share:
        return
    # the diagrams stay in host memory: each library worker uploads its own pair
    # inside its front end, overlapping the others (no up-front bulk copy)
    ctx = _lib.context(dev)
    ptrs = (ctypes.c_void_p * max(1, len(pts)))(*[_lib.addr(p) for p in pts])
    sizes = np.array([p.shape[0] for p in pts], dtype=np.int64)
    ctx.call("w1g_corpus_set_host", ptrs, _lib.i64p(sizes), len(pts))
    pairs = np.ascontiguousarray(np.asarray(share, dtype=np.int32).reshape(-1, 2))
    delta = getattr(params, "delta", None)
    ctx.call("w1g_batch_begin", pairs.ctypes.data, pairs.shape[0], float(params.s),
             1 if params.use_condensation else 0, 0 if delta is None else 1,
             0.0 if delta is None else float(delta), float(getattr(params, "k", 0.99)),
             ctypes.c_uint64(int(params.seed) & 0xFFFFFFFFFFFFFFFF), int(streams), 0)
    lib = ctx.lib
    try:
        r = _lib.BatchResult()
        while True:
            rc = lib.w1g_batch_next(ctx.handle, ctypes.byref(r))
            if rc == _lib.W1G_DONE:
                break
            _lib.check(rc)
            if r.status != _lib.W1G_OK:
                _lib.raise_code(r.status, r.message.decode(errors="replace"))
            diag = _diagnostics(r.info)
            net = None
            if not r.info.short_circuit:
                net = TransshipmentNetwork(int(r.info.node_count), *_lib.result_arrays(r))
            on_network(int(r.i), int(r.j), net, diag)
    finally:
        lib.w1g_batch_end(ctx.handle)


def _run_pairs(pts, todo, params: ApproxParams, devs, streams_per_device: int, on_network) -> None:
    """Front ends of `todo` pairs: round-robin over devices (one consumer thread
    and one context each, no collective), each device's share run by the native
    batch executor with `streams_per_device` concurrent child contexts.
    on_network(i, j, net, diag) runs in the device's consumer thread."""
    shards = [todo[d::len(devs)] for d in range(len(devs))]
    streams = max(1, streams_per_device)
    if len(devs) == 1:
        _device_pairs(pts, shards[0], params, devs[0], streams, on_network)
        return
    with ThreadPoolExecutor(max_workers=len(devs)) as wp:
        futs = [wp.submit(_device_pairs, pts, sh, params, d, streams, on_network) for d, sh in zip(devs, shards)]
        for f in futs:
            f.result()


def sparsify_batch(diagrams, params: ApproxParams, pairs: list[tuple[int, int]] | None = None, devices=None,
                   streams_per_device: int = 4, on_network=None) -> int:
    """The front end of every pair (i < j, or `pairs`) of a diagram batch, sharded
    over devices and streams; on_network(i, j, network | None, diag) receives each
    result (in a worker thread).  Returns the number of pairs processed."""
    pts = [points_of(d) for d in diagrams]
    n = len(pts)
    todo = pairs if pairs is not None else [(i, j) for i in range(n) for j in range(i + 1, n)]
    _run_pairs(pts, todo, params, _devices(devices), streams_per_device, on_network or (lambda *a: None))
    return len(todo)


def pairwise_w1(diagrams, params: ApproxParams, devices=None, solver_threads: int | None = None,
                pairs: list[tuple[int, int]] | None = None, streams_per_device: int = 4) -> np.ndarray:
    """Symmetric matrix of approx_w1(D[i], D[j]) for i < j, mirrored to (j, i).

    Pairs are sharded round-robin over `devices` x `streams_per_device` (one host
    thread and one context each, no collective); the networks go to a pool of
    `solver_threads` host threads running the reference solver (numba, GIL
    released).  `pairs` restricts the work to a subset (other entries NaN).
    """
    pts = [points_of(d) for d in diagrams]
    n = len(pts)
    devs = _devices(devices)
    todo = pairs if pairs is not None else [(i, j) for i in range(n) for j in range(i + 1, n)]
    out = np.full((n, n), np.nan)
    np.fill_diagonal(out, 0.0)
    if solver_threads is None:
        solver_threads = max(1, (os.cpu_count() or 1) - len(devs) * max(1, streams_per_device))
    pool = ThreadPoolExecutor(max_workers=solver_threads)
    futures = []
    lock = threading.Lock()
    # every queued network holds a page-locked result block until it is solved:
    # bound the networks in flight so fast front ends cannot pin host memory
    # without limit while the (much slower) host solver drains the queue
    in_flight = threading.BoundedSemaphore(2 * solver_threads + len(devs) * max(1, streams_per_device))

    def solve_one(net, diag):
        try:
            return solve_network(net, params, diag)
        finally:
            in_flight.release()

    def on_network(i, j, net, diag):
        if net is None:
            out[i, j] = out[j, i] = 0.0
            return
        in_flight.acquire()
        try:
            f = pool.submit(solve_one, net, diag)
        except BaseException:
            in_flight.release()
            raise
        with lock:
            futures.append((i, j, f))

    _run_pairs(pts, todo, params, devs, streams_per_device, on_network)
    for i, j, f in futures:
        out[i, j] = out[j, i] = f.result()
    pool.shutdown()
    return out


# ---------------------------------------------------------------- staged nearest-neighbour search

WCD_STAGE = "wcd"
RWMD_STAGE = "rwmd"
PDFLOW_STAGE = "pdflow"
EXACT_STAGE = "exact"
_STAGE_NAMES = (WCD_STAGE, RWMD_STAGE, PDFLOW_STAGE, EXACT_STAGE)


@dataclass(frozen=True)
class PipelineStage:
    """One filtering stage: a distance algorithm and its survivor count (pipeline.py:153-169)."""

    algorithm: str
    keep: int
    s: float | None = None

    def __post_init__(self):
        if self.algorithm not in _STAGE_NAMES:
            raise ValueError(f"unknown stage algorithm {self.algorithm!r}")
        if self.keep < 1:
            raise ValueError("stage must keep at least one candidate")
        if self.algorithm == PDFLOW_STAGE and (self.s is None or self.s <= 0):
            raise ValueError("pdflow stages need a positive sparsity parameter")


@dataclass(frozen=True)
class PipelineSpec:
    """Staged filtering plan with strictly decreasing survivor counts (pipeline.py:172-185)."""

    stages: tuple[PipelineStage, ...]

    def __post_init__(self):
        if not self.stages:
            raise ValueError("pipeline needs at least one stage")
        keeps = [st.keep for st in self.stages]
        if keeps[-1] != 1:
            raise ValueError("the final stage must keep exactly one candidate")
        if any(x <= y for x, y in zip(keeps, keeps[1:])):
            raise ValueError("survivor counts must be strictly decreasing")


@dataclass
class NNDiagnostics:
    stage_survivors: list[list[int]] = field(default_factory=list)
    stage_scores: list[dict[int, float]] = field(default_factory=list)


def _stage_scores(stage, ctx, query, corpus, survivors, seed: int, threads: int, device) -> list[float]:
    """One stage's scores for the surviving candidates (pipeline.py:191-207).

    wcd and rwmd score every survivor against the device-resident corpus in one
    library call; pdflow runs the GPU front end per candidate (pairs of the
    batch path, several streams) and the reference solver; exact builds the
    dense network on the GPU and solves it on the host."""
    from .exact import exact_w1_dense
    from .lower_bound import corpus_scores

    if stage.algorithm in (WCD_STAGE, RWMD_STAGE):
        return [float(v) for v in corpus_scores(ctx, stage.algorithm, query, survivors)]
    if stage.algorithm == EXACT_STAGE:
        def one(i):
            return exact_w1_dense(query, corpus[i], device=device)
    else:
        # an explicit s in the spec acknowledges best-effort values s <= 2
        params = ApproxParams(s=stage.s, seed=seed, best_effort=True, threads=1)

        def one(i):
            return approx_w1(query, corpus[i], params, device=device)[0]
    if threads > 1 and len(survivors) > 1:
        with ThreadPoolExecutor(max_workers=threads) as pool:
            return list(pool.map(one, survivors))
    return [one(i) for i in survivors]


def nn_search(query, corpus, spec: PipelineSpec, seed: int = 0, threads: int = 1,
              device: int | None = None) -> tuple[int, NNDiagnostics]:
    """Index of the corpus diagram the staged pipeline ranks nearest (pipeline.py:210-243).

    Each stage rescores the surviving candidates and keeps its `keep` best;
    ties break toward the lower corpus index.  The corpus is uploaded to the
    device once for all stages."""
    from .lower_bound import load_corpus

    if not corpus:
        raise ValueError("corpus must be nonempty")
    ctx = load_corpus(corpus, device)
    diag = NNDiagnostics()
    survivors = list(range(len(corpus)))
    for stage in spec.stages:
        scores = _stage_scores(stage, ctx, query, corpus, survivors, seed, threads, device)
        ranked = sorted(zip(scores, survivors), key=lambda t: (t[0], t[1]))
        diag.stage_scores.append({i: sc for sc, i in ranked})
        survivors = [i for _, i in ranked[: stage.keep]]
        diag.stage_survivors.append(list(survivors))
    return survivors[0], diag
