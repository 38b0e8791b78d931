"""Relaxed-transport (RWMD) lower bound (reference: w1flow/lower_bound.py:43-75).

Runs on the B200: an FP32 all-pairs tile pass bounds every source's nearest
opposite-side node, an exact fp64 pass recomputes the reference's IEEE
distance inside that bound, and numpy's pairwise summation tree is evaluated
on device, so the value is bit-identical to the reference's.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .diagram import SuppliedNodes, load_nodes


def rwmd_sides(nodes: SuppliedNodes, device: int | None = None) -> tuple[float, float, float]:
    """(L, L_A, L_B) with L = max(L_A, L_B) (lower_bound.py:61-75)."""
    if nodes.points.shape[0] == 0:
        return 0.0, 0.0, 0.0
    ctx = _lib.context(device)
    load_nodes(ctx, _lib.NODES0, nodes)
    L, la, lb = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    ctx.call("w1g_rwmd", ctypes.byref(L), ctypes.byref(la), ctypes.byref(lb))
    return L.value, la.value, lb.value


def rwmd(nodes: SuppliedNodes, workers: int = 1) -> float:
    """Relaxed-transport lower bound on W1 for a condensed node set.

    `workers` is accepted for signature compatibility; the device decides
    its own parallelism and the result does not depend on it."""
    return rwmd_sides(nodes)[0]


def rwmd_best(nodes: SuppliedNodes, side: str = "a", device: int | None = None) -> np.ndarray:
    """Per-source min(nn distance, diagonal distance), sources in node order
    (the `best` vector of lower_bound.py:51-57), for kernel-level checks."""
    ctx = _lib.context(device)
    load_nodes(ctx, _lib.NODES0, nodes)
    L = ctypes.c_double()
    ctx.call("w1g_rwmd", ctypes.byref(L), None, None)
    s = 0 if side == "a" else 1
    n = ctypes.c_int64(0)
    ctx.call("w1g_fetch_rwmd_best", s, None, ctypes.byref(n))
    out = np.empty(int(n.value), dtype=np.float64)
    if out.size:
        ctx.call("w1g_fetch_rwmd_best", s, _lib.f64p(out), ctypes.byref(n))
    return out


def _corpus_arrays(diagrams) -> tuple[np.ndarray, np.ndarray]:
    """Points of a list of diagrams back to back plus row offsets (n + 1)."""
    from .diagram import points_of

    pts = [points_of(d) for d in diagrams]
    off = np.zeros(len(pts) + 1, dtype=np.int64)
    if pts:
        off[1:] = np.cumsum([p.shape[0] for p in pts])
    flat = np.ascontiguousarray(np.concatenate(pts, axis=0)) if pts else np.empty((0, 2))
    return flat.reshape(-1, 2), off


def load_corpus(diagrams, device: int | None = None):
    """Upload a diagram corpus to the device once (w1g_corpus_load); returns the context."""
    ctx = _lib.context(device)
    flat, off = _corpus_arrays(diagrams)
    ctx.call("w1g_corpus_load", _lib.f64p(flat), _lib.i64p(off), len(off) - 1)
    return ctx


def corpus_scores(ctx, kind: str, query, candidates) -> np.ndarray:
    """Scores of `query` against the loaded corpus' `candidates`: kind "wcd" (one
    launch for all of them, lower_bound.py:78-92) or "rwmd" (rwmd(zero_condense(
    query, candidate)), pipeline.py:202-203)."""
    from .diagram import points_of

    q = points_of(query)
    cand = np.ascontiguousarray(candidates, dtype=np.int64)
    out = np.empty(cand.shape[0], dtype=np.float64)
    if cand.shape[0]:
        ctx.call("w1g_wcd_corpus" if kind == "wcd" else "w1g_rwmd_corpus", _lib.f64p(q), q.shape[0],
                 _lib.i64p(cand), cand.shape[0], _lib.f64p(out))
    return out


def wcd(a, b, device: int | None = None) -> float:
    """Centroid-difference lower bound on W1 (lower_bound.py:78-92), on device:
    N * |mean(A u proj(B)) - mean(B u proj(A))| / 2 with numpy's summation order
    and glibc's hypot, bit for bit."""
    ctx = load_corpus([b], device)
    return float(corpus_scores(ctx, "wcd", a, [0])[0])
