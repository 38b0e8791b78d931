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
