"""CSR transshipment network (reference: w1flow/network.py).

`build_network` / `assemble` run on the B200 (network.cu): validation in the
reference's order, radix sort of (tail, head), min-cost dedup, row offsets.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import NetworkError
from .diagram import SuppliedNodes, load_nodes
from .spanner import ArcList


@dataclass(frozen=True)
class TransshipmentNetwork:
    node_count: int
    supplies: np.ndarray  # (n,) int64
    tails: np.ndarray  # (m,) int64, sorted by (tail, head)
    heads: np.ndarray  # (m,) int64
    costs: np.ndarray  # (m,) float64
    row_offsets: np.ndarray  # (n + 1,) int64

    @property
    def arc_count(self) -> int:
        return self.tails.shape[0]

    def dump(self) -> str:
        """Debug text dump (network.py:35-41)."""
        lines = [f"{self.node_count} {self.arc_count}"]
        lines.append(" ".join(str(int(s)) for s in self.supplies))
        for t, h, c in zip(self.tails, self.heads, self.costs):
            lines.append(f"{int(t)} {int(h)} {float(c)!r}")
        return "\n".join(lines) + "\n"


def fetch_network(ctx, n: int, m: int) -> TransshipmentNetwork:
    # result arrays live in pooled page-locked memory: one full-speed D2H each,
    # no host-side copy (the block returns to the pool when the arrays die)
    sup, tails, heads, costs, ro = _lib.pinned_arrays(
        [((n,), np.int64), ((m,), np.int64), ((m,), np.int64), ((m,), np.float64), ((n + 1,), np.int64)])
    ctx.call("w1g_fetch_network", _lib.i64p(sup), _lib.i64p(tails), _lib.i64p(heads), _lib.f64p(costs),
             _lib.i64p(ro))
    return TransshipmentNetwork(n, sup, tails, heads, costs, ro)


def _load_arcs(ctx, tails, heads, costs):
    t, h = _lib.as_i64(tails), _lib.as_i64(heads)
    c = np.ascontiguousarray(costs, dtype=np.float64)
    if t.shape != h.shape or t.shape != c.shape:
        raise NetworkError("tail/head/cost arrays must have equal length")
    ctx.call("w1g_load_arcs", _lib.i64p(t), _lib.i64p(h), _lib.f64p(c), t.shape[0])


def build_network(supplies, tails, heads, costs, device: int | None = None) -> TransshipmentNetwork:
    """Validate, sort and deduplicate raw arc arrays into a CSR network (network.py:44-85)."""
    sup = _lib.as_i64(supplies).reshape(-1)
    n = sup.shape[0]
    if int(sup.sum()) != 0:
        raise NetworkError(f"unbalanced supplies (sum = {int(sup.sum())})")
    ctx = _lib.context(device)
    _load_arcs(ctx, tails, heads, costs)
    m = ctypes.c_int64(0)
    ctx.call("w1g_build_network", _lib.i64p(sup), n, ctypes.byref(m))
    return fetch_network(ctx, n, int(m.value))


def assemble(nodes: SuppliedNodes, arcs: ArcList, device: int | None = None) -> TransshipmentNetwork:
    """Network for supplied nodes plus the two virtual nodes (network.py:88-93)."""
    ctx = _lib.context(device)
    load_nodes(ctx, _lib.NODES, nodes)
    _load_arcs(ctx, arcs.tails, arcs.heads, arcs.costs)
    n = ctypes.c_int64(0)
    m = ctypes.c_int64(0)
    ctx.call("w1g_assemble", ctypes.byref(n), ctypes.byref(m))
    return fetch_network(ctx, int(n.value), int(m.value))
