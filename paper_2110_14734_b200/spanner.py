"""Arc sparsification: split tree, WSPD, arcs (reference: w1flow/spanner.py).

All three stages run on the B200 (tree.cu, wspd.cu, network.cu).  The
dataclasses, node layout (points 0..k-1, abar = k, bbar = k+1) and error
behaviour mirror the reference.  `build_wspd` returns the pairs in the
reference's exact layout (owner node ascending, DFS pop order) so its arrays
compare equal to the reference's, not only as sets.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .diagram import SuppliedNodes, load_nodes

ABAR_OFFSET = 0
BBAR_OFFSET = 1


def abar_index(n_points: int) -> int:
    return n_points + ABAR_OFFSET


def bbar_index(n_points: int) -> int:
    return n_points + BBAR_OFFSET


@dataclass(frozen=True)
class SplitTree:
    """Array-backed split tree (spanner.py:37-64); children have larger ids."""

    points: np.ndarray  # (n, 2) float64
    left: np.ndarray  # (N,) int64
    right: np.ndarray  # (N,) int64
    bbox: np.ndarray  # (N, 4) float64: xmin, ymin, xmax, ymax
    rep: np.ndarray  # (N,) int64
    size: np.ndarray  # (N,) int64
    root: int  # -1 for an empty tree

    @property
    def n_nodes(self) -> int:
        return self.left.shape[0]

    def internal_nodes(self) -> np.ndarray:
        return np.flatnonzero(self.left >= 0)

    def leaf_count(self) -> int:
        return int(np.count_nonzero(self.left < 0))


@dataclass(frozen=True)
class WSPairList:
    """Well-separated pairs (spanner.py:67-81)."""

    node_pairs: np.ndarray  # (P, 2) int64 tree node ids
    indices: np.ndarray  # (P, 2) int64 representative point indices
    points: np.ndarray  # (n, 2)

    def __len__(self) -> int:
        return self.node_pairs.shape[0]


@dataclass(frozen=True)
class ArcList:
    """Directed arcs (tail, head, cost) over supplied-node indices (spanner.py:84-93)."""

    tails: np.ndarray
    heads: np.ndarray
    costs: np.ndarray

    def __len__(self) -> int:
        return self.tails.shape[0]


def _fetch_tree(ctx, pts: np.ndarray, nn: int) -> SplitTree:
    left = np.empty(nn, dtype=np.int64)
    right = np.empty(nn, dtype=np.int64)
    bbox = np.empty((nn, 4), dtype=np.float64)
    rep = np.empty(nn, dtype=np.int64)
    size = np.empty(nn, dtype=np.int64)
    if nn:
        ctx.call("w1g_fetch_tree", _lib.i64p(left), _lib.i64p(right), _lib.f64p(bbox), _lib.i64p(rep),
                 _lib.i64p(size))
    return SplitTree(pts, left, right, bbox, rep, size, 0 if nn else -1)


def build_split_tree(points, device: int | None = None) -> SplitTree:
    """Split tree of a set of distinct planar points (spanner.py:96-159), on device."""
    pts = _lib.as_points(points)
    n = pts.shape[0]
    if n == 0:
        e = np.empty(0, dtype=np.int64)
        return SplitTree(pts, e, e.copy(), np.empty((0, 4)), e.copy(), e.copy(), -1)
    ctx = _lib.context(device)
    z = np.zeros(n, dtype=np.int64)
    load_nodes(ctx, _lib.NODES, SuppliedNodes(pts, z, z, 0, 0))
    nn = ctypes.c_int64(0)
    depth = ctypes.c_int32(0)
    ctx.call("w1g_split_tree", _lib.NODES, ctypes.byref(nn), ctypes.byref(depth))
    return _fetch_tree(ctx, pts, int(nn.value))


def well_separated(box_u: np.ndarray, box_v: np.ndarray, s: float) -> bool:
    """Scalar separation predicate with np.hypot (spanner.py:162-173); a test
    helper in the reference, not on the device path."""
    ru = 0.5 * np.hypot(box_u[2] - box_u[0], box_u[3] - box_u[1])
    rv = 0.5 * np.hypot(box_v[2] - box_v[0], box_v[3] - box_v[1])
    r = max(ru, rv)
    dx = 0.5 * (box_u[0] + box_u[2]) - 0.5 * (box_v[0] + box_v[2])
    dy = 0.5 * (box_u[1] + box_u[3]) - 0.5 * (box_v[1] + box_v[3])
    return bool(np.hypot(dx, dy) - 2.0 * r >= s * r)


def _load_tree(ctx, tree: SplitTree) -> None:
    pts = _lib.as_points(tree.points)
    left = _lib.as_i64(tree.left)
    right = _lib.as_i64(tree.right)
    bbox = np.ascontiguousarray(tree.bbox, dtype=np.float64).reshape(-1, 4)
    rep = _lib.as_i64(tree.rep)
    ctx.call("w1g_load_tree", _lib.f64p(pts), pts.shape[0], _lib.i64p(left), _lib.i64p(right),
             _lib.f64p(bbox), _lib.i64p(rep), left.shape[0])


def _run_wspd(tree: SplitTree, s: float, device: int | None):
    ctx = _lib.context(device)
    _load_tree(ctx, tree)
    P = ctypes.c_int64(0)
    ctx.call("w1g_wspd", float(s), 1, ctypes.byref(P))
    return ctx, int(P.value)


def _counts(ctx) -> np.ndarray:
    ni = ctypes.c_int64(0)
    ctx.call("w1g_fetch_pair_counts", None, ctypes.byref(ni))
    out = np.empty(int(ni.value), dtype=np.int64)
    if out.size:
        ctx.call("w1g_fetch_pair_counts", _lib.i64p(out), ctypes.byref(ni))
    return out


def count_pairs(tree: SplitTree, s: float, workers: int = 1, device: int | None = None) -> np.ndarray:
    """WS pair count of the recursion rooted at each internal node (spanner.py:263-271)."""
    if s <= 0:
        raise ValueError("s must be positive")
    if tree.n_nodes < 2:
        return np.zeros(0, dtype=np.int64)
    ctx, _ = _run_wspd(tree, s, device)
    return _counts(ctx)


def _fetch_pairs(ctx, P: int, points) -> WSPairList:
    node_pairs = np.empty((P, 2), dtype=np.int64)
    indices = np.empty((P, 2), dtype=np.int64)
    if P:
        ctx.call("w1g_fetch_pairs", _lib.i64p(node_pairs), _lib.i64p(indices))
    return WSPairList(node_pairs, indices, points)


def write_pairs(tree: SplitTree, s: float, offsets: np.ndarray, counts: np.ndarray, workers: int = 1,
                device: int | None = None) -> WSPairList:
    """Pairs laid out in the ranges of the exclusive prefix sum of `counts`
    (spanner.py:274-297), with the reference's argument checks."""
    internal = tree.internal_nodes()
    if offsets.shape[0] != internal.shape[0] or counts.shape[0] != internal.shape[0]:
        raise AssertionError("offsets/counts do not match the internal node count")
    expected = np.concatenate([[0], np.cumsum(counts)])[:-1].astype(np.int64)
    if not np.array_equal(np.asarray(offsets, dtype=np.int64), expected):
        raise AssertionError("offsets are not the exclusive prefix sum of counts")
    if internal.shape[0] == 0:
        return WSPairList(np.empty((0, 2), np.int64), np.empty((0, 2), np.int64), tree.points)
    ctx, P = _run_wspd(tree, s, device)
    if not np.array_equal(_counts(ctx), np.asarray(counts, dtype=np.int64)):
        raise AssertionError("WSPD write pass disagrees with counted offsets")
    return _fetch_pairs(ctx, P, tree.points)


def build_wspd(tree: SplitTree, s: float, workers: int = 1, device: int | None = None) -> WSPairList:
    """WSPD of a split tree (spanner.py:303-307), reference pair order."""
    if s <= 0:
        raise ValueError("s must be positive")
    if tree.n_nodes < 2:
        e = np.empty((0, 2), dtype=np.int64)
        return WSPairList(e, e.copy(), tree.points)
    ctx, P = _run_wspd(tree, s, device)
    return _fetch_pairs(ctx, P, tree.points)


def emit_arcs(pairs: WSPairList, nodes: SuppliedNodes, device: int | None = None) -> ArcList:
    """Spanner biarcs plus diagonal arcs (spanner.py:310-337), on device."""
    ctx = _lib.context(device)
    load_nodes(ctx, _lib.NODES, nodes)
    idx = _lib.as_i64(pairs.indices).reshape(-1, 2)
    pts = _lib.as_points(pairs.points)
    ctx.call("w1g_load_pairs", _lib.i64p(idx), idx.shape[0], _lib.f64p(pts), pts.shape[0])
    m = ctypes.c_int64(0)
    ctx.call("w1g_emit_arcs", ctypes.byref(m))
    m = int(m.value)
    tails = np.empty(m, dtype=np.int64)
    heads = np.empty(m, dtype=np.int64)
    costs = np.empty(m, dtype=np.float64)
    ctx.call("w1g_fetch_arcs", _lib.i64p(tails), _lib.i64p(heads), _lib.f64p(costs))
    return ArcList(tails, heads, costs)
