"""Persistence diagrams and 0-condensation (reference: w1flow/diagram.py).

`zero_condense` runs on the B200 (condense.cu: 128-bit key radix sort,
run-length unique, per-side multiplicities); the dataclasses and validation
mirror the reference so objects flow unchanged into the rest of the API.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Iterable, Iterator, NamedTuple

import numpy as np

from . import _lib

SQRT2 = math.sqrt(2.0)


class DiagramFormatError(ValueError):
    """Invalid diagram content (diagram.py:20-21)."""


class PDPoint(NamedTuple):
    birth: float
    death: float


def diagonal_distance(p: PDPoint) -> float:
    """(death - birth)/sqrt(2), diagram.py:35-37 (scalar helper)."""
    return (p.death - p.birth) / SQRT2


def diagonal_projection(p: PDPoint) -> tuple[float, float]:
    """((b+d)/2, (b+d)/2), diagram.py:29-32 (scalar helper)."""
    m = 0.5 * (p.birth + p.death)
    return (m, m)


def diagonal_distances(points) -> np.ndarray:
    """|y - x| / sqrt(2) per row of an (n, 2) array (diagram.py:40-47).  The
    device kernels evaluate the same two IEEE operations inline (rwmd.cu,
    network.cu); this is the host helper of the public API."""
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 2)
    return np.abs(pts[:, 1] - pts[:, 0]) / SQRT2


def diagonal_projections(points) -> np.ndarray:
    """((x+y)/2, (x+y)/2) per row of an (n, 2) array (diagram.py:50-54)."""
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 2)
    m = 0.5 * (pts[:, 0] + pts[:, 1])
    return np.stack([m, m], axis=1)


class PersistenceDiagram:
    """Finite multiset of (birth, death) points with death > birth (diagram.py:57-95)."""

    __slots__ = ("points",)

    def __init__(self, points: Iterable | np.ndarray = ()):
        pts = np.asarray(points, dtype=np.float64)
        if pts.size == 0:
            pts = np.empty((0, 2), dtype=np.float64)
        if pts.ndim != 2 or pts.shape[1] != 2:
            raise DiagramFormatError("expected an (n, 2) array of (birth, death) pairs")
        if not np.all(np.isfinite(pts)):
            raise DiagramFormatError("non-finite coordinate in diagram")
        if np.any(pts[:, 1] <= pts[:, 0]):
            raise DiagramFormatError("every point must satisfy death > birth")
        self.points = pts

    def __len__(self) -> int:
        return self.points.shape[0]

    def __iter__(self) -> Iterator[PDPoint]:
        for b, d in self.points:
            yield PDPoint(float(b), float(d))

    def __eq__(self, other) -> bool:
        if not isinstance(other, PersistenceDiagram):
            return NotImplemented
        if len(self) != len(other):
            return False
        a = self.points[np.lexsort((self.points[:, 1], self.points[:, 0]))]
        b = other.points[np.lexsort((other.points[:, 1], other.points[:, 0]))]
        return bool(np.array_equal(a, b))

    def __repr__(self) -> str:
        return f"PersistenceDiagram({len(self)} points)"


def _parse_pair(lineno: int, tokens: list[str]) -> tuple[float, float]:
    """One data line of the diagram text format -> (birth, death), validated."""
    if len(tokens) != 2:
        raise DiagramFormatError(f"line {lineno}: expected two numbers, got {len(tokens)} tokens")
    try:
        pair = (float(tokens[0]), float(tokens[1]))
    except ValueError:
        raise DiagramFormatError(f"line {lineno}: non-numeric token") from None
    if not all(map(math.isfinite, pair)):
        raise DiagramFormatError(f"line {lineno}: non-finite coordinate")
    if pair[1] < pair[0]:
        raise DiagramFormatError(f"line {lineno}: death < birth")
    return pair


def parse_diagram(text: str) -> tuple[PersistenceDiagram, int]:
    """Diagram text, one "birth death" pair per line (diagram.py:98-131).

    Blank lines and lines starting with '#' are skipped; repeated lines are
    multiplicity; zero-persistence points (death == birth) are dropped and
    counted; any malformed line rejects the input with its line number."""
    rows = []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        body = raw.strip()
        if body and body[0] != "#":
            rows.append(_parse_pair(lineno, body.split()))
    pts = np.array(rows, dtype=np.float64).reshape(-1, 2)
    keep = pts[:, 1] != pts[:, 0]
    return PersistenceDiagram(pts[keep]), int(pts.shape[0] - np.count_nonzero(keep))


def serialize_diagram(diagram: PersistenceDiagram) -> str:
    """Inverse of parse_diagram up to point order (diagram.py:134-137): repr()
    of each coordinate, so a round trip is exact."""
    lines = [f"{float(b)!r} {float(d)!r}" for b, d in points_of(diagram)]
    return "\n".join(lines) + ("\n" if lines else "")


def load_diagram(path) -> tuple[PersistenceDiagram, int]:
    """parse_diagram of a file; errors carry the path (diagram.py:140-147)."""
    with open(path, "r", encoding="utf-8") as fh:
        text = fh.read()
    try:
        return parse_diagram(text)
    except DiagramFormatError as exc:
        raise DiagramFormatError(f"{path}: {exc}") from None


def points_of(d) -> np.ndarray:
    """(n, 2) float64 C-contiguous points of a diagram-like object."""
    pts = d.points if hasattr(d, "points") else d
    return _lib.as_points(pts)


def pinned_points(d) -> np.ndarray:
    """A page-locked (n, 2) float64 copy of a diagram's points.  Passing it to
    sparsify / approx_w1 lets the front end DMA the input straight to the
    device instead of staging it through its own pinned buffer."""
    p = points_of(d)
    (out,) = _lib.pinned_arrays([(p.shape, np.float64)])
    out[...] = p
    return out


@dataclass(frozen=True)
class SuppliedNodes:
    """Deduplicated planar nodes with per-side integer masses (diagram.py:150-187)."""

    points: np.ndarray  # (k, 2) float64, pairwise distinct
    a_mass: np.ndarray  # (k,) int64
    b_mass: np.ndarray  # (k,) int64
    abar_supply: int
    bbar_supply: int

    @property
    def supply(self) -> np.ndarray:
        return self.a_mass - self.b_mass

    @property
    def a_member(self) -> np.ndarray:
        return self.a_mass > 0

    @property
    def b_member(self) -> np.ndarray:
        return self.b_mass > 0

    def n_points(self) -> int:
        return int(self.a_mass.sum() + self.b_mass.sum())

    def total_balance(self) -> int:
        return int(self.supply.sum()) + self.abar_supply + self.bbar_supply


def _empty_nodes(abar: int = 0, bbar: int = 0) -> SuppliedNodes:
    z = np.zeros(0, dtype=np.int64)
    return SuppliedNodes(np.empty((0, 2), dtype=np.float64), z, z.copy(), abar, bbar)


def fetch_nodes(ctx, slot: int, abar: int, bbar: int) -> SuppliedNodes:
    k = ctypes.c_int64(0)
    ctx.call("w1g_nodes_size", slot, ctypes.byref(k))
    k = int(k.value)
    pts = np.empty((k, 2), dtype=np.float64)
    am = np.empty(k, dtype=np.int64)
    bm = np.empty(k, dtype=np.int64)
    if k:
        ctx.call("w1g_fetch_nodes", slot, _lib.f64p(pts), _lib.i64p(am), _lib.i64p(bm))
    return SuppliedNodes(pts, am, bm, abar, bbar)


def load_nodes(ctx, slot: int, nodes: SuppliedNodes) -> None:
    pts = _lib.as_points(nodes.points)
    am = _lib.as_i64(nodes.a_mass)
    bm = _lib.as_i64(nodes.b_mass)
    ctx.call("w1g_load_nodes", slot, _lib.f64p(pts), _lib.i64p(am), _lib.i64p(bm), pts.shape[0],
             int(nodes.abar_supply), int(nodes.bbar_supply))


def zero_condense(a, b, device: int | None = None) -> SuppliedNodes:
    """Merge coincident points of both diagrams (diagram.py:190-208), on device."""
    ap, bp = points_of(a), points_of(b)
    na, nb = ap.shape[0], bp.shape[0]
    if na + nb == 0:
        return _empty_nodes()
    ctx = _lib.context(device)
    k0 = ctypes.c_int64(0)
    bal = ctypes.c_int32(0)
    ctx.call("w1g_zero_condense", _lib.f64p(ap), na, _lib.f64p(bp), nb, ctypes.byref(k0), ctypes.byref(bal))
    return fetch_nodes(ctx, _lib.NODES0, -na, nb)
