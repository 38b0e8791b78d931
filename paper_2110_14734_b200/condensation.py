"""Lattice (delta-) condensation (reference: w1flow/condensation.py).

`delta_condense` runs on the B200 (condense.cu): exact fp64 snapping with the
reference's round-half-away, radix sort of the integer cells, reduce-by-key
of the masses and splitmix64 per-cell offsets.  The host-side scalars (pitch,
half width, delta) are computed here with the reference's own expressions so
they are bit-identical.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .diagram import SuppliedNodes, fetch_nodes, load_nodes

_SQRT2 = math.sqrt(2.0)


@dataclass(frozen=True)
class CondensationParams:
    """Lattice pitch, fraction and RNG seed for one pass (condensation.py:29-44)."""

    epsilon: float
    delta: float
    k: float = 0.99
    seed: int = 0

    def __post_init__(self):
        if self.epsilon <= 0:
            raise ValueError("epsilon must be positive")
        if self.delta < 0:
            raise ValueError("delta must be nonnegative")
        if not (0.5 <= self.k < 1.0):
            raise ValueError("k must lie in [0.5, 1)")


def compute_delta(epsilon: float, lower_bound: float, n_points: int) -> float:
    """Lattice pitch 2*eps*L / (sqrt(2) * n) (condensation.py:47-59)."""
    if epsilon <= 0:
        raise ValueError("epsilon must be positive")
    if n_points < 1:
        raise ValueError("n_points must be >= 1")
    if lower_bound < 0:
        raise ValueError("lower bound must be nonnegative")
    return 2.0 * epsilon * lower_bound / (_SQRT2 * n_points)


def snap_points(points, delta: float, k: float, device: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Snap points to the k*delta lattice, round half away from zero
    (condensation.py:66-77), on device: cells = sign(t) floor(|t| + 0.5) with
    t = p / pitch, snapped = cells * pitch.  Returns (snapped, int64 cells)."""
    if delta <= 0:
        raise ValueError("delta must be positive")
    pitch = k * delta
    pts = _lib.as_points(points)
    n = pts.shape[0]
    snapped = np.empty((n, 2), dtype=np.float64)
    cells = np.empty((n, 2), dtype=np.int64)
    ctx = _lib.context(device)
    ctx.call("w1g_snap_points", _lib.f64p(pts), n, float(pitch), _lib.f64p(snapped), _lib.i64p(cells))
    return snapped, cells


def snap_point(p, delta: float, k: float = 0.99) -> tuple[float, float]:
    """condensation.py:80-82."""
    snapped, _ = snap_points(np.asarray(p, dtype=np.float64).reshape(1, 2), delta, k)
    return (float(snapped[0, 0]), float(snapped[0, 1]))


def delta_condense(nodes: SuppliedNodes, params: CondensationParams,
                   device: int | None = None) -> SuppliedNodes:
    """Snap nodes to the k*delta lattice, merge supplies, perturb merged nodes
    (condensation.py:105-124).  delta == 0 returns the input unchanged."""
    if params.delta == 0.0 or nodes.points.shape[0] == 0:
        return nodes
    ctx = _lib.context(device)
    load_nodes(ctx, _lib.NODES0, nodes)
    pitch = params.k * params.delta                       # condensation.py:73,123
    half_width = (1.0 - params.k) * params.delta / 2.0    # condensation.py:121
    k = ctypes.c_int64(0)
    ctx.call("w1g_delta_condense", float(params.delta), pitch, half_width,
             ctypes.c_uint64(int(params.seed) & 0xFFFFFFFFFFFFFFFF), ctypes.byref(k))
    return fetch_nodes(ctx, _lib.NODES, nodes.abar_supply, nodes.bbar_supply)
