"""Synthetic Gaussian-cluster persistence diagrams (benchmark workload).

Restates the reference generator (/root/reference/pkg/src/w1flow/synth.py:12-54)
draw for draw, so bench.py and the parity tests see byte-identical inputs to
the reference's own benchmark configurations.  This is
workload plumbing, not part of the sparsify hot path.
"""

from __future__ import annotations

import numpy as np

_MIN_LIFE = 1e-6


def _centres(rng, n_clusters: int, scale: float):
    # synth.py:46-51: uniform births, uniform lifetimes in [1, scale/2), Dirichlet weights
    c = np.stack(
        [rng.uniform(0.0, scale, n_clusters), rng.uniform(1.0, scale / 2, n_clusters)], axis=1
    )
    w = rng.dirichlet(np.ones(n_clusters))
    return c, w


def sample_points(rng, centres, weights, n: int, spread: float) -> np.ndarray:
    """synth.py:12-17 (_sample_points)."""
    idx = rng.choice(centres.shape[0], size=n, p=weights)
    births = centres[idx, 0] + rng.normal(0.0, spread, size=n)
    lives = np.maximum(np.abs(centres[idx, 1] + rng.normal(0.0, spread, size=n)), _MIN_LIFE)
    return np.stack([births, births + lives], axis=1)


def gaussian_cluster_pair(n_a: int, n_b: int, seed: int = 0, n_clusters: int = 8,
                          spread: float = 0.5, scale: float = 50.0):
    """synth.py:37-54 -> two (n, 2) float64 arrays around shared centres."""
    rng = np.random.default_rng(seed)
    c, w = _centres(rng, n_clusters, scale)
    return sample_points(rng, c, w, n_a, spread), sample_points(rng, c, w, n_b, spread)


def gaussian_cluster_diagram(n: int, seed: int = 0, n_clusters: int = 8, spread: float = 0.5,
                             scale: float = 50.0) -> np.ndarray:
    """synth.py:20-34."""
    rng = np.random.default_rng(seed)
    c, w = _centres(rng, n_clusters, scale)
    return sample_points(rng, c, w, n, spread)


def shared_centre_batch(n_diagrams: int, n_points: int, seed: int = 0, n_clusters: int = 8,
                        spread: float = 0.5, scale: float = 50.0) -> list[np.ndarray]:
    """cfg4: centres/weights drawn from default_rng(seed) as
    gaussian_cluster_pair does; diagram i from default_rng(1000 + i)."""
    c, w = _centres(np.random.default_rng(seed), n_clusters, scale)
    return [sample_points(np.random.default_rng(1000 + i), c, w, n_points, spread)
            for i in range(n_diagrams)]
