import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")


def golden_cases():
    return sorted(
        os.path.basename(p)[:-4]
        for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
        if not os.path.basename(p).startswith(("arith", "scalars", "retrieval"))
    )


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def bits_equal(x, y):
    x = np.ascontiguousarray(x)
    y = np.ascontiguousarray(y)
    return x.shape == y.shape and x.dtype == y.dtype and x.tobytes() == y.tobytes()


def numpy_build_network(supplies, tails, heads, costs):
    """network.py:70-85 restated with numpy itself (np.lexsort + np.minimum.at)."""
    order = np.lexsort((heads, tails))
    t, h, c = tails[order], heads[order], costs[order]
    new = np.empty(t.shape[0], dtype=bool)
    new[0] = True
    new[1:] = (t[1:] != t[:-1]) | (h[1:] != h[:-1])
    gid = np.cumsum(new) - 1
    cmin = np.full(int(gid[-1]) + 1, np.inf)
    np.minimum.at(cmin, gid, c)
    ro = np.zeros(supplies.shape[0] + 1, dtype=np.int64)
    ro[1:] = np.cumsum(np.bincount(t[new], minlength=supplies.shape[0]))
    return t[new], h[new], cmin, ro


def row_class_arcs(n_huge, n=6000, seed=7):
    """Arc lists exercising every CSR row class (<= 32, <= 256, <= 4096 arcs, and
    n_huge rows of 6000), many duplicate (tail, head) pairs, costs tying at +0.0 / -0.0."""
    rng = np.random.default_rng(seed + n_huge)
    lengths = np.concatenate([rng.integers(0, 33, n // 2), rng.integers(33, 257, n // 30),
                              rng.integers(257, 4097, 6), np.full(n_huge, 6000)])
    tails = np.repeat(rng.permutation(n)[: lengths.shape[0]], lengths)
    heads = rng.integers(0, n, tails.shape[0])
    dup = rng.random(tails.shape[0]) < 0.3
    heads[dup] = (tails[dup] + 1 + rng.integers(0, 4, int(dup.sum()))) % n
    heads[heads == tails] = (heads[heads == tails] + 1) % n
    costs = rng.choice(np.array([0.0, -0.0, 1.5, 2.25, 7.0]), tails.shape[0])
    order = rng.permutation(tails.shape[0])
    return n, tails[order], heads[order], costs[order]
