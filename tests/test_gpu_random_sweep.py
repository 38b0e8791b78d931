"""A deterministic randomized sweep of the fused front end against the C oracle:
point distributions that stress different parts of the path -- Gaussian clusters,
integer-lattice points (exact distances: glibc hypot's zero-correction branch, many
ties in the sorts), points on a line (deep split trees, long WSPD recursions),
tiny and huge coordinates (hypot's scaling branches, the RWMD frame), heavy
duplication across the two diagrams -- at sizes and (s, delta) that exercise every
CSR row class, the windowed and full-K bitmap ranks and the depth-first WSPD's
stack spills and work sharing.  Every network array is compared bit for bit."""
import numpy as np
import pytest

from conftest import bits_equal

pytestmark = pytest.mark.gpu

NET_FIELDS = ("supplies", "tails", "heads", "costs", "row_offsets")


def _diagram(rng, kind: str, n: int) -> np.ndarray:
    if kind == "clusters":
        c = rng.uniform(0, 100, (6, 2))
        p = c[rng.integers(0, 6, n)] + rng.normal(0, 2.0, (n, 2))
    elif kind == "lattice":
        p = rng.integers(0, 60, (n, 2)).astype(np.float64)
    elif kind == "line":
        t = np.sort(rng.exponential(1.0, n)).cumsum()
        p = np.stack([t, 2.0 * t + 1.0], axis=1)
    elif kind == "tiny":
        p = rng.uniform(0, 1, (n, 2)) * 1e-160
    elif kind == "huge":
        p = rng.uniform(0, 1, (n, 2)) * 1e150
    else:  # "dups": few distinct points, many repeats
        base = rng.uniform(0, 10, (max(4, n // 20), 2))
        p = base[rng.integers(0, base.shape[0], n)]
    return np.ascontiguousarray(p)


CASES = [
    ("clusters", 3000, 1.0, 0.01), ("clusters", 3000, 16.0, None), ("clusters", 4000, 40.0, 0.001),
    ("lattice", 3000, 1.0, 0.0), ("lattice", 3000, 8.0, 0.5), ("lattice", 2500, 24.0, 0.0),
    ("line", 2000, 4.0, 0.0), ("line", 3000, 16.0, 0.001),
    ("tiny", 2000, 4.0, 0.0), ("huge", 2000, 4.0, 0.0),
    ("dups", 4000, 2.0, 0.0), ("dups", 4000, 12.0, None),
    ("clusters", 20000, 16.0, 0.001), ("lattice", 15000, 4.0, 0.0), ("line", 10000, 8.0, 0.0),
    ("dups", 20000, 1.0, 0.01),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_random_sweep_matches_oracle(case):
    import paper_2110_14734_b200 as w1g
    from oracle import w1oracle as O

    kind, n, s, delta = CASES[case]
    rng = np.random.default_rng(1000 + case)
    a, b = _diagram(rng, kind, n), _diagram(rng, kind, n - n // 7)
    if kind == "dups":  # half of b coincides with points of a
        b[: b.shape[0] // 2] = a[rng.integers(0, a.shape[0], b.shape[0] // 2)]
    fixed = delta is not None and delta > 0.0
    params = w1g.ApproxParams(s=s, best_effort=True, delta=delta if fixed else None,
                              use_condensation=delta is None or delta > 0.0)
    net, diag = w1g.sparsify(a, b, params)
    fe = O.front_end(a, b, s, delta=delta if fixed else None, use_condensation=delta is None or delta > 0.0)
    if fe.short_circuit:
        assert net is None
        return
    assert diag.n_pairs == fe.node_pairs.shape[0]
    for f in NET_FIELDS:
        assert bits_equal(getattr(net, f), getattr(fe.network, f)), (kind, n, s, delta, f)
