"""Parity at the BASELINE.json configurations' own sizes (the CUDA path through
the C-ABI against the C oracle, itself pinned to the reference by
tests/test_oracle_golden.py and tests/test_oracle_vs_reference.py).

* cfg3: one 1M+1M pair (s = 1, delta = 0.01): the whole network bit for bit and
  L equal to the reference's own scalar (tests/golden/scalars.npz, measured by
  running w1flow on this input);
* cfg5: all nine (delta, s) cells at 100k+100k, including the 90M-arc
  delta = 0.001 / s = 16 cell;
* cfg4: pairs of the 64 x 20k shared-centre batch;
* cfg2 with the reference's own delta schedule (delta derived from L);
* WSPD recursions deeper than 128 levels through the standalone stage API.
"""

import numpy as np
import pytest

from conftest import bits_equal, load_golden

pytestmark = pytest.mark.gpu

NET_FIELDS = ("supplies", "tails", "heads", "costs", "row_offsets")


@pytest.fixture(scope="module")
def w1g():
    import paper_2110_14734_b200 as m

    return m


def _front_end_vs_oracle(w1g, a, b, s, delta):
    from oracle import w1oracle as O

    fe = O.front_end(a, b, s, delta=delta)
    net, diag = w1g.sparsify(a, b, w1g.ApproxParams(s=s, best_effort=True, delta=delta))
    assert diag.lower_bound == fe.lower_bound
    assert diag.delta == fe.delta
    assert diag.n_pairs == fe.node_pairs.shape[0]
    assert diag.n_nodes == fe.network.supplies.shape[0]
    for f in NET_FIELDS:
        assert bits_equal(getattr(net, f), getattr(fe.network, f)), f
    return fe, net, diag


def test_cfg3_1m_network_and_lower_bound(w1g):
    from paper_2110_14734_b200 import synth

    a, b = synth.gaussian_cluster_pair(1_000_000, 1_000_000, seed=0)
    fe, net, diag = _front_end_vs_oracle(w1g, a, b, 1.0, 0.01)
    ref_L = float(load_golden("scalars")["cfg3_L"])
    assert diag.lower_bound == ref_L == fe.lower_bound
    assert diag.n_nodes - 2 == 342_392  # K at cfg3, delta = 0.01


@pytest.mark.parametrize("delta", [0.1, 0.01, 0.001])
@pytest.mark.parametrize("s", [1.0, 4.0, 16.0])
def test_cfg5_sweep_cell(w1g, s, delta):
    from paper_2110_14734_b200 import synth

    a, b = synth.gaussian_cluster_pair(100_000, 100_000, seed=0)
    fe, net, diag = _front_end_vs_oracle(w1g, a, b, s, delta)
    if (s, delta) == (16.0, 0.001):
        assert net.arc_count == 89_878_894  # the largest network of the sweep


@pytest.mark.parametrize("i,j", [(0, 1), (17, 42), (62, 63)])
def test_cfg4_pair(w1g, i, j):
    from paper_2110_14734_b200 import synth

    diags = synth.shared_centre_batch(64, 20_000, seed=0)
    _front_end_vs_oracle(w1g, diags[i], diags[j], 1.0, 0.01)


def test_cfg4_batch_entry_matches_oracle(w1g):
    """The batched C entry (w1g_front_end_batch) over a slice of the cfg4 matrix."""
    from oracle import w1oracle as O
    from paper_2110_14734_b200 import synth

    diags = synth.shared_centre_batch(64, 20_000, seed=0)
    pairs = [(0, 5), (3, 9), (10, 11), (40, 63)]
    got = {}
    w1g.sparsify_batch(diags, w1g.ApproxParams(s=1.0, best_effort=True, delta=0.01), pairs=pairs,
                       on_network=lambda i, j, net, d: got.__setitem__((i, j), net))
    assert sorted(got) == sorted(pairs)
    for i, j in pairs:
        fe = O.front_end(diags[i], diags[j], 1.0, delta=0.01)
        for f in NET_FIELDS:
            assert bits_equal(getattr(got[(i, j)], f), getattr(fe.network, f)), (i, j, f)


def test_cfg2_reference_delta_schedule(w1g):
    """delta = None: delta = 2 eps L / (sqrt2 n) from the RWMD bound (pipeline.py:116-122),
    the sequential schedule with a host read of L."""
    from paper_2110_14734_b200 import synth

    a, b = synth.gaussian_cluster_pair(100_000, 100_000, seed=0)
    fe, net, diag = _front_end_vs_oracle(w1g, a, b, 1.0, None)
    assert diag.lower_bound == float(load_golden("scalars")["cfg2_L"])


@pytest.mark.parametrize("name,s", [("deep_pm2i", 2.0), ("deep_pm2i_s8", 8.0)])
def test_wspd_deeper_than_128_levels(w1g, name, s):
    """build_wspd / count_pairs / write_pairs in the reference's exact order on trees
    whose WSPD recursion is 169 / 147 levels deep (the reference's explicit stack
    has no depth limit, spanner.py:206-241)."""
    g = load_golden(name)
    tree = w1g.build_split_tree(g["nodes_points"])
    for f in ("left", "right", "bbox", "rep", "size"):
        assert bits_equal(getattr(tree, f), g["tree_" + f]), f
    counts = w1g.count_pairs(tree, s)
    assert bits_equal(counts, g["wspd_counts"])
    pairs = w1g.build_wspd(tree, s)
    assert bits_equal(pairs.node_pairs, g["node_pairs"])
    assert bits_equal(pairs.indices, g["pair_indices"])
    offsets = np.concatenate([[0], np.cumsum(counts)])[:-1].astype(np.int64)
    again = w1g.write_pairs(tree, s, offsets, counts)
    assert bits_equal(again.node_pairs, g["node_pairs"])
    net, _ = w1g.sparsify(g["a"], g["b"], w1g.ApproxParams(s=s, best_effort=True, use_condensation=False))
    for f in NET_FIELDS:
        assert bits_equal(getattr(net, f), g["net_" + f]), f
