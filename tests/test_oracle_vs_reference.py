"""Differential check of the C oracle against the LIVE reference package.

Runs only where /root/reference is importable (the build container); the GPU
box has no reference tree and relies on the committed golden fixtures.
"""

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree not present")


@pytest.fixture(scope="module")
def w1flow():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_w1g")
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import w1flow as m
    return m


@pytest.mark.parametrize("n,s,delta", [(20000, 1.0, 0.01), (5000, 4.0, None), (3000, 16.0, 0.001)])
def test_chain_bit_exact(w1flow, n, s, delta):
    from oracle import w1oracle as O
    from w1flow import condensation, diagram, lower_bound, network, pipeline, spanner, synth

    a, b = synth.gaussian_cluster_pair(n, n, seed=1)
    n0 = diagram.zero_condense(a, b)
    L = lower_bound.rwmd(n0)
    eps = pipeline.condensation_epsilon(s)
    d = condensation.compute_delta(eps, L, n0.n_points()) if delta is None else delta
    nodes = condensation.delta_condense(n0, condensation.CondensationParams(eps, d, seed=0))
    tree = spanner.build_split_tree(nodes.points)
    pairs = spanner.build_wspd(tree, s)
    net = network.assemble(nodes, spanner.emit_arcs(pairs, nodes))

    fe = O.front_end(a.points, b.points, s, delta=delta)
    assert fe.lower_bound == L
    assert np.array_equal(fe.nodes.points, nodes.points)
    assert np.array_equal(fe.node_pairs, pairs.node_pairs)
    for f in ("supplies", "tails", "heads", "costs", "row_offsets"):
        assert getattr(fe.network, f).tobytes() == getattr(net, f).tobytes()


def test_synth_restatement_matches_reference(w1flow):
    from paper_2110_14734_b200 import synth as mine
    from w1flow import synth

    a, b = synth.gaussian_cluster_pair(3000, 2000, seed=4)
    x, y = mine.gaussian_cluster_pair(3000, 2000, seed=4)
    assert np.array_equal(a.points, x) and np.array_equal(b.points, y)
    d = synth.gaussian_cluster_diagram(500, seed=9)
    assert np.array_equal(d.points, mine.gaussian_cluster_diagram(500, seed=9))
