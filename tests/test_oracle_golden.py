"""Pin the C oracle (oracle/w1oracle.c) to the reference's own outputs.

The fixtures in tests/golden were produced by running the live reference
(tests/golden/make_golden.py); the oracle must reproduce every stage bit for
bit before it is trusted as the checker for the CUDA path.
"""

import numpy as np
import pytest

from conftest import bits_equal, golden_cases, load_golden, numpy_build_network, row_class_arcs
from oracle import w1oracle as O


@pytest.mark.parametrize("name", golden_cases())
def test_front_end_matches_reference(name):
    g = load_golden(name)
    fixed = float(g["fixed_delta"])
    fe = O.front_end(g["a"], g["b"], float(g["s"]), delta=None if np.isnan(fixed) else fixed,
                     seed=int(g["seed"]))
    assert bits_equal(fe.nodes0.points, g["n0_points"])
    assert bits_equal(fe.nodes0.a_mass, g["n0_a"])
    assert bits_equal(fe.nodes0.b_mass, g["n0_b"])
    assert fe.short_circuit == bool(g["short_circuit"])
    if fe.short_circuit:
        return
    L, LA, LB = O.rwmd(fe.nodes0)
    assert L == float(g["L"]) and LA == float(g["LA"]) and LB == float(g["LB"])
    assert fe.delta == float(g["delta"])
    assert bits_equal(fe.nodes.points, g["nodes_points"])
    assert bits_equal(fe.nodes.a_mass, g["nodes_a"])
    assert bits_equal(fe.nodes.b_mass, g["nodes_b"])
    t = fe.tree
    for f in ("left", "right", "bbox", "rep", "size"):
        assert bits_equal(getattr(t, f), g["tree_" + f]), f
    counts, pairs, indices = O.wspd(t, float(g["s"]))
    assert bits_equal(counts, g["wspd_counts"])
    assert bits_equal(pairs, g["node_pairs"])
    if "arc_tails" in g:
        tl, hd, cs = O.emit_arcs(indices, fe.nodes)
        assert bits_equal(tl, g["arc_tails"]) and bits_equal(hd, g["arc_heads"])
        assert bits_equal(cs, g["arc_costs"])
    net = fe.network
    for f in ("supplies", "tails", "heads", "costs", "row_offsets"):
        assert bits_equal(getattr(net, f), g["net_" + f]), f


def test_hypot_port_matches_numpy():
    g = load_golden("arith")
    port = np.array([O.hypot_port(x, y) for x, y in zip(g["hx"], g["hy"])])
    libm = np.array([O.hypot_libm(x, y) for x, y in zip(g["hx"], g["hy"])])
    assert bits_equal(libm, g["h"])
    assert bits_equal(port, g["h"])


def test_pairwise_sum_matches_numpy():
    g = load_golden("arith")
    for k in g:
        if k.startswith("v"):
            n = k[1:]
            assert O.pairwise_sum(g[k]) == float(g["s" + n])


def test_hypot_port_random_bulk():
    rng = np.random.default_rng(5)
    x = rng.uniform(-80, 80, 20000) * rng.choice([1.0, 1e-5, 1e5], 20000)
    y = rng.uniform(-80, 80, 20000)
    port = np.array([O.hypot_port(a, b) for a, b in zip(x, y)])
    assert bits_equal(port, np.hypot(x, y))


def test_error_paths():
    with pytest.raises(ValueError, match="duplicate"):
        O.split_tree(np.array([[1.0, 1.0], [1.0, 1.0]]))
    nodes = O.zero_condense(np.array([[0.0, 1e300]]), np.empty((0, 2)))
    with pytest.raises(ValueError, match="lattice"):
        O.delta_condense(nodes, 1e-300)
    with pytest.raises(ValueError, match="self-loop"):
        O.build_network([1, -1], [0], [0], [1.0])
    with pytest.raises(ValueError, match="unbalanced"):
        O.build_network([1, -2], [0], [1], [1.0])
    net = O.build_network([1, -1], [0, 0], [1, 1], [5.0, 3.0])
    assert net.arc_count == 1 and net.costs[0] == 3.0


def test_build_network_matches_numpy_ties():
    """Duplicate arcs whose minimal costs tie as +0.0 / -0.0: np.minimum.at keeps the later arc."""
    n, tails, heads, costs = row_class_arcs(1, n=3000, seed=11)
    sup = np.zeros(n, dtype=np.int64)
    net = O.build_network(sup, tails, heads, costs)
    t, h, c, ro = numpy_build_network(sup, tails, heads, costs)
    assert bits_equal(net.tails, t) and bits_equal(net.heads, h)
    assert bits_equal(net.costs, c)
    assert bits_equal(net.row_offsets, ro)
