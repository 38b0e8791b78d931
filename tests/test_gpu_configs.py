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


@pytest.mark.parametrize("G", [2, 3, 4])
def test_rwmd_sharded_over_contexts(w1g, G):
    """w1g_rwmd_sharded: the rows of one pair over G contexts (here all on device 0,
    each with its own stream and host thread) recombine to w1g_rwmd bit for bit."""
    import ctypes

    from paper_2110_14734_b200 import _lib, lower_bound, synth
    from paper_2110_14734_b200.diagram import load_nodes

    a, b = synth.gaussian_cluster_pair(70000, 60000, seed=13)
    n0 = w1g.zero_condense(a, b)
    L, la, lb = lower_bound.rwmd_sides(n0)
    ctxs = [_lib.Context(0) for _ in range(G)]
    for c in ctxs:
        load_nodes(c, _lib.NODES0, n0)
    arr = (ctypes.c_void_p * G)(*[c.handle.value for c in ctxs])
    out = [ctypes.c_double() for _ in range(3)]
    _lib.check(_lib.load().w1g_rwmd_sharded(arr, G, *[ctypes.byref(x) for x in out]))
    assert (out[0].value, out[1].value, out[2].value) == (L, la, lb)
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("G,s,delta", [(2, 1.0, 0.01), (3, 4.0, 0.001), (5, 16.0, 0.1)])
def test_wspd_shards_partition_the_network(w1g, G, s, delta):
    """The sharded WSPD (w1g_wspd_shard) over G shards: the shards' arc slices (rank 0's
    with the diagonal arcs) assemble into exactly the single-GPU network."""
    import ctypes

    from paper_2110_14734_b200 import _lib, synth
    from paper_2110_14734_b200.network import fetch_network

    a, b = synth.gaussian_cluster_pair(100_000, 100_000, seed=0)
    ref, _ = w1g.sparsify(a, b, w1g.ApproxParams(s=s, best_effort=True, delta=delta))
    ctx = _lib.context()
    ap, bp = np.ascontiguousarray(a), np.ascontiguousarray(b)
    k0, bal = ctypes.c_int64(), ctypes.c_int32()
    ctx.call("w1g_zero_condense", _lib.f64p(ap), ap.shape[0], _lib.f64p(bp), bp.shape[0], ctypes.byref(k0),
             ctypes.byref(bal))
    kk = ctypes.c_int64()
    ctx.call("w1g_delta_condense", delta, 0.99 * delta, (1.0 - 0.99) * delta / 2.0, ctypes.c_uint64(0),
             ctypes.byref(kk))
    nn, depth = ctypes.c_int64(), ctypes.c_int32()
    ctx.call("w1g_split_tree", _lib.NODES, ctypes.byref(nn), ctypes.byref(depth))
    parts = []
    total_pairs = 0
    for g in range(G):
        P, m = ctypes.c_int64(), ctypes.c_int64()
        ctx.call("w1g_wspd_shard", s, g, G, ctypes.byref(P))
        total_pairs += P.value
        ctx.call("w1g_emit_pair_arcs", 1 if g == 0 else 0, ctypes.byref(m))
        t, h, c = np.empty(m.value, np.int64), np.empty(m.value, np.int64), np.empty(m.value)
        ctx.call("w1g_fetch_arcs", _lib.i64p(t), _lib.i64p(h), _lib.f64p(c))
        parts.append((t, h, c))
    assert total_pairs > 0
    t = np.concatenate([p[0] for p in parts])
    h = np.concatenate([p[1] for p in parts])
    c = np.concatenate([p[2] for p in parts])
    ctx.call("w1g_load_arcs", _lib.i64p(t), _lib.i64p(h), _lib.f64p(c), t.shape[0])
    n, m = ctypes.c_int64(), ctypes.c_int64()
    ctx.call("w1g_assemble", ctypes.byref(n), ctypes.byref(m))
    net = fetch_network(ctx, n.value, m.value)
    for f in NET_FIELDS:
        assert bits_equal(getattr(net, f), getattr(ref, f)), f


def test_sparsify_sharded_nccl_world1(w1g):
    """distributed.sparsify_sharded through a real NCCL process group (world size 1 on
    this box's one GPU): the replicated stages, rwmd_rows, the WSPD shard, the arc
    path through torch tensors over the library's device buffers, assemble."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    from paper_2110_14734_b200 import synth
    from paper_2110_14734_b200.distributed import sparsify_sharded

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        a, b = synth.gaussian_cluster_pair(100_000, 100_000, seed=0)
        for delta in (0.01, None):
            params = w1g.ApproxParams(s=1.0, best_effort=True, delta=delta)
            net, diag = sparsify_sharded(a, b, params, 0, 1)
            ref, rdiag = w1g.sparsify(a, b, params)
            assert diag.lower_bound == rdiag.lower_bound and diag.delta == rdiag.delta
            for f in NET_FIELDS:
                assert bits_equal(getattr(net, f), getattr(ref, f)), f
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("G", [2, 4])
def test_gathered_shard_pairs_build_the_network(w1g, G):
    """The sharded front end's gather: each shard's node pairs (w1g_pairs_device), concatenated
    on "rank 0" (w1g_load_pairs_device) and turned into the network by the fused builder
    (w1g_network_from_pairs) -- bit-identical to the single-GPU front end."""
    import ctypes

    import torch

    from paper_2110_14734_b200 import _lib, synth
    from paper_2110_14734_b200.network import fetch_network

    a, b = synth.gaussian_cluster_pair(100_000, 100_000, seed=3)
    ref, _ = w1g.sparsify(a, b, w1g.ApproxParams(s=2.0, best_effort=True, delta=0.01))
    ctx = _lib.context()
    k0, bal = ctypes.c_int64(), ctypes.c_int32()
    ap, bp = np.ascontiguousarray(a), np.ascontiguousarray(b)
    ctx.call("w1g_zero_condense", _lib.f64p(ap), ap.shape[0], _lib.f64p(bp), bp.shape[0], ctypes.byref(k0),
             ctypes.byref(bal))
    kk = ctypes.c_int64()
    ctx.call("w1g_delta_condense", 0.01, 0.99 * 0.01, (1.0 - 0.99) * 0.01 / 2.0, ctypes.c_uint64(0), ctypes.byref(kk))
    nn, depth = ctypes.c_int64(), ctypes.c_int32()
    ctx.call("w1g_split_tree", _lib.NODES, ctypes.byref(nn), ctypes.byref(depth))
    parts = []
    for g in range(G):
        P = ctypes.c_int64()
        ctx.call("w1g_wspd_shard", 2.0, g, G, ctypes.byref(P))
        up = ctypes.c_void_p()
        ctx.call("w1g_pairs_device", ctypes.byref(up), ctypes.byref(P))
        ctx.call("w1g_synchronize")
        n = 2 * P.value
        buf = torch.empty(n, dtype=torch.int32, device="cuda")
        src = torch.as_tensor(type("A", (), {"__cuda_array_interface__": {
            "shape": (n,), "typestr": "<i4", "data": (up.value, False), "version": 3, "strides": None}})(),
            device="cuda")
        buf.copy_(src)
        parts.append(buf)
    allp = torch.cat(parts)
    torch.cuda.synchronize()
    ctx.call("w1g_load_pairs_device", allp.data_ptr(), allp.shape[0] // 2)
    n_, m_ = ctypes.c_int64(), ctypes.c_int64()
    ctx.call("w1g_network_from_pairs", ctypes.byref(n_), ctypes.byref(m_))
    net = fetch_network(ctx, n_.value, m_.value)
    for f in NET_FIELDS:
        assert bits_equal(getattr(net, f), getattr(ref, f)), f


def test_wspd_capacity_regrow(w1g, monkeypatch):
    """The WSPD's pair and frontier / pool capacities start far too small
    (W1G_WSPD_TINY_CAPS=1): the overflow flags and the regrow-and-retry path give the
    same network (depth-first kernel) and the same reference-order pairs (standalone
    build_wspd) as the normal capacities."""
    from paper_2110_14734_b200 import synth

    a, b = synth.gaussian_cluster_pair(20_000, 20_000, seed=3)
    params = w1g.ApproxParams(s=4.0, best_effort=True, delta=0.001)
    ref, _ = w1g.sparsify(a, b, params)
    nodes = w1g.zero_condense(a, b)
    tree = w1g.build_split_tree(nodes.points)
    ref_pairs = w1g.build_wspd(tree, 4.0)
    monkeypatch.setenv("W1G_WSPD_TINY_CAPS", "1")
    got, _ = w1g.sparsify(a, b, params)
    for f in NET_FIELDS:
        assert bits_equal(getattr(got, f), getattr(ref, f)), f
    got_pairs = w1g.build_wspd(tree, 4.0)
    for f in ("node_pairs", "indices"):
        assert bits_equal(getattr(got_pairs, f), getattr(ref_pairs, f)), f
