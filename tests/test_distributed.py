"""Multi-rank host logic on CPU (gloo, world_size 2 and 4).

The device work of each rank is replaced by the C oracle so the sharding,
the all-gathers and the tree-order recombination are exercised without a
GPU; on the B200 the same code calls w1g_rwmd_range / approx_w1.
"""

import os
import socket

import numpy as np
import pytest

from paper_2110_14734_b200.distributed import pairwise_combine, pairwise_plan


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("n", [0, 1, 7, 127, 128, 129, 300, 1000, 4099, 100003])
@pytest.mark.parametrize("pieces", [1, 2, 3, 4, 8])
def test_plan_combine_is_numpy_sum(n, pieces):
    rng = np.random.default_rng(n * 10 + pieces)
    v = rng.uniform(0, 5, n) * rng.integers(1, 4, n)
    plan = pairwise_plan(n, pieces)
    assert plan[0][0] == 0 and plan[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(plan, plan[1:]))
    partials = [np.sum(v[b:e]) for b, e in plan]
    assert pairwise_combine(n, pieces, partials) == float(np.sum(v))


def _rwmd_worker(rank, world, port, n, out):
    import torch.distributed as dist

    from oracle import w1oracle as O
    from paper_2110_14734_b200 import synth
    from paper_2110_14734_b200.diagram import SuppliedNodes
    from paper_2110_14734_b200.distributed import rwmd_rows

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = synth.gaussian_cluster_pair(n, n + 17, seed=5)
    on = O.zero_condense(a, b)
    nodes = SuppliedNodes(on.points, on.a_mass, on.b_mass, on.abar_supply, on.bbar_supply)
    best = {0: O.rwmd_best(on, "a"), 1: O.rwmd_best(on, "b")}
    mass = {0: on.a_mass[on.a_mass > 0], 1: on.b_mass[on.b_mass > 0]}

    def partial(side, b_, e_):
        terms = mass[side][b_:e_].astype(np.float64) * best[side][b_:e_]
        return float(np.sum(terms))

    L, la, lb = rwmd_rows(nodes, rank, world, partial_fn=partial)
    ref = O.rwmd(on)
    out[rank] = (L == ref[0] and la == ref[1] and lb == ref[2], L, ref[0])
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_rwmd_rows_gloo_bit_exact(world):
    import torch.multiprocessing as mp

    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_rwmd_worker, args=(world, _free_port(), 3000, out), nprocs=world, join=True)
    assert len(out) == world
    for r in range(world):
        assert out[r][0], out[r]


def _pairs_worker(rank, world, port, out):
    import torch.distributed as dist

    from paper_2110_14734_b200 import ApproxParams
    from paper_2110_14734_b200.distributed import pairwise_w1_ranks

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    diagrams = [None] * 9
    done = []

    def compute(i, j):
        done.append((i, j))
        return i * 100.0 + j

    m = pairwise_w1_ranks(diagrams, ApproxParams(s=1, best_effort=True), rank, world, compute=compute)
    out[rank] = (m.tolist(), done)
    dist.destroy_process_group()


def test_pairwise_ranks_gloo():
    import torch.multiprocessing as mp

    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_pairs_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    mats = [np.array(out[r][0]) for r in range(world)]
    for m in mats:
        for i in range(9):
            for j in range(i + 1, 9):
                assert m[i, j] == m[j, i] == i * 100.0 + j
    work = sorted(out[0][1] + out[1][1])
    assert work == [(i, j) for i in range(9) for j in range(i + 1, 9)]
    assert not set(out[0][1]) & set(out[1][1])


def _gather_worker(rank, world, port, sizes, out):
    import torch
    import torch.distributed as dist

    from paper_2110_14734_b200.distributed import gather_arcs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(rank)
    m = sizes[rank]
    t = torch.from_numpy(rng.integers(0, 1000, m))
    h = torch.from_numpy(rng.integers(0, 1000, m))
    c = torch.from_numpy(rng.uniform(0, 9, m))
    got = gather_arcs(t, h, c, rank, world)
    out[rank] = None if got is None else [x.numpy().tolist() for x in got]
    dist.destroy_process_group()


@pytest.mark.parametrize("sizes", [[5, 7], [0, 4, 9], [3, 0, 0, 2]])
def test_gather_arcs_gloo(sizes):
    """The arc-list gather of the sharded front end: rank 0 receives every slice in rank order."""
    import torch.multiprocessing as mp

    world = len(sizes)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gather_worker, args=(world, _free_port(), sizes, out), nprocs=world, join=True)
    want = [[], [], []]
    for r, m in enumerate(sizes):
        rng = np.random.default_rng(r)
        want[0] += rng.integers(0, 1000, m).tolist()
        want[1] += rng.integers(0, 1000, m).tolist()
        want[2] += rng.uniform(0, 9, m).tolist()
    assert out[0] == want
    assert all(out[r] is None for r in range(1, world))


def _shard_worker(rank, world, port, out):
    """The sharded front end's data flow with the C oracle standing in for each
    rank's device: replicated condense + tree, the WSPD owner loop split by
    w % world, this rank's arcs (rank 0 adds the diagonal arcs), gather on rank 0,
    assemble there."""
    import torch
    import torch.distributed as dist

    from oracle import w1oracle as O
    from paper_2110_14734_b200 import synth
    from paper_2110_14734_b200.distributed import gather_arcs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = synth.gaussian_cluster_pair(3000, 2500, seed=8)
    n0 = O.zero_condense(a, b)
    nodes = O.delta_condense(n0, 0.01)
    tree = O.split_tree(nodes.points)
    counts, pairs, idx = O.wspd(tree, 2.0)
    owners = np.repeat(np.flatnonzero(tree.left >= 0), counts)
    mine = idx[owners % world == rank]
    t, h, c = O.emit_arcs(mine, nodes)
    if rank != 0:  # only the pairs' arcs: both directions
        P = mine.shape[0]
        t, h, c = t[:2 * P], h[:2 * P], c[:2 * P]
    got = gather_arcs(torch.from_numpy(t), torch.from_numpy(h), torch.from_numpy(c), rank, world)
    if rank == 0:
        net = O.assemble(nodes, *[x.numpy() for x in got])
        ref = O.front_end(a, b, 2.0, delta=0.01).network
        out[0] = all(getattr(net, f).tobytes() == getattr(ref, f).tobytes()
                     for f in ("supplies", "tails", "heads", "costs", "row_offsets"))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_wspd_arc_gather_gloo(world):
    import torch.multiprocessing as mp

    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_shard_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert out[0] is True
