"""Generate golden fixtures by running the LIVE reference (w1flow) on fixed inputs.

Run in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Every array written here is an output of the reference's own functions
(/root/reference/pkg/src/w1flow), not of this repo's code, so the fixtures
pin both the C oracle (tests/test_oracle_golden.py) and the CUDA path
(tests/test_gpu_parity.py) to the reference bit for bit.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from w1flow import condensation, diagram, lower_bound, network, pipeline, spanner, synth  # noqa: E402
from w1flow.diagram import PersistenceDiagram  # noqa: E402


def chain(a, b, s, delta=None, seed=0):
    """pipeline.py:105-130 with an optional fixed delta (test_acceptance.py:224-237)."""
    out = {}
    n0 = diagram.zero_condense(a, b)
    out.update(n0_points=n0.points, n0_a=n0.a_mass, n0_b=n0.b_mass)
    if n0.points.shape[0] == 0 or np.array_equal(n0.a_mass, n0.b_mass):
        out["short_circuit"] = np.array(1)
        return out
    out["short_circuit"] = np.array(0)
    a_sel, b_sel = n0.a_member, n0.b_member
    la = lower_bound._one_sided(n0.points[a_sel], n0.a_mass[a_sel], n0.points[b_sel], 1)
    lb = lower_bound._one_sided(n0.points[b_sel], n0.b_mass[b_sel], n0.points[a_sel], 1)
    L = lower_bound.rwmd(n0)
    out.update(L=np.array(L), LA=np.array(la), LB=np.array(lb))
    eps = pipeline.condensation_epsilon(s)
    nodes = n0
    d = 0.0
    if L > 0.0:
        d = condensation.compute_delta(eps, L, n0.n_points()) if delta is None else delta
        if d > 0.0:
            nodes = condensation.delta_condense(n0, condensation.CondensationParams(eps, d, seed=seed))
    out.update(delta=np.array(d), nodes_points=nodes.points, nodes_a=nodes.a_mass, nodes_b=nodes.b_mass)
    tree = spanner.build_split_tree(nodes.points)
    out.update(tree_left=tree.left, tree_right=tree.right, tree_bbox=tree.bbox, tree_rep=tree.rep,
               tree_size=tree.size)
    counts = spanner.count_pairs(tree, s)
    pairs = spanner.build_wspd(tree, s)
    out.update(wspd_counts=counts, node_pairs=pairs.node_pairs, pair_indices=pairs.indices)
    arcs = spanner.emit_arcs(pairs, nodes)
    out.update(arc_tails=arcs.tails, arc_heads=arcs.heads, arc_costs=arcs.costs)
    net = network.assemble(nodes, arcs)
    out.update(net_supplies=net.supplies, net_tails=net.tails, net_heads=net.heads,
               net_costs=net.costs, net_row_offsets=net.row_offsets)
    return out


def random_diagram(rng, max_points=12, scale=10.0, min_points=0):
    # pkg/tests/helpers.py:10-17
    n = int(rng.integers(min_points, max_points + 1))
    if n == 0:
        return PersistenceDiagram()
    births = rng.uniform(0.0, scale, n)
    lifetimes = rng.uniform(1e-3, scale / 2.0, n)
    return PersistenceDiagram(np.stack([births, births + lifetimes], axis=1))


def save(name, a, b, s, delta=None, seed=0, w1=False, **extra):
    out = chain(a, b, s, delta, seed)
    out.update(a=a.points, b=b.points, s=np.array(float(s)), seed=np.array(seed),
               fixed_delta=np.array(np.nan if delta is None else delta))
    if w1:
        params = pipeline.ApproxParams(s=s, best_effort=True, seed=seed)
        value, diag = pipeline.approx_w1(a, b, params)
        out.update(w1=np.array(value), w1_status=np.array(diag.status), w1_n_arcs=np.array(diag.n_arcs))
    out.update(extra)
    if out.get("node_pairs") is not None and out["node_pairs"].shape[0] > 20000:
        # large cases: the CSR network already holds the arc set; indices = rep[node_pairs]
        for key in ("arc_tails", "arc_heads", "arc_costs", "pair_indices"):
            out.pop(key, None)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, {k: v.shape for k, v in out.items() if hasattr(v, "shape") and v.ndim})


def deep_cases():
    """Inputs whose WSPD recursion is far deeper than 128 levels (the reference's
    explicit stack has no limit, spanner.py:206-241): births +-2^-i, deaths b+1."""
    P = PersistenceDiagram
    births = np.array([sg * 2.0 ** -i for i in range(100) for sg in (1.0, -1.0)])
    deep = P(np.stack([births, births + 1.0], axis=1))
    save("deep_pm2i", deep, P([(0.5, 1.5)]), 2.0, delta=0.0)
    save("deep_pm2i_s8", deep, P([(0.25, 2.5), (0.0, 1.0)]), 8.0, delta=0.0)


def retrieval_cases():
    """nn_search stages (pipeline.py:191-243), WCD (lower_bound.py:78-92) and the dense
    exact oracle (oracle.py:66-108) on a mixed corpus, from the live reference."""
    from w1flow import oracle

    rng = np.random.default_rng(77)
    P = PersistenceDiagram
    corpus = [random_diagram(rng, max_points=30, min_points=1) for _ in range(14)]
    corpus += list(synth.gaussian_cluster_pair(400, 300, seed=11))
    corpus += [synth.gaussian_cluster_diagram(250 + 50 * i, seed=20 + i) for i in range(6)]
    corpus.append(P())  # an empty diagram
    corpus.append(P(np.array([[-3.5, -0.0], [-0.0, 2.0], [1.0, 2.5]])))  # signed zeros, negatives
    query = synth.gaussian_cluster_diagram(300, seed=20)
    out = {"query": query.points, "n_corpus": np.array(len(corpus))}
    for i, d in enumerate(corpus):
        out[f"c{i}"] = d.points
    out["wcd"] = np.array([lower_bound.wcd(query, d) for d in corpus])
    out["wcd_rev"] = np.array([lower_bound.wcd(d, query) for d in corpus])
    out["rwmd"] = np.array([lower_bound.rwmd(diagram.zero_condense(query, d)) for d in corpus])
    specs = {
        "spec_wcd_rwmd_pdflow": (("wcd", 12, None), ("rwmd", 5, None), ("pdflow", 1, 12.0)),
        "spec_rwmd_exact": (("rwmd", 4, None), ("exact", 1, None)),
        "spec_wcd_only": (("wcd", 1, None),),
    }
    for name, stages in specs.items():
        spec = pipeline.PipelineSpec(tuple(pipeline.PipelineStage(a, k, s) for a, k, s in stages))
        best, nd = pipeline.nn_search(query, corpus, spec, seed=3)
        out[name + "_best"] = np.array(best)
        for si, (surv, sc) in enumerate(zip(nd.stage_survivors, nd.stage_scores)):
            out[f"{name}_s{si}_survivors"] = np.array(surv, dtype=np.int64)
            keys = np.array(sorted(sc), dtype=np.int64)
            out[f"{name}_s{si}_ids"] = keys
            out[f"{name}_s{si}_scores"] = np.array([sc[k] for k in keys])
    # dense oracle networks and exact W1
    for i, (x, y) in enumerate([(query, corpus[15]), (corpus[0], corpus[1]), (corpus[22], corpus[14]),
                                (corpus[23], query)]):
        nodes = diagram.zero_condense(x, y)
        net = oracle.dense_network(nodes)
        out.update({f"dense{i}_a": x.points, f"dense{i}_b": y.points,
                    f"dense{i}_supplies": net.supplies, f"dense{i}_tails": net.tails,
                    f"dense{i}_heads": net.heads, f"dense{i}_costs": net.costs,
                    f"dense{i}_row_offsets": net.row_offsets,
                    f"dense{i}_w1": np.array(oracle.exact_w1_dense(x, y))})
    np.savez_compressed(os.path.join(HERE, "retrieval.npz"), **out)
    print("retrieval", len(out), "arrays")


def main():
    deep_cases()
    retrieval_cases()
    # cfg1: BASELINE.json configs[0] -- 1k points each, s=1, delta=0.01
    a, b = synth.gaussian_cluster_pair(1000, 1000, seed=0)
    save("cfg1_s1_d001", a, b, 1.0, delta=0.01)
    # the reference's own delta schedule (approx_w1) at s=1 and s=12, with W1
    save("cfg1_s1_auto", a, b, 1.0, w1=True)
    save("cfg1_s12_auto", a, b, 12.0, w1=True)
    # 2k shared-centre pair at s=4 (more pairs per node)
    a2, b2 = synth.gaussian_cluster_pair(1200, 900, seed=5)
    save("gauss1k_s4_d005", a2, b2, 4.0, delta=0.05, seed=3)
    # delta = 0: nodes stay lexicographic (rep == min index path)
    save("gauss1k_s2_nodelta", a2, b2, 2.0, delta=0.0)

    # hand examples from pkg/tests/test_lower_bound.py:48-81 and SPEC vectors
    P = PersistenceDiagram
    hands = {
        "hand_single_pair": (P([(0, 2)]), P([(0, 3)])),
        "hand_two_vs_one": (P([(0, 2), (0, 4)]), P([(0, 3)])),
        "hand_identical": (P([(0, 2), (1, 4)]), P([(0, 2), (1, 4)])),
        "hand_one_empty": (P([(0, 2)]), P()),
        "hand_both_empty": (P(), P()),
        "hand_far_diag": (P([(0, 2)]), P([(0, 100)])),
        "hand_multiset": (P([(0, 2), (0, 2), (1, 5)]), P([(0, 2), (3, 4)])),
        "hand_L0_dual": (P([(0, 2), (0, 2)]), P([(0, 2)])),
        "hand_B_empty4": (P([(0, 2), (1, 3), (2, 4), (0, 1)]), P()),
    }
    for name, (x, y) in hands.items():
        save(name, x, y, 2.0, w1=True)

    # random small pairs (helpers.random_pair), several s, auto delta and W1
    rng = np.random.default_rng(2024)
    rand = []
    for i in range(40):
        x, y = random_diagram(rng), random_diagram(rng)
        s = [1.0, 2.0, 4.0, 12.0, 20.0][i % 5]
        rand.append((x, y, s, i))
    for x, y, s, i in rand:
        save(f"rand_{i:02d}", x, y, s, seed=i, w1=True)

    # H0-like diagrams: every birth is 0 (one huge run of equal x)
    r = np.random.default_rng(7)
    h0a = P(np.stack([np.zeros(300), r.uniform(0.1, 9, 300)], 1))
    h0b = P(np.stack([np.zeros(200), r.uniform(0.1, 9, 200)], 1))
    save("h0_births_zero", h0a, h0b, 2.0, w1=True)
    # negative coordinates and repeated points, fixed delta hits half-away rounding
    na = np.round(r.uniform(-20, 20, (400, 1)), 1)
    nega = P(np.concatenate([na, na + np.round(r.uniform(0.1, 5, (400, 1)), 1)], 1))
    nb_ = np.round(r.uniform(-20, 20, (300, 1)), 1)
    negb = P(np.concatenate([nb_, nb_ + np.round(r.uniform(0.1, 5, (300, 1)), 1)], 1))
    save("neg_grid_d02", nega, negb, 3.0, delta=0.2 / 0.99)
    # adjacent floats (split-tree midpoint fallback, spanner.py:139-144)
    base = r.uniform(0, 1, (5, 1))
    xs = np.repeat(base, 40, axis=0) + r.uniform(0, 1e-14, (200, 1))
    adj = P(np.concatenate([xs, xs + 1.0 + r.uniform(0, 1e-14, (200, 1))], 1))
    save("adjacent_floats", adj, P([(0.5, 1.5)]), 2.0, delta=0.0)

    # arithmetic kernels: glibc hypot and numpy pairwise sum
    hx = np.concatenate([r.uniform(-100, 100, 8000), r.normal(0, 1e-3, 2000), r.uniform(-1, 1, 1000) * 1e-300,
                         r.uniform(-1, 1, 1000) * 1e300])
    hy = np.concatenate([r.uniform(-100, 100, 8000), r.normal(0, 1e-3, 2000), r.uniform(-1, 1, 1000) * 1e-300,
                         r.uniform(-1, 1, 1000) * 1e300])
    hy[:500] = hx[:500] * 1e-17  # tiny-ratio branch
    sums = {}
    for n in (0, 1, 7, 8, 9, 127, 128, 129, 1000, 12345, 100003):
        v = r.uniform(0, 3, n) * r.integers(1, 4, n)
        sums[f"v{n}"] = v
        sums[f"s{n}"] = np.array(np.sum(v))
    np.savez_compressed(os.path.join(HERE, "arith.npz"), hx=hx, hy=hy, h=np.hypot(hx, hy), **sums)

    # fingerprints of the full-size benchmark inputs and the reference's scalars
    sc = {}
    for n in (1000, 100000):
        a, b = synth.gaussian_cluster_pair(n, n, seed=0)
        sc[f"sha_{n}"] = np.array(hashlib.sha256(a.points.tobytes() + b.points.tobytes()).hexdigest())
    # published in SURVEY.md / BASELINE.md (reference, measured in this container)
    sc["cfg2_L"] = np.array(949.0501340320344)
    sc["cfg2_W1_s1_d001"] = np.array(8776.545620305833)
    sc["cfg3_L"] = np.array(3013.4490112970716)
    np.savez_compressed(os.path.join(HERE, "scalars.npz"), **sc)


if __name__ == "__main__":
    if sys.argv[1:] == ["deep"]:
        deep_cases()
    elif sys.argv[1:] == ["retrieval"]:
        retrieval_cases()
    else:
        main()
