"""Measurements for the BASELINE configs other than the bench default (cfg2).

  python tools/report_configs.py cfg1   # 1k pair: W1 vs the exact dense oracle (empirical error)
  python tools/report_configs.py cfg3   # 1M pair: front end + RWMD tile kernel roofline at n=1M
  python tools/report_configs.py cfg4   # 64 x 20k shared-centre diagrams: 2016-pair sparsify throughput
  python tools/report_configs.py cfg5   # delta x s sweep at 100k+100k: nodes, pairs, arcs, time, parity

Every line printed is one JSON object; results are device-timed with CUDA
events on the library stream (front-end stage_ms) or wall-clock for the
host-side pieces, as labelled.
"""

from __future__ import annotations

import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2110_14734_b200 as w1g  # noqa: E402
from paper_2110_14734_b200 import _lib, synth  # noqa: E402
from paper_2110_14734_b200.diagram import load_nodes  # noqa: E402

FP32_PEAK = 148 * 128 * 2 * 1.965e9 / 1e12


def emit(d):
    print(json.dumps(d), flush=True)


def front_end(a, b, s, delta, reps=3):
    params = w1g.ApproxParams(s=s, best_effort=True, delta=delta)
    ctx = _lib.context()
    from paper_2110_14734_b200.pipeline import _front_end

    infos = []
    for _ in range(reps + 1):
        infos.append(_front_end(ctx, a, b, params))
    inf = infos[1:]
    ms = sorted(i.stage_ms[7] for i in inf)[len(inf) // 2]
    stages = {n: float(np.median([i.stage_ms[k] for i in inf])) for k, n in enumerate(_lib.STAGES)}
    i = inf[-1]
    return ms, stages, i


def tile_roofline(a, b):
    ctx = _lib.context()
    n0 = w1g.zero_condense(a, b)
    load_nodes(ctx, _lib.NODES0, n0)
    ctx.call("w1g_set_rwmd_culling", 0)
    ms, ev = ctypes.c_float(), ctypes.c_int64()
    ctx.call("w1g_profile_rwmd_tile", 2, ctypes.byref(ms), ctypes.byref(ev))
    ctx.call("w1g_set_rwmd_culling", 1)
    tf = 5.0 * ev.value / (ms.value * 1e-3) / 1e12
    return {"kernel": "k_rwmd_f32 full brute force", "ms_per_launch": ms.value, "evals_per_launch": ev.value,
            "tflops_5flop": tf, "frac_nominal_fp32": tf / FP32_PEAK}


def cfg1():
    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    from w1flow import oracle as ref_oracle
    from w1flow.diagram import PersistenceDiagram

    a, b = synth.gaussian_cluster_pair(1000, 1000, seed=0)
    t0 = time.perf_counter()
    exact = w1g.exact_w1_dense(a, b)  # the dense network built on the B200, the reference simplex
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    exact_ref = ref_oracle.exact_w1_dense(PersistenceDiagram(a), PersistenceDiagram(b))
    t_ref = time.perf_counter() - t0
    emit({"config": "cfg1", "exact_w1_dense": exact, "reference_exact_w1_dense": exact_ref,
          "rel_diff": abs(exact - exact_ref) / exact_ref, "seconds_dropin": t_gpu, "seconds_reference": t_ref})
    for s, delta in ((1.0, 0.01), (1.0, None), (12.0, None), (40.0, None)):
        params = w1g.ApproxParams(s=s, best_effort=True, delta=delta)
        w1g.sparsify(a, b, params)  # warm: device buffers sized for this s (first-use allocations)
        v, d = w1g.approx_w1(a, b, params)
        emit({"config": "cfg1", "s": s, "delta": d.delta, "w1": v, "exact_w1": exact,
              "empirical_rel_error": (v - exact) / exact, "arcs": d.n_arcs, "status": d.status,
              "front_end_ms": d.stage_ms.get("total")})


def cfg3():
    a, b = synth.gaussian_cluster_pair(1_000_000, 1_000_000, seed=0)
    ms, stages, i = front_end(a, b, 1.0, 0.01, reps=6)
    sc = np.load(os.path.join(ROOT, "tests", "golden", "scalars.npz"))
    emit({"config": "cfg3", "n_each": 1_000_000, "front_end_ms": ms, "stage_ms": stages,
          "lower_bound": i.lower_bound, "reference_lower_bound": float(sc["cfg3_L"]),
          "lower_bound_bit_exact": i.lower_bound == float(sc["cfg3_L"]),
          "nodes": i.n_points, "pairs": i.n_pairs, "arcs": i.n_arcs})
    import bench

    emit({"config": "cfg3", "hbm_stages": bench.hbm_stages(2_000_000, i.n_points0, i.n_points, i.n_pairs,
                                                          i.n_arcs, stages)})
    emit({"config": "cfg3", "roofline": tile_roofline(a, b)})
    params = w1g.ApproxParams(s=1.0, best_effort=True, delta=0.01)
    ap, bp = w1g.pinned_points(a), w1g.pinned_points(b)
    w1g.sparsify(ap, bp, params)  # warm: sizes the pinned output target
    times = []
    for it in range(5):
        if it:
            del net  # its page-locked block returns to the pool for the next call
        t0 = time.perf_counter()
        net, d = w1g.sparsify(ap, bp, params)
        times.append(1e3 * (time.perf_counter() - t0))
    emit({"config": "cfg3", "e2e_ms": float(np.median(times)), "e2e_ms_samples": times,
          "arcs": d.n_arcs, "inputs": "page-locked (w1g.pinned_points)"})
    if "--oracle" in sys.argv:
        from oracle import w1oracle as O

        t0 = time.perf_counter()
        fe = O.front_end(a, b, 1.0, delta=0.01)
        t1 = time.perf_counter()
        same = all(getattr(net, f).tobytes() == getattr(fe.network, f).tobytes()
                   for f in ("supplies", "tails", "heads", "costs", "row_offsets"))
        emit({"config": "cfg3", "oracle_front_end_s": t1 - t0, "network_bit_exact_vs_oracle": same})


def cfg4():
    diags = synth.shared_centre_batch(64, 20_000, seed=0)
    params = w1g.ApproxParams(s=1.0, best_effort=True, delta=0.01)
    pairs = [(i, j) for i in range(64) for j in range(i + 1, 64)]
    for i, j in pairs[:3]:
        w1g.sparsify(diags[i], diags[j], params)
    for spd in (1, 2, 3, 4):
        w1g.sparsify_batch(diags, params, pairs=pairs[: 4 * spd], streams_per_device=spd)  # warm contexts
        arcs = [0]
        lock = __import__("threading").Lock()

        def count(i, j, net, d):
            with lock:
                arcs[0] += net.arc_count

        t0 = time.perf_counter()
        w1g.sparsify_batch(diags, params, pairs=pairs, streams_per_device=spd, on_network=count)
        el = time.perf_counter() - t0
        emit({"config": "cfg4", "pairs": len(pairs), "streams_per_device": spd, "sparsify_e2e_s": el,
              "pairs_per_s": len(pairs) / el, "mean_arcs": arcs[0] / len(pairs), "n_gpus": 1})
    t0 = time.perf_counter()
    sub = pairs[:4]
    vals = [w1g.approx_w1(diags[i], diags[j], params)[0] for i, j in sub]
    el = time.perf_counter() - t0
    emit({"config": "cfg4", "w1_pairs": len(sub), "w1_s": el, "w1_pairs_per_s_1_solver_thread": len(sub) / el,
          "w1": vals})


def cfg5():
    from oracle import w1oracle as O

    a, b = synth.gaussian_cluster_pair(100_000, 100_000, seed=0)
    for delta in (0.001, 0.01, 0.1):
        for s in (1.0, 4.0, 16.0):
            ms, stages, i = front_end(a, b, s, delta, reps=2)
            row = {"config": "cfg5", "delta": delta, "s": s, "front_end_ms": ms, "stage_ms": stages,
                   "nodes": i.n_points, "pairs": i.n_pairs, "arcs": i.n_arcs, "lower_bound": i.lower_bound}
            if "--oracle" in sys.argv and not (delta == 0.001 and s == 16.0):
                net, _ = w1g.sparsify(a, b, w1g.ApproxParams(s=s, best_effort=True, delta=delta))
                t0 = time.perf_counter()
                fe = O.front_end(a, b, s, delta=delta)
                row["oracle_front_end_s"] = time.perf_counter() - t0
                row["network_bit_exact_vs_oracle"] = all(
                    getattr(net, f).tobytes() == getattr(fe.network, f).tobytes()
                    for f in ("supplies", "tails", "heads", "costs", "row_offsets"))
            emit(row)
    # W1 through the host solver last: its worker threads would otherwise share
    # the host with the next front end's launches and round trips
    for s in (1.0, 4.0, 16.0):
        v, d = w1g.approx_w1(a, b, w1g.ApproxParams(s=s, best_effort=True, delta=0.1))
        emit({"config": "cfg5", "delta": 0.1, "s": s, "w1": v, "w1_status": d.status,
              "bracket_lower": d.lower_bound})


if __name__ == "__main__":
    {"cfg1": cfg1, "cfg3": cfg3, "cfg4": cfg4, "cfg5": cfg5}[sys.argv[1]]()
