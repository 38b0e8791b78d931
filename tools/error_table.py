"""cfg5's empirical-error table (BASELINE.json configs[4]): W1 of every
(delta, s) cell at 100k+100k points, and the certified bracket [RWMD L, the
condensation-off (spanner-only) W1] that contains the true W1 (the exact dense
oracle needs 1e10 arcs at this size: unavailable).

    python tools/error_table.py [--jobs J] [--cells d,s d,s ...] > profiles/r02_cfg5_error_table.jsonl

Each cell's network is the front end's network: built here by the C restatement
(oracle/w1oracle.c), which tests/test_gpu_configs.py::test_cfg5_sweep_cell pins
bit for bit to the B200 front end's network for every one of these cells, so the
solve needs no GPU and runs on the host cores while the GPU is busy with other
work.  Each network is solved by the reference's own host simplex (w1flow),
single-threaded, one cell per process.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor, as_completed

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CELLS = [(d, s) for d in (0.1, 0.01, 0.001) for s in (1.0, 4.0, 16.0)]
NO_COND = [1.0, 4.0]  # condensation off (the bracket's upper end)


def solve_cell(delta, s, n=100_000):
    from oracle import w1oracle as O
    from paper_2110_14734_b200 import solver, synth

    a, b = synth.gaussian_cluster_pair(n, n, seed=0)
    t0 = time.perf_counter()
    fe = O.front_end(a, b, s, delta=delta if delta is not None else 0.0, use_condensation=delta is not None)
    t1 = time.perf_counter()
    res = solver.solve(fe.network)
    t2 = time.perf_counter()
    return {"config": "cfg5", "n_each": n, "delta": delta, "s": s, "condensation": delta is not None,
            "w1": res.objective, "status": res.status, "pivots": res.pivots, "lower_bound_L": fe.lower_bound,
            "nodes": int(fe.network.supplies.shape[0]), "arcs": int(fe.network.tails.shape[0]),
            "front_end_s_cpu_port": t1 - t0, "solve_s": t2 - t1, "solver": "reference w1flow.simplex, 1 thread"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=4)
    ap.add_argument("--cells", nargs="*", default=None)
    args = ap.parse_args()
    todo = [(d, s) for d, s in CELLS] + [(None, s) for s in NO_COND]
    if args.cells:
        todo = [(None if d == "off" else float(d), float(s)) for d, s in (c.split(",") for c in args.cells)]
    # the largest networks first: they take longest
    order = sorted(todo, key=lambda c: (c[0] or 0.0, -c[1]))
    with ProcessPoolExecutor(max_workers=args.jobs) as ex:
        futs = {ex.submit(solve_cell, d, s): (d, s) for d, s in order}
        for f in as_completed(futs):
            d, s = futs[f]
            try:
                row = f.result()
            except Exception as exc:  # noqa: BLE001
                row = {"config": "cfg5", "delta": d, "s": s, "error": repr(exc)}
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
