"""Benchmark of the sparsify front end (BASELINE.json configs[1], cfg2; --workload cfg4 for configs[3]).

Workload (default, cfg2): a fixed batch of PAIRS synthetic persistence-diagram
pairs of 100,000 points each (reference generator,
synth.gaussian_cluster_pair(100000, 100000, seed=p), p = 0..PAIRS-1), s = 1,
delta = 0.01 (fixed, the chain of test_acceptance.py:224-237), k = 0.99.  A step
is the full sparsify front end (pipeline.py:105-130: zero_condense -> rwmd ->
delta_condense -> split tree -> WSPD -> emit arcs -> CSR network) of every pair
of the batch.  Under torchrun every rank runs its own batch of PAIRS pairs (seeds
rank * PAIRS + p): weak scaling -- the pairs are independent, so they shard with no
collective; value = all ranks' pairs / the max-over-ranks time.

Our arm (default):
  value    -- pairs/s of the whole job: the batch with the diagrams already in
              HBM and the networks left in HBM (w1g_front_end_batch: the native
              batch executor, STREAMS child contexts per GPU), device makespan
              from CUDA events on the library stream that every child stream
              joins, L2 flushed (256 MiB write) before every step, max over ranks;
  e2e      -- the same through the public API (paper_2110_14734_b200.sparsify_batch):
              host numpy diagrams in (pageable, as a user passes them), host
              numpy TransshipmentNetworks out, every H2D / D2H copy inside the
              timed region; plus single-pair variants (pinned / pageable input,
              the reference's own delta schedule);
  roofline -- the production RWMD kernels of the step, timed with CUDA events
              on the stream each runs on (w1g_profile_rwmd) with device counters
              of the distance evaluations they perform: the exact fp64 refine
              (FP64 pipe) and the culled FP32 tile pass;
  north_star_kernel -- the FP32 all-pairs tile kernel in full brute-force mode
              at n = 1M (BASELINE.json: "at n=1M, the RWMD kernel reaches >= 70 %
              of FP32 pipe peak"), 5 FLOP x 2|A||B| evaluations;
  cpu_baseline -- the reference itself (w1flow from baseline/_ref, the
              stage chain of pipeline.py:105-130) on one pair, rank 0, at
              workers = all host threads and workers = 1; and the C port.
  cfg4     -- the batched matrix workload (64 diagrams x 20k, 2016 pairs) dealt
              over the ranks, front-end pairs/s (strong scaling).
Reference arm (--impl reference): the reference's own front end (w1flow) on the
host cores, rank 0 only, one pair per step.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sparsify-stage ms & W1 pairs/sec at n=100k; RWMD kernel % of FP32 peak"
N_POINTS = 100_000
S = 1.0
DELTA = 0.01
K_LATTICE = 0.99
PAIRS = 64
STREAMS = 6  # child contexts per GPU for the cfg2 batch (value 2021 vs 1990 with 4, e2e 1142 vs 1118)
CFG4 = (64, 20_000)
CFG4_STREAMS = 4  # the 20k-point pairs are launch-bound: more contexts do not help (3266 vs 3150 with 6)


def _peaks() -> dict:
    """Roofline denominators: HBM from MEASURED_PEAKS.json (driver-measured copy
    bandwidth); FP32 / FP64 pipe peaks derived from the SM count and the max SM
    clock there (MEASURED_PEAKS.json has no FP32/FP64 figure)."""
    mp = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
    except (OSError, ValueError):
        pass
    mhz = float(mp.get("sm_max_mhz", 1965.0))
    return {
        "hbm_gbs": float(mp.get("hbm_gbs", 6553.6)),
        "hbm_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in mp else "B200_PROFILING.md fallback",
        "fp32_tflops": 148 * 128 * 2 * mhz * 1e6 / 1e12,
        "fp64_tflops": 148 * 64 * 2 * mhz * 1e6 / 1e12,
        "fp_source": f"derived nominal: 148 SM x (128 FP32 | 64 FP64 lanes) x 2 x {mhz:.0f} MHz "
                     "(sm_max_mhz of MEASURED_PEAKS.json)",
    }


PEAKS = _peaks()


def _ncu_capture(fname: str, kernel: str) -> dict | None:
    """The committed `ncu --set full` summary of `kernel` for this workload (profiles/,
    tools/ncu_summary.py): DRAM bytes per launch and pipe utilisation.  ncu cannot run
    inside the timed bench, so the capture of the same configuration is read here."""
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    try:
        with open(os.path.join(ROOT, "profiles", fname)) as f:
            for line in f:
                row = json.loads(line)
                if kernel not in row["kernel"]:
                    continue
                out = {"capture": "profiles/" + fname}
                tr = 0.0
                for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    v, u = row[key].split()
                    tr += float(v) * scale[u]
                out["dram_bytes_per_launch"] = int(tr)
                for key, name in (("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_pct"),
                                  ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_pct"),
                                  ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_pct"),
                                  ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct")):
                    if key in row:
                        out[name] = float(row[key].split()[0])
                return out
    except (OSError, KeyError, ValueError, IndexError):
        pass
    return None


def workload_config(args) -> dict:
    if args.workload == "cfg4":
        return {"workload": f"cfg4: sparsify front ends of the {CFG4[0] * (CFG4[0] - 1) // 2} pairs of "
                            f"{CFG4[0]} shared-centre diagrams x {CFG4[1]} points, s={args.s}, delta={args.delta}, "
                            f"k={K_LATTICE}",
                "pairs_per_step": CFG4[0] * (CFG4[0] - 1) // 2, "diagram_points": CFG4[1],
                "l2": "flushed (256 MiB write) before every step"}
    return {"workload": f"cfg2: sparsify front end, {args.n}+{args.n} points per pair, s={args.s}, "
                        f"delta={args.delta}, k={K_LATTICE}",
            "pairs_per_step_per_gpu": args.pairs, "l2": "flushed (256 MiB write) before every step"}


def scaling_of(args) -> str:
    # cfg2: every rank its own batch of independent pairs, no collective (weak scaling: the
    # pairs partition the work); cfg4: one fixed matrix dealt over the ranks (strong)
    return "strong" if args.workload == "cfg4" else "weak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=["cfg2", "cfg4", "cfg3"])
    ap.add_argument("--n", type=int, default=N_POINTS)
    ap.add_argument("--pairs", type=int, default=PAIRS)
    ap.add_argument("--streams", type=int, default=None,
                    help=f"child contexts per GPU (default {STREAMS}; {CFG4_STREAMS} for --workload cfg4)")
    ap.add_argument("--s", type=float, default=S)
    ap.add_argument("--delta", type=float, default=DELTA)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="value / e2e only (profiling runs)")
    ap.add_argument("--w1", dest="w1", action="store_true", default=True)
    ap.add_argument("--no-w1", dest="w1", action="store_false")
    args = ap.parse_args()
    if args.streams is None:
        args.streams = CFG4_STREAMS if args.workload == "cfg4" else STREAMS
    return args


class Dist:
    """torch.distributed plumbing (barrier, max over ranks); single process without torchrun."""

    def __init__(self, gpus: int, backend: str = "nccl"):
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        # W1G_BENCH_SHARE_GPU=1 (checks only, never a bench number): every rank on GPU 0 with a
        # gloo group, to exercise the multi-rank code path where one GPU is available (the
        # ranks' kernels never wait on one another; only host barriers join them)
        if os.environ.get("W1G_BENCH_SHARE_GPU") == "1" and backend:
            self.local = 0
            backend = "gloo"
        if self.world > 1 and backend:
            import torch
            import torch.distributed as dist

            self.torch, self.dist = torch, dist
            if backend == "nccl":
                torch.cuda.set_device(self.local)
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
                self.dev = torch.device("cuda", self.local)
            else:
                dist.init_process_group("gloo")
                self.dev = torch.device("cpu")
            self.pg = True

    def barrier(self):
        if self.pg:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.pg:
            self.dist.destroy_process_group()


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = "index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active," \
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def wait_first(self, timeout: float = 3.0):
        """Block until the sampler produces output (nvidia-smi takes a moment to start),
        so the samples cover the timed region that follows."""
        t0 = time.monotonic()
        while self.proc and not self.lines and time.monotonic() - t0 < timeout:
            time.sleep(0.01)

    def mark(self):
        return time.monotonic()

    def stop(self, window=None) -> dict:
        """Summary of the samples taken inside `window` = (t_start, t_end) (monotonic)."""
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for t, ln in self.lines:
            if window and not (window[0] <= t <= window[1] + 0.06):
                continue
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm), "sample_period_ms": 20,
                "window_s": (window[1] - window[0]) if window else None}


# ---------------------------------------------------------------- inputs

def cfg2_inputs(args, rank: int = 0) -> list[np.ndarray]:
    """Diagrams 2p, 2p+1 = gaussian_cluster_pair(n, n, seed=rank * pairs + p) for every pair p
    of this rank's batch (rank 0: seeds 0..pairs-1)."""
    from paper_2110_14734_b200 import synth

    out = []
    for p in range(args.pairs):
        a, b = synth.gaussian_cluster_pair(args.n, args.n, seed=rank * args.pairs + p)
        out += [a, b]
    return out


def rank_share(pairs: list[tuple[int, int]], rank: int, world: int) -> list[tuple[int, int]]:
    return pairs[rank::world]


# ---------------------------------------------------------------- the reference (CPU) front end

def _reference_modules():
    from paper_2110_14734_b200 import solver

    solver.reference_simplex()  # puts baseline/_ref on sys.path when that is where the reference lives
    import w1flow  # noqa: F401
    from w1flow import condensation, diagram, lower_bound, network, pipeline, spanner
    return condensation, diagram, lower_bound, network, pipeline, spanner


def reference_front_end(a, b, s: float, delta: float, workers: int):
    """pipeline.py:105-130 with the given delta (the fixed-delta chain of
    test_acceptance.py:224-237), run by the reference package itself."""
    condensation, diagram, lower_bound, network, pipeline, spanner = _reference_modules()
    nodes0 = diagram.zero_condense(diagram.PersistenceDiagram(a), diagram.PersistenceDiagram(b))
    lower = lower_bound.rwmd(nodes0, workers=workers)
    nodes = nodes0
    if lower > 0.0 and delta > 0.0:
        nodes = condensation.delta_condense(
            nodes0, condensation.CondensationParams(pipeline.condensation_epsilon(s), delta, k=K_LATTICE))
    pairs = spanner.build_wspd(spanner.build_split_tree(nodes.points), s, workers=workers)
    return network.assemble(nodes, spanner.emit_arcs(pairs, nodes))


def host_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def cpu_baselines(a, b, args) -> dict:
    """The reference's own front end on this host (rank 0, one pair): all host
    threads (the reference's `workers`) and one thread; the C port beside it."""
    out = {}
    threads = host_threads()
    try:
        tiny = np.array([[0.0, 1.0], [0.5, 2.0], [1.0, 1.5]])
        reference_front_end(tiny, tiny[:2] + 0.25, args.s, args.delta, 1)  # numba compilation, untimed
        for w in (threads, 1):
            t0 = time.perf_counter()
            net = reference_front_end(a, b, args.s, args.delta, w)
            el = time.perf_counter() - t0
            out[w] = (el, int(net.tails.shape[0]))
    except Exception as exc:  # noqa: BLE001
        return {"value": None, "unit": "pairs/s", "cores": threads, "kind": "reference",
                "sample": f"reference unavailable: {exc!r}"}
    el, m = out[threads]
    res = {"value": 1.0 / el, "unit": "pairs/s", "cores": threads, "kind": "reference",
           "sample": f"one cfg2 pair (seed 0) through the reference's own stage chain (w1flow from "
                     f"baseline/_ref, pipeline.py:105-130, delta={args.delta}) with workers={threads}: "
                     f"{el:.2f} s; {m} arcs",
           "one_thread": {"value": 1.0 / out[1][0], "cores": 1, "seconds": out[1][0]}}
    try:
        from oracle import w1oracle as O

        O.lib()
        t0 = time.perf_counter()
        O.front_end(a, b, args.s, delta=args.delta)
        el = time.perf_counter() - t0
        res["c_port"] = {"value": 1.0 / el, "cores": 1, "kind": "port", "seconds": el,
                         "note": "scalar C restatement of the reference (oracle/w1oracle.c)"}
    except Exception as exc:  # noqa: BLE001
        res["c_port"] = {"value": None, "note": repr(exc)}
    return res


def run_reference(args, dist: Dist):
    if dist.rank != 0:
        return
    from paper_2110_14734_b200 import synth

    threads = host_threads()
    if args.workload == "cfg4":
        diags = synth.shared_centre_batch(*CFG4, seed=0)
        todo = [(i, j) for i in range(CFG4[0]) for j in range(i + 1, CFG4[0])]
        inputs = [(diags[i], diags[j]) for i, j in todo[:: max(1, len(todo) // 64)]]
    else:
        inputs = [synth.gaussian_cluster_pair(args.n, args.n, seed=p) for p in range(min(args.pairs, 4))]
    tiny = np.array([[0.0, 1.0], [0.5, 2.0], [1.0, 1.5]])
    reference_front_end(tiny, tiny[:2] + 0.25, args.s, args.delta, 1)  # numba compilation
    for i in range(args.warmup):
        reference_front_end(*inputs[i % len(inputs)], args.s, args.delta, threads)
    t0 = time.perf_counter()
    for i in range(args.steps):
        reference_front_end(*inputs[i % len(inputs)], args.s, args.delta, threads)
    el = time.perf_counter() - t0
    v = args.steps / el
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "pairs/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
        "higher_is_better": True, "scaling": scaling_of(args), "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator)", "config": workload_config(args),
        "cpu_baseline": {"value": v, "unit": "pairs/s", "cores": threads, "kind": "reference",
                         "sample": f"{args.steps} timed steps after {args.warmup} warm-up; each step one pair "
                                   f"of the workload through the reference's own front end (w1flow from "
                                   f"baseline/_ref, pipeline.py:105-130) with workers={threads}"},
        "e2e": {"value": v, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm

class Batch:
    """Device-resident batch of pairs on this rank's GPU (w1g_front_end_batch)."""

    def __init__(self, ctx, diagrams, pairs, args):
        from paper_2110_14734_b200 import _lib
        from paper_2110_14734_b200.lower_bound import load_corpus

        self.ctx = ctx
        self.lib = ctx.lib
        load_corpus(diagrams, ctx.device)
        self.pairs = np.ascontiguousarray(np.asarray(pairs, dtype=np.int32).reshape(-1, 2))
        self.infos = (_lib.FrontEndInfo * max(1, len(pairs)))()
        self.args = args

    def run(self) -> float:
        from paper_2110_14734_b200 import _lib

        ms = ctypes.c_float(0)
        if self.pairs.shape[0]:
            _lib.check(self.lib.w1g_front_end_batch(
                self.ctx.handle, self.pairs.ctypes.data, self.pairs.shape[0], float(self.args.s), 1, 1,
                float(self.args.delta), K_LATTICE, ctypes.c_uint64(0), int(self.args.streams), self.infos,
                ctypes.byref(ms)))
        return ms.value


def time_batch(batch: Batch, steps: int, warmup: int, flush, dist: Dist, clocks=None):
    from paper_2110_14734_b200 import _lib

    for _ in range(warmup):
        flush()
        batch.run()
    if clocks:
        clocks.start()
        clocks.wait_first()
    dist.barrier()
    t_start = time.monotonic()
    launches0 = _lib.launch_count()
    times = []
    for _ in range(steps):
        flush()  # ordered on the library stream before the batch's start event
        times.append(batch.run())
    launches = (_lib.launch_count() - launches0) // max(steps, 1)
    clk = clocks.stop((t_start, time.monotonic())) if clocks else None
    dist.barrier()
    return dist.max(statistics.mean(times)), launches, clk


def rwmd_roofline(ctx, w1g, a, b) -> dict:
    """The production RWMD kernels (culled FP32 tile + exact fp64 refine, both
    sides) on one cfg2 pair: per-launch device time from CUDA events on the stream
    each kernel runs on, work = the (source, target) distance evaluations each
    performs x 5 FLOP (2 sub, 2 mul, 1 add), against the FP64 / FP32 pipe peaks."""
    from paper_2110_14734_b200 import _lib
    from paper_2110_14734_b200.diagram import load_nodes

    n0 = w1g.zero_condense(a, b, device=ctx.device)
    load_nodes(ctx, _lib.NODES0, n0)
    ms = (ctypes.c_float * 4)()
    ev = (ctypes.c_int64 * 4)()
    directed = ctypes.c_int64(0)
    ctx.call("w1g_profile_rwmd", 1, ms, ev, ctypes.byref(directed))  # warm
    ctx.call("w1g_profile_rwmd", 5, ms, ev, ctypes.byref(directed))
    names = ["tile_a", "refine_a", "tile_b", "refine_b"]
    per = {nm: {"ms": float(ms[i]), "evals": int(ev[i])} for i, nm in enumerate(names)}
    ref_ms = (ms[1] + ms[3]) / 2
    ref_ev = (ev[1] + ev[3]) / 2
    tile_ms = (ms[0] + ms[2]) / 2
    tile_ev = (ev[0] + ev[2]) / 2
    f64 = 5.0 * ref_ev / (ref_ms * 1e-3) / 1e12 if ref_ms else 0.0
    f32 = 5.0 * tile_ev / (tile_ms * 1e-3) / 1e12 if tile_ms else 0.0
    total = sum(ms[i] for i in range(4))
    ncu_ref = _ncu_capture("r02c_ncu_cfg2_rwmd.jsonl", "k_refine")
    ncu_tile = _ncu_capture("r02c_ncu_cfg2_rwmd.jsonl", "k_rwmd_f32")
    return {
        "bound": "fp64", "kernel": "k_refine (rwmd.cu): exact fp64 nearest-neighbour refine, the production RWMD",
        "achieved": f64, "peak": PEAKS["fp64_tflops"], "unit": "TFLOP/s", "frac": f64 / PEAKS["fp64_tflops"],
        "traffic": ncu_ref["dram_bytes_per_launch"] if ncu_ref else None,
        "ncu": ncu_ref,
        "ms_per_launch": ref_ms, "flop_per_launch": 5.0 * ref_ev, "evals_per_launch": ref_ev,
        "note": "achieved = 5 FLOP x the distance evaluations the launch performs (device counter) / its "
                "event-timed duration; peak " + PEAKS["fp_source"],
        "tile": {"bound": "fp32", "kernel": "k_rwmd_f32<R,1,256> (rwmd_tile.cu): culled FP32 seed pass, R = 1 source per thread below "
                           "300k sources",
                 "achieved": f32, "peak": PEAKS["fp32_tflops"], "unit": "TFLOP/s",
                 "frac": f32 / PEAKS["fp32_tflops"], "ms_per_launch": tile_ms, "evals_per_launch": tile_ev,
                 "ncu": ncu_tile},
        "per_kernel": per,
        "rwmd_algorithmic": {
            "directed_evals": int(directed.value),
            "kernel_ms_both_sides": total,
            "brute_force_equivalent_tflops": 5.0 * directed.value / (total * 1e-3) / 1e12 if total else None,
            "evals_performed_frac": (sum(ev[i] for i in range(4)) / directed.value) if directed.value else None,
            "note": "W = 2|A||B| directed evaluations (SURVEY 8d); culling performs the fraction above"},
    }


def north_star_kernel(ctx, w1g, n: int) -> dict:
    """FP32 all-pairs tile kernel, full brute force, at n points per side."""
    from paper_2110_14734_b200 import _lib, synth
    from paper_2110_14734_b200.diagram import load_nodes

    a, b = synth.gaussian_cluster_pair(n, n, seed=0)
    n0 = w1g.zero_condense(a, b, device=ctx.device)
    load_nodes(ctx, _lib.NODES0, n0)
    ctx.call("w1g_set_rwmd_culling", 0)
    ms = ctypes.c_float(0)
    evals = ctypes.c_int64(0)
    try:
        ctx.call("w1g_profile_rwmd_tile", 1, ctypes.byref(ms), ctypes.byref(evals))
        ctx.call("w1g_profile_rwmd_tile", 2, ctypes.byref(ms), ctypes.byref(evals))
    finally:
        ctx.call("w1g_set_rwmd_culling", 1)
    tflops = 5.0 * evals.value / (ms.value * 1e-3) / 1e12
    return {"bound": "fp32", "kernel": "k_rwmd_f32<8,0,1024,1> (rwmd_tile.cu), culling off, two sources packed per FP32x2 lane pair",
            "config": f"{n}+{n} points (gaussian_cluster_pair seed 0)", "achieved": tflops,
            "peak": PEAKS["fp32_tflops"], "unit": "TFLOP/s", "frac": tflops / PEAKS["fp32_tflops"],
            "ms_per_launch": ms.value, "evals_per_launch": evals.value,
            "traffic": (_ncu_capture("r02c_ncu_brute_1m.jsonl", "k_rwmd_f32") or {}).get("dram_bytes_per_launch"),
            "ncu": _ncu_capture("r02c_ncu_brute_1m.jsonl", "k_rwmd_f32"),
            "note": "5 FLOP per directed (source, target) evaluation (4 FMA FLOP executed: 2 FFMA per evaluation)"}


def e2e_batch(w1g, diagrams, pairs, args, dist: Dist, reps: int) -> dict:
    """sparsify_batch with host numpy in and host networks out, max over ranks."""
    params = w1g.ApproxParams(s=args.s, best_effort=True, delta=args.delta, k=K_LATTICE)
    nbytes = {"d2h": 0, "net": 0}
    lock = threading.Lock()
    # the batch executor's compact transfer (batch.cu) does not copy the tails (rebuilt on the
    # host from the row offsets) and copies the heads as int32: the bytes that cross the link
    compact = os.environ.get("W1G_BATCH_COMPACT", "1") != "0"

    def keep(i, j, net, d):
        with lock:
            nbytes["net"] += sum(getattr(net, f).nbytes for f in ("supplies", "tails", "heads", "costs",
                                                                  "row_offsets"))
            nbytes["d2h"] += sum(getattr(net, f).nbytes for f in ("supplies", "costs", "row_offsets")) + (
                net.heads.nbytes // 2 if compact else net.heads.nbytes + net.tails.nbytes)

    used = sorted({i for p in pairs for i in p})
    h2d = sum(diagrams[i].nbytes for i in used)
    w1g.sparsify_batch(diagrams, params, pairs=pairs, devices=[dist.local], streams_per_device=args.streams,
                       on_network=keep)  # warm (pool blocks, child contexts)
    dist.barrier()
    times = []
    for _ in range(reps):
        nbytes["d2h"] = nbytes["net"] = 0
        t0 = time.perf_counter()
        w1g.sparsify_batch(diagrams, params, pairs=pairs, devices=[dist.local], streams_per_device=args.streams,
                           on_network=keep)
        times.append(time.perf_counter() - t0)
    dist.barrier()
    t = dist.max(statistics.mean(times))
    return {"seconds": t, "h2d": int(h2d), "d2h": int(nbytes["d2h"]), "net_bytes": int(nbytes["net"]),
            "compact": compact, "reps_ms": [round(1e3 * x, 2) for x in times]}


def e2e_single(w1g, a, b, args, device: int, flush, reps: int) -> dict:
    """One pair through sparsify(): pinned input, pageable input, and the reference's
    own delta schedule (delta derived from L with a host read of L)."""
    import torch

    out = {}
    cases = {
        "pinned_input": (w1g.pinned_points(a), w1g.pinned_points(b),
                         w1g.ApproxParams(s=args.s, best_effort=True, delta=args.delta)),
        "pageable_input": (a, b, w1g.ApproxParams(s=args.s, best_effort=True, delta=args.delta)),
        "auto_delta": (a, b, w1g.ApproxParams(s=args.s, best_effort=True)),
    }
    for name, (x, y, params) in cases.items():
        keep = []
        for _ in range(3):
            keep.append(w1g.sparsify(x, y, params, device=device))
            keep = keep[-2:]
        del keep
        ts = []
        net = diag = None
        for _ in range(reps):
            flush()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            net, diag = w1g.sparsify(x, y, params, device=device)
            ts.append(time.perf_counter() - t0)
        t = statistics.median(ts)
        d2h = sum(getattr(net, f).nbytes for f in ("supplies", "tails", "heads", "costs", "row_offsets"))
        out[name] = {"value": 1.0 / t, "unit": "pairs/s", "ms_per_pair": 1e3 * t,
                     "h2d_bytes_per_step": int(a.nbytes + b.nbytes), "d2h_bytes_per_step": int(d2h),
                     "delta": diag.delta, "device_ms": diag.stage_ms.get("total")}
    return out


def run_sharded(args, dist: Dist):
    """--workload cfg3: ONE 1M+1M pair, its front end sharded over the ranks
    (distributed.sparsify_sharded: replicated condensing and tree, RWMD rows along
    numpy's summation tree with one all-gather, WSPD owners by rank, arc slices
    gathered on rank 0 with grouped NCCL send/recv).  Wall time of each step with a
    device synchronisation on both sides and a barrier, max over ranks (the step has
    host round trips and collectives; no single stream brackets it)."""
    import torch

    from paper_2110_14734_b200 import ApproxParams, synth
    from paper_2110_14734_b200.distributed import sparsify_sharded

    device = dist.local
    torch.cuda.set_device(device)
    n = args.n if args.n != N_POINTS else 1_000_000
    import paper_2110_14734_b200 as w1g

    a, b = synth.gaussian_cluster_pair(n, n, seed=0)
    a, b = w1g.pinned_points(a), w1g.pinned_points(b)  # page-locked: the 32 MB upload is one DMA
    params = ApproxParams(s=args.s, best_effort=True, delta=args.delta)
    for _ in range(max(3, args.warmup)):
        sparsify_sharded(a, b, params, dist.rank, dist.world, device=device)
    ts = []
    net = None
    for _ in range(args.steps):
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        net, diag = sparsify_sharded(a, b, params, dist.rank, dist.world, device=device)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    t = dist.max(statistics.mean(ts))
    if dist.rank != 0:
        return
    d2h = sum(getattr(net, f).nbytes for f in ("supplies", "tails", "heads", "costs", "row_offsets"))
    print(json.dumps({
        "metric": METRIC, "value": 1.0 / t, "unit": "pairs/s", "n_gpus": dist.world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": 1e3 * t, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (the reference generator)",
        "config": {"workload": f"cfg3: one {n}+{n}-point pair, front end sharded over {dist.world} rank(s), "
                               f"s={args.s}, delta={args.delta}", "pairs_per_step": 1},
        "e2e": {"value": 1.0 / t, "unit": "pairs/s", "h2d_bytes_per_step": int(a.nbytes + b.nbytes),
                "d2h_bytes_per_step": int(d2h), "api": "paper_2110_14734_b200.distributed.sparsify_sharded"},
        "timing": "wall clock per step between device synchronisations and a barrier, max over ranks",
        "lower_bound": diag.lower_bound, "arcs": int(net.tails.shape[0]), "gpu_launches": None,
        "roofline": None}), flush=True)


def run_ours(args, dist: Dist):
    import torch

    import paper_2110_14734_b200 as w1g
    from paper_2110_14734_b200 import _lib, synth

    device = dist.local
    torch.cuda.set_device(device)
    ctx = _lib.context(device)
    stream = torch.cuda.ExternalStream(ctx.stream, device=device)
    flush_buf = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{device}")

    def flush():
        with torch.cuda.stream(stream):
            flush_buf.fill_(1)

    if args.workload == "cfg4":
        diagrams = synth.shared_centre_batch(*CFG4, seed=0)
        all_pairs = [(i, j) for i in range(CFG4[0]) for j in range(i + 1, CFG4[0])]
    else:
        diagrams = cfg2_inputs(args, dist.rank)
        all_pairs = [(2 * p, 2 * p + 1) for p in range(args.pairs)]
    # cfg2: each rank runs its own batch (weak scaling); cfg4: the matrix dealt over the ranks
    mine = rank_share(all_pairs, dist.rank, dist.world) if args.workload == "cfg4" else all_pairs
    batch = Batch(ctx, diagrams, mine, args)
    clocks = Clocks(device)
    step_ms, launches, clk = time_batch(batch, args.steps, max(3, args.warmup), flush, dist, clocks)
    infos = [batch.infos[i] for i in range(len(mine))]
    e2e = e2e_batch(w1g, diagrams, mine, args, dist, reps=max(2, min(5, args.steps // 4)))

    extra = {}
    if not args.no_extras:
        a, b = diagrams[0], diagrams[1]
        # single-pair latency on the device (the stage split of one front end)
        single = Batch(ctx, [a, b], [(0, 1)], args)
        single.args = argparse.Namespace(**{**vars(args), "streams": 1})
        one_ms, _, _ = time_batch(single, max(5, args.steps), 3, flush, _NoDist())
        extra["single_pair"] = {"device_ms": one_ms, "stage_ms": {nm: float(single.infos[0].stage_ms[i])
                                                                 for i, nm in enumerate(_lib.STAGES)},
                                "nodes": int(single.infos[0].n_points), "pairs": int(single.infos[0].n_pairs),
                                "arcs": int(single.infos[0].n_arcs)}
        extra["e2e_single_pair"] = e2e_single(w1g, a, b, args, device, flush, reps=max(5, args.steps))
        if args.workload == "cfg2":
            extra["roofline"] = rwmd_roofline(ctx, w1g, a, b)
            if dist.rank == 0:
                extra["north_star_kernel"] = north_star_kernel(ctx, w1g, 1_000_000)
            # the cfg4 matrix over the same ranks (strong scaling of the batched workload)
            c4 = synth.shared_centre_batch(*CFG4, seed=0)
            p4 = [(i, j) for i in range(CFG4[0]) for j in range(i + 1, CFG4[0])]
            b4 = Batch(ctx, c4, rank_share(p4, dist.rank, dist.world),
                       argparse.Namespace(**{**vars(args), "streams": CFG4_STREAMS}))
            ms4, _, _ = time_batch(b4, 2, 1, flush, dist)
            extra["cfg4"] = {"workload": f"{len(p4)} pairs of {CFG4[0]} shared-centre diagrams x {CFG4[1]} points, "
                                         f"s={args.s}, delta={args.delta}, dealt round-robin over {dist.world} GPU(s)",
                             "value": len(p4) / (ms4 * 1e-3), "unit": "pairs/s", "ms_per_step": ms4,
                             "scaling": "strong", "streams_per_gpu": CFG4_STREAMS}
        if dist.rank == 0 and not args.no_cpu_baseline:
            extra["cpu_baseline"] = cpu_baselines(a, b, args)
        if dist.rank == 0 and args.w1 and args.workload == "cfg2":
            params = w1g.ApproxParams(s=args.s, best_effort=True, delta=args.delta)
            t0 = time.perf_counter()
            value, d = w1g.approx_w1(a, b, params, device=device)
            t_w1 = time.perf_counter() - t0
            extra["w1"] = {"value": value, "status": d.status, "pivots": d.pivots, "seconds": t_w1,
                           "solver": "reference w1flow.simplex (host, 1 thread)"}
            # W1 pairs/s end to end on the batched matrix: front ends on the GPU, the networks
            # handed (page-locked, zero-copy) to a pool of host solver threads
            c4 = synth.shared_centre_batch(*CFG4, seed=0)
            sub = [(i, j) for i in range(CFG4[0]) for j in range(i + 1, CFG4[0])][:48]
            threads = max(1, host_threads() - 2)
            t0 = time.perf_counter()
            m = w1g.pairwise_w1(c4, params, devices=[device], pairs=sub, solver_threads=threads)
            t_m = time.perf_counter() - t0
            extra["w1_pairs"] = {"value": len(sub) / t_m, "unit": "W1 pairs/s", "pairs": len(sub),
                                 "seconds": t_m, "solver_threads": threads,
                                 "workload": f"{len(sub)} pairs of the cfg4 batch (64 x {CFG4[1]} points), "
                                             "approx_w1 end to end (GPU front end + reference host simplex)",
                                 "finite": bool(np.isfinite([m[i, j] for i, j in sub]).all())}
    if dist.rank != 0:
        return
    total_pairs = len(all_pairs) * (1 if args.workload == "cfg4" else dist.world)
    cfg = workload_config(args)  # identical to the reference arm's
    batch_info = {"streams_per_gpu": args.streams, "pairs_per_gpu": len(mine),
                  "nodes_pair0": int(infos[0].n_points) if infos else 0,
                  "tree_pairs_pair0": int(infos[0].n_pairs) if infos else 0,
                  "arcs_pair0": int(infos[0].n_arcs) if infos else 0}
    line = {
        "metric": METRIC,
        "value": total_pairs / (step_ms * 1e-3),
        "unit": "pairs/s",
        "n_gpus": dist.world,
        "steps": args.steps,
        "warmup": max(3, args.warmup),
        "ms_per_step": step_ms,
        "higher_is_better": True,
        "scaling": scaling_of(args),
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (the reference generator, restated draw for draw in synth.py)",
        "config": cfg,
        "batch": batch_info,
        "e2e": {"value": total_pairs / e2e["seconds"], "unit": "pairs/s", "ms_per_step": 1e3 * e2e["seconds"],
                "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"], "reps_ms": e2e["reps_ms"],
                "network_bytes_per_step": e2e["net_bytes"],
                "transfer": ("compact: tails rebuilt on the host from the row offsets, heads as int32 widened on the "
                             "host (batch.cu expanders)") if e2e["compact"] else "every network array copied",
                "api": "paper_2110_14734_b200.sparsify_batch (host numpy diagrams -> host TransshipmentNetworks)"},
        "gpu_launches": int(launches),
        "clocks": clk,
        "peaks": PEAKS,
    }
    if "roofline" not in extra:
        line["roofline"] = None
    line.update(extra)
    print(json.dumps(line), flush=True)


class _NoDist:
    """Single-rank stand-in (per-rank measurements that need no barrier)."""

    def barrier(self):
        pass

    def max(self, x):
        return x


def main():
    args = parse()
    # the reference arm runs on rank 0 alone: no process group (other ranks exit at once)
    dist = Dist(args.gpus, None if args.impl == "reference" else "nccl")
    try:
        if args.impl == "reference":
            run_reference(args, dist)
        elif args.workload == "cfg3":
            run_sharded(args, dist)
        else:
            run_ours(args, dist)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
