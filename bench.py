"""Benchmark of the sparsify front end (BASELINE.json configs[1], cfg2).

Workload: one synthetic persistence-diagram pair of 100,000 points each
(reference generator, synth.gaussian_cluster_pair(100000, 100000, seed)),
s = 1, delta = 0.01 (fixed, the chain of test_acceptance.py:224-237), k = 0.99.
A step is one full sparsify front end (pipeline.py:105-130: zero_condense ->
rwmd -> delta_condense -> split tree -> WSPD -> emit arcs -> CSR network).

Our arm (default):
  value  -- pairs/s of the front end with the diagrams already in HBM and the
            network left in HBM (w1g_front_end_device), CUDA events on the
            library stream, L2 flushed (256 MiB write) before every step;
  e2e    -- pairs/s through the public API (paper_2110_14734_b200.sparsify):
            host numpy diagrams in (page-locked, w1g.pinned_points), host numpy
            TransshipmentNetwork out, all H2D / D2H copies inside the timed region;
  roofline -- the FP32 all-pairs RWMD tile kernel (w1g_profile_rwmd_tile):
            5 FLOP x 2|A||B| directed evaluations per pair of launches;
  cpu_baseline -- the C restatement of the reference front end (oracle/),
            one bounded sample on rank 0.
  w1     -- one approx_w1 (front end + the reference's host simplex) outside
            the timed loop (rank 0, --w1).
Reference arm (--impl reference): the same front end by the CPU port on the
host cores, rank 0 only.

Multi-GPU (torchrun): every rank runs its own pair (seed = rank): the pairs
workload shards with no collective; scaling is weak.  Timing is the max over
ranks (all-reduce MAX of the per-rank device time).
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
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # 74.4, derived nominal (no FP32 figure in MEASURED_PEAKS.json)
N_POINTS = 100_000
S = 1.0
DELTA = 0.01
NCU_SUMMARY = os.path.join(ROOT, "profiles", "r01_ncu_rwmd_tile.jsonl")


def _ncu_traffic(kernel: str, capture: str = "prof_rwmd_all"):
    """dram__bytes_read.sum + dram__bytes_write.sum of one launch of `kernel` at this workload,
    from the committed `ncu --set full` capture summary (cfg2, same command as this bench)."""
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    try:
        with open(NCU_SUMMARY) as f:
            for line in f:
                row = json.loads(line)
                if row["capture"] == capture and kernel in row["Kernel Name"]:
                    total = 0.0
                    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                        v, u = row[key].split()
                        total += float(v) * scale[u]
                    return int(total)
    except (OSError, KeyError, ValueError):
        pass
    return None


HBM_PEAK_GBS = 6528.7  # MEASURED_PEAKS.json hbm_gbs (copy bandwidth, read + write)


def hbm_stages(n_in: int, k0: int, k: int, p: int, m: int, stage_ms: dict) -> dict:
    """Algorithmic HBM bytes of the byte-moving stages (each stage's inputs read once and
    outputs written once) over their measured device time, against
    the measured copy bandwidth.  emit_arcs is fused into the CSR assembly (the pairs
    and node arrays are read, the network written; no arc list in between)."""
    nn = max(2 * k - 1, 0)
    bytes_ = {
        "zero_condense": 16 * n_in + 32 * k0,
        "delta_condense": 32 * k0 + 32 * k,
        "split_tree": 16 * k + 64 * nn,
        "wspd": 40 * nn + 24 * p,
        "emit_arcs+assemble": 16 * p + 32 * k + 24 * m + 16 * (k + 3),
    }
    out = {}
    for name, b in bytes_.items():
        t = sum(stage_ms.get(x) or 0.0 for x in name.split("+"))
        if not t:
            continue
        gbs = b / (t * 1e-3) / 1e9
        out[name] = {"bytes": int(b), "ms": t, "gbs": gbs, "frac": gbs / HBM_PEAK_GBS}
    return out


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=N_POINTS)
    ap.add_argument("--s", type=float, default=S)
    ap.add_argument("--delta", type=float, default=DELTA)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--w1", dest="w1", action="store_true", default=True)
    ap.add_argument("--no-w1", dest="w1", action="store_false")
    ap.add_argument("--profile-only", action="store_true", help="a few steps, no extras (for ncu)")
    return ap.parse_args()


class Dist:
    """torch.distributed plumbing (barrier, max over ranks); single process if no torchrun."""

    def __init__(self, gpus: int):
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        if self.world > 1:
            import torch
            import torch.distributed as dist

            torch.cuda.set_device(self.local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            self.torch, self.dist = torch, dist
            self.pg = True

    def barrier(self):
        if self.pg:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device="cuda")
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
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
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
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_front_end_sample(a, b, s, delta, repeats: int = 2) -> dict:
    """The C oracle (restatement of the reference front end), rank 0, bounded sample."""
    from oracle import w1oracle as O

    O.lib()
    times = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        O.front_end(a, b, s, delta=delta)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    return {"value": 1.0 / t, "unit": "pairs/s", "cores": 1, "kind": "port",
            "sample": f"{repeats} full cfg2 front ends (one {a.shape[0]}+{b.shape[0]}-point pair each), "
                      f"median {t * 1e3:.1f} ms/pair, scalar C port of the reference (oracle/w1oracle.c)"}


def run_reference(args, dist: Dist):
    if dist.rank != 0:
        return
    from paper_2110_14734_b200 import synth

    a, b = synth.gaussian_cluster_pair(args.n, args.n, seed=0)
    from concurrent.futures import ThreadPoolExecutor

    from oracle import w1oracle as O

    O.lib()
    # every host thread the process may use runs its own front end (the C port
    # releases the GIL): one step = `threads` pairs processed concurrently
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    pool = ThreadPoolExecutor(max_workers=threads)

    def step():
        list(pool.map(lambda _: O.front_end(a, b, args.s, delta=args.delta), range(threads)))

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    pool.shutdown()
    v = threads * args.steps / el
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "pairs/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator)",
        "config": {"workload": f"cfg2: sparsify front end, {args.n}+{args.n} points, s={args.s}, delta={args.delta}",
                   "host_threads": threads},
        "cpu_baseline": {"value": v, "unit": "pairs/s", "cores": threads, "kind": "port",
                         "sample": f"{args.steps} timed steps after {args.warmup} warm-up, each {threads} concurrent "
                                   f"front ends (one per host thread) of the scalar C port"},
        "e2e": {"value": v, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, dist: Dist):
    import paper_2110_14734_b200 as w1g
    from paper_2110_14734_b200 import _lib, synth

    device = dist.local
    ctx = _lib.context(device)
    lib = ctx.lib
    a, b = synth.gaussian_cluster_pair(args.n, args.n, seed=dist.rank)
    params = w1g.ApproxParams(s=args.s, best_effort=True, delta=args.delta)

    # device-resident inputs for the `value` leg (torch is plumbing only: device
    # buffers, the L2 flush and CUDA events on the library's own stream)
    import torch

    torch.cuda.set_device(device)
    stream = torch.cuda.ExternalStream(ctx.stream, device=device)
    da = torch.from_numpy(a).to(f"cuda:{device}")
    db = torch.from_numpy(b).to(f"cuda:{device}")
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{device}")
    torch.cuda.synchronize()
    info = _lib.FrontEndInfo()

    def device_step():
        _lib.check(lib.w1g_front_end_device(ctx.handle, ctypes.c_void_p(da.data_ptr()), a.shape[0],
                                            ctypes.c_void_p(db.data_ptr()), b.shape[0], float(args.s), 1, 1,
                                            float(args.delta), 0.99, ctypes.c_uint64(0), ctypes.byref(info)))

    def flush_l2():
        with torch.cuda.stream(stream):
            flush.fill_(1)

    for _ in range(args.warmup):
        flush_l2()
        device_step()
    torch.cuda.synchronize()
    dist.barrier()
    clocks = Clocks(device)
    clocks.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = _lib.launch_count()
    stage_ms = []
    wall0 = time.perf_counter()
    for i in range(args.steps):
        flush_l2()
        ev[i][0].record(stream)
        device_step()
        ev[i][1].record(stream)
        stage_ms.append([float(x) for x in info.stage_ms])
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    launches = (_lib.launch_count() - launches0) // max(args.steps, 1)
    dev_ms = sum(s.elapsed_time(e) for s, e in ev) / args.steps
    dist.barrier()
    dev_ms_max = dist.max(dev_ms)
    clk = clocks.stop()

    # e2e through the public API (host numpy in, host numpy network out); the
    # inputs live in page-locked host memory (w1g.pinned_points), so every step
    # DMAs them to the device; warm-up also fills the pinned result pool
    a_host, b_host = w1g.pinned_points(a), w1g.pinned_points(b)
    keep = []
    for _ in range(max(3, args.warmup)):
        keep.append(w1g.sparsify(a_host, b_host, params, device=device))
        keep = keep[-2:]
    del keep
    e2e_times = []
    net = None
    for _ in range(args.steps):
        flush_l2()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        net, diag = w1g.sparsify(a_host, b_host, params, device=device)
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = dist.max(statistics.mean(e2e_times))
    h2d = a.nbytes + b.nbytes
    d2h = net.supplies.nbytes + net.tails.nbytes + net.heads.nbytes + net.costs.nbytes + net.row_offsets.nbytes

    # roofline of the dominant kernel: FP32 all-pairs RWMD tile pass (full brute force)
    n0 = w1g.zero_condense(a, b, device=device)
    from paper_2110_14734_b200.diagram import load_nodes

    load_nodes(ctx, _lib.NODES0, n0)
    ctx.call("w1g_set_rwmd_culling", 0)
    ms = ctypes.c_float(0)
    evals = ctypes.c_int64(0)
    ctx.call("w1g_profile_rwmd_tile", 3, ctypes.byref(ms), ctypes.byref(evals))
    ctx.call("w1g_set_rwmd_culling", 1)
    tflops = 5.0 * evals.value / (ms.value * 1e-3) / 1e12
    roofline = {"bound": "fp32", "achieved": tflops, "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": tflops / FP32_PEAK_TFLOPS, "traffic": _ncu_traffic("k_rwmd_f32<8, 0, 1024>"),
                "traffic_unit": "bytes/launch (dram read+write, ncu --set full, profiles/r01_ncu_rwmd_tile.jsonl)",
                "kernel": "k_rwmd_f32 (rwmd_tile.cu)",
                "ms_per_launch": ms.value, "evals_per_launch": evals.value,
                "note": "5 FLOP per directed (source,target) evaluation, full brute force (culling off); "
                        "peak = derived nominal 148 SM x 128 lanes x 2 x 1.965 GHz"}
    stage_names = list(_lib.STAGES)
    stage_avg = {nm: statistics.mean(s[i] for s in stage_ms) for i, nm in enumerate(stage_names)}

    extra = {}
    if dist.rank == 0 and not args.profile_only:
        if not args.no_cpu_baseline:
            extra["cpu_baseline"] = cpu_front_end_sample(a, b, args.s, args.delta)
        if args.w1:
            t0 = time.perf_counter()
            value, d = w1g.approx_w1(a, b, params, device=device)
            t_w1 = time.perf_counter() - t0
            extra["w1"] = {"value": value, "status": d.status, "pivots": d.pivots, "seconds": t_w1,
                           "pairs_per_s": 1.0 / t_w1, "solver": "reference w1flow.simplex (host, 1 thread)"}
    if dist.rank == 0:
        n = dist.world
        hs = hbm_stages(2 * args.n, int(info.n_points0), int(info.n_points), int(info.n_pairs), int(info.n_arcs),
                        stage_avg)
        if hs:
            # the timed step's longest byte-moving stage against HBM (the RWMD tile above is
            # the north star's named kernel; this says where the step's own time goes)
            nm, st = max(hs.items(), key=lambda kv: kv[1]["ms"])
            roofline["step_longest_stage"] = {
                "stage": nm, "bound": "hbm", "achieved": st["gbs"], "peak": HBM_PEAK_GBS, "unit": "GB/s",
                "frac": st["frac"], "ms": st["ms"], "algorithmic_bytes": st["bytes"],
                "note": "latency-bound: dependent grid-wide phases (levels, sorts, round trips), "
                        "not bandwidth; see DESIGN.md section 4"}
        line = {
            "metric": METRIC,
            "value": n / (dev_ms_max * 1e-3),
            "unit": "pairs/s",
            "n_gpus": n,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": dev_ms_max,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (reference generator gaussian_cluster_pair, seed = rank)",
            "config": {"workload": f"cfg2: sparsify front end, {args.n}+{args.n} points, s={args.s}, "
                                   f"delta={args.delta}, k=0.99",
                       "pairs_per_gpu_per_step": 1, "l2": "flushed (256 MiB write) before every step",
                       "nodes": int(info.n_points), "pairs": int(info.n_pairs), "arcs": int(info.n_arcs)},
            "sparsify_ms": dev_ms_max,
            "stage_ms": stage_avg,
            "wall_s": wall,
            "e2e": {"value": n / e2e_s, "unit": "pairs/s", "ms_per_pair": e2e_s * 1e3,
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
            "roofline": roofline,
            "hbm_stages": {"peak_gbs": HBM_PEAK_GBS, "note": "algorithmic bytes / stage device time; "
                           "latency-bound at this size (few-microsecond dependent phases), see DESIGN.md",
                           "stages": hs},
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        line.update(extra)
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    dist = Dist(args.gpus)
    try:
        if args.impl == "reference":
            run_reference(args, dist)
        else:
            run_ours(args, dist)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
