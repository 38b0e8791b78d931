"""Summarise an ncu --set full report (.ncu-rep) into one JSON line per kernel launch:
duration, pipe utilisation, issue / warp activity, DRAM bytes and throughput.

    python tools/ncu_summary.py gpurun_out/r02_cfg5w_top.ncu-rep > profiles/r02_....jsonl
"""
import csv
import io
import json
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
           "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
           "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
           "launch__occupancy_limit_registers", "sm__maximum_warps_per_active_cycle_pct"]

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
ki = hdr.index("Kernel Name")
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    d = {"kernel": r[ki].split("(")[0].replace("w1g::<unnamed>::", "").replace("w1g::", "")}
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            d[m] = f"{r[i]} {units[i]}".strip()
    print(json.dumps(d))
