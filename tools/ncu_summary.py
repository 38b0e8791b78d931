"""Summarise an ncu --set full report (.ncu-rep) into one JSON line per kernel launch."""
import csv, io, json, subprocess, sys

METRICS = ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__grid_size", "launch__registers_per_thread"]

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
