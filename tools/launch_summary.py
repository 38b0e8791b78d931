"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel:
launches, total and mean duration, share of the total.

    python tools/launch_summary.py gpurun_out/launches_cfg2.csv [skip_first_n]
"""
import csv
import sys
from collections import defaultdict

rows = []
with open(sys.argv[1]) as f:
    lines = [ln for ln in f if not ln.startswith("==")]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}[unit]
    name = r["Kernel Name"].split("(")[0].replace("w1g::<unnamed>::", "").replace("w1g::", "")
    rows.append((int(r["ID"]), name, v * scale))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = [x for x in rows if x[0] >= skip]
agg = defaultdict(lambda: [0, 0.0])
for _, nm, us in rows:
    agg[nm][0] += 1
    agg[nm][1] += us
total = sum(v[1] for v in agg.values())
print(f"{len(rows)} launches, {total:.1f} us total (serialised, cold-cache ncu replay)")
for nm, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{us:10.1f} us {100 * us / total:5.1f} %  x{n:<4d} {us / n:9.1f} us/launch  {nm}")
