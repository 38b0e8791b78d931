"""Summarise an ncu launch list (gpu__time_duration.sum per launch)."""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ki, vi = hdr.index('Kernel Name'), hdr.index('Metric Value')
data = [(r[ki].split('(')[0].replace('w1g::<unnamed>::', '').replace('w1g::', ''), float(r[vi])) for r in rows[1:]]
agg = collections.defaultdict(lambda: [0, 0.0])
for k, v in data:
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(v for _, v in data)
print(f"launches={len(data)} total_kernel_ms={tot/1e6:.3f} (cold-cache, serialised: compare shares)")
print(f"{'ms':>9} {'share':>6} {'n':>5} {'us/launch':>9}  kernel")
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{v/1e6:9.3f} {100*v/tot:5.1f}% {n:5d} {v/1e3/n:9.1f}  {k[:90]}")
