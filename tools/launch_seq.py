"""Print the last N launches of an ncu launch list in order (one front end's kernel sequence)."""
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ki, vi = hdr.index('Kernel Name'), hdr.index('Metric Value')
gi = hdr.index('Grid Size') if 'Grid Size' in hdr else None
data = [(r[ki].split('(')[0].replace('w1g::<unnamed>::', '').replace('w1g::', ''), float(r[vi]), r[gi] if gi is not None else '') for r in rows[1:]]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 120
tot = 0.0
for k, v, g in data[-n:]:
    tot += v
    print(f"{v/1e3:8.1f} us  {g:>14}  {k[:80]}")
print(f"sum of last {n}: {tot/1e3:.1f} us")
