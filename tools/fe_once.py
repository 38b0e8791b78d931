"""One warm fused front end at a given size (for ncu launch lists: ncu -s skips the warm-up).

    python tools/fe_once.py N S DELTA [REPEATS]
"""
import sys

sys.path.insert(0, ".")
import paper_2110_14734_b200 as w1g  # noqa: E402
from paper_2110_14734_b200 import _lib, synth  # noqa: E402
from paper_2110_14734_b200.pipeline import _front_end  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
s = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
delta = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
a, b = synth.gaussian_cluster_pair(n, n, seed=0)
p = w1g.ApproxParams(s=s, best_effort=True, delta=delta)
ctx = _lib.context()
_front_end(ctx, a, b, p)  # warm
c0 = _lib.launch_count()
tot = []
for _ in range(reps):
    info = _front_end(ctx, a, b, p)
    tot.append(float(info.stage_ms[7]))
c1 = _lib.launch_count()
tot.sort()
print(f"n={n} s={s} delta={delta}: launches per front end {(c1 - c0) // reps}, device ms {info.stage_ms[7]:.3f} "
      f"(min {tot[0]:.3f}, median {tot[len(tot) // 2]:.3f} of {reps}), "
      f"K={info.n_points} P={info.n_pairs} M={info.n_arcs} wspd_levels={info.n_levels_wspd}")
if reps > 1:
    print("device ms, sorted:", [round(x, 3) for x in tot])
print({nm: round(float(info.stage_ms[i]), 4) for i, nm in enumerate(_lib.STAGES)})
