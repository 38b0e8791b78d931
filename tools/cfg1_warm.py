import sys; sys.path.insert(0,'.')
import paper_2110_14734_b200 as w1g
from paper_2110_14734_b200 import synth
a,b=synth.gaussian_cluster_pair(1000,1000,seed=0)
for s in (1.0, 12.0, 40.0):
    for rep in range(3):
        net,d=w1g.sparsify(a,b,w1g.ApproxParams(s=s,best_effort=True))
        print(s, rep, round(d.stage_ms['total'],3), {k:round(v,3) for k,v in d.stage_ms.items()}, d.n_arcs, d.n_pairs)
