import sys, time; sys.path.insert(0,'.')
import paper_2110_14734_b200 as w1g
from paper_2110_14734_b200 import synth
a,b=synth.gaussian_cluster_pair(1000,1000,seed=0)
t0=time.perf_counter()
net,d=w1g.sparsify(a,b,w1g.ApproxParams(s=40.0,best_effort=True))
print("wall", time.perf_counter()-t0, {k:round(v,3) for k,v in d.stage_ms.items()})
