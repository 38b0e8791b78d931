import sys, os; sys.path.insert(0, '.')
import numpy as np
import paper_2110_14734_b200 as w1g
from paper_2110_14734_b200 import lower_bound
d = np.load('tests/golden/%s.npz' % sys.argv[1])
a, b = d['a'], d['b']
print('sizes', len(a), len(b), flush=True)
n0 = w1g.zero_condense(a, b)
print('zc ok', flush=True)
for s in 'ab':
    r = lower_bound.rwmd_best(n0, s)
    print('side', s, 'ok', r[:4], flush=True)
