import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_08152_b200 import _build
if len(sys.argv) > 1: _build.LIB = sys.argv[1]; _build.needs_build = lambda: False
import numpy as np, qfgen, paper_2306_08152_b200 as qf
for (n,p,seed,ar) in [(4,1,3,(3,)),(4,6,3,(3,))]:
    locs, kinds, cm = qfgen.random_template(n, p, arities=ar, seed=seed, const_frac=0.0)
    V = qfgen.haar(qfgen.stream_key(seed, qfgen.PURPOSE_TARGET, 0, 0), 2 ** n)[0]
    init = qfgen.initial_gates(n, locs, kinds, 3000 + seed, 0, 1)
    c = qf.Circuit(n, locs, kinds, cm)
    out=[qf.qf_instantiate(c, V, init, max_iters=1, engine=e) for e in (1,2)]
    print(_build.LIB[-30:], n,p,'delta stream',out[0].delta,'resident',out[1].delta)
