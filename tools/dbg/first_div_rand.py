"""First sweep where the GPU leaves the oracle on a random template (debug)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import oracle, qfgen
import paper_2306_08152_b200 as qf
n, p, seed = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
ar = tuple(int(x) for x in sys.argv[4].split(",")) if len(sys.argv) > 4 else (1, 2)
S, R = 4, 20
locs, kinds, cm = qfgen.random_template(n, p, arities=ar, seed=seed, const_frac=0.25)
print(locs, kinds)
V = qfgen.haar(qfgen.stream_key(seed, qfgen.PURPOSE_TARGET, 0, 0), 2 ** n)[0]
init = qfgen.initial_gates(n, locs, kinds, 3000 + seed, 0, S)
c = qf.Circuit(n, locs, kinds, cm)
g = qf.qf_instantiate(c, V, init, record_starts=np.arange(S), record_sweeps=R, max_iters=R)
o = oracle.instantiate(oracle.Circuit(n, locs, kinds, cm), V, init,
                       oracle.default_params(max_iters=R), record_sweeps=R, record_gates=R)
for s in range(S):
    d = np.abs(g.cost_hist[s] - o.cost_hist[s])
    d = d[np.isfinite(d)]
    print(s, "max |dDelta|", d.max() if len(d) else None, "verdicts", g.verdict[s], o.verdict[s], g.iters[s], o.iters[s])
