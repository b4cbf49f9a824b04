"""First sweep where the GPU's per-sweep Delta leaves the oracle's (debug)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import oracle, qfgen
import paper_2306_08152_b200 as qf
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
S = int(sys.argv[2]) if len(sys.argv) > 2 else 4
R = int(sys.argv[3]) if len(sys.argv) > 3 else 50
w = qfgen.workload(name)
init = w.initial(0, S)
V = w.target_unitary()
c = qf.Circuit.from_workload(w)
g = qf.qf_instantiate(c, V, init, record_starts=np.arange(S), record_sweeps=R, max_iters=R)
o = oracle.instantiate(oracle.Circuit(w.n, w.locs, w.kinds, w.const_mats), V, init,
                       oracle.default_params(max_iters=R), record_sweeps=R, record_gates=R)
for s in range(S):
    d = np.abs(g.cost_hist[s] - o.cost_hist[s])
    gd = np.abs(g.gates_hist[s] - o.gates_hist[s]).max(axis=1)
    bad = np.nonzero(d > 1e-10)[0]
    print(s, "first Delta divergence at sweep", bad[0] + 1 if len(bad) else None,
          "max |dDelta| by sweep 1..10:", d[:10].max(), "gate err by sweep:", np.array2string(gd[:R:5], precision=1))
