import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, qfgen, paper_2306_08152_b200 as qf
for (n,p,seed,ar) in [(4,2,3,(3,)),(4,1,3,(3,))]:
    locs, kinds, cm = qfgen.random_template(n, p, arities=ar, seed=seed, const_frac=0.0)
    print(locs)
    V = qfgen.haar(qfgen.stream_key(seed, qfgen.PURPOSE_TARGET, 0, 0), 2 ** n)[0]
    init = qfgen.initial_gates(n, locs, kinds, 3000 + seed, 0, 1)
    c = qf.Circuit(n, locs, kinds, cm)
    for mi in (0, 1):
        out=[]
        for eng in (1, 2):
            r = qf.qf_instantiate(c, V, init, record_starts=[0], record_sweeps=1, max_iters=mi, engine=eng)
            out.append(r)
        print(n,p,'max_iters',mi,'delta',out[0].delta, out[1].delta, 'gates diff', np.abs(out[0].gates-out[1].gates).max(), 'moved', np.abs(out[1].gates-init).max(), np.abs(out[0].gates-init).max())
