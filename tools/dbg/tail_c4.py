"""C4 to verdict at several start counts (whole waves of 444 resident starts
and the bench's 4096): time per start-sweep shows the tail of the last wave."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2306_08152_b200 as qf, qfgen
w = qfgen.workload("C4")
c = qf.Circuit.from_workload(w)
dev = torch.device("cuda:0")
V = torch.from_numpy(np.ascontiguousarray(w.target_unitary())).to(dev)
for S in [int(a) for a in (sys.argv[1:] or ["3552", "3996", "4096", "4440"])]:
    ws = torch.empty(qf.qf_workspace_size(c, S, max_iters=w.max_iters), dtype=torch.uint8, device=dev)
    kw = dict(max_iters=w.max_iters, seed=w.init_seed, num_starts=S)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = qf.qf_instantiate_device(c, V, None, ws, **kw)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    ss = r.stats["start_sweeps"]
    print(f"S {S} waves {S/444:.2f} ms {1e3*min(ts[1:]):.1f} start-sweeps {ss} us/start-sweep {1e6*min(ts[1:])/ss:.4f}", flush=True)
