import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2306_08152_b200 as qf, qfgen
for name in ("C1", "C2"):
    w = qfgen.workload(name)
    dev = torch.device("cuda:0")
    c = qf.Circuit.from_workload(w)
    dV = torch.from_numpy(np.ascontiguousarray(w.target_unitary())).to(dev)
    dI = torch.from_numpy(w.initial()).to(dev)
    ws = torch.empty(qf.qf_workspace_size(c, w.starts, max_iters=w.max_iters), dtype=torch.uint8, device=dev)
    for _ in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = qf.qf_instantiate_device(c, dV, dI, ws, max_iters=w.max_iters, profile=1)
        torch.cuda.synchronize(); t1 = time.perf_counter()
    it = r.iters.max()
    print(name, "call ms", 1e3 * (t1 - t0), "resident kernel ms", r.stats["resident_ms"], "max sweeps", it,
          "us per step (slowest start)", 1e3 * r.stats["resident_ms"] / (it * 2 * w.p), "launches", r.stats["kernel_launches"])
