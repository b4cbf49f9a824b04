"""Per-call overhead of qf_instantiate_device (max_iters = 0 and 1) for C1."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2306_08152_b200 as qf, qfgen
w = qfgen.workload("C1")
dev = torch.device("cuda:0")
c = qf.Circuit.from_workload(w)
dV = torch.from_numpy(np.ascontiguousarray(w.target_unitary())).to(dev)
dI = torch.from_numpy(w.initial()).to(dev)
ws = torch.empty(qf.qf_workspace_size(c, w.starts, max_iters=w.max_iters), dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream()
for mi in (0, 1, w.max_iters):
    for want in (True, False):
        ts = []
        for _ in range(20):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            qf.qf_instantiate_device(c, dV, dI, ws, st, max_iters=mi, want_result=want)
            torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(10):
            qf.qf_instantiate_device(c, dV, dI, ws, st, max_iters=mi, want_result=want)
        e1.record(st); torch.cuda.synchronize()
        print(f"max_iters {mi} want_result {want}: wall median {1e3*sorted(ts)[10]:.3f} ms, events {e0.elapsed_time(e1)/10:.3f} ms/call")
