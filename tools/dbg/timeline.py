"""GPU timeline of one qf_instantiate_device call (CUPTI via torch.profiler):
every kernel / memcpy / memset with its start offset and duration, to find
per-call overhead.  usage: python tools/dbg/timeline.py C1 [max_iters]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
import paper_2306_08152_b200 as qf, qfgen
name = sys.argv[1] if len(sys.argv) > 1 else "C1"
w = qfgen.workload(name)
mi = int(sys.argv[2]) if len(sys.argv) > 2 else w.max_iters
dev = torch.device("cuda:0")
c = qf.Circuit.from_workload(w)
dV = torch.from_numpy(np.ascontiguousarray(w.target_unitary())).to(dev)
dI = torch.from_numpy(w.initial()).to(dev)
ws = torch.empty(qf.qf_workspace_size(c, w.starts, max_iters=mi), dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream()
for _ in range(3):
    qf.qf_instantiate_device(c, dV, dI, ws, st, max_iters=mi)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    qf.qf_instantiate_device(c, dV, dI, ws, st, max_iters=mi)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start if evs else 0
prev = t0
for e in evs:
    s, d = e.time_range.start, e.time_range.end - e.time_range.start
    print(f"{(s - t0):10.1f} us  gap {(s - prev):8.1f}  dur {d:9.1f}  {e.name[:90]}")
    prev = e.time_range.end
cpu = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU]
cpu.sort(key=lambda e: e.time_range.start)
print("host API calls:")
c0 = cpu[0].time_range.start if cpu else 0
for e in cpu[:80]:
    print(f"  {(e.time_range.start - c0):10.1f} us dur {(e.time_range.end - e.time_range.start):8.1f} {e.name[:80]}")
