"""Short, fixed workload for ncu captures: one qf_instantiate_device call on a
config with max_iters capped (same kernels and launch configuration as
bench.py's step).  Usage: python tools/profile_case.py C4 2"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_08152_b200 as qf  # noqa: E402
import qfgen  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
w = qfgen.workload(name)
dev = torch.device("cuda:0")
c = qf.Circuit.from_workload(w)
dV = torch.from_numpy(np.ascontiguousarray(w.target_unitary())).to(dev)
dI = torch.from_numpy(w.initial()).to(dev)
ws = torch.empty(qf.qf_workspace_size(c, w.starts, max_iters=iters), dtype=torch.uint8, device=dev)
eng = {"stream": qf.QF_ENGINE_STREAM, "resident": qf.QF_ENGINE_RESIDENT}.get(
    os.environ.get("QF_ENGINE", "auto"), qf.QF_ENGINE_AUTO)
for _ in range(reps):
    r = qf.qf_instantiate_device(c, dV, dI, ws, max_iters=iters, profile=1, engine=eng)
torch.cuda.synchronize()
print(name, "iters", iters, "stats", r.stats)
