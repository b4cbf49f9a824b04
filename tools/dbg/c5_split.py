"""C5 init + 2 sweeps with per-launch events: sandwich vs environment split."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2306_08152_b200 as qf, qfgen
w = qfgen.workload("C5")
dev = torch.device("cuda:0")
c = qf.Circuit.from_workload(w)
V = torch.from_numpy(np.ascontiguousarray(w.target_unitary())).to(dev)
ws = torch.empty(qf.qf_workspace_size(c, w.starts, max_iters=2), dtype=torch.uint8, device=dev)
kw = dict(max_iters=2, seed=w.init_seed, num_starts=w.starts)
qf.qf_instantiate_device(c, V, None, ws, want_result=False, **kw)
r = qf.qf_instantiate_device(c, V, None, ws, profile=1, **kw)
st = r.stats
print("fuse", os.environ.get("QF_GROUP_FUSE", "2"), "tsum", os.environ.get("QF_GROUP_TSUM", "1"), "sandwich ms", round(st["sandwich_ms"], 1), "launches", st["sandwich_launches"],
      "GB/s", round(st["sandwich_bytes"] / 1e9 / (st["sandwich_ms"] / 1e3)),
      "| env ms", round(st["env_ms"], 1), "launches", st["env_launches"],
      "useful GB/s", round(st["env_bytes"] / 1e9 / (st["env_ms"] / 1e3)))
