"""A/B of library builds on C1/C2 per-step latency: python tools/dbg/small_ab.py LIB_A LIB_B"""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
code = r'''
import sys, os, time
sys.path.insert(0, %r)
from paper_2306_08152_b200 import _build
_build.LIB = sys.argv[1]
import numpy as np, torch
import paper_2306_08152_b200 as qf, qfgen
out = []
for name in ("C1", "C2"):
    w = qfgen.workload(name)
    dev = torch.device("cuda:0")
    c = qf.Circuit.from_workload(w)
    dV = torch.from_numpy(np.ascontiguousarray(w.target_unitary())).to(dev)
    dI = torch.from_numpy(w.initial()).to(dev)
    ws = torch.empty(qf.qf_workspace_size(c, w.starts, max_iters=w.max_iters), dtype=torch.uint8, device=dev)
    best = 1e9
    for _ in range(3):
        r = qf.qf_instantiate_device(c, dV, dI, ws, max_iters=w.max_iters, profile=1)
        best = min(best, r.stats["resident_ms"])
    out.append(f"{name} {1e3 * best / (r.iters.max() * 2 * w.p):.4f}")
print(" ".join(out))
''' % ROOT
for rep in range(2):
    for lib in sys.argv[1:]:
        o = subprocess.run([sys.executable, "-c", code, lib], capture_output=True, text=True)
        print(lib, "us/step:", o.stdout.strip() or o.stderr[-300:], flush=True)
