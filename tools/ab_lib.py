"""A/B timing of library builds / switches on one box:
  python tools/ab_lib.py SPEC_A SPEC_B [SPEC_C ...] [--reps R] [--config C]
SPEC = path/to/lib.so[@VAR=value[,VAR=value]] (environment for that arm).
C4 (or `config`), 3 sweeps (or --sweeps K), resident engine (AB_ENGINE=stream for the
streaming one); alternates the arms to cancel drift and prints each run's
wall time of the whole call (ms, best of the last two of three), the
start-sweeps it ran and the time per start-sweep."""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
args = sys.argv[1:]
reps, cfg, sweeps = 3, "C4", 3
if "--reps" in args:
    i = args.index("--reps")
    reps = int(args[i + 1])
    del args[i:i + 2]
if "--sweeps" in args:
    i = args.index("--sweeps")
    sweeps = int(args[i + 1])
    del args[i:i + 2]
if "--config" in args:
    i = args.index("--config")
    cfg = args[i + 1]
    del args[i:i + 2]
libs = args
code = r'''
import sys, os
sys.path.insert(0, %r)
from paper_2306_08152_b200 import _build
_build.LIB = sys.argv[1]
import numpy as np, torch
import paper_2306_08152_b200 as qf, qfgen
w = qfgen.workload(sys.argv[2] if len(sys.argv) > 2 else "C4")
dev = torch.device("cuda:0")
c = qf.Circuit.from_workload(w)
dV = torch.from_numpy(np.ascontiguousarray(w.target_unitary())).to(dev)
dI = torch.from_numpy(w.initial()).to(dev)
MI = int(sys.argv[3])
ws = torch.empty(qf.qf_workspace_size(c, w.starts, max_iters=MI), dtype=torch.uint8, device=dev)
eng = {"stream": qf.QF_ENGINE_STREAM, "resident": qf.QF_ENGINE_RESIDENT}[os.environ.get("AB_ENGINE", "resident")]
import time
ms = []
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = qf.qf_instantiate_device(c, dV, dI, ws, max_iters=MI, engine=eng)
    torch.cuda.synchronize()
    ms.append(1e3 * (time.perf_counter() - t0))
print(r.stats["start_sweeps"], min(ms[1:]))
''' % ROOT
res = {l: [] for l in libs}
for _ in range(reps):
    for l in libs:
        path, _, envs = l.partition("@")
        env = dict(os.environ)
        for kv in filter(None, envs.split(",")):
            k, _, v = kv.partition("=")
            env[k] = v
        out = subprocess.run([sys.executable, "-c", code, path, cfg, str(sweeps)], capture_output=True, text=True,
                             env=env)
        f = out.stdout.strip().split()
        res[l].append((float(f[-1]), int(f[-2])))
for l in libs:
    t = [x for x, _ in res[l]]
    ss = res[l][0][1]
    print(l, " ".join(f"{x:.2f}" for x in t), "min", f"{min(t):.2f}", "start-sweeps", ss,
          f"us/start-sweep {1e3 * min(t) / ss:.4f}")
