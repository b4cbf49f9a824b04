"""Builds a debug copy of the library with -DQF_POLAR_COUNT and reports the mean
Newton-Schulz iterations per polar factor on a workload (default C4, 3 sweeps).
usage: python tools/polar_stats.py [config] [sweeps] [engine]"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2306_08152_b200 import _build  # noqa: E402

dbg = os.path.join(ROOT, "paper_2306_08152_b200", "libqfactor_debug.so")
subprocess.check_call([_build.NVCC, *_build.ARCH, *_build.FLAGS, "-DQF_POLAR_COUNT", *_build.sources(),
                       "-o", dbg])
_build.LIB = dbg  # load the debug library through the normal binding
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2306_08152_b200 as qf  # noqa: E402
import qfgen  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
eng = {"stream": 1, "resident": 2}.get(sys.argv[3] if len(sys.argv) > 3 else "auto", 0)
w = qfgen.workload(name)
c = qf.Circuit.from_workload(w)
r = qf.qf_instantiate(c, w.target_unitary(), w.initial(), max_iters=iters, engine=eng)
out = (ctypes.c_ulonglong * 20)()
qf.lib().qf_debug_polar_counts(out)
print(f"{name} {iters} sweeps: NS calls {out[0]}, NS iterations {out[1]} "
      f"({out[1] / max(1, out[0]):.2f} per call), Jacobi sweeps {out[2]}")
if out[5]:
    print(f"  resident: per step serial {out[3] / out[5]:.0f} cycles, sandwich {out[4] / out[5]:.0f} "
          f"cycles ({out[5]} steps)")
if out[9]:
    print(f"  gather (all threads, before the barrier) {out[6] / out[9]:.0f}, form A {out[7] / out[9]:.0f}, "
          f"polar {out[8] / out[9]:.0f} cycles")

if out[13]:
    print(f"  WIDE overlapped phase A on warp 0: env from T {out[10] / out[13]:.0f} (incl. the u_old "
          f"load issue), u_old staged {out[11] / out[13]:.0f}, prepare (form A + polar + L/R) "
          f"{out[12] / out[13]:.0f} cycles ({out[13]} steps)")
    print(f"  phase A per step: warp 0 {out[3] / out[5]:.0f}, warp 1 (sandwich) {out[4] / out[5]:.0f}; "
          f"after the barrier (tile table + T gather) {out[6] / out[5]:.0f} cycles")

if out[19]:
    nl = out[19]
    print(f"  k_lean per step: sandwich {out[14] / nl:.0f}, env {out[15] / nl:.0f}, form A {out[16] / nl:.0f}, "
          f"polar {out[17] / nl:.0f}, L/R {out[18] / nl:.0f} cycles ({nl} steps)")

rc = (ctypes.c_ulonglong * 5)()
qf.lib().qf_debug_rows_counts(rc)
if rc[4]:
    print(f"  row-tile d=8 per tile (consumer thread 0): wait {rc[0] / rc[4]:.0f}, phase 1 "
          f"{rc[1] / rc[4]:.0f}, phase 2 {rc[2] / rc[4]:.0f}, epilogue+handoff {rc[3] / rc[4]:.0f} cycles "
          f"({rc[4]} tiles)")
