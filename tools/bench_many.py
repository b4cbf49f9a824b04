"""NEXT-2 measurement: 1024 independent 3-qubit blocks x 32 multistarts
(qfgen.many_workload, the shape the paper's partitioned flow produces, P:740,
P:886-895) instantiated (a) in ONE qf_instantiate_many launch and (b) one
qf_instantiate call per block (the single-problem path, what a per-block
driver without process packing does).  Both through the host API (inputs
from pinned host memory, results back to host).  Prints one JSON line.
usage: python tools/bench_many.py [blocks] [steps]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_08152_b200 as qf  # noqa: E402
import qfgen  # noqa: E402

blocks = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ws = qfgen.many_workload(blocks)
cs = [qf.Circuit.from_workload(w) for w in ws]
Vs = [np.ascontiguousarray(w.target_unitary()) for w in ws]
Is = [w.initial() for w in ws]
S = sum(x.shape[0] for x in Is)
mi = ws[0].max_iters


def many():
    return qf.qf_instantiate_many(cs, Vs, Is, max_iters=mi)


def per_block():
    return [qf.qf_instantiate(c, V, x, max_iters=mi) for c, V, x in zip(cs, Vs, Is)]


out = {"workload": f"{blocks} x 3-qubit self-target blocks (ladders of 4-10 VAR U(4)), 32 starts each",
       "starts": S, "max_iters": mi}
for name, fn in (("many_one_launch", many), ("one_call_per_block", per_block)):
    fn()  # warm-up
    t0 = time.perf_counter()
    for _ in range(steps):
        r = fn()
    dt = (time.perf_counter() - t0) / steps
    succ = sum(int((x.summary["delta"] < 1e-8).sum()) for x in r)
    sweeps = sum(int(x.summary["iters"].sum()) for x in r)
    out[name] = {"s_per_step": dt, "instantiations_per_s": S / dt, "blocks_per_s": blocks / dt,
                 "successes": succ, "mean_sweeps": sweeps / S}
out["speedup_many_vs_per_block"] = (out["one_call_per_block"]["s_per_step"] /
                                   out["many_one_launch"]["s_per_step"])
print(json.dumps(out))
