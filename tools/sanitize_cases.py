"""Small cases of every device path, for compute-sanitizer (racecheck,
synccheck, memcheck; one tool per gpurun call, B200_PROFILING.md):

  compute-sanitizer --tool racecheck python tools/sanitize_cases.py [case ...]

resident engine: C1 / C2 / C2+ (register-resident k_reg), C2+ also on k_lean and
the SMALL k_resident variant, C3 (SMALL variant, n <= 4), C4 (128-thread
kernel), C4 WIDE (256-thread MMA variant, overlapped steps), C3+ under the
paper's batch policy (cooperative launch, grid barrier per sweep), many
(heterogeneous problems in one launch); streaming engine: C4 (register
sandwich), C5 (row-tile bulk-copy ring with mbarriers + fused partials,
grouped steps), n = 10 (tile kernel).  Every case checks its verdicts are set.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2306_08152_b200 as qf  # noqa: E402
import qfgen  # noqa: E402


def run(name, S, iters, engine=qf.QF_ENGINE_AUTO, env=None, **kw):
    old = {}
    for k, v in (env or {}).items():
        old[k] = os.environ.get(k)
        os.environ[k] = v
    try:
        w = qfgen.workload(name)
        c = qf.Circuit.from_workload(w)
        r = qf.qf_instantiate(c, w.target_unitary(), None, num_starts=S, seed=w.init_seed,
                              max_iters=iters, engine=engine, **kw)
        assert np.all(r.verdict != qf.QF_RUNNING), r.verdict
        return r
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


CASES = {
    "res_C1": lambda: run("C1", 4, 20),                        # k_reg<2>
    "res_C2": lambda: run("C2", 8, 20),                        # k_reg<3>
    "res_C2p": lambda: run("C2+", 8, 10),                      # k_reg<3>, 2-qubit VARIABLE
    "res_C2p_lean": lambda: run("C2+", 8, 10, env={"QF_REG_RES": "0"}),  # k_lean<3>
    "res_C2p_small": lambda: run("C2+", 8, 10, env={"QF_LEAN": "0"}),
    "res_C3": lambda: run("C3", 16, 3),
    "res_C4": lambda: run("C4", 6, 2),
    "res_C4_sliced": lambda: run("C4", 24, 50, reset_iters=20),  # time slicing, waits
    "res_C3_sliced": lambda: run("C3", 40, 30, reset_iters=10),
    "res_C4_wide": lambda: run("C4", 6, 2, env={"QF_RES_WIDE": "1"}),
    "batch_C3p": lambda: run("C3+", 12, 8, batch_policy=qf.QF_BATCH_PAPER),
    "stream_C4": lambda: run("C4", 6, 1, engine=qf.QF_ENGINE_STREAM),
    "stream_C5": lambda: run("C5", 3, 1),
    "stream_C6": lambda: run("C6", 1, 1),
}


def many():
    w = qfgen.workload("C2+")
    w3 = qfgen.workload("C3+")
    cs = [qf.Circuit.from_workload(w), qf.Circuit.from_workload(w3)]
    out = qf.qf_instantiate_many(cs, [w.target_unitary(), w3.target_unitary()],
                                 [w.initial(0, 4), w3.initial(0, 4)], max_iters=5)
    assert all(np.all(r.verdict != qf.QF_RUNNING) for r in out)


CASES["many"] = many

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
        print("case ok:", n, flush=True)
