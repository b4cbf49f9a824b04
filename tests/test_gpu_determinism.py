"""Race evidence without compute-sanitizer (closed on the GPU pool): every
device path must give bitwise the same per-start results when a call is
repeated -- shared-memory races, a missing barrier or an unordered reduction
would show up as run-to-run differences (the reductions are fixed-order by
design).  Each path runs 3 times on the same inputs; the bounds-
checked build (tools/checked_build.py, -DQF_DEVICE_CHECKS) runs the same
cases with device traps on out-of-range indices."""
import os

import numpy as np
import pytest

import paper_2306_08152_b200 as qf
import qfgen

pytestmark = pytest.mark.gpu

CASES = [
    # (name, config, starts, sweeps, engine, env, extra params)
    ("register-resident k_reg n=2", "C1", 4, 30, qf.QF_ENGINE_AUTO, {}, {}),
    ("register-resident k_reg n=3", "C2", 16, 40, qf.QF_ENGINE_AUTO, {}, {}),
    ("register-resident k_reg n=3, 2-qubit VARIABLE", "C2+", 16, 20, qf.QF_ENGINE_AUTO, {}, {}),
    ("one-warp k_lean n=3", "C2+", 16, 20, qf.QF_ENGINE_AUTO, {"QF_REG_RES": "0"}, {}),
    ("resident SMALL n=3", "C2+", 16, 20, qf.QF_ENGINE_AUTO, {"QF_LEAN": "0"}, {}),
    ("resident SMALL n=4", "C3", 64, 10, qf.QF_ENGINE_AUTO, {}, {}),
    ("resident 128-thread n=6", "C4", 96, 6, qf.QF_ENGINE_AUTO, {}, {}),
    ("resident time-sliced n=6", "C4", 96, 50, qf.QF_ENGINE_AUTO, {}, {"reset_iters": 20}),
    ("resident WIDE n=6", "C4", 96, 6, qf.QF_ENGINE_AUTO, {"QF_RES_WIDE": "1"}, {}),
    ("resident batch policy", "C3+", 48, 20, qf.QF_ENGINE_AUTO, {},
     {"batch_policy": qf.QF_BATCH_PAPER}),
    ("streaming register sandwich", "C4", 32, 2, qf.QF_ENGINE_STREAM, {}, {}),
    ("streaming row tiles + groups", "C5", 8, 2, qf.QF_ENGINE_AUTO, {}, {}),
    ("streaming row tiles, fused partials", "C5", 8, 1, qf.QF_ENGINE_AUTO,
     {"QF_GROUP": "0"}, {}),
    ("streaming tile kernel n=10", "C6", 2, 1, qf.QF_ENGINE_AUTO, {}, {}),
]


@pytest.mark.parametrize("name,cfg,S,iters,engine,env,extra", CASES, ids=[c[0] for c in CASES])
def test_repeat_bitwise(name, cfg, S, iters, engine, env, extra, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    w = qfgen.workload(cfg)
    c = qf.Circuit.from_workload(w)
    V = w.target_unitary()
    runs = [qf.qf_instantiate(c, V, None, num_starts=S, seed=w.init_seed, max_iters=iters,
                              engine=engine, **extra) for _ in range(3)]
    for r in runs[1:]:
        assert np.array_equal(r.summary, runs[0].summary), name
        assert np.array_equal(r.gates, runs[0].gates), name
    assert np.all(runs[0].verdict != qf.QF_RUNNING)
