"""C-ABI boundary (include/qf.h) without a GPU: the library loads, exports
every declared symbol, validates its arguments, and fails loudly (QF_E_CUDA)
instead of computing anything when no device is present."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

import paper_2306_08152_b200 as qf
import qfgen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "qf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qf_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    L = qf.lib()
    syms = declared_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(qf.EXPORTS) == syms


def test_params_default_matches_paper():
    g = json.load(open(os.path.join(GOLD, "hyperparams_P532.json")))
    p = qf.qf_params_default()
    for k in ("dist_tol", "diff_tol_a", "diff_tol_r", "long_diff_count", "long_diff_r",
              "min_iters", "max_iters", "reset_iters", "beta"):
        assert getattr(p, k) == g[k], k
    assert p.num_starts == g["multistarts"]
    assert ctypes.sizeof(qf.qf_summary) == 16


def test_circuit_create_and_errors():
    c = qf.Circuit(3, [(0, 1), (2,), (1, 2, 0)], [0, 0, 0])
    assert c.var_doubles == 2 * (16 + 4 + 64)
    assert qf.lib().qf_circuit_num_qubits(c.h) == 3
    cases = [
        (lambda: qf.Circuit(0, [], []), qf.QF_E_DIM),
        (lambda: qf.Circuit(13, [], []), qf.QF_E_DIM),
        (lambda: qf.Circuit(3, [(0, 1, 2, 0)], [0]), qf.QF_E_DIM),
        (lambda: qf.Circuit(2, [(0, 2)], [0]), qf.QF_E_LOCATION),
        (lambda: qf.Circuit(2, [(1, 1)], [0]), qf.QF_E_LOCATION),
        (lambda: qf.Circuit(2, [(0, 1)], [1], [None]), qf.QF_E_ARG),
        (lambda: qf.Circuit(2, [(0, 1)], [1], [2 * np.eye(4)]), qf.QF_E_NOT_UNITARY),
        (lambda: qf.Circuit(2, [(0, 1)], [7]), qf.QF_E_ARG),
    ]
    for fn, status in cases:
        with pytest.raises(qf.QfError) as e:
            fn()
        assert e.value.status == status, (e.value, status)
        assert qf.qf_last_error()
    c = qf.Circuit(2, [(0, 1)], [1], [qfgen.CNOT])
    assert c.var_doubles == 0


def test_param_validation_precedes_device():
    w = qfgen.workload("C1")
    c = qf.Circuit.from_workload(w)
    V = w.target_unitary()
    g = w.initial()
    for bad, status in (({"beta": 1.5}, qf.QF_E_ARG), ({"dist_tol": 0.0}, qf.QF_E_ARG),
                        ({"max_iters": -1}, qf.QF_E_ARG), ({"reset_iters": 0}, qf.QF_E_ARG),
                        ({"batch_policy": 2}, qf.QF_E_ARG), ({"start_offset": -1}, qf.QF_E_ARG),
                        ({"batch_policy": qf.QF_BATCH_PAPER, "engine": qf.QF_ENGINE_RESIDENT},
                         qf.QF_E_ARG)):
        with pytest.raises(qf.QfError) as e:
            qf.qf_instantiate(c, V, g, **bad)
        assert e.value.status == status


def test_no_device_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    w = qfgen.workload("C1")
    c = qf.Circuit.from_workload(w)
    with pytest.raises(qf.QfError) as e:
        qf.qf_instantiate(c, w.target_unitary(), w.initial())
    assert e.value.status == qf.QF_E_CUDA
    with pytest.raises(qf.QfError) as e:  # seeded starts: no host fallback either
        qf.qf_instantiate(c, w.target_unitary(), None, num_starts=4, seed=1)
    assert e.value.status == qf.QF_E_CUDA


def test_workspace_size_monotone():
    w = qfgen.workload("C4")
    c = qf.Circuit.from_workload(w)
    a = qf.qf_workspace_size(c, 16)
    b = qf.qf_workspace_size(c, 4096)
    assert b > a > 16 * 64 * 64 * 16
    assert b >= 4096 * 64 * 64 * 16


def test_select_best_host():
    s = np.zeros(5, dtype=qf.SUMMARY_DTYPE)
    s["delta"] = [0.3, np.nan, 0.1, 0.1, 0.2]
    assert qf.qf_select_best_host(s) == 2
    s["delta"] = [np.nan, np.nan, 0.5, 0.5, 0.6]
    assert qf.qf_select_best_host(s) == 2
    s["delta"] = np.nan
    assert qf.qf_select_best_host(s) == 0


def test_instantiate_many_validation_precedes_device():
    w = qfgen.workload("C1")
    c = qf.Circuit.from_workload(w)
    big = qf.Circuit(7, [(0, 1)], [qfgen.VARIABLE], [None])
    rng = np.random.default_rng(0)
    cases = [
        (([c, big], [w.target_unitary(), np.eye(128)], [w.initial(), rng.standard_normal((2, 32))]), {}),
        (([c], [w.target_unitary()], [w.initial()]), {"batch_policy": qf.QF_BATCH_PAPER}),
        (([c], [w.target_unitary()], [w.initial()]), {"engine": qf.QF_ENGINE_STREAM}),
        (([c], [w.target_unitary()], [w.initial()]), {"beta": 2.0}),
    ]
    for args, kw in cases:
        with pytest.raises(qf.QfError) as e:
            qf.qf_instantiate_many(*args, **kw)
        assert e.value.status == qf.QF_E_ARG
