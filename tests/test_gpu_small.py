"""Smallest blocks (n <= 3): the register-resident kernel k_reg (tensor in the
warp's registers; VARIABLE and CONSTANT gates of <= 2 qubits, CONSTANT 0/1
permutations applied as relabellings)
against the shared-memory kernel k_lean it replaces (QF_REG_RES=0) -- bitwise
equal summaries, gates and per-sweep records, since every output is formed
with k_lean's operand and summation order -- and against the oracle within the
north_star tolerance.  Templates cover every gate position at n = 1, 2, 3
(the n = 3 layout keeps row bit 2 in the register index), reversed and
non-adjacent CONSTANT pairs, CONSTANT one-qubit gates, beta != 0 and resets."""
import numpy as np
import pytest

import paper_2306_08152_b200 as qf
import qfgen
from helpers import haar_np
from test_gpu_parity import _compare, _run_pair

pytestmark = pytest.mark.gpu

CNOT = np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]], dtype=complex)


def _template(n, p, seed, var2=0.0):
    """One-qubit VARIABLE gates on random qubits, CONSTANT CNOT / Haar 4 x 4
    on random ordered pairs (any order, any distance), CONSTANT Haar 2 x 2;
    with probability var2 a 2-qubit VARIABLE gate on a random ordered pair."""
    rng = np.random.default_rng(seed)
    locs, kinds, cm = [], [], []
    for k in range(p):
        u = rng.random()
        if n >= 2 and rng.random() < var2:
            q = rng.choice(n, 2, replace=False)
            locs.append((int(q[0]), int(q[1])))
            kinds.append(qfgen.VARIABLE)
            cm.append(None)
        elif n >= 2 and u < 0.35:
            q = rng.choice(n, 2, replace=False)
            locs.append((int(q[0]), int(q[1])))
            kinds.append(qfgen.CONSTANT)
            cm.append(CNOT if rng.random() < 0.5 else haar_np(rng, 4))
        elif u < 0.45:
            locs.append((int(rng.integers(n)),))
            kinds.append(qfgen.CONSTANT)
            cm.append(haar_np(rng, 2))
        else:
            locs.append((int(rng.integers(n)),))
            kinds.append(qfgen.VARIABLE)
            cm.append(None)
    if qfgen.VARIABLE not in kinds:
        locs[0], kinds[0], cm[0] = (0,), qfgen.VARIABLE, None
    return locs, kinds, cm


def _both(c, V, init, monkeypatch, **kw):
    a = qf.qf_instantiate(c, V, init, **kw)
    monkeypatch.setenv("QF_REG_RES", "0")
    b = qf.qf_instantiate(c, V, init, **kw)
    monkeypatch.delenv("QF_REG_RES")
    assert a.stats["resident_kernel"] == 3 and b.stats["resident_kernel"] == 2
    return a, b


def _same(a, b):
    assert np.array_equal(a.summary, b.summary)
    assert np.array_equal(a.gates, b.gates)
    if a.cost_hist is not None:
        assert np.array_equal(a.cost_hist, b.cost_hist, equal_nan=True)
        assert np.array_equal(a.gates_hist, b.gates_hist, equal_nan=True)


@pytest.mark.parametrize("name,iters", [("C1", None), ("C2", 300), ("C2+", None)])
def test_reg_bitwise_lean_configs(name, iters, monkeypatch):
    w = qfgen.workload(name)
    c = qf.Circuit.from_workload(w)
    S = w.starts
    a, b = _both(c, w.target_unitary(), w.initial(), monkeypatch,
                 max_iters=iters or w.max_iters, record_starts=np.arange(min(S, 16)),
                 record_sweeps=10)
    _same(a, b)


@pytest.mark.parametrize("n,p,seed,var2,params", [
    (1, 3, 1, 0.0, {}),
    (2, 9, 2, 0.0, {}),
    (2, 14, 3, 0.0, {"beta": 0.1, "reset_iters": 7}),
    (3, 12, 4, 0.0, {}),
    (3, 30, 5, 0.0, {"reset_iters": 5}),
    (3, 20, 6, 0.0, {"beta": 0.05}),
    (2, 10, 7, 0.4, {}),
    (3, 16, 8, 0.4, {"beta": 0.05, "reset_iters": 6}),
    (3, 24, 9, 0.3, {}),
])
def test_reg_bitwise_lean_random(n, p, seed, var2, params, monkeypatch):
    locs, kinds, cm = _template(n, p, seed, var2)
    c = qf.Circuit(n, locs, kinds, cm)
    V = qfgen.haar(qfgen.stream_key(seed, qfgen.PURPOSE_TARGET, 0, 0), 2 ** n)[0]
    init = qfgen.initial_gates(n, locs, kinds, 4000 + seed, 0, 37)
    a, b = _both(c, V, init, monkeypatch, max_iters=200, record_starts=np.arange(37),
                 record_sweeps=10, **params)
    _same(a, b)


@pytest.mark.parametrize("n,p,seed,var2", [(2, 9, 12, 0.0), (3, 16, 13, 0.0), (3, 24, 14, 0.0),
                                            (3, 14, 15, 0.4)])
def test_reg_parity_oracle(n, p, seed, var2):
    """k_reg against the oracle: 37 starts, 10 recorded sweeps, to verdict
    within 300 sweeps (north_star tolerance, R21 readings as in test_gpu_parity)."""
    locs, kinds, cm = _template(n, p, seed, var2)
    V = qfgen.haar(qfgen.stream_key(seed, qfgen.PURPOSE_TARGET, 0, 0), 2 ** n)[0]
    init = qfgen.initial_gates(n, locs, kinds, 4000 + seed, 0, 37)
    gpu, orc, idx = _run_pair(n, locs, kinds, cm, V, init, R=10, max_iters=300)
    assert gpu.stats["resident_kernel"] == 3
    _compare(gpu, orc, idx, 10, 2 ** n)


def test_reg_zero_iters(monkeypatch):
    """max_iters = 0: the cost of the initial gates only."""
    w = qfgen.workload("C1")
    c = qf.Circuit.from_workload(w)
    a, b = _both(c, w.target_unitary(), w.initial(), monkeypatch, max_iters=0)
    _same(a, b)
    assert np.all(a.verdict == qf.QF_MAX_ITER)
