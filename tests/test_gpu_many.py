"""NEXT-2 on the GPU: heterogeneous batched instantiation (qf_instantiate_many,
P:740-752) -- several problems with their own templates, targets
and starts in one resident launch.  Each start runs the arithmetic of a
single-problem resident call, so:
  - problems of equal n (same CTA shape) give bitwise the single-call results;
  - mixed n agree with the single calls on every verdict and sweep count and
    on Delta within 1e-12, and with the oracle within the north_star 1e-10."""
import numpy as np
import pytest

import oracle
import paper_2306_08152_b200 as qf
import qfgen
from helpers import haar_np
from test_gpu_parity import _compare

pytestmark = pytest.mark.gpu


def _random_problem(seed, n, p, S, arity=(2,), target="haar"):
    rng = np.random.default_rng(seed)
    locs, kinds = [], []
    for k in range(p):
        m = arity[k % len(arity)]
        q0 = int(rng.integers(0, n - m + 1))
        locs.append(tuple(range(q0, q0 + m)))
        kinds.append(qfgen.VARIABLE)
    cm = [None] * p
    init = np.stack([np.concatenate([haar_np(rng, 2 ** len(l)).view(np.float64).ravel()
                                     for l in locs]) for _ in range(S)])
    V = haar_np(rng, 2 ** n)
    return (n, locs, kinds, cm), V, init


def _single(prob, V, init, max_iters):
    n, locs, kinds, cm = prob
    return qf.qf_instantiate(qf.Circuit(n, locs, kinds, cm), V, init, max_iters=max_iters,
                             engine=qf.QF_ENGINE_RESIDENT)


def _many(probs, Vs, inits, max_iters):
    cs = [qf.Circuit(*pr) for pr in probs]
    return qf.qf_instantiate_many(cs, Vs, inits, max_iters=max_iters)


def test_many_same_n_bitwise():
    probs, Vs, inits = [], [], []
    w = qfgen.workload("C4")
    probs.append((w.n, w.locs, w.kinds, w.const_mats))
    Vs.append(w.target_unitary())
    inits.append(w.initial(0, 24))
    for i, (p, S) in enumerate([(20, 16), (45, 8), (7, 40)]):
        pr, V, init = _random_problem(100 + i, 6, p, S)
        probs.append(pr), Vs.append(V), inits.append(init)
    got = _many(probs, Vs, inits, max_iters=150)
    for q in range(len(probs)):
        ref = _single(probs[q], Vs[q], inits[q], 150)
        assert np.array_equal(got[q].summary, ref.summary), q
        assert np.array_equal(got[q].gates, ref.gates), q
        assert got[q].best == ref.best


def test_many_mixed_against_single_and_oracle(monkeypatch):
    # mixed n runs the 128-thread resident kernel; the single-problem
    # references take the same kernel (QF_RES_WIDE=0: no 256-thread variant
    # for the n = 5 problem), so verdicts and sweep counts must match exactly
    monkeypatch.setenv("QF_RES_WIDE", "0")
    monkeypatch.setenv("QF_LEAN", "0")  # nor the one-warp kernel for the n <= 3 problems
    probs, Vs, inits = [], [], []
    for name, S in (("C1", 4), ("C2+", 16), ("C3+", 48)):
        w = qfgen.workload(name)
        probs.append((w.n, w.locs, w.kinds, w.const_mats))
        Vs.append(w.target_unitary())
        inits.append(w.initial(0, S))
    for i, (n, p, S, ar) in enumerate([(3, 6, 12, (3, 2)), (5, 24, 10, (2,)), (2, 3, 20, (1, 2))]):
        pr, V, init = _random_problem(200 + i, n, p, S, arity=ar)
        probs.append(pr), Vs.append(V), inits.append(init)
    mi = 400
    got = _many(probs, Vs, inits, max_iters=mi)
    for q in range(len(probs)):
        ref = _single(probs[q], Vs[q], inits[q], mi)
        g, r = got[q].summary, ref.summary
        assert np.array_equal(g["verdict"], r["verdict"]) and np.array_equal(g["iters"], r["iters"]), q
        assert np.abs(g["delta"] - r["delta"]).max() < 1e-12, q
        n, locs, kinds, cm = probs[q]
        P = oracle.default_params(max_iters=mi)
        o = oracle.instantiate(oracle.Circuit(n, locs, kinds, cm), Vs[q], inits[q], P,
                               record_sweeps=mi)
        # (verdict, sweeps, Delta) within 1e-10, rounding-borderline stops
        # accepted as in the single-problem parity tests (reading R21)
        border = _compare(got[q], (o, P), np.arange(len(g)), 0, 2 ** n)
        same = [j for j in range(len(g)) if j not in {b[0] for b in border}]
        assert np.abs(got[q].gates[same] - o.gates[same]).max() < 1e-10, q


def test_many_degenerate(monkeypatch):
    """A problem with zero starts and a constant-only circuit ride along."""
    monkeypatch.setenv("QF_LEAN", "0")  # the reference call on k_resident, as the launch
    w = qfgen.workload("C2+")
    pr = (w.n, w.locs, w.kinds, w.const_mats)
    cx = np.eye(4)[[0, 1, 3, 2]]
    const_only = (2, [(0, 1)], [qfgen.CONSTANT], [cx])
    got = _many([pr, pr, const_only], [w.target_unitary()] * 2 + [cx],
                [w.initial(0, 8), w.initial(0, 0), np.zeros((3, 0))], max_iters=50)
    ref = _single(pr, w.target_unitary(), w.initial(0, 8), 50)
    assert np.array_equal(got[0].summary, ref.summary)
    assert got[1].summary.shape == (0,)
    assert np.all(got[2].summary["delta"] < 1e-15)  # V = CNOT, circuit = CNOT
