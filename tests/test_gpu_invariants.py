"""GPU-side checks of the facts the paper fixes, on the GPU's own records --
including starts and sweeps the oracle does not cover -- and of the polar
factor's fallback paths (rank-deficient environments, Jacobi).

  * every updated gate is unitary to 1e-12 (north_star);
  * |Tr(V^dag U)| <= N, i.e. Delta >= 0;
  * the cost never increases: every single update raises |Tr| or keeps it
    (P:448-452), so Delta is non-increasing from sweep to sweep;
  * a rank-deficient environment still gives a unitary update whose value
    Re Tr(E u_new) is the sum of the singular values (SURVEY
    Sec. 8c reading #13: for singular E only that value is unique).
"""
import numpy as np
import pytest

import oracle
import paper_2306_08152_b200 as qf
import qfgen
from test_gpu_parity import ENGINES, _compare, _run_pair

pytestmark = pytest.mark.gpu


def _unitarity_err(packed, locs, kinds):
    """max |u^dag u - I| over every VARIABLE gate of every row of `packed`."""
    err, off = 0.0, 0
    flat = packed.reshape(-1, packed.shape[-1])
    for l, k in zip(locs, kinds):
        if k == qfgen.CONSTANT:
            continue
        d = 1 << len(l)
        u = np.ascontiguousarray(flat[:, off:off + 2 * d * d]).view(np.complex128)
        u = u.reshape(-1, d, d)
        g = np.einsum("sji,sjk->sik", u.conj(), u) - np.eye(d)
        err = max(err, float(np.abs(g).max()))
        off += 2 * d * d
    return err


def _check_invariants(w, res, R):
    N = 2 ** w.n
    eta = 64 * N * np.finfo(float).eps
    ch = res.cost_hist[:, :R]
    ok = np.isfinite(ch)
    assert np.all(ch[ok] >= -eta), ch[ok].min()          # |Tr| <= N
    assert np.all(ch[ok] <= 1.0 + eta)
    d = np.diff(np.where(ok, ch, np.nan), axis=1)       # non-increasing
    dd = d[np.isfinite(d)]
    assert dd.size == 0 or dd.max() <= eta, dd.max()
    assert np.all(res.delta >= -eta)
    assert _unitarity_err(res.gates, w.locs, w.kinds) < 1e-12
    assert _unitarity_err(res.gates_hist[:, :R][ok], w.locs, w.kinds) < 1e-12


@pytest.mark.parametrize("engine", [qf.QF_ENGINE_AUTO, qf.QF_ENGINE_STREAM])
def test_invariants_C4_all_starts(engine):
    """Every one of C4's 4096 starts run to its verdict: final gates unitary,
    Delta in [0, 1]; 512 recorded starts spread over the batch: Delta
    non-increasing over the first 20 sweeps and every recorded gate unitary."""
    w = qfgen.workload("C4")
    rec = np.linspace(0, w.starts - 1, 512).astype(np.int32)
    r = qf.qf_instantiate(qf.Circuit.from_workload(w), w.target_unitary(), w.initial(),
                          record_starts=rec, record_sweeps=20, max_iters=w.max_iters,
                          engine=engine)
    assert np.all(r.verdict != qf.QF_RUNNING)
    _check_invariants(w, r, 20)


def test_invariants_C5_full_batch():
    """All 8192 C5 starts for 3 sweeps in bench.py's launch configuration:
    every start's gates unitary and Delta non-increasing on 64 recorded
    starts spread over the batch."""
    w = qfgen.workload("C5")
    rec = np.linspace(0, w.starts - 1, 64).astype(np.int32)
    r = qf.qf_instantiate(qf.Circuit.from_workload(w), w.target_unitary(), w.initial(),
                          record_starts=rec, record_sweeps=3, max_iters=3)
    assert np.all(r.iters == 3)
    _check_invariants(w, r, 3)


# ------------------------------------------------------------------ polar fallback
def _cnot_on(n, c, t):
    """Dense CNOT(c -> t) on n qubits (qubit 0 = MSB) from its definition."""
    N = 2 ** n
    M = np.zeros((N, N))
    for i in range(N):
        j = i ^ (1 << (n - 1 - t)) if (i >> (n - 1 - c)) & 1 else i
        M[j, i] = 1.0
    return M.astype(np.complex128)


RANK_DEFICIENT = [
    # (n, VARIABLE gate location, CNOT (c, t) of the target): the environment
    # of the single gate is PT over t of CNOT = I x diag(2, 0) on the gate's
    # qubits -- half its singular values are 0, sum sigma = N / 2.
    (2, (0,), (0, 1)),
    (3, (0, 1), (1, 2)),
    (4, (0, 1, 2), (2, 3)),
]


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("n,loc,cnot", RANK_DEFICIENT)
@pytest.mark.parametrize("polar", ["ns", "jacobi"])
def test_polar_rank_deficient(n, loc, cnot, engine, polar, monkeypatch):
    """A singular environment (rank d/2): the update must still be unitary
    to 1e-12, and its value Re Tr(E u_new) = sum sigma(E) = N/2,
    so Delta = 1/2 after every sweep; the oracle agrees on Delta (the gate
    itself is not unique here)."""
    if polar == "jacobi":
        monkeypatch.setenv("QF_POLAR", "jacobi")
    V = _cnot_on(n, *cnot)
    locs, kinds, cm = [loc], [qfgen.VARIABLE], [None]
    init = qfgen.initial_gates(n, locs, kinds, 77, 0, 9)
    c = qf.Circuit(n, locs, kinds, cm)
    r = qf.qf_instantiate(c, V, init, record_starts=np.arange(9), record_sweeps=3,
                          max_iters=3, engine=engine)
    ch = r.cost_hist[:, :3]
    m = np.isfinite(ch)  # the short plateau stops every start after sweep 2
    assert _unitarity_err(r.gates, locs, kinds) < 1e-12
    assert _unitarity_err(r.gates_hist[m], locs, kinds) < 1e-12
    assert m[:, :2].all() and np.abs(ch[m] - 0.5).max() < 1e-12, ch
    # the unique part (Delta) against the oracle
    o = oracle.instantiate(oracle.Circuit(n, locs, kinds, cm), V, init,
                           oracle.default_params(max_iters=3), record_sweeps=3)
    assert np.array_equal(m, np.isfinite(o.cost_hist))
    assert np.abs(ch[m] - o.cost_hist[m]).max() < 1e-12
    assert np.array_equal(r.verdict, o.verdict) and np.array_equal(r.iters, o.iters)


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("n,p,seed", [(4, 8, 11), (5, 7, 12), (6, 6, 13)])
def test_parity_jacobi_polar(n, p, seed, engine, monkeypatch):
    """QF_POLAR=jacobi (the one-sided Jacobi that finishes a non-converging
    Newton-Schulz iteration) against the oracle on random templates with
    1-, 2- and 3-qubit gates: the polar factor is unique for non-singular E,
    so the Jacobi path must meet the same 1e-10 bar."""
    monkeypatch.setenv("QF_POLAR", "jacobi")
    locs, kinds, cm = qfgen.random_template(n, p, seed=seed, const_frac=0.2)
    V = qfgen.haar(qfgen.stream_key(seed, qfgen.PURPOSE_TARGET, 0, 0), 2 ** n)[0]
    init = qfgen.initial_gates(n, locs, kinds, 4000 + seed, 0, 21)
    gpu, orc, idx = _run_pair(n, locs, kinds, cm, V, init, R=10, max_iters=10, engine=engine)
    _compare(gpu, orc, idx, 10, 2 ** n)
