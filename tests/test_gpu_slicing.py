"""Time slicing of the resident engine (per-start policy): a start runs in
slices of min(reset_iters, 10) sweeps; a slice beginning on a reset point
begins with InitCircuitTensor exactly where the reset (reading R10) would
rebuild the tensor, any other one restores the tensor its predecessor saved,
so every per-start result is bitwise the one of a start run to its verdict in
one CTA (QF_SLICE=0).  Cases: more starts than resident CTAs and fewer (a start's next
slice then waits on its previous one), the SMALL (n <= 4) and 128-thread
(n = 6) kernels, records across slice boundaries, a start that fails."""
import numpy as np
import pytest

import paper_2306_08152_b200 as qf
import qfgen

pytestmark = pytest.mark.gpu


def _run(w, S, monkeypatch, slice_on, **kw):
    if not slice_on:
        monkeypatch.setenv("QF_SLICE", "0")
    c = qf.Circuit.from_workload(w)
    r = qf.qf_instantiate(c, w.target_unitary(), w.initial(0, S), engine=qf.QF_ENGINE_RESIDENT,
                          **kw)
    monkeypatch.delenv("QF_SLICE", raising=False)
    return r


@pytest.mark.parametrize("name,S,iters,reset", [
    ("C4", 96, 100, 40),     # fewer starts than CTAs: slices wait on their predecessors
    ("C4", 700, 60, 20),     # more starts than CTAs
    ("C3", 200, 90, 30),     # SMALL kernel
    ("C3+", 64, 50, 7),      # short slices, starts converging inside a slice
    ("C4", 300, 60, 13),     # slices of 10 across resets at 13, 26, ...: saved tensors
])
def test_slicing_bitwise(name, S, iters, reset, monkeypatch):
    w = qfgen.workload(name)
    kw = dict(max_iters=iters, reset_iters=reset, record_starts=np.arange(0, S, 7),
              record_sweeps=min(iters, 2 * reset + 3))
    a = _run(w, S, monkeypatch, True, **kw)
    b = _run(w, S, monkeypatch, False, **kw)
    assert np.array_equal(a.summary, b.summary)
    assert np.array_equal(a.gates, b.gates)
    assert np.array_equal(a.cost_hist, b.cost_hist, equal_nan=True)
    assert np.array_equal(a.gates_hist, b.gates_hist, equal_nan=True)
    assert a.best == b.best


def test_slicing_failed_start(monkeypatch):
    """A start whose tensor turns non-finite retires at once; the others run on."""
    w = qfgen.workload("C4")
    monkeypatch.setenv("QF_DEBUG_POISON", "5")
    a = _run(w, 64, monkeypatch, True, max_iters=90, reset_iters=30)
    b = _run(w, 64, monkeypatch, False, max_iters=90, reset_iters=30)
    assert a.verdict[5] == qf.QF_NUMERIC_FAIL and a.iters[5] == 1
    assert np.array_equal(a.verdict, b.verdict) and np.array_equal(a.iters, b.iters)
    assert np.array_equal(a.delta, b.delta, equal_nan=True)  # the failed start's is NaN
    assert np.array_equal(a.gates, b.gates, equal_nan=True)
