"""NEXT-1 on the GPU: the batch termination policy (reading R22)
(resident engine for co-resident batches, streaming otherwise) against the
batch oracle (tests/test_batch_policy.py
pins the oracle side), on the same seeded inputs: every start's verdict and
sweep count agree and the final Delta within the north_star 1e-10.  The
cross-process reduction is exercised through qf_params.batch_reduce with a
callback that stands in for other ranks."""
import numpy as np
import pytest

import oracle
import paper_2306_08152_b200 as qf
import qfgen
from helpers import haar_np

pytestmark = pytest.mark.gpu

TOL = 1e-10


def _plateau_case():
    rng = np.random.default_rng(2306)
    locs = [(0, 1), (1, 2), (0, 1)]
    kinds = [qfgen.VARIABLE] * 3
    V = haar_np(rng, 8)
    init = np.stack([np.concatenate([haar_np(rng, 4).view(np.float64).ravel() for _ in locs])
                     for _ in range(12)])
    return 3, locs, kinds, [None] * 3, V, init


def _pair(n, locs, kinds, cm, V, init, **params):
    P = oracle.default_params(**params)
    orc = oracle.instantiate_batch(oracle.Circuit(n, locs, kinds, cm), V, init, P)
    gpu = qf.qf_instantiate(qf.Circuit(n, locs, kinds, cm), V, init,
                            batch_policy=qf.QF_BATCH_PAPER, **params)
    return gpu, orc


def _check(gpu, orc):
    g = gpu.summary
    assert np.array_equal(g["verdict"], orc.verdict), (g["verdict"], orc.verdict)
    assert np.array_equal(g["iters"], orc.iters), (g["iters"], orc.iters)
    assert np.abs(g["delta"] - orc.delta).max() < TOL
    assert np.array_equal(g["delta"] < 1e-8, orc.delta < 1e-8)


@pytest.mark.parametrize("name", ["C1", "C2+", "C3+"])
def test_batch_success_path(name):
    w = qfgen.workload(name)
    gpu, orc = _pair(w.n, w.locs, w.kinds, w.const_mats, w.target_unitary(), w.initial(),
                     max_iters=w.max_iters)
    _check(gpu, orc)
    assert (orc.verdict == oracle.CONVERGED).sum() >= 1
    assert np.all(np.isin(orc.verdict, [oracle.CONVERGED, oracle.BATCH_STOPPED]))


def test_batch_plateau_path():
    n, locs, kinds, cm, V, init = _plateau_case()
    gpu, orc = _pair(n, locs, kinds, cm, V, init, max_iters=3000)
    _check(gpu, orc)
    assert np.all(np.isin(orc.verdict, [oracle.PLATEAU_SHORT, oracle.PLATEAU_LONG]))


def test_batch_c4_subset():
    """C4 shape (n = 6, 80 U(4)), 64 starts: every start stalls; the batch
    runs until the last one has hit its long plateau."""
    w = qfgen.workload("C4")
    init = w.initial(0, 64)
    gpu, orc = _pair(w.n, w.locs, w.kinds, w.const_mats, w.target_unitary(), init,
                     max_iters=w.max_iters)
    _check(gpu, orc)


def test_batch_reduce_other_rank_converges():
    """A callback that reports one converged start of another rank at sweep
    k: every start here stops at k, BATCH_STOPPED unless it had plateaued --
    the batch oracle capped at k, with MAX_ITER read as BATCH_STOPPED."""
    n, locs, kinds, cm, V, init = _plateau_case()
    k = 7
    calls = []

    def fn(user, counts, m):
        calls.append([counts[i] for i in range(m)])
        if len(calls) == k:
            counts[0] += 1
        return 0

    cb = qf.BATCH_REDUCE_FN(fn)
    gpu = qf.qf_instantiate(qf.Circuit(n, locs, kinds, cm), V, init,
                            batch_policy=qf.QF_BATCH_PAPER, batch_reduce=cb, max_iters=3000)
    orc = oracle.instantiate_batch(oracle.Circuit(n, locs, kinds, cm), V, init,
                                   oracle.default_params(max_iters=k))
    want = np.where(orc.verdict == oracle.MAX_ITER, oracle.BATCH_STOPPED, orc.verdict)
    assert len(calls) == k
    assert all(c[2] == init.shape[0] for c in calls)  # every start running
    assert np.array_equal(gpu.summary["verdict"], want)
    assert np.all(gpu.summary["iters"] == k)
    assert np.abs(gpu.summary["delta"] - orc.delta).max() < TOL


def test_batch_reduce_other_rank_never_plateaus():
    """Another rank that never plateaus holds the batch to max_iters."""
    n, locs, kinds, cm, V, init = _plateau_case()

    def fn(user, counts, m):
        counts[1] += 1
        counts[2] += 1
        return 0

    cb = qf.BATCH_REDUCE_FN(fn)
    cap = 400
    gpu = qf.qf_instantiate(qf.Circuit(n, locs, kinds, cm), V, init,
                            batch_policy=qf.QF_BATCH_PAPER, batch_reduce=cb, max_iters=cap)
    orc = oracle.instantiate(oracle.Circuit(n, locs, kinds, cm), V, init,
                             oracle.default_params(max_iters=cap))
    assert np.all(gpu.summary["iters"] == cap)
    plateaued = orc.iters < cap
    assert np.array_equal(gpu.summary["verdict"][plateaued], orc.verdict[plateaued])
    assert np.all(gpu.summary["verdict"][~plateaued] == oracle.MAX_ITER)


def test_batch_reduce_failure_is_reported():
    n, locs, kinds, cm, V, init = _plateau_case()
    cb = qf.BATCH_REDUCE_FN(lambda user, counts, m: 1)
    with pytest.raises(qf.QfError) as e:
        qf.qf_instantiate(qf.Circuit(n, locs, kinds, cm), V, init,
                          batch_policy=qf.QF_BATCH_PAPER, batch_reduce=cb, max_iters=10)
    assert e.value.status == qf.QF_E_NCCL


def test_batch_resident_matches_streaming():
    """The co-resident batch (one CTA per start, grid barrier per sweep) and
    the streaming batch (host decision per sweep) give the same verdicts and
    sweep counts, Delta within 1e-10."""
    import os

    w = qfgen.workload("C3+")
    c = qf.Circuit(w.n, w.locs, w.kinds, w.const_mats)
    V, init = w.target_unitary(), w.initial(0, 256)
    a = qf.qf_instantiate(c, V, init, batch_policy=qf.QF_BATCH_PAPER, max_iters=w.max_iters)
    old = os.environ.get("QF_RES_BATCH")
    os.environ["QF_RES_BATCH"] = "0"
    try:
        b = qf.qf_instantiate(c, V, init, batch_policy=qf.QF_BATCH_PAPER, max_iters=w.max_iters)
    finally:
        if old is None:
            del os.environ["QF_RES_BATCH"]
        else:
            os.environ["QF_RES_BATCH"] = old
    assert a.stats["engine"] == qf.QF_ENGINE_RESIDENT and b.stats["engine"] == qf.QF_ENGINE_STREAM
    assert np.array_equal(a.verdict, b.verdict) and np.array_equal(a.iters, b.iters)
    assert np.abs(a.delta - b.delta).max() < TOL


@pytest.mark.parametrize("policy", [qf.QF_BATCH_PER_START, qf.QF_BATCH_PAPER])
def test_numeric_fail_start_both_engines(policy, monkeypatch):
    """A start whose circuit tensor turns non-finite (fault injection,
    QF_DEBUG_POISON) fails alone: NUMERIC_FAIL after its first sweep, with the
    Delta and sweep count of that sweep, on the resident engine (cooperative
    batch launch) and on the streaming engine alike; the other starts are
    untouched (same results as the call without the fault)."""
    w = qfgen.workload("C3+")
    c = qf.Circuit.from_workload(w)
    V, init = w.target_unitary(), w.initial(0, 24)
    kw = dict(batch_policy=policy, max_iters=30)
    clean = qf.qf_instantiate(c, V, init, **kw)
    monkeypatch.setenv("QF_DEBUG_POISON", "5")
    res = qf.qf_instantiate(c, V, init, **kw)
    monkeypatch.setenv("QF_RES_BATCH", "0")
    stream = qf.qf_instantiate(c, V, init, engine=qf.QF_ENGINE_STREAM, **kw)
    for r in (res, stream):
        assert r.verdict[5] == qf.QF_NUMERIC_FAIL and r.iters[5] == 1, (r.verdict[5], r.iters[5])
        assert not np.isfinite(r.delta[5])
    assert np.array_equal(res.verdict, stream.verdict) and np.array_equal(res.iters, stream.iters)
    others = np.arange(24) != 5
    if policy == qf.QF_BATCH_PER_START:
        assert np.array_equal(res.summary[others], clean.summary[others])
    else:  # a failed start does not hold or stop the batch
        assert np.array_equal(res.verdict[others], clean.verdict[others])
        assert np.array_equal(res.iters[others], clean.iters[others])
