"""NEXT-3 on the GPU: grouped steps on the streaming engine (QF_GROUP=umax,
k_group + one sandwich pass per group) against the oracle, north_star
tolerances as tests/test_gpu_parity.py; the grouping must also cut the
sandwich passes."""
import os

import numpy as np
import pytest

import paper_2306_08152_b200 as qf
import qfgen
from helpers import haar_np
from test_gpu_parity import _compare, _run_pair

pytestmark = pytest.mark.gpu


def u3_cnot_template(n, layers):
    """The paper's gate set (U3 + CNOT): a VAR U(2) on every qubit,
    then `layers` x [CNOT(i, i+1), VAR U(2) on i, VAR U(2) on i+1] along a
    ladder."""
    cx = np.eye(4)[[0, 1, 3, 2]]
    locs, kinds, cm = [(q,) for q in range(n)], [qfgen.VARIABLE] * n, [None] * n
    for l in range(layers):
        i = l % (n - 1)
        locs += [(i, i + 1), (i,), (i + 1,)]
        kinds += [qfgen.CONSTANT, qfgen.VARIABLE, qfgen.VARIABLE]
        cm += [cx, None, None]
    return locs, kinds, cm


@pytest.fixture
def group(request):
    old = os.environ.get("QF_GROUP")
    os.environ["QF_GROUP"] = str(request.param)
    yield request.param
    if old is None:
        del os.environ["QF_GROUP"]
    else:
        os.environ["QF_GROUP"] = old


@pytest.mark.parametrize("group", [2, 3], indirect=True)
def test_grouped_u3_cnot(group):
    n = 8
    locs, kinds, cm = u3_cnot_template(n, 10)
    V = haar_np(np.random.default_rng(11), 2 ** n)
    init = qfgen.initial_gates(n, locs, kinds, 5100, 0, 12)
    gpu, orc, idx = _run_pair(n, locs, kinds, cm, V, init, R=5, max_iters=5,
                              engine=qf.QF_ENGINE_STREAM)
    _compare(gpu, orc, idx, 5, 2 ** n)
    # 2p = 76 steps per sweep; a CNOT and its two U(2)s share a pair
    passes_per_sweep = gpu.stats["sandwich_launches"] / 5
    assert passes_per_sweep < 2 * len(locs) * 0.6, passes_per_sweep


@pytest.mark.parametrize("group", [1, 2, 3], indirect=True)
@pytest.mark.parametrize("n,p,seed", [(7, 9, 61), (8, 7, 62), (9, 5, 63)])
def test_grouped_random(group, n, p, seed):
    locs, kinds, cm = qfgen.random_template(n, p, seed=seed, const_frac=0.3)
    V = qfgen.haar(qfgen.stream_key(seed, qfgen.PURPOSE_TARGET, 0, 0), 2 ** n)[0]
    init = qfgen.initial_gates(n, locs, kinds, 5200 + seed, 0, 9)
    gpu, orc, idx = _run_pair(n, locs, kinds, cm, V, init, R=4, max_iters=4,
                              engine=qf.QF_ENGINE_STREAM)
    _compare(gpu, orc, idx, 4, 2 ** n)


@pytest.mark.parametrize("group", [3], indirect=True)
def test_grouped_c5_sample(group):
    w = qfgen.workload("C5")
    init = w.initial(0, 6)
    gpu, orc, idx = _run_pair(w.n, w.locs, w.kinds, w.const_mats, w.target_unitary(), init,
                              R=2, max_iters=2, engine=qf.QF_ENGINE_STREAM)
    _compare(gpu, orc, idx, 2, 2 ** w.n)


@pytest.mark.parametrize("group", [3], indirect=True)
@pytest.mark.parametrize("n,p,seed", [(8, 9, 64), (9, 7, 65)])
def test_grouped_fused_partials(group, n, p, seed, monkeypatch):
    """QF_GROUP_FUSE=1: a d = 8 group flush on the row-tile kernel leaves the
    next group's T as tile partials (W as a pseudo-gate) and k_group sums them
    instead of gathering; same oracle bar (DESIGN 9e; off by default)."""
    monkeypatch.setenv("QF_GROUP_FUSE", "1")
    locs, kinds, cm = qfgen.random_template(n, p, seed=seed, const_frac=0.2)
    V = qfgen.haar(qfgen.stream_key(seed, qfgen.PURPOSE_TARGET, 0, 0), 2 ** n)[0]
    init = qfgen.initial_gates(n, locs, kinds, 5300 + seed, 0, 6)
    gpu, orc, idx = _run_pair(n, locs, kinds, cm, V, init, R=4, max_iters=4,
                              engine=qf.QF_ENGINE_STREAM)
    _compare(gpu, orc, idx, 4, 2 ** n)
    # the partial path really ran: the gather path sums in another order
    monkeypatch.setenv("QF_GROUP_FUSE", "0")
    c = qf.Circuit(n, locs, kinds, cm)
    ref = qf.qf_instantiate(c, V, init, max_iters=4, engine=qf.QF_ENGINE_STREAM)
    assert not np.array_equal(gpu.gates, ref.gates)
    assert np.max(np.abs(gpu.gates - ref.gates)) < 1e-11
