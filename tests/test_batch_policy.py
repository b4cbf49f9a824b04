"""NEXT-1: the paper's GPU multistart termination (
DESIGN.md reading R22), oracle side.

The batch oracle is pinned to the per-start oracle (itself pinned in
test_oracle_pins.py) through what the definition fixes, given that starts
never exchange data (their trajectories are the same whether they run alone
or in a batch):
  - a batch of one start is the per-start run;
  - on a template where every start converges, the batch stops at the first
    sweep any start converges; the others are BATCH_STOPPED with the cost
    their own trajectory has at that sweep;
  - on a template where every start plateaus, the batch stops at the last
    first-plateau sweep, each start keeping the kind its own run stopped on;
  - a max_iters cap below that stops the batch at the cap (MAX_ITER for the
    starts that had not plateaued yet)."""
import numpy as np
import pytest

import qfgen
from helpers import haar_np


def _circ(orc, w):
    return orc.Circuit(w.n, w.locs, w.kinds, w.const_mats)


def _plateau_case():
    """3 qubits, 3 VARIABLE U(4) gates, Haar target: too few parameters to
    reach the target (Delta stays ~1e-1), so every start plateaus fast."""
    rng = np.random.default_rng(2306)
    locs = [(0, 1), (1, 2), (0, 1)]
    kinds = [qfgen.VARIABLE] * 3
    V = haar_np(rng, 8)
    S = 12
    init = np.stack([np.concatenate([haar_np(rng, 4).view(np.float64).ravel() for _ in locs])
                     for _ in range(S)])
    return 3, locs, kinds, V, init


def test_batch_of_one_is_per_start(orc):
    w = qfgen.workload("C1")
    C = _circ(orc, w)
    P = orc.default_params(max_iters=w.max_iters)
    init = w.initial()
    per = orc.instantiate(C, w.target_unitary(), init, P)
    for s in range(init.shape[0]):
        b = orc.instantiate_batch(C, w.target_unitary(), init[s:s + 1], P)
        assert b.verdict[0] == per.verdict[s] and b.iters[0] == per.iters[s]
        assert b.delta[0] == per.delta[s]
        assert np.array_equal(b.gates[0], per.gates[s])
    n, locs, kinds, V, init = _plateau_case()
    C = orc.Circuit(n, locs, kinds, [None] * len(locs))
    P = orc.default_params(max_iters=3000)
    per = orc.instantiate(C, V, init, P)
    for s in range(3):
        b = orc.instantiate_batch(C, V, init[s:s + 1], P)
        assert (b.verdict[0], b.iters[0], b.delta[0]) == (per.verdict[s], per.iters[s], per.delta[s])


@pytest.mark.parametrize("name", ["C1", "C2+"])
def test_batch_stops_on_first_success(orc, name):
    w = qfgen.workload(name)
    C = _circ(orc, w)
    P = orc.default_params(max_iters=w.max_iters)
    init = w.initial()
    per = orc.instantiate(C, w.target_unitary(), init, P, record_sweeps=w.max_iters)
    assert np.all(per.verdict == orc.CONVERGED)  # the success-path template
    T = int(per.iters.min())
    b = orc.instantiate_batch(C, w.target_unitary(), init, P)
    assert np.all(b.iters == T)
    first = per.iters == T
    assert np.array_equal(b.verdict == orc.CONVERGED, first)
    assert np.all(b.verdict[~first] == orc.BATCH_STOPPED)
    # every start's Delta is its own trajectory's cost at sweep T
    assert np.array_equal(b.delta, per.cost_hist[:, T - 1])


def test_batch_waits_for_every_plateau(orc):
    n, locs, kinds, V, init = _plateau_case()
    C = orc.Circuit(n, locs, kinds, [None] * len(locs))
    P = orc.default_params(max_iters=3000)
    per = orc.instantiate(C, V, init, P, record_sweeps=3000)
    assert np.all((per.verdict == orc.PLATEAU_SHORT) | (per.verdict == orc.PLATEAU_LONG))
    assert per.iters.min() < per.iters.max()  # the batch really waits
    T = int(per.iters.max())
    b = orc.instantiate_batch(C, V, init, P)
    assert np.all(b.iters == T)
    assert np.array_equal(b.verdict, per.verdict)  # first plateau kind kept
    last = per.iters == T
    assert np.array_equal(b.delta[last], per.delta[last])
    assert np.all(b.delta[~last] > 1e-3)  # still far from the target: no escape here

    # a cap below the last plateau: MAX_ITER for the starts still unplateaued
    cap = int(np.sort(per.iters)[len(per.iters) // 2])
    Pc = orc.default_params(max_iters=cap)
    bc = orc.instantiate_batch(C, V, init, Pc)
    assert np.all(bc.iters == cap)
    done = per.iters <= cap
    assert np.array_equal(bc.verdict[done], per.verdict[done])
    assert np.all(bc.verdict[~done] == orc.MAX_ITER)
    alive = per.iters >= cap  # own trajectory known at the cap
    assert np.array_equal(bc.delta[alive], per.cost_hist[alive, cap - 1])


def test_batch_max_iter_zero(orc):
    w = qfgen.workload("C2+")
    C = _circ(orc, w)
    g = w.initial(0, 3)
    a = orc.instantiate(C, w.target_unitary(), g, orc.default_params(max_iters=0))
    b = orc.instantiate_batch(C, w.target_unitary(), g, orc.default_params(max_iters=0))
    assert np.all(b.verdict == orc.MAX_ITER) and np.all(b.iters == 0)
    assert np.array_equal(a.delta, b.delta)
