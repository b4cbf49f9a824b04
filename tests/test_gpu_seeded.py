"""Seeded multistarts inside the library ("The initial random unitaries
for each gate are controlled by a seed parameter"; initial ==
NULL => keyed Haar starts).  The device generator implements the same
counter-based SplitMix64 recipe as the input module qfgen (each side its own
code), so:
  * the gates it generates equal qfgen.initial_gates to 4e-14 (a few ulp);
  * a NULL-initial call meets the same oracle parity as the explicit call;
  * start s's gates depend only on (seed, start_offset + s, gate): sharding
    a job over calls with their own start_offset is bitwise invariant.
"""
import numpy as np
import pytest

import paper_2306_08152_b200 as qf
import qfgen
from test_gpu_parity import _compare, _oracle

pytestmark = pytest.mark.gpu


def _rz_template():
    locs = [(0,), (0, 1), (1,), (1, 2), (0, 1, 2), (2,)]
    kinds = [qfgen.RZ, qfgen.VARIABLE, qfgen.CONSTANT, qfgen.VARIABLE, qfgen.VARIABLE, qfgen.RZ]
    cm = [None, None, qfgen.haar(qfgen.stream_key(3, 9, 0, 0), 2)[0], None, None, None]
    return 3, locs, kinds, cm


@pytest.mark.parametrize("case", ["C1", "C4", "C5", "rz"])
def test_seeded_gates_match_input_module(case):
    """max_iters = 0 returns the starting gates untouched: they must be
    qfgen's (seed, global start, gate)-keyed Haar / R_z draws."""
    if case == "rz":
        n, locs, kinds, cm = _rz_template()
        V = qfgen.haar(qfgen.stream_key(5, qfgen.PURPOSE_TARGET, 0, 0), 8)[0]
        seed = 123456789012345
    else:
        w = qfgen.workload(case)
        n, locs, kinds, cm = w.n, w.locs, w.kinds, w.const_mats
        V, seed = w.target_unitary(), w.init_seed
    S, off = 37, 1000003
    c = qf.Circuit(n, locs, kinds, cm)
    r = qf.qf_instantiate(c, V, None, num_starts=S, seed=seed, start_offset=off, max_iters=0)
    ref = qfgen.initial_gates(n, locs, kinds, seed, off, S)
    # the transcendental functions (log, cos, sin) of the two sides differ in
    # the last ulp; Gram-Schmidt on d <= 8 columns spreads that to ~d eps
    assert np.abs(r.gates - ref).max() < 4e-14
    assert np.all(r.verdict == qf.QF_MAX_ITER)


def test_seeded_parity_against_oracle():
    """C2+ from a start count alone: same oracle parity (10 recorded sweeps,
    to verdict) as the call with qfgen's arrays, and the same verdicts."""
    w = qfgen.workload("C2+")
    c = qf.Circuit.from_workload(w)
    V = w.target_unitary()
    idx = np.arange(w.starts)
    gpu = qf.qf_instantiate(c, V, None, num_starts=w.starts, seed=w.init_seed,
                            record_starts=idx, record_sweeps=10, max_iters=w.max_iters)
    orc = _oracle(w.n, w.locs, w.kinds, w.const_mats, V, w.initial(), 10,
                  max_iters=w.max_iters)
    _compare(gpu, orc, idx, 10, 2 ** w.n)
    exp = qf.qf_instantiate(c, V, w.initial(), max_iters=w.max_iters)
    assert np.array_equal(gpu.verdict, exp.verdict) and np.array_equal(gpu.iters, exp.iters)
    assert np.abs(gpu.delta - exp.delta).max() < 1e-12


@pytest.mark.parametrize("engine", [qf.QF_ENGINE_STREAM, qf.QF_ENGINE_RESIDENT])
def test_seeded_shard_invariance_bitwise(engine):
    """100 seeded starts in one call == two calls of 50 with start_offset 0
    and 50 (the multi-GPU split), bitwise."""
    w = qfgen.workload("C3")
    c = qf.Circuit.from_workload(w)
    V = w.target_unitary()
    kw = dict(seed=w.init_seed, max_iters=200, engine=engine)
    a = qf.qf_instantiate(c, V, None, num_starts=100, **kw)
    b1 = qf.qf_instantiate(c, V, None, num_starts=50, start_offset=0, **kw)
    b2 = qf.qf_instantiate(c, V, None, num_starts=50, start_offset=50, **kw)
    assert np.array_equal(a.summary, np.concatenate([b1.summary, b2.summary]))
    assert np.array_equal(a.gates, np.concatenate([b1.gates, b2.gates]))


def test_seeded_device_entry():
    """qf_instantiate_device with d_initial = None equals the host call."""
    import torch

    w = qfgen.workload("C3+")
    c = qf.Circuit.from_workload(w)
    V = w.target_unitary()
    host = qf.qf_instantiate(c, V, None, num_starts=64, seed=7, start_offset=64, max_iters=40)
    dev = torch.device("cuda:0")
    dV = torch.from_numpy(np.ascontiguousarray(V)).to(dev)
    ws = torch.empty(qf.qf_workspace_size(c, 64, max_iters=40), dtype=torch.uint8, device=dev)
    gout = torch.empty((64, c.var_doubles), dtype=torch.float64, device=dev)
    r = qf.qf_instantiate_device(c, dV, None, ws, d_gates_out=gout, num_starts=64, seed=7,
                                 start_offset=64, max_iters=40)
    torch.cuda.synchronize()
    assert np.array_equal(r.summary, host.summary)
    assert np.array_equal(gout.cpu().numpy(), host.gates)
