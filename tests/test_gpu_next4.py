"""NEXT-4 on the GPU: templates with R_z(theta) gates (analytic update,
P:538-575, reading R19) and beta regularisation, both engines, against the
oracle (north_star tolerances, as tests/test_gpu_parity.py)."""
import numpy as np
import pytest

import paper_2306_08152_b200 as qf
import qfgen
from helpers import haar_np
from test_gpu_parity import ENGINES, _compare, _run_pair
from test_next4 import _rz_template

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("beta", [0.0, 0.25])
def test_parity_rz_template(engine, beta):
    n, locs, kinds, cm = _rz_template()
    V = haar_np(np.random.default_rng(9), 8)
    init = qfgen.initial_gates(n, locs, kinds, 4100, 0, 33)
    gpu, orc, idx = _run_pair(n, locs, kinds, cm, V, init, R=10, max_iters=60, engine=engine,
                              beta=beta)
    _compare(gpu, orc, idx, 10, 2 ** n)


@pytest.mark.parametrize("engine", ENGINES)
def test_parity_rz_mixed_random(engine):
    """Random template on 5 qubits with every 1-qubit gate an R_z."""
    locs, kinds, cm = qfgen.random_template(5, 12, arities=(1, 2), seed=41, const_frac=0.2)
    kinds = [qfgen.RZ if (k == qfgen.VARIABLE and len(l) == 1) else k for l, k in zip(locs, kinds)]
    V = haar_np(np.random.default_rng(41), 32)
    init = qfgen.initial_gates(5, locs, kinds, 4200, 0, 21)
    gpu, orc, idx = _run_pair(5, locs, kinds, cm, V, init, R=8, max_iters=8, engine=engine)
    _compare(gpu, orc, idx, 8, 32)


def test_rz_initial_form_checked():
    n, locs, kinds, cm = _rz_template()
    init = qfgen.initial_gates(n, locs, kinds, 4100, 0, 2)
    init[1, 3 * 8: 3 * 8 + 8] = qfgen.haar(qfgen.stream_key(1, 1, 0, 0), 2)[0].view(np.float64).ravel()
    with pytest.raises(qf.QfError) as e:
        qf.qf_instantiate(qf.Circuit(n, locs, kinds, cm), haar_np(np.random.default_rng(1), 8), init,
                          max_iters=3)
    assert e.value.status == qf.QF_E_NOT_UNITARY
