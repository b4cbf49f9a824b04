"""NEXT-4: update variants, CPU side.
  - R_z(theta) gates (reading R19): the oracle's analytic update is
    pinned by brute force over theta and by the closed-form maximum
    Re M_00 + |M_11|; a sweep with R_z gates never lowers |Tr|;
    a single R_z gate reaches a reachable target in one update.
  - U3 / ZYZ angle extraction: e^{i gamma} U3(theta, phi,
    lambda) rebuilds u (exact to rounding), angles in their ranges."""
import numpy as np
import pytest

import paper_2306_08152_b200 as qf
import qfgen
from helpers import haar_np


def _rz(t):
    return np.diag([1.0, np.exp(1j * t)])


def _u3(t, p, l):
    return np.array([[np.cos(t / 2), -np.exp(1j * l) * np.sin(t / 2)],
                     [np.exp(1j * p) * np.sin(t / 2), np.exp(1j * (p + l)) * np.cos(t / 2)]])


@pytest.mark.parametrize("beta", [0.0, 0.3])
def test_rz_update_brute_force(orc, beta):
    rng = np.random.default_rng(538)
    grid = np.linspace(0, 2 * np.pi, 200001)
    for _ in range(50):
        E = rng.standard_normal((2, 2)) + 1j * rng.standard_normal((2, 2))
        u_old = _rz(rng.uniform(0, 2 * np.pi))
        u = orc.optimize_rz(E, u_old, beta)
        M = (1 - beta) * E + beta * u_old.conj().T
        val = np.real(np.trace(M @ u))
        brute = np.max(np.real(M[0, 0] + M[1, 1] * np.exp(1j * grid)))
        assert val >= brute - 1e-12
        assert abs(val - (M[0, 0].real + abs(M[1, 1]))) < 1e-12  # closed-form maximum
        assert np.allclose(u[0], [1, 0]) and abs(u[1, 0]) == 0 and abs(abs(u[1, 1]) - 1) < 1e-15
    E = np.array([[1.0, 2.0], [3.0, 0.0]], dtype=complex)  # M_11 = 0: keep u_old
    assert np.array_equal(orc.optimize_rz(E, _rz(0.7), 0.0), _rz(0.7))


def _rz_template():
    """3 qubits: U(2) layer, then 3 x [CNOT(0,1), RZ q1, CNOT(1,2), RZ q2, U(2) q0]."""
    cx = np.eye(4)[[0, 1, 3, 2]]
    locs, kinds, cm = [(0,), (1,), (2,)], [qfgen.VARIABLE] * 3, [None] * 3
    for _ in range(3):
        locs += [(0, 1), (1,), (1, 2), (2,), (0,)]
        kinds += [qfgen.CONSTANT, qfgen.RZ, qfgen.CONSTANT, qfgen.RZ, qfgen.VARIABLE]
        cm += [cx, None, cx, None, None]
    return 3, locs, kinds, cm


def test_rz_sweep_monotone(orc):
    n, locs, kinds, cm = _rz_template()
    C = orc.Circuit(n, locs, kinds, cm)
    V = haar_np(np.random.default_rng(5), 8)
    g = qfgen.initial_gates(n, locs, kinds, 77, 0, 1)[0]
    ct = orc.init_ct(C, V, g)
    # every update maximises Re Tr(E u): Re Tr never drops
    # (|Tr| may: an R_z update cannot rotate the phase of Tr freely)
    last = -np.inf
    for _ in range(5):
        ct, g, log = orc.sweep(C, ct, g, log=True)
        a = np.real(log)
        assert a[0] >= last - 1e-12 and np.all(np.diff(a) >= -1e-12)
        last = a[-1]
    for u, k in zip(qfgen.unpack_gates(locs, kinds, g), kinds):  # R_z form kept
        if k == qfgen.RZ:
            assert abs(u[0, 0] - 1) < 1e-15 and abs(u[0, 1]) == 0 and abs(u[1, 0]) == 0


def test_rz_single_gate_reaches_target(orc):
    """One R_z gate, target R_z(theta*): the first update is exact.  (With a
    global phase on the target it is not: R_z's fixed 1 cannot absorb the
    phase, and the update maximises Re Tr, not |Tr|.)"""
    C = orc.Circuit(1, [(0,)], [qfgen.RZ], [None])
    V = _rz(2.1)
    r = orc.instantiate(C, V, qfgen.initial_gates(1, [(0,)], [qfgen.RZ], 3, 0, 4),
                        orc.default_params(max_iters=5))
    assert np.all(r.delta < 1e-15) and np.all(r.verdict == orc.CONVERGED) and np.all(r.iters == 1)


def test_rz_rejected_on_two_qubits():
    with pytest.raises(qf.QfError) as e:
        qf.Circuit(2, [(0, 1)], [qfgen.RZ], [None])
    assert e.value.status == qf.QF_E_ARG


def test_u3_angles_rebuild():
    rng = np.random.default_rng(173)
    cases = [haar_np(rng, 2) for _ in range(300)]
    cases += [np.eye(2), np.diag([1, -1]), np.array([[0, 1], [1, 0]]), np.array([[0, 1j], [1j, 0]]),
              np.exp(0.3j) * _rz(1.2), np.array([[1, 1], [1, -1]]) / np.sqrt(2),
              np.exp(-2.0j) * np.array([[0, -np.exp(0.5j)], [np.exp(-1.1j), 0]])]
    for u in cases:
        t, p, l, g = qf.qf_unitary_to_u3(u)
        assert 0 <= t <= np.pi
        for a in (p, l, g):
            assert -np.pi < a <= np.pi
        assert np.abs(np.exp(1j * g) * _u3(t, p, l) - u).max() < 1e-13, u
    with pytest.raises(qf.QfError) as e:
        qf.qf_unitary_to_u3(np.array([[1, 1], [0, 1]]))
    assert e.value.status == qf.QF_E_NOT_UNITARY
