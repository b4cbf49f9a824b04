"""Input generators (qfgen): determinism, sharding invariance, Haar sanity,
and the dense circuit unitary against an independent Kronecker build."""
import json
import os

import numpy as np
import pytest

import qfgen
from helpers import dense_circuit, dense_embed

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_haar_unitary_and_deterministic():
    for d in (2, 4, 8, 16):
        keys = qfgen.stream_key(7, 1, np.arange(50), 3)
        U = qfgen.haar(keys, d)
        I = np.eye(d)
        err = np.abs(np.einsum("kji,kjl->kil", U.conj(), U) - I).max()
        assert err < 1e-13
        assert np.array_equal(U, qfgen.haar(keys, d))


def test_haar_moments():
    # E|U_00|^2 = 1/d and E U_00 = 0 under Haar measure
    d = 4
    U = qfgen.haar(qfgen.stream_key(11, 1, np.arange(20000), 0), d)
    assert abs(np.mean(np.abs(U[:, 0, 0]) ** 2) - 1 / d) < 0.01
    assert abs(np.mean(U[:, 0, 0])) < 0.02


def test_initial_gates_shard_invariant():
    w = qfgen.workload("C3")
    a = w.initial(0, 40)
    b = w.initial(17, 9)
    assert np.array_equal(a[17:26], b)


def test_cnot_golden_and_embedding():
    g = json.load(open(os.path.join(GOLD, "cnot_S141.json")))
    assert np.array_equal(qfgen.CNOT.real, np.array(g["matrix"]))
    # CNOT on (2, 0) of n = 3: i -> i ^ (4 * (i & 1))
    U = qfgen.circuit_unitary(3, [(2, 0)], [qfgen.CONSTANT], [qfgen.CNOT], np.zeros(0))
    P = np.zeros((8, 8))
    for i in range(8):
        P[i ^ (4 * (i & 1)), i] = 1
    assert np.array_equal(U, P)


def test_x_embedding_kron():
    X = np.array([[0, 1], [1, 0]], dtype=complex)
    I = np.eye(2)
    for loc, ref in (((0,), np.kron(X, I)), ((1,), np.kron(I, X))):
        U = qfgen.circuit_unitary(2, [loc], [qfgen.CONSTANT], [X], np.zeros(0))
        assert np.array_equal(U, ref)


@pytest.mark.parametrize("seed", range(4))
def test_circuit_unitary_matches_kron_build(seed):
    n = 4
    locs, kinds, cm = qfgen.random_template(n, 9, seed=seed, const_frac=0.3)
    packed = qfgen.initial_gates(n, locs, kinds, 5, 0, 1)[0]
    U = qfgen.circuit_unitary(n, locs, kinds, cm, packed)
    mats = [m if k == qfgen.CONSTANT else u
            for m, k, u in zip(cm, kinds, qfgen.unpack_gates(locs, kinds, packed))]
    assert np.abs(U - dense_circuit(n, locs, mats)).max() < 1e-13


def test_workload_shapes():
    c1 = qfgen.workload("C1")
    assert (c1.n, c1.p, c1.starts) == (2, 11, 4)
    assert sum(k == qfgen.CONSTANT for k in c1.kinds) == 3
    c2 = qfgen.workload("C2")
    assert (c2.n, c2.p, c2.starts) == (3, 45, 64)
    assert sum(k == qfgen.CONSTANT for k in c2.kinds) == 14
    c3 = qfgen.workload("C3")
    assert (c3.n, c3.p, c3.starts) == (4, 20, 1024)
    c4 = qfgen.workload("C4")
    assert (c4.n, c4.p, c4.starts) == (6, 80, 4096)
    c5 = qfgen.workload("C5")
    assert (c5.n, c5.p, c5.starts) == (8, 200, 8192)
    assert sum(len(l) == 2 for l in c5.locs) == 110
    assert sum(len(l) == 3 for l in c5.locs) == 90
    for name in qfgen.ALL:
        w = qfgen.workload(name)
        for l in w.locs:
            assert len(set(l)) == len(l) and all(0 <= q < w.n for q in l)


def test_self_target_unitary():
    w = qfgen.workload("C3")
    V = w.target_unitary()
    assert np.abs(V.conj().T @ V - np.eye(16)).max() < 1e-12
