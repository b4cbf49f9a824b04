"""Pins of the CPU oracle against facts the paper and mathematics fix.

What pins each oracle function (none of these retypes the oracle's formula):
  apply_left/right -- dense Kronecker+permutation embedding (helpers.dense_embed)
                      and numpy tensordot circuit unitary; inverse cancellation
                      (SPEC S:259); identity gate.
  env              -- brute force by linearity: E[a,b] =
                      Tr(V^dag C_k[|b><a|]) with dense circuits; Tr(E u_k) =
                      Tr(V^dag U); linearity; golden S:275.
  trace            -- numpy trace; eq:cost identity (golden S:350).
  svd              -- reconstruction + unitarity; singular values equal numpy's
                      LAPACK values; rank-deficient diag(3,0).
  optimize_gate    -- Procrustes closed form via numpy SVD; Re Tr(E u_new) =
                      sum sigma; beats 1000 Haar unitaries;
                      dense 1-qubit grid e^{i g}U3 (north_star); beta limits
                      (P:526-528).
  init_ct/sweep    -- full-matrix equality ct = U_dense V^dag after init and
                      after every sweep; |Tr| non-decreasing over single
                      updates; |Tr| <= N; special cases
                      (self-target fixed point, whole-register gate, product
                      target, C1 KAK universality, global phase invariance);
                      the half-sweep order p..1 then 1..p by a
                      dense brute-force sweep with LAPACK Procrustes updates.
  terminate        -- hand-built cost sequences for every verdict.
"""
import json
import os

import numpy as np
import pytest

import qfgen
from helpers import dense_circuit, dense_embed, ginibre, haar_np, pack, u3

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rand_ct(rng, n):
    N = 2 ** n
    return rng.standard_normal((N, N)) + 1j * rng.standard_normal((N, N))


# ------------------------------------------------------------------ apply
@pytest.mark.parametrize("n,loc", [(1, (0,)), (2, (1,)), (2, (1, 0)), (3, (0, 2)),
                                   (3, (2, 0, 1)), (4, (3,)), (4, (1, 3)), (5, (4, 0, 2)),
                                   (5, (2, 3))])
def test_apply_matches_dense_embedding(orc, n, loc):
    rng = np.random.default_rng(n * 31 + len(loc))
    ct = rand_ct(rng, n)
    u = ginibre(rng, 2 ** len(loc))  # any matrix: E is linear in u
    E = dense_embed(n, loc, u)
    assert np.abs(orc.apply_left(ct, u, loc) - E @ ct).max() < 1e-12
    assert np.abs(orc.apply_right(ct, u, loc) - ct @ E).max() < 1e-12
    Ed = dense_embed(n, loc, u.conj().T)
    assert np.abs(orc.apply_left(ct, u, loc, True) - Ed @ ct).max() < 1e-12
    assert np.abs(orc.apply_right(ct, u, loc, True) - ct @ Ed).max() < 1e-12
    # tensordot-built single-gate unitary (independent of dense_embed)
    T = qfgen.circuit_unitary(n, [loc], [qfgen.CONSTANT], [u], np.zeros(0))
    assert np.abs(T - E).max() < 1e-12


def test_apply_inverse_cancels_and_identity(orc):
    rng = np.random.default_rng(3)
    ct = rand_ct(rng, 4)
    u = haar_np(rng, 4)
    for loc in ((0, 3), (2, 1)):
        a = orc.apply_left(orc.apply_left(ct, u, loc), u, loc, True)
        b = orc.apply_right(orc.apply_right(ct, u, loc), u, loc, True)
        assert np.abs(a - ct).max() < 1e-12 and np.abs(b - ct).max() < 1e-12
        assert np.array_equal(orc.apply_left(ct, np.eye(4), loc), ct)


# ------------------------------------------------------------------ env
def _brute_env(n, locs, mats, V, k):
    """E[a,b] = Tr(V^dag C_k[|b><a|]) (linearity of Tr(V^dag U) in u_k)."""
    d = 2 ** len(locs[k])
    E = np.zeros((d, d), dtype=complex)
    for a in range(d):
        for b in range(d):
            unit = np.zeros((d, d), dtype=complex)
            unit[b, a] = 1.0
            mk = list(mats)
            mk[k] = unit
            E[a, b] = np.trace(V.conj().T @ dense_circuit(n, locs, mk))
    return E


@pytest.mark.parametrize("seed", range(6))
def test_env_brute_force(orc, seed):
    rng = np.random.default_rng(100 + seed)
    n = 3 + seed % 2
    locs, kinds, cm = qfgen.random_template(n, 6, seed=seed)
    mats = [haar_np(rng, 2 ** len(l)) for l in locs]
    V = haar_np(rng, 2 ** n)
    p = len(locs)
    for k in range(p):
        # peeled tensor at step k: E(u_{k-1})..E(u_1) V^dag E(u_p)..E(u_{k+1})
        ct = V.conj().T.copy()
        for j in range(k):
            ct = orc.apply_left(ct, mats[j], locs[j])
        for j in range(p - 1, k, -1):
            ct = orc.apply_right(ct, mats[j], locs[j])
        E = orc.env(ct, locs[k])
        assert np.abs(E - _brute_env(n, locs, mats, V, k)).max() < 1e-12
        # Tr(E u_k) = Tr(V^dag U)
        tr = np.trace(V.conj().T @ dense_circuit(n, locs, mats))
        assert abs(np.trace(E @ mats[k]) - tr) < 1e-12
        # linearity
        x, y = haar_np(rng, E.shape[0]), haar_np(rng, E.shape[0])
        al, be = 0.3 - 0.7j, 1.1 + 0.2j
        assert abs(np.trace(E @ (al * x + be * y)) - al * np.trace(E @ x)
                   - be * np.trace(E @ y)) < 1e-12


def test_env_golden_S275(orc):
    g = json.load(open(os.path.join(GOLD, "env_identity_S275.json")))
    E = orc.env(np.eye(2 ** g["n"], dtype=complex), tuple(g["location"]))
    ref = np.array(g["env_re"]) + 1j * np.array(g["env_im"])
    assert np.array_equal(E, ref)


# ------------------------------------------------------------------ cost
def test_cost_identity_eq_cost(orc):
    g = json.load(open(os.path.join(GOLD, "frob_S350.json")))
    V, U = np.array(g["V_re"], dtype=complex), np.array(g["U_re"], dtype=complex)
    re_tr = orc.trace(V.conj().T @ U).real
    assert re_tr == g["re_trace"]
    n = g["n"]
    assert 2 ** (n + 1) * (1 - re_tr / 2 ** n) == g["frob_sq"] == np.sum(np.abs(U - V) ** 2)
    rng = np.random.default_rng(5)
    for _ in range(200):
        n = int(rng.integers(1, 5))
        U, V = haar_np(rng, 2 ** n), haar_np(rng, 2 ** n)
        tr = orc.trace(V.conj().T @ U)
        assert abs(tr - np.trace(V.conj().T @ U)) < 1e-12
        lhs = np.sum(np.abs(U - V) ** 2)
        assert abs(lhs - 2 ** (n + 1) * (1 - tr.real / 2 ** n)) < 1e-9
        # Delta and the phase-aligned Frobenius distance: ||e^{-i phi}U - V||^2 = 2N Delta
        delta = 1 - abs(tr) / 2 ** n
        ph = np.exp(-1j * np.angle(tr))
        assert abs(np.sum(np.abs(ph * U - V) ** 2) - 2 * 2 ** n * delta) < 1e-9


# ------------------------------------------------------------------ svd
@pytest.mark.parametrize("d", [2, 4, 8, 16])
def test_svd_reconstruction(orc, d):
    rng = np.random.default_rng(d)
    for _ in range(25):
        M = ginibre(rng, d)
        X, D, Y = orc.svd(M)
        assert np.abs(X @ np.diag(D) @ Y.conj().T - M).max() < 1e-12
        assert np.abs(X.conj().T @ X - np.eye(d)).max() < 1e-12
        assert np.abs(Y.conj().T @ Y - np.eye(d)).max() < 1e-12
        assert np.all(np.diff(D) <= 0)
        assert np.abs(D - np.linalg.svd(M, compute_uv=False)).max() < 1e-12


def test_svd_rank_deficient_S73(orc):
    M = np.diag([3.0, 0.0]).astype(complex)
    X, D, Y = orc.svd(M)
    assert np.array_equal(D, [3.0, 0.0])
    assert np.abs(X @ np.diag(D) @ Y.conj().T - M).max() == 0.0
    assert np.abs(X.conj().T @ X - np.eye(2)).max() < 1e-15
    X, D, Y = orc.svd(np.eye(2, dtype=complex))
    assert np.array_equal(D, [1.0, 1.0])
    # rank-1 4x4 and zero matrix still give unitary factors
    rng = np.random.default_rng(0)
    v = ginibre(rng, 4)[:, :1]
    for M in (v @ v.conj().T, np.zeros((4, 4), dtype=complex)):
        X, D, Y = orc.svd(M)
        assert np.abs(X.conj().T @ X - np.eye(4)).max() < 1e-12
        assert np.abs(X @ np.diag(D) @ Y.conj().T - M).max() < 1e-12


# ------------------------------------------------------------------ update
@pytest.mark.parametrize("d", [2, 4, 8])
def test_optimize_gate_procrustes(orc, d):
    rng = np.random.default_rng(40 + d)
    for _ in range(100):
        E = ginibre(rng, d)
        u, ssum = orc.optimize_gate(E, haar_np(rng, d))
        assert np.abs(u.conj().T @ u - np.eye(d)).max() < 1e-12
        # textbook Procrustes: argmax Re Tr(E u) = V_E U_E^dag for E = U_E S V_E^dag
        Ue, s, Vh = np.linalg.svd(E)
        ustar = Vh.conj().T @ Ue.conj().T
        assert np.abs(u - ustar).max() < 1e-10
        val = np.trace(E @ u).real
        assert abs(val - s.sum()) < 1e-12 * max(1, s.sum())
        assert abs(ssum - s.sum()) < 1e-12 * max(1, s.sum())
    # 1000 random unitaries never beat it
    E = ginibre(rng, d)
    u, _ = orc.optimize_gate(E, np.eye(d))
    best = np.trace(E @ u).real
    for _ in range(1000):
        assert np.trace(E @ haar_np(rng, d)).real <= best + 1e-10


def test_optimize_gate_special_S83_S362(orc):
    rng = np.random.default_rng(9)
    assert np.abs(orc.optimize_gate(np.eye(2, dtype=complex), haar_np(rng, 2))[0]
                  - np.eye(2)).max() < 1e-15
    W = haar_np(rng, 4)
    assert np.abs(orc.optimize_gate(W, np.eye(4))[0] - W.conj().T).max() < 1e-12


def test_optimize_gate_grid_1q(orc):
    """Each single-gate update is the brute-force optimum over a dense grid of
    U(2) = e^{i g} U3(theta, phi, lambda) (north_star)."""
    rng = np.random.default_rng(77)
    K = 48
    th = np.linspace(0, np.pi, K)
    an = np.linspace(-np.pi, np.pi, K, endpoint=False)
    T, P, L, G = np.meshgrid(th, an, an, an, indexing="ij")
    c, s = np.cos(T / 2), np.sin(T / 2)
    eg = np.exp(1j * G)
    U = np.stack([np.stack([c, -np.exp(1j * L) * s], -1),
                  np.stack([np.exp(1j * P) * s, np.exp(1j * (P + L)) * c], -1)], -2)
    U = U * eg[..., None, None]
    assert np.abs(U[3, 5, 7, 9] - np.exp(1j * G[3, 5, 7, 9]) * u3(T[3, 5, 7, 9], P[3, 5, 7, 9],
                                                                   L[3, 5, 7, 9])).max() < 1e-14
    for _ in range(3):
        E = ginibre(rng, 2)
        u, ssum = orc.optimize_gate(E, np.eye(2))
        val = np.trace(E @ u).real
        grid = np.einsum("ab,...ba->...", E, U).real
        assert val >= grid.max() - 1e-12
        assert val <= ssum + 1e-12
        assert grid.max() > val - 0.05  # the grid is fine enough to come close


def test_beta_limits(orc):
    """beta = 1 keeps the gate; beta = 0.5 maximises Re Tr(M u)."""
    rng = np.random.default_rng(4)
    E, u0 = ginibre(rng, 4), haar_np(rng, 4)
    u1, _ = orc.optimize_gate(E, u0, beta=1.0)
    assert np.abs(u1 - u0).max() < 1e-12
    u5, _ = orc.optimize_gate(E, u0, beta=0.5)
    M = 0.5 * E + 0.5 * u0.conj().T
    assert abs(np.trace(M @ u5).real - np.linalg.svd(M, compute_uv=False).sum()) < 1e-12


# ------------------------------------------------------------------ init / sweep
def _circ(orc, n, locs, kinds, cm):
    return orc.Circuit(n, locs, kinds, cm)


def _mats(locs, kinds, cm, packed):
    return [c if k == qfgen.CONSTANT else u
            for c, k, u in zip(cm, kinds, qfgen.unpack_gates(locs, kinds, packed))]


@pytest.mark.parametrize("seed", range(4))
def test_init_and_sweep_bookkeeping(orc, seed):
    """After init and after every sweep, ct = U_dense(current gates) V^dag as a
    full matrix (InitCircuitTensor P:584-592, TwoSidedSweep P:596-621)."""
    n = 3 + seed % 2
    locs, kinds, cm = qfgen.random_template(n, 8, seed=seed, const_frac=0.25)
    rng = np.random.default_rng(seed)
    V = haar_np(rng, 2 ** n)
    g = qfgen.initial_gates(n, locs, kinds, 50 + seed, 0, 1)[0]
    C = _circ(orc, n, locs, kinds, cm)
    ct = orc.init_ct(C, V, g)
    U = dense_circuit(n, locs, _mats(locs, kinds, cm, g))
    assert np.abs(ct - U @ V.conj().T).max() < 1e-12
    assert abs(orc.trace(ct) - np.trace(V.conj().T @ U)) < 1e-12
    for _ in range(3):
        ct, g2, log = orc.sweep(C, ct, g, log=True)
        # CONSTANT gates never change (reading R14)
        U2 = dense_circuit(n, locs, _mats(locs, kinds, cm, g2))
        assert np.abs(ct - U2 @ V.conj().T).max() < 1e-11
        g = g2


def _brute_sweep(n, locs, kinds, mats, V, order):
    """One sweep by brute force: at every step k of `order` the environment of
    gate k is built densely by linearity from the CURRENT gates,
    and a VARIABLE gate is replaced by the textbook Procrustes maximiser of
    Re Tr(E u) from numpy's LAPACK SVD.  Returns the gates and
    Tr(V^dag U) after every step."""
    mats = [np.array(m) for m in mats]
    log = []
    for k in order:
        if kinds[k] == qfgen.VARIABLE:
            Ue, _, Vh = np.linalg.svd(_brute_env(n, locs, mats, V, k))
            mats[k] = Vh.conj().T @ Ue.conj().T
        log.append(np.trace(V.conj().T @ dense_circuit(n, locs, mats)))
    return mats, np.array(log)


@pytest.mark.parametrize("seed", range(3))
def test_sweep_order_brute_force(orc, seed):
    """TwoSidedSweep visits k = p..1 first ("reversed"), then
    k = 1..p, each update using the gates as already updated in this
    sweep.  The oracle's per-step traces and final gates must
    equal a dense brute-force sweep in that order; the swapped halves, the
    forward half alone first, or updates from stale gates all give other
    values (checked below, so the pin is sensitive to those mistakes); an
    update from stale gates would not match the brute force, which always
    builds the environment from the current ones."""
    n = 3
    locs = [(0, 1), (1, 2), (2, 0), (1,)]
    kinds = [qfgen.VARIABLE, qfgen.VARIABLE, qfgen.CONSTANT, qfgen.VARIABLE]
    cm = [None, None, qfgen.CNOT, None]
    rng = np.random.default_rng(500 + seed)
    V = haar_np(rng, 2 ** n)
    g = qfgen.initial_gates(n, locs, kinds, 70 + seed, 0, 1)[0]
    mats = _mats(locs, kinds, cm, g)
    p = len(locs)
    order = list(range(p - 1, -1, -1)) + list(range(p))
    ref_mats, ref_log = _brute_sweep(n, locs, kinds, mats, V, order)
    C = _circ(orc, n, locs, kinds, cm)
    _, g2, log = orc.sweep(C, orc.init_ct(C, V, g), g, log=True)
    assert np.abs(log - ref_log).max() < 1e-11
    got = _mats(locs, kinds, cm, g2)
    for k in range(p):
        assert np.abs(got[k] - ref_mats[k]).max() < 1e-10
    # sensitivity: plausible wrong schedules disagree with the oracle
    for bad in (list(range(p)) + list(range(p - 1, -1, -1)),      # halves swapped
                list(range(p)) * 2,                                # forward only
                list(range(p - 1, -1, -1)) * 2):                   # backward only
        _, bad_log = _brute_sweep(n, locs, kinds, mats, V, bad)
        assert np.abs(log - bad_log).max() > 1e-6


@pytest.mark.parametrize("seed", range(5))
def test_sweep_monotone_and_bounded(orc, seed):
    """|Tr| never decreases across single updates, never exceeds
    N, and is real and equal to sum sigma after each VARIABLE
    update (reading R16)."""
    n = 3 + seed % 2
    locs, kinds, cm = qfgen.random_template(n, 10, seed=10 + seed, const_frac=0.2)
    rng = np.random.default_rng(seed)
    V = haar_np(rng, 2 ** n)
    g = qfgen.initial_gates(n, locs, kinds, 60 + seed, 0, 1)[0]
    C = _circ(orc, n, locs, kinds, cm)
    ct = orc.init_ct(C, V, g)
    N = 2 ** n
    prev = abs(orc.trace(ct))
    order = list(range(len(locs) - 1, -1, -1)) + list(range(len(locs)))
    for _ in range(20):
        ct, g, log = orc.sweep(C, ct, g, log=True)
        for t, k in zip(log, order):
            assert abs(t) >= prev - 1e-12 * N
            assert abs(t) <= N * (1 + 1e-12)
            if kinds[k] == qfgen.VARIABLE:
                assert abs(t.imag) < 1e-12 * N and t.real >= 0
            prev = abs(t)


def test_self_target_fixed_point(orc):
    """V = C(alpha0), start at alpha0: ct = I, Delta ~ 0, gates are a fixed
    point (north_star)."""
    w = qfgen.workload("C3")
    V = w.target_unitary()
    g0 = qfgen.initial_gates(w.n, w.locs, w.kinds, w.target_seed, 0, 1,
                             purpose=qfgen.PURPOSE_SELF)[0]
    C = _circ(orc, w.n, w.locs, w.kinds, w.const_mats)
    ct = orc.init_ct(C, V, g0)
    assert np.abs(ct - np.eye(16)).max() < 1e-13
    ct2, g1, _ = orc.sweep(C, ct, g0)
    assert np.abs(g1 - g0).max() < 1e-12
    assert 1 - abs(orc.trace(ct2)) / 16 < 1e-14


def test_whole_register_gate(orc):
    """One VARIABLE gate on all qubits: u <- argmax Re Tr(V^dag u) = V."""
    rng = np.random.default_rng(8)
    for n in (2, 3):
        V = haar_np(rng, 2 ** n)
        loc = tuple(rng.permutation(n))
        C = _circ(orc, n, [loc], [qfgen.VARIABLE], [None])
        g = pack([haar_np(rng, 2 ** n)])
        ct = orc.init_ct(C, V, g)
        ct, g, _ = orc.sweep(C, ct, g)
        u = g.view(complex).reshape(2 ** n, 2 ** n)
        assert np.abs(dense_embed(n, loc, u) - V).max() < 1e-12
        assert 1 - abs(orc.trace(ct)) / 2 ** n < 1e-14


def test_product_target(orc):
    """V = V_A (x) V_B and two VARIABLE gates on A and B: |Tr| = N after the
    two updates of the backward half."""
    rng = np.random.default_rng(12)
    VA, VB = haar_np(rng, 4), haar_np(rng, 2)
    V = np.kron(VA, VB)
    C = _circ(orc, 3, [(0, 1), (2,)], [qfgen.VARIABLE] * 2, [None, None])
    g = pack([haar_np(rng, 4), haar_np(rng, 2)])
    ct = orc.init_ct(C, V, g)
    _, _, log = orc.sweep(C, ct, g, log=True)
    assert abs(abs(log[1]) - 8) < 1e-12


def test_c1_kak_universal(orc):
    """C1's 3-CNOT template is universal for SU(4) (KAK): converged
    starts reach Delta <= dist_tol = 1e-10, and at least one converges."""
    w = qfgen.workload("C1")
    C = _circ(orc, w.n, w.locs, w.kinds, w.const_mats)
    res = orc.instantiate(C, w.target_unitary(), w.initial(),
                          orc.default_params(max_iters=w.max_iters))
    assert (res.verdict == orc.CONVERGED).sum() >= 1
    assert np.all(res.delta[res.verdict == orc.CONVERGED] <= 1e-10)


def test_global_phase_invariance(orc):
    """V -> e^{i phi} V leaves the Delta trajectory unchanged."""
    w = qfgen.workload("C2+")
    C = _circ(orc, w.n, w.locs, w.kinds, w.const_mats)
    V = w.target_unitary()
    P = orc.default_params(max_iters=30, diff_tol_r=0.0, long_diff_count=0)
    a = orc.instantiate(C, V, w.initial(0, 3), P, record_sweeps=30)
    for phi in (np.pi / 3, np.pi):
        b = orc.instantiate(C, np.exp(1j * phi) * V, w.initial(0, 3), P, record_sweeps=30)
        assert np.array_equal(a.iters, b.iters) and np.array_equal(a.verdict, b.verdict)
        assert np.array_equal(np.isnan(a.cost_hist), np.isnan(b.cost_hist))
        assert np.nanmax(np.abs(a.cost_hist - b.cost_hist)) < 1e-13


def test_beta_one_sweep_noop(orc):
    w = qfgen.workload("C2+")
    C = _circ(orc, w.n, w.locs, w.kinds, w.const_mats)
    g = w.initial(0, 1)[0]
    ct = orc.init_ct(C, w.target_unitary(), g)
    _, g2, _ = orc.sweep(C, ct, g, beta=1.0)
    assert np.abs(g2 - g).max() < 1e-12


def test_reset_stability(orc):
    """reset_iter in {1, 40} gives the same final Delta within 1e-8."""
    w = qfgen.workload("C2+")
    C = _circ(orc, w.n, w.locs, w.kinds, w.const_mats)
    V = w.target_unitary()
    a = orc.instantiate(C, V, w.initial(0, 4), orc.default_params(max_iters=300, reset_iters=40))
    b = orc.instantiate(C, V, w.initial(0, 4), orc.default_params(max_iters=300, reset_iters=1))
    assert np.abs(a.delta - b.delta).max() < 1e-8
    assert np.array_equal(a.verdict, b.verdict)


def test_max_iter_zero_S384(orc):
    w = qfgen.workload("C2+")
    C = _circ(orc, w.n, w.locs, w.kinds, w.const_mats)
    V = w.target_unitary()
    g = w.initial(0, 2)
    res = orc.instantiate(C, V, g, orc.default_params(max_iters=0))
    assert np.all(res.verdict == orc.MAX_ITER) and np.all(res.iters == 0)
    for s in range(2):
        U = dense_circuit(w.n, w.locs, _mats(w.locs, w.kinds, w.const_mats, g[s]))
        ref = 1 - abs(np.trace(V.conj().T @ U)) / 2 ** w.n
        assert abs(res.delta[s] - ref) < 1e-13
        assert np.array_equal(res.gates[s], g[s])


# ------------------------------------------------------------------ termination
def test_terminate_sequences(orc):
    P = orc.default_params()  # 1e-10, 0, 1e-5, 100, 0.1, min 0, max 1e5
    T = orc.terminate
    assert T(P, [0.5]) == orc.RUNNING
    assert T(P, [0.5, 1e-11]) == orc.CONVERGED
    assert T(P, [1e-10]) == orc.CONVERGED  # <= dist_tol, even at sweep 1
    # short plateau: |c_i - c_{i-1}| <= 1e-5 c_i, never at it = 1
    assert T(P, [0.3, 0.3]) == orc.PLATEAU_SHORT
    assert T(P, [0.3, 0.3 * (1 - 0.9e-5)]) == orc.PLATEAU_SHORT
    assert T(P, [0.3, 0.3 * (1 - 2e-5)]) == orc.RUNNING
    # converged beats plateau (reading R17)
    assert T(P, [1e-11, 1e-11]) == orc.CONVERGED
    # long plateau: c_{i-L} - c_i <= 0.1 c_{i-L}, only for i > L
    seq = list(0.5 * (1 - 0.0009) ** np.arange(101))  # 8.6% decrease over 100 sweeps
    assert T(P, seq[:100]) == orc.RUNNING
    assert T(P, seq) == orc.PLATEAU_LONG
    seq2 = list(0.5 * (1 - 0.0012) ** np.arange(101))  # 11.3% decrease
    assert T(P, seq2) == orc.RUNNING
    P0 = orc.default_params(long_diff_count=0)
    assert T(P0, seq) == orc.RUNNING
    # max_iter
    Pm = orc.default_params(max_iters=3)
    assert T(Pm, [0.5, 0.4, 0.3]) == orc.MAX_ITER
    assert T(Pm, [0.5, 0.4, 1e-12]) == orc.CONVERGED
    # min_iter gates everything but MAX_ITER
    Pn = orc.default_params(min_iters=5, max_iters=4)
    assert T(Pn, [1e-12, 1e-12]) == orc.RUNNING
    assert T(Pn, [0.1] * 4) == orc.MAX_ITER
    # non-finite
    assert T(P, [0.5, float("nan")]) == orc.NUMERIC_FAIL


def test_default_params_golden(orc):
    g = json.load(open(os.path.join(GOLD, "hyperparams_P532.json")))
    P = orc.default_params()
    for k in ("dist_tol", "diff_tol_a", "diff_tol_r", "long_diff_count", "long_diff_r",
              "min_iters", "max_iters", "reset_iters", "beta"):
        assert getattr(P, k) == g[k], k


def test_oracle_regression_C1_golden(orc):
    """Regression fixture written by tests/golden/make_golden.py (oracle only)."""
    g = json.load(open(os.path.join(GOLD, "oracle_C1_trajectories.json")))
    w = qfgen.workload("C1")
    r = orc.instantiate(orc.Circuit(w.n, w.locs, w.kinds, w.const_mats), w.target_unitary(),
                        w.initial(), orc.default_params(max_iters=w.max_iters), record_sweeps=30,
                        nthreads=1)
    assert r.verdict.tolist() == g["verdict"] and r.iters.tolist() == g["iters"]
    assert np.abs(r.delta - np.array(g["delta"])).max() < 1e-13
    ref = np.array([[np.nan if x is None else x for x in row] for row in g["cost_first30"]])
    assert np.array_equal(np.isnan(ref), np.isnan(r.cost_hist))
    assert np.nanmax(np.abs(ref - r.cost_hist)) < 1e-13
