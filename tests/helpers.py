"""Dense, independent constructions used by the pin tests (numpy only).

Nothing here is imported by the product path; nothing here calls the oracle.
"""
import numpy as np


def dense_embed(n, loc, u):
    """E(u) as a dense 2^n x 2^n matrix, built by Kronecker product with the
    identity on the other qubits and a basis permutation that moves the
    location's qubits to the front (qubit 0 = MSB, loc[0] = MSB; SPEC
    S:153-161)."""
    m = len(loc)
    rest = [q for q in range(n) if q not in loc]
    order = list(loc) + rest
    big = np.kron(np.asarray(u, dtype=np.complex128), np.eye(2 ** (n - m)))
    idx = np.arange(2 ** n)
    shifts = n - 1 - np.arange(n)
    bits = (idx[:, None] >> shifts[None, :]) & 1
    new = (bits[:, order] << shifts[None, :]).sum(1)
    P = np.zeros((2 ** n, 2 ** n))
    P[new, idx] = 1.0
    return P.T @ big @ P


def dense_circuit(n, locs, mats):
    """U = E(u_p) ... E(u_1) by dense products."""
    U = np.eye(2 ** n, dtype=np.complex128)
    for l, u in zip(locs, mats):
        U = dense_embed(n, l, u) @ U
    return U


def haar_np(rng, d):
    z = (rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))) / np.sqrt(2)
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))


def ginibre(rng, d):
    return rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))


def u3(theta, phi, lam):
    """U3 as in SPEC S:136 (standard half-angle form)."""
    c, s = np.cos(theta / 2), np.sin(theta / 2)
    return np.array([[c, -np.exp(1j * lam) * s],
                     [np.exp(1j * phi) * s, np.exp(1j * (phi + lam)) * c]])


def pack(mats):
    return np.concatenate([np.ascontiguousarray(m, dtype=np.complex128).ravel().view(np.float64)
                           for m in mats if m is not None])
