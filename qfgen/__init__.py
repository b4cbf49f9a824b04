"""Seeded synthetic inputs for QFactor instantiation (shared by both sides).

This module is the ONLY code the oracle side (``oracle/``, ``tests/``) and
the product side (``bench.py``, the CUDA path's callers) share.  It holds
none of QFactor's arithmetic (no gate application to a circuit tensor, no
environment, no polar update, no cost): it draws random numbers, builds Haar
unitaries, names templates, and builds the target V.

Recipe:
  * counter-based SplitMix64 streams keyed by (seed, purpose, start, gate),
    so a start's initial gates do not depend on how starts are sharded;
  * Haar unitaries on U(d) by QR of a complex Ginibre matrix with the
    diagonal-phase fix (Mezzadri 2007);
  * targets: Haar on U(2^n) or "self" targets V = C(alpha*) with alpha*
    Haar gates (the paper re-instantiates partitions to their own unitary,
    P:686-689);
  * templates C1..C5 (+ success-path variants) of SURVEY.md Sec. 8d, shaped
    like the paper's workloads (3-8 qubit blocks, QSearch/ladder templates,
    multistart; BASELINE.json configs).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

VARIABLE, CONSTANT = 0, 1
RZ = 2  # NEXT-4: parameterised R_z(theta) = diag(1, e^{i theta}), a VARIABLE-like gate

PURPOSE_INIT = 1  # initial unitaries of the multistarts
PURPOSE_TARGET = 2  # Haar targets
PURPOSE_SELF = 3  # alpha* of self-targets

# CNOT with location (control, target), location[0] = MSB
CNOT = np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]], dtype=np.complex128)

_G1 = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_G2 = np.uint64(0xD1B54A32D192ED03)


def splitmix64(x):
    """SplitMix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + _G1
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def stream_key(seed, purpose, start, gate):
    """Key of the counter stream for (seed, purpose, start, gate)."""
    k = splitmix64(np.uint64(seed))
    k = splitmix64(k ^ np.asarray(purpose, dtype=np.uint64))
    k = splitmix64(k ^ np.asarray(start, dtype=np.uint64))
    return splitmix64(k ^ np.asarray(gate, dtype=np.uint64))


def uniforms(keys, count):
    """(len(keys), count) uniforms in (0, 1) from counter streams."""
    keys = np.asarray(keys, dtype=np.uint64).reshape(-1, 1)
    ctr = np.arange(count, dtype=np.uint64).reshape(1, -1)
    with np.errstate(over="ignore"):
        x = splitmix64(keys + ctr * _G2)
    return ((x >> np.uint64(11)).astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)


def haar(keys, d):
    """Haar-random U(d) matrices, one per key: QR of Ginibre + phase fix."""
    keys = np.asarray(keys, dtype=np.uint64).ravel()
    u = uniforms(keys, 2 * d * d)
    u1, u2 = u[:, 0::2], u[:, 1::2]
    r = np.sqrt(-2.0 * np.log(u1))
    z = (r * np.cos(2 * np.pi * u2) + 1j * r * np.sin(2 * np.pi * u2)) / np.sqrt(2.0)
    z = z.reshape(-1, d, d)
    # Q of the QR factorisation with a positive real diagonal of R ("phase
    # fix", Mezzadri 2007), by twice-iterated modified Gram-Schmidt vectorised
    # over the batch (the same unique Q as LAPACK QR + phase fix, much faster
    # for millions of small matrices); columns laid out batch-contiguous and
    # processed in cache-sized chunks
    q = np.empty_like(z)
    for c0 in range(0, z.shape[0], 16384):
        zt = np.ascontiguousarray(z[c0:c0 + 16384].transpose(2, 1, 0))  # [col][row][batch]
        qt = np.empty_like(zt)
        for j in range(d):
            v = zt[j].copy()
            for _ in range(2):
                for i in range(j):
                    v -= np.sum(np.conj(qt[i]) * v, axis=0) * qt[i]
            qt[j] = v / np.sqrt(np.sum(v.real ** 2 + v.imag ** 2, axis=0))
        q[c0:c0 + 16384] = qt.transpose(2, 1, 0)
    return q


@dataclass
class Workload:
    name: str
    n: int
    locs: list
    kinds: list
    const_mats: list
    starts: int
    max_iters: int
    target: str  # "haar" | "self"
    cid: int
    desc: str = ""
    params: dict = field(default_factory=dict)

    @property
    def p(self):
        return len(self.locs)

    @property
    def var_doubles(self):
        return sum(2 * 4 ** len(l) for l, k in zip(self.locs, self.kinds) if k != CONSTANT)

    @property
    def target_seed(self):
        return 1000 + self.cid

    @property
    def init_seed(self):
        return 2000 + self.cid

    def initial(self, start_begin=0, count=None, seed=None):
        """(count, var_doubles) float64: interleaved Haar initial gates for
        global starts [start_begin, start_begin+count)."""
        count = self.starts if count is None else count
        return initial_gates(self.n, self.locs, self.kinds,
                             self.init_seed if seed is None else seed, start_begin, count)

    def target_unitary(self):
        if self.target == "haar":
            return haar(stream_key(self.target_seed, PURPOSE_TARGET, 0, 0), 1 << self.n)[0]
        g = initial_gates(self.n, self.locs, self.kinds, self.target_seed, 0, 1,
                          purpose=PURPOSE_SELF)[0]
        return circuit_unitary(self.n, self.locs, self.kinds, self.const_mats, g)


def initial_gates(n, locs, kinds, seed, start_begin, count, purpose=PURPOSE_INIT):
    """Pack the starting values of the parameterised gates, gate order,
    row-major, interleaved: Haar for VARIABLE gates; R_z(theta) with theta
    uniform in [0, 2 pi) for RZ gates."""
    var_idx = [k for k, kd in enumerate(kinds) if kd != CONSTANT]
    sizes = [2 * 4 ** len(locs[k]) for k in var_idx]
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    out = np.zeros((count, int(offs[-1])), dtype=np.float64)
    starts = np.arange(start_begin, start_begin + count, dtype=np.uint64)
    for d in sorted({1 << len(locs[k]) for k in var_idx if kinds[k] == VARIABLE}):
        ks = [j for j, k in enumerate(var_idx) if (1 << len(locs[k])) == d and kinds[k] == VARIABLE]
        gate_ids = np.array([var_idx[j] for j in ks], dtype=np.uint64)
        keys = stream_key(seed, purpose, starts[:, None], gate_ids[None, :])
        us = haar(keys.ravel(), d).reshape(count, len(ks), d * d)
        for col, j in enumerate(ks):
            out[:, offs[j]:offs[j + 1]] = np.ascontiguousarray(us[:, col]).view(np.float64)
    for j, k in enumerate(var_idx):
        if kinds[k] != RZ:
            continue
        keys = stream_key(seed, purpose, starts, np.uint64(k))
        th = 2 * np.pi * uniforms(keys, 1)[:, 0]
        m = np.zeros((count, 4), dtype=np.complex128)
        m[:, 0] = 1.0
        m[:, 3] = np.exp(1j * th)
        out[:, offs[j]:offs[j + 1]] = m.view(np.float64)
    return out


def unpack_gates(locs, kinds, packed):
    """Inverse of the packing: list of (d, d) complex (None for CONSTANT)."""
    out, off = [], 0
    for l, k in zip(locs, kinds):
        if k == CONSTANT:
            out.append(None)
            continue
        d = 1 << len(l)
        out.append(np.asarray(packed[off:off + 2 * d * d]).view(np.complex128).reshape(d, d))
        off += 2 * d * d
    return out


def circuit_unitary(n, locs, kinds, const_mats, packed):
    """Dense U = E(u_p) ... E(u_1) (gate p leftmost), by
    contracting each gate into the 2n-leg tensor of the running unitary
    with numpy.tensordot (qubit 0 = leading axis = MSB)."""
    N = 1 << n
    T = np.eye(N, dtype=np.complex128).reshape((2,) * (2 * n))
    gates = unpack_gates(locs, kinds, packed)
    for l, k, u, c in zip(locs, kinds, gates, const_mats):
        g = u if k != CONSTANT else np.asarray(c, dtype=np.complex128)
        m = len(l)
        G = g.reshape((2,) * (2 * m))
        # contract gate input legs with the output legs l of T
        T = np.tensordot(G, T, axes=(list(range(m, 2 * m)), list(l)))
        # tensordot puts the gate's output legs first; move them back to l
        T = np.moveaxis(T, list(range(m)), list(l))
    return T.reshape(N, N)


# ------------------------------------------------------------------ templates
def _c1():
    locs, kinds, cm = [(0,), (1,)], [VARIABLE, VARIABLE], [None, None]
    for _ in range(3):
        locs += [(0, 1), (0,), (1,)]
        kinds += [CONSTANT, VARIABLE, VARIABLE]
        cm += [CNOT, None, None]
    return locs, kinds, cm


def _c2():
    locs, kinds, cm = [(0,), (1,), (2,)], [VARIABLE] * 3, [None] * 3
    for i in range(14):
        a = (0, 1) if i % 2 == 0 else (1, 2)
        locs += [a, (a[0],), (a[1],)]
        kinds += [CONSTANT, VARIABLE, VARIABLE]
        cm += [CNOT, None, None]
    return locs, kinds, cm


def _brick4(p):
    layers = [[(0, 1), (2, 3)], [(1, 2)]]
    locs, li = [], 0
    while len(locs) < p:
        for l in layers[li % 2]:
            if len(locs) < p:
                locs.append(l)
        li += 1
    return locs, [VARIABLE] * p, [None] * p


def _ladder(n, p):
    locs = [(k % (n - 1), k % (n - 1) + 1) for k in range(p)]
    return locs, [VARIABLE] * p, [None] * p


def _c5():
    locs = []
    while len(locs) < 200:
        for i in range(7):
            locs.append((i, i + 1))
        for i in range(6):
            locs.append((i, i + 1, i + 2))
    locs = locs[:200]
    return locs, [VARIABLE] * 200, [None] * 200


def _round(n, p):
    """C5's pattern on n qubits: a cyclic round of n-1 U(4) on (i, i+1), then
    n-2 U(8) on (i, i+1, i+2), truncated to p gates."""
    locs = []
    while len(locs) < p:
        locs += [(i, i + 1) for i in range(n - 1)] + [(i, i + 1, i + 2) for i in range(n - 2)]
    return locs[:p], [VARIABLE] * p, [None] * p


def _u3_cnot(n, layers):
    """The paper's gate set (U3 + CNOT): a VAR U(2) on every qubit,
    then `layers` x [CNOT(i, i+1), VAR U(2) i, VAR U(2) i+1] down a ladder."""
    cx = np.eye(4)[[0, 1, 3, 2]]
    locs, kinds, cm = [(q,) for q in range(n)], [VARIABLE] * n, [None] * n
    for l in range(layers):
        i = l % (n - 1)
        locs += [(i, i + 1), (i,), (i + 1,)]
        kinds += [CONSTANT, VARIABLE, VARIABLE]
        cm += [cx, None, None]
    return locs, kinds, cm


def workload(name: str) -> Workload:
    """The configs of BASELINE.json / SURVEY.md Sec. 8d (C1-C5, C2+, C3+) and
    the NEXT-3 size probes C6 (n = 10), C7 (n = 12) and C8 (n = 10, the
    paper's U3 + CNOT gate set)."""
    if name == "C1":
        l, k, c = _c1()
        return Workload("C1", 2, l, k, c, 4, 10000, "haar", 1,
                        "2-qubit 3-CNOT + U(2) KAK template vs Haar SU(4), 4 starts")
    if name == "C2":
        l, k, c = _c2()
        return Workload("C2", 3, l, k, c, 64, 10000, "haar", 2,
                        "3-qubit QSearch-style 14-CNOT ladder vs Haar, 64 starts")
    if name == "C3":
        l, k, c = _brick4(20)
        return Workload("C3", 4, l, k, c, 1024, 5000, "self", 3,
                        "4-qubit brick of 20 VAR U(4), self-target, 1024 starts")
    if name == "C4":
        l, k, c = _ladder(6, 80)
        return Workload("C4", 6, l, k, c, 4096, 2000, "self", 4,
                        "6-qubit ladder of 80 VAR U(4), self-target, 4096 starts")
    if name == "C5":
        l, k, c = _c5()
        return Workload("C5", 8, l, k, c, 8192, 1000, "self", 5,
                        "8-qubit 110 VAR U(4) + 90 VAR U(8), self-target, 8192 starts")
    if name == "C2+":
        l, k, c = _ladder(3, 12)
        return Workload("C2+", 3, l, k, c, 64, 2000, "haar", 6,
                        "3-qubit ladder of 12 VAR U(4) vs Haar, 64 starts")
    if name == "C3+":
        l, k, c = _ladder(4, 40)
        return Workload("C3+", 4, l, k, c, 1024, 2000, "haar", 7,
                        "4-qubit ladder of 40 VAR U(4) vs Haar, 1024 starts")
    if name == "C6":
        l, k, c = _round(10, 60)
        return Workload("C6", 10, l, k, c, 256, 1000, "self", 8,
                        "10-qubit round of VAR U(4) + U(8) (C5 pattern), 60 gates, self-target, 256 starts")
    if name == "C7":
        l, k, c = _round(12, 40)
        return Workload("C7", 12, l, k, c, 32, 1000, "self", 9,
                        "12-qubit round of VAR U(4) + U(8) (C5 pattern), 40 gates, self-target, 32 starts")
    if name == "C8":
        l, k, c = _u3_cnot(10, 60)
        return Workload("C8", 10, l, k, c, 256, 1000, "self", 10,
                        "10-qubit U3+CNOT ladder (10 + 60 x [CNOT, U(2), U(2)] = 190 gates), "
                        "self-target, 256 starts")
    raise KeyError(name)


ALL = ["C1", "C2", "C3", "C4", "C5", "C2+", "C3+"]


def many_workload(count=1024, starts=32, max_iters=1000):
    """NEXT-2 workload: `count` independent
    3-qubit blocks, the shape partitioning produces; block q is a ladder of
    4 + (q mod 7) VARIABLE U(4) gates re-instantiated to its own unitary
    (self-target, seeds 1100 + q / 2100 + q), 32 multistarts each."""
    out = []
    for q in range(count):
        l, k, c = _ladder(3, 4 + q % 7)
        out.append(Workload(f"B{q}", 3, l, k, c, starts, max_iters, "self", 100 + q,
                            f"3-qubit block {q}: ladder of {len(l)} VAR U(4), self-target"))
    return out


def random_template(n, p, arities=(1, 2, 3), seed=0, const_frac=0.0):
    """A random template for tests: random arity, random distinct, randomly
    ordered locations; a fraction of CONSTANT gates (Haar matrices)."""
    rng = np.random.default_rng(seed)
    locs, kinds, cm = [], [], []
    for k in range(p):
        m = int(rng.choice([a for a in arities if a <= n]))
        locs.append(tuple(int(q) for q in rng.permutation(n)[:m]))
        if rng.random() < const_frac:
            kinds.append(CONSTANT)
            cm.append(haar(stream_key(seed, 99, 0, k), 1 << m)[0])
        else:
            kinds.append(VARIABLE)
            cm.append(None)
    return locs, kinds, cm
