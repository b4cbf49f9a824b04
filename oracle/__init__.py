"""ctypes wrapper of the plain CPU oracle (oracle/qf_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product path (``paper_2306_08152_b200``) never imports it and
shares no code with it.

The oracle is Alg. 1 of arXiv 2306.08152 written out
literally; see ``qf_oracle.h`` for the conventions and citations and
``tests/test_oracle_pins.py`` for what pins each function.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "qf_oracle.c")
# ORACLE_SANITIZE=1: an AddressSanitizer + UndefinedBehaviorSanitizer build
# (liboracle_asan.so; run under LD_PRELOAD=$(gcc -print-file-name=libasan.so),
# ASAN_OPTIONS=detect_leaks=0) -- tools/oracle_sanitize.sh
_SAN = os.environ.get("ORACLE_SANITIZE") == "1"
_LIB = os.path.join(_HERE, "liboracle_asan.so" if _SAN else "liboracle.so")

VARIABLE, CONSTANT, RZ = 0, 1, 2
RUNNING, CONVERGED, PLATEAU_SHORT, PLATEAU_LONG, MAX_ITER, NUMERIC_FAIL, BATCH_STOPPED = range(7)


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc -O2 -ffp-contract=off."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "qf_oracle.h"))
    ):
        tmp = _LIB + f".tmp{os.getpid()}"
        san = (["-g", "-fno-omit-frame-pointer", "-fsanitize=address,undefined",
                "-fno-sanitize-recover=undefined"] if _SAN else [])
        subprocess.check_call(
            ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
             "-D_GNU_SOURCE", "-fPIC", "-shared", "-pthread", *san, _SRC, "-o", tmp, "-lm"]
        )
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _declare(_lib)
    return _lib


class Params(ctypes.Structure):
    _fields_ = [
        ("dist_tol", ctypes.c_double),
        ("diff_tol_a", ctypes.c_double),
        ("diff_tol_r", ctypes.c_double),
        ("long_diff_count", ctypes.c_int),
        ("long_diff_r", ctypes.c_double),
        ("min_iters", ctypes.c_int),
        ("max_iters", ctypes.c_int),
        ("reset_iters", ctypes.c_int),
        ("beta", ctypes.c_double),
    ]


class _Circuit(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int),
        ("p", ctypes.c_int),
        ("arity", ctypes.POINTER(ctypes.c_int)),
        ("loc", ctypes.POINTER(ctypes.c_int)),
        ("kind", ctypes.POINTER(ctypes.c_int)),
        ("const_mats", ctypes.POINTER(ctypes.c_double)),
    ]


_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int)


def _declare(L):
    L.oracle_apply_left.argtypes = [ctypes.c_int, ctypes.c_int, _I, _D, ctypes.c_int, _D]
    L.oracle_apply_right.argtypes = [ctypes.c_int, ctypes.c_int, _I, _D, ctypes.c_int, _D]
    L.oracle_env.argtypes = [ctypes.c_int, ctypes.c_int, _I, _D, _D]
    L.oracle_trace.argtypes = [ctypes.c_int, _D, _D]
    L.oracle_svd.argtypes = [ctypes.c_int, _D, _D, _D, _D]
    L.oracle_svd.restype = ctypes.c_int
    L.oracle_optimize_gate.argtypes = [ctypes.c_int, _D, _D, ctypes.c_double, _D, _D]
    L.oracle_optimize_rz.argtypes = [_D, _D, ctypes.c_double, _D]
    L.oracle_init_ct.argtypes = [ctypes.POINTER(_Circuit), _D, _D, _D]
    L.oracle_sweep.argtypes = [ctypes.POINTER(_Circuit), _D, _D, ctypes.c_double, _D]
    L.oracle_terminate.argtypes = [ctypes.POINTER(Params), ctypes.c_int, _D]
    L.oracle_terminate.restype = ctypes.c_int
    L.oracle_var_doubles.argtypes = [ctypes.POINTER(_Circuit)]
    L.oracle_var_doubles.restype = ctypes.c_int
    L.oracle_instantiate.argtypes = [
        ctypes.POINTER(_Circuit), _D, ctypes.c_int, _D, ctypes.POINTER(Params),
        ctypes.c_int, ctypes.c_int, ctypes.c_int, _D, _I, _I, _D, _D, _D]
    L.oracle_instantiate.restype = ctypes.c_int
    L.oracle_instantiate_batch.argtypes = [
        ctypes.POINTER(_Circuit), _D, ctypes.c_int, _D, ctypes.POINTER(Params),
        ctypes.c_int, _D, _I, _I, _D]
    L.oracle_instantiate_batch.restype = ctypes.c_int


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_D)


def _ip(a: np.ndarray):
    return a.ctypes.data_as(_I)


def _cplx(a) -> np.ndarray:
    """complex ndarray -> contiguous interleaved float64 view-copy."""
    a = np.ascontiguousarray(a, dtype=np.complex128)
    return a.view(np.float64)


def default_params(**kw) -> Params:
    """Paper defaults, P:532 (max_iter 1e5, reset 40, beta 0, ...)."""
    p = Params(1e-10, 0.0, 1e-5, 100, 0.1, 0, 100000, 40, 0.0)
    for k, v in kw.items():
        setattr(p, k, v)
    return p


@dataclass
class Circuit:
    """A template: gate k acts on qubits locs[k]."""

    n: int
    locs: list  # list of tuples of qubit indices
    kinds: list  # VARIABLE / CONSTANT per gate
    const_mats: list  # per gate: complex (d, d) array or None

    def _c(self):
        arity = np.array([len(l) for l in self.locs], dtype=np.int32)
        loc = np.array([q for l in self.locs for q in l], dtype=np.int32)
        kind = np.array(self.kinds, dtype=np.int32)
        cm = [np.asarray(m, dtype=np.complex128).ravel() for m, k in
              zip(self.const_mats, self.kinds) if k == CONSTANT]
        cmat = _cplx(np.concatenate(cm)) if cm else np.zeros(2, dtype=np.float64)
        keep = (arity, loc, kind, cmat)
        c = _Circuit(self.n, len(self.locs), _ip(arity), _ip(loc), _ip(kind), _dp(cmat))
        return c, keep

    @property
    def var_doubles(self) -> int:
        return sum(2 * 4 ** len(l) for l, k in zip(self.locs, self.kinds) if k != CONSTANT)


# ---------------------------------------------------------------- blocks
def apply_left(ct: np.ndarray, u: np.ndarray, loc, dagger=False) -> np.ndarray:
    n = int(np.log2(ct.shape[0]))
    out = _cplx(ct).copy()
    L = np.array(loc, dtype=np.int32)
    uu = _cplx(u)
    lib().oracle_apply_left(n, len(loc), _ip(L), _dp(uu), int(dagger), _dp(out))
    return out.view(np.complex128).reshape(ct.shape)


def apply_right(ct: np.ndarray, u: np.ndarray, loc, dagger=False) -> np.ndarray:
    n = int(np.log2(ct.shape[0]))
    out = _cplx(ct).copy()
    L = np.array(loc, dtype=np.int32)
    uu = _cplx(u)
    lib().oracle_apply_right(n, len(loc), _ip(L), _dp(uu), int(dagger), _dp(out))
    return out.view(np.complex128).reshape(ct.shape)


def env(ct: np.ndarray, loc) -> np.ndarray:
    n = int(np.log2(ct.shape[0]))
    d = 1 << len(loc)
    out = np.zeros((d, d), dtype=np.complex128)
    L = np.array(loc, dtype=np.int32)
    c = _cplx(ct)
    lib().oracle_env(n, len(loc), _ip(L), _dp(c), _dp(out.view(np.float64)))
    return out


def trace(ct: np.ndarray) -> complex:
    n = int(np.log2(ct.shape[0]))
    out = np.zeros(2)
    lib().oracle_trace(n, _dp(_cplx(ct)), _dp(out))
    return complex(out[0], out[1])


def svd(M: np.ndarray):
    d = M.shape[0]
    X = np.zeros((d, d), dtype=np.complex128)
    Y = np.zeros((d, d), dtype=np.complex128)
    D = np.zeros(d)
    lib().oracle_svd(d, _dp(_cplx(M)), _dp(X.view(np.float64)), _dp(D), _dp(Y.view(np.float64)))
    return X, D, Y


def optimize_gate(E: np.ndarray, u_old: np.ndarray, beta: float = 0.0):
    d = E.shape[0]
    out = np.zeros((d, d), dtype=np.complex128)
    ss = np.zeros(1)
    lib().oracle_optimize_gate(d, _dp(_cplx(E)), _dp(_cplx(u_old)), float(beta),
                               _dp(out.view(np.float64)), _dp(ss))
    return out, float(ss[0])


def optimize_rz(E: np.ndarray, u_old: np.ndarray, beta: float = 0.0):
    """R_z(theta) update of a 2 x 2 environment (reading R19)."""
    out = np.zeros((2, 2), dtype=np.complex128)
    lib().oracle_optimize_rz(_dp(_cplx(E)), _dp(_cplx(u_old)), float(beta), _dp(out.view(np.float64)))
    return out


def init_ct(circ: Circuit, target: np.ndarray, gates: np.ndarray) -> np.ndarray:
    c, keep = circ._c()
    N = 1 << circ.n
    ct = np.zeros((N, N), dtype=np.complex128)
    g = np.ascontiguousarray(gates, dtype=np.float64)
    lib().oracle_init_ct(ctypes.byref(c), _dp(_cplx(target)), _dp(g), _dp(ct.view(np.float64)))
    return ct


def sweep(circ: Circuit, ct: np.ndarray, gates: np.ndarray, beta: float = 0.0,
          log: bool = False):
    """One TwoSidedSweep; returns (ct, gates, trace_log or None)."""
    c, keep = circ._c()
    ct = np.ascontiguousarray(ct, dtype=np.complex128).copy()
    g = np.ascontiguousarray(gates, dtype=np.float64).copy()
    tl = np.zeros(2 * 2 * len(circ.locs)) if log else None
    lib().oracle_sweep(ctypes.byref(c), _dp(ct.view(np.float64)), _dp(g), float(beta),
                       _dp(tl) if log else None)
    return ct, g, (tl.view(np.complex128) if log else None)


def terminate(params: Params, costs) -> int:
    """costs = [c_1, ..., c_it]; returns the verdict after sweep it."""
    c = np.concatenate([[np.nan], np.asarray(costs, dtype=np.float64)])
    return int(lib().oracle_terminate(ctypes.byref(params), len(costs), _dp(c)))


@dataclass
class Result:
    delta: np.ndarray
    iters: np.ndarray
    verdict: np.ndarray
    gates: np.ndarray  # (S, var_doubles)
    cost_hist: np.ndarray  # (S, R)
    gates_hist: np.ndarray | None  # (S, R, var_doubles)
    threads: int


def instantiate(circ: Circuit, target: np.ndarray, initial: np.ndarray,
                params: Params | None = None, record_sweeps: int = 0,
                record_gates: bool | int = False, nthreads: int = 0) -> Result:
    """Multi-start Qfactor over the S rows of `initial`.
    record_sweeps: costs kept for sweeps 1..R; record_gates: True (gates for
    the same R sweeps) or an int R_g (gates for sweeps 1..R_g)."""
    params = params or default_params()
    c, keep = circ._c()
    initial = np.ascontiguousarray(initial, dtype=np.float64)
    S = initial.shape[0]
    var = circ.var_doubles
    assert initial.shape == (S, var), (initial.shape, var)
    delta = np.zeros(S)
    iters = np.zeros(S, dtype=np.int32)
    verdict = np.zeros(S, dtype=np.int32)
    gates = np.zeros((S, var))
    R = int(record_sweeps)
    Rg = (R if record_gates is True else int(record_gates)) if record_gates else 0
    ch = np.zeros((S, max(R, 1)))
    gh = np.zeros((S, max(Rg, 1), var)) if Rg else None
    th = lib().oracle_instantiate(
        ctypes.byref(c), _dp(_cplx(target)), S, _dp(initial), ctypes.byref(params),
        R, Rg, int(nthreads), _dp(delta), _ip(iters), _ip(verdict), _dp(gates), _dp(ch),
        _dp(gh) if gh is not None else None)
    return Result(delta, iters, verdict, gates, ch[:, :R],
                  gh[:, :Rg] if gh is not None else None, th)


def instantiate_batch(circ: Circuit, target: np.ndarray, initial: np.ndarray,
                      params: Params | None = None, nthreads: int = 0) -> Result:
    """The paper's GPU multistart termination (reading R22): all
    starts advance sweep by sweep; stop on the first convergence, or once
    every running start has hit a plateau, or at max_iters."""
    params = params or default_params()
    c, keep = circ._c()
    initial = np.ascontiguousarray(initial, dtype=np.float64)
    S = initial.shape[0]
    var = circ.var_doubles
    assert initial.shape == (S, var), (initial.shape, var)
    delta = np.zeros(S)
    iters = np.zeros(S, dtype=np.int32)
    verdict = np.zeros(S, dtype=np.int32)
    gates = np.zeros((S, var))
    th = lib().oracle_instantiate_batch(
        ctypes.byref(c), _dp(_cplx(target)), S, _dp(initial), ctypes.byref(params),
        int(nthreads), _dp(delta), _ip(iters), _ip(verdict), _dp(gates))
    return Result(delta, iters, verdict, gates, np.zeros((S, 0)), None, th)
