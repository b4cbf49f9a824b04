"""Python binding of libqfactor.so (include/qf.h): argument marshalling only.

Every step of the QFactor sweep (arXiv 2306.08152, Alg. 1) runs in the
sm_100a kernels of ``csrc/``; this module converts numpy arrays / torch
tensors to pointers and back.  PyTorch is used for device memory, streams and
process groups only.  There is no CPU fallback: if the CUDA library is
missing or no device is present, calls raise ``QfError``.

Names follow the C ABI (``qf_circuit_create``, ``qf_instantiate``, ...);
``Circuit`` / ``instantiate`` / ``instantiate_device`` are thin conveniences.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _build

QF_OK, QF_E_ARG, QF_E_DIM, QF_E_LOCATION, QF_E_NOT_UNITARY, QF_E_OOM, QF_E_CUDA, QF_E_NCCL = range(8)
QF_GATE_VARIABLE, QF_GATE_CONSTANT, QF_GATE_RZ = 0, 1, 2
(QF_RUNNING, QF_CONVERGED, QF_PLATEAU_SHORT, QF_PLATEAU_LONG, QF_MAX_ITER, QF_NUMERIC_FAIL,
 QF_BATCH_STOPPED) = range(7)
QF_ENGINE_AUTO, QF_ENGINE_STREAM, QF_ENGINE_RESIDENT = range(3)
QF_BATCH_PER_START, QF_BATCH_PAPER = range(2)

ENGINE_NAMES = {0: "auto", 1: "stream", 2: "resident"}
VERDICT_NAMES = {0: "RUNNING", 1: "CONVERGED", 2: "PLATEAU_SHORT", 3: "PLATEAU_LONG",
                 4: "MAX_ITER", 5: "NUMERIC_FAIL", 6: "BATCH_STOPPED"}

EXPORTS = [
    "qf_params_default", "qf_circuit_create", "qf_circuit_destroy", "qf_circuit_var_doubles",
    "qf_circuit_num_qubits", "qf_instantiate", "qf_workspace_size", "qf_instantiate_device",
    "qf_result_get", "qf_result_best", "qf_result_num_starts", "qf_result_trace",
    "qf_result_stats", "qf_result_destroy", "qf_select_best_device", "qf_select_best_host",
    "qf_last_error", "qf_version", "qf_instantiate_many", "qf_unitary_to_u3",
    "qf_result_summaries", "qf_result_gates",
]


class QfError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"qf status {status}: {msg}")
        self.status = status


# qf_batch_reduce_fn: sums int64 counts[0..n) in place over the batch's processes
BATCH_REDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64),
                                   ctypes.c_int32)


class qf_params(ctypes.Structure):
    _fields_ = [
        ("dist_tol", ctypes.c_double),
        ("diff_tol_a", ctypes.c_double),
        ("diff_tol_r", ctypes.c_double),
        ("long_diff_count", ctypes.c_int32),
        ("long_diff_r", ctypes.c_double),
        ("min_iters", ctypes.c_int32),
        ("max_iters", ctypes.c_int32),
        ("reset_iters", ctypes.c_int32),
        ("beta", ctypes.c_double),
        ("num_starts", ctypes.c_int32),
        ("engine", ctypes.c_int32),
        ("record_sweeps", ctypes.c_int32),
        ("record_count", ctypes.c_int32),
        ("record_starts", ctypes.POINTER(ctypes.c_int32)),
        ("profile", ctypes.c_int32),
        ("batch_policy", ctypes.c_int32),
        ("batch_reduce", BATCH_REDUCE_FN),
        ("batch_user", ctypes.c_void_p),
        ("seed", ctypes.c_uint64),
        ("start_offset", ctypes.c_int64),
    ]


class qf_summary(ctypes.Structure):
    _fields_ = [("delta", ctypes.c_double), ("iters", ctypes.c_int32), ("verdict", ctypes.c_int32)]


SUMMARY_DTYPE = np.dtype([("delta", "<f8"), ("iters", "<i4"), ("verdict", "<i4")])
assert SUMMARY_DTYPE.itemsize == ctypes.sizeof(qf_summary) == 16


class qf_stats(ctypes.Structure):
    _fields_ = [
        ("kernel_launches", ctypes.c_int64),
        ("sweeps", ctypes.c_int32),
        ("engine", ctypes.c_int32),
        ("start_sweeps", ctypes.c_int64),
        ("h2d_bytes", ctypes.c_int64),
        ("d2h_bytes", ctypes.c_int64),
        ("alg_bytes_total", ctypes.c_double),
        ("sandwich_bytes", ctypes.c_double),
        ("env_bytes", ctypes.c_double),
        ("sandwich_launches", ctypes.c_int64),
        ("env_launches", ctypes.c_int64),
        ("sandwich_ms", ctypes.c_double),
        ("env_ms", ctypes.c_double),
        ("resident_ms", ctypes.c_double),
        ("sweep_flops", ctypes.c_double),
        ("resident_kernel", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int)
_VP = ctypes.c_void_p
_lib = None


def lib():
    """Load (building in-tree first if stale) libqfactor.so."""
    global _lib
    if _lib is None and os.environ.get("QF_LIB"):  # an alternative build (checked / A-B)
        L = ctypes.CDLL(os.environ["QF_LIB"])
        _declare(L)
        _lib = L
    if _lib is None:
        if _build.needs_build():
            if not os.path.exists(_build.NVCC):
                raise QfError(QF_E_CUDA, f"{_build.LIB} missing and nvcc not found")
            _build.build()
        L = ctypes.CDLL(_build.LIB)
        _declare(L)
        _lib = L
    return _lib


def _declare(L):
    c = ctypes
    L.qf_params_default.argtypes = [c.POINTER(qf_params)]
    L.qf_params_default.restype = None
    L.qf_circuit_create.argtypes = [c.c_int, c.c_int, _I, _I, _I, c.POINTER(_D), c.POINTER(_VP)]
    L.qf_circuit_destroy.argtypes = [_VP]
    L.qf_circuit_destroy.restype = None
    L.qf_circuit_var_doubles.argtypes = [_VP]
    L.qf_circuit_num_qubits.argtypes = [_VP]
    L.qf_instantiate.argtypes = [_VP, _D, _D, c.POINTER(qf_params), c.POINTER(_VP)]
    L.qf_workspace_size.argtypes = [_VP, c.POINTER(qf_params)]
    L.qf_workspace_size.restype = c.c_size_t
    L.qf_instantiate_device.argtypes = [_VP, _VP, _VP, c.POINTER(qf_params), _VP, c.c_size_t,
                                        _VP, _VP, _VP, c.POINTER(_VP)]
    L.qf_result_get.argtypes = [_VP, c.c_int, _D, _I, _I, _D]
    L.qf_result_best.argtypes = [_VP]
    L.qf_result_num_starts.argtypes = [_VP]
    L.qf_result_trace.argtypes = [_VP, c.c_int, _D, _D, _I]
    L.qf_result_stats.argtypes = [_VP, c.POINTER(qf_stats)]
    L.qf_result_destroy.argtypes = [_VP]
    L.qf_result_destroy.restype = None
    L.qf_select_best_device.argtypes = [_VP, c.c_int64, _VP, _VP]
    L.qf_select_best_host.argtypes = [c.POINTER(qf_summary), c.c_int64, c.POINTER(c.c_int64)]
    L.qf_instantiate_many.argtypes = [c.c_int32, c.POINTER(_VP), c.POINTER(_D), c.POINTER(_D),
                                      _I, c.POINTER(qf_params), c.POINTER(_VP)]
    L.qf_unitary_to_u3.argtypes = [_D, _D]
    L.qf_result_summaries.argtypes = [_VP, _VP, c.c_int64]
    L.qf_result_gates.argtypes = [_VP, _D, c.c_int64]
    L.qf_last_error.restype = c.c_char_p
    L.qf_last_error.argtypes = []
    L.qf_version.restype = c.c_char_p
    L.qf_version.argtypes = []


def _check(status):
    if status != QF_OK:
        raise QfError(status, lib().qf_last_error().decode())


def qf_last_error() -> str:
    return lib().qf_last_error().decode()


def qf_version() -> str:
    return lib().qf_version().decode()


def qf_params_default(**overrides) -> qf_params:
    p = qf_params()
    lib().qf_params_default(ctypes.byref(p))
    for k, v in overrides.items():
        setattr(p, k, v)
    return p


def _cplx(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128).view(np.float64)


class Circuit:
    """Owning wrapper of a qf_circuit_t (qf_circuit_create)."""

    def __init__(self, n, locs, kinds, const_mats=None):
        p = len(locs)
        const_mats = const_mats or [None] * p
        arity = np.array([len(l) for l in locs], dtype=np.int32)
        loc = np.array([q for l in locs for q in l], dtype=np.int32)
        kind = np.array(kinds, dtype=np.int32)
        keep = [None if m is None else _cplx(m) for m in const_mats]
        ptrs = (_D * max(p, 1))(*[(m.ctypes.data_as(_D) if m is not None else _D()) for m in keep])
        h = _VP()
        _check(lib().qf_circuit_create(int(n), p, arity.ctypes.data_as(_I), loc.ctypes.data_as(_I),
                                       kind.ctypes.data_as(_I), ptrs, ctypes.byref(h)))
        self.h = h
        self.n = int(n)
        self.var_doubles = lib().qf_circuit_var_doubles(h)

    @classmethod
    def from_workload(cls, w):
        return cls(w.n, w.locs, w.kinds, w.const_mats)

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and _lib is not None:
            _lib.qf_circuit_destroy(h)
            self.h = None


def qf_circuit_create(n, locs, kinds, const_mats=None) -> Circuit:
    return Circuit(n, locs, kinds, const_mats)


@dataclass
class Result:
    summary: np.ndarray  # structured (delta, iters, verdict)
    best: int
    gates: np.ndarray | None  # (S, var) for host calls; (1, var) best only for device calls
    cost_hist: np.ndarray | None  # (record_count, R)
    gates_hist: np.ndarray | None  # (record_count, R, var)
    stats: dict

    @property
    def delta(self):
        return self.summary["delta"]

    @property
    def iters(self):
        return self.summary["iters"]

    @property
    def verdict(self):
        return self.summary["verdict"]


def _make_params(S, record_starts=None, record_sweeps=0, **kw):
    p = qf_params_default(num_starts=int(S), **kw)
    keep = None
    if record_starts is not None and len(record_starts) and record_sweeps > 0:
        keep = np.ascontiguousarray(record_starts, dtype=np.int32)
        p.record_sweeps = int(record_sweeps)
        p.record_count = len(keep)
        p.record_starts = keep.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    return p, keep


def _collect(h, var, all_gates) -> Result:
    L = lib()
    S = L.qf_result_num_starts(h)
    summ = np.zeros(S, dtype=SUMMARY_DTYPE)
    if S:
        _check(L.qf_result_summaries(h, _VP(summ.ctypes.data), S))
    best = L.qf_result_best(h)
    if all_gates:
        gates = np.zeros((S, var))
        if S and var:
            _check(L.qf_result_gates(h, gates.ctypes.data_as(_D), S * var))
    else:
        gates = np.zeros((1, var))
        if var and best >= 0:
            _check(L.qf_result_get(h, -1, None, None, None, gates[0].ctypes.data_as(_D)))
    st = qf_stats()
    _check(L.qf_result_stats(h, ctypes.byref(st)))
    stats = {f: getattr(st, f) for f, _ in qf_stats._fields_}
    return Result(summ, best, gates, None, None, stats)


def _collect_trace(h, res: Result, count, R, var):
    ch = np.full((count, R), np.nan)
    gh = np.zeros((count, R, var))
    n = ctypes.c_int()
    for i in range(count):
        _check(lib().qf_result_trace(h, i, ch[i].ctypes.data_as(_D),
                                     gh[i].ctypes.data_as(_D) if var else None, ctypes.byref(n)))
    res.cost_hist, res.gates_hist = ch, gh


def qf_instantiate(circ: Circuit, target, initial=None, record_starts=None, record_sweeps=0,
                   num_starts=None, **params) -> Result:
    """Blocking instantiation from host buffers (the end-to-end call).
    initial=None: `num_starts` seeded starts generated on the device from
    params seed / start_offset (qf.h qf_params)."""
    if initial is None:
        S = int(num_starts)
        iptr = None
    else:
        initial = np.ascontiguousarray(initial, dtype=np.float64)
        S = initial.shape[0]
        assert initial.shape == (S, circ.var_doubles)
        assert num_starts is None or num_starts == S
        iptr = initial.ctypes.data_as(_D)
    p, keep = _make_params(S, record_starts, record_sweeps, **params)
    t = _cplx(target)
    h = _VP()
    _check(lib().qf_instantiate(circ.h, t.ctypes.data_as(_D), iptr,
                                ctypes.byref(p), ctypes.byref(h)))
    try:
        res = _collect(h, circ.var_doubles, True)
        if keep is not None:
            _collect_trace(h, res, p.record_count, p.record_sweeps, circ.var_doubles)
    finally:
        lib().qf_result_destroy(h)
    return res


instantiate = qf_instantiate


def qf_instantiate_many(circuits, targets, initials, **params) -> list:
    """NEXT-2: several problems (own template, target, starts) in one resident
    launch (qf.h qf_instantiate_many).  Returns one Result per problem."""
    P = len(circuits)
    assert len(targets) == P and len(initials) == P
    ts = [_cplx(t) for t in targets]
    ins = [np.ascontiguousarray(x, dtype=np.float64) for x in initials]
    for c, x in zip(circuits, ins):
        assert x.ndim == 2 and x.shape[1] == c.var_doubles, (x.shape, c.var_doubles)
    S = np.array([x.shape[0] for x in ins], dtype=np.int32)
    p, _ = _make_params(1, **params)
    hs = (_VP * P)(*[c.h for c in circuits])
    tp = (_D * P)(*[t.ctypes.data_as(_D) for t in ts])
    ip = (_D * P)(*[x.ctypes.data_as(_D) for x in ins])
    out = (_VP * P)()
    _check(lib().qf_instantiate_many(P, hs, tp, ip, S.ctypes.data_as(_I), ctypes.byref(p), out))
    res = []
    try:
        for q in range(P):
            res.append(_collect(out[q], circuits[q].var_doubles, True))
    finally:
        for q in range(P):
            lib().qf_result_destroy(out[q])
    return res


instantiate_many = qf_instantiate_many


def qf_unitary_to_u3(u) -> tuple:
    """(theta, phi, lambda, gamma) with u = e^{i gamma} U3(theta, phi, lambda)."""
    a = _cplx(np.asarray(u).reshape(2, 2))
    out = np.zeros(4)
    _check(lib().qf_unitary_to_u3(a.ctypes.data_as(_D), out.ctypes.data_as(_D)))
    return tuple(float(x) for x in out)


unitary_to_u3 = qf_unitary_to_u3


def qf_workspace_size(circ: Circuit, S, **params) -> int:
    p = qf_params_default(num_starts=int(S), **params)
    return int(lib().qf_workspace_size(circ.h, ctypes.byref(p)))


def qf_instantiate_device(circ: Circuit, d_target, d_initial, workspace, stream=None,
                          d_gates_out=None, d_summary_out=None, want_result=True,
                          record_starts=None, record_sweeps=0, **params):
    """Blocking instantiation from device-resident torch tensors.

    d_target: complex128 (N, N) or float64 (N, N, 2) CUDA tensor; d_initial:
    float64 (S, var) CUDA tensor, or None for `num_starts` seeded starts
    (params seed / start_offset); workspace: uint8 CUDA tensor of at least
    qf_workspace_size bytes; stream: torch.cuda.Stream (default: current)."""
    import torch

    S = int(d_initial.shape[0]) if d_initial is not None else int(params.pop("num_starts"))
    params.pop("num_starts", None)
    p, keep = _make_params(S, record_starts, record_sweeps, **params)
    st = stream if stream is not None else torch.cuda.current_stream()
    h = _VP()
    _check(lib().qf_instantiate_device(
        circ.h, _VP(d_target.data_ptr()),
        _VP(d_initial.data_ptr()) if d_initial is not None else None, ctypes.byref(p),
        _VP(workspace.data_ptr()), int(workspace.numel() * workspace.element_size()),
        _VP(st.cuda_stream), _VP(d_gates_out.data_ptr()) if d_gates_out is not None else None,
        _VP(d_summary_out.data_ptr()) if d_summary_out is not None else None,
        ctypes.byref(h) if want_result else None))
    if not want_result:
        return None
    try:
        res = _collect(h, circ.var_doubles, False)
        if keep is not None:
            _collect_trace(h, res, p.record_count, p.record_sweeps, circ.var_doubles)
    finally:
        lib().qf_result_destroy(h)
    return res


instantiate_device = qf_instantiate_device


def qf_select_best_device(d_summaries, count, d_best, stream=None):
    """argmin kernel over `count` qf_summary records in a CUDA tensor."""
    import torch

    st = stream if stream is not None else torch.cuda.current_stream()
    _check(lib().qf_select_best_device(_VP(d_summaries.data_ptr()), int(count),
                                       _VP(st.cuda_stream), _VP(d_best.data_ptr())))


def qf_select_best_host(summaries: np.ndarray) -> int:
    s = np.ascontiguousarray(summaries, dtype=SUMMARY_DTYPE)
    out = ctypes.c_int64()
    _check(lib().qf_select_best_host(s.ctypes.data_as(ctypes.POINTER(qf_summary)), len(s),
                                     ctypes.byref(out)))
    return int(out.value)


def qf_instantiate_ptr(circ: Circuit, target_ptr: int, initial_ptr: int, S: int, **params) -> dict:
    """qf_instantiate on raw HOST pointers (e.g. pinned torch tensors); returns
    the call's qf_stats plus the best start's summary (bench e2e leg)."""
    p, _ = _make_params(S, **params)
    h = _VP()
    _check(lib().qf_instantiate(circ.h, ctypes.cast(target_ptr, _D),
                                ctypes.cast(initial_ptr, _D) if initial_ptr else None,
                                ctypes.byref(p), ctypes.byref(h)))
    try:
        st = qf_stats()
        _check(lib().qf_result_stats(h, ctypes.byref(st)))
        out = {f: getattr(st, f) for f, _ in qf_stats._fields_}
        out["best"] = lib().qf_result_best(h)
    finally:
        lib().qf_result_destroy(h)
    return out
