"""NEXT-3 host logic on CPU: the grouping of the sweep schedule into runs of
steps on <= umax qubits (qf_engine.cu make_groups), read through the
library's debug export.  Checked against the definition: the groups list the
2p steps of TwoSidedSweep in order (backward p-1..0, forward 0..p-1); every
gate of a group lies in its W; |W| <= max(umax, arity); a group never grows
past the point where the next step would exceed the bound."""
import ctypes

import numpy as np
import pytest

import paper_2306_08152_b200 as qf
import qfgen
from test_gpu_next3 import u3_cnot_template


def groups(c: qf.Circuit, umax):
    L = qf.lib()
    f = L.qf_debug_groups
    f.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_int]
    buf = (ctypes.c_int * 100000)()
    n = f(c.h, umax, buf, len(buf))
    assert n >= 0
    out, i = [], 0
    while i < n:
        w = buf[i]
        wq = list(buf[i + 1:i + 1 + w])
        ns = buf[i + 1 + w]
        st = [(buf[i + 2 + w + 2 * j], buf[i + 3 + w + 2 * j]) for j in range(ns)]
        out.append((wq, st))
        i += 2 + w + 2 * ns
    return out


def schedule(p):
    return [(p - 1 - j, 0) for j in range(p)] + [(j, 1) for j in range(p)]


@pytest.mark.parametrize("umax", [1, 2, 3])
@pytest.mark.parametrize("case", ["u3cnot", "random", "c5"])
def test_groups_cover_schedule(case, umax):
    if case == "u3cnot":
        n = 8
        locs, kinds, cm = u3_cnot_template(n, 10)
    elif case == "random":
        n = 7
        locs, kinds, cm = qfgen.random_template(n, 15, seed=9, const_frac=0.3)
    else:
        w = qfgen.workload("C5")
        n, locs, kinds, cm = w.n, w.locs, w.kinds, w.const_mats
    c = qf.Circuit(n, locs, kinds, cm)
    g = groups(c, umax)
    flat = [s for _, st in g for s in st]
    assert flat == schedule(len(locs))  # every step once, in sweep order
    for wq, st in g:
        assert wq == sorted(set(wq))
        qs = set()
        for k, _ in st:
            assert set(locs[k]) <= set(wq)
            qs |= set(locs[k])
        assert qs == set(wq)  # W is exactly the union of the group's locations
        assert len(wq) <= max(umax, max(len(locs[k]) for k, _ in st))
        assert len(wq) <= 3
    # maximality: the first step of a group would not have fit into the previous one
    for (wq0, st0), (wq1, st1) in zip(g, g[1:]):
        k = st1[0][0]
        union = set(wq0) | set(locs[k])
        bound = min(3, max(umax, len(locs[k])))
        assert len(union) > bound or len(st0) >= 48


def test_u3cnot_pairs_group():
    """[CNOT(i,i+1), U(2) i, U(2) i+1] share a pair: with umax = 2 the
    backward and forward sweeps need at most ~1/3 of the passes."""
    n = 8
    locs, kinds, cm = u3_cnot_template(n, 10)
    g = groups(qf.Circuit(n, locs, kinds, cm), 2)
    assert len(g) <= 0.45 * 2 * len(locs)
