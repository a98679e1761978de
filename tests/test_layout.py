"""Host-side Tanner-graph layouts (csrc/layout.h) on the CPU: the colored
layout's coloring invariants (one edge of every color per variable, q or
q+1 per check matching its rotation, slots by color) and the slot layout's
clash-freedom, on the BASELINE codes."""
import ctypes
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_1204_0556_b200 import baseline_code

HERE = Path(__file__).resolve().parent


@pytest.fixture(scope="module")
def harness(tmp_path_factory):
    out = tmp_path_factory.mktemp("layout") / "liblayout_harness.so"
    subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", str(out),
                    str(HERE / "native" / "layout_harness.cpp")], check=True)
    lib = ctypes.CDLL(str(out))
    P, I, LL, U = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_uint64
    lib.layout_colored.argtypes = [I, I, P, P, I, I, LL, U, P, P, P, P]
    lib.layout_slots.argtypes = [I, I, P, P, I, LL, U, P, P, P]
    return lib


def _arr(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


@pytest.mark.parametrize("name,D", [("cfg1_n96", 6), ("cfg2_n1008", 6), ("cfg4_n1040", 13)])
def test_colored_layout_invariants(harness, name, D):
    code = baseline_code(name)
    M, N, DV = code.n_checks, code.n_vars, 3
    ptr, ev = _arr(code.check_ptr, np.int32), _arr(code.edge_var, np.int32)
    slot = np.zeros(M * D, np.int32)
    rot = np.zeros(M, np.int32)
    sov = np.zeros(N, np.int32)
    costs = np.zeros(2)
    rc = harness.layout_colored(N, M, ptr.ctypes.data, ev.ctypes.data, D, DV, 200000, 7, slot.ctypes.data,
                                rot.ctypes.data, sov.ctypes.data, costs.ctypes.data)
    assert rc == 0
    assert sorted(sov.tolist()) == list(range(N))  # a permutation
    slot = slot.reshape(M, D)
    color = (slot + rot[:, None]) % DV  # color of every edge (check-major, sorted rows)
    for c in range(M):
        assert sorted(slot[c].tolist()) == list(range(D))  # every slot used once
        counts = np.bincount(color[c], minlength=DV)
        want = np.full(DV, D // DV)
        if D % DV:
            want[rot[c]] += 1
        assert np.array_equal(counts, want)
    per_var = [[] for _ in range(N)]
    for c in range(M):
        for r in range(D):
            per_var[ev[ptr[c] + r]].append(color[c, r])
    assert all(sorted(v) == list(range(DV)) for v in per_var)
    assert costs[1] <= costs[0]


def test_colored_layout_rejects_unsupported_shapes(harness):
    # (3,7): D mod DV = 1 but M (DV - 1) / DV is not an integer for 3 checks of 7
    from paper_1204_0556_b200 import ParityCheckMatrix

    code = ParityCheckMatrix.from_dense(np.ones((1, 5), dtype=int))  # one check of degree 5, DV = 1
    ptr, ev = _arr(code.check_ptr, np.int32), _arr(code.edge_var, np.int32)
    out = [np.zeros(5, np.int32), np.zeros(1, np.int32), np.zeros(5, np.int32), np.zeros(2)]
    rc = harness.layout_colored(5, 1, ptr.ctypes.data, ev.ctypes.data, 5, 2, 1000, 1, *(o.ctypes.data for o in out))
    assert rc == 1


@pytest.mark.parametrize("name,D", [("cfg2_n1008", 6), ("cfg4_n1040", 13)])
def test_slot_layout_is_clash_free(harness, name, D):
    code = baseline_code(name)
    M, N = code.n_checks, code.n_vars
    ptr, ev = _arr(code.check_ptr, np.int32), _arr(code.edge_var, np.int32)
    slot = np.zeros(M * D, np.int32)
    sov = np.zeros(N, np.int32)
    costs = np.zeros(2)
    rc = harness.layout_slots(N, M, ptr.ctypes.data, ev.ctypes.data, D, 400000, 12345, slot.ctypes.data,
                              sov.ctypes.data, costs.ctypes.data)
    assert rc == 0  # every variable's edges in distinct slots
    slot = slot.reshape(M, D)
    seen = [set() for _ in range(N)]
    for c in range(M):
        for r in range(D):
            v = ev[ptr[c] + r]
            assert slot[c, r] not in seen[v]
            seen[v].add(slot[c, r])
