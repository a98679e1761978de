"""Host-side Tanner-graph model, alist I/O and the code builder.  CPU only."""
import pickle

import numpy as np
import pytest

from conftest import golden_code, load_golden
from paper_1204_0556_b200.codes import (
    AlistParseError, BASELINE_CODES, CodeGenerationError, ParityCheckMatrix, baseline_code,
    emit_alist, gen_regular_ldpc, is_codeword, make_ldpc, parse_alist)

HAMMING = [[1, 1, 0, 1, 1, 0, 0], [1, 0, 1, 1, 0, 1, 0], [0, 1, 1, 1, 0, 0, 1]]


def test_edge_arrays_follow_reference_layout():
    c = ParityCheckMatrix(5, [[3, 0, 1], [4, 2], [1, 2, 4]])
    assert c.edge_var.tolist() == [0, 1, 3, 2, 4, 1, 2, 4]     # sorted per check (codes.py:42)
    assert c.check_ptr.tolist() == [0, 3, 5, 8]
    assert c.var_degrees.tolist() == [1, 2, 2, 1, 2]
    assert c.n_edges == 8
    assert set(c.checks_by_degree) == {2, 3}
    assert c.checks_by_degree[3].tolist() == [[0, 1, 2], [5, 6, 7]]
    ptr, eids = c.var_edges
    assert ptr.tolist() == [0, 1, 3, 5, 6, 8]
    assert c.edge_var[eids].tolist() == [0, 1, 1, 2, 2, 3, 4, 4]
    assert [a.tolist() for a in c.var_neighborhoods] == [[0], [0, 2], [1, 2], [0], [1, 2]]


def test_validation_errors():
    with pytest.raises(ValueError):
        ParityCheckMatrix(0, [[0]])
    with pytest.raises(ValueError):
        ParityCheckMatrix(3, [])
    with pytest.raises(ValueError):
        ParityCheckMatrix(3, [[0, 0]])
    with pytest.raises(ValueError):
        ParityCheckMatrix(3, [[0, 3]])
    with pytest.raises(ValueError):
        ParityCheckMatrix(3, [[]])


def test_dense_roundtrip_pickle_and_codeword():
    c = ParityCheckMatrix.from_dense(HAMMING)
    assert np.array_equal(c.to_dense(), np.array(HAMMING, dtype=np.uint8))
    assert pickle.loads(pickle.dumps(c)) == c
    assert is_codeword(c, np.zeros(7, np.uint8))
    assert not is_codeword(c, np.eye(7, dtype=np.uint8)[0])
    with pytest.raises(ValueError):
        is_codeword(c, np.zeros(6))
    with pytest.raises(ValueError):
        is_codeword(c, np.full(7, 2))


def test_alist_roundtrip_and_errors():
    c = make_ldpc(48, 3, 6, seed=2)
    assert parse_alist(emit_alist(c)) == c
    with pytest.raises(AlistParseError):
        parse_alist("3\n")
    bad = emit_alist(c).splitlines()
    bad[4] = "1 2"
    with pytest.raises(AlistParseError):
        parse_alist("\n".join(bad))


def test_gen_regular_ldpc_reference_semantics():
    c = gen_regular_ldpc(30, 3, 6, seed=1)
    assert set(c.var_degrees.tolist()) == {3} and set(c.check_degrees.tolist()) == {6}
    assert gen_regular_ldpc(30, 3, 6, seed=1) == c  # deterministic per seed
    with pytest.raises(CodeGenerationError):
        gen_regular_ldpc(20, 3, 13 if False else 4, seed=0, max_attempts=0)
    with pytest.raises(ValueError):
        gen_regular_ldpc(10, 3, 4, seed=0)


@pytest.mark.parametrize("name", ["cfg1_n96", "cfg2_n1008", "cfg4_n1040"])
def test_baseline_codes(name):
    n, dv, dc, g6 = BASELINE_CODES[name]
    c = baseline_code(name)
    assert c.n_vars == n and c.n_checks == n * dv // dc
    assert set(c.var_degrees.tolist()) == {dv} and set(c.check_degrees.tolist()) == {dc}
    if g6:
        assert c.girth_at_least_6()
    assert baseline_code(name) == c


@pytest.mark.parametrize("fixture,name", [("decode_cfg1.npz", "cfg1_n96"), ("decode_cfg2.npz", "cfg2_n1008"),
                                          ("decode_cfg4.npz", "cfg4_n1040")])
def test_builder_is_pinned_by_golden(fixture, name):
    assert golden_code(load_golden(fixture)) == baseline_code(name)


def test_make_ldpc_girth_and_repair():
    c = make_ldpc(240, 3, 6, seed=11)
    assert c.girth_at_least_6()
    c2 = make_ldpc(96, 3, 6, seed=5, girth6=False)
    assert all(len(set(r.tolist())) == r.size for r in c2.check_neighborhoods)
