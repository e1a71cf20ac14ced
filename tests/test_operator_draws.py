"""The host mirror draws R bit-identically to the reference (CPU only).

R is never regenerated on the GPU; these tests pin our draws (draws.py via
operators.py) against the reference's own arrays and hashes recorded in
tests/golden (make_golden.py), plus the reference's validation behaviour.
"""

import hashlib
import math

import numpy as np
import pytest

from conftest import seed_of
from paper_2302_01977_b200 import sketching as sk


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _build(case):
    kw = {}
    if case["kind"] == "sjlt":
        kw = dict(alpha=case["alpha"], construction=case["construction"])
    (rows0, s0), *rest = case["blocks"]
    op = sk.new_operator(case["kind"], case["n"], rows0, seed_of(s0), **kw)
    for rows, s in rest:
        op = sk.append_columns(op, rows, seed_of(s))
    return op


def test_block_draws_match_reference(golden):
    arrays, man = golden
    for case in man["cases"]:
        op = _build(case)
        assert op.d == case["d"]
        for bi, blk in enumerate(op.blocks):
            p = f"{case['name']}/b{bi}/"
            if case["kind"] == "sjlt":
                np.testing.assert_array_equal(blk._pos, arrays[p + "pos"])
                np.testing.assert_array_equal(blk._signs, arrays[p + "signs"])
                assert blk._pos.dtype == np.intp and blk._signs.dtype == np.int8
            elif case["kind"] == "gaussian":
                np.testing.assert_array_equal(blk.matrix, arrays[p + "matrix"])
            else:
                np.testing.assert_array_equal(blk.signs, arrays[p + "signs"])
                np.testing.assert_array_equal(blk.sample, arrays[p + "sample"])
                assert blk.n_pad == case["n_pad"]
        dense = sk.dense_rows(op, np.arange(op.n), np.arange(op.d))
        np.testing.assert_array_equal(dense, arrays[case["name"] + "/dense"])


def test_config_size_draws_match_reference_hashes(golden):
    _, man = golden
    for dr in man["draws"]:
        kw = dict(alpha=dr["alpha"], construction=dr["construction"]) if dr["kind"] == "sjlt" else {}
        op = sk.new_operator(dr["kind"], dr["n"], dr["d"],
                             np.random.SeedSequence(tuple(dr["seed_sequence"])), **kw)
        b = op.blocks[0]
        if dr["kind"] == "sjlt":
            assert _sha(np.asarray(b._pos, dtype=np.int64)) == dr["sha"]["pos"]
            assert _sha(b._signs) == dr["sha"]["signs"]
        elif dr["kind"] == "gaussian":
            assert _sha(b.matrix) == dr["sha"]["matrix"]
        else:
            assert _sha(b.signs) == dr["sha"]["signs"]
            assert _sha(np.asarray(b.sample, dtype=np.int64)) == dr["sha"]["sample"]


def test_worked_pattern_storage(golden):
    arrays, man = golden
    w = man["patterns"][0]
    blk = sk.SjltBlock.from_pattern(4, 3, 2, w["pos"], w["signs"])
    st = blk.storage
    assert st.scale == 1.0 / math.sqrt(2.0)
    for f in ("plus_rowptr", "plus_cols", "minus_rowptr", "minus_cols",
              "plus_colptr", "plus_rows", "minus_colptr", "minus_rows"):
        np.testing.assert_array_equal(getattr(st, f), arrays[f"worked_pattern/{f}"], err_msg=f)
    np.testing.assert_array_equal(blk.dense_rows(np.arange(4), np.arange(3)),
                                  arrays["worked_pattern/dense"])


def test_validation_matches_reference():
    with pytest.raises(ValueError):
        sk.new_operator(sk.SJLT, 4, 3, seed=0, alpha=2, construction=sk.BLOCK)
    with pytest.raises(ValueError):
        sk.new_operator(sk.SJLT, 16, 4, seed=0, alpha=0, construction=sk.GRAPH)
    with pytest.raises(ValueError):
        sk.new_operator(sk.SJLT, 16, 4, seed=0, alpha=5, construction=sk.GRAPH)
    with pytest.raises(ValueError):
        sk.new_operator(sk.SJLT, 16, 4, seed=0, alpha=None, construction=sk.GRAPH)
    with pytest.raises(ValueError):
        sk.new_operator(sk.SJLT, 16, 4, seed=0, alpha=2, construction="dense")
    with pytest.raises(ValueError):
        sk.new_operator(sk.GAUSSIAN, 8, 0, seed=0)
    with pytest.raises(ValueError):
        sk.new_operator(sk.GAUSSIAN, 8, 9, seed=0)
    with pytest.raises(ValueError):
        sk.new_operator("fourier", 8, 4, seed=0)
    op = sk.new_operator(sk.GAUSSIAN, 8, 2, seed=0)
    with pytest.raises(ValueError):
        sk.append_columns(op, 0, seed=1)


def test_apply_dimension_mismatch_raises_before_device():
    # shape validation happens on the host, so it holds without a GPU
    op = sk.new_operator(sk.GAUSSIAN, 8, 4, seed=0)
    with pytest.raises(ValueError):
        sk.apply_right(np.zeros((3, 9)), op)
    with pytest.raises(ValueError):
        sk.apply_right_transposed(np.zeros((9, 3)), op)


def test_append_shares_blocks_and_preserves_prefix():
    op = sk.new_operator(sk.SRHT, 32, 6, seed=21)
    before = sk.dense_rows(op, np.arange(32), np.arange(6))
    grown = sk.append_columns(op, 5, seed=99)
    assert grown.d == 11 and grown.blocks[0] is op.blocks[0]
    np.testing.assert_array_equal(sk.dense_rows(grown, np.arange(32), np.arange(6)), before)


def test_sjlt_structure():
    for cons in (sk.BLOCK, sk.GRAPH):
        op = sk.new_operator(sk.SJLT, 40, 8, seed=11, alpha=4, construction=cons)
        Rt = sk.dense_rows(op, np.arange(40), np.arange(8))
        np.testing.assert_array_equal(np.sum(Rt ** 2, axis=1), 1.0)
        np.testing.assert_array_equal(np.count_nonzero(Rt, axis=1), 4)
    op = sk.new_operator(sk.SJLT, 25, 12, seed=13, alpha=3, construction=sk.BLOCK)
    Rt = sk.dense_rows(op, np.arange(25), np.arange(12))
    for row in Rt:
        np.testing.assert_array_equal(np.sort(np.flatnonzero(row)) // 4, [0, 1, 2])


def test_dense_rows_bounds_and_subsets():
    op = sk.new_operator(sk.GAUSSIAN, 10, 6, seed=1)
    full = sk.dense_rows(op, np.arange(10), np.arange(6))
    rows, cols = np.array([7, 2, 2]), np.array([5, 0])
    np.testing.assert_array_equal(sk.dense_rows(op, rows, cols), full[np.ix_(rows, cols)])
    assert sk.dense_rows(op, np.array([], dtype=int), np.arange(6)).shape == (0, 6)
    with pytest.raises(IndexError):
        sk.dense_rows(op, np.array([10]), np.arange(6))
    with pytest.raises(IndexError):
        sk.dense_rows(op, np.array([0]), np.array([6]))


def test_dense_accessor_contract():
    A = np.arange(12.0).reshape(3, 4)
    acc = sk.DenseAccessor(A)
    buf = acc.dense()
    assert buf.flags.f_contiguous and acc.dense() is buf and acc.shape == (3, 4)
    np.testing.assert_array_equal(acc.extract([2, 0], [1, 3]), A[np.ix_([2, 0], [1, 3])])
