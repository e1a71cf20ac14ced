"""Pin the CPU oracle (oracle/hsk_oracle.c) against the reference.

The golden fixtures were produced by the reference itself
(tests/golden/make_golden.py).  SJLT (both directions) and SRHT must match
BIT-EXACTLY: the oracle restates the reference's operation order, including
np.add.reduceat's pairwise summation.  The Gaussian product uses OpenBLAS in
the reference, whose order is not reproducible: 1e-13 relative there.
"""

import math

import numpy as np
import pytest
import scipy.linalg as sla

from conftest import case_inputs
from oracle import oracle as O


def _blocks(arrays, case):
    out = []
    for bi, (rows, _seed) in enumerate(case["blocks"]):
        p = f"{case['name']}/b{bi}/"
        out.append((rows, p))
    return out


def _oracle_case(arrays, case, A, B):
    S, St = [], []
    for rows, p in _blocks(arrays, case):
        if case["kind"] == "sjlt":
            s = 1.0 / math.sqrt(case["alpha"])
            S.append(O.sjlt_right(A, arrays[p + "pos"], arrays[p + "signs"], rows, s))
            St.append(O.sjlt_right_t(B, arrays[p + "pos"], arrays[p + "signs"], rows, s))
        elif case["kind"] == "gaussian":
            S.append(O.gauss(A, arrays[p + "matrix"], False))
            St.append(O.gauss(B, arrays[p + "matrix"], True))
        else:
            sc = 1.0 / math.sqrt(rows)
            S.append(O.srht(A, arrays[p + "signs"], arrays[p + "sample"], rows, sc, False))
            St.append(O.srht(B, arrays[p + "signs"], arrays[p + "sample"], rows, sc, True))
    return np.hstack(S), np.hstack(St)


def test_inputs_regenerate_bit_exactly(golden):
    import hashlib
    arrays, man = golden
    for case in man["cases"]:
        A, B = case_inputs(case)
        assert hashlib.sha256(A.tobytes()).hexdigest() == case["sha_A"], case["name"]
        assert hashlib.sha256(B.tobytes()).hexdigest() == case["sha_B"], case["name"]


def test_oracle_matches_reference_bit_exactly(golden):
    arrays, man = golden
    for case in man["cases"]:
        A, B = case_inputs(case)
        S, St = _oracle_case(arrays, case, A, B)
        ref_S, ref_St = arrays[case["name"] + "/S"], arrays[case["name"] + "/St"]
        if case["kind"] == "gaussian":
            assert O.rel_frobenius(S, ref_S) <= 1e-13, case["name"]
            assert O.rel_frobenius(St, ref_St) <= 1e-13, case["name"]
        else:
            np.testing.assert_array_equal(S, ref_S, err_msg=case["name"])
            np.testing.assert_array_equal(St, ref_St, err_msg=case["name"])


def test_oracle_matches_dense_materialisation(golden):
    arrays, man = golden
    for case in man["cases"]:
        A, B = case_inputs(case)
        S, St = _oracle_case(arrays, case, A, B)
        dense = arrays[case["name"] + "/dense"]
        tol = 1e-12 * max(np.linalg.norm(A), np.linalg.norm(B))
        assert np.max(np.abs(S - A @ dense)) <= tol
        assert np.max(np.abs(St - B.T @ dense)) <= tol


def test_worked_pattern_and_empty_buckets(golden):
    arrays, man = golden
    w = man["patterns"][0]
    A = np.random.default_rng(w["data_seed"]).standard_normal((5, 4))
    s = 1.0 / math.sqrt(2.0)
    np.testing.assert_array_equal(O.sjlt_right(A, w["pos"], w["signs"], 3, s),
                                  arrays["worked_pattern/S"])
    np.testing.assert_array_equal(O.sjlt_right_t(A.T, w["pos"], w["signs"], 3, s),
                                  arrays["worked_pattern/St"])
    e = man["patterns"][1]
    Ae = np.arange(6.0).reshape(2, 3)
    np.testing.assert_array_equal(O.sjlt_right_t(Ae, e["pos"], e["signs"], 3, 1.0),
                                  arrays["trailing_empty/St"])
    np.testing.assert_array_equal(O.sjlt_right(Ae.T, e["pos"], e["signs"], 3, 1.0),
                                  arrays["trailing_empty/S"])


def test_reduceat_restatement(golden):
    arrays, man = golden
    for L in man["reduceat_lengths"]:
        x = arrays[f"reduceat/{L}/x"]
        assert O.reduceat_segment(x) == arrays[f"reduceat/{L}/y"][0]


def test_reduceat_restatement_random_lengths():
    rng = np.random.default_rng(7)
    for L in list(range(1, 140)) + [255, 256, 257, 511, 1000, 4097]:
        x = rng.standard_normal(L) * np.exp(4 * rng.standard_normal(L))
        ref = np.add.reduceat(np.concatenate([x, [0.0]]), [0, L])[0]
        assert O.reduceat_segment(x) == ref, L


def test_fwht_known_answers(golden):
    arrays, _ = golden
    np.testing.assert_array_equal(O.fwht([1.0, 1.0, 1.0, 1.0]), arrays["fwht/const4"])
    X = np.random.default_rng(1).standard_normal((3, 16))
    np.testing.assert_array_equal(O.fwht(X), arrays["fwht/rows16"])
    for n in (1, 2, 4, 8, 32, 64):
        x = np.random.default_rng(n).standard_normal(n)
        np.testing.assert_allclose(O.fwht(x), sla.hadamard(n) @ x / math.sqrt(n), atol=1e-12)
    with pytest.raises(ValueError):
        O.fwht(np.ones(6))


def test_oracle_threads_do_not_change_results():
    rng = np.random.default_rng(3)
    A = rng.standard_normal((300, 257))
    pos = rng.integers(0, 40, size=(257, 4))
    sg = (rng.integers(0, 2, size=(257, 4)) * 2 - 1).astype(np.int8)
    one = O.sjlt_right(A, pos, sg, 40, 0.5, nthreads=1)
    many = O.sjlt_right(A, pos, sg, 40, 0.5, nthreads=4)
    np.testing.assert_array_equal(one, many)
    one_t = O.sjlt_right_t(A.T.copy(order="F"), pos, sg, 40, 0.5, nthreads=1)
    many_t = O.sjlt_right_t(A.T.copy(order="F"), pos, sg, 40, 0.5, nthreads=4)
    np.testing.assert_array_equal(one_t, many_t)


def test_row_and_column_slab_oracles_are_exact():
    # rows of S depend only on rows of A; rows of S' only on columns of A
    rng = np.random.default_rng(11)
    A = rng.standard_normal((120, 96))
    pos = rng.integers(0, 16, size=(96, 3))
    sg = (rng.integers(0, 2, size=(96, 3)) * 2 - 1).astype(np.int8)
    full = O.sjlt_right(A, pos, sg, 16, 0.5)
    np.testing.assert_array_equal(O.sjlt_right(A[37:81], pos, sg, 16, 0.5), full[37:81])
    pos2 = rng.integers(0, 16, size=(120, 3))
    sg2 = (rng.integers(0, 2, size=(120, 3)) * 2 - 1).astype(np.int8)
    full_t = O.sjlt_right_t(A, pos2, sg2, 16, 0.5)
    np.testing.assert_array_equal(O.sjlt_right_t(A[:, 10:50], pos2, sg2, 16, 0.5), full_t[10:50])
