"""GPU parity: libhsk kernels through the public API vs reference + oracle.

Tolerances (BASELINE.json north_star): the sketch must match the reference's
on the same inputs and the same R within 1e-12 relative Frobenius (fp64);
the reference's own kernel tests use max|diff| <= 1e-12..1e-14 * ||A||_F
(test_sketching.py:53-131, test_acceptance.py:66-93), asserted here too.
R is bit-exact by construction (tests/test_operator_draws.py).
"""

import math

import numpy as np
import pytest

from conftest import case_inputs, seed_of
from oracle import oracle as O
from paper_2302_01977_b200 import adaptive, device
from paper_2302_01977_b200 import sketching as sk

pytestmark = pytest.mark.gpu

REL = 1e-12


def _op(case):
    kw = dict(alpha=case["alpha"], construction=case["construction"]) if case["kind"] == "sjlt" else {}
    (r0, s0), *rest = case["blocks"]
    op = sk.new_operator(case["kind"], case["n"], r0, seed_of(s0), **kw)
    for rows, s in rest:
        op = sk.append_columns(op, rows, seed_of(s))
    return op


def _close(x, ref, scale_norm, rel=REL):
    assert x.shape == ref.shape
    assert O.rel_frobenius(x, ref) <= rel
    assert np.max(np.abs(x - ref), initial=0.0) <= 1e-12 * scale_norm


def test_golden_cases(golden, cuda):
    arrays, man = golden
    for case in man["cases"]:
        op = _op(case)
        A, B = case_inputs(case)
        S = sk.apply_right(A, op)
        St = sk.apply_right_transposed(B, op)
        assert S.flags.f_contiguous and St.flags.f_contiguous
        _close(S, arrays[case["name"] + "/S"], np.linalg.norm(A))
        _close(St, arrays[case["name"] + "/St"], np.linalg.norm(B))


def test_worked_pattern_and_trailing_empty(golden, cuda):
    arrays, man = golden
    w = man["patterns"][0]
    blk = sk.SjltBlock.from_pattern(4, 3, 2, w["pos"], w["signs"])
    A = np.random.default_rng(w["data_seed"]).standard_normal((5, 4))
    np.testing.assert_allclose(blk.apply_right(np.asfortranarray(A)),
                               arrays["worked_pattern/S"], atol=1e-14)
    np.testing.assert_allclose(blk.apply_right_transposed(np.asfortranarray(A.T)),
                               arrays["worked_pattern/St"], atol=1e-14)
    e = man["patterns"][1]
    blk = sk.SjltBlock.from_pattern(2, 3, 1, e["pos"], e["signs"])
    Ae = np.arange(6.0).reshape(2, 3)
    np.testing.assert_array_equal(blk.apply_right_transposed(np.asfortranarray(Ae)),
                                  arrays["trailing_empty/St"])


def test_acceptance_criterion_2(cuda):
    """Reference acceptance 2 (test_acceptance.py:66-93) through the GPU."""
    rng = np.random.default_rng(2024)
    for trial in range(100):
        m = int(rng.integers(8, 65))
        n = int(rng.integers(8, 65))
        A = rng.standard_normal((m, n))
        tol = 1e-12 * np.linalg.norm(A)
        alpha = (1, 2, 4)[trial % 3]
        for cons in (sk.BLOCK, sk.GRAPH):
            if cons == sk.BLOCK:
                d_r = alpha * int(rng.integers(1, min(32, n) // alpha + 1))
                d_l = alpha * int(rng.integers(1, min(32, m) // alpha + 1))
            else:
                d_r = int(rng.integers(alpha, min(32, n) + 1))
                d_l = int(rng.integers(alpha, min(32, m) + 1))
            op_r = sk.new_operator(sk.SJLT, n, d_r, seed=(2, trial), alpha=alpha, construction=cons)
            Rt = sk.dense_rows(op_r, np.arange(n), np.arange(d_r))
            assert np.max(np.abs(sk.apply_right(A, op_r) - A @ Rt)) <= tol
            op_l = sk.new_operator(sk.SJLT, m, d_l, seed=(3, trial), alpha=alpha, construction=cons)
            Lt = sk.dense_rows(op_l, np.arange(m), np.arange(d_l))
            assert np.max(np.abs(sk.apply_right_transposed(A, op_l) - A.T @ Lt)) <= tol


@pytest.mark.parametrize("m,n,d,alpha,cons", [
    (1, 64, 8, 2, "graph"), (31, 100, 3, 1, "graph"), (33, 129, 63, 3, "graph"),
    (64, 64, 64, 8, "block"), (65, 300, 65, 5, "graph"), (127, 1000, 128, 4, "block"),
    (129, 517, 200, 8, "graph"), (200, 2048, 256, 4, "graph"), (333, 1500, 300, 4, "block"),
    (96, 4096, 512, 8, "block"), (70, 3000, 513, 3, "graph"), (40, 5000, 2048, 8, "block"),
    (50, 700, 600, 33, "graph"), (20, 400, 300, 100, "graph"),
])
def test_sjlt_shapes_vs_oracle(cuda, m, n, d, alpha, cons):
    rng = np.random.default_rng(m * 1000 + d)
    op = sk.new_operator(sk.SJLT, n, d, seed=(m, n, d), alpha=alpha, construction=cons)
    b = op.blocks[0]
    A = rng.standard_normal((m, n))
    ref = O.sjlt_right(A, b._pos, b._signs, d, b._scale)
    _close(sk.apply_right(A, op), ref, np.linalg.norm(A))
    B = rng.standard_normal((n, m))
    ref_t = O.sjlt_right_t(B, b._pos, b._signs, d, b._scale)
    _close(sk.apply_right_transposed(B, op), ref_t, np.linalg.norm(B))


@pytest.mark.parametrize("m,n,d,alpha", [
    (5000, 3000, 300, 4), (9000, 1000, 64, 8), (4000, 2600, 700, 4), (3000, 5000, 2048, 8),
    (150, 20000, 512, 4),
])
def test_sjlt_schedules_vs_oracle(cuda, tune, m, n, d, alpha):
    """Whole-tile (k-split) and persistent stream-K schedules, with and without
    TMA multicast across slab clusters: all match the oracle, and stream-K's
    cross-CTA tile fixup is bitwise repeatable."""
    rng = np.random.default_rng(m + n + d)
    op = sk.new_operator(sk.SJLT, n, d, seed=(m, d), alpha=alpha, construction=sk.BLOCK)
    b = op.blocks[0]
    A = rng.standard_normal((m, n))
    B = rng.standard_normal((n, m))
    ref = O.sjlt_right(A, b._pos, b._signs, d, b._scale)
    ref_t = O.sjlt_right_t(B, b._pos, b._signs, d, b._scale)
    dA, dB = device.DeviceMatrix.from_host(A), device.DeviceMatrix.from_host(B)
    # whole-tile / stream-K schedules, each with and without slab-cluster
    # TMA multicast (opt-in path)
    for mode, mc in (("0", "0"), ("1", "0"), ("0", "1"), ("1", "1")):
        tune("HSK_SJLT_STREAMK", mode)
        tune("HSK_SJLT_MC", mc)
        s1 = sk.apply_right_device(dA, op).to_host()
        s2 = sk.apply_right_device(dA, op).to_host()
        _close(s1, ref, np.linalg.norm(A))
        np.testing.assert_array_equal(s1, s2)
        t1 = sk.apply_right_transposed_device(dB, op).to_host()
        t2 = sk.apply_right_transposed_device(dB, op).to_host()
        _close(t1, ref_t, np.linalg.norm(B))
        np.testing.assert_array_equal(t1, t2)


@pytest.mark.parametrize("ws", ["16", "20", "24"])
def test_sjlt_warp_shapes_vs_oracle(cuda, tune, ws):
    """S's consumer-warp shapes (16 x 16, 20 x 13, 24 x 11: slabs of 256 / 260 /
    264 buckets, the last one partial) under both schedules; a forced shape
    leaves S' on its 16 x 16 kernels."""
    m, n, d = 1000, 3000, 700
    rng = np.random.default_rng(7)
    op = sk.new_operator(sk.SJLT, n, d, seed=(m, d), alpha=4, construction=sk.BLOCK)
    b = op.blocks[0]
    A = rng.standard_normal((m, n))
    B = rng.standard_normal((n, m))
    tune("HSK_SJLT_W32", ws)
    for mode in ("0", "1"):
        tune("HSK_SJLT_STREAMK", mode)
        _close(sk.apply_right(A, op), O.sjlt_right(A, b._pos, b._signs, d, b._scale), np.linalg.norm(A))
        _close(sk.apply_right_transposed(B, op), O.sjlt_right_t(B, b._pos, b._signs, d, b._scale),
               np.linalg.norm(B))


@pytest.mark.parametrize("m,n,d,alpha", [
    (5000, 3000, 128, 4),      # single slab, a = 4: transposed tile by default
    (7000, 2000, 256, 8),      # a = 8
    (6000, 1500, 64, 8),       # paired plan (default: natural layout)
    (9000, 1100, 512, 4),      # two slabs, a = 2 (default: natural layout)
    (300, 9000, 200, 5),       # few row tiles, long rows: k-split clusters
    (8000, 1500, 64, 4),       # 128-row tiles (d <= 64): transposed tile by default
    (4100, 2000, 32, 2),
])
def test_sjlt_transposed_tile_paths_vs_oracle(cuda, tune, m, n, d, alpha):
    """S' tiles in both layouts (HSK_SJLT_XP = 0: the TMA-landed natural layout
    of 64-row tiles, modes 3 / 1, and the XOR-transposed 128-row tiles, modes
    4 / 1; = 1: transposed in shared memory into the S layout, modes 5 / 6)
    under both schedules, for aligned (TMA) and odd-ld
    (cp.async) operands; every variant is bitwise repeatable."""
    rng = np.random.default_rng(m + d)
    B = rng.standard_normal((n, m))
    # one operator for both settings: its cached device plan is rebuilt when the
    # knobs change (hsk_tuning_generation, device.block_state)
    op = sk.new_operator(sk.SJLT, n, d, seed=(m, d), alpha=alpha, construction=sk.BLOCK)
    b = op.blocks[0]
    ref_t = O.sjlt_right_t(B, b._pos, b._signs, d, b._scale)
    for xp in ("0", "1"):
        tune("HSK_SJLT_XP", xp)
        for ld in (n + (n & 1), n + 1 - (n & 1)):       # even (TMA) / odd (cp.async)
            dB = device.DeviceMatrix(n, m, ld=ld)
            dB.upload(B)
            for mode in ("0", "1"):
                tune("HSK_SJLT_STREAMK", mode)
                t1 = sk.apply_right_transposed_device(dB, op).to_host()
                t2 = sk.apply_right_transposed_device(dB, op).to_host()
                _close(t1, ref_t, np.linalg.norm(B))
                np.testing.assert_array_equal(t1, t2)


def test_odd_leading_dimension_and_column_offset(cuda):
    rng = np.random.default_rng(5)
    m, n, d = 77, 333, 96
    A = rng.standard_normal((m, n))
    for kind, kw in ((sk.SJLT, dict(alpha=4, construction=sk.GRAPH)), (sk.GAUSSIAN, {}),
                     (sk.SRHT, {})):
        op = sk.new_operator(kind, n, d, seed=7, **kw)
        ref = O.apply_right(A, op)
        dA = device.DeviceMatrix(m, n, ld=m)          # odd ld: unaligned columns
        dA.upload(A)
        out = device.DeviceMatrix.zeros(m, d + 10, ld=m + 3)
        sk.apply_right_device(dA, op, out=out, col0=5)
        got = out.to_host()
        _close(got[:, 5:5 + d], ref, np.linalg.norm(A))
        assert np.all(got[:, :5] == 0) and np.all(got[:, 5 + d:] == 0)
        B = rng.standard_normal((n, m))
        dB = device.DeviceMatrix(n, m, ld=n + 2)  # odd: unaligned columns (cp.async producers)
        dB.upload(B)
        ref_t = O.apply_right_transposed(B, op)
        _close(sk.apply_right_transposed_device(dB, op).to_host(), ref_t, np.linalg.norm(B))


def test_results_are_deterministic(cuda):
    rng = np.random.default_rng(9)
    A = rng.standard_normal((1000, 2000))
    for kind, kw in ((sk.SJLT, dict(alpha=8, construction=sk.BLOCK)), (sk.GAUSSIAN, {}),
                     (sk.SRHT, {})):
        op = sk.new_operator(kind, 2000, 256, seed=1, **kw)
        acc = sk.DenseAccessor(A)
        s1 = sk.apply_right(acc, op)
        s2 = sk.apply_right(acc, op)
        np.testing.assert_array_equal(s1, s2)
        t1 = sk.apply_right_transposed(acc, sk.new_operator(kind, 1000, 128, seed=2, **kw))
        t2 = sk.apply_right_transposed(acc, sk.new_operator(kind, 1000, 128, seed=2, **kw))
        np.testing.assert_array_equal(t1, t2)


def test_symmetric_sides_and_zero_matrix(cuda):
    rng = np.random.default_rng(6)
    Bm = rng.standard_normal((300, 300))
    A = Bm + Bm.T
    op = sk.new_operator(sk.SJLT, 300, 40, seed=3, alpha=2, construction=sk.GRAPH)
    np.testing.assert_allclose(sk.apply_right(A, op), sk.apply_right_transposed(A, op), atol=1e-12)
    for kind, kw in ((sk.SRHT, {}), (sk.SJLT, dict(alpha=3)), (sk.GAUSSIAN, {})):
        op = sk.new_operator(kind, 12, 4, seed=0, **kw) if kind != sk.SJLT else \
            sk.new_operator(kind, 12, 6, seed=0, **kw)
        np.testing.assert_array_equal(sk.apply_right(np.zeros((5, 12)), op), 0.0)


def test_accessor_equivalence_and_device_cache(cuda):
    rng = np.random.default_rng(7)
    A = rng.standard_normal((60, 180))
    op = sk.new_operator(sk.GAUSSIAN, 180, 16, seed=8)
    acc = sk.DenseAccessor(A)
    np.testing.assert_array_equal(sk.apply_right(acc, op), sk.apply_right(A, op))
    d1 = sk.device_matrix_of(acc)
    d2 = sk.device_matrix_of(acc)
    assert d1 is d2  # uploaded once (dense() contract)


def test_gaussian_vs_oracle(cuda):
    rng = np.random.default_rng(12)
    for m, n, d in ((1, 7, 1), (130, 257, 129), (300, 2048, 512), (513, 1000, 64)):
        A = rng.standard_normal((m, n))
        op = sk.new_operator(sk.GAUSSIAN, n, d, seed=m)
        _close(sk.apply_right(A, op), O.apply_right(A, op), np.linalg.norm(A))
        B = rng.standard_normal((n, m))
        _close(sk.apply_right_transposed(B, op), O.apply_right_transposed(B, op),
               np.linalg.norm(B))


def test_srht_vs_oracle(cuda):
    rng = np.random.default_rng(13)
    for m, n, d in ((3, 1, 1), (40, 100, 24), (33, 256, 64), (65, 1000, 100), (64, 4096, 512),
                    (17, 5000, 300), (32, 70000, 64)):
        A = rng.standard_normal((m, n))
        op = sk.new_operator(sk.SRHT, n, d, seed=n)
        _close(sk.apply_right(A, op), O.apply_right(A, op), np.linalg.norm(A))
        if n <= 5000:
            B = rng.standard_normal((n, m))
            _close(sk.apply_right_transposed(B, op), O.apply_right_transposed(B, op),
                   np.linalg.norm(B))


def test_srht_duplicate_samples(cuda):
    op = sk.new_operator(sk.SRHT, 64, 60, seed=4)
    sample = op.blocks[0].sample
    assert len(np.unique(sample)) < len(sample)  # drawn with replacement
    A = np.random.default_rng(1).standard_normal((10, 64))
    S = sk.apply_right(A, op)
    for t in range(60):
        for u in range(60):
            if sample[t] == sample[u]:
                np.testing.assert_array_equal(S[:, t], S[:, u])


def test_fwht_gpu_known_answers(golden, cuda):
    arrays, _ = golden
    np.testing.assert_allclose(sk.fwht([1.0, 1.0, 1.0, 1.0]), arrays["fwht/const4"], atol=0)
    X = np.random.default_rng(1).standard_normal((3, 16))
    np.testing.assert_allclose(sk.fwht(X), arrays["fwht/rows16"], atol=1e-14)
    H = sk.fwht(np.eye(64))
    np.testing.assert_allclose(H.T @ H, np.eye(64), atol=1e-12)
    with pytest.raises(ValueError):
        sk.fwht(np.ones(6))


@pytest.mark.parametrize("keep_t,sym", [(True, False), (False, False), (True, True), (None, False)])
def test_adaptive_append_matches_one_shot(cuda, keep_t, sym):
    """Appended increments match the one-shot products; with keep_t True the
    sketch keeps A^T from the fifth extension on and runs S' as A^T R^T, or,
    for a symmetric A, copies S' from S (None: only for an A of at least
    DeviceSketch.MIN_BYTES -- not this one)."""
    rng = np.random.default_rng(21)
    n = 1500
    A = rng.standard_normal((n, n))
    if sym:
        A = A + A.T
    for kind, kw in ((sk.SJLT, dict(alpha=8, construction=sk.BLOCK)), (sk.GAUSSIAN, {}),
                     (sk.SRHT, {})):
        op = sk.new_operator(kind, n, 128, seed=(0, 0), **kw)
        ds = adaptive.DeviceSketch(sk.DenseAccessor(A), 128 + 6 * 64, keep_transpose=keep_t).start(op)
        for r in range(1, 7):      # the shortcut starts at the fifth extension
            op = sk.append_columns(op, 64, seed=(0, r))
            ds.extend(op)
        assert ds.d == op.d
        assert (ds.At is not None) == (keep_t is True and not sym)
        assert ds.sym == (keep_t is True and sym)
        _close(ds.right(), O.apply_right(A, op), np.linalg.norm(A))
        _close(ds.transposed(), O.apply_right_transposed(A, op), np.linalg.norm(A))
        # the one-shot API gives the identical bytes (same kernels, same order)
        np.testing.assert_array_equal(ds.right(), sk.apply_right(A, op))


@pytest.mark.parametrize("rows,cols,ld", [(1, 1, 2), (33, 70, 34), (257, 100, 258), (1000, 3001, 1000)])
def test_device_transpose_exact(cuda, rows, cols, ld):
    rng = np.random.default_rng(rows + cols)
    B = rng.standard_normal((rows, cols))
    dm = device.DeviceMatrix.from_host(B, ld=ld)
    t = dm.transposed()
    assert t.shape == (cols, rows)
    np.testing.assert_array_equal(t.to_host(), B.T)


@pytest.mark.parametrize("n,ld", [(1, 2), (64, 64), (65, 66), (200, 201), (1000, 1000)])
def test_device_symmetry_check(cuda, n, ld):
    rng = np.random.default_rng(n)
    B = rng.standard_normal((n, n))
    S = B + B.T
    assert device.DeviceMatrix.from_host(S, ld=ld).is_symmetric()
    if n > 1:
        S2 = S.copy()
        S2[n - 1, 0] = np.nextafter(S2[n - 1, 0], np.inf)   # one ulp off the mirror
        assert not device.DeviceMatrix.from_host(S2, ld=ld).is_symmetric()
        assert not device.DeviceMatrix.from_host(B, ld=ld).is_symmetric()


def test_streamed_pinned_host_path_is_bit_identical(cuda, monkeypatch):
    """Pinned host matrices are streamed in slabs (H2D / kernels / D2H
    overlapped); rows of S and S' depend only on their own rows / columns of
    A, so the result must equal the one-shot device path bit for bit."""
    import torch
    monkeypatch.setattr(sk, "STREAM_MIN_BYTES", 1)
    rng = np.random.default_rng(21)
    m, n = 1111, 1500                          # odd sizes: ragged last slab
    pin = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
    pin.copy_(torch.from_numpy(rng.standard_normal((n, m))))
    A = pin.numpy().T                          # F-ordered m x n view of pinned memory
    pinT = torch.empty((m, n), dtype=torch.float64, pin_memory=True)
    pinT.copy_(torch.from_numpy(np.ascontiguousarray(A)))
    B = pinT.numpy().T                         # F-ordered n x m (for S' over n rows)
    assert sk._pinned_host_buffer(A) is not None and sk._pinned_host_buffer(B) is not None
    for kind, kw in ((sk.SJLT, dict(alpha=4, construction=sk.BLOCK)), (sk.GAUSSIAN, {}),
                     (sk.SRHT, {})):
        op = sk.new_operator(kind, n, 96, seed=5, **kw)
        ref = sk.apply_right_device(device.DeviceMatrix.from_host(A), op).to_host()
        np.testing.assert_array_equal(sk.apply_right(A, op), ref)
        ref_t = sk.apply_right_transposed_device(device.DeviceMatrix.from_host(B), op).to_host()
        np.testing.assert_array_equal(sk.apply_right_transposed(B, op), ref_t)


def test_streamed_pageable_host_path_is_bit_identical(cuda, monkeypatch):
    """Plain (pageable) numpy arrays -- what the reference's callers pass --
    are staged slab by slab through pinned buffers by host threads; same
    bytes as the one-shot device path, ragged last slab included."""
    monkeypatch.setattr(sk, "STREAM_MIN_BYTES", 1)
    rng = np.random.default_rng(22)
    m, n = 1111, 1500
    A = np.asfortranarray(rng.standard_normal((m, n)))
    B = np.asfortranarray(rng.standard_normal((n, m)))
    assert sk._pinned_host_buffer(A) is None and sk._pageable_host_buffer(A) is not None
    for kind, kw in ((sk.SJLT, dict(alpha=4, construction=sk.BLOCK)), (sk.GAUSSIAN, {}),
                     (sk.SRHT, {})):
        op = sk.new_operator(kind, n, 96, seed=6, **kw)
        ref = sk.apply_right_device(device.DeviceMatrix.from_host(A), op).to_host()
        np.testing.assert_array_equal(sk.apply_right(A, op), ref)
        ref_t = sk.apply_right_transposed_device(device.DeviceMatrix.from_host(B), op).to_host()
        np.testing.assert_array_equal(sk.apply_right_transposed(B, op), ref_t)


@pytest.mark.parametrize("m,n,d,alpha", [
    (64, 64, 64, 8), (100, 1000, 64, 8), (3000, 9000, 64, 8), (257, 4100, 128, 16),
    (70, 20000, 64, 8), (1, 300, 64, 8),
    # TK < 128: the quarter fold's 64 KB must still fit one ring slot
    (130, 3000, 1024, 128), (70, 9000, 704, 88),
])
def test_sjlt_paired_plan_vs_oracle(cuda, tune, m, n, d, alpha):
    """Chunked (block-construction) patterns with d/alpha = 8 take the paired
    plan (one tile read feeds a warp's two chunks, k-groups folded per row
    tile): oracle parity on every schedule, odd leading dimensions (cp.async
    producers) and column offsets; bitwise repeatable; the unpaired plan of the
    same operator (HSK_SJLT_NOCHUNK=1) agrees to the same tolerance."""
    rng = np.random.default_rng(m + n + d)
    A = rng.standard_normal((m, n))
    B = rng.standard_normal((n, m))
    res = {}
    for nochunk in ("0", "1"):
        tune("HSK_SJLT_NOCHUNK", nochunk)
        op = sk.new_operator(sk.SJLT, n, d, seed=(m, n, d), alpha=alpha, construction=sk.BLOCK)
        b = op.blocks[0]
        ref = O.sjlt_right(A, b._pos, b._signs, d, b._scale)
        ref_t = O.sjlt_right_t(B, b._pos, b._signs, d, b._scale)
        assert device.block_state(b).flags == (0 if nochunk == "1" else device.HSK_SJLT_CHUNKED)
        for sched in ("0", "1"):
            tune("HSK_SJLT_STREAMK", sched)
            for ld_pad in (0, 1):
                dA = device.DeviceMatrix(m, n, ld=m + ld_pad)
                dA.upload(A)
                out = device.DeviceMatrix.zeros(m, d + 3)
                sk.apply_right_device(dA, op, out=out, col0=2)
                s1 = out.to_host()
                _close(s1[:, 2:2 + d], ref, np.linalg.norm(A))
                assert np.all(s1[:, :2] == 0) and np.all(s1[:, 2 + d:] == 0)
                sk.apply_right_device(dA, op, out=out, col0=2)
                np.testing.assert_array_equal(out.to_host(), s1)
                dB = device.DeviceMatrix(n, m, ld=n + ld_pad)
                dB.upload(B)
                t1 = sk.apply_right_transposed_device(dB, op).to_host()
                _close(t1, ref_t, np.linalg.norm(B))
                np.testing.assert_array_equal(sk.apply_right_transposed_device(dB, op).to_host(), t1)
                res[(nochunk, sched, ld_pad)] = (s1[:, 2:2 + d], t1)
    a, b = res[("0", "0", 0)], res[("1", "0", 0)]
    assert O.rel_frobenius(a[0], b[0]) <= REL and O.rel_frobenius(a[1], b[1]) <= REL


def test_sjlt_chunk_property_detection(cuda):
    """Only patterns with entry t in chunk t take the paired plan: graph
    construction at the same shape, and a from_pattern block that breaks the
    property, stay on the general plan (and still match the oracle)."""
    n, d, alpha = 500, 64, 8
    g = sk.new_operator(sk.SJLT, n, d, seed=3, alpha=alpha, construction=sk.GRAPH).blocks[0]
    blk = sk.new_operator(sk.SJLT, n, d, seed=3, alpha=alpha, construction=sk.BLOCK).blocks[0]
    pos = np.array(blk._pos)
    pos[7, [0, 1]] = pos[7, [1, 0]]  # entries 0 and 1 of k = 7 swap chunks
    bad = sk.SjltBlock.from_pattern(n, d, alpha, pos, blk._signs)
    good = sk.SjltBlock.from_pattern(n, d, alpha, blk._pos, blk._signs)
    assert device.block_state(good).flags == device.HSK_SJLT_CHUNKED
    A = np.random.default_rng(1).standard_normal((90, n))
    for b in (g, bad):
        assert device.block_state(b).flags == 0
    # the C ABI refuses HSK_SJLT_CHUNKED for a pattern without the property
    import torch
    from paper_2302_01977_b200 import _lib
    st = device.block_state(bad)
    nb = _lib.load().hsk_sjlt_plan_bytes_ex(n, d, alpha, device.HSK_SJLT_CHUNKED)
    plan = torch.empty(int(nb), dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError, match="chunk"):
        _lib.call("hsk_sjlt_plan_build_ex", st.pos.data_ptr(), st.sgn.data_ptr(), n, d, alpha,
                  device.HSK_SJLT_CHUNKED, plan.data_ptr(), int(nb), device.current_stream_ptr())
    for b in (g, bad, good):
        op = sk.SketchOperator(sk.SJLT, n, (b,), alpha=alpha)
        ref = O.sjlt_right(A, b._pos, b._signs, d, b._scale)
        _close(sk.apply_right(A, op), ref, np.linalg.norm(A))
        ref_t = O.sjlt_right_t(np.asfortranarray(A.T), b._pos, b._signs, d, b._scale)
        _close(sk.apply_right_transposed(np.asfortranarray(A.T), op), ref_t, np.linalg.norm(A))
