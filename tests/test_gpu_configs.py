"""GPU parity at BASELINE.json config sizes.

A is generated in HBM (matgen) and the oracle sees the SAME bytes, copied
back in full (C1, C2) or as row/column slabs (C3-C5): rows of S depend only
on rows of A and rows of S' only on columns of A, so slab oracles are exact
restrictions of the full product (tests/test_oracle.py pins this).
Tolerance: relative Frobenius <= 1e-12 (BASELINE.json north_star).
"""

import gc

import numpy as np
import pytest

from oracle import oracle as O
from paper_2302_01977_b200 import adaptive, device, matgen
from paper_2302_01977_b200 import sketching as sk

pytestmark = pytest.mark.gpu
REL = 1e-12


def _free():
    import torch
    gc.collect()
    torch.cuda.empty_cache()


def _rows(dm, r0, r1):
    return np.asfortranarray(dm.row_view(r0, r1 - r0).to_host())


def _cols(dm, c0, c1):
    return np.asfortranarray(dm.to_host(c0, c1 - c0))


def test_c1_full_size(cuda):
    n = 4096
    A = matgen.gaussian_kernel(n, 8, 0.5)
    Ah = A.to_host()
    op = sk.new_operator(sk.SJLT, n, 256, np.random.SeedSequence((0, 0)), alpha=4,
                         construction=sk.GRAPH)
    S = sk.apply_right_device(A, op).to_host()
    St = sk.apply_right_transposed_device(A, op).to_host()
    assert O.rel_frobenius(S, O.apply_right(Ah, op)) <= REL
    assert O.rel_frobenius(St, O.apply_right_transposed(Ah, op)) <= REL
    for kind in (sk.GAUSSIAN, sk.SRHT):
        op2 = sk.new_operator(kind, n, 256, np.random.SeedSequence((0, 0)))
        S2 = sk.apply_right_device(A, op2).to_host()
        rows = slice(0, 512)
        assert O.rel_frobenius(S2[rows], O.apply_right(Ah[rows], op2)) <= REL
    del A
    _free()


def test_c2_full_size(cuda):
    n = 16384
    A = matgen.gaussian_kernel(n, 8, 0.5)
    op = sk.new_operator(sk.SJLT, n, 512, np.random.SeedSequence((0, 0)), alpha=4,
                         construction=sk.BLOCK)
    S = sk.apply_right_device(A, op).to_host()
    Ah = A.to_host()
    assert O.rel_frobenius(S, O.apply_right(Ah, op)) <= REL
    St = sk.apply_right_transposed_device(A, op)
    cols = (5000, 5600)
    assert O.rel_frobenius(St.to_host()[cols[0]:cols[1]],
                           O.apply_right_transposed(np.asfortranarray(Ah[:, cols[0]:cols[1]]), op)) <= REL
    gop = sk.new_operator(sk.GAUSSIAN, n, 512, np.random.SeedSequence((0, 0)))
    G = sk.apply_right_device(A, gop).to_host()
    rows = slice(777, 777 + 384)
    assert O.rel_frobenius(G[rows], O.apply_right(np.asfortranarray(Ah[rows]), gop)) <= REL
    # Gaussian S' = A^T R^T: rows of S' are columns of A
    Gt = sk.apply_right_transposed_device(A, gop).to_host()
    cols = (9000, 9000 + 384)
    assert O.rel_frobenius(Gt[cols[0]:cols[1]],
                           O.apply_right_transposed(np.asfortranarray(Ah[:, cols[0]:cols[1]]), gop)) <= REL
    del A, Ah
    _free()


def test_c3_adaptive_full_size(cuda):
    n = 65536
    A = matgen.toeplitz_sin(n)
    op = sk.new_operator(sk.SJLT, n, 64, np.random.SeedSequence((0, 0)), alpha=8,
                         construction=sk.BLOCK)
    ds = adaptive.DeviceSketch(A, 1024).start(op)
    for r in range(1, 16):
        op = sk.append_columns(op, 64, np.random.SeedSequence((0, r)))
        ds.extend(op)
    assert ds.d == 1024
    r0, r1 = 40000, 40192
    S_rows = ds.S.row_view(r0, r1 - r0).to_host()[:, :1024]
    assert O.rel_frobenius(S_rows, O.apply_right(_rows(A, r0, r1), op)) <= REL
    c0, c1 = 1234, 1426
    St_rows = ds.St.row_view(c0, c1 - c0).to_host()[:, :1024]
    assert O.rel_frobenius(St_rows, O.apply_right_transposed(_cols(A, c0, c1), op)) <= REL
    # appending block by block gives the same bytes as one launch per block
    one = sk.apply_right_device(A, op)
    np.testing.assert_array_equal(one.row_view(r0, r1 - r0).to_host(), S_rows)
    del A, ds, one
    _free()


def test_c4_srht_full_size(cuda):
    n = 65536
    A = matgen.gaussian_kernel(n, 8, 0.25)
    op = sk.new_operator(sk.SRHT, n, 512, np.random.SeedSequence((0, 0)))
    S = sk.apply_right_device(A, op)
    for r0 in (0, 33000):
        r1 = r0 + 64
        got = S.row_view(r0, 64).to_host()
        assert O.rel_frobenius(got, O.apply_right(_rows(A, r0, r1), op)) <= REL
    # S' = A^T R^T (columns of A transformed; TMA staging + in-smem transpose):
    # column slabs of A against the oracle
    St = sk.apply_right_transposed_device(A, op)
    for c0 in (0, 40000):
        c1 = c0 + 48
        got = St.row_view(c0, c1 - c0).to_host()
        assert O.rel_frobenius(got, O.apply_right_transposed(_cols(A, c0, c1), op)) <= REL
    del A, S, St
    _free()


@pytest.mark.slow
def test_c5_single_gpu_full_size(cuda):
    n = 131072
    A = matgen.gaussian_kernel(n, 16, 1.0)   # 137 GB in HBM
    op = sk.new_operator(sk.SJLT, n, 2048, np.random.SeedSequence((0, 0)), alpha=8,
                         construction=sk.BLOCK)
    S = sk.apply_right_device(A, op)
    r0 = 70000
    assert O.rel_frobenius(S.row_view(r0, 64).to_host(), O.apply_right(_rows(A, r0, r0 + 64), op)) <= REL
    del S
    _free()
    # S' = A^T R^T: a column slab of A against the oracle (rows of S')
    St = sk.apply_right_transposed_device(A, op)
    c0 = 100000
    assert O.rel_frobenius(St.row_view(c0, 64).to_host(),
                           O.apply_right_transposed(_cols(A, c0, c0 + 64), op)) <= REL
    del St
    _free()
    gop = sk.new_operator(sk.GAUSSIAN, n, 512, np.random.SeedSequence((0, 0)))
    G = sk.apply_right_device(A, gop)
    assert O.rel_frobenius(G.row_view(r0, 32).to_host(), O.apply_right(_rows(A, r0, r0 + 32), gop)) <= REL
    del G
    _free()
    Gt = sk.apply_right_transposed_device(A, gop)
    assert O.rel_frobenius(Gt.row_view(c0, 32).to_host(),
                           O.apply_right_transposed(_cols(A, c0, c0 + 32), gop)) <= REL
    del A, Gt
    _free()
