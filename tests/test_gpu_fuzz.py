"""GPU parity over a seeded random sweep of operator shapes.

The fixed shape lists of test_gpu_sketch.py pin the cases the reference tests
name; this module walks the geometry rules of the kernels instead (slab and
warp-shape boundaries in d, the wide path at n >= 8192, chunk sizes TK * alpha
near the 12-bit local index, paired plans, multi-block operators with column
offsets, odd row counts) with shapes drawn from a fixed seed, every product
checked against the CPU oracle (oracle/hsk_oracle.c: the reference's
summation order, sketching.py:322-351 / :86-191 / :123-141) at the north-star
tolerance, 1e-12 relative Frobenius.
"""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2302_01977_b200 import sketching as sk

pytestmark = pytest.mark.gpu

REL = 1e-12

# d values either side of every slab / warp-shape switch of hsk_sjlt.cu
# (warp_shape, geom_dir): 64 | 128 | 256 | 260 | 264 | 384 | 512 | 520 | 640
_D_EDGES = (1, 2, 7, 63, 64, 65, 127, 128, 129, 255, 256, 257, 260, 261, 264, 265, 320, 383, 384,
            385, 511, 512, 513, 520, 521, 528, 639, 640, 641, 704, 1024, 1040, 2048, 2049)
# n values either side of the long-row rule (n >= 8192) and of chunk multiples
_N_EDGES = (1, 2, 15, 16, 17, 127, 128, 129, 207, 208, 209, 255, 256, 257, 415, 416, 417, 1000,
            4095, 4096, 4097, 8191, 8192, 8193, 8320, 9000)


def _draw_sjlt(rng):
    n = int(rng.choice(_N_EDGES)) if rng.random() < 0.7 else int(rng.integers(1, 9000))
    d = int(rng.choice(_D_EDGES)) if rng.random() < 0.7 else int(rng.integers(1, 2100))
    d = min(d, n)
    cons = sk.BLOCK if rng.random() < 0.5 else sk.GRAPH
    if cons == sk.BLOCK:
        divs = [a for a in range(1, d + 1) if d % a == 0]
        # mostly small alpha, sometimes the d/alpha = 8 paired shapes, sometimes huge
        pick = rng.random()
        if pick < 0.25 and d % 8 == 0:
            alpha = d // 8
        elif pick < 0.85:
            small = [a for a in divs if a <= 16]
            alpha = int(rng.choice(small))
        else:
            alpha = int(rng.choice(divs))
    else:
        alpha = int(rng.integers(1, min(d, 12) + 1)) if rng.random() < 0.85 else int(rng.integers(1, d + 1))
    m = int(rng.choice((1, 2, 31, 32, 33, 63, 64, 65, 127, 128, 129, 200)))
    return m, n, d, alpha, cons


def _close(x, ref, what):
    assert x.shape == ref.shape, what
    err = O.rel_frobenius(x, ref)
    assert err <= REL, f"{what}: rel Frobenius {err:.3e}"


@pytest.mark.parametrize("chunk", range(8))
def test_sjlt_random_shapes(cuda, chunk):
    rng = np.random.default_rng((20230201977, chunk))
    for trial in range(20):
        m, n, d, alpha, cons = _draw_sjlt(rng)
        # keep the graph draw's n x d `taken` table and the oracle quick
        if cons == sk.GRAPH and n * d > 6_000_000:
            n = max(d, 6_000_000 // d)
        what = f"chunk {chunk} trial {trial}: m={m} n={n} d={d} alpha={alpha} {cons}"
        op = sk.new_operator(sk.SJLT, n, d, seed=(chunk, trial), alpha=alpha, construction=cons)
        b = op.blocks[0]
        A = rng.standard_normal((m, n))
        B = rng.standard_normal((n, m))
        _close(sk.apply_right(A, op), O.sjlt_right(A, b._pos, b._signs, d, b._scale), what + " S")
        _close(sk.apply_right_transposed(B, op), O.sjlt_right_t(B, b._pos, b._signs, d, b._scale),
               what + " S'")


def test_multiblock_random_operators(cuda):
    """Operators grown by append_columns (sketching.py:417-428): blocks of
    different kinds of geometry side by side, each writing its own column slice."""
    rng = np.random.default_rng(977)
    for trial in range(12):
        n = int(rng.choice((64, 300, 1000, 4096, 8192)))
        m = int(rng.choice((1, 33, 64, 129)))
        kind = (sk.SJLT, sk.SJLT, sk.GAUSSIAN, sk.SRHT)[trial % 4]
        kw = {}
        if kind == sk.SJLT:
            alpha = int(rng.choice((1, 2, 4, 8)))
            kw = dict(alpha=alpha, construction=sk.BLOCK if trial % 2 else sk.GRAPH)
            widths = [alpha * int(rng.integers(1, 40)) for _ in range(int(rng.integers(2, 5)))]
        else:
            widths = [int(rng.integers(1, 70)) for _ in range(int(rng.integers(2, 5)))]
        widths = [min(w, n) for w in widths]
        op = sk.new_operator(kind, n, widths[0], seed=(5, trial), **kw)
        for i, w in enumerate(widths[1:]):
            op = sk.append_columns(op, w, seed=(5, trial, i))
        A = rng.standard_normal((m, n))
        B = rng.standard_normal((n, m))
        what = f"trial {trial}: {kind} n={n} m={m} widths={widths}"
        tol = 1e-11 if kind == sk.GAUSSIAN else REL  # DMMA vs the oracle's dot order
        s, st = sk.apply_right(A, op), sk.apply_right_transposed(B, op)
        assert O.rel_frobenius(s, O.apply_right(A, op)) <= tol, what
        assert O.rel_frobenius(st, O.apply_right_transposed(B, op)) <= tol, what


def test_srht_random_shapes(cuda):
    rng = np.random.default_rng(4242)
    for trial in range(24):
        n = int(rng.choice((1, 2, 3, 21, 64, 100, 1023, 1024, 1025, 4096, 5000, 16384, 20000)))
        d = int(rng.integers(1, min(n, 600) + 1))
        m = int(rng.choice((1, 7, 32, 33, 100)))
        op = sk.new_operator(sk.SRHT, n, d, seed=(9, trial))
        A = rng.standard_normal((m, n))
        B = rng.standard_normal((n, m))
        what = f"trial {trial}: n={n} d={d} m={m}"
        _close(sk.apply_right(A, op), O.apply_right(A, op), what + " S")
        _close(sk.apply_right_transposed(B, op), O.apply_right_transposed(B, op), what + " S'")


def test_gaussian_random_shapes(cuda):
    rng = np.random.default_rng(1717)
    for trial in range(24):
        n = int(rng.choice((1, 5, 63, 64, 65, 129, 1000, 4097)))
        d = int(rng.integers(1, min(n, 300) + 1))
        m = int(rng.choice((1, 15, 64, 65, 130, 257)))
        op = sk.new_operator(sk.GAUSSIAN, n, d, seed=(11, trial))
        A = rng.standard_normal((m, n))
        B = rng.standard_normal((n, m))
        # a dense product: the reference's own bound is the dense-equivalence
        # tolerance 1e-12 * ||A||_F (test_acceptance.py:66-93), not bit parity
        for got, ref, M in ((sk.apply_right(A, op), O.apply_right(A, op), A),
                            (sk.apply_right_transposed(B, op), O.apply_right_transposed(B, op), B)):
            assert got.shape == ref.shape
            assert np.max(np.abs(got - ref), initial=0.0) <= 1e-12 * np.linalg.norm(M), \
                f"trial {trial}: n={n} d={d} m={m}"
