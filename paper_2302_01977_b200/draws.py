"""Random operator draws, bit-identical to the reference's.

The GPU engine never regenerates R: an operator block is drawn on the host
with numpy's PCG64 Generator, consuming the stream in exactly the order the
reference does, and the resulting integers/doubles are uploaded once.  Each
function names the reference code it restates (hsskit sketching.py) and is
pinned against reference-generated fixtures (tests/test_operator_draws.py).

Stream order per block (a fresh `default_rng(seed)` per block):
  gaussian  standard_normal((rows, n)) / sqrt(rows)          sketching.py:131-132
  srht      integers(0,2,n_pad)*2-1, then integers(0,n_pad,rows)  :157-159
  sjlt      positions (block or graph), then integers(0,2,(n,alpha))*2-1  :246-253
"""

from __future__ import annotations

import math

import numpy as np


def next_pow2(n: int) -> int:
    """Smallest power of two >= n (1 for n <= 1); sketching.py:115-116."""
    if n <= 1:
        return 1
    return 1 << (int(n) - 1).bit_length()


def gaussian_matrix(n: int, rows: int, seed) -> np.ndarray:
    """rows x n i.i.d. N(0, 1/rows) (per-block variance)."""
    gen = np.random.default_rng(seed)
    return gen.standard_normal((rows, n)) / math.sqrt(rows)


def srht_draw(n: int, rows: int, seed) -> tuple[np.ndarray, np.ndarray, int]:
    """(signs of length n_pad as float64 +-1, sample of `rows` indices drawn
    WITH replacement from [0, n_pad), n_pad)."""
    n_pad = next_pow2(n)
    gen = np.random.default_rng(seed)
    signs = 2.0 * gen.integers(0, 2, size=n_pad) - 1.0
    sample = gen.integers(0, n_pad, size=rows)
    return signs, sample, n_pad


def _sjlt_block_positions(gen, n: int, rows: int, alpha: int) -> np.ndarray:
    # one offset inside each of the alpha chunks of length rows // alpha
    width = rows // alpha
    base = np.arange(alpha) * width
    return base + gen.integers(0, width, size=(n, alpha))


def _sjlt_graph_positions(gen, n: int, rows: int, alpha: int) -> np.ndarray:
    # Floyd's algorithm run column-parallel: for step j = rows-alpha..rows-1
    # draw c in [0, j]; keep c unless already used in that column, else j.
    used = np.zeros((n, rows), dtype=bool)
    out = np.empty((n, alpha), dtype=np.intp)
    every = np.arange(n)
    for t in range(alpha):
        j = rows - alpha + t
        cand = gen.integers(0, j + 1, size=n)
        pick = np.where(used[every, cand], j, cand)
        used[every, pick] = True
        out[:, t] = pick
    return out


def sjlt_draw(n: int, rows: int, seed, alpha: int,
              construction: str) -> tuple[np.ndarray, np.ndarray]:
    """(pos n x alpha intp in [0, rows), signs n x alpha int8 +-1)."""
    gen = np.random.default_rng(seed)
    if construction == "block":
        pos = _sjlt_block_positions(gen, n, rows, alpha)
    else:
        pos = _sjlt_graph_positions(gen, n, rows, alpha)
    signs = 2 * gen.integers(0, 2, size=(n, alpha)) - 1
    return np.asarray(pos, dtype=np.intp), np.asarray(signs, dtype=np.int8)
