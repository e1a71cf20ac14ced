"""Sketch operators: immutable stacks of independently drawn blocks.

Host-side mirror of the reference's operator model (hsskit sketching.py:
blocks :123-360, SketchOperator :367-387, construction/append :390-428,
dense_rows :460-476; jl_dimension_bound :479-499 is a sizing helper
outside the sketch path and is not restated).  A block carries only
its random draw (draws.py) plus the metadata the GPU engine needs; block
products (`apply_right`, `apply_right_transposed`) launch libhsk.so kernels
through device.py -- there is no host implementation of them here.

Block attribute names follow the reference (`_pos`, `_signs`, `_scale`,
`matrix`, `signs`, `sample`, `scale`, `n_pad`), so the engine accepts the
reference's own block objects unchanged (plugin.py) and ours interchangeably.
"""

from __future__ import annotations

import math

import numpy as np

from . import draws

GAUSSIAN, SRHT, SJLT = "gaussian", "srht", "sjlt"
KINDS = (GAUSSIAN, SRHT, SJLT)
BLOCK, GRAPH = "block", "graph"
CONSTRUCTIONS = (BLOCK, GRAPH)


def _gpu_block_product(block, buf, transpose: bool) -> np.ndarray:
    from . import device
    dA = device.DeviceMatrix.from_host(buf)
    out_rows = dA.cols if transpose else dA.rows
    out = device.DeviceMatrix.empty(out_rows, block.rows)
    device.apply_block(block, dA, transpose, out, 0)
    return out.to_host()


class _Block:
    """Common block protocol: kind, n, rows, two GPU products, dense_rows."""

    kind = ""

    def apply_right(self, buf: np.ndarray) -> np.ndarray:
        """buf @ R_b^T on the GPU (buf is rows_A x n)."""
        return _gpu_block_product(self, buf, False)

    def apply_right_transposed(self, buf: np.ndarray) -> np.ndarray:
        """buf^T @ R_b^T on the GPU (buf is n x cols_A)."""
        return _gpu_block_product(self, buf, True)

    def dense_rows(self, I: np.ndarray, cols: np.ndarray) -> np.ndarray:
        raise NotImplementedError


class GaussianBlock(_Block):
    """Dense block with i.i.d. N(0, 1/rows) entries (`matrix` is rows x n)."""

    kind = GAUSSIAN

    def __init__(self, n: int, rows: int, seed):
        self.n, self.rows = n, rows
        self.matrix = draws.gaussian_matrix(n, rows, seed)

    def dense_rows(self, I, cols):
        return self.matrix[np.ix_(cols, I)].T


class SrhtBlock(_Block):
    """R = sqrt(n_pad/rows) P H D on the zero-padded space; the Hadamard
    normalisation and sampling factor fold into `scale` = 1/sqrt(rows)."""

    kind = SRHT

    def __init__(self, n: int, rows: int, seed):
        self.n, self.rows = n, rows
        self.signs, self.sample, self.n_pad = draws.srht_draw(n, rows, seed)
        self.scale = 1.0 / math.sqrt(rows)

    def dense_rows(self, I, cols):
        # H[i, s] = (-1)^popcount(i & s) (unnormalised Walsh-Hadamard)
        s = self.sample[cols].astype(np.int64)
        bits = np.bitwise_count(np.bitwise_and.outer(I.astype(np.int64), s)) & 1
        return (self.signs[I, None] * (1.0 - 2.0 * bits)) * self.scale


class SjltStorage:
    """Index-only CSR/CSC views of the B+ and B- patterns (§6.1).

    Kept for API parity; the GPU consumes a re-blocked plan built on device
    from `_pos`/`_signs` (hsk_sjlt_plan_build)."""

    __slots__ = ("scale", "plus_rowptr", "plus_cols", "minus_rowptr", "minus_cols",
                 "plus_colptr", "plus_rows", "minus_colptr", "minus_rows")

    def __init__(self, scale, *views):
        self.scale = scale
        (self.plus_rowptr, self.plus_cols, self.minus_rowptr, self.minus_cols,
         self.plus_colptr, self.plus_rows, self.minus_colptr, self.minus_rows) = views


def _csr_csc(k_idx: np.ndarray, j_idx: np.ndarray, n: int, d: int):
    """CSR (over k) and CSC (over j, stable in k) of coordinates listed in
    row-major order."""
    rowptr = np.concatenate(([0], np.cumsum(np.bincount(k_idx, minlength=n)))).astype(np.intp)
    colptr = np.concatenate(([0], np.cumsum(np.bincount(j_idx, minlength=d)))).astype(np.intp)
    by_col = k_idx[np.argsort(j_idx, kind="stable")]
    return rowptr, np.asarray(j_idx, dtype=np.intp), colptr, by_col


class SjltBlock(_Block):
    """alpha nonzeros +-1/sqrt(alpha) per column of R, placed by the block
    (one per chunk of rows/alpha) or graph (distinct, Floyd) construction."""

    kind = SJLT

    def __init__(self, n: int, rows: int, seed, alpha: int, construction: str,
                 _pattern=None):
        self.n, self.rows, self.alpha, self.construction = n, rows, alpha, construction
        if _pattern is None:
            pos, sg = draws.sjlt_draw(n, rows, seed, alpha, construction)
        else:
            pos, sg = _pattern
        self._pos = np.asarray(pos, dtype=np.intp)
        self._signs = np.asarray(sg, dtype=np.int8)
        self._scale = 1.0 / math.sqrt(alpha)
        self._storage = None

    @classmethod
    def from_pattern(cls, n: int, rows: int, alpha: int, pos, signs) -> "SjltBlock":
        """Block from an explicit (pos, signs) pattern (testing hook)."""
        return cls(n, rows, seed=0, alpha=alpha, construction=GRAPH,
                   _pattern=(np.asarray(pos, dtype=np.intp), np.asarray(signs)))

    @property
    def storage(self) -> SjltStorage:
        if self._storage is None:
            ks = np.repeat(np.arange(self.n, dtype=np.intp), self.alpha)
            js = self._pos.ravel()
            plus = self._signs.ravel() > 0
            p = _csr_csc(ks[plus], js[plus], self.n, self.rows)
            m = _csr_csc(ks[~plus], js[~plus], self.n, self.rows)
            self._storage = SjltStorage(self._scale, p[0], p[1], m[0], m[1],
                                        p[2], p[3], m[2], m[3])
        return self._storage

    def dense_rows(self, I, cols):
        block = np.zeros((len(I), self.rows))
        block[np.arange(len(I))[:, None], self._pos[I]] = self._signs[I] * self._scale
        whole = cols.size == self.rows and np.array_equal(cols, np.arange(self.rows))
        return block if whole else block[:, cols]


class SketchOperator:
    """Ordered, immutable tuple of blocks; logical shape d x n."""

    def __init__(self, kind: str, n: int, blocks: tuple, alpha=None, construction=None):
        self.kind, self.n = kind, n
        self.blocks = tuple(blocks)
        self.alpha, self.construction = alpha, construction

    @property
    def d(self) -> int:
        return int(sum(b.rows for b in self.blocks))

    def block_offsets(self) -> list[int]:
        acc = [0]
        for b in self.blocks:
            acc.append(acc[-1] + b.rows)
        return acc


def _draw_block(kind, n, rows, seed, alpha, construction):
    if kind == GAUSSIAN:
        return GaussianBlock(n, rows, seed)
    if kind == SRHT:
        return SrhtBlock(n, rows, seed)
    if alpha is None or not 1 <= alpha <= rows:
        raise ValueError(f"SJLT needs 1 <= alpha <= block rows (alpha={alpha}, rows={rows})")
    if construction not in CONSTRUCTIONS:
        raise ValueError(f"unknown SJLT construction {construction!r}")
    if construction == BLOCK and rows % alpha:
        raise ValueError(f"block construction needs alpha | d (alpha={alpha}, d={rows})")
    return SjltBlock(n, rows, seed, alpha, construction)


def new_operator(kind: str, n: int, d: int, seed, *, alpha: int | None = None,
                 construction: str = BLOCK) -> SketchOperator:
    """One freshly drawn block of d rows (validation as sketching.py:407-418)."""
    if kind not in KINDS:
        raise ValueError(f"unknown operator kind {kind!r}")
    if not 1 <= d <= n:
        raise ValueError(f"need 1 <= d <= n (d={d}, n={n})")
    blk = _draw_block(kind, n, d, seed, alpha, construction)
    if kind == SJLT:
        return SketchOperator(kind, n, (blk,), alpha, construction)
    return SketchOperator(kind, n, (blk,))


def append_columns(op: SketchOperator, dd: int, seed) -> SketchOperator:
    """New operator sharing op's blocks plus one fresh block of dd rows."""
    if dd < 1:
        raise ValueError("dd must be >= 1")
    blk = _draw_block(op.kind, op.n, dd, seed, op.alpha, op.construction)
    return SketchOperator(op.kind, op.n, op.blocks + (blk,), op.alpha, op.construction)


def dense_rows(op: SketchOperator, I, col_range) -> np.ndarray:
    """R^T restricted to rows I and sketch columns col_range (host)."""
    I = np.asarray(I, dtype=np.intp)
    cols = np.asarray(col_range, dtype=np.intp)
    if I.size and not (0 <= I.min() and I.max() < op.n):
        raise IndexError("row indices out of range")
    if cols.size and not (0 <= cols.min() and cols.max() < op.d):
        raise IndexError("column indices out of range")
    if len(op.blocks) == 1:
        return op.blocks[0].dense_rows(I, cols)
    out = np.empty((len(I), len(cols)))
    bounds = op.block_offsets()
    for blk, lo, hi in zip(op.blocks, bounds[:-1], bounds[1:]):
        sel = (cols >= lo) & (cols < hi)
        if sel.any():
            out[:, sel] = blk.dense_rows(I, cols[sel] - lo)
    return out

