"""Adaptive sketching with append-in-place device buffers.

The reference grows its sketch by drawing a fresh block
(`append_columns`), sketching only that block against A, and concatenating
on the host (hss_compress.py:168-182; append-only, earlier
columns are never recomputed).  DeviceSketch keeps S = A R^T and
S' = A^T R^T in HBM with capacity d_max columns; each increment launches the
kernels once for the new block, writing straight into columns
[d, d + dd) (hsk_*_apply `col0`).  Old columns are neither re-read nor moved.

S' = A^T R^T of a TMA-landed A tile reads 8-byte column values whose
16-row groups share 8 bank pairs (2-way conflicts), while
S = A R^T reads contiguous rows conflict-free.  An adaptive run applies S' to
the same A once per increment, so in a long run (when HBM holds a second
copy) the sketch keeps A^T -- one transpose, 2 x bytes(A) of traffic
-- and runs every later S' increment as S = A^T R^T (same entries, same
per-bucket summation order over the input indices).  The copy is made at the
fifth extension (AFTER_EXTENSIONS), so short runs never pay for it.  A bitwise
symmetric A (kernel and covariance matrices) needs no copy: A^T R^T = A R^T
exactly, so from then on S' columns are the S columns just computed (one
symmetry check, hsk_is_symmetric, instead of the transpose).
"""

from __future__ import annotations

import numpy as np

from . import device as _dev
from . import sketching as _sk


class DeviceSketch:
    """S = A R^T and S' = A^T R^T in HBM, column-major with `capacity` columns.

    growable=True doubles the capacity when an increment does not fit (the
    sketched columns are copied once into the larger buffer); otherwise an
    overflow raises ValueError."""

    def __init__(self, A, n_cols_max: int, *, right: bool = True, transposed: bool = True,
                 growable: bool = False, keep_transpose: bool | None = None):
        self.A = _sk.device_matrix_of(A)
        # A^T (or the symmetry shortcut) for the S' increments: None = for an A
        # of at least MIN_BYTES that fits twice in HBM (the default), True =
        # whenever it fits, False = never
        self.keep_transpose = keep_transpose
        self.At = None
        self.sym = False      # A == A^T bitwise: S' increments are copies of S
        self._extensions = 0
        self.capacity = int(n_cols_max)
        self.growable = growable
        self.d = 0
        self.op = None
        self.S = _dev.DeviceMatrix.empty(self.A.rows, self.capacity) if right else None
        self.St = _dev.DeviceMatrix.empty(self.A.cols, self.capacity) if transposed else None

    def _grow(self, need: int):
        cap = max(need, 2 * self.capacity)
        for name in ("S", "St"):
            old = getattr(self, name)
            if old is None:
                continue
            new = _dev.DeviceMatrix.empty(old.rows, cap)
            if self.d:
                new.t[:self.d].copy_(old.t[:self.d])
            setattr(self, name, new)
        self.capacity = cap

    def _sketch_block(self, blk):
        if self.d + blk.rows > self.capacity:
            if self.growable:
                self._grow(self.d + blk.rows)
            else:
                raise ValueError(f"sketch capacity {self.capacity} exceeded "
                                 f"(d={self.d}, block rows={blk.rows})")
        if self.S is not None:
            _dev.apply_block(blk, self.A, False, self.S, self.d)
        if self.St is not None:
            if self.sym and self.S is not None:    # A^T R^T = A R^T, bit for bit
                n = self.A.rows
                self.St.t[self.d:self.d + blk.rows, :n].copy_(self.S.t[self.d:self.d + blk.rows, :n])
            elif self.At is not None:     # S' = (A^T) R^T on the kept transpose
                _dev.apply_block(blk, self.At, False, self.St, self.d)
            else:
                _dev.apply_block(blk, self.A, True, self.St, self.d)
        self.d += blk.rows

    # below this size of A the adaptive S' shortcuts are not tried (measured:
    # n = 8000, 3-18 blocks ran up to 2x slower with them; C3 at 34 GB and the
    # covariance n = 27000 runs at 5.8 GB gain)
    MIN_BYTES = 4 << 30
    # ... and only from this extension on: the copy costs ~9 increments' S'
    # savings (2 x bytes(A) at 5.7 TB/s vs ~0.3 x bytes(A) saved per S'), so a
    # rent-or-buy wait bounds the loss of short runs (Table 7.1's 4-extension
    # covariance runs at n = 27000 were 10-20 % slower with the copy at the
    # second extension) while long ones (C3: 15 extensions) still gain
    AFTER_EXTENSIONS = 5

    def _maybe_transpose(self):
        """Keep A^T for the remaining S' increments if it fits in free HBM
        (with a quarter of A as margin); a bitwise-symmetric A needs no copy.
        keep_transpose None: only for an A of at least MIN_BYTES."""
        if self.St is None or self.At is not None or self.sym or self.keep_transpose is False:
            return
        if self.keep_transpose is None and 8 * self.A.rows * self.A.cols < self.MIN_BYTES:
            return  # small A: the check, the copy and its allocation cost more than they save
        if self.S is not None and self.A.is_symmetric():
            self.sym = True
            return
        import torch
        free, _ = torch.cuda.mem_get_info()
        if free < 1.25 * 8 * self.A.rows * self.A.cols + (1 << 30):
            return
        self.At = self.A.transposed()

    def start(self, op) -> "DeviceSketch":
        """Sketch every block of a fresh operator (init_sketch)."""
        if self.S is not None and op.n != self.A.cols:
            raise ValueError("operator dimension does not match A's columns")
        if self.St is not None and op.n != self.A.rows:
            raise ValueError("operator dimension does not match A's rows")
        self.d = 0
        self.At = None   # a fresh schedule pays for its own transpose / check
        self.sym = False
        self._extensions = 0
        for blk in op.blocks:
            self._sketch_block(blk)
        self.op = op
        return self

    def extend(self, op) -> "DeviceSketch":
        """Sketch only the blocks op has beyond the current operator
        (extend_sketch after append_columns)."""
        known = 0 if self.op is None else len(self.op.blocks)
        if self.op is not None and tuple(op.blocks[:known]) != tuple(self.op.blocks):
            raise ValueError("operator is not an extension of the sketched one")
        self._extensions += len(op.blocks) > known
        if self._extensions >= self.AFTER_EXTENSIONS:  # a run long enough to repay the copy
            self._maybe_transpose()
        for blk in op.blocks[known:]:
            self._sketch_block(blk)
        self.op = op
        return self

    # bookkeeping for benchmarks: per schedule of `incs` single-block increments
    fused = False

    def products_per_schedule(self, incs: int) -> int:
        return incs * ((self.S is not None) + (self.St is not None))

    def passes_per_schedule(self, incs: int) -> int:
        """Full passes over A (HBM streams) per schedule."""
        return self.products_per_schedule(incs)

    def launches_per_schedule(self, incs: int) -> int:
        return self.products_per_schedule(incs)

    def right(self) -> np.ndarray:
        return self.S.to_host(0, self.d)

    def transposed(self) -> np.ndarray:
        return self.St.to_host(0, self.d)
