"""Public sketch API: a drop-in for hsskit.sketching with GPU products.

Every public name of the reference module
(/root/reference/pkg/src/hsskit/sketching.py) is available here with the
same argument meaning, return type and exception class:

  MatrixAccessor, DenseAccessor     matrix access      sketching.py:37-79
  fwht                              normalised FWHT    sketching.py:100-112
  GaussianBlock, SrhtBlock,
  SjltBlock, SjltStorage            operator blocks    sketching.py:123-360
  SketchOperator, new_operator,
  append_columns                    operators          sketching.py:367-428
  apply_right                       S  = A R^T         sketching.py:431-442
  apply_right_transposed            S' = A^T R^T       sketching.py:445-457
  dense_rows, jl_dimension_bound    host helpers       sketching.py:460-499

The two products (and fwht) run sm_100a kernels from libhsk.so; operator
draws are bit-identical to the reference's (draws.py).  Results are float64,
Fortran-ordered, freshly allocated and owned by the caller.

Extensions beyond the reference API (device-resident workflows):
  DeviceAccessor, device_matrix_of, apply_right_device,
  apply_right_transposed_device.
"""

from __future__ import annotations

import numpy as np

from . import device as _dev
from .operators import (BLOCK, CONSTRUCTIONS, GAUSSIAN, GRAPH, KINDS, SJLT, SRHT,
                        GaussianBlock, SjltBlock, SjltStorage, SketchOperator, SrhtBlock,
                        append_columns, dense_rows, jl_dimension_bound, new_operator)
from .draws import next_pow2 as _next_pow2

__all__ = [
    "GAUSSIAN", "SRHT", "SJLT", "KINDS", "BLOCK", "GRAPH", "CONSTRUCTIONS",
    "MatrixAccessor", "DenseAccessor", "DeviceAccessor", "fwht",
    "GaussianBlock", "SrhtBlock", "SjltBlock", "SjltStorage", "SketchOperator",
    "new_operator", "append_columns", "apply_right", "apply_right_transposed",
    "dense_rows", "jl_dimension_bound", "device_matrix_of", "apply_right_device",
    "apply_right_transposed_device",
]


class MatrixAccessor:
    """Matrix interface: `shape`, `extract(rows, cols)` and `dense()`.

    `dense()` returns a column-major float64 buffer and must hand back the
    SAME buffer on every call, which callers never mutate.  The GPU engine
    relies on this to upload A once and reuse the HBM copy (device.A_CACHE).
    """

    @property
    def shape(self) -> tuple[int, int]:
        raise NotImplementedError

    def extract(self, rows, cols) -> np.ndarray:
        raise NotImplementedError

    def dense(self) -> np.ndarray:
        raise NotImplementedError


class DenseAccessor(MatrixAccessor):
    """MatrixAccessor over an in-memory array (stored Fortran-ordered)."""

    def __init__(self, values):
        self._a = np.asfortranarray(np.atleast_2d(np.asarray(values, dtype=float)))

    @property
    def shape(self) -> tuple[int, int]:
        return self._a.shape

    def extract(self, rows, cols) -> np.ndarray:
        r = np.asarray(rows, dtype=np.intp)
        c = np.asarray(cols, dtype=np.intp)
        return self._a[np.ix_(r, c)]

    def dense(self) -> np.ndarray:
        return self._a


class DeviceAccessor(MatrixAccessor):
    """MatrixAccessor whose buffer lives in HBM (a device.DeviceMatrix).

    Products use the device copy directly (no host round trip); extract()
    gathers the requested entries on the device."""

    def __init__(self, dm: "_dev.DeviceMatrix"):
        self.dm = dm

    @property
    def shape(self) -> tuple[int, int]:
        return self.dm.shape

    def extract(self, rows, cols) -> np.ndarray:
        import torch
        dev = self.dm.t.device
        r = torch.as_tensor(np.asarray(rows, dtype=np.int64), device=dev)
        c = torch.as_tensor(np.asarray(cols, dtype=np.int64), device=dev)
        sub = self.dm.t.index_select(0, c).index_select(1, r)
        return np.ascontiguousarray(sub.cpu().numpy().T)

    def dense(self) -> np.ndarray:
        return self.dm.to_host()


def _buffer_of(A) -> np.ndarray:
    if isinstance(A, MatrixAccessor):
        return A.dense()
    return np.asfortranarray(np.atleast_2d(np.asarray(A, dtype=float)))


def _is_accessor(A) -> bool:
    # duck-typed so the reference's MatrixAccessor subclasses qualify too
    return isinstance(A, MatrixAccessor) or (
        callable(getattr(A, "dense", None)) and callable(getattr(A, "extract", None)))


def device_matrix_of(A) -> "_dev.DeviceMatrix":
    """HBM copy of A (MatrixAccessor, DeviceMatrix or array-like).

    Accessor buffers are cached by identity (the dense() contract); raw
    arrays may be mutated by the caller, so they are uploaded every call."""
    if isinstance(A, _dev.DeviceMatrix):
        return A
    if isinstance(A, DeviceAccessor):
        return A.dm
    if _is_accessor(A):
        buf = A.dense()
        if not (buf.dtype == np.float64 and buf.flags.f_contiguous):
            buf = np.asfortranarray(buf, dtype=np.float64)
        return _dev.A_CACHE.get(buf)
    return _dev.DeviceMatrix.from_host(_buffer_of(A))


def _shape_of(A) -> tuple[int, int]:
    if isinstance(A, _dev.DeviceMatrix) or _is_accessor(A):
        return tuple(A.shape)
    a = np.asarray(A)
    return a.shape if a.ndim == 2 else np.atleast_2d(a).shape


def fwht(x) -> np.ndarray:
    """Normalised Walsh-Hadamard transform of a vector or of each matrix row
    (length a power of two), computed by the hsk_fwht kernel."""
    arr = np.atleast_2d(np.array(x, dtype=float, copy=True))
    n = arr.shape[1]
    if n == 0 or n & (n - 1):
        raise ValueError("fwht length must be a power of two")
    _dev.require_cuda()
    import torch
    from . import _lib
    t = torch.from_numpy(np.ascontiguousarray(arr)).cuda()
    _lib.call("hsk_fwht", t.data_ptr(), arr.shape[0], n, 1, _dev.current_stream_ptr())
    out = t.cpu().numpy()
    return out[0] if np.ndim(x) == 1 else out


def _run_blocks(dA, op, transpose: bool, out, col0: int):
    lo = col0
    for blk in op.blocks:
        _dev.apply_block(blk, dA, transpose, out, lo)
        lo += blk.rows
    return out


def apply_right_device(A, op, out=None, col0: int = 0) -> "_dev.DeviceMatrix":
    """A R^T into a device buffer (columns [col0, col0 + op.d))."""
    dA = device_matrix_of(A)
    if dA.cols != op.n:
        raise ValueError(f"operator is over dimension {op.n}, matrix has {dA.cols} columns")
    out = out if out is not None else _dev.DeviceMatrix.empty(dA.rows, op.d)
    return _run_blocks(dA, op, False, out, col0)


def apply_right_transposed_device(A, op, out=None, col0: int = 0) -> "_dev.DeviceMatrix":
    """A^T R^T into a device buffer (columns [col0, col0 + op.d))."""
    dA = device_matrix_of(A)
    if dA.rows != op.n:
        raise ValueError(f"operator is over dimension {op.n}, matrix has {dA.rows} rows")
    out = out if out is not None else _dev.DeviceMatrix.empty(dA.cols, op.d)
    return _run_blocks(dA, op, True, out, col0)


def apply_right(A, op: SketchOperator) -> np.ndarray:
    """S = A R^T (m x op.d) for every block of op, on the GPU."""
    m, k = _shape_of(A)
    if k != op.n:
        raise ValueError(f"operator is over dimension {op.n}, matrix has {k} columns")
    if m == 0:
        return np.empty((0, op.d), order="F")
    return apply_right_device(A, op).to_host()


def apply_right_transposed(A, op: SketchOperator) -> np.ndarray:
    """S' = A^T R^T (n_A x op.d) for every block of op, on the GPU."""
    k, m = _shape_of(A)
    if k != op.n:
        raise ValueError(f"operator is over dimension {op.n}, matrix has {k} rows")
    if m == 0:
        return np.empty((0, op.d), order="F")
    return apply_right_transposed_device(A, op).to_host()
