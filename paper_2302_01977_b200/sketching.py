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
  dense_rows                        host helper        sketching.py:460-476

(jl_dimension_bound, sketching.py:479-499, sizes operators from the
Table 4.1 bounds; it is not on the sketch path and is not restated.)

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
                        append_columns, dense_rows, new_operator)
from .draws import next_pow2 as _next_pow2

__all__ = [
    "GAUSSIAN", "SRHT", "SJLT", "KINDS", "BLOCK", "GRAPH", "CONSTRUCTIONS",
    "MatrixAccessor", "DenseAccessor", "DeviceAccessor", "fwht",
    "GaussianBlock", "SrhtBlock", "SjltBlock", "SjltStorage", "SketchOperator",
    "new_operator", "append_columns", "apply_right", "apply_right_transposed",
    "dense_rows", "device_matrix_of", "apply_right_device",
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
    gathers the requested entries on the device.  dense() honours the
    accessor contract (sketching.py:41-43: the same buffer on every call): the
    host copy is made once, on first request, and cached."""

    def __init__(self, dm: "_dev.DeviceMatrix"):
        self.dm = dm
        self._host = None

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
        if self._host is None:
            self._host = self.dm.to_host()
        return self._host


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
    buf = _pinned_host_buffer(A)
    if buf is not None:
        return _streamed(buf, op, transpose=False)
    buf = _pageable_host_buffer(A)
    if buf is not None:
        return _streamed(buf, op, transpose=False, staged=True)
    return apply_right_device(A, op).to_host()


def apply_right_transposed(A, op: SketchOperator) -> np.ndarray:
    """S' = A^T R^T (n_A x op.d) for every block of op, on the GPU."""
    k, m = _shape_of(A)
    if k != op.n:
        raise ValueError(f"operator is over dimension {op.n}, matrix has {k} rows")
    if m == 0:
        return np.empty((0, op.d), order="F")
    buf = _pinned_host_buffer(A)
    if buf is not None:
        return _streamed(buf, op, transpose=True)
    buf = _pageable_host_buffer(A)
    if buf is not None:
        return _streamed(buf, op, transpose=True, staged=True)
    return apply_right_transposed_device(A, op).to_host()


# ------------------------------------------------- streamed host matrices
# A pinned host matrix of at least STREAM_MIN_BYTES is moved in slabs whose
# H2D copy overlaps the previous slab's kernels and D2H copy (three streams,
# two device slab buffers): the transfer, not the sketch, bounds this path,
# and everything but the last slab's compute hides under it.  S rows (S'
# rows) depend only on the same rows (columns) of A, so the result is
# bit-identical to the one-shot device path.
STREAM_MIN_BYTES = 256 << 20
STREAM_SLABS = int(__import__("os").environ.get("HSK_STREAM_SLABS", "8"))


def _pinned_host_buffer(A):
    """The F-ordered float64 host buffer of a raw array if it is page-locked
    and large enough to stream; otherwise None."""
    if isinstance(A, _dev.DeviceMatrix) or _is_accessor(A) or not isinstance(A, np.ndarray):
        return None
    if A.ndim != 2 or A.dtype != np.float64 or not A.flags.f_contiguous:
        return None
    if A.nbytes < STREAM_MIN_BYTES:
        return None
    try:
        import torch
        pinned = torch.from_numpy(A.T).is_pinned()  # (cols, rows) C-contiguous view
    except Exception:  # noqa: BLE001
        return None
    return A if pinned else None


def _pageable_host_buffer(A):
    """A large F-ordered float64 host array that is NOT page-locked (what the
    reference's callers hand over): streamed through pinned staging."""
    if isinstance(A, _dev.DeviceMatrix) or _is_accessor(A) or not isinstance(A, np.ndarray):
        return None
    if A.ndim != 2 or A.dtype != np.float64 or not A.flags.f_contiguous:
        return None
    return A if A.nbytes >= STREAM_MIN_BYTES else None


_STAGE_POOL = None


def _stage_pool():
    global _STAGE_POOL
    if _STAGE_POOL is None:
        import concurrent.futures
        import os
        n = int(os.environ.get("HSK_STAGE_THREADS", "0")) or min(32, os.cpu_count() or 1)
        _STAGE_POOL = concurrent.futures.ThreadPoolExecutor(max_workers=n)
    return _STAGE_POOL


def _stage_copy(dst: np.ndarray, src: np.ndarray):
    """dst[...] = src with the pool's threads over column blocks (numpy's copy
    loops release the GIL, so the pageable -> pinned memcpy runs in parallel)."""
    pool = _stage_pool()
    k = dst.shape[1]
    parts = min(pool._max_workers, max(1, k))
    bounds = [(k * i) // parts for i in range(parts + 1)]
    futs = [pool.submit(np.copyto, dst[:, a:b], src[:, a:b]) for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
    for f in futs:
        f.result()


def _streamed(buf: np.ndarray, op: SketchOperator, transpose: bool, staged: bool = False) -> np.ndarray:
    """Slab pipeline.  staged=True (pageable host array): each slab is first
    copied by host threads into one of two pinned staging buffers (the copy
    of slab i+1 overlaps slab i's DMA and kernels), then DMA'd from there."""
    import torch
    from . import _lib
    rows, cols = buf.shape
    m_out = cols if transpose else rows       # output rows
    nslab = max(1, min(STREAM_SLABS, m_out // 256))
    step = -(-m_out // nslab)
    step += step & 1                          # even leading dimension (16-byte TMA rows)
    comp = torch.cuda.current_stream()
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    # slab buffers: S: `step` rows of A (ld step); S': `step` columns (ld rows)
    sl_ld = step if not transpose else _dev.even_ld(rows)
    sl_cols = cols if not transpose else step
    slabs = [_dev.DeviceMatrix(step if not transpose else rows, sl_cols, ld=sl_ld) for _ in range(2)]
    out = _dev.DeviceMatrix.empty(m_out, op.d)
    host = torch.empty((op.d, m_out), dtype=torch.float64, pin_memory=True)
    # the slab and output buffers come from the caching allocator on `comp`:
    # kernels still queued there may have used those blocks last
    h2d.wait_stream(comp)
    d2h.wait_stream(comp)
    ev_in = [torch.cuda.Event() for _ in range(nslab)]
    ev_k = [torch.cuda.Event() for _ in range(nslab)]
    base = buf.ctypes.data
    stage = None
    if staged:  # two pinned slab images: S: h x cols (pitch h); S': rows x h
        shape = (cols, step) if not transpose else (step, rows)
        stage = [torch.empty(shape, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    for i in range(nslab):
        r0 = i * step
        r1 = min(m_out, r0 + step)
        if r0 >= r1:
            break
        h = r1 - r0
        b = slabs[i % 2]
        if i >= 2:
            h2d.wait_event(ev_k[i - 2])       # slab buffer free
        if staged:
            if i >= 2:
                ev_in[i - 2].synchronize()    # staging buffer's DMA has landed
            sg = stage[i % 2]
            if transpose:
                img = sg[:h].numpy().T        # rows x h, F-ordered
                _stage_copy(img, buf[:, r0:r1])
                _lib.call("hsk_memcpy2d", b.ptr, b.ld * 8, sg.data_ptr(), rows * 8, rows * 8, h, 1,
                          h2d.cuda_stream)
            else:
                img = sg[:, :h].numpy().T     # h x cols view, pitch step
                _stage_copy(img, buf[r0:r1, :])
                _lib.call("hsk_memcpy2d", b.ptr, b.ld * 8, sg.data_ptr(), step * 8, h * 8, cols, 1,
                          h2d.cuda_stream)
        elif transpose:   # columns [r0, r1) of A: h contiguous columns of `rows` doubles
            _lib.call("hsk_memcpy2d", b.ptr, b.ld * 8, base + r0 * rows * 8, rows * 8, rows * 8, h, 1,
                      h2d.cuda_stream)
        else:           # rows [r0, r1) of A: `cols` columns of h doubles, pitch `rows`
            _lib.call("hsk_memcpy2d", b.ptr, b.ld * 8, base + r0 * 8, rows * 8, h * 8, cols, 1,
                      h2d.cuda_stream)
        ev_in[i].record(h2d)
        comp.wait_event(ev_in[i])
        view = _dev.DeviceMatrix.__new__(_dev.DeviceMatrix)
        if transpose:
            view.rows, view.cols, view.ld, view.t = rows, h, b.ld, b.t[:h]
            apply_right_transposed_device(view, op, out=out.row_view(r0, h))
        else:
            view.rows, view.cols, view.ld, view.t = h, cols, b.ld, b.t
            apply_right_device(view, op, out=out.row_view(r0, h))
        ev_k[i].record(comp)
        d2h.wait_event(ev_k[i])
        _lib.call("hsk_memcpy2d", host.data_ptr() + r0 * 8, m_out * 8, out.ptr + r0 * 8, out.ld * 8,
                  h * 8, op.d, 2, d2h.cuda_stream)
    d2h.synchronize()
    comp.synchronize()
    del slabs
    return host.numpy().T                     # (m_out, d) F-contiguous, caller-owned
