"""Device residency for the sketch engine: HBM matrices and per-block R.

PyTorch is used only as plumbing here (device allocation, streams, host
<-> device copies); every sketch product is a libhsk.so kernel.

* DeviceMatrix   column-major fp64 matrix in HBM (rows x cols, even leading
                 dimension so TMA bulk copies of column segments are 16-byte
                 aligned), the layout the reference computes on
                 (`_buffer_of` -> Fortran order, sketching.py:76-79).
* block_state    per-operator-block device copy of R, uploaded once and
                 cached on the (immutable) block object: the
                 reference's own draw, bit-exact (SJLT `_pos`/`_signs` ->
                 device plan, Gaussian `matrix`, SRHT `signs`/`sample`).
* apply_block    launches the kernel for one block into a column slice of
                 a preallocated device output (the per-block loop of
                 sketching.py:431-457).
"""

from __future__ import annotations

import math
import os
import weakref

import numpy as np

from . import _lib

try:
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None

_CHUNK_BYTES = 256 << 20


def cuda_ready() -> bool:
    return torch is not None and torch.cuda.is_available()


def require_cuda():
    if not cuda_ready():
        raise RuntimeError("no CUDA device available: the sm_100a sketch engine has no CPU "
                           "fallback (run on a B200)")
    _lib.load()


def current_stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def even_ld(rows: int) -> int:
    return max(2, rows + (rows & 1))


class DeviceMatrix:
    """Column-major float64 matrix in device memory.

    Backed by a torch tensor of shape (cols, ld): tensor row j is column j.
    """

    __slots__ = ("rows", "cols", "ld", "t", "__weakref__")

    def __init__(self, rows: int, cols: int, ld: int | None = None, tensor=None, device=None):
        require_cuda()
        self.rows = int(rows)
        self.cols = int(cols)
        self.ld = int(ld) if ld is not None else even_ld(self.rows)
        if self.ld < max(1, self.rows):
            raise ValueError("leading dimension smaller than the row count")
        if tensor is None:
            dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
            tensor = torch.empty((max(self.cols, 1), self.ld), dtype=torch.float64, device=dev)
        self.t = tensor

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    @property
    def shape(self) -> tuple[int, int]:
        return (self.rows, self.cols)

    @classmethod
    def empty(cls, rows: int, cols: int, ld: int | None = None) -> "DeviceMatrix":
        return cls(rows, cols, ld)

    @classmethod
    def zeros(cls, rows: int, cols: int, ld: int | None = None) -> "DeviceMatrix":
        m = cls(rows, cols, ld)
        m.t.zero_()
        return m

    @classmethod
    def from_host(cls, buf: np.ndarray, ld: int | None = None) -> "DeviceMatrix":
        """Upload a host matrix (any layout; copied as column-major)."""
        buf = np.asfortranarray(np.atleast_2d(np.asarray(buf, dtype=np.float64)))
        m = cls(buf.shape[0], buf.shape[1], ld)
        m.upload(buf)
        return m

    def upload(self, buf: np.ndarray, col0: int = 0):
        """Copy host columns buf (F-order rows x k) into columns [col0, col0+k)."""
        buf = np.asfortranarray(buf, dtype=np.float64)
        if buf.shape[0] != self.rows or col0 + buf.shape[1] > self.cols:
            raise ValueError("upload shape mismatch")
        if buf.size == 0:
            return
        src = torch.from_numpy(buf.T)  # (k, rows) C-contiguous view, no copy
        k = buf.shape[1]
        if self.ld == self.rows:
            self.t[col0:col0 + k].copy_(src, non_blocking=True)
            return
        step = max(1, _CHUNK_BYTES // (8 * max(self.rows, 1)))
        for c0 in range(0, k, step):
            c1 = min(k, c0 + step)
            self.t[col0 + c0:col0 + c1, :self.rows].copy_(src[c0:c1], non_blocking=True)

    def to_host(self, col0: int = 0, ncols: int | None = None) -> np.ndarray:
        """Fresh host copy of columns [col0, col0+ncols) in Fortran order."""
        ncols = self.cols - col0 if ncols is None else ncols
        if self.rows == 0 or ncols == 0:
            return np.zeros((self.rows, ncols), order="F")
        # D2H straight into pinned memory from torch's caching host allocator:
        # full-rate DMA and no first-touch page faults on a fresh pageable
        # buffer (which cost more than the copy itself).  The numpy view keeps
        # the pinned block alive; it returns to the pool when the caller drops it.
        host = torch.empty((ncols, self.rows), dtype=torch.float64, pin_memory=True)
        host.copy_(self.t[col0:col0 + ncols, :self.rows])
        return host.numpy().T  # (rows, ncols) F-contiguous, owned by the caller

    def transposed(self) -> "DeviceMatrix":
        """A fresh device copy of this matrix's transpose (hsk_transpose)."""
        out = DeviceMatrix(self.cols, self.rows)
        _lib.call("hsk_transpose", self.ptr, self.rows, self.cols, self.ld, out.ptr, out.ld,
                  current_stream_ptr())
        return out

    def is_symmetric(self) -> bool:
        """True if this square matrix equals its transpose bit for bit
        (hsk_is_symmetric; one host sync)."""
        if self.rows != self.cols:
            return False
        flag = torch.empty(1, dtype=torch.int32, device=self.t.device)
        _lib.call("hsk_is_symmetric", self.ptr, self.rows, self.ld, flag.data_ptr(),
                  current_stream_ptr())
        return int(flag.item()) == 0

    def column_view(self, col0: int, ncols: int) -> "DeviceMatrix":
        sub = DeviceMatrix.__new__(DeviceMatrix)
        sub.rows, sub.cols, sub.ld = self.rows, ncols, self.ld
        sub.t = self.t[col0:col0 + ncols]
        return sub

    def row_view(self, row0: int, nrows: int) -> "DeviceMatrix":
        """Rows [row0, row0+nrows) as a strided view (same leading dimension)."""
        sub = DeviceMatrix.__new__(DeviceMatrix)
        sub.rows, sub.cols, sub.ld = nrows, self.cols, self.ld
        sub.t = self.t[:, row0:row0 + nrows]
        return sub


class RawMatrix:
    """Column-major rows x cols view of device memory this process does not
    own through torch -- e.g. a peer GPU's receive slot mapped by CUDA IPC
    (distributed.PeerSlots).  Kernel outputs only; no host transfers."""

    __slots__ = ("rows", "cols", "ld", "ptr")

    def __init__(self, ptr: int, rows: int, cols: int, ld: int):
        if ld < max(1, rows):
            raise ValueError("leading dimension smaller than the row count")
        self.ptr, self.rows, self.cols, self.ld = int(ptr), int(rows), int(cols), int(ld)

    @property
    def shape(self) -> tuple[int, int]:
        return (self.rows, self.cols)


# --------------------------------------------------------------- R on device

class _SjltState:
    __slots__ = ("pos", "sgn", "plan", "n", "d", "alpha", "scale", "flags", "gen")


HSK_SJLT_CHUNKED = 1  # include/hsk.h


def sjlt_chunked(pos: np.ndarray, d: int, alpha: int, construction=None) -> bool:
    """Whether to build the paired plan: only for the shapes it serves (d/alpha
    = 8, d a multiple of 64; include/hsk.h), and only for patterns with the
    block construction's chunk property (sketching.py:246-250: entry t of
    every input index in chunk t of d/alpha buckets) -- guaranteed by the
    reference's block construction, checked on the pattern otherwise
    (from_pattern blocks qualify too).  HSK_SJLT_NOCHUNK=1 turns it off (A/B
    runs)."""
    if os.environ.get("HSK_SJLT_NOCHUNK") == "1" or pos.size == 0:
        return False
    if d % 64 or alpha * 8 != d:
        return False
    if construction == "block":
        return True
    return bool((pos // (d // alpha) == np.arange(alpha, dtype=pos.dtype)).all())


class _GaussState:
    __slots__ = ("R", "n", "d")


class _SrhtState:
    __slots__ = ("signs", "sample", "n", "n_pad", "d", "scale")


_STATE_ATTR = "_hsk_device_state"


def _device_key() -> int:
    return torch.cuda.current_device()


def block_state(block):
    """Device copy of a block's random draw; uploaded once per device."""
    require_cuda()
    cache = block.__dict__.setdefault(_STATE_ATTR, {})
    key = _device_key()
    st = cache.get(key)
    # an SJLT plan is tied to the tuning knobs it was built under
    gen = _lib.load().hsk_tuning_generation() if block.kind == "sjlt" else 0
    if st is not None and getattr(st, "gen", 0) == gen:
        return st
    kind = block.kind
    dev = torch.device("cuda", key)
    stream = current_stream_ptr()
    if kind == "sjlt":
        pos = np.ascontiguousarray(block._pos)
        n, alpha = int(block.n), int(block.alpha)
        d = int(block.rows)
        if pos.shape != (n, alpha):
            pos = pos.reshape(n, alpha)
        if pos.size and (pos.min() < 0 or pos.max() >= d):
            raise ValueError(f"SJLT pattern positions must lie in [0, {d})")
        st = _SjltState()
        st.pos = torch.from_numpy(pos.astype(np.int32, copy=False).reshape(-1)).to(dev)
        st.sgn = torch.from_numpy(np.ascontiguousarray(block._signs, dtype=np.int8).reshape(-1)).to(dev)
        st.n, st.d, st.alpha = n, d, alpha
        st.scale = float(block._scale)
        chunked = sjlt_chunked(pos, d, alpha, getattr(block, "construction", None))
        st.flags = HSK_SJLT_CHUNKED if chunked else 0
        st.gen = gen
        nbytes = _lib.load().hsk_sjlt_plan_bytes_ex(n, d, alpha, st.flags)
        _lib.check(nbytes, "hsk_sjlt_plan_bytes_ex")
        st.plan = torch.empty(int(nbytes), dtype=torch.uint8, device=dev)
        _lib.call("hsk_sjlt_plan_build_ex", st.pos.data_ptr(), st.sgn.data_ptr(), n, d, alpha,
                  st.flags, st.plan.data_ptr(), int(nbytes), stream)
    elif kind == "gaussian":
        st = _GaussState()
        st.R = torch.from_numpy(np.ascontiguousarray(block.matrix, dtype=np.float64)).to(dev)
        st.d, st.n = st.R.shape
    elif kind == "srht":
        st = _SrhtState()
        st.signs = torch.from_numpy(np.ascontiguousarray(block.signs, dtype=np.float64)).to(dev)
        st.sample = torch.from_numpy(np.ascontiguousarray(block.sample, dtype=np.int64)).to(dev)
        st.n, st.n_pad, st.d = int(block.n), int(block.n_pad), int(block.rows)
        st.scale = float(block.scale)
    else:
        raise ValueError(f"unknown operator kind {kind!r}")
    cache[key] = st
    return st


def apply_block(block, A: DeviceMatrix, transpose: bool, S: DeviceMatrix, col0: int,
                stream: int | None = None):
    """S[:, col0:col0+block.rows] = A R_b^T (or A^T R_b^T) on the device."""
    st = block_state(block)
    stream = current_stream_ptr() if stream is None else stream
    trans = 1 if transpose else 0
    m_out = A.cols if transpose else A.rows
    if S.rows != m_out or col0 + block.rows > S.cols:
        raise ValueError("output buffer does not match the sketch shape")
    kind = block.kind
    if kind == "sjlt":
        _lib.call("hsk_sjlt_apply_ex", A.ptr, A.rows, A.cols, A.ld, trans, st.plan.data_ptr(),
                  st.n, st.d, st.alpha, st.flags, st.scale, S.ptr, S.ld, col0, stream)
    elif kind == "gaussian":
        _lib.call("hsk_gauss_apply", A.ptr, A.rows, A.cols, A.ld, trans, st.R.data_ptr(),
                  st.n, st.d, S.ptr, S.ld, col0, stream)
    else:
        _lib.call("hsk_srht_apply", A.ptr, A.rows, A.cols, A.ld, trans, st.signs.data_ptr(),
                  st.n, st.n_pad, st.sample.data_ptr(), st.d, st.scale, S.ptr, S.ld, col0,
                  stream)


# ------------------------------------------------------ host buffer cache

class _ACache:
    """Device copies of accessor buffers, keyed by buffer identity.

    Legal because MatrixAccessor.dense() must return the same buffer on
    every call and callers never mutate it (sketching.py:37-44).  Raw arrays
    passed directly are NOT cached (they may be mutated between calls).
    """

    def __init__(self, capacity: int = 2):
        self.capacity = capacity
        self.entries: list[tuple] = []  # (weakref(buf), key, DeviceMatrix)

    def get(self, buf: np.ndarray) -> DeviceMatrix:
        key = (buf.ctypes.data, buf.shape, buf.strides, _device_key())
        alive = []
        hit = None
        for ref, k, dm in self.entries:
            b = ref()
            if b is None:
                continue
            alive.append((ref, k, dm))
            if b is buf and k == key:
                hit = dm
        self.entries = alive
        if hit is not None:
            return hit
        dm = DeviceMatrix.from_host(buf)
        self.entries.append((weakref.ref(buf), key, dm))
        while len(self.entries) > self.capacity:
            self.entries.pop(0)
        return dm

    def clear(self):
        self.entries = []


A_CACHE = _ACache()


def sjlt_scale(alpha: int) -> float:
    return 1.0 / math.sqrt(alpha)
