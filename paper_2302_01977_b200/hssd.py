"""`.hssd` dense-matrix files read straight into HBM.

Mirrors the reference's file format and loader (`hsskit/matgen.py:16-22,
191-221`: magic ``HSSD``, little-endian u64 rows and cols, then the entries as
binary64 in column-major order) with the same validation order, messages and
exception class (`FileFormatError`, a `TypeError`).  The reference reads the
whole payload into host memory and wraps it in a DenseAccessor; `from_file`
here streams whole-column slabs from the file through two pinned staging
buffers into a `DeviceMatrix` (file read of slab i+1 overlapped with the H2D
copy of slab i), so an n x n matrix never exists in host memory and the
result is a `DeviceAccessor` the sketch products use in place.  Header
validation runs before anything touches the device, so malformed files fail
the same way with or without a GPU.
"""

from __future__ import annotations

import os
import struct

import numpy as np

from . import device as _dev

MAGIC = b"HSSD"
_HEADER = 4 + 16
_SLAB_BYTES = 64 << 20


class FileFormatError(TypeError):
    """Raised for malformed dense-matrix files (hsskit.matgen.FileFormatError)."""


def write_file(path, values) -> None:
    """Serialize a dense matrix exactly as `hsskit.matgen.write_file` does."""
    a = np.atleast_2d(np.asarray(values, dtype=float))
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(struct.pack("<QQ", a.shape[0], a.shape[1]))
        fh.write(a.astype("<f8").tobytes(order="F"))


def read_header(path) -> tuple[int, int]:
    """(rows, cols) of a well-formed file; FileFormatError otherwise, with the
    reference's checks in the reference's order (matgen.py:203-219)."""
    with open(path, "rb") as fh:
        magic = fh.read(4)
        if magic != MAGIC:
            raise FileFormatError(f"bad magic {magic!r}; expected {MAGIC.decode()!r}")
        header = fh.read(16)
        if len(header) < 16:
            raise FileFormatError("truncated header")
        rows, cols = struct.unpack("<QQ", header)
        held = os.fstat(fh.fileno()).st_size - _HEADER
    expected = rows * cols * 8
    if expected > 2**40:
        raise FileFormatError(f"dimensions {rows}x{cols} overflow sane size")
    if held != expected:
        raise FileFormatError(
            f"truncated payload: header promises {rows * cols} values "
            f"({expected} bytes), file holds {held} bytes")
    return int(rows), int(cols)


def from_file(path, slab_bytes: int = _SLAB_BYTES):
    """Load a file written by write_file into HBM; returns a DeviceAccessor.

    Column slabs of about `slab_bytes` alternate between two pinned buffers:
    the host reads slab i+1 from the file while slab i is in flight to the
    device (one copy stream, an event per buffer)."""
    import torch

    from .sketching import DeviceAccessor

    rows, cols = read_header(path)
    _dev.require_cuda()
    dm = _dev.DeviceMatrix.empty(rows, cols)
    if rows == 0 or cols == 0:
        return DeviceAccessor(dm)
    step = max(1, min(cols, slab_bytes // (8 * rows)))
    bufs = [torch.empty((step, rows), dtype=torch.float64, pin_memory=True) for _ in range(2)]
    done = [None, None]
    stream = torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())  # dm's block may still be in use there
    with open(path, "rb", buffering=0) as fh:
        fh.seek(_HEADER)
        for i, c0 in enumerate(range(0, cols, step)):
            k = min(step, cols - c0)
            b = i & 1
            if done[b] is not None:
                done[b].synchronize()  # the copy that last used this buffer has landed
            view = bufs[b][:k]
            mv = memoryview(view.numpy()).cast("B")
            got = 0
            while got < mv.nbytes:
                r = fh.readinto(mv[got:])
                if not r:
                    raise FileFormatError("truncated payload: file shrank while reading")
                got += r
            with torch.cuda.stream(stream):
                dm.t[c0:c0 + k, :rows].copy_(view, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
            done[b] = ev
    torch.cuda.current_stream().wait_stream(stream)
    stream.synchronize()
    return DeviceAccessor(dm)
