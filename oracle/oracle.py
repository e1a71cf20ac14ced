"""ctypes wrapper around the CPU oracle (oracle/hsk_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline leg as the parity checker / CPU baseline.  The
product package (paper_2302_01977_b200) never imports this module.

Each wrapper restates one reference function of hsskit
(/root/reference/pkg/src/hsskit/sketching.py) bit-exactly except the
Gaussian product (OpenBLAS order is not reproducible; see hsk_oracle.c):

  sjlt_right      SjltBlock.apply_right              sketching.py:322-332
  sjlt_right_t    SjltBlock.apply_right_transposed   sketching.py:334-351
  srht            SrhtBlock._transform               sketching.py:162-176
  fwht            fwht                               sketching.py:100-112
  gauss           GaussianBlock.apply_right(_t)      sketching.py:134-138
  apply_right / apply_right_transposed   module dispatch  sketching.py:431-457
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_d = ctypes.c_double
_i64 = ctypes.c_int64
_int = ctypes.c_int
_p = ctypes.c_void_p


def build() -> str:
    """Compile liboracle.so in place (gcc; seconds)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return os.path.join(_HERE, "liboracle.so")


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        src = os.path.join(_HERE, "hsk_oracle.c")
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
            build()
        L = ctypes.CDLL(path)
        L.oracle_sjlt_right.argtypes = [_p, _i64, _i64, _i64, _p, _p, _int, _int, _d, _p, _i64, _int]
        L.oracle_sjlt_right_t.argtypes = [_p, _i64, _i64, _i64, _p, _p, _int, _int, _d, _p, _i64, _int]
        L.oracle_srht.argtypes = [_p, _i64, _i64, _i64, _int, _p, _i64, _p, _int, _d, _p, _i64, _int]
        L.oracle_gauss.argtypes = [_p, _i64, _i64, _i64, _int, _p, _int, _p, _i64, _int]
        L.oracle_fwht.argtypes = [_p, _i64, _i64, _int]
        L.oracle_reduceat_segment.argtypes = [_p, _i64]
        L.oracle_reduceat_segment.restype = _d
        L.oracle_num_threads.restype = _int
        _LIB = L
    return _LIB


def num_threads() -> int:
    return lib().oracle_num_threads()


def _fbuf(A) -> np.ndarray:
    return np.asfortranarray(np.atleast_2d(np.asarray(A, dtype=np.float64)))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_p)


def _check(rc: int, name: str):
    if rc != 0:
        raise ValueError(f"{name} failed with code {rc}")


def reduceat_segment(seg) -> float:
    seg = np.ascontiguousarray(seg, dtype=np.float64)
    return lib().oracle_reduceat_segment(_ptr(seg), seg.size)


def sjlt_right(buf, pos, signs, d: int, scale: float, nthreads: int = 0) -> np.ndarray:
    buf = _fbuf(buf)
    m, n = buf.shape
    pos = np.ascontiguousarray(pos, dtype=np.int64).reshape(n, -1)
    sg = np.ascontiguousarray(signs, dtype=np.int8).reshape(n, -1)
    out = np.empty((m, d), order="F")
    _check(lib().oracle_sjlt_right(_ptr(buf), m, n, max(m, 1), _ptr(pos), _ptr(sg),
                                   pos.shape[1], d, scale, _ptr(out), max(m, 1), nthreads),
           "oracle_sjlt_right")
    return out


def sjlt_right_t(buf, pos, signs, d: int, scale: float, nthreads: int = 0) -> np.ndarray:
    buf = _fbuf(buf)
    nr, nc = buf.shape
    pos = np.ascontiguousarray(pos, dtype=np.int64).reshape(nr, -1)
    sg = np.ascontiguousarray(signs, dtype=np.int8).reshape(nr, -1)
    out = np.empty((nc, d), order="F")
    _check(lib().oracle_sjlt_right_t(_ptr(buf), nr, nc, max(nr, 1), _ptr(pos), _ptr(sg),
                                     pos.shape[1], d, scale, _ptr(out), max(nc, 1), nthreads),
           "oracle_sjlt_right_t")
    return out


def srht(buf, signs, sample, d: int, scale: float, transpose: bool,
         nthreads: int = 0) -> np.ndarray:
    buf = _fbuf(buf)
    signs = np.ascontiguousarray(signs, dtype=np.float64)
    sample = np.ascontiguousarray(sample, dtype=np.int64)
    if transpose:
        n, m = buf.shape
    else:
        m, n = buf.shape
    out = np.empty((m, d), order="F")
    _check(lib().oracle_srht(_ptr(buf), m, n, max(buf.shape[0], 1), int(transpose),
                             _ptr(signs), signs.size, _ptr(sample), d, scale,
                             _ptr(out), max(m, 1), nthreads), "oracle_srht")
    return out


def gauss(buf, R, transpose: bool, nthreads: int = 0) -> np.ndarray:
    buf = _fbuf(buf)
    R = np.ascontiguousarray(R, dtype=np.float64)
    d, n = R.shape
    m = buf.shape[1] if transpose else buf.shape[0]
    out = np.empty((m, d), order="F")
    _check(lib().oracle_gauss(_ptr(buf), m, n, max(buf.shape[0], 1), int(transpose),
                              _ptr(R), d, _ptr(out), max(m, 1), nthreads), "oracle_gauss")
    return out


def fwht(x, normalize: bool = True) -> np.ndarray:
    arr = np.array(x, dtype=np.float64, copy=True)
    squeeze = arr.ndim == 1
    arr = np.ascontiguousarray(np.atleast_2d(arr))
    _check(lib().oracle_fwht(_ptr(arr), arr.shape[0], arr.shape[1], int(normalize)),
           "oracle_fwht")
    return arr[0] if squeeze else arr


# --------------------------------------------------------------------------
# operator-level restatement of the module dispatch (sketching.py:431-457).
# Blocks are duck-typed: any object exposing the reference's block
# attributes (kind, rows, _pos/_signs/_scale, matrix, signs/sample/scale).

def block_apply(block, buf, transpose: bool, nthreads: int = 0) -> np.ndarray:
    kind = block.kind
    if kind == "sjlt":
        f = sjlt_right_t if transpose else sjlt_right
        return f(buf, block._pos, block._signs, block.rows, block._scale, nthreads)
    if kind == "gaussian":
        return gauss(buf, block.matrix, transpose, nthreads)
    if kind == "srht":
        return srht(buf, block.signs, block.sample, block.rows, block.scale, transpose, nthreads)
    raise ValueError(f"unknown block kind {kind!r}")


def apply_right(A, op, nthreads: int = 0) -> np.ndarray:
    buf = _fbuf(A)
    if buf.shape[1] != op.n:
        raise ValueError("dimension mismatch")
    out = np.empty((buf.shape[0], op.d), order="F")
    lo = 0
    for b in op.blocks:
        out[:, lo:lo + b.rows] = block_apply(b, buf, False, nthreads)
        lo += b.rows
    return out


def apply_right_transposed(A, op, nthreads: int = 0) -> np.ndarray:
    buf = _fbuf(A)
    if buf.shape[0] != op.n:
        raise ValueError("dimension mismatch")
    out = np.empty((buf.shape[1], op.d), order="F")
    lo = 0
    for b in op.blocks:
        out[:, lo:lo + b.rows] = block_apply(b, buf, True, nthreads)
        lo += b.rows
    return out


def rel_frobenius(x, ref) -> float:
    ref = np.asarray(ref)
    den = float(np.linalg.norm(ref))
    num = float(np.linalg.norm(np.asarray(x) - ref))
    return num / den if den > 0 else num


def sjlt_scale(alpha: int) -> float:
    return 1.0 / math.sqrt(alpha)
