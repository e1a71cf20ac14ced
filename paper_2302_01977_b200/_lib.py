"""ctypes binding of libhsk.so (include/hsk.h).

The product path has no CPU fallback: if the library or a CUDA device is
missing, every compute entry point raises RuntimeError.  Status codes map
onto the reference's exception classes (hsk.h): HSK_EINVAL -> ValueError,
HSK_ERANGE -> IndexError, CUDA failures -> RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhsk.so")

HSK_OK, HSK_EINVAL, HSK_ERANGE, HSK_ECUDA, HSK_ENODEV = 0, -1, -2, -3, -4

_c_i32 = ctypes.c_int32
_c_i64 = ctypes.c_int64
_c_d = ctypes.c_double
_c_p = ctypes.c_void_p

# name -> (restype, argtypes); mirrors include/hsk.h
SIGNATURES = {
    "hsk_abi_version": (ctypes.c_int, []),
    "hsk_tuning_reload": (ctypes.c_int, []),
    "hsk_tuning_generation": (ctypes.c_int, []),
    "hsk_last_error": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_size_t]),
    "hsk_device_info": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                       ctypes.POINTER(ctypes.c_int), ctypes.POINTER(_c_i64)]),
    "hsk_sjlt_plan_bytes": (_c_i64, [_c_i64, _c_i32, _c_i32]),
    "hsk_sjlt_plan_build": (ctypes.c_int, [_c_p, _c_p, _c_i64, _c_i32, _c_i32, _c_p, _c_i64, _c_p]),
    "hsk_sjlt_apply": (ctypes.c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_i32, _c_p, _c_i64, _c_i32,
                                      _c_i32, _c_d, _c_p, _c_i64, _c_i64, _c_p]),
    "hsk_sjlt_plan_bytes_ex": (_c_i64, [_c_i64, _c_i32, _c_i32, _c_i32]),
    "hsk_sjlt_plan_build_ex": (ctypes.c_int, [_c_p, _c_p, _c_i64, _c_i32, _c_i32, _c_i32, _c_p, _c_i64,
                                              _c_p]),
    "hsk_sjlt_apply_ex": (ctypes.c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_i32, _c_p, _c_i64, _c_i32,
                                         _c_i32, _c_i32, _c_d, _c_p, _c_i64, _c_i64, _c_p]),
    "hsk_gauss_apply": (ctypes.c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_i32, _c_p, _c_i64, _c_i32,
                                       _c_p, _c_i64, _c_i64, _c_p]),
    "hsk_srht_apply": (ctypes.c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_i32, _c_p, _c_i64, _c_i64,
                                      _c_p, _c_i32, _c_d, _c_p, _c_i64, _c_i64, _c_p]),
    "hsk_fwht": (ctypes.c_int, [_c_p, _c_i64, _c_i64, _c_i32, _c_p]),
    "hsk_gen_gauss_kernel": (ctypes.c_int, [_c_p, _c_i64, _c_i32, _c_d, _c_d, _c_i64, _c_i64,
                                            _c_i64, _c_i64, _c_p, _c_i64, _c_p]),
    "hsk_gen_toeplitz_sin": (ctypes.c_int, [_c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_p, _c_i64,
                                            _c_p]),
    "hsk_l2_flush": (ctypes.c_int, [_c_p, _c_i64, _c_p]),
    "hsk_transpose": (ctypes.c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_i64, _c_p]),
    "hsk_is_symmetric": (ctypes.c_int, [_c_p, _c_i64, _c_i64, _c_p, _c_p]),
    "hsk_ipc_alloc": (ctypes.c_int, [_c_i64, ctypes.POINTER(_c_p), _c_p]),
    "hsk_ipc_free": (ctypes.c_int, [_c_p]),
    "hsk_ipc_open": (ctypes.c_int, [_c_p, ctypes.POINTER(_c_p)]),
    "hsk_ipc_close": (ctypes.c_int, [_c_p]),
    "hsk_sum_slices": (ctypes.c_int, [_c_p, _c_i32, _c_i64, _c_i64, _c_i64, _c_i64, _c_p, _c_i64,
                                      _c_p]),
    "hsk_pqr_work_bytes": (_c_i64, [_c_i64, _c_i64]),
    "hsk_pqr": (ctypes.c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_d, _c_d, _c_p, _c_p, _c_i64, _c_p, _c_p,
                               _c_i64, _c_p]),
    "hsk_dmma_probe_flops": (_c_i64, [_c_i64]),
    "hsk_dmma_probe": (ctypes.c_int, [_c_i64, _c_p, _c_p]),
    "hsk_memcpy2d": (ctypes.c_int, [_c_p, _c_i64, _c_p, _c_i64, _c_i64, _c_i64, _c_i32, _c_p]),
}

_lock = threading.Lock()
_lib = None


class HskError(RuntimeError):
    """CUDA-side failure inside libhsk."""


def load(path: str | None = None):
    """Load libhsk.so (building it first if the sources are newer)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        # HSK_LIB: load another build of the same ABI (A/B timing of kernel
        # revisions on one GPU box; tools/ab_build.sh)
        path = path or os.environ.get("HSK_LIB") or LIB_PATH
        if not os.path.exists(path):
            try:
                from . import build as _build
                _build.build()
            except Exception as exc:  # noqa: BLE001
                raise RuntimeError(
                    f"libhsk.so is missing at {path} and could not be built ({exc}); "
                    "the sm_100a sketch engine has no CPU fallback") from exc
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.hsk_abi_version() != 1:
            raise RuntimeError("libhsk ABI version mismatch")
        _lib = lib
        return lib


def last_error() -> str:
    buf = ctypes.create_string_buffer(512)
    load().hsk_last_error(buf, 512)
    return buf.value.decode(errors="replace")


def check(rc: int, what: str = "") -> int:
    if rc >= 0:
        return rc
    msg = last_error() or what
    if rc == HSK_EINVAL:
        raise ValueError(msg)
    if rc == HSK_ERANGE:
        raise IndexError(msg)
    raise HskError(msg)


def call(name: str, *args):
    return check(getattr(load(), name)(*args), name)


def exported_symbols() -> list[str]:
    return list(SIGNATURES)
