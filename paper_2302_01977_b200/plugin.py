"""Install the GPU sketch engine into the reference package (hsskit).

The reference compressor calls `sketching.apply_right(self.A, op)` and
`sketching.apply_right_transposed(self.A, op)` through the module
attribute, resolved at call time (hss_compress.py:21,164-165,178-179).
`install()` rebinds exactly those two attributes of `hsskit.sketching` to
GPU implementations that accept the reference's own SketchOperator / block
objects (duck-typed on `_pos`/`_signs`/`_scale`, `matrix`,
`signs`/`sample`/`scale`/`n_pad`), so R is the reference's own draw and
`new_operator`, `append_columns`, `dense_rows` and the whole compressor stay
untouched.  `uninstall()` restores the originals.

    import hsskit
    from paper_2302_01977_b200 import plugin
    plugin.install()          # every compress() sketch now runs on sm_100a

`install(compressor=True)` additionally rebinds `hsskit.hss_compress._Driver`
(resolved by `compress()` at call time, hss_compress.py:385) to
hss_device.DeviceDriver: the reference's sweep logic with the sketch, the
local samples, the gate QR / projections and the interpolative
decompositions kept on the device.
"""

from __future__ import annotations

import importlib

import numpy as np

from . import device as _dev
from . import sketching as _sk

_saved: dict = {}


def _module(mod=None):
    if mod is not None:
        return mod
    return importlib.import_module("hsskit.sketching")


def gpu_apply_right(A, op) -> np.ndarray:
    """Drop-in for hsskit.sketching.apply_right (sketching.py:431-442)."""
    m, k = _sk._shape_of(A)
    if k != op.n:
        raise ValueError(f"operator is over dimension {op.n}, matrix has {k} columns")
    if m == 0:
        return np.empty((0, op.d), order="F")
    return _sk.apply_right_device(A, op).to_host()


def gpu_apply_right_transposed(A, op) -> np.ndarray:
    """Drop-in for hsskit.sketching.apply_right_transposed (sketching.py:445-457)."""
    k, m = _sk._shape_of(A)
    if k != op.n:
        raise ValueError(f"operator is over dimension {op.n}, matrix has {k} rows")
    if m == 0:
        return np.empty((0, op.d), order="F")
    return _sk.apply_right_transposed_device(A, op).to_host()


def _compress_module(mod):
    """hsskit.hss_compress of the package whose sketching module is `mod`."""
    pkg = mod.__name__.rsplit(".", 1)[0]
    return importlib.import_module(pkg + ".hss_compress")


def install(mod=None, compressor: bool = False) -> None:
    """Route the reference's sketch products through libhsk.so (and, with
    compressor=True, the whole compression sweep through the device driver)."""
    _dev.require_cuda()
    mod = _module(mod)
    key = id(mod)
    if key not in _saved:
        _saved[key] = (mod, mod.apply_right, mod.apply_right_transposed)
    mod.apply_right = gpu_apply_right
    mod.apply_right_transposed = gpu_apply_right_transposed
    if compressor:
        from . import hss_device
        hc = _compress_module(mod)
        ck = ("driver", id(hc))
        if ck not in _saved:
            _saved[ck] = (hc, hc._Driver)
        hc._Driver = hss_device.device_driver_class(hc, base=_saved[ck][1])


def uninstall(mod=None) -> None:
    mod = _module(mod)
    entry = _saved.pop(id(mod), None)
    if entry is not None:
        _, ar, art = entry
        mod.apply_right = ar
        mod.apply_right_transposed = art
    try:
        hc = _compress_module(mod)
    except ImportError:
        return
    dentry = _saved.pop(("driver", id(hc)), None)
    if dentry is not None:
        hc._Driver = dentry[1]


def installed(mod=None) -> bool:
    mod = _module(mod)
    return mod.apply_right is gpu_apply_right
