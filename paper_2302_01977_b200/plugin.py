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


def install(mod=None) -> None:
    """Route the reference's sketch products through libhsk.so."""
    _dev.require_cuda()
    mod = _module(mod)
    key = id(mod)
    if key not in _saved:
        _saved[key] = (mod, mod.apply_right, mod.apply_right_transposed)
    mod.apply_right = gpu_apply_right
    mod.apply_right_transposed = gpu_apply_right_transposed


def uninstall(mod=None) -> None:
    mod = _module(mod)
    entry = _saved.pop(id(mod), None)
    if entry is not None:
        _, ar, art = entry
        mod.apply_right = ar
        mod.apply_right_transposed = art


def installed(mod=None) -> bool:
    mod = _module(mod)
    return mod.apply_right is gpu_apply_right
