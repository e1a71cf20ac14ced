"""The C-ABI library loads and exports every symbol include/hsk.h declares.

CPU-only: no compute calls that need a device.  The entry points validate
their arguments on the host before touching CUDA, so the reference's error
behaviour (ValueError on shape mismatch) is checked here too.
"""

import ctypes
import os
import re

import pytest

from paper_2302_01977_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    with open(os.path.join(ROOT, "include", "hsk.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(hsk_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert _declared() == sorted(_lib.exported_symbols())


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.hsk_abi_version() == 1


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_plan_bytes_is_host_only_and_validates():
    lib = _lib.load()
    b1 = lib.hsk_sjlt_plan_bytes(4096, 256, 4)
    b2 = lib.hsk_sjlt_plan_bytes(8192, 256, 4)
    assert 0 < b1 < b2
    assert lib.hsk_sjlt_plan_bytes(4096, 0, 4) == _lib.HSK_EINVAL
    assert lib.hsk_sjlt_plan_bytes(4096, 256, 0) == _lib.HSK_EINVAL


def test_chunked_plan_flag():
    """HSK_SJLT_CHUNKED changes the plan only for the paired shapes (d/alpha
    = 8, d a multiple of 64); unknown flags are rejected on the host."""
    lib = _lib.load()
    assert lib.hsk_sjlt_plan_bytes_ex(16384, 512, 4, 1) == lib.hsk_sjlt_plan_bytes(16384, 512, 4)
    assert lib.hsk_sjlt_plan_bytes_ex(65536, 64, 8, 0) == lib.hsk_sjlt_plan_bytes(65536, 64, 8)
    paired = lib.hsk_sjlt_plan_bytes_ex(65536, 64, 8, 1)
    assert 0 < paired < lib.hsk_sjlt_plan_bytes(65536, 64, 8)  # alpha/2 entries per index
    assert lib.hsk_sjlt_plan_bytes_ex(65536, 64, 8, 2) == _lib.HSK_EINVAL
    rc = lib.hsk_sjlt_apply_ex(None, 5, 12, 5, 0, None, 12, 64, 8, 4, 0.5, None, 5, 0, None)
    assert rc == _lib.HSK_EINVAL and "unknown flags" in _lib.last_error()


def test_apply_dimension_mismatch_is_einval():
    lib = _lib.load()
    # S = A R^T needs cols == n: 10 columns vs an operator over 12
    rc = lib.hsk_sjlt_apply(None, 5, 10, 5, 0, None, 12, 4, 2, 0.5, None, 5, 0, None)
    assert rc == _lib.HSK_EINVAL
    assert "operator is over dimension 12" in _lib.last_error()
    with pytest.raises(ValueError):
        _lib.check(rc)
    rc = lib.hsk_gauss_apply(None, 9, 3, 9, 1, None, 8, 4, None, 3, 0, None)
    assert rc == _lib.HSK_EINVAL
    rc = lib.hsk_srht_apply(None, 4, 6, 4, 0, None, 6, 6, None, 2, 1.0, None, 4, 0, None)
    assert rc == _lib.HSK_EINVAL  # n_pad not a power of two
    rc = lib.hsk_fwht(None, 1, 6, 1, None)
    assert rc == _lib.HSK_EINVAL


def test_bad_trans_and_lda_rejected():
    lib = _lib.load()
    assert lib.hsk_sjlt_apply(None, 4, 4, 4, 2, None, 4, 4, 2, 0.5, None, 4, 0, None) == _lib.HSK_EINVAL
    assert lib.hsk_gauss_apply(None, 4, 4, 3, 0, None, 4, 4, None, 4, 0, None) == _lib.HSK_EINVAL


def test_oracle_library_exports():
    from oracle import oracle as O
    lib = O.lib()
    for name in ("oracle_sjlt_right", "oracle_sjlt_right_t", "oracle_srht", "oracle_gauss",
                 "oracle_fwht", "oracle_reduceat_segment"):
        assert hasattr(lib, name)
    assert isinstance(lib, ctypes.CDLL)


def test_chunked_flag_host_rule():
    """device.sjlt_chunked: only the paired shapes, trusted for the reference's
    block construction, checked on the pattern otherwise."""
    import numpy as np
    from paper_2302_01977_b200 import device, operators
    blk = operators.new_operator("sjlt", 300, 64, seed=1, alpha=8, construction="block").blocks[0]
    pos = np.asarray(blk._pos)
    assert device.sjlt_chunked(pos, 64, 8, "block")
    assert device.sjlt_chunked(pos, 64, 8, None)
    bad = pos.copy()
    bad[5, [0, 1]] = bad[5, [1, 0]]
    assert not device.sjlt_chunked(bad, 64, 8, "graph")
    b2 = operators.new_operator("sjlt", 600, 512, seed=1, alpha=4, construction="block").blocks[0]
    assert not device.sjlt_chunked(np.asarray(b2._pos), 512, 4, "block")  # not a paired shape


def test_plan_geometry_sweep_host_only():
    """hsk_sjlt_plan_bytes_ex walks the chunk / tile-layout rules (geom_dir,
    xp_rule, the TK fits) on the host: over a sweep of operator shapes --
    including huge alpha, one-bucket operators and every HSK_SJLT_XP setting --
    it returns a size that holds both directions' entry words and never less
    than one 4-byte word per entry, and the tuning generation counts reloads."""
    import os
    lib = _lib.load()
    gen0 = lib.hsk_tuning_generation()
    shapes = [(n, d, a) for n in (1, 17, 4096, 8192, 70000)
              for d in (1, 2, 64, 65, 128, 129, 256, 257, 384, 512, 513, 2048, 4096)
              for a in (1, 2, 3, 4, 8, 64, 4096) if a <= d]
    saved = os.environ.get("HSK_SJLT_XP")
    try:
        for xp in (None, "0", "1"):
            if xp is None:
                os.environ.pop("HSK_SJLT_XP", None)
            else:
                os.environ["HSK_SJLT_XP"] = xp
            assert lib.hsk_tuning_reload() == 0
            for n, d, a in shapes:
                for flags in (0, 1):
                    nbytes = lib.hsk_sjlt_plan_bytes_ex(n, d, a, flags)
                    paired = flags and d % 64 == 0 and a * 8 == d
                    per_dir = n * (a // 2 if paired else a) * 4
                    assert nbytes >= 2 * per_dir, (xp, n, d, a, flags, nbytes)
                    assert nbytes <= 2 * (8 * per_dir + 64 * (n + 4096) + (1 << 22)), (xp, n, d, a, flags, nbytes)
    finally:
        if saved is None:
            os.environ.pop("HSK_SJLT_XP", None)
        else:
            os.environ["HSK_SJLT_XP"] = saved
        lib.hsk_tuning_reload()
    assert lib.hsk_tuning_generation() == gen0 + 4
