"""`.hssd` files straight into HBM (paper_2302_01977_b200.hssd).

The CPU tests restate the reference's file tests (hsskit tests/test_matgen.py:
120-162: round trip, error class, bad magic, truncated header, truncated
payload, oversized header) against the device loader's validation, which runs
before anything touches a GPU; the GPU test streams a multi-slab file with an
odd row count into a DeviceMatrix and sketches it in place."""

import struct

import numpy as np
import pytest

from paper_2302_01977_b200 import hssd


def test_file_error_class():
    assert issubclass(hssd.FileFormatError, TypeError)


def test_header_roundtrip(tmp_path):
    A = np.random.default_rng(5).standard_normal((7, 5))
    path = tmp_path / "m.hssd"
    hssd.write_file(path, A)
    assert hssd.read_header(path) == (7, 5)
    raw = path.read_bytes()
    assert raw[:4] == b"HSSD" and struct.unpack("<QQ", raw[4:20]) == (7, 5)
    np.testing.assert_array_equal(np.frombuffer(raw[20:], "<f8").reshape((7, 5), order="F"), A)


def test_file_bad_magic(tmp_path):
    path = tmp_path / "bad.hssd"
    path.write_bytes(b"NOPE" + b"\x00" * 24)
    with pytest.raises(hssd.FileFormatError, match="HSSD"):
        hssd.from_file(path)


def test_file_truncated_header(tmp_path):
    path = tmp_path / "short.hssd"
    path.write_bytes(b"HSSD\x01\x00")
    with pytest.raises(hssd.FileFormatError, match="truncated header"):
        hssd.from_file(path)


def test_file_truncated_payload(tmp_path):
    path = tmp_path / "trunc.hssd"
    path.write_bytes(b"HSSD" + struct.pack("<QQ", 4, 4) + np.ones(15).tobytes())
    with pytest.raises(hssd.FileFormatError, match="truncat") as ei:
        hssd.from_file(path)
    assert "promises 16 values (128 bytes), file holds 120 bytes" in str(ei.value)


def test_file_oversized_header_rejected(tmp_path):
    path = tmp_path / "huge.hssd"
    path.write_bytes(b"HSSD" + struct.pack("<QQ", 2**40, 2**40))
    with pytest.raises(hssd.FileFormatError, match="overflow"):
        hssd.from_file(path)


@pytest.mark.gpu
def test_file_to_device_and_sketch(tmp_path, cuda):
    from oracle import oracle as O
    from paper_2302_01977_b200 import sketching as sk

    rng = np.random.default_rng(11)
    A = rng.standard_normal((301, 517))          # odd rows: padded leading dimension
    path = tmp_path / "a.hssd"
    hssd.write_file(path, A)
    acc = hssd.from_file(path, slab_bytes=301 * 8 * 37)  # 14 slabs through 2 buffers
    assert isinstance(acc, sk.DeviceAccessor) and acc.shape == (301, 517)
    np.testing.assert_array_equal(acc.dense(), A)
    np.testing.assert_array_equal(acc.extract([3, 0, 300], [516, 2]), A[np.ix_([3, 0, 300], [516, 2])])
    op = sk.new_operator(sk.SJLT, 517, 64, seed=1, alpha=4, construction=sk.BLOCK)
    assert O.rel_frobenius(sk.apply_right(acc, op), O.apply_right(A, op)) <= 1e-12
    op_t = sk.new_operator(sk.GAUSSIAN, 301, 32, seed=2)
    assert O.rel_frobenius(sk.apply_right_transposed(acc, op_t),
                           O.apply_right_transposed(A, op_t)) <= 1e-12
    empty = tmp_path / "e.hssd"
    hssd.write_file(empty, np.zeros((0, 3)))
    assert hssd.from_file(empty).shape == (0, 3)
