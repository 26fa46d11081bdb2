"""FP8T container parity (tensor_io.hpp:18-45, tensor_io.cpp:47-192) -- CPU.

libfp8b200's native writer/reader against the reference's own tensor_io.cpp
(compiled into oracle/_ref): byte-identical files, cross reads, and the same
IoError messages for garbled files (test_tensor_io.cpp's cases and more).
Host-only code: no GPU needed.
"""
import os
import struct

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def F():
    import paper_1905_12334_b200 as F
    return F


def _qt(F, codes, shape, fmt, mode="nearest-even"):
    import torch
    from paper_1905_12334_b200 import _lib
    c = np.ascontiguousarray(np.asarray(codes, dtype=np.uint16).reshape(-1))
    t = torch.from_numpy(c.astype(np.uint8)) if fmt == "fp8" else torch.from_numpy(c.view(np.int16))
    return F.QuantizedTensor(t, list(shape), _lib.E5M2 if fmt == "fp8" else _lib.FP16,
                             F._MODE[mode], F.Counters("cpu"))


SHAPES = [[], [0], [7], [3, 5], [2, 3, 4], [1, 1, 1, 9]]


@pytest.mark.parametrize("shape", SHAPES, ids=str)
def test_fp32_byte_identical_and_cross_read(F, tmp_path, shape):
    rng = np.random.default_rng(len(shape))
    a = rng.standard_normal(int(np.prod(shape)) if shape else 1).astype(np.float32).reshape(shape)
    if a.size:
        a.reshape(-1)[0] = np.float32(-0.0)
        if a.size > 2:
            a.reshape(-1)[1] = np.inf
            a.reshape(-1)[2] = np.nan
    ours, theirs = tmp_path / "ours.fp8t", tmp_path / "ref.fp8t"
    F.save_tensor(ours, a)
    O.ref_fp8t_save_f32(theirs, a)
    assert ours.read_bytes() == theirs.read_bytes()
    back = O.ref_fp8t_load_f32(ours)
    assert list(back.shape) == list(shape)
    np.testing.assert_array_equal(back.view(np.uint32), a.view(np.uint32))
    mine = F.load_tensor_fp32(theirs, device="cpu").numpy()
    np.testing.assert_array_equal(mine.view(np.uint32), a.view(np.uint32))
    assert F.peek_tensor_dtype(ours) == "fp32"


@pytest.mark.parametrize("fmt", ["fp8", "fp16"])
@pytest.mark.parametrize("mode,tag", [("nearest-even", 1), ("stochastic", 2), ("truncate", 3)])
@pytest.mark.parametrize("shape", SHAPES[1:], ids=str)
def test_codes_byte_identical_and_cross_read(F, tmp_path, fmt, mode, tag, shape):
    rng = np.random.default_rng(7)
    n = int(np.prod(shape))
    codes = rng.integers(0, 256 if fmt == "fp8" else 65536, n).astype(np.uint16)
    ours, theirs = tmp_path / "ours.fp8t", tmp_path / "ref.fp8t"
    F.save_tensor(ours, _qt(F, codes, shape, fmt, mode))
    O.ref_fp8t_save_codes(theirs, codes, shape, fmt, tag)
    assert ours.read_bytes() == theirs.read_bytes()
    back, bfmt, bmode = O.ref_fp8t_load_codes(ours)
    assert bfmt == fmt and bmode == tag and list(back.shape) == list(shape)
    np.testing.assert_array_equal(back.reshape(-1), codes)
    q = F.load_tensor_codes(theirs, device="cpu")
    assert q.format == ("FP8" if fmt == "fp8" else "FP16") and q.mode == mode
    assert q.shape == list(shape)
    np.testing.assert_array_equal(q.codes_u16().reshape(-1), codes)
    assert F.peek_tensor_dtype(theirs) == fmt


def _header(dtype=1, rank=1, mode=1, version=1, dims=(4,)):
    return b"FP8T" + bytes([version, dtype, rank, mode]) + bytes(8) + b"".join(
        struct.pack(">Q", d) for d in dims)


GARBLED = [
    ("bad_magic", b"FP9T" + bytes(12)),
    ("short_magic", b"FP"),
    ("truncated_header", b"FP8T" + bytes([1, 1])),
    ("bad_version", _header(version=2)),
    ("bad_dtype", _header(dtype=3)),
    ("truncated_dims", _header(rank=2, dims=(4,))),
    ("truncated_codes", _header() + bytes(3)),
    ("truncated_fp32", _header(dtype=0) + bytes(15)),
    ("bad_mode_tag", _header(mode=9) + bytes(4)),
    ("fp32_as_codes", _header(dtype=0) + bytes(16)),
    ("codes_as_fp32", _header(dtype=1) + bytes(4)),
    # shape_numel (tensor.cpp:9-16): a negative dimension is rejected, also when
    # two of them multiply to a positive element count
    ("negative_dim", _header(rank=2, dims=(2**64 - 2, 3)) + bytes(6)),
    ("two_negative_dims", _header(rank=2, dims=(2**64 - 2, 2**64 - 2)) + bytes(4)),
    ("negative_dim_fp32", _header(dtype=0, rank=1, dims=(2**64 - 1,))),
]


@pytest.mark.parametrize("name,blob", GARBLED, ids=[g[0] for g in GARBLED])
def test_garbled_files_same_ioerror(F, tmp_path, name, blob):
    p = tmp_path / f"{name}.fp8t"
    p.write_bytes(blob)
    want_fp32 = name in ("truncated_fp32", "codes_as_fp32", "negative_dim_fp32")
    ref_load = O.ref_fp8t_load_f32 if want_fp32 else O.ref_fp8t_load_codes
    our_load = F.load_tensor_fp32 if want_fp32 else F.load_tensor_codes
    with pytest.raises(O.RefIoError) as r:
        ref_load(p)
    with pytest.raises(F.IoError) as o:
        our_load(p, device="cpu")
    assert str(o.value) == str(r.value)


def test_missing_file(F, tmp_path):
    p = tmp_path / "nope.fp8t"
    with pytest.raises(O.RefIoError) as r:
        O.ref_fp8t_load_codes(p)
    with pytest.raises(F.IoError) as o:
        F.load_tensor_codes(p, device="cpu")
    assert str(o.value) == str(r.value)
    with pytest.raises(F.IoError, match="cannot open for writing"):
        F.save_tensor(os.path.join(str(tmp_path), "no_dir", "x.fp8t"), np.zeros(2, np.float32))


def test_huge_dims_fail_cleanly(F, tmp_path):
    """A header whose dimension product overflows is an IoError, not an abort
    across the C ABI; saving with a negative dimension is refused the same way."""
    import ctypes as C
    from paper_1905_12334_b200 import _lib
    p = tmp_path / "huge.fp8t"
    p.write_bytes(_header(rank=3, dims=(2**40, 2**40, 2**40)) + bytes(8))
    with pytest.raises(F.IoError, match="overflows"):
        F.load_tensor_codes(p, device="cpu")
    dims = (C.c_int64 * 2)(-1, 2)
    buf = np.zeros(4, np.float32)
    with pytest.raises(F.IoError, match="negative dimension"):
        _lib.check(_lib.LIB.fp8b_fp8t_save(str(tmp_path / "neg.fp8t").encode(), _lib.FP8T_F32, 0,
                                           2, dims, buf.ctypes.data))
