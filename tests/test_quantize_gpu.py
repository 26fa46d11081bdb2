"""GPU parity: quantize / dequantize / transpose kernels vs the reference's golden
vectors and the CPU oracle, bit-exact (codes and counters)."""
import json
import math
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def fp8():
    import paper_1905_12334_b200 as F
    F.init()
    return F


def _f(v):
    return {"nan": math.nan, "inf": math.inf, "-inf": -math.inf}.get(v, v) if isinstance(v, str) else v


def test_known_answers(fp8):
    ka = json.load(open(os.path.join(GOLD, "known_answers.json")))
    for c in ka["encode"]:
        code, ovf, unf = fp8.encode(_f(c["x"]), c["fmt"], c["mode"], 1, bool(c["saturate"]))
        assert (code, int(ovf), int(unf)) == (c["code"], c["overflowed"], c["underflowed"]), c
    for c in ka["decode"]:
        v = fp8.decode(c["code"], c["fmt"])
        w = _f(c["value"])
        assert (math.isnan(v) and math.isnan(w)) or (v == w and math.copysign(1, v) == math.copysign(1, w)), c
    for c in ka["quantize"]:
        q = fp8.quantize(np.array([_f(v) for v in c["x"]], np.float32), c["fmt"],
                         saturate=bool(c["saturate"]))
        assert list(q.codes_u16()) == c["codes"]
        assert (q.overflow_count, q.underflow_count) == (c["overflow"], c["underflow"])


QG = np.load(os.path.join(GOLD, "quantize_golden.npz"))
QMETA = json.load(open(os.path.join(GOLD, "quantize_golden.json")))


@pytest.mark.parametrize("m", QMETA, ids=lambda m: m["key"])
def test_quantize_golden_streams(fp8, m):
    """GPU == fp8emu::quantize on 3 full 4096-blocks + a partial block, all modes,
    including the reference LFSR stochastic stream."""
    q = fp8.quantize(QG["x"], m["fmt"], m["mode"], int(m["seed"]), bool(m["saturate"]))
    np.testing.assert_array_equal(q.codes_u16(), QG[m["key"]])
    assert (q.overflow_count, q.underflow_count) == (m["overflow"], m["underflow"])
    assert q.nan_count == int(np.isnan(QG["x"]).sum())


def _config2(fp8, n, seed=0):
    import torch
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    fp8.fill_synthetic(x, "config2", seed, 0.01)
    return x


@pytest.mark.parametrize("fmt", ["fp8", "fp16"])
@pytest.mark.parametrize("mode,bits", [("nearest-even", "lfsr"), ("truncate", "lfsr"),
                                       ("stochastic", "lfsr"), ("stochastic", "counter")])
@pytest.mark.parametrize("sat", [False, True])
def test_quantize_vs_oracle_config2(fp8, fmt, mode, bits, sat):
    n = (1 << 20) + 4096 * 3 + 777  # many blocks + ragged tail
    x = _config2(fp8, n, seed=5)
    q = fp8.quantize(x, fmt, mode, 1234567, sat, bits=bits)
    xh = x.cpu().numpy()
    codes, cnt = O.quantize(xh, fmt, mode, 1234567, sat, bits=bits)
    np.testing.assert_array_equal(q.codes_u16(), codes)
    assert q.counters.values() == tuple(int(v) for v in cnt)


def test_supplied_bits(fp8):
    import torch
    n = 300001
    x = _config2(fp8, n, 7)
    rb = torch.randint(-2 ** 31, 2 ** 31 - 1, (n,), dtype=torch.int32, device="cuda")
    for fmt in ("fp8", "fp16"):
        q = fp8.quantize(x, fmt, "stochastic", 9, bits="supplied", rbits=rb)
        codes, cnt = O.quantize(x.cpu().numpy(), fmt, "stochastic", 9, bits="supplied",
                                rbits=rb.cpu().numpy().view(np.uint32))
        np.testing.assert_array_equal(q.codes_u16(), codes)
        assert q.counters.values() == tuple(int(v) for v in cnt)


@pytest.mark.parametrize("fmt", ["fp8", "fp16"])
def test_sr_all_bit_patterns_supplied_bits(fp8, fmt):
    """Uniformly random FP32 bit patterns (every exponent, NaN/Inf, denormals)
    with random supplied bits: the carry-add SR kernels == the oracle's
    reference-derived rule; saturate on and off."""
    import torch
    n = 1 << 20
    rng = np.random.default_rng(17)
    bits = rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
    rb = rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
    x = torch.from_numpy(bits.view(np.float32)).cuda()
    rbt = torch.from_numpy(rb.view(np.int32)).cuda()
    for sat in (False, True):
        for mode in ("stochastic", "truncate"):
            q = fp8.quantize(x, fmt, mode, 3, sat, bits="supplied", rbits=rbt)
            codes, cnt = O.quantize(bits.view(np.float32), fmt, mode, 3, sat, bits="supplied",
                                    rbits=rb)
            np.testing.assert_array_equal(q.codes_u16(), codes)
            assert q.counters.values() == tuple(int(v) for v in cnt)
        q = fp8.quantize(x, fmt, "stochastic", 3, sat, bits="lfsr")
        codes, cnt = O.quantize(bits.view(np.float32), fmt, "stochastic", 3, sat, bits="lfsr")
        np.testing.assert_array_equal(q.codes_u16(), codes)
        assert q.counters.values() == tuple(int(v) for v in cnt)


def test_block_offset_sharding(fp8):
    """A rank holding blocks [b0, b1) with block_offset=b0 reproduces its slice
    of the whole-tensor SR codes."""
    n = 4096 * 40
    x = _config2(fp8, n, 3)
    whole = fp8.quantize(x, "fp8", "stochastic", 77).codes_u16()
    for b0, b1 in [(0, 13), (13, 27), (27, 40)]:
        part = fp8.quantize(x[b0 * 4096:b1 * 4096], "fp8", "stochastic", 77, block_offset=b0)
        np.testing.assert_array_equal(part.codes_u16(), whole[b0 * 4096:b1 * 4096])


@pytest.mark.parametrize("n", [1, 3, 4, 4095, 4096, 4097, 12345])
@pytest.mark.parametrize("mode", ["nearest-even", "stochastic"])
def test_ragged_and_unaligned(fp8, n, mode):
    import torch
    base = _config2(fp8, n + 3, 11)
    for off in (0, 1, 3):  # off != 0 -> misaligned pointers take the scalar path
        x = base[off:off + n]
        q = fp8.quantize(x, "fp8", mode, 5)
        codes, cnt = O.quantize(x.cpu().numpy(), "fp8", mode, 5)
        np.testing.assert_array_equal(q.codes_u16(), codes)
        assert q.counters.values() == tuple(int(v) for v in cnt)


def test_empty(fp8):
    q = fp8.quantize(np.zeros(0, np.float32), "fp8")
    assert q.codes.numel() == 0 and q.overflow_count == 0


def test_zero_seed_raises(fp8):
    with pytest.raises(ValueError):
        fp8.quantize(np.ones(4, np.float32), "fp8", "stochastic", 0)


@pytest.mark.parametrize("fmt", ["fp8", "fp16"])
def test_dequantize_all_codes(fp8, fmt):
    import torch
    ncodes = 256 if fmt == "fp8" else 65536
    dt = torch.uint8 if fmt == "fp8" else torch.int16
    codes = torch.arange(ncodes, dtype=torch.int32, device="cuda").to(dt)
    q = fp8.QuantizedTensor(codes, [ncodes], 0 if fmt == "fp8" else 1, 0, fp8.Counters())
    got = fp8.dequantize(q).cpu().numpy()
    want = O.dequantize(np.arange(ncodes, dtype=np.uint16), fmt)
    # bitwise, NaN included: every NaN code decodes to the reference's 0x7FC00000
    np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))


def test_roundtrip_all_finite_codes(fp8):
    """bindings test_smoke.py:23-30 / test_float_format.cpp:148-162."""
    vals = np.array([O.decode(c) for c in range(256)], dtype=np.float32)
    fin = vals[np.isfinite(vals)]
    for mode in ("nearest-even", "truncate", "stochastic"):
        q = fp8.quantize(fin, "fp8", mode, 3)
        assert q.overflow_count == 0
        np.testing.assert_array_equal(fp8.dequantize(q).cpu().numpy().view(np.uint32),
                                      fin.view(np.uint32))


def test_transpose(fp8):
    x = np.arange(6, dtype=np.float32).reshape(2, 3) + 1
    qt = fp8.transpose(fp8.quantize(x))
    assert qt.shape == [3, 2]
    np.testing.assert_array_equal(fp8.dequantize(qt).cpu().numpy(), x.T)


@pytest.mark.slow
@pytest.mark.parametrize("fmt", ["fp8", "fp16"])
@pytest.mark.parametrize("sat", [False, True])
def test_exhaustive_rne_vs_torch_cast(fp8, fmt, sat):
    """All 2^32 FP32 inputs: the RNE kernel equals PyTorch's own float->fp8/fp16
    cast (an independent IEEE RNE) after the reference's two documented
    deviations from IEEE: |x| > max normal overflows (Inf, or the
    max code when saturating) and NaN is the canonical unsigned NaN. Counters
    are checked against the same independent derivation."""
    import torch
    chunk = 1 << 28
    maxbits = 0x47600000 if fmt == "fp8" else 0x477FE000
    signbit = 0x80 if fmt == "fp8" else 0x8000
    inf, mx, nanc = (0x7C, 0x7B, 0x7E) if fmt == "fp8" else (0x7C00, 0x7BFF, 0x7E00)
    tdt = torch.float8_e5m2 if fmt == "fp8" else torch.float16
    cnt = fp8.Counters()
    exp_ovf = exp_unf = exp_nan = 0
    for c0 in range(0, 1 << 32, chunk):
        bits = torch.arange(c0, c0 + chunk, dtype=torch.int64, device="cuda").to(torch.int32)
        x = bits.view(torch.float32)
        q = fp8.quantize(x, fmt, "nearest-even", 1, sat, counters=cnt)
        got = q.codes.to(torch.int32) & (0xFF if fmt == "fp8" else 0xFFFF)
        hw = x.to(tdt).view(torch.uint8 if fmt == "fp8" else torch.int16).to(torch.int32)
        hw = hw & (0xFF if fmt == "fp8" else 0xFFFF)
        a = bits & 0x7FFFFFFF
        isnan = a > 0x7F800000
        big = (a > maxbits) & ~isnan
        neg = bits < 0
        ovcode = torch.where(neg, torch.full_like(hw, signbit), torch.zeros_like(hw)) | (mx if sat else inf)
        want = torch.where(big, ovcode, hw)
        want = torch.where(isnan, torch.full_like(hw, nanc), want)
        bad = int((got != want).sum())
        assert bad == 0, (fmt, sat, hex(c0), bad)
        mag = want & (signbit - 1)
        exp_ovf += int(big.sum())
        exp_nan += int(isnan.sum())
        exp_unf += int(((mag == 0) & (a != 0) & ~isnan & ~big).sum())
        del bits, x, q, got, hw, want
    assert cnt.values() == (exp_ovf, exp_unf, exp_nan)


@pytest.mark.slow
@pytest.mark.parametrize("fmt", ["fp8", "fp16"])
def test_exhaustive_fast_paths_vs_scalar_rule(fp8, fmt):
    """All 2^32 FP32 inputs: the vectorised SR/TRUNC kernels (packed carry-add
    representation) and the TMA-staged LFSR kernel equal the scalar integer
    rule (encode_int, SURVEY A2', itself pinned to the oracle above), which the
    library runs for misaligned buffers. Codes and counters."""
    import torch
    chunk = 1 << 28
    buf = torch.empty(chunk + 4, dtype=torch.float32, device="cuda")
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1)
    for c0 in range(0, 1 << 32, chunk):
        bits = torch.arange(c0, c0 + chunk, dtype=torch.int64, device="cuda").to(torch.int32)
        x = bits.view(torch.float32)
        buf[1:chunk + 1].copy_(x)
        xu = buf[1:chunk + 1]  # misaligned view -> scalar path
        rb = torch.randint(-2 ** 31, 2 ** 31 - 1, (chunk,), dtype=torch.int32, device="cuda",
                           generator=gen)
        for mode, bits_src in [("stochastic", "supplied"), ("truncate", "lfsr"),
                               ("stochastic", "lfsr"), ("stochastic", "counter")]:
            for sat in (False, True):
                ca, cb = fp8.Counters(), fp8.Counters()
                qa = fp8.quantize(x, fmt, mode, 11, sat, bits=bits_src,
                                  rbits=rb if bits_src == "supplied" else None, counters=ca)
                qb = fp8.quantize(xu, fmt, mode, 11, sat, bits=bits_src,
                                  rbits=rb if bits_src == "supplied" else None, counters=cb)
                bad = int((qa.codes != qb.codes).sum())
                assert bad == 0, (fmt, mode, bits_src, sat, hex(c0), bad)
                assert ca.values() == cb.values(), (fmt, mode, bits_src, sat, hex(c0))
        del bits, x, rb, qa, qb


@pytest.mark.parametrize("fmt", ["fp8", "fp16"])
@pytest.mark.parametrize("off", [1, 2, 4, 8])
@pytest.mark.parametrize("mode,bits", [("stochastic", "lfsr"), ("nearest-even", "lfsr"),
                                       ("stochastic", "counter"), ("truncate", "lfsr")])
def test_unaligned_codes_output(fp8, fmt, off, mode, bits):
    """Codes written into a view at any element offset (out=buf[off:]): the
    vector-store kernels are only chosen when the output base allows their
    8/16-byte stores; results equal the oracle either way."""
    import torch
    n = 4096 * 5 + 100
    x = _config2(fp8, n, 13)
    dt = torch.uint8 if fmt == "fp8" else torch.int16
    buf = torch.zeros(n + 16, dtype=dt, device="cuda")
    q = fp8.quantize(x, fmt, mode, 5, bits=bits, out=buf[off:off + n])
    torch.cuda.synchronize()
    codes, cnt = O.quantize(x.cpu().numpy(), fmt, mode, 5, bits=bits)
    np.testing.assert_array_equal(q.codes_u16(), codes)
    assert q.counters.values() == tuple(int(v) for v in cnt)
    # the guard bytes around the view are untouched
    assert int(buf[:off].abs().sum()) == 0 and int(buf[off + n:].abs().sum()) == 0
