"""GPU parity for gemm_fp8 (kernels.cpp:37-62).

* FP8B_GEMM_SEQUENTIAL is bitwise equal to the reference (same k-ascending
  FP32 running sum; products are exact).
* FP8B_GEMM_TENSOR (tcgen05) is checked against the exact sum with the stated
  tolerance |C - C_exact| <= tau * (|A||B|)_ij, tau = 1e-6, and its
  fused E5M2 outputs may differ from Q_RNE(C_ref) only by adjacent codes across
  a rounding midpoint (counted and reported).
"""
import json
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
GG = np.load(os.path.join(GOLD, "gemm_golden.npz"))
GMETA = json.load(open(os.path.join(GOLD, "gemm_golden.json")))
TAU = 1e-6


@pytest.fixture(scope="module")
def fp8():
    import paper_1905_12334_b200 as F
    F.init()
    return F


def _codes_dev(c, fmt):
    import torch
    c = np.ascontiguousarray(c)
    if fmt == "fp8":
        return torch.from_numpy(c.astype(np.uint8)).to("cuda")
    return torch.from_numpy(c.astype(np.uint16).view(np.int16)).to("cuda")


@pytest.mark.parametrize("m", GMETA, ids=lambda m: f"{m['m']}x{m['k']}x{m['n']}")
@pytest.mark.parametrize("fmt", ["fp8", "fp16"])
def test_sequential_engine_bitwise_golden(fp8, m, fmt):
    i = m["i"]
    a, b = _codes_dev(GG[f"a_{i}_{fmt}"], fmt), _codes_dev(GG[f"b_{i}_{fmt}"], fmt)
    c, _ = fp8.gemm_codes(a, b, m["m"], m["n"], m["k"], fmt, engine="sequential")
    np.testing.assert_array_equal(c.cpu().numpy().reshape(-1).view(np.uint32),
                                  GG[f"c_{i}_{fmt}"].reshape(-1).view(np.uint32))


def _rand_codes(rng, rows, cols, fmt, scale=1.0):
    x = (rng.standard_normal(rows * cols) * scale).astype(np.float32)
    c, _ = O.quantize(x, fmt)
    return c.reshape(rows, cols)


@pytest.mark.parametrize("a_major", ["k", "m"])
@pytest.mark.parametrize("b_major", ["n", "k"])
@pytest.mark.parametrize("fmt", ["fp8", "fp16"])
def test_layouts_sequential_bitwise(fp8, a_major, b_major, fmt):
    rng = np.random.default_rng(12)
    m, k, n = 96, 160, 72
    A = _rand_codes(rng, m, k, fmt)
    B = _rand_codes(rng, k, n, fmt)
    want = O.gemm(A, B, m, k, n, fmt)
    a_st = A if a_major == "k" else A.T.copy()
    b_st = B if b_major == "n" else B.T.copy()
    c, _ = fp8.gemm_codes(_codes_dev(a_st, fmt), _codes_dev(b_st, fmt), m, n, k, fmt,
                          a_major=a_major, b_major=b_major, engine="sequential")
    np.testing.assert_array_equal(c.cpu().numpy().view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("out_mode", ["nearest-even", "truncate", "stochastic"])
def test_fused_epilogue_sequential(fp8, out_mode):
    import torch
    rng = np.random.default_rng(13)
    m, k, n = 64, 128, 96
    A, B = _rand_codes(rng, m, k, "fp8"), _rand_codes(rng, k, n, "fp8")
    bias = rng.standard_normal(n).astype(np.float32)
    cnt = fp8.Counters()
    c, cq = fp8.gemm_codes(_codes_dev(A, "fp8"), _codes_dev(B, "fp8"), m, n, k, "fp8",
                           engine="sequential", bias=torch.from_numpy(bias).cuda(),
                           out_fmt="fp8", out_mode=out_mode, out_seed=17, out_counters=cnt)
    y = O.gemm(A, B, m, k, n, "fp8")
    y = (y + bias[None, :]).astype(np.float32)
    np.testing.assert_array_equal(c.cpu().numpy().view(np.uint32), y.view(np.uint32))
    codes, k_ = O.quantize(y, "fp8", out_mode, 17, bits="counter")
    np.testing.assert_array_equal(cq.cpu().numpy(), codes.astype(np.uint8))
    assert cnt.values() == tuple(int(v) for v in k_)


def _tolerance_check(c_gpu, A, B, m, k, n, fmt):
    exact, absdot = O.gemm_exact(A, B, m, k, n, fmt)
    err = np.abs(c_gpu.astype(np.float64) - exact)
    bound = TAU * absdot + 1e-30
    assert (err <= bound).all(), float((err / np.maximum(absdot, 1e-30)).max())
    return float((err / np.maximum(absdot, 1e-30)).max())


@pytest.mark.parametrize("shape", [(128, 256, 128), (256, 512, 256), (200, 96, 136),
                                   (512, 1024, 1024), (1, 64, 16), (130, 48, 40)])
@pytest.mark.parametrize("a_major,b_major", [("k", "n"), ("k", "k"), ("m", "n")])
def test_tensor_engine_tolerance(fp8, shape, a_major, b_major):
    rng = np.random.default_rng(sum(shape))
    m, k, n = shape
    A, B = _rand_codes(rng, m, k, "fp8"), _rand_codes(rng, k, n, "fp8")
    a_st = A if a_major == "k" else A.T.copy()
    b_st = B if b_major == "n" else B.T.copy()
    ad, bd = _codes_dev(a_st, "fp8"), _codes_dev(b_st, "fp8")
    inner_ok = (m if a_major == "m" else k) % 16 == 0 and (n if b_major == "n" else k) % 16 == 0
    assert fp8.gemm_tensor_supported(ad, bd, m, n, k, "fp8", a_major, b_major) == inner_ok
    c, _ = fp8.gemm_codes(ad, bd, m, n, k, "fp8", a_major=a_major, b_major=b_major,
                          engine="tensor")
    _tolerance_check(c.cpu().numpy(), A, B, m, k, n, "fp8")


@pytest.mark.parametrize("shape", [(128, 128, 256), (256, 320, 128), (96, 64, 200)])
@pytest.mark.parametrize("a_major,b_major", [("k", "n"), ("k", "k"), ("m", "n")])
def test_tensor_engine_fp16_operands(fp8, shape, a_major, b_major):
    """FP16 x FP16 codes (the reference accepts them, kernels.cpp:9-13) on kind::f16."""
    rng = np.random.default_rng(sum(shape) + 1)
    m, k, n = shape
    A, B = _rand_codes(rng, m, k, "fp16"), _rand_codes(rng, k, n, "fp16")
    a_st = A if a_major == "k" else A.T.copy()
    b_st = B if b_major == "n" else B.T.copy()
    ad, bd = _codes_dev(a_st, "fp16"), _codes_dev(b_st, "fp16")
    assert fp8.gemm_tensor_supported(ad, bd, m, n, k, "fp16", a_major, b_major)
    c, _ = fp8.gemm_codes(ad, bd, m, n, k, "fp16", a_major=a_major, b_major=b_major,
                          engine="tensor")
    _tolerance_check(c.cpu().numpy(), A, B, m, k, n, "fp16")


@pytest.mark.parametrize("out_mode", ["nearest-even", "truncate", "stochastic"])
@pytest.mark.parametrize("out_fmt", ["fp8", "fp16"])
def test_tensor_engine_fused_epilogue(fp8, out_mode, out_fmt):
    """Bias + output Q node fused into the tcgen05 epilogue. Codes may differ
    from Q(C_seq) only where C_tensor and C_seq straddle a rounding boundary;
    with these small-K shapes the sums are exact, so codes must match exactly."""
    import torch
    rng = np.random.default_rng(5)
    m, k, n = 256, 64, 512
    # operands on a coarse grid so every partial sum is exact in FP32
    A = O.quantize((rng.integers(-4, 5, m * k) * 0.25).astype(np.float32))[0].reshape(m, k)
    B = O.quantize((rng.integers(-4, 5, k * n) * 0.5).astype(np.float32))[0].reshape(k, n)
    bias = (rng.integers(-8, 8, n) * 0.125).astype(np.float32)
    cnt = fp8.Counters()
    c, cq = fp8.gemm_codes(_codes_dev(A, "fp8"), _codes_dev(B, "fp8"), m, n, k, "fp8",
                           engine="tensor", bias=torch.from_numpy(bias).cuda(), out_fmt=out_fmt,
                           out_mode=out_mode, out_seed=9, out_counters=cnt)
    y = (O.gemm(A, B, m, k, n, "fp8") + bias[None, :]).astype(np.float32)
    np.testing.assert_array_equal(c.cpu().numpy(), y)
    codes, k_ = O.quantize(y * np.float32(3e-5), out_fmt, out_mode, 9, bits="counter")
    # scale into the underflow/subnormal range too: run again with a scaled bias-free GEMM
    codes, k_ = O.quantize(y, out_fmt, out_mode, 9, bits="counter")
    got = cq.cpu().numpy()
    got = got.view(np.uint16) if out_fmt == "fp16" else got
    np.testing.assert_array_equal(got, codes.astype(got.dtype))
    assert cnt.values() == tuple(int(v) for v in k_)


def test_tensor_vs_sequential_large(fp8):
    """2048^3 (config 3): tensor engine vs the bitwise-reference CUDA-core engine
    under tau, plus E5M2 output flips only at rounding midpoints."""
    import torch
    m = n = k = 2048
    x = torch.empty(m * k + k * n, dtype=torch.float32, device="cuda")
    fp8.fill_synthetic(x, "normal", 21, 1.0)
    qa = fp8.quantize(x[: m * k])
    qb = fp8.quantize(x[m * k:])
    ct, cqt = fp8.gemm_codes(qa.codes, qb.codes, m, n, k, "fp8", engine="tensor", out_fmt="fp8")
    cs, _ = fp8.gemm_codes(qa.codes, qb.codes, m, n, k, "fp8", engine="sequential")
    da = fp8.dequantize(qa).double().reshape(m, k)
    db = fp8.dequantize(qb).double().reshape(k, n)
    absdot = da.abs() @ db.abs()
    err_t = (ct.double() - da @ db).abs()
    err_s = (cs.double() - da @ db).abs()
    assert bool((err_t <= TAU * absdot + 1e-30).all())
    assert bool((err_s <= TAU * absdot + 1e-30).all())
    # E5M2 output codes: Q_RNE(C_seq) vs fused epilogue codes
    ref_codes = fp8.quantize(cs).codes
    diff = (cqt != ref_codes)
    nflip = int(diff.sum())
    if nflip:
        # every flip must be a neighbouring code whose midpoint separates C_gpu and C_seq
        idx = diff.nonzero().squeeze(1)
        a_ = fp8.dequantize(fp8.QuantizedTensor(cqt[idx], [idx.numel()], 0, 0, fp8.Counters()))
        b_ = fp8.dequantize(fp8.QuantizedTensor(ref_codes[idx], [idx.numel()], 0, 0, fp8.Counters()))
        mid = (a_.double() + b_.double()) / 2
        cg, cr = ct.reshape(-1)[idx].double(), cs.reshape(-1)[idx].double()
        assert bool((((cg - mid) * (cr - mid)) <= 0).all())
    assert nflip <= m * n * 1e-4


@pytest.fixture
def splitk_env():
    old = os.environ.get("FP8B_GEMM_SPLITK")
    yield
    if old is None:
        os.environ.pop("FP8B_GEMM_SPLITK", None)
    else:
        os.environ["FP8B_GEMM_SPLITK"] = old


@pytest.mark.parametrize("splits", ["", "3", "7"])
@pytest.mark.parametrize("out_mode,out_fmt", [("nearest-even", "fp8"), ("truncate", "fp8"),
                                              ("stochastic", "fp8"), ("nearest-even", "fp16")])
@pytest.mark.parametrize("a_major", ["k", "m"])
def test_splitk_exact_grid(fp8, splitk_env, splits, out_mode, out_fmt, a_major):
    """Split-K (FP32 partials per K range -> fixed-order sum -> bias / C / fused
    Q node / counters): on a coarse operand grid every partial sum is exact, so
    C, the codes and the counters must equal the exact result bit for bit, with
    ragged K ranges (3, 7 splits) and the automatic choice (wgrad-like shape:
    small M x N, long K)."""
    import torch
    os.environ["FP8B_GEMM_SPLITK"] = splits
    rng = np.random.default_rng(31)
    m, k, n = 512, 8192, 768
    A = O.quantize((rng.integers(-4, 5, m * k) * 0.25).astype(np.float32))[0].reshape(m, k)
    B = O.quantize((rng.integers(-4, 5, k * n) * 0.5).astype(np.float32))[0].reshape(k, n)
    bias = (rng.integers(-8, 8, n) * 0.125).astype(np.float32)
    a_st = A if a_major == "k" else A.T.copy()
    cnt = fp8.Counters()
    c, cq = fp8.gemm_codes(_codes_dev(a_st, "fp8"), _codes_dev(B, "fp8"), m, n, k, "fp8",
                           a_major=a_major, engine="tensor", bias=torch.from_numpy(bias).cuda(),
                           out_fmt=out_fmt, out_mode=out_mode, out_seed=9, out_counters=cnt)
    da = O.dequantize(A).astype(np.float64).reshape(m, k)
    db = O.dequantize(B).astype(np.float64).reshape(k, n)
    y = ((da @ db).astype(np.float32) + bias[None, :]).astype(np.float32)
    np.testing.assert_array_equal(c.cpu().numpy(), y)
    codes, k_ = O.quantize(y, out_fmt, out_mode, 9, bits="counter")
    got = cq.cpu().numpy()
    got = got.view(np.uint16) if out_fmt == "fp16" else got
    np.testing.assert_array_equal(got, codes.astype(got.dtype))
    assert cnt.values() == tuple(int(v) for v in k_)


@pytest.mark.parametrize("splits", ["", "5"])
def test_splitk_tolerance_long_k(fp8, splitk_env, splits):
    """Config-5 wgrad shape class (dW[512 x 1024] over 65536 tokens): split-K
    result within tau of the exact sum."""
    import torch
    os.environ["FP8B_GEMM_SPLITK"] = splits
    m, k, n = 512, 65536, 1024
    x = torch.empty(m * k + k * n, dtype=torch.float32, device="cuda")
    fp8.fill_synthetic(x, "normal", 41, 1.0)
    qa = fp8.quantize(x[: m * k])
    qb = fp8.quantize(x[m * k:])
    # A stored [K, M] (MN-major): X^T of a [tokens, features] activation
    c, _ = fp8.gemm_codes(qa.codes, qb.codes, m, n, k, "fp8", a_major="m", engine="tensor")
    da = fp8.dequantize(qa).double().reshape(k, m).t()
    db = fp8.dequantize(qb).double().reshape(k, n)
    ex = da @ db
    absdot = da.abs() @ db.abs()
    assert bool(((c.double() - ex).abs() <= TAU * absdot + 1e-30).all())


@pytest.fixture
def nb_env():
    old = {k: os.environ.get(k) for k in ("FP8B_GEMM_NB",)}
    yield
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


@pytest.mark.parametrize("m,k,n,nb", [(512, 8192, 1024, "2"), (768, 512, 1280, ""),
                                      (256, 2048, 512, "1")])
def test_lean_codes_only_exact_grid(fp8, nb_env, m, k, n, nb):
    """The LEAN kernels (fused E5M2 RNE output only, no FP32 C; 256x512 and
    256x256 pair tiles): on an exact operand grid the codes and all three
    counters must equal Q_RNE of the exact result, with bias columns that force
    overflow (> 57344), underflow (tiny nonzero outputs) and NaN."""
    import torch
    os.environ["FP8B_GEMM_NB"] = nb
    rng = np.random.default_rng(77)
    A = O.quantize((rng.integers(-2, 3, m * k) * 0.5).astype(np.float32))[0].reshape(m, k)
    B = O.quantize((rng.integers(-2, 3, k * n) * 0.25).astype(np.float32))[0].reshape(k, n)
    B[:, 5::97] = 0  # zero columns: output = bias exactly
    bias = (rng.integers(-8, 8, n) * 0.125).astype(np.float32)
    bias[3::61] = 60000.0
    bias[5::97] = 1e-6
    bias[7::211] = np.nan
    cnt = fp8.Counters()
    _, cq = fp8.gemm_codes(_codes_dev(A, "fp8"), _codes_dev(B, "fp8"), m, n, k, "fp8",
                           engine="tensor", want_c=False, bias=torch.from_numpy(bias).cuda(),
                           out_fmt="fp8", out_mode="nearest-even", out_counters=cnt)
    da = O.dequantize(A).astype(np.float64).reshape(m, k)
    db = O.dequantize(B).astype(np.float64).reshape(k, n)
    y = ((da @ db).astype(np.float32) + bias[None, :]).astype(np.float32)
    codes, k_ = O.quantize(y, "fp8", "nearest-even", 1)
    np.testing.assert_array_equal(cq.cpu().numpy(), codes.astype(np.uint8))
    assert cnt.values() == tuple(int(v) for v in k_)
    assert k_[0] > 0 and k_[1] > 0 and k_[2] > 0


@pytest.mark.parametrize("b_major", ["n", "k"])
@pytest.mark.parametrize("m,k,n", [(40000, 320, 1000), (5000, 512, 256)])
def test_astat_codes_exact_grid(fp8, nb_env, b_major, m, k, n):
    """The A-stationary short-K pair kernel (resident A k-blocks, B-only ring;
    forced with FP8B_GEMM_AST=1): ragged M / N / K, several M blocks per cluster,
    both B layouts; codes and counters equal Q_RNE of the exact result, with
    overflow / underflow / NaN bias columns."""
    import torch
    old = os.environ.get("FP8B_GEMM_AST")
    os.environ["FP8B_GEMM_AST"] = "1"
    try:
        rng = np.random.default_rng(91)
        A = O.quantize((rng.integers(-2, 3, m * k) * 0.5).astype(np.float32))[0].reshape(m, k)
        B = O.quantize((rng.integers(-2, 3, k * n) * 0.25).astype(np.float32))[0].reshape(k, n)
        B[:, 5::97] = 0
        bias = (rng.integers(-8, 8, n) * 0.125).astype(np.float32)
        bias[3::61] = 60000.0
        bias[5::97] = 1e-6
        bias[7::211] = np.nan
        bdev = B if b_major == "n" else np.ascontiguousarray(B.T)
        cnt = fp8.Counters()
        _, cq = fp8.gemm_codes(_codes_dev(A, "fp8"), _codes_dev(bdev, "fp8"), m, n, k, "fp8",
                               b_major=b_major, engine="tensor", want_c=False,
                               bias=torch.from_numpy(bias).cuda(), out_fmt="fp8",
                               out_mode="nearest-even", out_counters=cnt)
        da = O.dequantize(A).astype(np.float64).reshape(m, k)
        db = O.dequantize(B).astype(np.float64).reshape(k, n)
        y = ((da @ db).astype(np.float32) + bias[None, :]).astype(np.float32)
        codes, k_ = O.quantize(y, "fp8", "nearest-even", 1)
        np.testing.assert_array_equal(cq.cpu().numpy().reshape(-1), codes.astype(np.uint8).reshape(-1))
        assert cnt.values() == tuple(int(v) for v in k_)
    finally:
        if old is None:
            os.environ.pop("FP8B_GEMM_AST", None)
        else:
            os.environ["FP8B_GEMM_AST"] = old



@pytest.mark.parametrize("b_major", ["n", "k"])
@pytest.mark.parametrize("m,k,n", [(3000, 64, 256), (1500, 256, 1000), (777, 96, 320)])
def test_short_k_16_warp_epilogue_exact_grid(fp8, b_major, m, k, n):
    """K <= 256 with codes-only E5M2 output takes the 256x256 pair kernel with 16
    epilogue warps (the 1x1 conv fprop / dgrad shapes): ragged M / N / K, both B
    layouts; codes and counters equal Q_RNE of the exact result, with overflow /
    underflow / NaN bias columns."""
    import torch
    rng = np.random.default_rng(123)
    A = O.quantize((rng.integers(-2, 3, m * k) * 0.5).astype(np.float32))[0].reshape(m, k)
    B = O.quantize((rng.integers(-2, 3, k * n) * 0.25).astype(np.float32))[0].reshape(k, n)
    B[:, 5::97] = 0
    bias = (rng.integers(-8, 8, n) * 0.125).astype(np.float32)
    bias[3::61] = 60000.0
    bias[5::97] = 1e-6
    bias[7::211] = np.nan
    bdev = B if b_major == "n" else np.ascontiguousarray(B.T)
    cnt = fp8.Counters()
    _, cq = fp8.gemm_codes(_codes_dev(A, "fp8"), _codes_dev(bdev, "fp8"), m, n, k, "fp8",
                           b_major=b_major, engine="tensor", want_c=False,
                           bias=torch.from_numpy(bias).cuda(), out_fmt="fp8",
                           out_mode="nearest-even", out_counters=cnt)
    da = O.dequantize(A).astype(np.float64).reshape(m, k)
    db = O.dequantize(B).astype(np.float64).reshape(k, n)
    y = ((da @ db).astype(np.float32) + bias[None, :]).astype(np.float32)
    codes, k_ = O.quantize(y, "fp8", "nearest-even", 1)
    np.testing.assert_array_equal(cq.cpu().numpy().reshape(-1), codes.astype(np.uint8).reshape(-1))
    assert cnt.values() == tuple(int(v) for v in k_)
    assert k_[0] > 0 and k_[1] > 0 and k_[2] > 0

@pytest.mark.parametrize("n,b_major", [(2048, "n"), (1536, "k"), (32000, "n")])
def test_astat_equals_streaming_at_config5_size(fp8, n, b_major):
    """Config-5 fprop shapes at full size (2^20 tokens x 512 -> n): the
    A-stationary kernel and the streaming pair kernel issue the same MMAs in the
    same K order, so codes and counters must be identical bit for bit."""
    import torch
    T, k = 1 << 20, 512
    if n == 32000:
        T = 1 << 17  # 4 GB of output codes per run otherwise
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    a = torch.randint(0, 256, (T * k,), dtype=torch.uint8, device="cuda", generator=g)
    a[(a & 0x7F) >= 0x7C] = 0x3C  # finite codes only
    b = torch.randint(0, 0x40, (k * n,), dtype=torch.uint8, device="cuda", generator=g)
    b |= (torch.randint(0, 2, (k * n,), dtype=torch.uint8, device="cuda", generator=g) << 7)
    outs = []
    old = os.environ.get("FP8B_GEMM_AST")
    try:
        for mode in ("2", "0"):  # default selection (A-stationary here), streaming
            os.environ["FP8B_GEMM_AST"] = mode
            cnt = fp8.Counters()
            _, cq = fp8.gemm_codes(a, b, T, n, k, "fp8", b_major=b_major, engine="tensor",
                                   want_c=False, out_fmt="fp8", out_counters=cnt)
            outs.append((cq, cnt.values()))
    finally:
        if old is None:
            os.environ.pop("FP8B_GEMM_AST", None)
        else:
            os.environ["FP8B_GEMM_AST"] = old
    assert torch.equal(outs[0][0], outs[1][0])
    assert outs[0][1] == outs[1][1]


@pytest.mark.parametrize("c_off,q_off", [(1, 1), (2, 4), (3, 8), (0, 1), (1, 0)])
@pytest.mark.parametrize("out_fmt", ["fp8", "fp16"])
def test_tensor_engine_unaligned_outputs(fp8, c_off, q_off, out_fmt):
    """FP32 C and output codes written into views at element offsets that are
    not 16-byte aligned: TMA stores are off for them and the direct-store
    epilogue must not use vector stores (no misaligned-address fault); results
    equal the aligned call bit for bit."""
    import torch
    rng = np.random.default_rng(41)
    m, k, n = 256, 256, 512
    A, B = _rand_codes(rng, m, k, "fp8"), _rand_codes(rng, k, n, "fp8")
    ad, bd = _codes_dev(A, "fp8"), _codes_dev(B, "fp8")
    qdt = torch.uint8 if out_fmt == "fp8" else torch.int16
    c_ref, q_ref = fp8.gemm_codes(ad, bd, m, n, k, "fp8", engine="tensor", out_fmt=out_fmt)
    cbuf = torch.zeros(m * n + 8, dtype=torch.float32, device="cuda")
    qbuf = torch.zeros(m * n + 16, dtype=qdt, device="cuda")
    c = cbuf[c_off:c_off + m * n].view(m, n)
    cq = qbuf[q_off:q_off + m * n]
    fp8.gemm_codes(ad, bd, m, n, k, "fp8", engine="tensor", c=c, out_fmt=out_fmt, out_codes=cq)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(c.cpu().numpy().view(np.uint32), c_ref.cpu().numpy().view(np.uint32))
    np.testing.assert_array_equal(cq.cpu().numpy(), q_ref.cpu().numpy())
    # codes-only (the lean E5M2 epilogue) into a misaligned view
    cq2 = qbuf[q_off:q_off + m * n]
    cq2.zero_()
    fp8.gemm_codes(ad, bd, m, n, k, "fp8", engine="tensor", want_c=False, out_fmt=out_fmt,
                   out_codes=cq2)
    _, q_ref2 = fp8.gemm_codes(ad, bd, m, n, k, "fp8", engine="tensor", want_c=False,
                               out_fmt=out_fmt)
    np.testing.assert_array_equal(cq2.cpu().numpy(), q_ref2.cpu().numpy())
