"""GPU parity for the weight-stationary halo-slab conv kernel (conv_halo.cu):
narrow NHWC stride-1 layers (C * bytes in {64, 128}, F <= 256), fprop and dgrad
(dgrad is fprop over E with the flipped weights).

On an exact operand grid (every partial sum exact in FP32) the halo kernel, the
im2col tensor kernel (FP8B_CONV_HALO=0) and the float64 reference agree bit for
bit -- FP32 output, fused output codes and the reference's counters -- so any
misplaced row shift, pad column or tile edge shows up as a hard mismatch."""
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fp8():
    import paper_1905_12334_b200 as F
    F.init()
    return F


@pytest.fixture
def env():
    keys = ("FP8B_CONV_HALO", "FP8B_CONV_WGRAD_BLOCK", "FP8B_CONV_1X1_WGRAD_PIX")
    old = {k: os.environ.get(k) for k in keys}
    yield os.environ
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def _qt(F, codes, shape, fmt):
    import torch
    from paper_1905_12334_b200 import _lib
    c = np.ascontiguousarray(codes).reshape(-1)
    if fmt == "fp8":
        t, fid = torch.from_numpy(c.astype(np.uint8)).to("cuda"), _lib.E5M2
    else:
        t, fid = torch.from_numpy(c.astype(np.uint16).view(np.int16)).to("cuda"), _lib.FP16
    return F.QuantizedTensor(t, list(shape), fid, _lib.RNE, F.Counters())


def _grid(rng, size, fmt, step):
    return O.quantize((rng.integers(-2, 3, size) * step).astype(np.float32), fmt)[0]


def _fwd_exact(x, w, k, pad):
    from numpy.lib.stride_tricks import sliding_window_view as swv
    xp = np.pad(x, ((0, 0), (pad, pad), (pad, pad), (0, 0)))
    win = swv(xp, (k, k), axis=(1, 2))
    return np.einsum("nhwcij,fijc->nhwf", win, w, optimize=True)


HALO_SHAPES = [  # n, c, h, w, f, k, pad, fmt
    (2, 64, 56, 56, 64, 3, 1, "fp8"),    # ResNet-50 3x3 @56 (R = 2 rows per tile)
    (2, 128, 28, 28, 128, 3, 1, "fp8"),  # 3x3 @28, 128-byte rows (R = 4)
    (3, 64, 13, 9, 48, 3, 1, "fp8"),     # F not a multiple of 64, ragged last tile
    (2, 64, 10, 17, 64, 5, 2, "fp8"),    # 5x5
    (2, 64, 9, 12, 80, 3, 0, "fp8"),     # no padding (OW = Wp - 2)
    (1, 128, 3, 126, 64, 3, 1, "fp8"),   # Wp = 128: one output row per tile
    (2, 32, 14, 14, 64, 3, 1, "fp16"),   # kind::f16, 64-byte rows
    (2, 64, 7, 7, 128, 3, 1, "fp16"),    # kind::f16, 128-byte rows
]


@pytest.mark.parametrize("shape", HALO_SHAPES, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("out", ["f32", "codes"])
def test_halo_exact_grid(fp8, env, shape, out):
    import torch
    n, c, h, w, f, k, pad, fmt = shape
    oh, ow = h + 2 * pad - k + 1, w + 2 * pad - k + 1
    rng = np.random.default_rng(n * 7 + c + f + k)
    xc = _grid(rng, n * h * w * c, fmt, 0.5).reshape(n, h, w, c)
    wc = _grid(rng, f * k * k * c, fmt, 0.25).reshape(f, k, k, c)
    ec = _grid(rng, n * oh * ow * f, fmt, 0.5).reshape(n, oh, ow, f)
    dec = lambda a: O.dequantize(a.reshape(-1), fmt).astype(np.float64).reshape(a.shape)
    wflip = np.ascontiguousarray(dec(wc)[:, ::-1, ::-1, :].transpose(3, 1, 2, 0))
    y_ex = _fwd_exact(dec(xc), dec(wc), k, pad).astype(np.float32)
    dx_ex = _fwd_exact(dec(ec), wflip, k, k - 1 - pad).astype(np.float32)
    X, W, E = (_qt(fp8, a, a.shape, fmt) for a in (xc, wc, ec))
    kw = dict(layout="nhwc", engine="tensor", out_fmt="fp8", out_mode="nearest-even")
    res = {}
    for halo in ("1", "0"):
        env["FP8B_CONV_HALO"] = halo
        cy, cdx = fp8.Counters(), fp8.Counters()
        y, qy = fp8.conv2d(X, W, 1, pad, out_counters=cy, want_y=out == "f32", **kw)
        dx, qdx = fp8.conv2d_backward_data(E, W, 1, pad, h, w, out_counters=cdx,
                                           want_y=out == "f32", **kw)
        torch.cuda.synchronize()
        res[halo] = (y, qy.codes.cpu().numpy(), cy.values(), dx, qdx.codes.cpu().numpy(), cdx.values())
    for name, ex, i in [("y", y_ex, 0), ("dx", dx_ex, 3)]:
        codes, cnt = O.quantize(ex.reshape(-1), "fp8", "nearest-even")
        for halo in ("1", "0"):
            got_t, got_q, got_c = res[halo][i], res[halo][i + 1], res[halo][i + 2]
            if out == "f32":
                np.testing.assert_array_equal(got_t.cpu().numpy().reshape(-1), ex.reshape(-1),
                                              err_msg=f"{name} halo={halo}")
            np.testing.assert_array_equal(got_q, codes.astype(np.uint8), err_msg=f"{name} halo={halo}")
            assert got_c == tuple(int(v) for v in cnt), (name, halo)


def test_halo_taken_for_resnet_layers(fp8):
    """The halo kernel covers the config-4 3x3 layers with 64 / 128 channels
    (fprop and dgrad), not the 256 / 512-channel ones."""
    for (c, hw) in [(64, 56), (128, 28)]:
        for kind in ("fprop", "dgrad"):
            assert fp8.conv_halo_supported(256, c, hw, hw, c, 3, 1, 1, "fp8", kind)
    assert not fp8.conv_halo_supported(256, 256, 14, 14, 256, 3, 1, 1, "fp8", "fprop")
    assert fp8.conv_halo_supported(256, 64, 56, 56, 64, 3, 1, 1, "fp8", "wgrad")
    assert not fp8.conv_halo_supported(256, 128, 28, 28, 128, 3, 1, 1, "fp8", "wgrad")
    assert not fp8.conv_halo_supported(2, 32, 14, 14, 32, 3, 1, 1, "fp16", "wgrad")
    for shape in HALO_SHAPES:
        n, c, h, w, f, k, pad, fmt = shape
        assert fp8.conv_halo_supported(n, c, h, w, f, k, 1, pad, fmt, "fprop"), shape


@pytest.mark.parametrize("shape", [(4, 256, 14, 14, 64), (2, 64, 7, 9, 512), (3, 128, 5, 6, 96),
                                   (2, 64, 12, 11, 256)], ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("out", ["f32", "codes"])
def test_1x1_gemm_route_exact(fp8, shape, out):
    """1x1 stride-1 fprop and dgrad routed to the pair-tile GEMM engine (y = x .
    w^T with w K-major, dx = e . w with w N-major) equal the im2col kernel and
    the exact result bit for bit on an exact operand grid, codes and counters
    included."""
    n, c, h, w, f = shape
    rng = np.random.default_rng(c + f)
    wc = _grid(rng, f * c, "fp8", 0.25).reshape(f, 1, 1, c)
    xc = _grid(rng, n * h * w * c, "fp8", 0.5).reshape(n, h, w, c)
    ec = _grid(rng, n * h * w * f, "fp8", 0.5).reshape(n, h, w, f)
    dec = lambda a: O.dequantize(a.reshape(-1), "fp8").astype(np.float64).reshape(a.shape)
    y_ex = np.einsum("nhwc,fc->nhwf", dec(xc), dec(wc).reshape(f, c)).astype(np.float32)
    dx_ex = np.einsum("nhwf,fc->nhwc", dec(ec), dec(wc).reshape(f, c)).astype(np.float32)
    X, W, E = _qt(fp8, xc, xc.shape, "fp8"), _qt(fp8, wc, wc.shape, "fp8"), _qt(fp8, ec, ec.shape, "fp8")
    old = os.environ.get("FP8B_CONV_1X1_GEMM")
    try:
        for route in ("1", "0"):
            os.environ["FP8B_CONV_1X1_GEMM"] = route
            for name, call, ex in [
                ("fprop", lambda **a: fp8.conv2d(X, W, 1, 0, **a), y_ex),
                ("dgrad", lambda **a: fp8.conv2d_backward_data(E, W, 1, 0, h, w, **a), dx_ex),
            ]:
                cnt = fp8.Counters()
                t, q = call(layout="nhwc", engine="tensor", out_fmt="fp8", out_counters=cnt,
                            want_y=out == "f32")
                codes, k_ = O.quantize(ex.reshape(-1), "fp8", "nearest-even")
                if out == "f32":
                    np.testing.assert_array_equal(t.cpu().numpy().reshape(-1), ex.reshape(-1))
                np.testing.assert_array_equal(q.codes.cpu().numpy(), codes.astype(np.uint8))
                assert cnt.values() == tuple(int(v) for v in k_), (route, name)
    finally:
        if old is None:
            os.environ.pop("FP8B_CONV_1X1_GEMM", None)
        else:
            os.environ["FP8B_CONV_1X1_GEMM"] = old


WGRAD_SHAPES = [  # n, c, h, w, f, pad, fmt  (3x3, 64-byte channel / filter rows)
    (2, 64, 56, 56, 64, 1, "fp8"),   # ResNet-50 3x3 @56 (2 rows per tile)
    (3, 64, 13, 9, 64, 1, "fp8"),    # ragged last tile
    (2, 64, 10, 30, 64, 0, "fp8"),   # no padding
    (1, 64, 6, 126, 64, 1, "fp8"),   # Wp = 128: one row per tile
    (300, 64, 7, 7, 64, 1, "fp8"),   # more tiles than SMs, tiny images
]


@pytest.mark.parametrize("shape", WGRAD_SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_halo_wgrad_exact_grid(fp8, env, shape):
    """Halo-slab wgrad (tap-pair accumulators resident in TMEM, fixed-order sum
    over CTAs) == the im2col wgrad == the exact result, bit for bit, on an
    exact operand grid; fused output Q node and counters included."""
    n, c, h, w, f, pad, fmt = shape
    k = 3
    assert fp8.conv_halo_supported(n, c, h, w, f, k, 1, pad, fmt, "wgrad")
    oh, ow = h + 2 * pad - k + 1, w + 2 * pad - k + 1
    rng = np.random.default_rng(n + h + w + pad)
    xc = _grid(rng, n * h * w * c, fmt, 0.5).reshape(n, h, w, c)
    ec = _grid(rng, n * oh * ow * f, fmt, 0.25).reshape(n, oh, ow, f)
    dec = lambda a: O.dequantize(a.reshape(-1), fmt).astype(np.float64).reshape(a.shape)
    from numpy.lib.stride_tricks import sliding_window_view as swv
    xp = np.pad(dec(xc), ((0, 0), (pad, pad), (pad, pad), (0, 0)))
    win = swv(xp, (k, k), axis=(1, 2))
    dw_ex = np.einsum("nhwf,nhwcij->fijc", dec(ec), win, optimize=True).astype(np.float32)
    X, E = _qt(fp8, xc, xc.shape, fmt), _qt(fp8, ec, ec.shape, fmt)
    codes, cnt = O.quantize(dw_ex.reshape(-1), "fp8", "nearest-even")
    for halo in ("1", "0"):
        env["FP8B_CONV_HALO"] = halo
        cq = fp8.Counters()
        dw, q = fp8.conv2d_backward_weights(X, E, k, k, 1, pad, layout="nhwc", engine="tensor",
                                            out_fmt="fp8", out_counters=cq)
        np.testing.assert_array_equal(dw.cpu().numpy().reshape(-1), dw_ex.reshape(-1),
                                      err_msg=f"halo={halo}")
        np.testing.assert_array_equal(q.codes.cpu().numpy(), codes.astype(np.uint8))
        assert cq.values() == tuple(int(v) for v in cnt), halo


@pytest.mark.parametrize("shape", [(4, 256, 7, 7, 512), (2, 512, 5, 6, 256), (3, 320, 4, 4, 384)],
                         ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("out_mode", ["nearest-even", "stochastic", "truncate"])
def test_1x1_wgrad_gemm_route_exact(fp8, shape, out_mode):
    """1x1 wgrad with few pixels routed to the pair-tile GEMM engine (dW = e^T . x,
    A = e MN-major, B = x N-major, split-K) equals the im2col wgrad and the exact
    result bit for bit on an exact operand grid; the fused Q(dW) node (RNE / TRUNC
    / SR with counter bits) equals the standalone quantize of dW, counters included."""
    n, c, h, w, f = shape
    rng = np.random.default_rng(c + f + 1)
    xc = _grid(rng, n * h * w * c, "fp8", 0.5).reshape(n, h, w, c)
    ec = _grid(rng, n * h * w * f, "fp8", 0.25).reshape(n, h, w, f)
    dec = lambda a: O.dequantize(a.reshape(-1), "fp8").astype(np.float64).reshape(a.shape)
    dw_ex = np.einsum("nhwf,nhwc->fc", dec(ec), dec(xc)).astype(np.float32)
    X, E = _qt(fp8, xc, xc.shape, "fp8"), _qt(fp8, ec, ec.shape, "fp8")
    old = os.environ.get("FP8B_CONV_1X1_WGRAD_PIX")
    try:
        got = []
        for lim in ("1000000", "0"):
            os.environ["FP8B_CONV_1X1_WGRAD_PIX"] = lim
            cnt = fp8.Counters()
            dw, q = fp8.conv2d_backward_weights(X, E, 1, 1, 1, 0, layout="nhwc", engine="tensor",
                                                out_fmt="fp8", out_mode=out_mode, out_seed=5,
                                                out_counters=cnt)
            np.testing.assert_array_equal(dw.cpu().numpy().reshape(-1), dw_ex.reshape(-1), err_msg=lim)
            ref = fp8.quantize(dw.reshape(-1), "fp8", out_mode, 5, bits="counter")
            assert (q.codes == ref.codes).all(), lim
            assert cnt.values() == ref.counters.values(), lim
            got.append(q.codes.cpu().numpy())
        np.testing.assert_array_equal(got[0], got[1])
    finally:
        if old is None:
            os.environ.pop("FP8B_CONV_1X1_WGRAD_PIX", None)
        else:
            os.environ["FP8B_CONV_1X1_WGRAD_PIX"] = old


@pytest.mark.parametrize("shape", [(2, 256, 6, 6, 256, 3, 1, "fp8"), (3, 512, 5, 7, 256, 1, 0, "fp8"),
                                   (2, 128, 9, 8, 256, 3, 1, "fp8"), (2, 64, 12, 10, 512, 1, 0, "fp8"),
                                   (2, 128, 6, 6, 256, 3, 1, "fp16"), (2, 64, 5, 9, 256, 1, 0, "fp16"),
                                   (2, 192, 6, 5, 256, 3, 1, "fp8")],
                         ids=lambda s: "x".join(map(str, s)))
def test_wgrad_block_tiles_exact_grid(fp8, env, shape):
    """im2col wgrad with block tiles (2 x 128 filter rows, 1 or 2 channel blocks
    per CTA: half the operand bytes per MAC) == the 128 x 128 tiles == the exact
    result, bit for bit, on an exact operand grid; Q(dW) codes and counters too."""
    n, c, h, w, f, k, pad, fmt = shape
    oh, ow = h + 2 * pad - k + 1, w + 2 * pad - k + 1
    rng = np.random.default_rng(c + f + k)
    xc = _grid(rng, n * h * w * c, fmt, 0.5).reshape(n, h, w, c)
    ec = _grid(rng, n * oh * ow * f, fmt, 0.25).reshape(n, oh, ow, f)
    dec = lambda a: O.dequantize(a.reshape(-1), fmt).astype(np.float64).reshape(a.shape)
    from numpy.lib.stride_tricks import sliding_window_view as swv
    xp = np.pad(dec(xc), ((0, 0), (pad, pad), (pad, pad), (0, 0)))
    win = swv(xp, (k, k), axis=(1, 2))
    dw_ex = np.einsum("nhwf,nhwcij->fijc", dec(ec), win, optimize=True).astype(np.float32)
    X, E = _qt(fp8, xc, xc.shape, fmt), _qt(fp8, ec, ec.shape, fmt)
    codes, cnt = O.quantize(dw_ex.reshape(-1), "fp8", "nearest-even")
    env["FP8B_CONV_1X1_WGRAD_PIX"] = "0"   # keep 1x1 shapes on the im2col kernel
    env["FP8B_CONV_HALO"] = "0"
    for blk in ("1", "0"):
        env["FP8B_CONV_WGRAD_BLOCK"] = blk
        cq = fp8.Counters()
        dw, q = fp8.conv2d_backward_weights(X, E, k, k, 1, pad, layout="nhwc", engine="tensor",
                                            out_fmt="fp8", out_counters=cq)
        np.testing.assert_array_equal(dw.cpu().numpy().reshape(-1), dw_ex.reshape(-1),
                                      err_msg=f"block={blk}")
        np.testing.assert_array_equal(q.codes.cpu().numpy(), codes.astype(np.uint8))
        assert cq.values() == tuple(int(v) for v in cnt), blk
