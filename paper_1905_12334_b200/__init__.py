"""B200-native FP8 (E5M2) training primitives -- the hot path of fp8emu on sm_100a.

This module mirrors the reference's Python surface (``fp8emu``,
/root/reference/proj/src/python/bindings.cpp:76-238) for the hot path:
``quantize``, ``dequantize``, ``gemm``, ``transpose``, ``encode``, ``decode``,
``LossScaler`` and the fused ``sgd_momentum_update``, with the same argument
names, meanings and error behaviour (``ValueError`` where the reference raises
``std::invalid_argument``). Every call runs hand-written CUDA kernels from
``libfp8b200.so`` through its C-ABI (include/fp8b200.h); tensors live in HBM
as torch CUDA tensors (torch is used for device memory and streams only).

Differences from the reference surface, all deliberate:
  * codes are 1 byte per E5M2 element (the reference widens to uint16);
    ``QuantizedTensor.codes_u16()`` returns the reference's layout;
  * inputs may be numpy arrays (copied to the current CUDA device) or CUDA
    tensors (used in place, no copy);
  * extensions: ``bits`` / ``block_offset`` / ``rbits`` for stochastic rounding
    (reference LFSR stream, counter bits, supplied bits), fused GEMM epilogues,
    MN-major operands, device-resident loss-scaler state.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib
from ._lib import LIB, check

__all__ = [
    "QuantizedTensor", "ScaleEvent", "LossScaler", "quantize", "dequantize", "transpose",
    "gemm", "gemm_codes", "encode", "decode", "sgd_momentum_update", "bias_grad",
    "count_nonfinite", "fill_synthetic", "stream_probe", "Counters", "launch_count", "version",
    "conv2d", "conv2d_backward_data", "conv2d_backward_weights", "im2col", "conv_out_dim", "conv_tensor_supported", "conv_halo_supported",
    "conv2d_im2col",
]

_FMT = {"fp8": _lib.E5M2, "FP8": _lib.E5M2, "e5m2": _lib.E5M2, "fp16": _lib.FP16,
        "FP16": _lib.FP16}
_MODE = {"nearest-even": _lib.RNE, "rne": _lib.RNE, "stochastic": _lib.SR,
         "truncate": _lib.TRUNC}
_BITS = {"lfsr": _lib.BITS_LFSR, "counter": _lib.BITS_COUNTER, "supplied": _lib.BITS_SUPPLIED}
_FMT_NAME = {_lib.E5M2: "FP8", _lib.FP16: "FP16"}
_MODE_NAME = {_lib.RNE: "nearest-even", _lib.SR: "stochastic", _lib.TRUNC: "truncate"}
_ACTION = {0: "none", 1: "backoff", 2: "growth", 3: "clamped_to_min"}


def _fmt(fmt: str) -> int:
    try:
        return _FMT[fmt]
    except KeyError:
        raise ValueError(f"unknown float format: {fmt}") from None


def _mode(mode: str) -> int:
    try:
        return _MODE[mode]
    except KeyError:
        raise ValueError(f"unknown rounding mode: {mode}") from None


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else t.data_ptr()


def _device_f32(x) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        if not x.is_cuda:
            x = x.to("cuda")
        if x.dtype != torch.float32:
            x = x.float()
        return x.contiguous()
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    return torch.from_numpy(arr).to("cuda")


def _code_dtype(fmt: int):
    return torch.uint8 if fmt == _lib.E5M2 else torch.int16


def version() -> str:
    return LIB.fp8b_version().decode()


def launch_count() -> int:
    """Number of libfp8b200 kernels launched by this process so far."""
    return int(LIB.fp8b_launch_count())


def init() -> None:
    check(LIB.fp8b_init(), "init")


class Counters:
    """Device int64[3] = {overflow, underflow, nan}; kernels accumulate into it."""

    def __init__(self, device=None):
        self.t = torch.zeros(3, dtype=torch.int64, device=device or "cuda")

    @property
    def ptr(self):
        return self.t.data_ptr()

    def zero_(self):
        self.t.zero_()
        return self

    def values(self) -> Tuple[int, int, int]:
        o, u, n = (int(v) for v in self.t.tolist())
        return o, u, n


class QuantizedTensor:
    """Mirror of fp8emu::QuantizedTensor (tensor.hpp:37-53) with device codes."""

    def __init__(self, codes: torch.Tensor, shape, fmt: int, mode: int, counters: Counters):
        self.codes = codes
        self.shape = list(shape)
        self.fmt_id = fmt
        self.mode_id = mode
        self.counters = counters

    @property
    def format(self) -> str:
        return _FMT_NAME[self.fmt_id]

    @property
    def mode(self) -> str:
        return _MODE_NAME[self.mode_id]

    @property
    def overflow_count(self) -> int:
        return self.counters.values()[0]

    @property
    def underflow_count(self) -> int:
        return self.counters.values()[1]

    @property
    def nan_count(self) -> int:
        return self.counters.values()[2]

    def numel(self) -> int:
        return int(np.prod(self.shape)) if self.shape else 1

    def codes_u16(self) -> np.ndarray:
        """Codes widened to the reference's uint16 storage, on the host."""
        c = self.codes.cpu().numpy()
        if self.fmt_id == _lib.FP16:
            c = c.view(np.uint16)
        return c.astype(np.uint16).reshape(self.shape)

    def reshaped(self, new_shape) -> "QuantizedTensor":
        if int(np.prod(new_shape)) != self.numel():
            raise ValueError("reshape changes element count")
        return QuantizedTensor(self.codes, new_shape, self.fmt_id, self.mode_id, self.counters)

    def __repr__(self):
        return f"QuantizedTensor({self.format}, shape={self.shape})"


def quantize(array, fmt: str = "fp8", mode: str = "nearest-even", seed: int = 1,
             saturate: bool = False, *, bits: str = "lfsr", block_offset: int = 0,
             rbits: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None,
             counters: Optional[Counters] = None, stream=None) -> QuantizedTensor:
    """fp8emu.quantize (bindings.cpp:167-176 -> tensor.cpp:46-81) on the GPU."""
    f, m = _fmt(fmt), _mode(mode)
    if bits not in _BITS:
        raise ValueError(f"unknown random-bits source: {bits}")
    x = _device_f32(array)
    shape = list(x.shape)
    n = x.numel()
    codes = out if out is not None else torch.empty(n, dtype=_code_dtype(f), device=x.device)
    cnt = counters if counters is not None else Counters(x.device)
    rb = None
    if rbits is not None:
        rb = rbits.reshape(-1).contiguous()
        if rb.dtype not in (torch.int32, torch.uint32) or rb.numel() != n or not rb.is_cuda:
            raise ValueError("rbits must be a CUDA int32/uint32 tensor with one word per element")
    cfg = _lib.QuantConfig(m, _BITS[bits], int(seed) & (2**64 - 1), int(bool(saturate)), 0,
                           int(block_offset), _ptr(rb))
    check(LIB.fp8b_quantize(x.data_ptr(), codes.data_ptr(), n, f, cfg, cnt.ptr, _stream(stream)),
          "quantize")
    return QuantizedTensor(codes, shape, f, m, cnt)


def dequantize(tensor: QuantizedTensor, stream=None) -> torch.Tensor:
    """fp8emu.dequantize (tensor.cpp:83-98)."""
    n = tensor.numel()
    out = torch.empty(n, dtype=torch.float32, device=tensor.codes.device)
    check(LIB.fp8b_dequantize(tensor.codes.data_ptr(), out.data_ptr(), n, tensor.fmt_id,
                              _stream(stream)), "dequantize")
    return out.reshape(tensor.shape)


def transpose(tensor: QuantizedTensor, stream=None) -> QuantizedTensor:
    """fp8emu transpose (tensor.cpp:135-150)."""
    if len(tensor.shape) != 2:
        raise ValueError("transpose expects a rank-2 tensor")
    r, c = tensor.shape
    out = torch.empty_like(tensor.codes)
    check(LIB.fp8b_transpose(tensor.codes.data_ptr(), out.data_ptr(), r, c, tensor.fmt_id,
                             _stream(stream)), "transpose")
    return QuantizedTensor(out, [c, r], tensor.fmt_id, tensor.mode_id, tensor.counters)


def gemm_codes(a_codes: torch.Tensor, b_codes: torch.Tensor, m: int, n: int, k: int,
               fmt: str = "fp8", *, a_major: str = "k", b_major: str = "n",
               engine: str = "tensor", c: Optional[torch.Tensor] = None, want_c: bool = True,
               bias: Optional[torch.Tensor] = None, out_fmt: Optional[str] = None,
               out_mode: str = "nearest-even", out_seed: int = 1, out_saturate: bool = False,
               out_codes: Optional[torch.Tensor] = None, out_counters: Optional[Counters] = None,
               stream=None):
    """Low-level GEMM over device code buffers (fp8b_gemm).

    a_major: "k" (A stored [M,K]) or "m" (A stored [K,M]);
    b_major: "n" (B stored [K,N], the reference layout) or "k" (B stored [N,K]).
    Returns (c, out_codes) -- either may be None.
    """
    f = _fmt(fmt)
    dev = a_codes.device
    if want_c and c is None:
        c = torch.empty((m, n), dtype=torch.float32, device=dev)
    cq = None
    cqf = 0
    if out_fmt is not None:
        cqf = _fmt(out_fmt)
        cq = out_codes if out_codes is not None else torch.empty(m * n, dtype=_code_dtype(cqf),
                                                                 device=dev)
    args = _lib.GemmArgs(
        _lib.K_MAJOR if a_major == "k" else _lib.MN_MAJOR,
        _lib.MN_MAJOR if b_major == "n" else _lib.K_MAJOR,
        _lib.GEMM_TENSOR if engine == "tensor" else _lib.GEMM_SEQUENTIAL, 0,
        _ptr(c) if want_c else None, _ptr(bias), _ptr(cq), cqf, _mode(out_mode),
        int(out_seed), int(bool(out_saturate)), 0,
        out_counters.ptr if out_counters is not None else None)
    check(LIB.fp8b_gemm(a_codes.data_ptr(), b_codes.data_ptr(), m, n, k, f, args,
                        _stream(stream)), "gemm_fp8")
    return (c if want_c else None), cq


def gemm_tensor_supported(a_codes, b_codes, m, n, k, fmt="fp8", a_major="k", b_major="n") -> bool:
    """True if the tcgen05 engine (not the CUDA-core fallback) runs this GEMM."""
    return bool(LIB.fp8b_gemm_tensor_supported(
        a_codes.data_ptr(), b_codes.data_ptr(), m, n, k, _fmt(fmt),
        _lib.K_MAJOR if a_major == "k" else _lib.MN_MAJOR,
        _lib.MN_MAJOR if b_major == "n" else _lib.K_MAJOR))


def gemm(a: QuantizedTensor, b: QuantizedTensor, *, engine: str = "tensor",
         stream=None) -> torch.Tensor:
    """fp8emu.gemm (bindings.cpp:183-189 -> kernels.cpp:37-62): FP32 [M, N]."""
    if len(a.shape) != 2 or len(b.shape) != 2:
        raise ValueError("gemm_fp8 expects rank-2 operands")
    if a.shape[1] != b.shape[0]:
        raise ValueError("gemm_fp8 inner dimensions disagree")
    if a.fmt_id != b.fmt_id:
        raise ValueError("kernel operands must share one format")
    m, k = a.shape
    n = b.shape[1]
    c, _ = gemm_codes(a.codes, b.codes, m, n, k, _FMT_NAME[a.fmt_id].lower(), engine=engine,
                      stream=stream)
    return c



# ---------------------------------------------------------------- convolutions


def conv_out_dim(size: int, k: int, stride: int, pad: int) -> int:
    """conv_out_dim (kernels.cpp:28-35)."""
    span = size + 2 * pad - k
    if span < 0 or stride < 1:
        raise ValueError("convolution geometry does not fit input")
    return span // stride + 1


def _conv_geom(n, c, h, w, f, kh, kw, stride, pad, layout, engine):
    if layout not in ("nchw", "nhwc"):
        raise ValueError(f"unknown layout: {layout}")
    if engine not in ("tensor", "sequential"):
        raise ValueError(f"unknown engine: {engine}")
    return _lib.ConvGeom(n, c, h, w, f, kh, kw, stride, pad,
                         _lib.NCHW if layout == "nchw" else _lib.NHWC,
                         _lib.GEMM_TENSOR if engine == "tensor" else _lib.GEMM_SEQUENTIAL)


def _conv_out_q(g, shape, device, out_fmt, out_mode, out_seed, out_saturate, out_counters):
    """Attach the fused output Q node to a ConvGeom; returns the code tensor."""
    if out_fmt is None:
        return None, None
    f = _fmt(out_fmt)
    n = int(np.prod(shape))
    codes = torch.empty(n, dtype=_code_dtype(f), device=device)
    cnt = out_counters if out_counters is not None else Counters(device)
    g.yq, g.yq_fmt, g.yq_mode = codes.data_ptr(), f, _mode(out_mode)
    g.yq_seed, g.yq_saturate, g.yq_counters = int(out_seed), int(bool(out_saturate)), cnt.ptr
    return QuantizedTensor(codes, list(shape), f, _mode(out_mode), cnt), cnt


def _conv_ret(y, q, want_y):
    if q is None:
        return y
    return (y if want_y else None), q


def _nchw_dims(shape, layout):
    if len(shape) != 4:
        return None
    if layout == "nchw":
        return shape[0], shape[1], shape[2], shape[3]
    return shape[0], shape[3], shape[1], shape[2]


def conv2d(x: QuantizedTensor, w: QuantizedTensor, stride: int = 1, pad: int = 0, *,
           layout: str = "nchw", engine: str = "sequential", out_fmt: Optional[str] = None,
           out_mode: str = "nearest-even", out_seed: int = 1, out_saturate: bool = False,
           out_counters: Optional[Counters] = None, want_y: bool = True, stream=None):
    """fp8emu.conv2d (bindings.cpp:191-198 -> kernels.cpp:106-151): FP32 output.

    layout "nchw": x [N,C,H,W], w [F,C,kH,kW] -> y [N,F,OH,OW] (the reference);
    layout "nhwc": x [N,H,W,C], w [F,kH,kW,C] -> y [N,OH,OW,F].
    engine "sequential" is bitwise the reference; "tensor" runs tcgen05 implicit
    GEMM where supported (NHWC E5M2 stride 1) within the GEMM tolerance.
    out_fmt: also emit the output's Q node (fused into the tensor epilogue);
    returns (y or None, QuantizedTensor) then. out_mode "stochastic" uses
    counter bits (seed out_seed)."""
    xd, wd = _nchw_dims(x.shape, layout), _nchw_dims(w.shape, layout)
    if xd is None or wd is None:
        raise ValueError("conv2d_fp8 expects [N,C,H,W] and [F,C,kH,kW]")
    n, c, h, wi = xd
    f, wc, kh, kw = wd
    if c != wc:
        raise ValueError("conv2d_fp8 channel counts disagree")
    if x.fmt_id != w.fmt_id:
        raise ValueError("kernel operands must share one format")
    oh, ow = conv_out_dim(h, kh, stride, pad), conv_out_dim(wi, kw, stride, pad)
    shape = (n, f, oh, ow) if layout == "nchw" else (n, oh, ow, f)
    g = _conv_geom(n, c, h, wi, f, kh, kw, stride, pad, layout, engine)
    q, _ = _conv_out_q(g, shape, x.codes.device, out_fmt, out_mode, out_seed, out_saturate,
                       out_counters)
    keep = want_y or q is None
    y = torch.empty(shape, dtype=torch.float32, device=x.codes.device) if keep else None
    check(LIB.fp8b_conv2d_fprop(x.codes.data_ptr(), w.codes.data_ptr(), _ptr(y), x.fmt_id,
                                g, _stream(stream)), "conv2d_fp8")
    return _conv_ret(y, q, keep)


def conv2d_backward_data(e: QuantizedTensor, w: QuantizedTensor, stride: int, pad: int, h: int,
                         w_dim: int, *, layout: str = "nchw", engine: str = "sequential",
                         out_fmt: Optional[str] = None, out_mode: str = "nearest-even",
                         out_seed: int = 1, out_saturate: bool = False,
                         out_counters: Optional[Counters] = None, want_y: bool = True,
                         stream=None):
    """conv2d_backward_data_fp8 (kernels.cpp:153-205): dx [N,C,H,W] (or NHWC)."""
    ed, wd = _nchw_dims(e.shape, layout), _nchw_dims(w.shape, layout)
    if ed is None or wd is None:
        raise ValueError("conv backward expects rank-4 operands")
    n, f, oh, ow = ed
    wf, c, kh, kw = wd
    if f != wf:
        raise ValueError("conv backward filter counts disagree")
    if e.fmt_id != w.fmt_id:
        raise ValueError("kernel operands must share one format")
    if conv_out_dim(h, kh, stride, pad) != oh or conv_out_dim(w_dim, kw, stride, pad) != ow:
        raise ValueError("conv backward geometry disagrees with error")
    shape = (n, c, h, w_dim) if layout == "nchw" else (n, h, w_dim, c)
    g = _conv_geom(n, c, h, w_dim, f, kh, kw, stride, pad, layout, engine)
    q, _ = _conv_out_q(g, shape, e.codes.device, out_fmt, out_mode, out_seed, out_saturate,
                       out_counters)
    keep = want_y or q is None
    dx = torch.empty(shape, dtype=torch.float32, device=e.codes.device) if keep else None
    check(LIB.fp8b_conv2d_dgrad(e.codes.data_ptr(), w.codes.data_ptr(), _ptr(dx), e.fmt_id,
                                g, _stream(stream)), "conv2d_backward_data_fp8")
    return _conv_ret(dx, q, keep)


def conv2d_backward_weights(x: QuantizedTensor, e: QuantizedTensor, kh: int, kw: int,
                            stride: int, pad: int, *, layout: str = "nchw",
                            engine: str = "sequential", out_fmt: Optional[str] = None,
                            out_mode: str = "nearest-even", out_seed: int = 1,
                            out_saturate: bool = False, out_counters: Optional[Counters] = None,
                            want_y: bool = True, stream=None):
    """conv2d_backward_weights_fp8 (kernels.cpp:207-253): dw [F,C,kH,kW] (or [F,kH,kW,C])."""
    xd, ed = _nchw_dims(x.shape, layout), _nchw_dims(e.shape, layout)
    if xd is None or ed is None or xd[0] != ed[0]:
        raise ValueError("conv backward expects matching rank-4 operands")
    if x.fmt_id != e.fmt_id:
        raise ValueError("kernel operands must share one format")
    n, c, h, wi = xd
    _, f, oh, ow = ed
    if conv_out_dim(h, kh, stride, pad) != oh or conv_out_dim(wi, kw, stride, pad) != ow:
        raise ValueError("conv backward geometry disagrees with error")
    shape = (f, c, kh, kw) if layout == "nchw" else (f, kh, kw, c)
    g = _conv_geom(n, c, h, wi, f, kh, kw, stride, pad, layout, engine)
    q, _ = _conv_out_q(g, shape, x.codes.device, out_fmt, out_mode, out_seed, out_saturate,
                       out_counters)
    keep = want_y or q is None
    dw = torch.empty(shape, dtype=torch.float32, device=x.codes.device) if keep else None
    check(LIB.fp8b_conv2d_wgrad(x.codes.data_ptr(), e.codes.data_ptr(), _ptr(dw), x.fmt_id,
                                g, _stream(stream)), "conv2d_backward_weights_fp8")
    return _conv_ret(dw, q, keep)


def conv2d_im2col(x: QuantizedTensor, w: QuantizedTensor, stride: int = 1, pad: int = 0, *,
                  engine: str = "sequential", stream=None) -> torch.Tensor:
    """conv2d_fp8_im2col (kernels.cpp:255-281): im2col + gemm_fp8, NCHW. With the
    sequential engine it is bitwise equal to conv2d (the reference's own check,
    test_kernels.cpp:97-118)."""
    if len(x.shape) != 4 or len(w.shape) != 4:
        raise ValueError("conv2d_fp8 expects [N,C,H,W] and [F,C,kH,kW]")
    n = x.shape[0]
    f, c, kh, kw = w.shape
    oh, ow = conv_out_dim(x.shape[2], kh, stride, pad), conv_out_dim(x.shape[3], kw, stride, pad)
    cols = im2col(x, kh, kw, stride, pad, stream=stream)
    flat = gemm(w.reshaped([f, c * kh * kw]), cols, engine=engine, stream=stream)  # [F, N*OH*OW]
    return flat.reshape(f, n, oh, ow).permute(1, 0, 2, 3).contiguous()


def conv_tensor_supported(n, c, h, w, f, k, stride=1, pad=0, fmt="fp8", kind="fprop",
                          layout="nhwc") -> bool:
    """True if engine="tensor" runs this conv on tcgen05 (else the sequential engine)."""
    g = _conv_geom(n, c, h, w, f, k, k, stride, pad, layout, "tensor")
    return bool(LIB.fp8b_conv_tensor_supported(g, _fmt(fmt),
                                               {"fprop": 0, "dgrad": 1, "wgrad": 2}[kind]))


def conv_halo_supported(n, c, h, w, f, k, stride=1, pad=0, fmt="fp8", kind="fprop") -> bool:
    """True if the tensor engine runs this NHWC conv on the weight-stationary
    halo-slab kernel (fprop / dgrad of narrow stride-1 layers)."""
    g = _conv_geom(n, c, h, w, f, k, k, stride, pad, "nhwc", "tensor")
    return bool(LIB.fp8b_conv_halo_supported(g, _fmt(fmt), {"fprop": 0, "dgrad": 1, "wgrad": 2}[kind]))


def im2col(x: QuantizedTensor, kh: int, kw: int, stride: int = 1, pad: int = 0, *,
           layout: str = "nchw", stream=None) -> QuantizedTensor:
    """im2col (kernels.cpp:64-104): NCHW -> [C*kH*kW, N*OH*OW] (the reference);
    NHWC -> [N*OH*OW, kH*kW*C]."""
    xd = _nchw_dims(x.shape, layout)
    if xd is None:
        raise ValueError("im2col expects [N, C, H, W]")
    n, c, h, wi = xd
    oh, ow = conv_out_dim(h, kh, stride, pad), conv_out_dim(wi, kw, stride, pad)
    rows, cols = (c * kh * kw, n * oh * ow) if layout == "nchw" else (n * oh * ow, kh * kw * c)
    out = torch.empty(rows * cols, dtype=x.codes.dtype, device=x.codes.device)
    g = _conv_geom(n, c, h, wi, 1, kh, kw, stride, pad, layout, "sequential")
    check(LIB.fp8b_im2col(x.codes.data_ptr(), out.data_ptr(), x.fmt_id, g, _stream(stream)),
          "im2col")
    return QuantizedTensor(out, [rows, cols], x.fmt_id, x.mode_id, x.counters)


def encode(x: float, fmt: str = "fp8", mode: str = "nearest-even", seed: int = 1,
           saturate: bool = False):
    """fp8emu.encode (bindings.cpp:138-152): (code, overflowed, underflowed_to_zero).
    SR draws from LfsrStream::split(seed, 0), as the binding does."""
    q = quantize(np.array([x], dtype=np.float32), fmt, mode, seed, saturate)
    code = int(q.codes_u16()[0])
    o, u, _ = q.counters.values()
    return code, bool(o), bool(u)


def decode(code: int, fmt: str = "fp8") -> float:
    """fp8emu.decode for one code (exact in FP32 for both formats)."""
    f = _fmt(fmt)
    dt = np.uint8 if f == _lib.E5M2 else np.uint16
    c = torch.from_numpy(np.array([code], dtype=dt).view(
        np.uint8 if f == _lib.E5M2 else np.int16)).to("cuda")
    q = QuantizedTensor(c, [1], f, _lib.RNE, Counters())
    return float(dequantize(q).cpu()[0])


@dataclass
class ScaleEvent:
    iteration: int
    action: str
    scale_after: float


class LossScaler:
    """fp8emu.LossScaler (loss_scaling.hpp:26-68) with its state in HBM.

    ``step`` launches one device kernel and does not synchronise; the
    ``scale``/event accessors copy the state back (they synchronise)."""

    def __init__(self, kind: str = "constant", scale: float = 1.0, backoff_factor: float = 0.5,
                 growth_factor: float = 2.0, growth_interval: int = 2000,
                 min_threshold_schedule: Sequence[Tuple[int, float]] = (), device=None):
        if kind == "constant":
            k = _lib.SCALER_CONSTANT
        elif kind == "dynamic-backoff":
            k = _lib.SCALER_DYNAMIC_BACKOFF
        else:
            raise ValueError(f"unknown scaler kind: {kind}")
        sched = list(min_threshold_schedule)
        if len(sched) > _lib.MAX_SCHEDULE:
            raise ValueError("min threshold schedule too long")
        h = _lib.LossScalerState()
        h.kind, h.n_schedule, h.scale = k, len(sched), float(scale)
        h.backoff_factor, h.growth_factor = float(backoff_factor), float(growth_factor)
        h.growth_interval = int(growth_interval)
        for i, (it, sc) in enumerate(sched):
            h.sched_iter[i] = int(it)
            h.sched_scale[i] = float(sc)
        self._host = h
        self.kind = kind
        self.schedule = sched
        nbytes = C_sizeof(_lib.LossScalerState)
        self.state = torch.zeros(nbytes, dtype=torch.uint8, device=device or "cuda")
        check(LIB.fp8b_loss_scaler_init(self.state.data_ptr(), h,
                                        _stream(None)), "LossScaler")

    @property
    def ptr(self):
        return self.state.data_ptr()

    def _read(self) -> _lib.LossScalerState:
        raw = self.state.cpu().numpy().tobytes()
        return _lib.LossScalerState.from_buffer_copy(raw)

    @property
    def scale(self) -> float:
        return self._read().scale

    @property
    def steps_since_overflow(self) -> int:
        return self._read().steps_since_overflow

    def min_threshold(self, iteration: int) -> float:
        thr = 1.0
        for it, sc in self.schedule:
            if it > iteration:
                break
            thr = sc
        return thr

    def step_async(self, grads_finite: bool = True, iteration: int = 0,
                   counters: Optional[Counters] = None, stream=None) -> None:
        check(LIB.fp8b_loss_scaler_step(self.ptr, counters.ptr if counters else None,
                                        int(bool(grads_finite)), int(iteration),
                                        _stream(stream)), "LossScaler.step")

    def step(self, grads_finite: bool, iteration: int) -> ScaleEvent:
        self.step_async(grads_finite, iteration)
        s = self._read()
        return ScaleEvent(int(s.last_iteration), _ACTION[s.last_action], s.last_scale_after)

    def state_dict(self) -> dict:
        """Device scaler state as a JSON-able dict (checkpoint extension)."""
        s = self._read()
        return {"kind": self.kind, "scale": s.scale, "steps_since_overflow": s.steps_since_overflow,
                "raw": self.state.cpu().numpy().tobytes().hex()}

    def load_state_dict(self, d: dict) -> None:
        raw = np.frombuffer(bytes.fromhex(d["raw"]), dtype=np.uint8)
        if raw.size != self.state.numel():
            raise ValueError("scaler state size mismatch")
        self.state.copy_(torch.from_numpy(raw.copy()))

    def unscale(self, gradients) -> torch.Tensor:
        g = _device_f32(gradients).clone()
        check(LIB.fp8b_unscale(g.data_ptr(), g.numel(), self.ptr, _stream(None)), "unscale")
        return g


def C_sizeof(t) -> int:
    import ctypes
    return ctypes.sizeof(t)


def sgd_momentum_update(grad: torch.Tensor, grad_fmt: str, master: torch.Tensor,
                        momentum: torch.Tensor, *, lr: float, mu: float,
                        two_lambda: float = 0.0, scale: float = 1.0,
                        scaler: Optional[LossScaler] = None,
                        skip_counters: Optional[Counters] = None,
                        master_mode: str = "nearest-even", bits: str = "lfsr", seed: int = 1,
                        block_offset: int = 0, rbits: Optional[torch.Tensor] = None,
                        master_counters: Optional[Counters] = None,
                        w_e5m2: Optional[torch.Tensor] = None, w_saturate: bool = False,
                        w_counters: Optional[Counters] = None,
                        step_scaler_iteration: Optional[int] = None,
                        skip_counters2: Optional[Counters] = None,
                        gate_out: Optional[Counters] = None,
                        clear_skip_counters: bool = False, stream=None) -> None:
    """update_tensor (nn.cpp:417-432) for one parameter tensor, in place.

    grad: device codes (grad_fmt "fp8"/"fp16") or FP32 values (grad_fmt "f32");
    master: FP16 codes (int16 tensor); momentum: FP32.
    step_scaler_iteration: when given (the iteration's last update), the update
    also runs LossScaler::step(grads_finite(skip_counters), iteration) on
    `scaler` once every CTA has read the scale -- no separate step launch.
    skip_counters2 / gate_out: the gate is skip_counters + skip_counters2, and
    (with step_scaler_iteration) the merged counts are stored in gate_out;
    clear_skip_counters then also zeroes the gate's inputs for the next step."""
    gf = {"fp8": _lib.E5M2, "e5m2": _lib.E5M2, "fp16": _lib.FP16, "f32": _lib.F32}.get(grad_fmt)
    if gf is None:
        raise ValueError(f"unknown gradient format: {grad_fmt}")
    n = master.numel()
    if momentum.numel() != n or grad.numel() != n:
        raise ValueError("update operands disagree in size")
    args = _lib.SgdArgs(float(lr), float(mu), float(two_lambda), float(scale),
                        scaler.ptr if scaler is not None else None,
                        skip_counters.ptr if skip_counters is not None else None,
                        _mode(master_mode), _BITS[bits], int(seed), int(block_offset),
                        _ptr(rbits), master_counters.ptr if master_counters else None,
                        _ptr(w_e5m2), int(bool(w_saturate)),
                        0 if step_scaler_iteration is None else (2 if clear_skip_counters else 1),
                        w_counters.ptr if w_counters else None,
                        0 if step_scaler_iteration is None else int(step_scaler_iteration),
                        skip_counters2.ptr if skip_counters2 is not None else None,
                        gate_out.ptr if gate_out is not None else None)
    check(LIB.fp8b_sgd_momentum_update(grad.data_ptr(), gf, master.data_ptr(),
                                       momentum.data_ptr(), n, args, _stream(stream)),
          "sgd_momentum_update")


def bias_grad(e: QuantizedTensor, stream=None) -> torch.Tensor:
    """db[j] = sum_r dequant(qe)[r, j] in row order (nn.cpp:308-314)."""
    rows, cols = e.shape
    db = torch.empty(cols, dtype=torch.float32, device=e.codes.device)
    check(LIB.fp8b_bias_grad(e.codes.data_ptr(), e.fmt_id, rows, cols, db.data_ptr(),
                             _stream(stream)), "bias_grad")
    return db


def count_nonfinite(x: torch.Tensor, counters: Counters, stream=None) -> None:
    check(LIB.fp8b_count_nonfinite(x.data_ptr(), x.numel(), counters.ptr, _stream(stream)),
          "count_nonfinite")


def fill_synthetic(out: torch.Tensor, kind: str, seed: int, p: float = 0.01, lo: float = -24.0,
                   hi: float = 17.0, stream=None) -> torch.Tensor:
    """Seeded synthetic data in HBM: kind "config2" (log-uniform + ties),
    "normal" (N(0, p^2)) or "halfnormal" (|N(0, p^2)|)."""
    k = {"config2": 0, "normal": 1, "halfnormal": 2}[kind]
    check(LIB.fp8b_fill_synthetic(out.data_ptr(), out.numel(), k, int(seed), float(p),
                                  float(lo), float(hi), _stream(stream)), "fill_synthetic")
    return out


def stream_probe(x: torch.Tensor, out: Optional[torch.Tensor], out_bytes: int, stream=None) -> None:
    """Measurement aid: stream x with the quantizer's access pattern, writing
    out_bytes (0, 1, 2 or 4) bytes per element and doing no arithmetic."""
    check(LIB.fp8b_stream_probe(x.data_ptr(), out.data_ptr() if out is not None else None,
                                x.numel(), int(out_bytes), _stream(stream)), "stream_probe")


class DenseLayer:
    """One quantized Dense layer trained on device (fp8b_dense_step).

    Mirrors what nn::Network does for a Dense layer in one training step
    (forward nn.cpp:187-203, backward nn.cpp:294-326, finiteness nn.cpp:401-411,
    apply_update nn.cpp:436-458, scaler.step nn.cpp:547): masters start as
    RNE_FP16(w) (nn.cpp:76-88) and the fprop weights as Q(decode(master)).
    ``w`` is [in, out] (row-major, as the reference stores Dense weights).
    """

    def __init__(self, w, bias=None, *, batch: int, lr: float, mu: float,
                 two_lambda: float = 0.0, scaler: LossScaler, engine: str = "tensor",
                 master_mode: str = "nearest-even", bits: str = "lfsr", seed: int = 1,
                 saturate: bool = False, want_dx: bool = True, want_y: bool = False):
        w = _device_f32(w)
        if w.dim() != 2:
            raise ValueError("Dense weights must be rank 2 [in, out]")
        self.in_features, self.out_features = w.shape
        self.batch = int(batch)
        dev = w.device
        I, O, B = self.in_features, self.out_features, self.batch
        self.w_master = quantize(w, "fp16").codes.reshape(I, O)
        wq = quantize(dequantize(QuantizedTensor(self.w_master.reshape(-1), [I * O], _lib.FP16,
                                                 _lib.RNE, Counters(dev))), "fp8")
        self.w_q = wq.codes.reshape(I, O)
        self.w_momentum = torch.zeros(I, O, dtype=torch.float32, device=dev)
        self.has_bias = bias is not None
        if self.has_bias:
            self.b_master = quantize(_device_f32(bias).reshape(-1), "fp16").codes
            self.b_momentum = torch.zeros(O, dtype=torch.float32, device=dev)
            self.b_value = torch.empty(O, dtype=torch.float32, device=dev)
            self.db = torch.empty(O, dtype=torch.float32, device=dev)
        self.qx = torch.empty(B, I, dtype=torch.uint8, device=dev)
        self.qy = torch.empty(B, O, dtype=torch.uint8, device=dev)
        self.qe = torch.empty(B, O, dtype=torch.uint8, device=dev)
        self.qdw = torch.empty(I, O, dtype=torch.uint8, device=dev)
        self.qdx = torch.empty(B, I, dtype=torch.uint8, device=dev) if want_dx else None
        self.y = torch.empty(B, O, dtype=torch.float32, device=dev) if want_y else None
        self.fwd_counters = torch.zeros(3, dtype=torch.int64, device=dev)
        self.counters = torch.zeros(6, dtype=torch.int64, device=dev)
        self.gate = torch.zeros(3, dtype=torch.int64, device=dev)
        self.scaler = scaler
        if bits not in _BITS:
            raise ValueError(f"unknown random-bits source: {bits}")
        self._s = _lib.DenseStep()
        s = self._s
        s.batch, s.in_features, s.out_features = B, I, O
        s.w_master, s.w_momentum, s.w_q = (self.w_master.data_ptr(), self.w_momentum.data_ptr(),
                                           self.w_q.data_ptr())
        if self.has_bias:
            s.b_master, s.b_momentum = self.b_master.data_ptr(), self.b_momentum.data_ptr()
            s.b_value, s.db = self.b_value.data_ptr(), self.db.data_ptr()
        s.qx, s.qy, s.qe, s.qdw = (self.qx.data_ptr(), self.qy.data_ptr(), self.qe.data_ptr(),
                                   self.qdw.data_ptr())
        s.qdx = _ptr(self.qdx)
        s.y = _ptr(self.y)
        s.fwd_counters, s.counters, s.gate = (self.fwd_counters.data_ptr(),
                                              self.counters.data_ptr(), self.gate.data_ptr())
        s.scaler = scaler.ptr
        s.lr, s.mu, s.two_lambda = float(lr), float(mu), float(two_lambda)
        s.engine = _lib.GEMM_TENSOR if engine == "tensor" else _lib.GEMM_SEQUENTIAL
        s.master_mode = _mode(master_mode)
        s.bits = _BITS[bits]
        s.saturate = int(bool(saturate))
        s.seed = int(seed)

    def step(self, x: torch.Tensor, e: torch.Tensor, iteration: int, stream=None) -> None:
        """Asynchronous: forward, backward, gated update and scaler step."""
        if x.numel() != self.batch * self.in_features or e.numel() != self.batch * self.out_features:
            raise ValueError("batch and layer sizes disagree")
        self._x, self._e = x, e
        self._s.x, self._s.e = x.data_ptr(), e.data_ptr()
        self._s.iteration = int(iteration)
        check(LIB.fp8b_dense_step(self._s, _stream(stream)), "dense_step")

    def refresh_fprop_weights(self) -> None:
        """Re-derive the fprop E5M2 weights Q(decode(master)) (nn.cpp:192) and the
        FP32 bias value decode(b_master) after the masters were replaced."""
        I, O = self.in_features, self.out_features
        dev = self.w_master.device
        wdec = dequantize(QuantizedTensor(self.w_master.reshape(-1), [I * O], _lib.FP16, _lib.RNE,
                                          Counters(dev)))
        quantize(wdec, "fp8", out=self.w_q.view(-1))
        if self.has_bias:
            self.b_value.copy_(dequantize(QuantizedTensor(self.b_master.reshape(-1), [O], _lib.FP16,
                                                          _lib.RNE, Counters(dev))))

    # step statistics (synchronise)
    def overflow_count(self) -> int:
        c = self.counters.tolist()
        return int(c[0] + c[3])

    def grads_finite(self) -> bool:
        g = self.gate.tolist()
        return g[0] + g[2] == 0

    def underflow_fraction(self) -> float:
        return float(self.counters[4].item()) / float(self.in_features * self.out_features)


from . import fp8t  # noqa: E402  (FP8T files and checkpoints)
from .fp8t import (IoError, load_checkpoint, load_tensor_codes, load_tensor_fp32,  # noqa: E402
                   peek_tensor_dtype, save_checkpoint, save_tensor)
__all__ += ["fp8t", "IoError", "save_tensor", "load_tensor_fp32", "load_tensor_codes",
            "peek_tensor_dtype", "save_checkpoint", "load_checkpoint"]
