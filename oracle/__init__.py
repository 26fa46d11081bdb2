"""TEST INFRASTRUCTURE ONLY -- ctypes bindings for the CPU oracle.

Two libraries live here:

* ``liboracle.so`` -- ``fp8_oracle.c``, a C restatement of the reference
  fp8emu hot path (codec, LFSR streams, quantize, gemm_fp8, update_tensor,
  LossScaler), each function citing the reference file:line it follows.
* ``_ref/libfp8emu_ref.so`` -- the UNMODIFIED reference sources
  (/root/reference/proj/src/*.cpp) compiled in place by ``oracle/Makefile``
  plus a ctypes shim (``ref_capi.cpp``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package. The product path
(``paper_1905_12334_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfp8emu_ref.so")

FMT = {"fp8": 0, "e5m2": 0, "fp16": 1}
MODE = {"nearest-even": 0, "rne": 0, "stochastic": 1, "truncate": 2}
BITS = {"lfsr": 0, "counter": 1, "supplied": 2}

_P = np.ctypeslib.ndpointer
_i64 = C.c_int64
_u64 = C.c_uint64


def build(force: bool = False) -> None:
    """Compile liboracle.so (and _ref when /root/reference is present)."""
    targets = []
    if force or not os.path.exists(ORACLE_SO):
        targets.append(ORACLE_SO)
    if os.path.isdir("/root/reference/proj") and (force or not os.path.exists(REF_SO)):
        targets.append("ref")
    if targets:
        subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _load_oracle():
    build()
    lib = C.CDLL(ORACLE_SO)
    lib.or_mix64.restype = _u64
    lib.or_mix64.argtypes = [_u64]
    lib.or_mix_seed.restype = _u64
    lib.or_mix_seed.argtypes = [_u64, _u64]
    lib.or_lfsr_split.restype = C.c_uint16
    lib.or_lfsr_split.argtypes = [_u64, _u64]
    lib.or_lfsr_next_bits.restype = C.c_uint32
    lib.or_lfsr_next_bits.argtypes = [C.POINTER(C.c_uint16), C.c_int]
    lib.or_decode.restype = C.c_double
    lib.or_decode.argtypes = [C.c_uint32, C.c_int]
    lib.or_encode.restype = C.c_uint32
    lib.or_encode.argtypes = [C.c_double, C.c_int, C.c_int, C.POINTER(C.c_uint16), C.c_int,
                              C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]
    lib.or_encode_bits.restype = C.c_uint32
    lib.or_encode_bits.argtypes = [C.c_uint32, C.c_int, C.c_int, C.c_uint32, C.c_int,
                                   C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]
    lib.or_quantize.restype = C.c_int
    lib.or_quantize.argtypes = [_P(np.float32, flags="C"), _i64, C.c_int, C.c_int, C.c_int,
                                _u64, C.c_int, _i64, C.c_void_p,
                                _P(np.uint16, flags="C"), _P(np.int64, flags="C")]
    lib.or_dequantize.restype = None
    lib.or_dequantize.argtypes = [_P(np.uint16, flags="C"), _i64, C.c_int,
                                  _P(np.float32, flags="C")]
    lib.or_gemm.restype = None
    lib.or_gemm.argtypes = [_P(np.uint16, flags="C"), _P(np.uint16, flags="C"), _i64, _i64,
                            _i64, C.c_int, _P(np.float32, flags="C")]
    lib.or_gemm_exact.restype = None
    lib.or_gemm_exact.argtypes = [_P(np.uint16, flags="C"), _P(np.uint16, flags="C"), _i64,
                                  _i64, _i64, C.c_int, _P(np.float64, flags="C"),
                                  _P(np.float64, flags="C")]
    lib.or_sgd_update.restype = C.c_int
    lib.or_sgd_update.argtypes = [_P(np.uint16, flags="C"), _P(np.float32, flags="C"),
                                  _P(np.float32, flags="C"), _i64, C.c_float, C.c_float,
                                  C.c_float, C.c_float, C.c_int, C.c_int, _u64, _i64,
                                  C.c_void_p, C.c_void_p, _P(np.int64, flags="C")]
    for fn in ("or_conv2d", "or_conv2d_dgrad", "or_conv2d_wgrad"):
        getattr(lib, fn).restype = None
        getattr(lib, fn).argtypes = [_P(np.uint16, flags="C"), _P(np.uint16, flags="C")] + \
            [_i64] * 9 + [C.c_int, _P(np.float32, flags="C")]
    lib.or_bias_grad.restype = None
    lib.or_bias_grad.argtypes = [_P(np.float32, flags="C"), _i64, _i64,
                                 _P(np.float32, flags="C")]
    lib.or_fnv1a64.restype = _u64
    lib.or_fnv1a64.argtypes = [C.c_void_p, _i64]
    lib.or_lfsr_tables.restype = None
    lib.or_lfsr_tables.argtypes = [_P(np.uint16, flags="C"), _P(np.uint16, flags="C")]
    lib.or_rand_fill_normal.restype = None
    lib.or_rand_fill_normal.argtypes = [C.c_void_p, _P(np.float32, flags="C"), _i64,
                                        C.c_double]
    lib.or_unscale.restype = None
    lib.or_unscale.argtypes = [_P(np.float32, flags="C"), _i64, C.c_double]
    return lib


_ORACLE = None
_REF = None


def lib():
    global _ORACLE
    if _ORACLE is None:
        _ORACLE = _load_oracle()
    return _ORACLE


def ref_available() -> bool:
    build()
    return os.path.exists(REF_SO)


def ref():
    """The compiled reference (oracle/_ref/libfp8emu_ref.so)."""
    global _REF
    if _REF is None:
        if not ref_available():
            raise FileNotFoundError(REF_SO)
        r = C.CDLL(REF_SO)
        r.ref_mix64.restype = _u64
        r.ref_mix64.argtypes = [_u64]
        r.ref_mix_seed.restype = _u64
        r.ref_mix_seed.argtypes = [_u64, _u64]
        r.ref_lfsr_split.restype = C.c_uint16
        r.ref_lfsr_split.argtypes = [_u64, _u64]
        r.ref_lfsr_samples.restype = None
        r.ref_lfsr_samples.argtypes = [C.c_uint16, _i64, _P(np.uint32, flags="C")]
        r.ref_decode.restype = C.c_double
        r.ref_decode.argtypes = [C.c_uint32, C.c_int]
        r.ref_encode.restype = C.c_uint32
        r.ref_encode.argtypes = [C.c_double, C.c_int, C.c_int, _u64, C.c_int,
                                 C.POINTER(C.c_int), C.POINTER(C.c_int)]
        r.ref_encode_state.restype = C.c_uint32
        r.ref_encode_state.argtypes = [C.c_double, C.c_int, C.c_int, C.POINTER(C.c_uint16),
                                       C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        r.ref_quantize.restype = C.c_int
        r.ref_quantize.argtypes = [_P(np.float32, flags="C"), _i64, C.c_int, C.c_int, _u64,
                                   C.c_int, _P(np.uint16, flags="C"), _P(np.int64, flags="C")]
        r.ref_quantize_mt.restype = C.c_int
        r.ref_quantize_mt.argtypes = [_P(np.float32, flags="C"), _i64, C.c_int, C.c_int, _u64,
                                      C.c_int, C.c_void_p, _P(np.int64, flags="C"), C.c_int]
        r.ref_dequantize.restype = None
        r.ref_dequantize.argtypes = [_P(np.uint16, flags="C"), _i64, C.c_int,
                                     _P(np.float32, flags="C")]
        r.ref_gemm.restype = C.c_int
        r.ref_gemm.argtypes = [_P(np.uint16, flags="C"), _P(np.uint16, flags="C"), _i64, _i64,
                               _i64, C.c_int, _P(np.float32, flags="C")]
        r.ref_gemm_mt.restype = C.c_int
        r.ref_gemm_mt.argtypes = [_P(np.uint16, flags="C"), _P(np.uint16, flags="C"), _i64,
                                  _i64, _i64, C.c_int, _P(np.float32, flags="C"), C.c_int]
        r.ref_conv.restype = C.c_int
        r.ref_conv.argtypes = [C.c_int, _P(np.uint16, flags="C"), _P(np.uint16, flags="C")] + \
            [_i64] * 9 + [C.c_int, _P(np.float32, flags="C")]
        r.ref_scaler_new.restype = C.c_void_p
        r.ref_scaler_new.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, _i64,
                                     C.c_int, C.c_void_p, C.c_void_p]
        r.ref_scaler_free.restype = None
        r.ref_scaler_free.argtypes = [C.c_void_p]
        r.ref_scaler_scale.restype = C.c_double
        r.ref_scaler_scale.argtypes = [C.c_void_p]
        r.ref_scaler_min_threshold.restype = C.c_double
        r.ref_scaler_min_threshold.argtypes = [C.c_void_p, _i64]
        r.ref_scaler_step.restype = C.c_int
        r.ref_scaler_step.argtypes = [C.c_void_p, C.c_int, _i64, C.POINTER(C.c_double)]
        r.ref_scaler_unscale.restype = None
        r.ref_scaler_unscale.argtypes = [C.c_void_p, _P(np.float32, flags="C"), _i64]
        r.ref_update.restype = C.c_int
        r.ref_update.argtypes = [_P(np.uint16, flags="C"), _P(np.float32, flags="C"),
                                 _P(np.float32, flags="C"), _i64, C.c_float, C.c_float,
                                 C.c_float, C.c_float, C.c_int, _u64, C.c_void_p]
        r.ref_rand_fill_normal.restype = None
        r.ref_rand_fill_normal.argtypes = [_P(np.uint64, flags="C"), C.POINTER(C.c_int),
                                           C.POINTER(C.c_double), _P(np.float32, flags="C"),
                                           _i64, C.c_double]
        _REF = r
    return _REF


# ---------------------------------------------------------------- oracle API
def encode(x: float, fmt="fp8", mode="nearest-even", r16=None, lfsr_state=None,
           saturate=False):
    """Reference-style scalar encode -> (code, overflowed, underflowed)."""
    o, u, c = C.c_int(), C.c_int(), C.c_int()
    st = C.c_uint16(lfsr_state if lfsr_state is not None else 1)
    code = lib().or_encode(float(x), FMT[fmt], MODE[mode], C.byref(st), int(saturate),
                           C.byref(o), C.byref(u), C.byref(c))
    return code, bool(o.value), bool(u.value)


def encode_bits(x_bits: int, fmt="fp8", mode="nearest-even", r16=0, saturate=False):
    o, u, ie = C.c_int(), C.c_int(), C.c_int()
    code = lib().or_encode_bits(int(x_bits) & 0xFFFFFFFF, FMT[fmt], MODE[mode], int(r16),
                                int(saturate), C.byref(o), C.byref(u), C.byref(ie))
    return code, bool(o.value), bool(u.value), bool(ie.value)


def decode(code: int, fmt="fp8") -> float:
    return lib().or_decode(int(code), FMT[fmt])


def quantize(x, fmt="fp8", mode="nearest-even", seed=1, saturate=False,
             bits="lfsr", block_offset=0, rbits=None):
    """Oracle quantize -> (codes uint16, [overflow, underflow, nan])."""
    x = np.ascontiguousarray(x, dtype=np.float32).reshape(-1)
    codes = np.zeros(x.size, dtype=np.uint16)
    cnt = np.zeros(3, dtype=np.int64)
    rb = None
    if rbits is not None:
        rbits = np.ascontiguousarray(rbits, dtype=np.uint32).reshape(-1)
        rb = rbits.ctypes.data
    rc = lib().or_quantize(x, x.size, FMT[fmt], MODE[mode], BITS[bits], int(seed),
                           int(saturate), int(block_offset), rb, codes, cnt)
    if rc != 0:
        raise ValueError("QuantConfig.seed must be nonzero")
    return codes, cnt


def dequantize(codes, fmt="fp8"):
    codes = np.ascontiguousarray(codes, dtype=np.uint16).reshape(-1)
    out = np.zeros(codes.size, dtype=np.float32)
    lib().or_dequantize(codes, codes.size, FMT[fmt], out)
    return out


def gemm(a_codes, b_codes, m, k, n, fmt="fp8"):
    a = np.ascontiguousarray(a_codes, dtype=np.uint16).reshape(-1)
    b = np.ascontiguousarray(b_codes, dtype=np.uint16).reshape(-1)
    c = np.zeros(m * n, dtype=np.float32)
    lib().or_gemm(a, b, m, k, n, FMT[fmt], c)
    return c.reshape(m, n)


def gemm_exact(a_codes, b_codes, m, k, n, fmt="fp8"):
    a = np.ascontiguousarray(a_codes, dtype=np.uint16).reshape(-1)
    b = np.ascontiguousarray(b_codes, dtype=np.uint16).reshape(-1)
    c = np.zeros(m * n, dtype=np.float64)
    d = np.zeros(m * n, dtype=np.float64)
    lib().or_gemm_exact(a, b, m, k, n, FMT[fmt], c, d)
    return c.reshape(m, n), d.reshape(m, n)


def conv_out(n, k, s, p):
    return (n + 2 * p - k) // s + 1


def conv2d(x_codes, w_codes, n, c, h, w, f, kh, kw, stride=1, pad=0, fmt="fp8", kind="fprop"):
    """Oracle conv family in NCHW / [F,C,kh,kw] (kernels.cpp:106-253).
    kind fprop: (x, w) -> y [N,F,OH,OW]; dgrad: (e, w) -> dx [N,C,H,W];
    wgrad: (x, e) -> dw [F,C,kh,kw]."""
    oh, ow = conv_out(h, kh, stride, pad), conv_out(w, kw, stride, pad)
    a = np.ascontiguousarray(x_codes, dtype=np.uint16).reshape(-1)
    b = np.ascontiguousarray(w_codes, dtype=np.uint16).reshape(-1)
    shape = {"fprop": (n, f, oh, ow), "dgrad": (n, c, h, w), "wgrad": (f, c, kh, kw)}[kind]
    out = np.zeros(int(np.prod(shape)), dtype=np.float32)
    fn = {"fprop": lib().or_conv2d, "dgrad": lib().or_conv2d_dgrad, "wgrad": lib().or_conv2d_wgrad}[kind]
    fn(a, b, n, c, h, w, f, kh, kw, stride, pad, FMT[fmt], out)
    return out.reshape(shape)


def ref_conv2d(a_codes, b_codes, n, c, h, w, f, kh, kw, stride=1, pad=0, fmt="fp8", kind="fprop"):
    oh, ow = conv_out(h, kh, stride, pad), conv_out(w, kw, stride, pad)
    a = np.ascontiguousarray(a_codes, dtype=np.uint16).reshape(-1)
    b = np.ascontiguousarray(b_codes, dtype=np.uint16).reshape(-1)
    shape = {"fprop": (n, f, oh, ow), "dgrad": (n, c, h, w), "wgrad": (f, c, kh, kw)}[kind]
    out = np.zeros(int(np.prod(shape)), dtype=np.float32)
    rc = ref().ref_conv({"fprop": 0, "dgrad": 1, "wgrad": 2}[kind], a, b, n, c, h, w, f, kh, kw,
                        stride, pad, FMT[fmt], out)
    if rc != 0:
        raise ValueError("convolution geometry does not fit input")
    return out.reshape(shape)


def sgd_update(master, momentum, g, scale, lr, mu, two_lambda=0.0, master_mode="nearest-even",
               bits="lfsr", seed=1, block_offset=0, rbits=None):
    """update_tensor arithmetic (nn.cpp:417-432); returns (master, momentum, w32, counters)."""
    master = np.array(master, dtype=np.uint16).reshape(-1)
    momentum = np.array(momentum, dtype=np.float32).reshape(-1)
    g = np.ascontiguousarray(g, dtype=np.float32).reshape(-1)
    w32 = np.zeros(master.size, dtype=np.float32)
    cnt = np.zeros(3, dtype=np.int64)
    rb = None
    if rbits is not None:
        rbits = np.ascontiguousarray(rbits, dtype=np.uint32).reshape(-1)
        rb = rbits.ctypes.data
    rc = lib().or_sgd_update(master, momentum, g, master.size, scale, lr, mu, two_lambda,
                             MODE[master_mode], BITS[bits], int(seed), int(block_offset), rb,
                             w32.ctypes.data, cnt)
    if rc != 0:
        raise ValueError("seed must be nonzero")
    return master, momentum, w32, cnt


def bias_grad(e, rows, cols):
    e = np.ascontiguousarray(e, dtype=np.float32).reshape(-1)
    db = np.zeros(cols, dtype=np.float32)
    lib().or_bias_grad(e, rows, cols, db)
    return db


def fnv1a64(arr) -> int:
    a = np.ascontiguousarray(arr)
    return int(lib().or_fnv1a64(a.ctypes.data, a.nbytes))


def lfsr_tables():
    tab = np.zeros(65535, dtype=np.uint16)
    pos = np.zeros(65536, dtype=np.uint16)
    lib().or_lfsr_tables(tab, pos)
    return tab, pos


class Rand:
    """rand.hpp:13-37 (the reference's counter RNG with Box-Muller spares)."""

    class _St(C.Structure):
        _fields_ = [("seed", C.c_uint64), ("n", C.c_uint64), ("have_spare", C.c_int),
                    ("spare", C.c_double)]

    def __init__(self, seed: int):
        self.st = Rand._St(seed, 0, 0, 0.0)

    def normal(self, count: int, stddev: float = 1.0) -> np.ndarray:
        out = np.zeros(count, dtype=np.float32)
        lib().or_rand_fill_normal(C.byref(self.st), out, count, stddev)
        return out


class OracleLossScaler:
    """loss_scaling.cpp state machine restated in Python over the C oracle's rules."""

    ACTIONS = {0: "none", 1: "backoff", 2: "growth", 3: "clamped_to_min"}

    def __init__(self, kind="constant", scale=1.0, backoff_factor=0.5, growth_factor=2.0,
                 growth_interval=2000, min_threshold_schedule=()):
        if not (scale > 0.0) or not np.isfinite(scale):
            raise ValueError("loss scale must be finite and positive")
        self.kind = kind
        self._scale = float(scale)
        self.backoff = backoff_factor
        self.growth = growth_factor
        self.interval = growth_interval
        self.schedule = list(min_threshold_schedule)
        self.steps_since_overflow = 0

    @property
    def scale(self):
        return self._scale

    def min_threshold(self, iteration):
        thr = 1.0
        for it, sc in self.schedule:
            if it > iteration:
                break
            thr = sc
        return thr

    def step(self, grads_finite, iteration):
        if self.kind == "constant":
            return "none", self._scale
        thr = self.min_threshold(iteration)
        act = "none"
        if not grads_finite:
            cand = self._scale * self.backoff
            if cand < thr:
                self._scale, act = thr, "clamped_to_min"
            else:
                self._scale, act = cand, "backoff"
            self.steps_since_overflow = 0
        else:
            self.steps_since_overflow += 1
            if self.steps_since_overflow >= self.interval:
                self._scale *= self.growth
                self.steps_since_overflow = 0
                act = "growth"
            if self._scale < thr:
                self._scale, act = thr, "clamped_to_min"
        return act, self._scale


# ------------------------------------------------------------- reference API
def ref_quantize(x, fmt="fp8", mode="nearest-even", seed=1, saturate=False):
    x = np.ascontiguousarray(x, dtype=np.float32).reshape(-1)
    codes = np.zeros(x.size, dtype=np.uint16)
    cnt = np.zeros(3, dtype=np.int64)
    rc = ref().ref_quantize(x, x.size, FMT[fmt], MODE[mode], int(seed), int(saturate), codes,
                            cnt)
    if rc != 0:
        raise ValueError("QuantConfig.seed must be nonzero")
    return codes, cnt[:2]


def ref_quantize_mt(x, fmt="fp8", mode="nearest-even", seed=1, saturate=False, nthreads=None):
    x = np.ascontiguousarray(x, dtype=np.float32).reshape(-1)
    nthreads = nthreads or os.cpu_count() or 1
    codes = np.zeros(x.size, dtype=np.uint8 if FMT[fmt] == 0 else np.uint16)
    cnt = np.zeros(3, dtype=np.int64)
    rc = ref().ref_quantize_mt(x, x.size, FMT[fmt], MODE[mode], int(seed), int(saturate),
                               codes.ctypes.data, cnt, int(nthreads))
    if rc != 0:
        raise ValueError("QuantConfig.seed must be nonzero")
    return codes, cnt[:2]


def ref_encode(x, fmt="fp8", mode="nearest-even", seed=1, saturate=False):
    o, u = C.c_int(), C.c_int()
    code = ref().ref_encode(float(x), FMT[fmt], MODE[mode], int(seed), int(saturate),
                            C.byref(o), C.byref(u))
    return code, bool(o.value), bool(u.value)


def ref_gemm(a_codes, b_codes, m, k, n, fmt="fp8", nthreads=1):
    a = np.ascontiguousarray(a_codes, dtype=np.uint16).reshape(-1)
    b = np.ascontiguousarray(b_codes, dtype=np.uint16).reshape(-1)
    c = np.zeros(m * n, dtype=np.float32)
    if nthreads > 1:
        ref().ref_gemm_mt(a, b, m, k, n, FMT[fmt], c, nthreads)
    else:
        rc = ref().ref_gemm(a, b, m, k, n, FMT[fmt], c)
        if rc != 0:
            raise ValueError("gemm_fp8: invalid arguments")
    return c.reshape(m, n)


def ref_update(master, momentum, g, scale, lr, mu, two_lambda=0.0, master_mode="nearest-even",
               seed=1):
    master = np.array(master, dtype=np.uint16).reshape(-1)
    momentum = np.array(momentum, dtype=np.float32).reshape(-1)
    g = np.ascontiguousarray(g, dtype=np.float32).reshape(-1)
    w32 = np.zeros(master.size, dtype=np.float32)
    rc = ref().ref_update(master, momentum, g, master.size, scale, lr, mu, two_lambda,
                          MODE[master_mode], int(seed), w32.ctypes.data)
    if rc != 0:
        raise ValueError("seed must be nonzero")
    return master, momentum, w32


class RefLossScaler:
    """The reference LossScaler itself (loss_scaling.cpp), through the shim."""

    ACTIONS = {0: "none", 1: "backoff", 2: "growth", 3: "clamped_to_min"}

    def __init__(self, kind="constant", scale=1.0, backoff_factor=0.5, growth_factor=2.0,
                 growth_interval=2000, min_threshold_schedule=()):
        sched = list(min_threshold_schedule)
        its = (C.c_int64 * max(1, len(sched)))(*[int(i) for i, _ in sched])
        scs = (C.c_double * max(1, len(sched)))(*[float(s) for _, s in sched])
        self.h = ref().ref_scaler_new(0 if kind == "constant" else 1, scale, backoff_factor,
                                      growth_factor, growth_interval, len(sched), its, scs)
        if not self.h:
            raise ValueError("invalid LossScaler options")

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_scaler_free(self.h)

    @property
    def scale(self):
        return ref().ref_scaler_scale(self.h)

    def min_threshold(self, it):
        return ref().ref_scaler_min_threshold(self.h, it)

    def step(self, grads_finite, iteration):
        sa = C.c_double()
        act = ref().ref_scaler_step(self.h, int(bool(grads_finite)), int(iteration),
                                    C.byref(sa))
        return self.ACTIONS[act], sa.value

    def unscale(self, g):
        g = np.array(g, dtype=np.float32).reshape(-1)
        ref().ref_scaler_unscale(self.h, g, g.size)
        return g


def ref_rand_normal(seed, counts_and_std):
    """Draw successive tensors from one Rand{seed} stream via the reference."""
    st = np.array([seed, 0], dtype=np.uint64)
    hs = C.c_int(0)
    sp = C.c_double(0.0)
    outs = []
    for count, std in counts_and_std:
        o = np.zeros(count, dtype=np.float32)
        ref().ref_rand_fill_normal(st, C.byref(hs), C.byref(sp), o, count, std)
        outs.append(o)
    return outs


def bitrev16(v: int) -> int:
    r = 0
    for i in range(16):
        r |= ((v >> i) & 1) << (15 - i)
    return r


# ---- FP8T container through the reference's own tensor_io.cpp -------------
def _ref_io():
    r = ref()
    if not getattr(r, "_io_ready", False):
        r.ref_fp8t_save_f32.restype = C.c_int
        r.ref_fp8t_save_f32.argtypes = [C.c_char_p, C.c_int, C.c_void_p, C.c_void_p, C.c_char_p]
        r.ref_fp8t_save_codes.restype = C.c_int
        r.ref_fp8t_save_codes.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                          C.c_void_p, C.c_char_p]
        r.ref_fp8t_load_f32.restype = C.c_int
        r.ref_fp8t_load_f32.argtypes = [C.c_char_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                        C.c_char_p]
        r.ref_fp8t_load_codes.restype = C.c_int
        r.ref_fp8t_load_codes.argtypes = [C.c_char_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p, C.c_char_p]
        r._io_ready = True
    return r


class RefIoError(RuntimeError):
    pass


def _dims64(shape):
    return np.ascontiguousarray(np.asarray(list(shape) or [0], dtype=np.int64))


def ref_fp8t_save_f32(path, arr):
    a = np.asarray(arr, dtype=np.float32)
    flat = np.ascontiguousarray(a.reshape(-1))  # (ascontiguousarray promotes 0-d to 1-d)
    d, msg = _dims64(a.shape), C.create_string_buffer(256)
    rc = _ref_io().ref_fp8t_save_f32(os.fsencode(path), a.ndim, d.ctypes.data, flat.ctypes.data, msg)
    if rc:
        raise RefIoError(msg.value.decode())


def ref_fp8t_save_codes(path, codes, shape, fmt="fp8", mode_tag=1):
    c = np.ascontiguousarray(np.asarray(codes, dtype=np.uint16).reshape(-1))
    d, msg = _dims64(shape), C.create_string_buffer(256)
    rc = _ref_io().ref_fp8t_save_codes(os.fsencode(path), FMT[fmt], mode_tag, len(shape),
                                       d.ctypes.data, c.ctypes.data, msg)
    if rc:
        raise RefIoError(msg.value.decode())


def ref_fp8t_load_f32(path, cap=1 << 20):
    out = np.empty(cap, dtype=np.float32)
    rank, dims, msg = C.c_int(), np.zeros(16, dtype=np.int64), C.create_string_buffer(256)
    rc = _ref_io().ref_fp8t_load_f32(os.fsencode(path), out.ctypes.data, cap, C.addressof(rank),
                                     dims.ctypes.data, msg)
    if rc:
        raise RefIoError(msg.value.decode())
    shape = [int(v) for v in dims[:rank.value]]
    return out[:int(np.prod(shape)) if shape else 1].reshape(shape)


def ref_fp8t_load_codes(path, cap=1 << 20):
    out = np.empty(cap, dtype=np.uint16)
    fmt, mode, rank = C.c_int(), C.c_int(), C.c_int()
    dims, msg = np.zeros(16, dtype=np.int64), C.create_string_buffer(256)
    rc = _ref_io().ref_fp8t_load_codes(os.fsencode(path), out.ctypes.data, cap, C.addressof(fmt),
                                       C.addressof(mode), C.addressof(rank), dims.ctypes.data, msg)
    if rc:
        raise RefIoError(msg.value.decode())
    shape = [int(v) for v in dims[:rank.value]]
    n = int(np.prod(shape)) if shape else 1
    return out[:n].reshape(shape), ("fp8" if fmt.value == 0 else "fp16"), mode.value
