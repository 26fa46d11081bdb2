"""ctypes binding of libfp8b200.so (the C-ABI declared in include/fp8b200.h).

The library is built in-tree (``make -C paper_1905_12334_b200``, or
``__graft_entry__.build()``). There is no Python or CPU fallback: if the shared
object is missing, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# FP8B200_LIB (diagnostic): another build of the same library, for A/B timing
LIB_PATH = os.environ.get("FP8B200_LIB") or os.path.join(HERE, "libfp8b200.so")

OK, EINVAL, ENOTSUP, ECUDA, EIO = 0, 22, 95, 1000, 5
FP8T_F32, FP8T_FP8, FP8T_FP16 = 0, 1, 2
FP8T_MAX_RANK = 255
E5M2, FP16, F32 = 0, 1, 2
RNE, SR, TRUNC = 0, 1, 2
BITS_LFSR, BITS_COUNTER, BITS_SUPPLIED = 0, 1, 2
K_MAJOR, MN_MAJOR = 0, 1
GEMM_TENSOR, GEMM_SEQUENTIAL = 0, 1
SCALER_CONSTANT, SCALER_DYNAMIC_BACKOFF = 0, 1
NCHW, NHWC = 0, 1
MAX_SCHEDULE = 16

_vp = C.c_void_p
_i32, _i64, _u64 = C.c_int32, C.c_int64, C.c_uint64


class QuantConfig(C.Structure):
    _fields_ = [("mode", _i32), ("bits", _i32), ("seed", _u64), ("saturate", _i32),
                ("reserved", _i32), ("block_offset", _i64), ("rbits", _vp)]


class GemmArgs(C.Structure):
    _fields_ = [("a_major", _i32), ("b_major", _i32), ("engine", _i32), ("reserved0", _i32),
                ("c", _vp), ("bias", _vp), ("cq", _vp), ("cq_fmt", _i32), ("cq_mode", _i32),
                ("cq_seed", _u64), ("cq_saturate", _i32), ("reserved1", _i32),
                ("cq_counters", _vp)]


class LossScalerState(C.Structure):
    _fields_ = [("kind", _i32), ("n_schedule", _i32), ("scale", C.c_double),
                ("backoff_factor", C.c_double), ("growth_factor", C.c_double),
                ("growth_interval", _i64), ("steps_since_overflow", _i64),
                ("sched_iter", _i64 * MAX_SCHEDULE), ("sched_scale", C.c_double * MAX_SCHEDULE),
                ("last_iteration", _i64), ("last_action", _i32), ("last_grads_finite", _i32),
                ("last_scale_after", C.c_double), ("step_ticket", C.c_uint32),
                ("reserved", C.c_uint32)]


class SgdArgs(C.Structure):
    _fields_ = [("lr", C.c_float), ("mu", C.c_float), ("two_lambda", C.c_float),
                ("scale", C.c_float), ("scaler", _vp), ("skip_counters", _vp),
                ("master_mode", _i32), ("bits", _i32), ("seed", _u64), ("block_offset", _i64),
                ("rbits", _vp), ("master_counters", _vp), ("w_e5m2", _vp),
                ("w_saturate", _i32), ("step_scaler", _i32), ("w_counters", _vp),
                ("step_iteration", _i64), ("skip_counters2", _vp), ("gate_out", _vp)]


class DenseStep(C.Structure):
    _fields_ = [("batch", _i64), ("in_features", _i64), ("out_features", _i64),
                ("x", _vp), ("e", _vp), ("w_master", _vp), ("w_momentum", _vp), ("w_q", _vp),
                ("b_master", _vp), ("b_momentum", _vp), ("b_value", _vp),
                ("qx", _vp), ("qy", _vp), ("qe", _vp), ("qdw", _vp), ("qdx", _vp),
                ("db", _vp), ("y", _vp), ("fwd_counters", _vp), ("counters", _vp),
                ("gate", _vp), ("scaler", _vp), ("iteration", _i64),
                ("lr", C.c_float), ("mu", C.c_float), ("two_lambda", C.c_float),
                ("engine", _i32), ("master_mode", _i32), ("bits", _i32), ("saturate", _i32),
                ("seed", _u64)]


class ConvGeom(C.Structure):
    _fields_ = [("n", _i64), ("c", _i64), ("h", _i64), ("w", _i64), ("f", _i64), ("kh", _i64),
                ("kw", _i64), ("stride", _i64), ("pad", _i64), ("layout", _i32), ("engine", _i32),
                ("yq", _vp), ("yq_fmt", _i32), ("yq_mode", _i32), ("yq_seed", _u64),
                ("yq_saturate", _i32), ("reserved", _i32), ("yq_counters", _vp)]


# every symbol include/fp8b200.h declares, with its ctypes signature
SIGNATURES = {
    "fp8b_quantize": (C.c_int, [_vp, _vp, _i64, _i32, C.POINTER(QuantConfig), _vp, _vp]),
    "fp8b_dequantize": (C.c_int, [_vp, _vp, _i64, _i32, _vp]),
    "fp8b_transpose": (C.c_int, [_vp, _vp, _i64, _i64, _i32, _vp]),
    "fp8b_count_nonfinite": (C.c_int, [_vp, _i64, _vp, _vp]),
    "fp8b_gemm": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _i32, C.POINTER(GemmArgs), _vp]),
    "fp8b_gemm_tensor_supported": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _i32, _i32, _i32]),
    "fp8b_loss_scaler_init": (C.c_int, [_vp, C.POINTER(LossScalerState), _vp]),
    "fp8b_loss_scaler_step": (C.c_int, [_vp, _vp, _i32, _i64, _vp]),
    "fp8b_unscale": (C.c_int, [_vp, _i64, _vp, _vp]),
    "fp8b_sgd_momentum_update": (C.c_int, [_vp, _i32, _vp, _vp, _i64, C.POINTER(SgdArgs), _vp]),
    "fp8b_bias_grad": (C.c_int, [_vp, _i32, _i64, _i64, _vp, _vp]),
    "fp8b_conv2d_fprop": (C.c_int, [_vp, _vp, _vp, _i32, C.POINTER(ConvGeom), _vp]),
    "fp8b_conv2d_dgrad": (C.c_int, [_vp, _vp, _vp, _i32, C.POINTER(ConvGeom), _vp]),
    "fp8b_conv2d_wgrad": (C.c_int, [_vp, _vp, _vp, _i32, C.POINTER(ConvGeom), _vp]),
    "fp8b_conv_tensor_supported": (C.c_int, [C.POINTER(ConvGeom), _i32, _i32]),
    "fp8b_conv_halo_supported": (C.c_int, [C.POINTER(ConvGeom), _i32, _i32]),
    "fp8b_im2col": (C.c_int, [_vp, _vp, _i32, C.POINTER(ConvGeom), _vp]),
    "fp8b_fp8t_save": (C.c_int, [C.c_char_p, _i32, _i32, _i32, _vp, _vp]),
    "fp8b_fp8t_peek": (C.c_int, [C.c_char_p, _vp, _vp, _vp, _vp, _i32]),
    "fp8b_fp8t_load": (C.c_int, [C.c_char_p, _i32, _vp, _i64]),
    "fp8b_dense_step": (C.c_int, [C.POINTER(DenseStep), _vp]),
    "fp8b_init": (C.c_int, []),
    "fp8b_last_error": (C.c_char_p, []),
    "fp8b_version": (C.c_char_p, []),
    "fp8b_launch_count": (C.c_int64, []),
    "fp8b_fill_synthetic": (C.c_int, [_vp, _i64, _i32, _u64, C.c_double, C.c_double,
                                      C.c_double, _vp]),
    "fp8b_stream_probe": (C.c_int, [_vp, _vp, _i64, _i32, _vp]),
    "fp8b_peer_alloc": (C.c_int, [C.POINTER(_vp), _i64, C.c_char_p]),
    "fp8b_peer_free": (C.c_int, [_vp]),
    "fp8b_peer_open": (C.c_int, [C.c_char_p, C.POINTER(_vp)]),
    "fp8b_peer_close": (C.c_int, [_vp]),
    "fp8b_peer_reduce_quantize": (C.c_int, [C.POINTER(_vp), _i32, _i64, _i64, _vp, _vp, _i32,
                                            C.POINTER(QuantConfig), _vp, _vp]),
}


def load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C {HERE}` "
            "(the CUDA extension is required; there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = load()


class Fp8bError(RuntimeError):
    pass


class IoError(RuntimeError):
    """fp8emu::IoError (tensor_io.hpp:13-15): unreadable or garbled files."""


def check(rc: int, what: str = "") -> None:
    if rc == OK:
        return
    msg = LIB.fp8b_last_error().decode(errors="replace")
    if rc == EINVAL:
        raise ValueError(f"{what}: {msg}" if what else msg)
    if rc == EIO:
        raise IoError(msg)
    raise Fp8bError(f"{what}: [{rc}] {msg}" if what else f"[{rc}] {msg}")
