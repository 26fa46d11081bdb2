"""FP8T tensor files and checkpoints (tensor_io.hpp:18-45, nn.cpp:632-701).

The container is read and written by libfp8b200's native host code
(``fp8b_fp8t_save/peek/load``, csrc/fp8t_io.cu); this module moves tensors
between HBM and host buffers around it. Errors raise ``IoError`` with the
reference's messages.

Checkpoints follow ``save_checkpoint`` / ``load_checkpoint`` (nn.cpp:632-701):
``layer{i}_w.fp8t`` / ``layer{i}_b.fp8t`` hold the FP16 master codes and
``manifest.txt`` lists the layers. As an extension the momentum
buffers (``layer{i}_w_mom.fp8t``, FP32) and the loss-scaler state
(``scaler.json``) are saved too, which the reference omits, so a resumed run
continues bit for bit.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import LIB, IoError, check

__all__ = ["IoError", "save_tensor", "load_tensor_fp32", "load_tensor_codes",
           "peek_tensor_dtype", "save_checkpoint", "load_checkpoint"]

_MODE_TAG = {_lib.RNE: 1, _lib.SR: 2, _lib.TRUNC: 3}
_TAG_MODE = {0: _lib.RNE, 1: _lib.RNE, 2: _lib.SR, 3: _lib.TRUNC}


def _b(path) -> bytes:
    return os.fsencode(os.fspath(path))


def _dims(shape):
    d = (C.c_int64 * max(1, len(shape)))(*[int(v) for v in shape])
    return d


def save_tensor(path, t) -> None:
    """save_tensor (tensor_io.cpp:107-140) for an FP32 torch tensor / numpy array
    or a QuantizedTensor (codes, with its rounding-mode tag)."""
    from . import QuantizedTensor
    if isinstance(t, QuantizedTensor):
        codes = t.codes.reshape(-1).cpu().numpy()
        if t.fmt_id == _lib.E5M2:
            host, dtype = np.ascontiguousarray(codes.astype(np.uint8)), _lib.FP8T_FP8
        else:
            host, dtype = np.ascontiguousarray(codes.view(np.uint16)), _lib.FP8T_FP16
        shape, mode = list(t.shape), _MODE_TAG.get(t.mode_id, 1)
    else:
        a = t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)
        if a.dtype != np.float32:
            raise ValueError("save_tensor expects FP32 data or a QuantizedTensor")
        host, dtype, shape, mode = np.ascontiguousarray(a.reshape(-1)), _lib.FP8T_F32, list(a.shape), 0
    check(LIB.fp8b_fp8t_save(_b(path), dtype, mode, len(shape), _dims(shape),
                             host.ctypes.data if host.size else None))


def _peek(path):
    dt, mode, rank = C.c_int32(), C.c_int32(), C.c_int32()
    dims = (C.c_int64 * _lib.FP8T_MAX_RANK)()
    check(LIB.fp8b_fp8t_peek(_b(path), C.byref(dt), C.byref(mode), C.byref(rank), dims,
                             _lib.FP8T_MAX_RANK))
    return dt.value, mode.value, [int(dims[i]) for i in range(rank.value)]


def peek_tensor_dtype(path) -> str:
    """peek_tensor_dtype (tensor_io.cpp:189-192): "fp32", "fp8" or "fp16"."""
    return {_lib.FP8T_F32: "fp32", _lib.FP8T_FP8: "fp8", _lib.FP8T_FP16: "fp16"}[_peek(path)[0]]


def load_tensor_fp32(path, device: str = "cuda") -> torch.Tensor:
    """load_tensor_fp32 (tensor_io.cpp:142-160)."""
    dt, _, shape = _peek(path)
    n = int(np.prod(shape)) if shape else 1
    host = np.empty(n, dtype=np.float32)
    check(LIB.fp8b_fp8t_load(_b(path), _lib.FP8T_F32, host.ctypes.data, n))
    return torch.from_numpy(host.reshape(shape)).to(device)


def load_tensor_codes(path, device: str = "cuda"):
    """load_tensor_codes (tensor_io.cpp:162-187) -> QuantizedTensor on ``device``."""
    from . import Counters, QuantizedTensor
    dt, mode, shape = _peek(path)
    n = int(np.prod(shape)) if shape else 1
    host = np.empty(n, dtype=np.uint8 if dt == _lib.FP8T_FP8 else np.uint16)
    check(LIB.fp8b_fp8t_load(_b(path), -1, host.ctypes.data, n))
    if dt == _lib.FP8T_FP8:
        codes, fmt = torch.from_numpy(host), _lib.E5M2
    else:
        codes, fmt = torch.from_numpy(host.view(np.int16)), _lib.FP16
    return QuantizedTensor(codes.to(device), shape, fmt, _TAG_MODE[mode], Counters(device))


def save_checkpoint(layers: Sequence, directory, scaler=None) -> None:
    """save_checkpoint (nn.cpp:632-674) for a stack of DenseLayer objects, plus
    the momentum buffers and the scaler state (extension)."""
    from . import QuantizedTensor
    os.makedirs(directory, exist_ok=True)
    manifest = []
    for i, L in enumerate(layers):
        manifest.append(f"layer {i} kind=dense precision=fp8 w=layer{i}_w.fp8t "
                        f"b=layer{i}_b.fp8t\n")
        I, O = L.in_features, L.out_features
        save_tensor(os.path.join(directory, f"layer{i}_w.fp8t"),
                    QuantizedTensor(L.w_master.reshape(-1), [I, O], _lib.FP16, _lib.RNE, None))
        save_tensor(os.path.join(directory, f"layer{i}_w_mom.fp8t"), L.w_momentum.reshape(I, O))
        if L.has_bias:
            save_tensor(os.path.join(directory, f"layer{i}_b.fp8t"),
                        QuantizedTensor(L.b_master.reshape(-1), [O], _lib.FP16, _lib.RNE, None))
            save_tensor(os.path.join(directory, f"layer{i}_b_mom.fp8t"), L.b_momentum.reshape(O))
    try:
        with open(os.path.join(directory, "manifest.txt"), "w") as f:
            f.write("".join(manifest))
        if scaler is not None:
            with open(os.path.join(directory, "scaler.json"), "w") as f:
                json.dump(scaler.state_dict(), f)
    except OSError as e:
        raise IoError(f"{directory}: cannot write checkpoint ({e})") from None


def load_checkpoint(layers: Sequence, directory, scaler=None) -> None:
    """load_checkpoint (nn.cpp:676-701): masters (and, when present, momentum and
    scaler state); the fprop E5M2 weights are re-derived as Q(decode(master))."""
    for i, L in enumerate(layers):
        I, O = L.in_features, L.out_features
        parts = [("w", L.w_master, [I, O], L.w_momentum)]
        if L.has_bias:
            parts.append(("b", L.b_master, [O], L.b_momentum))
        for tag, master, shape, mom in parts:
            path = os.path.join(directory, f"layer{i}_{tag}.fp8t")
            if peek_tensor_dtype(path) != "fp16":
                raise IoError(path + ": checkpoint shape/format mismatch")
            q = load_tensor_codes(path, device=str(master.device))
            if list(q.shape) != shape:
                raise IoError(path + ": checkpoint shape/format mismatch")
            master.view(-1).copy_(q.codes.view(-1))
            mpath = os.path.join(directory, f"layer{i}_{tag}_mom.fp8t")
            if os.path.exists(mpath):
                m = load_tensor_fp32(mpath, device=str(mom.device))
                if list(m.shape) != shape:
                    raise IoError(mpath + ": checkpoint shape mismatch")
                mom.copy_(m)
        L.refresh_fprop_weights()
    spath = os.path.join(directory, "scaler.json")
    if scaler is not None and os.path.exists(spath):
        with open(spath) as f:
            scaler.load_state_dict(json.load(f))
