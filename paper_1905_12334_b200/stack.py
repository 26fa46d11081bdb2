"""A stack of FP8 (E5M2) linear layers trained data-parallel -- the caller of
the hot path for BASELINE config 5 (Transformer-base, every linear GEMM in
E5M2 with FP32 accumulation, enhanced dynamic loss scaling, SR FP16 masters).

One training step over T tokens per rank, per layer l with weights W_l [in, out]
(the reference's Dense layout, nn.cpp:56-62):

  forward   (nn.cpp:187-203)  Y_l = Q(X_l) W_l          -> fused Q(Y_l), E5M2
  backward  (nn.cpp:294-326)  dX_l = E_l W_l^T           -> fused Q(dX_l)
                              dW_l = X_l^T E_l           -> Q(dW_l)
  update    (nn.cpp:436-458)  one SGD-momentum pass over every layer's
                              parameters, FP16 master with stochastic
                              rounding, next step's E5M2 weights written by
                              the same pass; skipped when any backward Q node
                              overflowed (nn.cpp:546)
  scaler    (nn.cpp:547)      LossScaler::step on the device

Parameters of all layers live in flat buffers (FP16 masters, FP32 momentum,
E5M2 weights, E5M2 dW), each layer at a 4096-aligned offset, so the update is a
single launch whose SR stream for layer l equals a per-layer update with
block_offset = offset_l / 4096 (tensor.cpp:58-62).

Data parallel: with world > 1 every rank computes FP32 dW for its
token shard into one flat FP32 buffer; one all-reduce (NCCL over NVLink on the
B200) sums them **before** the single Q(dW) pass, exactly as the reference's
one Q node sits on the full-batch sum (nn.cpp:302-303); the overflow gate is
all-reduced so every rank skips together. With world == 1 Q(dW) is fused into
the wgrad epilogue and no FP32 dW exists.

Attention softmax, layer norm, embedding and the loss are not in the
reference and are not run: each layer reads synthetic
E5M2 activations / errors of its shape.

The arithmetic goes through an ``ops`` object (dp.GpuOps by default); the CPU
tests substitute the oracle to check the orchestration over gloo.
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist

from .dp import BLOCK, GpuOps

LayerSpec = Tuple[str, int, int]   # (name, in_features, out_features)


def transformer_base_layers(d_model: int = 512, d_ff: int = 2048, n_enc: int = 6,
                            n_dec: int = 6, vocab: int = 32000) -> List[LayerSpec]:
    """The linear layers of Transformer-base (BASELINE config 5) in forward order.
    Encoder layer: fused QKV, attention output, FFN in/out. Decoder layer: fused
    self-attention QKV and output, cross-attention Q, fused cross K/V (on the
    encoder output) and output, FFN in/out. Then the output projection."""
    d, f = d_model, d_ff
    out: List[LayerSpec] = []
    for i in range(n_enc):
        out += [(f"enc{i}.qkv", d, 3 * d), (f"enc{i}.attn_out", d, d),
                (f"enc{i}.ffn_in", d, f), (f"enc{i}.ffn_out", f, d)]
    for i in range(n_dec):
        out += [(f"dec{i}.self_qkv", d, 3 * d), (f"dec{i}.self_out", d, d),
                (f"dec{i}.cross_q", d, d), (f"dec{i}.cross_kv", d, 2 * d),
                (f"dec{i}.cross_out", d, d), (f"dec{i}.ffn_in", d, f), (f"dec{i}.ffn_out", f, d)]
    out.append(("generator", d, vocab))
    return out


def linear_flops_per_token(layers: Sequence[LayerSpec]) -> float:
    """fprop + dgrad + wgrad FLOP per token of the linear layers (2 per MAC)."""
    return 3 * 2.0 * sum(i * o for _, i, o in layers)


class LinearStack:
    """FP8 linear layers of one model replica on this rank (see module doc)."""

    def __init__(self, layers: Sequence[LayerSpec], tokens: int, w_init: torch.Tensor, *,
                 lr: float, mu: float, two_lambda: float = 0.0, scaler=None, ops=None,
                 group=None, master_mode: str = "stochastic", seed: int = 1):
        self.ops = ops or GpuOps()
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.layers = list(layers)
        self.tokens = int(tokens)
        self.offsets = []
        off = 0
        for _, i, o in self.layers:
            self.offsets.append(off)
            off += (i * o + BLOCK - 1) // BLOCK * BLOCK
        self.nparams = off
        if w_init.numel() != off:
            raise ValueError(f"w_init must hold {off} values (4096-aligned layer offsets)")
        ops = self.ops
        dev = w_init.device
        # masters start as RNE_FP16(w), the fprop weights as Q(decode(master)) (nn.cpp:76-88, 192)
        self.master = ops.quantize(w_init.reshape(-1), "fp16").view(torch.int16)
        self.w_q = ops.quantize(ops.dequantize(self.master, "fp16"))
        self.momentum = torch.zeros(off, dtype=torch.float32, device=dev)
        self.qdw = torch.zeros(off, dtype=torch.uint8, device=dev)
        self.dw32 = torch.zeros(off, dtype=torch.float32, device=dev) if self.world > 1 else None
        self.lr, self.mu, self.two_lambda = lr, mu, two_lambda
        self.scaler = scaler
        self.master_mode, self.seed = master_mode, seed

    def weights(self, l: int) -> torch.Tensor:
        """E5M2 fprop weights of layer l, [in, out]."""
        _, i, o = self.layers[l]
        return self.w_q[self.offsets[l]:self.offsets[l] + i * o].view(i, o)

    def masters(self, l: int) -> torch.Tensor:
        _, i, o = self.layers[l]
        return self.master[self.offsets[l]:self.offsets[l] + i * o].view(i, o)

    def step(self, xs: Sequence[torch.Tensor], es: Sequence[torch.Tensor], iteration: int,
             ys: Optional[Sequence[torch.Tensor]] = None,
             dxs: Optional[Sequence[torch.Tensor]] = None):
        """One training step. xs[l]: E5M2 codes [T, in_l]; es[l]: E5M2 loss-scaled
        errors [T, out_l]. ys / dxs: optional output buffers for Q(Y_l) / Q(dX_l).
        Returns (forward counters, backward counters) -- backward is the gate."""
        ops, T = self.ops, self.tokens
        fwd, bwd = ops.counters(), ops.counters()
        multi = self.world > 1
        for l, (_, i, o) in enumerate(self.layers):
            ops.gemm_q(xs[l], self.weights(l), T, o, i, "k", "n", counters=fwd,
                       out=None if ys is None else ys[l])
        for l in reversed(range(len(self.layers))):
            _, i, o = self.layers[l]
            a, b = self.offsets[l], self.offsets[l] + i * o
            ops.gemm_q(es[l], self.weights(l), T, i, o, "k", "k", counters=bwd,
                       out=None if dxs is None else dxs[l])
            if multi:
                ops.gemm_f32(xs[l], es[l], i, o, T, "m", "n", out=self.dw32[a:b])
            else:
                ops.gemm_q(xs[l], es[l], i, o, T, "m", "n", counters=bwd, out=self.qdw[a:b])
        if multi:
            dist.all_reduce(self.dw32, op=dist.ReduceOp.SUM, group=self.group)
            ops.quantize(self.dw32, counters=bwd, out=self.qdw)
            gate = ops.ctensor(bwd)
            dist.all_reduce(gate, op=dist.ReduceOp.SUM, group=self.group)
        ops.update(self.qdw, self.master, self.momentum, lr=self.lr, mu=self.mu,
                   two_lambda=self.two_lambda, scaler=self.scaler, skip_counters=bwd,
                   master_mode=self.master_mode, seed=self.seed, w_e5m2=self.w_q)
        if self.scaler is not None and hasattr(self.scaler, "step_async"):
            self.scaler.step_async(True, iteration, counters=bwd)
        return fwd, bwd
