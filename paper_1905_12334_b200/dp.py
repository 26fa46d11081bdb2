"""Multi-GPU plumbing for the FP8 training primitives.

* ``block_shard``: contiguous ranges of whole 4096-element blocks per rank, with
  the ``block_offset`` that makes each rank's stochastic-rounding stream the
  slice of the single-GPU stream (the reference's schedule-independence
  contract, tensor.hpp:55-58). Quantize / update shard with no collective.
* ``DataParallelDense``: a Dense layer trained data-parallel. Each rank runs the
  forward, Q(e), bprop and a *FP32* wgrad on its batch shard; the FP32 partial
  dW are summed with one all-reduce (NCCL over NVLink on B200, gloo in the CPU
  tests) **before** the single Q(dW) node, matching the reference's one Q node
  on the full-batch sum (nn.cpp:302-303; only the FP32 summation order
  differs). The overflow counters are all-reduced too, so every rank skips the
  update together (nn.cpp:546), and every rank applies the identical update to
  its replica of the FP16 masters.

* ``ZeroDataParallelDense`` (ZeRO stage 1): the FP32 partial dW
  are reduce-scattered instead of all-reduced; each rank owns a block-aligned
  shard of the FP16 masters and momentum, runs Q(dW) and the update on it
  (``block_offset`` keeps the SR streams those of the unsharded update) and
  the E5M2 fprop weights are all-gathered: 4 + 1 bytes per parameter on the
  wire instead of 8, and 6/world bytes of optimizer state per parameter.

The arithmetic goes through an ``ops`` object; the default is this library's
CUDA kernels (``GpuOps``). Tests substitute a CPU implementation to cover the
multi-process orchestration with world_size 2 over gloo.
"""
from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist

BLOCK = 4096


def block_shard(n: int, world: int, rank: int, block: int = BLOCK):
    """(start, end, block_offset) of rank's share of n elements, whole blocks."""
    nblocks = (n + block - 1) // block
    per = (nblocks + world - 1) // world
    b0 = min(rank * per, nblocks)
    b1 = min(b0 + per, nblocks)
    return min(b0 * block, n), min(b1 * block, n), b0


class GpuOps:
    """The hot path on this library's kernels (tensors on the current CUDA device)."""

    def __init__(self, engine: str = "tensor"):
        from . import Counters, gemm_codes, quantize, sgd_momentum_update
        self._q, self._g, self._u, self._C = quantize, gemm_codes, sgd_momentum_update, Counters
        self.engine = engine
        self.device = torch.device("cuda", torch.cuda.current_device())

    def dequantize(self, codes, fmt="fp8"):
        from . import QuantizedTensor, dequantize, _fmt
        return dequantize(QuantizedTensor(codes.reshape(-1), [codes.numel()], _fmt(fmt), 0,
                                          self.counters()))

    def counters(self):
        return self._C(self.device)

    @staticmethod
    def ctensor(c):
        return c.t

    def quantize(self, x, fmt="fp8", mode="nearest-even", seed=1, block_offset=0, counters=None,
                 out=None):
        return self._q(x, fmt, mode, seed, block_offset=block_offset, counters=counters,
                       out=out).codes

    def gemm_f32(self, a, b, m, n, k, a_major="k", b_major="n", out=None):
        c, _ = self._g(a, b, m, n, k, "fp8", a_major=a_major, b_major=b_major, engine=self.engine,
                       c=None if out is None else out.view(m, n))
        return c

    def gemm_q(self, a, b, m, n, k, a_major="k", b_major="n", counters=None, out=None):
        _, cq = self._g(a, b, m, n, k, "fp8", a_major=a_major, b_major=b_major,
                        engine=self.engine, want_c=False, out_fmt="fp8", out_counters=counters,
                        out_codes=out)
        return cq

    def update(self, qdw, master, momentum, *, lr, mu, two_lambda, scaler, skip_counters,
               master_mode, seed, w_e5m2=None, block_offset=0):
        self._u(qdw, "fp8", master, momentum, lr=lr, mu=mu, two_lambda=two_lambda,
                scaler=scaler, skip_counters=skip_counters, master_mode=master_mode, seed=seed,
                w_e5m2=w_e5m2, block_offset=block_offset)


class DataParallelDense:
    """Batch-sharded Dense layer; weights [in, out] replicated on every rank."""

    def __init__(self, w_master, w_q, *, batch_per_rank: int, lr: float, mu: float,
                 two_lambda: float = 0.0, scaler=None, ops=None, group=None,
                 master_mode: str = "nearest-even", seed: int = 1):
        self.ops = ops or GpuOps()
        self.group = group
        self.w_master = w_master            # FP16 codes [in, out]
        self.w_q = w_q                      # E5M2 codes [in, out]: Q(decode(master))
        self.in_f, self.out_f = w_master.shape
        self.momentum = torch.zeros(self.in_f, self.out_f, dtype=torch.float32,
                                    device=w_master.device)
        self.bpr = batch_per_rank
        self.lr, self.mu, self.two_lambda = lr, mu, two_lambda
        self.scaler = scaler
        self.master_mode, self.seed = master_mode, seed

    def step(self, x_local, e_local, iteration: int):
        """One DP training step; returns (qy_local, qdx_local, gate counters)."""
        B, I, O = self.bpr, self.in_f, self.out_f
        ops = self.ops
        fwd = ops.counters()
        bwd = ops.counters()
        qx = ops.quantize(x_local.reshape(-1), counters=fwd)
        qy = ops.gemm_q(qx, self.w_q, B, O, I, "k", "n", counters=fwd)
        qe = ops.quantize(e_local.reshape(-1), counters=bwd)
        # FP32 partial dW on this rank's rows, summed across ranks before Q(dW)
        dw = ops.gemm_f32(qx, qe, I, O, B, "m", "n")
        if dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.all_reduce(dw, op=dist.ReduceOp.SUM, group=self.group)
        qdx = ops.gemm_q(qe, self.w_q, B, I, O, "k", "k", counters=bwd)
        qdw = ops.quantize(dw.reshape(-1), counters=bwd)
        gate = ops.ctensor(bwd)
        if dist.is_initialized() and dist.get_world_size(self.group) > 1:
            # every rank must agree on grads_finite (nn.cpp:401-411, 546)
            dist.all_reduce(gate, op=dist.ReduceOp.SUM, group=self.group)
        ops.update(qdw, self.w_master.reshape(-1), self.momentum.reshape(-1), lr=self.lr,
                   mu=self.mu, two_lambda=self.two_lambda, scaler=self.scaler,
                   skip_counters=bwd, master_mode=self.master_mode, seed=self.seed,
                   w_e5m2=self.w_q.reshape(-1))
        if self.scaler is not None and hasattr(self.scaler, "step_async"):
            self.scaler.step_async(True, iteration, counters=bwd)
        return qy, qdx, gate


class ZeroDataParallelDense:
    """Batch-sharded Dense layer with ZeRO-1 sharded optimizer state.

    Every rank keeps the full E5M2 fprop weights ``w_q`` [in, out]; the FP16
    masters and FP32 momentum exist only for this rank's block-aligned shard
    ``[start, end)`` of the flattened weights (block_shard). Per step:
    forward / Q(e) / bprop / FP32 wgrad on the local batch, reduce-scatter of
    the FP32 dW (padded to whole equal shards), Q(dW) and the gated update on
    the shard, all-reduce of the overflow gate, all-gather of the E5M2 shards.
    Bitwise equal to ``DataParallelDense`` (same FP32 sum order per element)."""

    def __init__(self, w_master_full, w_q, *, batch_per_rank: int, lr: float, mu: float,
                 two_lambda: float = 0.0, scaler=None, ops=None, group=None,
                 master_mode: str = "nearest-even", seed: int = 1,
                 transport: str = "collective"):
        """transport "collective": reduce-scatter / all-gather through the process
        group (NCCL on GPUs). "peer": one node, NVLink / NVSwitch peer memory --
        every rank's FP32 dW lives in a buffer its peers map, the shard owner's
        fused kernel sums the ranks' partials in rank order and applies Q(dW) in
        the same pass (peer.py, csrc/peer.cu), and the E5M2 weight shards are
        pulled from the owners' buffers; the two transports give identical bits
        when the FP32 sums are order-independent."""
        if transport not in ("collective", "peer"):
            raise ValueError(f"unknown transport: {transport}")
        self.transport = transport
        self.ops = ops or GpuOps()
        self.group = group
        distributed = dist.is_initialized()
        self.world = dist.get_world_size(group) if distributed else 1
        self.rank = dist.get_rank(group) if distributed else 0
        self.in_f, self.out_f = w_q.shape
        n = self.in_f * self.out_f
        self.n = n
        nblocks = (n + BLOCK - 1) // BLOCK
        self.per = ((nblocks + self.world - 1) // self.world) * BLOCK   # padded shard length
        self.start, self.end, self.block_offset = block_shard(n, self.world, self.rank)
        dev = w_q.device
        self.w_q = w_q                                                   # E5M2 [in, out]
        self.w_master = w_master_full.reshape(-1)[self.start:self.end].clone()   # FP16 shard
        self.momentum = torch.zeros(self.end - self.start, dtype=torch.float32, device=dev)
        self.bpr = batch_per_rank
        self.lr, self.mu, self.two_lambda = lr, mu, two_lambda
        self.scaler = scaler
        self.master_mode, self.seed = master_mode, seed
        if transport == "peer":
            from .peer import PeerBuffer
            if n % 4:
                raise ValueError("peer transport needs a parameter count that is a multiple of 4")
            self._dw_peer = PeerBuffer(4 * self.per * self.world, group)
            self._wq_peer = PeerBuffer(self.per * self.world, group)
            self._dw_full = self._dw_peer.view().view(torch.float32)
            self._dw_full.zero_()
            self._wq_pad = self._wq_peer.view()
            self._wq_pad.zero_()
        else:
            self._wq_pad = torch.zeros(self.per * self.world, dtype=w_q.dtype, device=dev)

    def _step_peer(self, x_local, e_local, iteration: int):
        """The step over peer memory (transport="peer")."""
        from .peer import fence, reduce_quantize
        B, I, O = self.bpr, self.in_f, self.out_f
        ops = self.ops
        fwd, bwd = ops.counters(), ops.counters()
        qx = ops.quantize(x_local.reshape(-1), counters=fwd)
        qy = ops.gemm_q(qx, self.w_q, B, O, I, "k", "n", counters=fwd)
        qe = ops.quantize(e_local.reshape(-1), counters=bwd)
        # this rank's FP32 partial dW, written where its peers can read it
        ops.gemm_f32(qx, qe, I, O, B, "m", "n", out=self._dw_full[: self.n])
        qdx = ops.gemm_q(qe, self.w_q, B, I, O, "k", "k", counters=bwd)
        fence(self.group)          # every rank's partial is complete
        ns = self.end - self.start
        qdw = torch.empty(ns, dtype=torch.uint8, device=self.w_q.device)
        if ns:
            reduce_quantize(self._dw_peer.ptrs, self.start, ns, qdw, counters=bwd,
                            block_offset=self.block_offset)
        gate = ops.ctensor(bwd)
        if self.world > 1:
            dist.all_reduce(gate, op=dist.ReduceOp.SUM, group=self.group)
        lo = self.rank * self.per
        if ns:
            self._wq_pad[lo: lo + ns].copy_(self.w_q.reshape(-1)[self.start:self.end])
            ops.update(qdw, self.w_master, self.momentum, lr=self.lr, mu=self.mu,
                       two_lambda=self.two_lambda, scaler=self.scaler, skip_counters=bwd,
                       master_mode=self.master_mode, seed=self.seed,
                       w_e5m2=self._wq_pad[lo: lo + ns], block_offset=self.block_offset)
        fence(self.group)          # every owner's new E5M2 shard is in its buffer
        for r in range(self.world):  # pull the other owners' shards over NVLink
            if r != self.rank:
                s0, s1, _ = block_shard(self.n, self.world, r)
                if s1 > s0:
                    self._wq_pad[r * self.per: r * self.per + (s1 - s0)].copy_(
                        self._wq_peer.view(r)[r * self.per: r * self.per + (s1 - s0)])
        wflat = self.w_q.reshape(-1)
        for r in range(self.world):
            s0, s1, _ = block_shard(self.n, self.world, r)
            wflat[s0:s1].copy_(self._wq_pad[r * self.per: r * self.per + (s1 - s0)])
        if self.scaler is not None and hasattr(self.scaler, "step_async"):
            self.scaler.step_async(True, iteration, counters=bwd)
        return qy, qdx, gate

    def step(self, x_local, e_local, iteration: int):
        if self.transport == "peer":
            return self._step_peer(x_local, e_local, iteration)
        B, I, O = self.bpr, self.in_f, self.out_f
        ops = self.ops
        fwd, bwd = ops.counters(), ops.counters()
        multi = self.world > 1
        qx = ops.quantize(x_local.reshape(-1), counters=fwd)
        qy = ops.gemm_q(qx, self.w_q, B, O, I, "k", "n", counters=fwd)
        qe = ops.quantize(e_local.reshape(-1), counters=bwd)
        dw = ops.gemm_f32(qx, qe, I, O, B, "m", "n").reshape(-1)
        qdx = ops.gemm_q(qe, self.w_q, B, I, O, "k", "k", counters=bwd)
        full = torch.zeros(self.per * self.world, dtype=torch.float32, device=dw.device)
        full[: self.n] = dw
        shard = torch.empty(self.per, dtype=torch.float32, device=dw.device)
        if multi:
            dist.reduce_scatter_tensor(shard, full, op=dist.ReduceOp.SUM, group=self.group)
        else:
            shard.copy_(full)
        ns = self.end - self.start
        qdw = ops.quantize(shard[:ns].contiguous(), block_offset=self.block_offset, counters=bwd) \
            if ns else shard[:0].to(torch.uint8)
        gate = ops.ctensor(bwd)
        if multi:
            dist.all_reduce(gate, op=dist.ReduceOp.SUM, group=self.group)
        wq_shard = self._wq_pad[self.rank * self.per: self.rank * self.per + ns]
        if ns:
            wq_shard.copy_(self.w_q.reshape(-1)[self.start:self.end])
            ops.update(qdw, self.w_master, self.momentum, lr=self.lr, mu=self.mu,
                       two_lambda=self.two_lambda, scaler=self.scaler, skip_counters=bwd,
                       master_mode=self.master_mode, seed=self.seed, w_e5m2=wq_shard,
                       block_offset=self.block_offset)
        if multi:
            # bytes moved as int32 words (shards are whole 4096-blocks): gloo has
            # no uint8 all-gather, NCCL does not care
            mine = self._wq_pad[self.rank * self.per:(self.rank + 1) * self.per].clone()
            dist.all_gather_into_tensor(self._wq_pad.view(torch.int32), mine.view(torch.int32),
                                        group=self.group)
        self.w_q.reshape(-1).copy_(self._wq_pad[: self.n])
        if self.scaler is not None and hasattr(self.scaler, "step_async"):
            self.scaler.step_async(True, iteration, counters=bwd)
        return qy, qdx, gate

    def gather_masters(self):
        """The full FP16 masters (for checks and checkpoints): all-gather of shards."""
        pad = torch.zeros(self.per, dtype=self.w_master.dtype, device=self.w_master.device)
        pad[: self.end - self.start] = self.w_master
        if self.world == 1:
            return pad[: self.n].reshape(self.in_f, self.out_f)
        out = torch.empty(self.per * self.world, dtype=pad.dtype, device=pad.device)
        dist.all_gather_into_tensor(out.view(torch.int32), pad.view(torch.int32), group=self.group)
        return out[: self.n].reshape(self.in_f, self.out_f)
