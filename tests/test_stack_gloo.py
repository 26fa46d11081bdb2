"""CPU, world_size 2 over gloo: the data-parallel FP8 linear stack
(paper_1905_12334_b200/stack.py, BASELINE config 5's caller of the hot path)
with the oracle standing in for the kernels.

* two ranks on half the tokens each, FP32 dW all-reduced before the single
  Q(dW) pass, equal the single-process stack (fused Q(dW)) bit for bit on
  inputs whose FP32 sums are exact -- masters, E5M2 weights and momentum, over
  two steps with SR FP16 masters;
* an overflowing Q(dX) on one rank makes every rank skip the update.
"""
import os

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1905_12334_b200.stack import LinearStack, linear_flops_per_token, transformer_base_layers
from test_dp_gloo import ConstScale, CpuOps, _free_port, _grid

LAYERS = [("l0", 64, 96), ("l1", 96, 64), ("l2", 64, 160)]
T = 32


class StackCpuOps(CpuOps):
    """CpuOps with output buffers and FP16 codes (test infrastructure only)."""

    def dequantize(self, codes, fmt="fp8"):
        c = codes.numpy().reshape(-1)
        c = c.view(np.uint16) if fmt == "fp16" else c.astype(np.uint16)
        return torch.from_numpy(O.dequantize(c, fmt).copy())

    def quantize(self, x, fmt="fp8", mode="nearest-even", seed=1, block_offset=0, counters=None,
                 out=None):
        codes, cnt = O.quantize(x.reshape(-1).numpy(), fmt, mode, seed, block_offset=block_offset)
        if counters is not None:
            counters += torch.from_numpy(cnt)
        t = torch.from_numpy(codes.view(np.int16).copy() if fmt == "fp16"
                             else codes.astype(np.uint8))
        if out is not None:
            out.copy_(t.reshape(out.shape))
            return out
        return t

    def gemm_f32(self, a, b, m, n, k, a_major="k", b_major="n", out=None):
        c = super().gemm_f32(a.reshape(-1), b.reshape(-1), m, n, k, a_major, b_major)
        if out is not None:
            out.copy_(c.reshape(-1))
            return out
        return c

    def gemm_q(self, a, b, m, n, k, a_major="k", b_major="n", counters=None, out=None):
        return self.quantize(self.gemm_f32(a, b, m, n, k, a_major, b_major).reshape(-1),
                             counters=counters, out=out)


def _offsets():
    offs, off = [], 0
    for _, i, o in LAYERS:
        offs.append(off)
        off += (i * o + 4095) // 4096 * 4096
    return offs, off


def _inputs():
    rng = np.random.default_rng(17)
    offs, total = _offsets()
    w = np.zeros(total, np.float32)
    for (_, i, o), a in zip(LAYERS, offs):
        w[a:a + i * o] = _grid(rng, i * o, 0.125, 4)
    xs = [O.quantize(_grid(rng, T * i, 0.25, 4))[0].astype(np.uint8).reshape(T, i)
          for _, i, _ in LAYERS]
    es = [O.quantize(_grid(rng, T * o, 0.5, 4))[0].astype(np.uint8).reshape(T, o)
          for _, _, o in LAYERS]
    return w, xs, es


def _run_stack(xs, es, tokens, w, steps=2):
    st = LinearStack(LAYERS, tokens, torch.from_numpy(w), lr=0.25, mu=0.5,
                     scaler=ConstScale(1.0), ops=StackCpuOps(), master_mode="stochastic", seed=7)
    gates = []
    for it in range(steps):
        _, bwd = st.step([torch.from_numpy(x) for x in xs], [torch.from_numpy(e) for e in es], it)
        gates.append(bwd.numpy().copy())
    return st, gates


def _worker(rank, world, port, mode, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w, xs, es = _inputs()
        tpr = T // world
        xs_r = [x[rank * tpr:(rank + 1) * tpr].copy() for x in xs]
        es_r = [e[rank * tpr:(rank + 1) * tpr].copy() for e in es]
        if mode == "overflow" and rank == 1:
            es_r[1] = O.quantize(np.full(es_r[1].size, 40000.0, np.float32))[0].astype(
                np.uint8).reshape(es_r[1].shape)          # dX = E W^T overflows E5M2
        st, gates = _run_stack(xs_r, es_r, tpr, w, steps=1 if mode == "overflow" else 2)
        out[rank] = (st.master.numpy().copy(), st.w_q.numpy().copy(), st.momentum.numpy().copy(),
                     gates[-1])
    finally:
        dist.destroy_process_group()


def _run(mode):
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, mode, out), nprocs=2, join=True)
    return dict(out)


def test_dp_stack_equals_single_process():
    w, xs, es = _inputs()
    ref, gates = _run_stack(xs, es, T, w)
    assert all(g[0] == 0 and g[2] == 0 for g in gates)
    m0, _ = O.quantize(w, "fp16")
    assert (ref.master.numpy().view(np.uint16) != m0).any()      # the update ran
    res = _run("step")
    for r in range(2):
        master, wq, mom, gate = res[r]
        np.testing.assert_array_equal(master, ref.master.numpy())
        np.testing.assert_array_equal(wq, ref.w_q.numpy())
        np.testing.assert_array_equal(mom.view(np.uint32), ref.momentum.numpy().view(np.uint32))
        assert gate[0] == 0 and gate[2] == 0


def test_dp_stack_overflow_on_one_rank_skips_everywhere():
    w, _, _ = _inputs()
    m0, _ = O.quantize(w, "fp16")
    res = _run("overflow")
    for r in range(2):
        master, _, mom, gate = res[r]
        assert gate[0] > 0
        np.testing.assert_array_equal(master.view(np.uint16), m0)
        assert not mom.any()


def test_transformer_base_shapes():
    layers = transformer_base_layers()
    assert len(layers) == 6 * 4 + 6 * 7 + 1
    params = sum(i * o for _, i, o in layers)
    assert params == 6 * (512 * 1536 + 512 * 512 + 2 * 512 * 2048) + \
        6 * (512 * 1536 + 3 * 512 * 512 + 512 * 1024 + 2 * 512 * 2048) + 512 * 32000
    # ~380 TFLOP per 2^20-token step
    assert abs(linear_flops_per_token(layers) * (1 << 20) / 1e12 - 380) < 15
