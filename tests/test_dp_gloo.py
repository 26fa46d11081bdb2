"""CPU, world_size 2 over gloo: the multi-rank orchestration of the FP8 path
(paper_1905_12334_b200/dp.py) with the oracle standing in for the kernels.

* block-aligned sharding + block_offset reproduces the single-process SR stream;
* the data-parallel Dense step (FP32 dW all-reduce before Q(dW), all-reduced
  overflow gate, replicated update) equals the single-process reference recipe
  on inputs whose FP32 sums are exact (so summation order cannot matter);
* one rank overflowing makes every rank skip the update.
"""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1905_12334_b200.dp import DataParallelDense, ZeroDataParallelDense, block_shard


class CpuOps:
    """Oracle-backed stand-in for GpuOps (test infrastructure only)."""
    device = torch.device("cpu")

    def counters(self):
        return torch.zeros(3, dtype=torch.int64)

    @staticmethod
    def ctensor(c):
        return c

    def quantize(self, x, fmt="fp8", mode="nearest-even", seed=1, block_offset=0, counters=None):
        codes, cnt = O.quantize(x.numpy(), fmt, mode, seed, block_offset=block_offset)
        if counters is not None:
            counters += torch.from_numpy(cnt)
        return torch.from_numpy(codes.astype(np.uint8))

    @staticmethod
    def _mat(codes, rows, cols, major_is_inner):
        a = codes.numpy().astype(np.uint16)
        return a.reshape(rows, cols) if major_is_inner else a.reshape(cols, rows).T.copy()

    def gemm_f32(self, a, b, m, n, k, a_major="k", b_major="n"):
        A = self._mat(a, m, k, a_major == "k")
        B = self._mat(b, k, n, b_major == "n")
        return torch.from_numpy(O.gemm(A, B, m, k, n).copy())

    def gemm_q(self, a, b, m, n, k, a_major="k", b_major="n", counters=None):
        return self.quantize(self.gemm_f32(a, b, m, n, k, a_major, b_major).reshape(-1),
                             counters=counters)

    def update(self, qdw, master, momentum, *, lr, mu, two_lambda, scaler, skip_counters,
               master_mode, seed, w_e5m2=None, block_offset=0):
        if int(skip_counters[0] + skip_counters[2]) != 0:
            return
        m1, mo1, _, _ = O.sgd_update(master.numpy().view(np.uint16), momentum.numpy(),
                                     O.dequantize(qdw.numpy().astype(np.uint16)), scaler.scale,
                                     lr, mu, np.float32(two_lambda), master_mode, "lfsr", seed,
                                     block_offset=block_offset)
        master.copy_(torch.from_numpy(m1.view(np.int16)))
        momentum.copy_(torch.from_numpy(mo1))
        if w_e5m2 is not None:
            q, _ = O.quantize(O.dequantize(m1, "fp16"))
            w_e5m2.copy_(torch.from_numpy(q.astype(np.uint8)))


class ConstScale:
    def __init__(self, s):
        self.scale = s


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _grid(rng, n, step, lim):
    return (rng.integers(-lim, lim + 1, n) * step).astype(np.float32)


def _data(B=8, I=64, O_=32, seed=0):
    rng = np.random.default_rng(seed)
    x = _grid(rng, B * I, 0.25, 4)        # |x| <= 1, multiples of 1/4
    w = _grid(rng, I * O_, 0.125, 4)      # |w| <= 0.5, exact in E5M2 and FP16
    e = _grid(rng, B * O_, 0.5, 4)        # |e| <= 2
    return x, w, e


def _worker(rank, world, port, mode, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if mode == "shard":
            n = 3 * 4096 + 123
            x = np.random.default_rng(5).standard_normal(n).astype(np.float32)
            s, e, boff = block_shard(n, world, rank)
            codes, _ = O.quantize(x[s:e], "fp8", "stochastic", 77, block_offset=boff)
            gathered = [None] * world
            dist.all_gather_object(gathered, codes)
            out[rank] = np.concatenate(gathered)
        elif mode.startswith("zero"):
            B, I, O_ = 8, 64, 200  # 12800 params: uneven block shards (2 + 1.125 blocks)
            x, w, e = _data(B, I, O_, seed=3)
            mm = "stochastic" if mode.endswith("sr") else "nearest-even"
            if mode.endswith("overflow") and rank == 0:
                e = e * np.float32(1e6)
            m0, _ = O.quantize(w, "fp16")
            wq, _ = O.quantize(O.dequantize(m0, "fp16"))
            bpr = B // world
            layer = ZeroDataParallelDense(
                torch.from_numpy(m0.view(np.int16).reshape(I, O_)).clone(),
                torch.from_numpy(wq.astype(np.uint8).reshape(I, O_)).clone(),
                batch_per_rank=bpr, lr=0.25, mu=0.5, scaler=ConstScale(1.0), ops=CpuOps(),
                master_mode=mm, seed=9)
            xs = torch.from_numpy(x.reshape(B, I)[rank * bpr:(rank + 1) * bpr].copy())
            es = torch.from_numpy(e.reshape(B, O_)[rank * bpr:(rank + 1) * bpr].copy())
            for it in range(2):
                qy, qdx, gate = layer.step(xs, es, it)
            out[rank] = (layer.gather_masters().numpy().copy(), layer.w_q.numpy().copy(),
                         qdx.numpy().copy(), gate.numpy().copy(),
                         (layer.start, layer.end, layer.block_offset))
        else:
            B, I, O_ = 8, 64, 32
            x, w, e = _data(B, I, O_)
            if mode == "overflow" and rank == 1:
                e = e * np.float32(1e6)  # this rank's Q(e) overflows
            m0, _ = O.quantize(w, "fp16")
            wq, _ = O.quantize(O.dequantize(m0, "fp16"))
            bpr = B // world
            layer = DataParallelDense(torch.from_numpy(m0.view(np.int16).reshape(I, O_)).clone(),
                                      torch.from_numpy(wq.astype(np.uint8).reshape(I, O_)).clone(),
                                      batch_per_rank=bpr, lr=0.25, mu=0.5,
                                      scaler=ConstScale(1.0), ops=CpuOps())
            xs = torch.from_numpy(x.reshape(B, I)[rank * bpr:(rank + 1) * bpr].copy())
            es = torch.from_numpy(e.reshape(B, O_)[rank * bpr:(rank + 1) * bpr].copy())
            qy, qdx, gate = layer.step(xs, es, 0)
            out[rank] = (layer.w_master.numpy().copy(), qy.numpy().copy(), qdx.numpy().copy(),
                         gate.numpy().copy())
    finally:
        dist.destroy_process_group()


def _run(mode):
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, mode, out), nprocs=world, join=True)
    return dict(out)


def test_block_shards_reproduce_single_process_sr_stream():
    res = _run("shard")
    n = 3 * 4096 + 123
    x = np.random.default_rng(5).standard_normal(n).astype(np.float32)
    whole, _ = O.quantize(x, "fp8", "stochastic", 77)
    for r in range(2):
        np.testing.assert_array_equal(res[r], whole)


def test_dp_dense_step_equals_single_process():
    res = _run("step")
    B, I, O_ = 8, 64, 32
    x, w, e = _data(B, I, O_)
    # single-process reference recipe (nn.cpp:187-203, 294-326, 417-432)
    m0, _ = O.quantize(w, "fp16")
    qw, _ = O.quantize(O.dequantize(m0, "fp16"))
    qx, _ = O.quantize(x)
    qy, _ = O.quantize(O.gemm(qx, qw, B, I, O_))
    qe, _ = O.quantize(e)
    qdw, _ = O.quantize(O.gemm(qx.reshape(B, I).T.copy(), qe, I, B, O_))
    qdx, _ = O.quantize(O.gemm(qe, qw.reshape(I, O_).T.copy(), B, O_, I))
    m1, _, _, _ = O.sgd_update(m0, np.zeros(I * O_, np.float32), O.dequantize(qdw), 1.0, 0.25,
                               0.5)
    for r in range(2):
        wm, qy_r, qdx_r, gate = res[r]
        np.testing.assert_array_equal(wm.reshape(-1).view(np.uint16), m1)
        np.testing.assert_array_equal(qy_r.reshape(-1),
                                      qy.reshape(B, O_)[r * 4:(r + 1) * 4].reshape(-1))
        np.testing.assert_array_equal(qdx_r.reshape(-1),
                                      qdx.reshape(B, I)[r * 4:(r + 1) * 4].reshape(-1))
        assert gate[0] == 0 and gate[2] == 0


def test_overflow_on_one_rank_skips_everywhere():
    res = _run("overflow")
    _, w, _ = _data()
    m0, _ = O.quantize(w, "fp16")
    for r in range(2):
        wm, _, _, gate = res[r]
        assert gate[0] > 0
        np.testing.assert_array_equal(wm.reshape(-1).view(np.uint16), m0)


def test_block_shard_partition():
    for n in (1, 4095, 4096, 4097, 5 * 4096 + 1):
        for world in (1, 2, 3, 8):
            covered = []
            for r in range(world):
                s, e, b0 = block_shard(n, world, r)
                assert s == min(b0 * 4096, n) and (s % 4096 == 0 or s == n)
                covered += list(range(s, e))
            assert covered == list(range(n))


def _zero_reference(master_mode, steps=2):
    """Single-process recipe for the ZeRO test (two steps, same batch)."""
    B, I, O_ = 8, 64, 200
    x, w, e = _data(B, I, O_, seed=3)
    m, _ = O.quantize(w, "fp16")
    mom = np.zeros(I * O_, np.float32)
    qx, _ = O.quantize(x)
    qe, _ = O.quantize(e)
    for _ in range(steps):
        qw, _ = O.quantize(O.dequantize(m, "fp16"))
        qdw, _ = O.quantize(O.gemm(qx.reshape(B, I).T.copy(), qe, I, B, O_))
        m, mom, _, _ = O.sgd_update(m, mom, O.dequantize(qdw), 1.0, 0.25, 0.5,
                                    master_mode=master_mode, seed=9)
    qw, _ = O.quantize(O.dequantize(m, "fp16"))
    return m, qw


def test_zero1_step_equals_single_process_rne():
    res = _run("zero_rne")
    m, qw = _zero_reference("nearest-even")
    shards = sorted(res[r][4] for r in range(2))
    assert shards == [(0, 8192, 0), (8192, 12800, 2)]
    for r in range(2):
        wm, wq, _, gate = res[r][:4]
        np.testing.assert_array_equal(wm.reshape(-1).view(np.uint16), m)
        np.testing.assert_array_equal(wq.reshape(-1), qw)
        assert gate[0] == 0 and gate[2] == 0


def test_zero1_step_sr_master_stream_is_unsharded():
    """Each shard's SR update draws the unsharded LFSR block streams (block_offset)."""
    res = _run("zero_sr")
    m, qw = _zero_reference("stochastic")
    for r in range(2):
        wm, wq = res[r][:2]
        np.testing.assert_array_equal(wm.reshape(-1).view(np.uint16), m)
        np.testing.assert_array_equal(wq.reshape(-1), qw)


def test_zero1_overflow_on_one_rank_skips_all_shards():
    res = _run("zero_overflow")
    _, w, _ = _data(8, 64, 200, seed=3)
    m0, _ = O.quantize(w, "fp16")
    qw0, _ = O.quantize(O.dequantize(m0, "fp16"))
    for r in range(2):
        wm, wq, _, gate = res[r][:4]
        assert gate[0] > 0
        np.testing.assert_array_equal(wm.reshape(-1).view(np.uint16), m0)
        np.testing.assert_array_equal(wq.reshape(-1), qw0)


def test_zero1_rejects_unknown_transport():
    import pytest
    w = torch.zeros(8, 8, dtype=torch.int16)
    with pytest.raises(ValueError):
        ZeroDataParallelDense(w, w.to(torch.uint8), batch_per_rank=2, lr=0.1, mu=0.9,
                              ops=CpuOps(), transport="carrier-pigeon")
