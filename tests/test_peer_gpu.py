"""GPU: the data-parallel exchange over peer memory (csrc/peer.cu, peer.py).

* fp8b_peer_reduce_quantize == rank-order FP32 sum + the standalone quantize, on
  several "virtual peers" (buffers of one process: the kernel only sees pointers);
* two PROCESSES on this one GPU (gloo for the control plane, CUDA IPC for the
  data plane; no kernel ever waits on a peer): the ZeRO-1 Dense step over peer
  memory equals the single-process step bit for bit on exact-sum inputs.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fp8():
    import paper_1905_12334_b200 as F
    F.init()
    return F


@pytest.mark.parametrize("world", [1, 2, 5])
@pytest.mark.parametrize("fmt,mode", [("fp8", "nearest-even"), ("fp8", "stochastic"),
                                      ("fp16", "truncate"), ("fp16", "stochastic")])
def test_reduce_quantize_equals_sum_then_quantize(fp8, world, fmt, mode):
    import torch
    from paper_1905_12334_b200.peer import PeerBuffer, reduce_quantize
    n_total, i0, n = 5 * 4096 + 64, 4096, 3 * 4096 + 36
    bufs = [PeerBuffer(4 * n_total) for _ in range(world)]
    parts = []
    for r, b in enumerate(bufs):
        t = b.view().view(torch.float32)
        fp8.fill_synthetic(t, "config2", 50 + r, 0.01)
        t[i0 + 7] = float("nan") if r == 0 else 1.0
        t[i0 + 11] = 1e30 if r == world - 1 else 2.0
        parts.append(t)
    s = parts[0][i0:i0 + n].clone()
    for t in parts[1:]:
        s = s + t[i0:i0 + n]          # rank order, binary32
    cnt = fp8.Counters()
    codes = torch.empty(n, dtype=torch.uint8 if fmt == "fp8" else torch.int16, device="cuda")
    sum_out = torch.empty(n, dtype=torch.float32, device="cuda")
    reduce_quantize([b.ptrs[0] for b in bufs], i0, n, codes, fmt=fmt, mode=mode, seed=77,
                    block_offset=1, counters=cnt, sum_out=sum_out)
    ref = fp8.quantize(s, fmt, mode, 77, bits="counter", block_offset=1)
    assert torch.equal(sum_out.view(torch.int32), s.view(torch.int32))
    assert torch.equal(codes.view(torch.uint8), ref.codes.view(torch.uint8))
    assert cnt.values() == ref.counters.values()
    assert cnt.values()[2] >= 1 and cnt.values()[0] >= 1
    for b in bufs:
        b.close()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _grid(rng, n, step, lim):
    return (rng.integers(-lim, lim + 1, n) * step).astype(np.float32)


def _data(B, I, O_, seed):
    rng = np.random.default_rng(seed)
    return (_grid(rng, B * I, 0.25, 4), _grid(rng, I * O_, 0.125, 4), _grid(rng, B * O_, 0.5, 4))


def _layer_run(F, torch, x, w, e, B, I, O_, world, rank, transport, mm):
    from paper_1905_12334_b200.dp import ZeroDataParallelDense
    m0 = F.quantize(torch.from_numpy(w).cuda(), "fp16").codes
    wq = F.quantize(F.dequantize(F.quantize(torch.from_numpy(w).cuda(), "fp16"))).codes
    bpr = B // world
    sc = F.LossScaler("constant", 1.0)
    layer = ZeroDataParallelDense(m0.reshape(I, O_).clone(), wq.reshape(I, O_).clone(),
                                  batch_per_rank=bpr, lr=0.25, mu=0.5, scaler=sc,
                                  master_mode=mm, seed=9, transport=transport)
    xs = torch.from_numpy(x.reshape(B, I)[rank * bpr:(rank + 1) * bpr].copy()).cuda()
    es = torch.from_numpy(e.reshape(B, O_)[rank * bpr:(rank + 1) * bpr].copy()).cuda()
    for it in range(2):
        qy, qdx, gate = layer.step(xs, es, it)
    return (layer.gather_masters().cpu().numpy().copy(), layer.w_q.cpu().numpy().copy(),
            gate.cpu().numpy().copy())


def _worker(rank, world, port, mm, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_1905_12334_b200 as F
        F.init()
        B, I, O_ = 512, 256, 200   # 51200 params: uneven block shards (7 + 5.5 blocks)
        x, w, e = _data(B, I, O_, 3)
        try:
            out[rank] = _layer_run(F, torch, x, w, e, B, I, O_, world, rank, "peer", mm)
        except RuntimeError as ex:   # no CUDA IPC in this sandbox: report, do not fail
            if "peer_open" in str(ex) or "peer_alloc" in str(ex):
                out[rank] = "noipc: " + str(ex)
                dist.barrier()
            else:
                raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mm", ["nearest-even", "stochastic"])
def test_zero1_peer_two_processes_equal_single_process(fp8, mm):
    import torch
    import torch.multiprocessing as mp
    world = 2
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    ctx = mp.spawn(_worker, args=(world, _free_port(), mm, out), nprocs=world, join=False)
    import time
    deadline = time.time() + 240
    while not ctx.join(timeout=5):
        if time.time() > deadline:   # a sandbox that stalls IPC must not hang the suite
            for p in ctx.processes:
                p.kill()
            pytest.skip("two-process peer run did not finish in 240 s")
    if any(isinstance(out.get(r), str) for r in range(world)):
        pytest.skip("CUDA IPC unavailable here: " + str(out[0]))
    B, I, O_ = 512, 256, 200
    x, w, e = _data(B, I, O_, 3)
    ref = _layer_run(fp8, torch, x, w, e, B, I, O_, 1, 0, "collective", mm)
    for r in range(world):
        np.testing.assert_array_equal(out[r][0], ref[0])   # FP16 masters (gathered)
        np.testing.assert_array_equal(out[r][1], ref[1])   # E5M2 fprop weights
    np.testing.assert_array_equal(out[0][2], out[1][2])    # the all-reduced gate
