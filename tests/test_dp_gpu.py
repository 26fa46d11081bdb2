"""GPU: the data-parallel layers on this library's kernels (single process).

ZeroDataParallelDense (sharded masters/momentum, block_offset updates) and
DataParallelDense (replicated) run the same step on the same device and must
agree bit for bit; both must match the fused fp8b_dense_step layer's masters.
(The multi-rank orchestration is covered by tests/test_dp_gloo.py.)"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("master_mode", ["nearest-even", "stochastic"])
def test_zero1_equals_replicated_on_gpu(master_mode):
    import torch
    import paper_1905_12334_b200 as F
    from paper_1905_12334_b200.dp import DataParallelDense, ZeroDataParallelDense
    F.init()
    B, I, Ou = 256, 512, 384
    rng = np.random.default_rng(1)
    w = (rng.standard_normal(I * Ou) / 20).astype(np.float32)
    x = torch.from_numpy(rng.standard_normal(B * I).astype(np.float32)).cuda()
    e = torch.from_numpy((rng.standard_normal(B * Ou) * 0.01 * 8192).astype(np.float32)).cuda()
    m0 = F.quantize(torch.from_numpy(w).cuda(), "fp16").codes.reshape(I, Ou)
    wq0 = F.quantize(F.dequantize(F.QuantizedTensor(m0.reshape(-1), [I * Ou], 1, 0, F.Counters())),
                     "fp8").codes.reshape(I, Ou)
    sc1, sc2 = F.LossScaler("constant", 8192.0), F.LossScaler("constant", 8192.0)
    rep = DataParallelDense(m0.clone(), wq0.clone(), batch_per_rank=B, lr=0.1, mu=0.9, scaler=sc1,
                            master_mode=master_mode, seed=5)
    zero = ZeroDataParallelDense(m0.clone(), wq0.clone(), batch_per_rank=B, lr=0.1, mu=0.9,
                                 scaler=sc2, master_mode=master_mode, seed=5)
    for it in range(3):
        ya, dxa, _ = rep.step(x, e, it)
        yb, dxb, _ = zero.step(x, e, it)
        assert torch.equal(ya, yb) and torch.equal(dxa, dxb)
    torch.cuda.synchronize()
    assert torch.equal(rep.w_master, zero.gather_masters())
    assert torch.equal(rep.w_q, zero.w_q)
    assert not torch.equal(rep.w_master, m0)  # the steps did update
