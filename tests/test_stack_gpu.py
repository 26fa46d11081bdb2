"""GPU parity of the FP8 linear stack (stack.py, BASELINE config 5's caller):
the stack on this library's kernels (tcgen05 GEMMs with fused Q(Y) / Q(dX) /
Q(dW) epilogues, one flat SR master update, device loss scaler) equals the
same orchestration on the CPU oracle, bit for bit, on inputs whose FP32 sums
are exact: step-1 outputs and gates, masters / E5M2 weights / momentum after
two steps."""
import numpy as np
import pytest
import torch

import oracle as O
from test_stack_gloo import StackCpuOps, _grid

pytestmark = pytest.mark.gpu

LAYERS = [("a", 128, 384), ("b", 384, 128), ("c", 128, 640)]
T = 512


def _inputs():
    rng = np.random.default_rng(23)
    offs, off = [], 0
    for _, i, o in LAYERS:
        offs.append(off)
        off += (i * o + 4095) // 4096 * 4096
    w = np.zeros(off, np.float32)
    for (_, i, o), a in zip(LAYERS, offs):
        w[a:a + i * o] = _grid(rng, i * o, 0.125, 4)
    xs = [O.quantize(_grid(rng, T * i, 0.25, 4))[0].astype(np.uint8).reshape(T, i)
          for _, i, _ in LAYERS]
    es = [O.quantize(_grid(rng, T * o, 0.5, 4))[0].astype(np.uint8).reshape(T, o)
          for _, _, o in LAYERS]
    return w, xs, es


class _Const:
    def __init__(self, s):
        self.scale = s


def test_stack_gpu_equals_oracle_orchestration():
    import paper_1905_12334_b200 as F
    from paper_1905_12334_b200.stack import LinearStack
    F.init()
    w, xs, es = _inputs()
    # CPU oracle run
    ref = LinearStack(LAYERS, T, torch.from_numpy(w), lr=0.25, mu=0.5, scaler=_Const(1.0),
                      ops=StackCpuOps(), master_mode="stochastic", seed=7)
    ys_c = [torch.zeros(T * o, dtype=torch.uint8) for _, _, o in LAYERS]
    dxs_c = [torch.zeros(T * i, dtype=torch.uint8) for _, i, _ in LAYERS]
    xs_c = [torch.from_numpy(x) for x in xs]
    es_c = [torch.from_numpy(e) for e in es]
    f_c, b_c = ref.step(xs_c, es_c, 0, ys=ys_c, dxs=dxs_c)
    ref.step(xs_c, es_c, 1)
    # GPU run (device scaler: constant 1.0)
    scaler = F.LossScaler("constant", 1.0)
    st = LinearStack(LAYERS, T, torch.from_numpy(w).cuda(), lr=0.25, mu=0.5, scaler=scaler,
                     master_mode="stochastic", seed=7)
    ys = [torch.zeros(T * o, dtype=torch.uint8, device="cuda") for _, _, o in LAYERS]
    dxs = [torch.zeros(T * i, dtype=torch.uint8, device="cuda") for _, i, _ in LAYERS]
    xs_d = [x.cuda() for x in xs_c]
    es_d = [e.cuda() for e in es_c]
    f_g, b_g = st.step(xs_d, es_d, 0, ys=ys, dxs=dxs)
    for l in range(len(LAYERS)):
        np.testing.assert_array_equal(ys[l].cpu().numpy(), ys_c[l].numpy())
        np.testing.assert_array_equal(dxs[l].cpu().numpy(), dxs_c[l].numpy())
    assert f_g.values() == tuple(int(v) for v in f_c)
    assert b_g.values() == tuple(int(v) for v in b_c)
    st.step(xs_d, es_d, 1)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(st.master.cpu().numpy(), ref.master.numpy())
    np.testing.assert_array_equal(st.w_q.cpu().numpy(), ref.w_q.numpy())
    np.testing.assert_array_equal(st.momentum.cpu().numpy().view(np.uint32),
                                  ref.momentum.numpy().view(np.uint32))
