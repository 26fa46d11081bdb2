"""GPU parity for the config-1 Dense layer step (BASELINE
configs[0]): X[512x1024], W[1024x1024] ~ N(0, 1/1024), dY ~ N(0, 1e-4) scaled by
2^13, E5M2 RNE Q nodes, SGD-momentum 0.9 / lr 0.1, FP16 masters.

Known answers come from the reference library (tests/golden/config1_golden.json,
written by tests/golden/gen_golden.py). With the sequential GEMM engine every
tensor of the step is bit-identical to the reference; with the tcgen05 engine
the Q nodes fed by a GEMM may differ only by boundary flips (counted)."""
import json
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "config1_golden.json")))


@pytest.fixture(scope="module")
def fp8():
    import paper_1905_12334_b200 as F
    F.init()
    return F


@pytest.fixture(scope="module")
def inputs():
    r = O.Rand(0)
    X = r.normal(524288)
    W = r.normal(1048576, 1 / 32)
    dY = r.normal(524288, 0.01)
    E = (dY * np.float32(8192.0)).astype(np.float32)
    assert f"{O.fnv1a64(X):016x}" == GOLD["X"]
    return X, W, E


def H(t):
    return f"{O.fnv1a64(t.contiguous().cpu().numpy()):016x}"


def _layer(fp8, W, engine, master_mode, scale=8192.0):
    import torch
    sc = fp8.LossScaler("constant", scale)
    return fp8.DenseLayer(torch.from_numpy(W.reshape(1024, 1024)).cuda(), batch=512, lr=0.1,
                          mu=0.9, scaler=sc, engine=engine, master_mode=master_mode, seed=1)


@pytest.mark.parametrize("master_mode", ["nearest-even", "stochastic"])
def test_config1_step_sequential_engine_bit_exact(fp8, inputs, master_mode):
    import torch
    X, W, E = inputs
    L = _layer(fp8, W, "sequential", master_mode)
    assert H(L.w_master) == GOLD["master0"]
    assert H(L.w_q) == GOLD["qW"]
    L.step(torch.from_numpy(X).cuda(), torch.from_numpy(E).cuda(), 0)
    torch.cuda.synchronize()
    for name, t in [("qX", L.qx), ("qY", L.qy), ("qE", L.qe), ("qdW", L.qdw), ("qdX", L.qdx)]:
        assert H(t) == GOLD[name], name
    c = L.counters.tolist()
    f = L.fwd_counters.tolist()
    g = GOLD["counters"]
    assert f[:2] == [g["qX"][0] + g["qY"][0], g["qX"][1] + g["qY"][1]]
    assert c[3:5] == g["qdW"] and [c[0], c[1]] == [g["qE"][0] + g["qdX"][0], g["qE"][1] + g["qdX"][1]]
    assert L.grads_finite() == bool(GOLD["grads_finite"])
    assert H(L.w_momentum) == GOLD["momentum1"]
    if master_mode == "nearest-even":
        assert H(L.w_master) == GOLD["master1_rne"]
    else:
        assert H(L.w_master) == GOLD["master1_sr1"]
        assert H(L.w_q) == GOLD["qW1"]


def test_config1_step_tensor_engine(fp8, inputs):
    """tcgen05 engine: input Q nodes and masters' inputs exact; GEMM-fed Q nodes
    may flip only at rounding boundaries (compared with the bit-exact step)."""
    import torch
    X, W, E = inputs
    xs, es = torch.from_numpy(X).cuda(), torch.from_numpy(E).cuda()
    Lt = _layer(fp8, W, "tensor", "nearest-even")
    Ls = _layer(fp8, W, "sequential", "nearest-even")
    Lt.step(xs, es, 0)
    Ls.step(xs, es, 0)
    torch.cuda.synchronize()
    assert H(Lt.qx) == GOLD["qX"] and H(Lt.qe) == GOLD["qE"]
    for a, b in [(Lt.qy, Ls.qy), (Lt.qdw, Ls.qdw), (Lt.qdx, Ls.qdx)]:
        diff = (a != b)
        nflip = int(diff.sum())
        assert nflip <= a.numel() * 1e-3, nflip
        if nflip:  # adjacent codes only
            d = (a[diff].to(torch.int32) - b[diff].to(torch.int32)).abs()
            assert int(d.max()) == 1
    assert Lt.grads_finite()


def test_overflow_skips_update_and_backs_off(fp8, inputs):
    """A huge loss scale overflows every backward Q node: the update is skipped on
    device and the dynamic scaler backs off (nn.cpp:546-547, test_nn.cpp:180-199)."""
    import torch
    X, W, E = inputs
    sc = fp8.LossScaler("dynamic-backoff", 2.0 ** 40, min_threshold_schedule=[(0, 8192.0)])
    L = fp8.DenseLayer(torch.from_numpy(W.reshape(1024, 1024)).cuda(), batch=512, lr=0.1, mu=0.9,
                       scaler=sc, engine="tensor")
    before = L.w_master.clone()
    big = torch.from_numpy(E).cuda() * (2.0 ** 27)  # errors scaled by 2^40 overall
    L.step(torch.from_numpy(X).cuda(), big, 7)
    torch.cuda.synchronize()
    assert not L.grads_finite() and L.overflow_count() > 0
    assert torch.equal(L.w_master, before)
    assert sc.scale == 2.0 ** 39


def test_step_with_bias_matches_reference_order(fp8):
    """Bias path: y += b in FP32 after the sum (nn.cpp:195-198), db = row-order
    column sums of dequant(qe) (nn.cpp:308-314), bias update without 2λ."""
    import torch
    rng = np.random.default_rng(3)
    B_, I_, O_ = 64, 128, 96
    x = rng.standard_normal(B_ * I_).astype(np.float32)
    w = (rng.standard_normal(I_ * O_) / np.sqrt(I_)).astype(np.float32)
    b = (rng.standard_normal(O_) * 0.1).astype(np.float32)
    e = (rng.standard_normal(B_ * O_) * 0.01 * 1024).astype(np.float32)
    sc = fp8.LossScaler("constant", 1024.0)
    L = fp8.DenseLayer(torch.from_numpy(w.reshape(I_, O_)).cuda(), torch.from_numpy(b).cuda(),
                       batch=B_, lr=0.05, mu=0.9, two_lambda=2e-4, scaler=sc, engine="sequential",
                       want_y=True)
    L.step(torch.from_numpy(x).cuda(), torch.from_numpy(e).cuda(), 0)
    torch.cuda.synchronize()
    # oracle composition
    m0, _ = O.quantize(w, "fp16")
    bm0, _ = O.quantize(b, "fp16")
    qx, _ = O.quantize(x)
    qw, _ = O.quantize(O.dequantize(m0, "fp16"))
    y = O.gemm(qx, qw, B_, I_, O_) + O.dequantize(bm0, "fp16")[None, :]
    np.testing.assert_array_equal(L.y.cpu().numpy().view(np.uint32), y.astype(np.float32).view(np.uint32))
    qe, _ = O.quantize(e)
    db = O.bias_grad(O.dequantize(qe), B_, O_)
    np.testing.assert_array_equal(L.db.cpu().numpy().view(np.uint32), db.view(np.uint32))
    dw = O.gemm(qx.reshape(B_, I_).T.copy(), qe, I_, B_, O_)
    qdw, _ = O.quantize(dw)
    m1, _, _, _ = O.sgd_update(m0, np.zeros(I_ * O_, np.float32), O.dequantize(qdw), 1024.0, 0.05,
                               0.9, np.float32(2e-4))
    bm1, _, _, _ = O.sgd_update(bm0, np.zeros(O_, np.float32), db, 1024.0, 0.05, 0.9, 0.0)
    np.testing.assert_array_equal(L.w_master.cpu().numpy().view(np.uint16).reshape(-1), m1)
    np.testing.assert_array_equal(L.b_master.cpu().numpy().view(np.uint16), bm1)


def test_step_cuda_graph_replay(fp8, inputs):
    """The whole step is capturable: graph replays == eager steps."""
    import torch
    X, W, E = inputs
    xs, es = torch.from_numpy(X).cuda(), torch.from_numpy(E).cuda()
    La = _layer(fp8, W, "tensor", "stochastic")
    Lb = _layer(fp8, W, "tensor", "stochastic")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        Lb.step(xs, es, 0)  # warm (TMA descriptors, LFSR tables)
    torch.cuda.synchronize()
    La.step(xs, es, 0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        Lb.step(xs, es, 1)
    g.replay()
    La.step(xs, es, 1)
    torch.cuda.synchronize()
    assert torch.equal(La.w_master, Lb.w_master) and torch.equal(La.w_q, Lb.w_q)


def test_checkpoint_resume_is_exact(fp8, inputs, tmp_path):
    """save_checkpoint/load_checkpoint (nn.cpp:632-701) + momentum and scaler
    state (extension): a resumed layer continues bit for bit."""
    import torch
    X, W, E = inputs
    xs, es = torch.from_numpy(X).cuda(), torch.from_numpy(E).cuda()
    sa = fp8.LossScaler("dynamic-backoff", 8192.0, growth_interval=2,
                        min_threshold_schedule=[(0, 4096.0)])
    A = fp8.DenseLayer(torch.from_numpy(W.reshape(1024, 1024)).cuda(), torch.zeros(1024).cuda(),
                       batch=512, lr=0.1, mu=0.9, scaler=sa, engine="tensor",
                       master_mode="stochastic", seed=3)
    for it in range(3):
        A.step(xs, es, it)
    torch.cuda.synchronize()
    fp8.save_checkpoint([A], tmp_path, scaler=sa)
    assert (tmp_path / "manifest.txt").read_text().startswith("layer 0 kind=dense precision=fp8")
    # the master file is a reference-readable FP16 code tensor
    codes, fmt, _ = O.ref_fp8t_load_codes(tmp_path / "layer0_w.fp8t", cap=1 << 21)
    assert fmt == "fp16" and codes.shape == (1024, 1024)
    np.testing.assert_array_equal(codes.reshape(-1), A.w_master.cpu().numpy().view(np.uint16).reshape(-1))
    sb = fp8.LossScaler("dynamic-backoff", 1.0, growth_interval=2,
                        min_threshold_schedule=[(0, 4096.0)])
    B = fp8.DenseLayer(torch.zeros(1024, 1024).cuda(), torch.ones(1024).cuda(), batch=512, lr=0.1,
                       mu=0.9, scaler=sb, engine="tensor", master_mode="stochastic", seed=3)
    fp8.load_checkpoint([B], tmp_path, scaler=sb)
    assert sb.scale == sa.scale
    for it in range(3, 6):
        A.step(xs, es, it)
        B.step(xs, es, it)
    torch.cuda.synchronize()
    assert torch.equal(A.w_master, B.w_master) and torch.equal(A.w_momentum, B.w_momentum)
    assert torch.equal(A.b_master, B.b_master) and torch.equal(A.w_q, B.w_q)
    assert sa.scale == sb.scale


def test_step_first_call_inside_capture(fp8, inputs):
    """A host thread whose first step is captured into a CUDA graph (no side
    stream may be created during capture) runs both branches on the caller's
    stream; replays equal eager steps."""
    import threading

    import torch
    X, W, E = inputs
    xs, es = torch.from_numpy(X).cuda(), torch.from_numpy(E).cuda()
    La = _layer(fp8, W, "tensor", "stochastic")
    Lb = _layer(fp8, W, "tensor", "stochastic")
    La.step(xs, es, 0)  # warms the process-wide state (TMA descriptors, LFSR tables)
    torch.cuda.synchronize()
    err = []

    def worker():
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                Lb.step(xs, es, 0)
            g.replay()
            torch.cuda.synchronize()
        except Exception as e:  # noqa: BLE001
            err.append(e)

    t = threading.Thread(target=worker)
    t.start()
    t.join()
    assert not err, err
    assert torch.equal(La.w_master, Lb.w_master) and torch.equal(La.w_q, Lb.w_q)
