"""GPU parity: fused SGD-momentum update into FP16 masters (update_tensor,
nn.cpp:417-432) and the device loss scaler (loss_scaling.cpp) vs the
reference's fixtures and the oracle; bit-exact."""
import json
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
UG = np.load(os.path.join(GOLD, "update_golden.npz"))
UMETA = json.load(open(os.path.join(GOLD, "update_golden.json")))


@pytest.fixture(scope="module")
def fp8():
    import paper_1905_12334_b200 as F
    F.init()
    return F


def _dev(a, dtype=None):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(a))
    return t.to("cuda") if dtype is None else t.to("cuda").view(dtype)


@pytest.mark.parametrize("m", UMETA, ids=lambda m: m["key"])
def test_update_golden(fp8, m):
    import torch
    master = _dev(UG["master0"].view(np.int16))
    mom = _dev(UG["mom0"])
    grad = _dev(UG["grad_e5m2"].astype(np.uint8))
    w8 = torch.empty(master.numel(), dtype=torch.uint8, device="cuda")
    fp8.sgd_momentum_update(grad, "fp8", master, mom, lr=m["lr"], mu=m["mu"],
                            two_lambda=float(np.float32(m["two_lambda"])), scale=m["scale"],
                            master_mode=m["master_mode"], seed=m["seed"], w_e5m2=w8)
    k = m["key"]
    np.testing.assert_array_equal(master.cpu().numpy().view(np.uint16), UG[f"master1_{k}"])
    np.testing.assert_array_equal(mom.cpu().numpy().view(np.uint32), UG[f"mom1_{k}"].view(np.uint32))
    # fused next-fprop weight == Q_RNE(decode(master1)) (nn.cpp:192)
    want, _ = O.quantize(O.dequantize(UG[f"master1_{k}"], "fp16"), "fp8")
    np.testing.assert_array_equal(w8.cpu().numpy(), want.astype(np.uint8))


@pytest.mark.parametrize("bits", ["counter", "supplied"])
@pytest.mark.parametrize("gfmt", ["fp8", "f32"])
def test_update_sr_bits_vs_oracle(fp8, bits, gfmt):
    import torch
    n = 70000 + 3
    r = O.Rand(5)
    master0, _ = O.quantize(r.normal(n, 1 / 32), "fp16")
    mom0 = r.normal(n, 1e-3)
    gf32 = r.normal(n, 1e-2)
    gq, _ = O.quantize(gf32, "fp8")
    g_used = O.dequantize(gq, "fp8") if gfmt == "fp8" else gf32
    rb = np.random.default_rng(2).integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
    master = _dev(master0.view(np.int16))
    mom = _dev(mom0)
    grad = _dev(gq.astype(np.uint8)) if gfmt == "fp8" else _dev(gf32)
    rbt = _dev(rb.view(np.int32)) if bits == "supplied" else None
    cnt = fp8.Counters()
    fp8.sgd_momentum_update(grad, gfmt, master, mom, lr=0.05, mu=0.9, two_lambda=1e-4,
                            scale=1024.0, master_mode="stochastic", bits=bits, seed=31,
                            block_offset=3, rbits=rbt, master_counters=cnt)
    m1, mo1, _, k = O.sgd_update(master0, mom0, g_used, 1024.0, 0.05, 0.9, np.float32(1e-4),
                                 "stochastic", bits, 31, 3, rb if bits == "supplied" else None)
    np.testing.assert_array_equal(master.cpu().numpy().view(np.uint16), m1)
    np.testing.assert_array_equal(mom.cpu().numpy().view(np.uint32), mo1.view(np.uint32))
    assert cnt.values() == tuple(int(v) for v in k)


def test_update_skipped_on_overflow(fp8):
    """Non-finite gradients freeze the parameters (nn.cpp:546, test_nn.cpp:180-199)."""
    import torch
    n = 5000
    master = _dev(UG["master0"][:n].view(np.int16)).clone()
    mom = _dev(UG["mom0"][:n]).clone()
    grad = _dev(UG["grad_e5m2"][:n].astype(np.uint8))
    m_before, mo_before = master.clone(), mom.clone()
    skip = fp8.Counters()
    skip.t[0] = 3  # three overflowing backward Q nodes
    fp8.sgd_momentum_update(grad, "fp8", master, mom, lr=0.1, mu=0.9, scale=8192.0,
                            skip_counters=skip)
    assert torch.equal(master, m_before) and torch.equal(mom, mo_before)
    skip.t.zero_()
    skip.t[2] = 1  # a NaN / non-finite db
    fp8.sgd_momentum_update(grad, "fp8", master, mom, lr=0.1, mu=0.9, scale=8192.0,
                            master_mode="stochastic", seed=3, skip_counters=skip)
    assert torch.equal(master, m_before)
    skip.t.zero_()
    fp8.sgd_momentum_update(grad, "fp8", master, mom, lr=0.1, mu=0.9, scale=8192.0,
                            skip_counters=skip)
    assert not torch.equal(master, m_before)


def test_zero_grads_keep_masters(fp8):
    """test_nn.cpp:133-160: zero weight gradients leave masters bit-identical
    (momentum 0)."""
    import torch
    n = 8000
    master = _dev(UG["master0"][:n].view(np.int16)).clone()
    before = master.clone()
    mom = torch.zeros(n, dtype=torch.float32, device="cuda")
    grad = torch.zeros(n, dtype=torch.uint8, device="cuda")
    for mode in ("nearest-even", "stochastic"):
        fp8.sgd_momentum_update(grad, "fp8", master, mom, lr=0.1, mu=0.9, scale=1024.0,
                                master_mode=mode, seed=4)
        assert torch.equal(master, before)


def test_update_unaligned_and_scaler_scale(fp8):
    import torch
    n = 4099
    master = _dev(UG["master0"][: n + 1].view(np.int16)).clone()[1:]
    mom = _dev(UG["mom0"][: n + 1]).clone()[1:]
    grad = _dev(UG["grad_e5m2"][: n + 1].astype(np.uint8))[1:]
    sc = fp8.LossScaler("dynamic-backoff", 8192.0)
    fp8.sgd_momentum_update(grad, "fp8", master, mom, lr=0.1, mu=0.9, scaler=sc)
    m1, mo1, _, _ = O.sgd_update(UG["master0"][1:n + 1], UG["mom0"][1:n + 1],
                                 O.dequantize(UG["grad_e5m2"][1:n + 1], "fp8"), 8192.0, 0.1, 0.9)
    np.testing.assert_array_equal(master.cpu().numpy().view(np.uint16), m1)


def test_bias_grad(fp8):
    rng = np.random.default_rng(8)
    e = rng.standard_normal((129, 77)).astype(np.float32)
    qe = fp8.quantize(e)
    db = fp8.bias_grad(qe).cpu().numpy()
    want = O.bias_grad(O.dequantize(qe.codes_u16(), "fp8"), 129, 77)
    np.testing.assert_array_equal(db.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("tr", json.load(open(os.path.join(GOLD, "scaler_golden.json"))),
                         ids=lambda t: t["cite"])
def test_loss_scaler_traces(fp8, tr):
    opts = dict(tr["opts"])
    if "min_threshold_schedule" in opts:
        opts["min_threshold_schedule"] = [tuple(v) for v in opts["min_threshold_schedule"]]
    s = fp8.LossScaler(**opts)
    steps = tr["steps"]
    # async path for long traces: drive the device state machine and compare the end
    # state, and step synchronously for the first 64 events
    for finite, it, act, sc in steps[:64]:
        ev = s.step(bool(finite), it)
        assert (ev.action, ev.scale_after) == (act, sc)
    for finite, it, act, sc in steps[64:]:
        s.step_async(bool(finite), it)
    if len(steps) > 64:
        assert s.scale == steps[-1][3]


def test_loss_scaler_reads_device_counters(fp8):
    s = fp8.LossScaler("dynamic-backoff", 1024.0, min_threshold_schedule=[(0, 256.0)])
    c = fp8.Counters()
    c.t[0] = 1
    s.step_async(True, 0, counters=c)  # counters override: overflow -> backoff
    assert s.scale == 512.0
    c.t.zero_()
    s.step_async(False, 1, counters=c)  # clean counters -> finite step
    assert s.scale == 512.0 and s.steps_since_overflow == 1


def test_unscale_true_division(fp8):
    """test_loss_scaling.cpp:156-176: unscale is FP32 true division."""
    s = fp8.LossScaler("constant", 3.0)
    assert float(s.unscale(np.array([9.0], np.float32)).cpu()[0]) == 3.0
    s = fp8.LossScaler("constant", 4096.0)
    u = s.unscale(np.array([4096.0, -8192.0, np.inf, np.nan], np.float32)).cpu().numpy()
    assert u[0] == 1.0 and u[1] == -2.0 and np.isinf(u[2]) and np.isnan(u[3])


@pytest.mark.parametrize("n", [5000, 3 * 4096, 1 << 20, 512 * 4096, 700 * 4096 + 33])
@pytest.mark.parametrize("mode,bits", [("nearest-even", "lfsr"), ("stochastic", "lfsr"),
                                       ("stochastic", "counter")])
@pytest.mark.parametrize("overflow", [False, True])
def test_fused_scaler_step_equals_update_then_step(fp8, n, mode, bits, overflow):
    """step_scaler: the update's last CTA runs LossScaler::step after every CTA
    has read the scale. Masters, momentum, E5M2 W and the whole scaler state
    equal the separate update + fp8b_loss_scaler_step, over several iterations
    (growth, backoff and floor clamps), with the update skipped on overflow."""
    import torch
    rng = np.random.default_rng(n % 1000 + len(mode))
    m0 = O.quantize(rng.normal(0, 1 / 32, n).astype(np.float32), "fp16")[0].view(np.int16)
    g0 = O.quantize(rng.normal(0, 1.0, n).astype(np.float32), "fp8")[0].astype(np.uint8)
    out = []
    for fused in (False, True):
        master, mom, grad = _dev(m0.copy()), _dev(np.zeros(n, np.float32)), _dev(g0)
        w8 = torch.empty(n, dtype=torch.uint8, device="cuda")
        sc = fp8.LossScaler("dynamic-backoff", 65536.0, growth_interval=2,
                            min_threshold_schedule=[(0, 8192.0), (3, 32768.0)])
        gate = fp8.Counters()
        trace = []
        for it in range(6):
            gate.zero_()
            if overflow and it in (1, 4):
                gate.t[0] = 3  # an overflow count: update skipped, scale backs off
            kw = dict(lr=0.05, mu=0.9, scaler=sc, skip_counters=gate, master_mode=mode, bits=bits,
                      seed=9 + it, w_e5m2=w8)
            if fused:
                fp8.sgd_momentum_update(grad, "fp8", master, mom, step_scaler_iteration=it, **kw)
            else:
                fp8.sgd_momentum_update(grad, "fp8", master, mom, **kw)
                sc.step_async(True, it, counters=gate)
            trace.append(sc.state.cpu().numpy().tobytes())
        out.append((master.cpu().numpy(), mom.cpu().numpy().view(np.uint32), w8.cpu().numpy(), trace))
    a, b = out
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])
    np.testing.assert_array_equal(a[2], b[2])
    assert a[3] == b[3]


@pytest.mark.parametrize("n", [3 * 4096 + 5, 512 * 4096])
def test_merged_gate_two_counter_sets(fp8, n):
    """skip_counters2 / gate_out: the update is gated on the sum of two counter
    sets (the step's forward-side and wgrad-side Q nodes), and its last CTA stores
    the merged gate and steps the scaler on it -- equal to a merge, an update and
    a step done separately."""
    import torch
    rng = np.random.default_rng(n % 977)
    m0 = O.quantize(rng.normal(0, 1 / 32, n).astype(np.float32), "fp16")[0].view(np.int16)
    g0 = O.quantize(rng.normal(0, 1.0, n).astype(np.float32), "fp8")[0].astype(np.uint8)
    for c1, c2 in [((0, 4, 0), (0, 1, 0)), ((0, 0, 0), (2, 0, 0)), ((0, 0, 1), (0, 0, 0))]:
        res = []
        for fused in (False, True):
            master, mom, grad = _dev(m0.copy()), _dev(np.zeros(n, np.float32)), _dev(g0)
            sc = fp8.LossScaler("dynamic-backoff", 65536.0, growth_interval=1,
                                min_threshold_schedule=[(0, 8192.0)])
            a, b, gate = fp8.Counters(), fp8.Counters(), fp8.Counters()
            a.t.copy_(torch.tensor(c1)); b.t.copy_(torch.tensor(c2))
            kw = dict(lr=0.05, mu=0.9, scaler=sc, master_mode="stochastic", seed=3)
            if fused:
                fp8.sgd_momentum_update(grad, "fp8", master, mom, skip_counters=a, skip_counters2=b,
                                        gate_out=gate, step_scaler_iteration=7, **kw)
            else:
                gate.t.copy_(a.t + b.t)
                fp8.sgd_momentum_update(grad, "fp8", master, mom, skip_counters=gate, **kw)
                sc.step_async(True, 7, counters=gate)
            res.append((master.cpu().numpy(), mom.cpu().numpy().view(np.uint32), gate.values(),
                        sc.state.cpu().numpy().tobytes()))
        assert res[0][2] == res[1][2] == tuple(x + y for x, y in zip(c1, c2))
        np.testing.assert_array_equal(res[0][0], res[1][0])
        np.testing.assert_array_equal(res[0][1], res[1][1])
        assert res[0][3] == res[1][3]


@pytest.mark.parametrize("n", [5000, 700 * 4096 + 33])
def test_fused_step_clears_gate_inputs(fp8, n):
    """clear_skip_counters (step_scaler = 2): after the update and the fused
    scaler step the gate's input counters are zero again, the merged gate is in
    gate_out, and masters / momentum / scaler state equal the non-clearing run."""
    import torch
    rng = np.random.default_rng(n % 911)
    m0 = O.quantize(rng.normal(0, 1 / 32, n).astype(np.float32), "fp16")[0].view(np.int16)
    g0 = O.quantize(rng.normal(0, 1.0, n).astype(np.float32), "fp8")[0].astype(np.uint8)
    res = []
    for clear in (False, True):
        master, mom, grad = _dev(m0.copy()), _dev(np.zeros(n, np.float32)), _dev(g0)
        sc = fp8.LossScaler("dynamic-backoff", 65536.0, growth_interval=2,
                            min_threshold_schedule=[(0, 8192.0)])
        a, b, gate = fp8.Counters(), fp8.Counters(), fp8.Counters()
        for it, (c1, c2) in enumerate([((0, 3, 0), (0, 1, 0)), ((1, 0, 0), (0, 0, 0)),
                                       ((0, 0, 0), (0, 2, 0))]):
            a.t.copy_(torch.tensor(c1)); b.t.copy_(torch.tensor(c2))
            fp8.sgd_momentum_update(grad, "fp8", master, mom, lr=0.05, mu=0.9, scaler=sc,
                                    skip_counters=a, skip_counters2=b, gate_out=gate,
                                    master_mode="stochastic", seed=3 + it,
                                    step_scaler_iteration=it, clear_skip_counters=clear)
            assert gate.values() == tuple(x + y for x, y in zip(c1, c2))
            if clear:
                assert a.values() == (0, 0, 0) and b.values() == (0, 0, 0)
            else:
                assert a.values() == c1 and b.values() == c2
        res.append((master.cpu().numpy(), mom.cpu().numpy().view(np.uint32),
                    sc.state.cpu().numpy().tobytes()))
    np.testing.assert_array_equal(res[0][0], res[1][0])
    np.testing.assert_array_equal(res[0][1], res[1][1])
    assert res[0][2] == res[1][2]
