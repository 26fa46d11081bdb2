"""CPU: pin the oracle restatement (oracle/fp8_oracle.c) against the reference's
frozen known answers and against fixtures produced by the reference itself
(tests/golden/gen_golden.py). When the compiled reference is present
(oracle/_ref, build container only) it is also compared directly."""
import json
import math
import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _f(v):
    return {"nan": math.nan, "inf": math.inf, "-inf": -math.inf}.get(v, v) if isinstance(v, str) else v


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


KA = _load("known_answers.json")


@pytest.mark.parametrize("case", KA["encode"], ids=lambda c: f"{c['fmt']}-{c['mode']}-{c['x']}")
def test_known_encode(case):
    x = _f(case["x"])
    st = 1
    code, ovf, unf = O.encode(x, case["fmt"], case["mode"], lfsr_state=st,
                              saturate=bool(case["saturate"]))
    assert (code, int(ovf), int(unf)) == (case["code"], case["overflowed"], case["underflowed"]), case["cite"]
    bits = int(np.array([x], dtype=np.float32).view(np.uint32)[0])
    c2, o2, u2, _ = O.encode_bits(bits, case["fmt"], case["mode"], r16=0,
                                  saturate=bool(case["saturate"]))
    if case["mode"] != "stochastic":
        assert (c2, int(o2), int(u2)) == (case["code"], case["overflowed"], case["underflowed"])


@pytest.mark.parametrize("case", KA["decode"], ids=lambda c: f"{c['fmt']}-{c['code']:#x}")
def test_known_decode(case):
    v = O.decode(case["code"], case["fmt"])
    want = _f(case["value"])
    if math.isnan(want):
        assert math.isnan(v)
    else:
        assert v == want and math.copysign(1, v) == math.copysign(1, want)


@pytest.mark.parametrize("case", KA["quantize"], ids=lambda c: c["cite"])
def test_known_quantize_counters(case):
    codes, cnt = O.quantize(np.array([_f(v) for v in case["x"]], dtype=np.float32), case["fmt"],
                            saturate=bool(case["saturate"]))
    assert list(codes) == case["codes"]
    assert (cnt[0], cnt[1]) == (case["overflow"], case["underflow"])


QG = np.load(os.path.join(GOLD, "quantize_golden.npz"))
QMETA = _load("quantize_golden.json")


@pytest.mark.parametrize("m", QMETA, ids=lambda m: m["key"])
def test_quantize_stream_golden(m):
    """Whole-tensor quantize (3 full 4096-blocks + a partial block) equals the
    reference's fp8emu::quantize bit for bit, counters included."""
    codes, cnt = O.quantize(QG["x"], m["fmt"], m["mode"], int(m["seed"]), m["saturate"])
    np.testing.assert_array_equal(codes, QG[m["key"]])
    assert (int(cnt[0]), int(cnt[1])) == (m["overflow"], m["underflow"])


def test_sr_constant_tensor_golden():
    codes, _ = O.quantize(QG["const_1p1"], "fp8", "stochastic", 31)
    np.testing.assert_array_equal(codes, QG["const_1p1_sr31"])
    ups = int((codes == 0x3D).sum())
    assert abs(ups - 1638) < 157  # test_quantize.cpp:76-92


def test_zero_seed_rejected():
    with pytest.raises(ValueError):
        O.quantize(np.ones(3, np.float32), "fp8", "stochastic", 0)
    with pytest.raises(ValueError):  # tensor.cpp:48 rejects seed 0 in every mode
        O.quantize(np.ones(3, np.float32), "fp8", "nearest-even", 0)


def test_block_offset_shards_reproduce_whole_tensor():
    """SR block streams are indexed by the global 4096-block (tensor.cpp:58-62)."""
    x = QG["x"][: 3 * 4096]
    whole, wc = O.quantize(x, "fp8", "stochastic", 1337)
    parts = [O.quantize(x[b * 4096:(b + 1) * 4096], "fp8", "stochastic", 1337, block_offset=b)
             for b in range(3)]
    np.testing.assert_array_equal(np.concatenate([p[0] for p in parts]), whole)
    assert sum(int(p[1][1]) for p in parts) == int(wc[1])


def test_integer_rule_equals_reference_rule_random():
    """SURVEY A2': the integer rule the kernels implement == encode() in double."""
    rng = np.random.default_rng(1)
    bits = rng.integers(0, 2 ** 32, 60000, dtype=np.uint64).astype(np.uint32)
    # bias towards interesting exponents as well
    mant = rng.integers(0, 2 ** 23, 60000, dtype=np.uint64).astype(np.uint32)
    expo = rng.integers(95, 145, 60000).astype(np.uint32)
    sign = rng.integers(0, 2, 60000).astype(np.uint32)
    bits = np.concatenate([bits, (sign << 31) | (expo << 23) | mant])
    r16s = rng.integers(0, 65536, bits.size)
    x = bits.view(np.float32)
    for fmt in ("fp8", "fp16"):
        for mode in ("nearest-even", "truncate", "stochastic"):
            bad = 0
            for i in range(0, bits.size, 3):
                r16 = int(r16s[i])
                c1, o1, u1, ie = O.encode_bits(int(bits[i]), fmt, mode, r16)
                if mode == "stochastic":
                    # encode() with an LFSR whose first sample is r16 (SURVEY 8c iv)
                    if r16 == 0:
                        continue
                    st = O.bitrev16(r16)
                    c2, o2, u2 = O.encode(float(x[i]), fmt, mode, lfsr_state=st)
                else:
                    c2, o2, u2 = O.encode(float(x[i]), fmt, mode)
                bad += (c1, o1, u1) != (c2, o2, u2)
            assert bad == 0, (fmt, mode)


def test_lfsr_jump_tables_reproduce_split_streams():
    """The GPU's stream addressing: sample j of split(seed, b) is
    tab[(pos[split(seed, b)] + j) mod 65535]."""
    tab, pos = O.lfsr_tables()
    assert len(set(tab.tolist())) == 65535  # D = 16 clocks is a single 65535-cycle
    for seed, b in [(0, 0), (1, 0), (81, 0), (1337, 5), (2 ** 64 - 1, 77)]:
        s0 = O.lib().or_lfsr_split(seed, b)
        st = O.C.c_uint16(s0)
        p = int(pos[s0])
        for j in range(5000):
            want = O.lib().or_lfsr_next_bits(O.C.byref(st), 16)
            assert tab[(p + j) % 65535] == want


def test_lfsr_split_landmarks():
    # SURVEY Appendix A probe1: split(0,0)=0x65F4, split(0,1)=0x454F, split(1,0)=0xEC67,
    # split(81,0)=0xEACE
    assert O.lib().or_lfsr_split(0, 0) == 0x65F4
    assert O.lib().or_lfsr_split(0, 1) == 0x454F
    assert O.lib().or_lfsr_split(1, 0) == 0xEC67
    assert O.lib().or_lfsr_split(81, 0) == 0xEACE


def test_lfsr_period():
    """test_lfsr.cpp:12-21: the register walks the full 2^16-1 cycle."""
    st = O.C.c_uint16(1)
    steps = 0
    while True:
        O.lib().or_lfsr_next_bits(O.C.byref(st), 1)
        steps += 1
        if st.value == 1 or steps > 70000:
            break
    assert steps == 65535


def test_counter_and_supplied_bits_agree():
    x = QG["x"][:5000]
    seed = 99
    c1, k1 = O.quantize(x, "fp8", "stochastic", seed, bits="counter", block_offset=2)
    gi = [2 * 4096 + i for i in range(x.size)]
    r = np.array([((O.lib().or_mix64(seed + (g >> 2) + 1) >> (16 * (g & 3))) & 0xFFFF) << 16
                  for g in gi], dtype=np.uint32)
    c2, k2 = O.quantize(x, "fp8", "stochastic", seed, bits="supplied", rbits=r)
    np.testing.assert_array_equal(c1, c2)
    np.testing.assert_array_equal(k1, k2)


GG = np.load(os.path.join(GOLD, "gemm_golden.npz"))
GMETA = _load("gemm_golden.json")


@pytest.mark.parametrize("m", GMETA, ids=lambda m: f"{m['m']}x{m['k']}x{m['n']}")
@pytest.mark.parametrize("fmt", ["fp8", "fp16"])
def test_gemm_golden_bitwise(m, fmt):
    i = m["i"]
    c = O.gemm(GG[f"a_{i}_{fmt}"], GG[f"b_{i}_{fmt}"], m["m"], m["k"], m["n"], fmt)
    np.testing.assert_array_equal(c.view(np.uint32), GG[f"c_{i}_{fmt}"].view(np.uint32))


def test_gemm_frozen_hand_computation():
    c = GG["c_0_fp8"].reshape(-1)
    assert list(c) == [2.25, -1.0, -1.625, 5.0]  # test_kernels.cpp:60-73


@pytest.mark.parametrize("tr", _load("scaler_golden.json"), ids=lambda t: t["cite"])
def test_scaler_traces_golden(tr):
    opts = dict(tr["opts"])
    if "min_threshold_schedule" in opts:
        opts["min_threshold_schedule"] = [tuple(v) for v in opts["min_threshold_schedule"]]
    s = O.OracleLossScaler(**opts)
    for finite, it, act, sc in tr["steps"]:
        a, v = s.step(bool(finite), it)
        assert (a, v) == (act, sc)


UG = np.load(os.path.join(GOLD, "update_golden.npz"))


@pytest.mark.parametrize("m", _load("update_golden.json"), ids=lambda m: m["key"])
def test_update_golden(m):
    g = O.dequantize(UG["grad_e5m2"], "fp8")
    master, mom, w32, _ = O.sgd_update(UG["master0"], UG["mom0"], g, m["scale"], m["lr"], m["mu"],
                                       np.float32(m["two_lambda"]), m["master_mode"], "lfsr",
                                       m["seed"])
    k = m["key"]
    np.testing.assert_array_equal(w32.view(np.uint32), UG[f"w32_{k}"].view(np.uint32))
    np.testing.assert_array_equal(mom.view(np.uint32), UG[f"mom1_{k}"].view(np.uint32))
    np.testing.assert_array_equal(master, UG[f"master1_{k}"])


def test_bias_grad_row_order():
    rng = np.random.default_rng(4)
    e = rng.standard_normal(37 * 11).astype(np.float32)
    db = O.bias_grad(e, 37, 11)
    for j in range(11):
        acc = np.float32(0)
        for r in range(37):
            acc = np.float32(acc + e[r * 11 + j])
        assert db[j] == acc


@pytest.mark.slow
def test_config1_known_answers():
    """SURVEY 8d config-1 recipe through the oracle == hashes from the reference."""
    gold = _load("config1_golden.json")
    H = lambda a: f"{O.fnv1a64(a):016x}"
    r = O.Rand(0)
    X, W, dY = r.normal(524288), r.normal(1048576, 1 / 32), r.normal(524288, 0.01)
    assert (H(X), H(W), H(dY)) == (gold["X"], gold["W"], gold["dY"])
    master0, _ = O.quantize(W, "fp16")
    assert H(master0) == gold["master0"]
    qX, kx = O.quantize(X)
    qW, kw = O.quantize(O.dequantize(master0, "fp16"))
    assert H(qX.astype(np.uint8)) == gold["qX"] and H(qW.astype(np.uint8)) == gold["qW"]
    assert list(kx[:2]) == gold["counters"]["qX"] and list(kw[:2]) == gold["counters"]["qW"]
    E = (dY * np.float32(8192)).astype(np.float32)
    qE, _ = O.quantize(E)
    assert H(qE.astype(np.uint8)) == gold["qE"]


# ------------------------------------------------ direct reference comparisons
ref_only = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@ref_only
@pytest.mark.parametrize("fmt", ["fp8", "fp16"])
@pytest.mark.parametrize("mode", ["nearest-even", "truncate", "stochastic"])
def test_oracle_vs_reference_random(fmt, mode):
    rng = np.random.default_rng(3)
    x = (np.exp2(rng.uniform(-30, 18, 50000)) * rng.choice([-1, 1], 50000)).astype(np.float32)
    for sat in (0, 1):
        c1, k1 = O.quantize(x, fmt, mode, 4242, sat)
        c2, k2 = O.ref_quantize(x, fmt, mode, 4242, sat)
        np.testing.assert_array_equal(c1, c2)
        np.testing.assert_array_equal(k1[:2], k2)


@ref_only
def test_reference_mt_harness_bit_identical():
    x = QG["x"]
    for mode in ("nearest-even", "stochastic"):
        c1, k1 = O.ref_quantize(x, "fp8", mode, 1337)
        c2, k2 = O.ref_quantize_mt(x, "fp8", mode, 1337, nthreads=4)
        np.testing.assert_array_equal(c1.astype(np.uint8), c2)
        np.testing.assert_array_equal(k1, k2)


CG = np.load(os.path.join(GOLD, "conv_golden.npz"))


@pytest.mark.parametrize("m", _load("conv_golden.json"), ids=lambda m: str(m["i"]))
def test_conv_family_golden_bitwise(m):
    """conv2d_fp8 / backward_data / backward_weights (kernels.cpp:106-253)."""
    i = m["i"]
    args = (m["n"], m["c"], m["h"], m["w"], m["f"], m["k"], m["k"], m["stride"], m["pad"])
    for kind, a, b, want in [("fprop", "x", "w", "y"), ("dgrad", "e", "w", "dx"),
                             ("wgrad", "x", "e", "dw")]:
        got = O.conv2d(CG[f"{a}_{i}"], CG[f"{b}_{i}"], *args, kind=kind)
        np.testing.assert_array_equal(got.view(np.uint32), CG[f"{want}_{i}"].view(np.uint32))
