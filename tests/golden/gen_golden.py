"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (it needs oracle/_ref/libfp8emu_ref.so, compiled from
/root/reference/proj/src by oracle/Makefile):

    python tests/golden/gen_golden.py

Every expected value below is produced by the unmodified reference library
(fp8emu::quantize / gemm_fp8 / LossScaler / encode), except the known-answer
table, which restates the constants frozen in the reference's own unit tests
(cited per entry) and is re-verified against the reference here before being
written. The GPU tests compare libfp8b200 against these files; the CPU tests
pin the oracle restatement (oracle/fp8_oracle.c) against them.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
import oracle as O  # noqa: E402

INF = float("inf")
NAN = float("nan")

# (x, fmt, mode, saturate, expected code, overflowed, underflowed, cite)
KNOWN = [
    (1.1, "fp8", "nearest-even", 0, 0x3C, 0, 0, "test_float_format.cpp:89"),
    (1.125, "fp8", "nearest-even", 0, 0x3C, 0, 0, "test_float_format.cpp:90"),
    (1.375, "fp8", "nearest-even", 0, 0x3E, 0, 0, "test_float_format.cpp:91"),
    (5e-5, "fp8", "nearest-even", 0, 0x03, 0, 0, "test_float_format.cpp:92"),
    (1e-4, "fp8", "nearest-even", 0, 0x07, 0, 0, "test_float_format.cpp:93"),
    (0.1, "fp8", "nearest-even", 0, 0x2E, 0, 0, "test_float_format.cpp:94"),
    (-0.3, "fp8", "nearest-even", 0, 0xB5, 0, 0, "test_float_format.cpp:95"),
    (2.2888184e-05, "fp8", "nearest-even", 0, 0x02, 0, 0, "test_float_format.cpp:96"),
    (0.0, "fp8", "nearest-even", 0, 0x00, 0, 0, "test_float_format.cpp:97"),
    (-0.0, "fp8", "nearest-even", 0, 0x80, 0, 0, "test_float_format.cpp:98"),
    (57344.0, "fp8", "nearest-even", 0, 0x7B, 0, 0, "test_float_format.cpp:104-106"),
    (57345.0, "fp8", "nearest-even", 0, 0x7C, 1, 0, "test_float_format.cpp:107-109"),
    (1e6, "fp8", "nearest-even", 0, 0x7C, 1, 0, "test_float_format.cpp:110-112"),
    (-1e6, "fp8", "nearest-even", 0, 0xFC, 1, 0, "test_float_format.cpp:113-115"),
    (1e6, "fp8", "nearest-even", 1, 0x7B, 1, 0, "test_float_format.cpp:117-119"),
    (7.0e-6, "fp8", "nearest-even", 0, 0x00, 0, 1, "test_float_format.cpp:123-125"),
    (7.62939453125e-06, "fp8", "nearest-even", 0, 0x00, 0, 1, "test_float_format.cpp:126-128"),
    (8.0e-6, "fp8", "nearest-even", 0, 0x01, 0, 0, "test_float_format.cpp:129-131"),
    (-7.0e-6, "fp8", "nearest-even", 0, 0x80, 0, 1, "test_float_format.cpp:132-134"),
    (INF, "fp8", "nearest-even", 0, 0x7C, 1, 0, "test_float_format.cpp:139"),
    (-INF, "fp8", "nearest-even", 0, 0xFC, 1, 0, "test_float_format.cpp:140-141"),
    (NAN, "fp8", "nearest-even", 0, 0x7E, 0, 0, "test_float_format.cpp:142-143"),
    (NAN, "fp16", "stochastic", 0, 0x7E00, 0, 0, "test_float_format.cpp:144-145"),
    (1.99, "fp8", "truncate", 0, 0x3F, 0, 0, "test_float_format.cpp:213 (1.75)"),
    (-1.99, "fp8", "truncate", 0, 0xBF, 0, 0, "test_float_format.cpp:214 (-1.75)"),
    (1.2499, "fp8", "truncate", 0, 0x3C, 0, 0, "test_float_format.cpp:215 (1.0)"),
    (5.5e-5, "fp8", "truncate", 0, 0x03, 0, 0, "test_float_format.cpp:216 (4.5776e-5)"),
    (0.1, "fp16", "nearest-even", 0, 0x2E66, 0, 0, "test_quantize.cpp:58 (0.0999755859375)"),
    (65504.0, "fp16", "nearest-even", 0, 0x7BFF, 0, 0, "test_quantize.cpp:59"),
    (70000.0, "fp16", "nearest-even", 0, 0x7C00, 1, 0, "test_quantize.cpp:56"),
]

# decode table (test_float_format.cpp:43-70)
DECODE = [
    (0x00, "fp8", 0.0), (0x01, "fp8", 1.52587890625e-05), (0x03, "fp8", 4.57763671875e-05),
    (0x04, "fp8", 6.103515625e-05), (0x3C, "fp8", 1.0), (0x3D, "fp8", 1.25), (0x3F, "fp8", 1.75),
    (0x42, "fp8", 3.0), (0xC2, "fp8", -3.0), (0x7B, "fp8", 57344.0), (0x7C, "fp8", INF),
    (0xFC, "fp8", -INF), (0x7E, "fp8", NAN), (0xFF, "fp8", NAN), (0x80, "fp8", -0.0),
    (0x3C00, "fp16", 1.0), (0x7BFF, "fp16", 65504.0), (0x0001, "fp16", 5.960464477539063e-08),
    (0x0400, "fp16", 6.103515625e-05), (0x2E66, "fp16", 0.0999755859375),
    (0x3555, "fp16", 0.333251953125), (0xC000, "fp16", -2.0),
]

# quantize counters (test_quantize.cpp:13-40)
QUANT_CASES = [
    ([1.0, 1e6, -2e6, 1e-6, -1e-6, 0.0], "fp8", 0, 2, 2, [0x3C, 0x7C, 0xFC, 0x00, 0x80, 0x00],
     "test_quantize.cpp:13-28"),
    ([1e6, -1e6], "fp8", 1, 2, 0, [0x7B, 0xFB], "test_quantize.cpp:30-40"),
]


def _json_float(v):
    if v != v:
        return "nan"
    if v in (INF, -INF):
        return "inf" if v > 0 else "-inf"
    return v


def config2_like(n, seed, tie_frac=0.01, lo=-24.0, hi=17.0):
    """Seeded sample of the SURVEY 8d config-2 distribution plus specials."""
    rng = np.random.default_rng(seed)
    u = rng.uniform(lo, hi, n)
    x = np.exp2(u) * rng.choice([-1.0, 1.0], n)
    ties = rng.random(n) < tie_frac
    c = rng.integers(0, 0x7B, n)
    mids = np.array([(O.decode(int(k)) + O.decode(int(k) + 1)) / 2 for k in range(0x7B)])
    x[ties] = mids[c[ties]] * rng.choice([-1.0, 1.0], int(ties.sum()))
    x = x.astype(np.float32)
    specials = np.array([0.0, -0.0, INF, -INF, NAN, 57344.0, 57345.0, 61439.0, 61440.0, 65504.0,
                         65519.0, 65520.0, 1e-45, -1e-45, 1.17549435e-38, 2.0 ** -17,
                         2.0 ** -16, 3 * 2.0 ** -17, 2.0 ** -25, 2.0 ** -24, 5.960464477539063e-08,
                         1.0, 1.125, 1.375, -1.625], dtype=np.float32)
    x[: specials.size] = specials
    # sprinkle specials across blocks too
    idx = rng.integers(0, n, 64)
    x[idx] = specials[rng.integers(0, specials.size, 64)]
    return x


def main():
    assert O.ref_available(), "needs oracle/_ref (run make -C oracle ref)"
    out = {}
    # ---- known answers, verified against the reference
    known = []
    for x, fmt, mode, sat, code, ovf, unf, cite in KNOWN:
        rc, ro, ru = O.ref_encode(x, fmt, mode, seed=1, saturate=sat)
        assert (rc, int(ro), int(ru)) == (code, ovf, unf), (x, fmt, mode, rc, ro, ru, cite)
        known.append({"x": _json_float(x), "fmt": fmt, "mode": mode, "saturate": sat,
                      "code": code, "overflowed": ovf, "underflowed": unf, "cite": cite})
    dec = []
    for code, fmt, v in DECODE:
        got = O.ref().ref_decode(code, O.FMT[fmt])
        assert (got == v) or (got != got and v != v), (code, fmt, got, v)
        if v == 0.0:
            assert np.signbit(got) == np.signbit(v)
        dec.append({"code": code, "fmt": fmt, "value": _json_float(v),
                    "cite": "test_float_format.cpp:43-70"})
    qc = []
    for xs, fmt, sat, ovf, unf, codes, cite in QUANT_CASES:
        c, k = O.ref_quantize(np.array(xs, dtype=np.float32), fmt, "nearest-even", 1, sat)
        assert list(c) == codes and int(k[0]) == ovf and int(k[1]) == unf, (xs, c, k)
        qc.append({"x": [_json_float(v) for v in xs], "fmt": fmt, "saturate": sat,
                   "codes": codes, "overflow": ovf, "underflow": unf, "cite": cite})
    with open(os.path.join(HERE, "known_answers.json"), "w") as f:
        json.dump({"encode": known, "decode": dec, "quantize": qc}, f, indent=1)

    # ---- quantize streams from the reference (3 full blocks + a partial one)
    n = 3 * 4096 + 1234
    x = config2_like(n, seed=20190529)
    arrays = {"x": x}
    meta = []
    for fmt in ("fp8", "fp16"):
        for mode in ("nearest-even", "truncate", "stochastic"):
            for sat in (0, 1):
                for seed in ((977,) if mode != "stochastic" else (977, 1337, 0xFFFFFFFFFFFFFFFF)):
                    codes, cnt = O.ref_quantize(x, fmt, mode, seed, sat)
                    key = f"{fmt}_{mode}_{sat}_{seed}"
                    arrays[key] = codes
                    meta.append({"key": key, "fmt": fmt, "mode": mode, "saturate": sat,
                                 "seed": str(seed), "overflow": int(cnt[0]),
                                 "underflow": int(cnt[1])})
    # a constant-tensor SR case (test_quantize.cpp:76-92 shape)
    xc = np.full(4096, 1.1, dtype=np.float32)
    arrays["const_1p1"] = xc
    arrays["const_1p1_sr31"], _ = O.ref_quantize(xc, "fp8", "stochastic", 31)
    np.savez_compressed(os.path.join(HERE, "quantize_golden.npz"), **arrays)
    with open(os.path.join(HERE, "quantize_golden.json"), "w") as f:
        json.dump(meta, f, indent=1)

    # ---- gemm_fp8 from the reference
    rng = np.random.default_rng(7)
    g = {}
    shapes = [(2, 2, 2)] + [tuple(int(v) for v in rng.integers(1, 17, 3)) for _ in range(12)] + \
             [(64, 96, 80), (128, 256, 64), (33, 517, 45)]
    gm = []
    for i, (m, k, n_) in enumerate(shapes):
        if i == 0:
            a = np.array([1.0, 2.0, 0.5, -1.75], dtype=np.float32)   # test_kernels.cpp:60-73
            b = np.array([0.25, 3.0, 1.0, -2.0], dtype=np.float32)
        else:
            a = rng.uniform(-2, 2, m * k).astype(np.float32)
            b = rng.uniform(-2, 2, k * n_).astype(np.float32)
        for fmt in ("fp8", "fp16"):
            qa, _ = O.ref_quantize(a, fmt)
            qb, _ = O.ref_quantize(b, fmt)
            c = O.ref_gemm(qa, qb, m, k, n_, fmt)
            g[f"a_{i}_{fmt}"], g[f"b_{i}_{fmt}"], g[f"c_{i}_{fmt}"] = qa, qb, c
        gm.append({"i": i, "m": m, "k": k, "n": n_})
    np.savez_compressed(os.path.join(HERE, "gemm_golden.npz"), **g)
    with open(os.path.join(HERE, "gemm_golden.json"), "w") as f:
        json.dump(gm, f, indent=1)

    # ---- conv family from the reference (kernels.cpp:106-253), NCHW
    rngc = np.random.default_rng(17)
    cg = {}
    cmeta = []
    shapes = [(2, 3, 7, 6, 4, 3, 1, 1), (1, 2, 9, 9, 3, 3, 2, 1), (2, 4, 5, 5, 2, 1, 1, 0),
              (1, 3, 8, 7, 2, 3, 2, 0), (2, 16, 6, 6, 8, 3, 1, 1), (1, 8, 5, 5, 16, 1, 1, 0)]
    for i, (n_, c, h, w, f, k, st, pd) in enumerate(shapes):
        oh, ow = O.conv_out(h, k, st, pd), O.conv_out(w, k, st, pd)
        x, _ = O.ref_quantize(rngc.uniform(-2, 2, n_ * c * h * w).astype(np.float32))
        wt, _ = O.ref_quantize(rngc.uniform(-2, 2, f * c * k * k).astype(np.float32))
        e, _ = O.ref_quantize(rngc.uniform(-2, 2, n_ * f * oh * ow).astype(np.float32))
        cg[f"x_{i}"], cg[f"w_{i}"], cg[f"e_{i}"] = x, wt, e
        cg[f"y_{i}"] = O.ref_conv2d(x, wt, n_, c, h, w, f, k, k, st, pd, kind="fprop")
        cg[f"dx_{i}"] = O.ref_conv2d(e, wt, n_, c, h, w, f, k, k, st, pd, kind="dgrad")
        cg[f"dw_{i}"] = O.ref_conv2d(x, e, n_, c, h, w, f, k, k, st, pd, kind="wgrad")
        cmeta.append({"i": i, "n": n_, "c": c, "h": h, "w": w, "f": f, "k": k, "stride": st,
                      "pad": pd})
    np.savez_compressed(os.path.join(HERE, "conv_golden.npz"), **cg)
    with open(os.path.join(HERE, "conv_golden.json"), "w") as f_:
        json.dump(cmeta, f_, indent=1)

    # ---- loss scaler traces from the reference
    traces = []
    def trace(opts, steps, cite):
        s = O.RefLossScaler(**opts)
        rows = []
        for finite, it in steps:
            act, sc = s.step(finite, it)
            rows.append([int(finite), int(it), act, sc])
        traces.append({"opts": {k: (list(map(list, v)) if k == "min_threshold_schedule" else v)
                                for k, v in opts.items()}, "steps": rows, "cite": cite})
    dyn = dict(kind="dynamic-backoff", scale=65536.0, growth_interval=100,
               min_threshold_schedule=[(40, 8192.0), (150, 32768.0)])
    trace(dyn, [(False, 10), (False, 10)] + [(False, 50)] * 10 + [(True, 100)] * 100 +
          [(True, 151)], "acceptance.cpp:255-283")
    trace(dict(kind="dynamic-backoff", scale=65536.0, min_threshold_schedule=[(40, 8192.0),
                                                                             (150, 32768.0)]),
          [(False, 148), (False, 149), (False, 150)], "test_loss_scaling.cpp:118-126")
    trace(dict(kind="dynamic-backoff", scale=1024.0, growth_interval=2000),
          [(True, i) for i in range(2000)] + [(False, 2000)] + [(True, 2001 + i) for i in range(2000)],
          "test_loss_scaling.cpp:84-104")
    trace(dict(kind="dynamic-backoff", scale=4096.0, min_threshold_schedule=[(40, 8192.0),
                                                                            (150, 32768.0)]),
          [(True, 10), (True, 40)], "test_loss_scaling.cpp:106-116")
    trace(dict(kind="constant", scale=1024.0), [(i % 7 != 0, i) for i in range(50)],
          "test_loss_scaling.cpp:23-34")
    trace(dict(kind="dynamic-backoff", scale=1024.0, backoff_factor=0.5, growth_factor=2.0,
               growth_interval=1000, min_threshold_schedule=[(0, 256.0)]),
          [(False, 0), (False, 1), (False, 2)], "tests/python/test_smoke.py:65-80")
    with open(os.path.join(HERE, "scaler_golden.json"), "w") as f:
        json.dump(traces, f, indent=1)

    # ---- update_tensor with RNE (reference) and SR (reference quantize) masters
    nu = 2 * 4096 + 100
    r = O.Rand(11)
    w = r.normal(nu, 1.0 / 32)
    master0, _ = O.ref_quantize(w, "fp16")
    mom0 = r.normal(nu, 1e-3)
    gq, _ = O.ref_quantize(r.normal(nu, 1e-4) * np.float32(8192.0), "fp8")
    gdec = O.dequantize(gq, "fp8")
    up = {"master0": master0, "mom0": mom0, "grad_e5m2": gq}
    umeta = []
    for tl in (0.0, 2e-4):
        for mm, seed in (("nearest-even", 1), ("stochastic", 5)):
            m1, mo1, w32 = O.ref_update(master0, mom0, gdec, 8192.0, 0.1, 0.9,
                                        np.float32(tl), mm, seed)
            key = f"{mm}_{tl}"
            up[f"master1_{key}"], up[f"mom1_{key}"], up[f"w32_{key}"] = m1, mo1, w32
            umeta.append({"key": key, "two_lambda": tl, "master_mode": mm, "seed": seed,
                          "scale": 8192.0, "lr": 0.1, "mu": 0.9})
    np.savez_compressed(os.path.join(HERE, "update_golden.npz"), **up)
    with open(os.path.join(HERE, "update_golden.json"), "w") as f:
        json.dump(umeta, f, indent=1)

    # ---- config-1 layer step known-answer hashes from the reference
    X, W, dY = O.ref_rand_normal(0, [(524288, 1.0), (1048576, 1.0 / 32), (524288, 0.01)])
    E = (dY * np.float32(8192.0)).astype(np.float32)
    H = O.fnv1a64
    c1 = {"X": H(X), "W": H(W), "dY": H(dY)}
    master0, _ = O.ref_quantize(W, "fp16")
    wv = O.dequantize(master0, "fp16")
    qX, kx = O.ref_quantize(X, "fp8")
    qW, kw = O.ref_quantize(wv, "fp8")
    Y = O.ref_gemm(qX, qW, 512, 1024, 1024, nthreads=os.cpu_count() or 8)
    qY, ky = O.ref_quantize(Y, "fp8")
    qE, ke = O.ref_quantize(E, "fp8")
    qXt = qX.reshape(512, 1024).T.copy()
    dW = O.ref_gemm(qXt, qE, 1024, 512, 1024, nthreads=os.cpu_count() or 8)
    qdW, kdw = O.ref_quantize(dW, "fp8")
    qWt = qW.reshape(1024, 1024).T.copy()
    dX = O.ref_gemm(qE, qWt, 512, 1024, 1024, nthreads=os.cpu_count() or 8)
    qdX, kdx = O.ref_quantize(dX, "fp8")
    g = O.dequantize(qdW, "fp8")
    finite = int(kdw[0] + ke[0] + kdx[0] == 0 and np.isfinite(g).all())
    mom = np.zeros(W.size, dtype=np.float32)
    m_rne, mom1, w32 = O.ref_update(master0, mom, g, 8192.0, 0.1, 0.9, 0.0, "nearest-even")
    m_sr, _, _ = O.ref_update(master0, mom, g, 8192.0, 0.1, 0.9, 0.0, "stochastic", 1)
    qW1, kw1 = O.ref_quantize(O.dequantize(m_sr, "fp16"), "fp8")
    u8 = lambda c: c.astype(np.uint8)
    c1.update({
        "master0": H(master0), "qX": H(u8(qX)), "qW": H(u8(qW)), "qY": H(u8(qY)),
        "qE": H(u8(qE)), "qdW": H(u8(qdW)), "qdX": H(u8(qdX)), "Y": H(Y), "dW": H(dW),
        "dX": H(dX), "momentum1": H(mom1), "w32": H(w32), "master1_rne": H(m_rne),
        "master1_sr1": H(m_sr), "qW1": H(u8(qW1)),
        "counters": {"qX": [int(v) for v in kx], "qW": [int(v) for v in kw],
                     "qY": [int(v) for v in ky], "qE": [int(v) for v in ke],
                     "qdW": [int(v) for v in kdw], "qdX": [int(v) for v in kdx],
                     "qW1": [int(v) for v in kw1]},
        "grads_finite": finite,
        "master1_rne_changed": int((m_rne != master0).sum()),
        "master1_sr_changed": int((m_sr != master0).sum()),
        "sr_vs_rne_differ": int((m_sr != m_rne).sum()),
        "recipe": "SURVEY 8d config 1: one Rand{0} stream X, W*1/32, dY*0.01; E = dY*8192; "
                  "master0 = RNE_FP16(W); qW = Q(decode(master0)); gemm_fp8 sequential; "
                  "update lr 0.1 mu 0.9 scale 8192; SR master seed 1",
    })
    c1 = {k: (f"{v:016x}" if isinstance(v, int) and k not in (
        "grads_finite", "master1_rne_changed", "master1_sr_changed", "sr_vs_rne_differ")
        else v) for k, v in c1.items()}
    with open(os.path.join(HERE, "config1_golden.json"), "w") as f:
        json.dump(c1, f, indent=1)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
