"""Stream-K vs data-parallel sweep (diagnostic): python scripts/sk_sweep.py
Times each shape under env variants (label=K:V,K:V), E5M2-out and FP32-out,
interleaved rounds, median."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12334_b200 as F  # noqa: E402

SHAPES = os.environ.get("SK_SHAPES", "2048x2048x2048,4096x4096x4096,16384x1024x16384,8192x8192x8192,"
                        "3072x3072x3072,6144x6144x6144").split(",")
VARIANTS = [v.split("=", 1) for v in (sys.argv[1:] or ["dp=FP8B_GEMM_SK:0", "sk=FP8B_GEMM_SK:1",
                                                        "auto="])]
ROUNDS = int(os.environ.get("SK_ROUNDS", "3"))
F.init()


def run(spec, fn):
    env = dict(kv.split(":") for kv in spec.split(",") if kv)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def timed(spec, fn, reps):
    for _ in range(3):
        run(spec, fn)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        run(spec, fn)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for sh in SHAPES:
    m, n, k = map(int, sh.split("x"))
    x = torch.empty(m * k + k * n, dtype=torch.float32, device="cuda")
    F.fill_synthetic(x, "normal", 3, 1.0)
    qa = F.quantize(x[: m * k]).codes
    qb = F.quantize(x[m * k:]).codes
    del x
    c = torch.empty((m, n), dtype=torch.float32, device="cuda")
    cq = torch.empty(m * n, dtype=torch.uint8, device="cuda")
    reps = max(5, min(200, int(2e12 / (2 * m * n * k))))
    for label, kw in [("e5m2", dict(want_c=False, out_fmt="fp8", out_codes=cq)), ("f32", dict(c=c))]:
        res = {lab: [] for lab, _ in VARIANTS}
        for _ in range(ROUNDS):
            for lab, spec in VARIANTS:
                res[lab].append(timed(spec, lambda: F.gemm_codes(qa, qb, m, n, k, "fp8", **kw), reps))
        line = " ".join(f"{lab} {statistics.median(v):.4f}ms {2*m*n*k/statistics.median(v)/1e9:7.1f}TF"
                        for lab, v in res.items())
        print(f"{sh:>18s} {label:5s} {line}", flush=True)
    del qa, qb, c, cq
    torch.cuda.empty_cache()
