"""Interleaved A/B timing of GEMM variants (env knobs set per call) against
cuBLASLt on the same box, same thermal state (diagnostic)."""
import os, statistics, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12334_b200 as F

variants = [v.split("=", 1) for v in sys.argv[1:]]  # label=ENVSPEC (k:v,k:v)
m = n = k = int(os.environ.get("AB_N", "8192"))
m = int(os.environ.get("AB_M", m))
n = int(os.environ.get("AB_NN", n))
k = int(os.environ.get("AB_K", k))
F.init()
x = torch.empty(m * k + k * n, dtype=torch.float32, device="cuda")
F.fill_synthetic(x, "normal", 3, 1.0)
qa = F.quantize(x[: m * k]).codes
qb = F.quantize(x[m * k:]).codes
qa0, qb0 = torch.zeros_like(qa), torch.zeros_like(qb)
c = torch.empty((m, n), dtype=torch.float32, device="cuda")
cq = torch.empty(m * n, dtype=torch.uint8, device="cuda")
a8 = x[: m * k].reshape(m, k).to(torch.float8_e4m3fn)
b8 = x[m * k:].reshape(n, k).to(torch.float8_e5m2)
one = torch.ones((), device="cuda")
del x


def run_ours(spec):
    env = dict(kv.split(":") for kv in spec.split(",") if kv)
    zeros = env.pop("zeros", None)
    outq = env.pop("q", None)
    old = {kk: os.environ.get(kk) for kk in env}
    os.environ.update(env)
    try:
        if outq:
            F.gemm_codes(qa, qb, m, n, k, "fp8", want_c=False, out_fmt="fp8", out_codes=cq)
        elif zeros:
            F.gemm_codes(qa0, qb0, m, n, k, "fp8", c=c)
        else:
            F.gemm_codes(qa, qb, m, n, k, "fp8", c=c)
    finally:
        for kk, vv in old.items():
            if vv is None:
                os.environ.pop(kk, None)
            else:
                os.environ[kk] = vv


def timed(fn, reps=20):
    for _ in range(2):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


res = {lab: [] for lab, _ in variants}
res["cublas"] = []
import time  # noqa: E402
ROUNDS = int(os.environ.get("AB_ROUNDS", "5"))
REPS = int(os.environ.get("AB_REPS", "20"))
COOL = float(os.environ.get("AB_SLEEP", "0"))  # seconds idle before each timing (power state)
for rnd in range(ROUNDS):
    for lab, spec in variants:
        time.sleep(COOL)
        res[lab].append(timed(lambda: run_ours(spec), REPS))
    time.sleep(COOL)
    res["cublas"].append(timed(lambda: torch._scaled_mm(a8, b8.t(), scale_a=one, scale_b=one,
                                                        out_dtype=torch.bfloat16), REPS))
base = statistics.median(res["cublas"])
for lab, v in res.items():
    md = statistics.median(v)
    print(f"{lab:14s} median {md:.4f} ms  {2*m*n*k/md/1e9:7.1f} TF/s  vs cublas {base/md:.3f}  all {[round(t,4) for t in v]}")
