"""tcgen05 E5M2 GEMM timings (iteration helper): python scripts/gemm_bench.py [--shapes MxNxK ...]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12334_b200 as F  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", nargs="*", default=["8192x8192x8192", "16384x1024x16384", "4096x4096x4096"])
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--outs", nargs="*", default=["f32", "e5m2"])
a = ap.parse_args()
F.init()
for sh in a.shapes:
    m, n, k = map(int, sh.split("x"))
    x = torch.empty(m * k + k * n, dtype=torch.float32, device="cuda")
    F.fill_synthetic(x, "normal", 3, 1.0)
    qa = F.quantize(x[: m * k]).codes
    qb = F.quantize(x[m * k:]).codes
    del x
    c = torch.empty((m, n), dtype=torch.float32, device="cuda")
    cq = torch.empty(m * n, dtype=torch.uint8, device="cuda")
    for label in a.outs:
        kw = dict(c=c) if label == "f32" else dict(want_c=False, out_fmt="fp8", out_codes=cq)
        for _ in range(3):
            F.gemm_codes(qa, qb, m, n, k, "fp8", **kw)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.reps):
            F.gemm_codes(qa, qb, m, n, k, "fp8", **kw)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        print(f"{m}x{n}x{k} {label} {ms:.4f} ms {2 * m * n * k / ms / 1e9:.1f} TF/s", flush=True)
    del qa, qb, c, cq
    torch.cuda.empty_cache()
