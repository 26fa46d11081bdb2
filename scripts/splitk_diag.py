"""Host vs device time per split-K GEMM call (diagnostic)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12334_b200 as F
F.init()
m, n, k = 512, 2048, 1 << 20
x = torch.empty(m * k + k * n, dtype=torch.float32, device="cuda")
F.fill_synthetic(x, "normal", 3, 1.0)
qa = F.quantize(x[: m * k]).codes
qb = F.quantize(x[m * k:]).codes
del x
c = torch.empty((m, n), dtype=torch.float32, device="cuda")
cq = torch.empty(m * n, dtype=torch.uint8, device="cuda")
for label in ["f32", "e5m2", "f32", "e5m2"]:
    kw = dict(c=c) if label == "f32" else dict(want_c=False, out_fmt="fp8", out_codes=cq)
    for _ in range(3):
        F.gemm_codes(qa, qb, m, n, k, "fp8", **kw)
    torch.cuda.synchronize()
    hs = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        t0 = time.perf_counter()
        F.gemm_codes(qa, qb, m, n, k, "fp8", **kw)
        hs.append((time.perf_counter() - t0) * 1e3)
    e1.record()
    torch.cuda.synchronize()
    print(label, "gpu ms/call", e0.elapsed_time(e1) / 10, "host ms/call", [round(h, 3) for h in hs], flush=True)
