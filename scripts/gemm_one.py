"""One-shape GEMM launcher for ncu (diagnostic): ours (env knobs apply) or cuBLASLt."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12334_b200 as F
which = sys.argv[1] if len(sys.argv) > 1 else "ours"
m = n = k = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
if len(sys.argv) > 4:  # explicit m n k
    m, n, k = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
F.init()
x = torch.empty(m * k + k * n, dtype=torch.float32, device="cuda")
F.fill_synthetic(x, "normal", 3, 1.0)
if which in ("ours", "ours_q"):
    qa = F.quantize(x[: m * k]).codes
    qb = F.quantize(x[m * k:]).codes
    c = torch.empty((m, n), dtype=torch.float32, device="cuda")
    cq = torch.empty(m * n, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        if which == "ours":
            F.gemm_codes(qa, qb, m, n, k, "fp8", c=c)
        else:
            F.gemm_codes(qa, qb, m, n, k, "fp8", want_c=False, out_fmt="fp8", out_codes=cq)
else:
    a8 = x[: m * k].reshape(m, k).to(torch.float8_e4m3fn)
    b8 = x[m * k:].reshape(n, k).to(torch.float8_e5m2)
    one = torch.ones((), device="cuda")
    for _ in range(3):
        torch._scaled_mm(a8, b8.t(), scale_a=one, scale_b=one, out_dtype=torch.bfloat16)
torch.cuda.synchronize()
