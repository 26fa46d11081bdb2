"""LFSR-stream SR quantize / update time vs tensor size, warp vs CTA kernels (A/B)."""
import os, sys, subprocess
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12334_b200 as F
F.init()
mode = os.environ.get("FP8B_LFSR_CTA_MAX", "default")
for lg in (16, 18, 20, 22, 24):
    n = 1 << lg
    x = torch.empty(n, device="cuda"); F.fill_synthetic(x, "config2", 1, 0.01)
    out = torch.empty(n, dtype=torch.uint8, device="cuda")
    g = torch.randint(0, 120, (n,), dtype=torch.uint8, device="cuda")
    m = torch.randint(0, 0x3C00, (n,), dtype=torch.int16, device="cuda")
    mom = torch.zeros(n, device="cuda")
    def q(): F.quantize(x, "fp8", "stochastic", 3, out=out)
    def u(): F.sgd_momentum_update(g, "fp8", m, mom, lr=0.1, mu=0.9, scale=8192.0, master_mode="stochastic", seed=5)
    res = []
    for fn in (q, u):
        for _ in range(3): fn()
        st = torch.cuda.Stream(); torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            for _ in range(20): fn()
        gr.replay(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); gr.replay(); b.record(); torch.cuda.synchronize()
        res.append(a.elapsed_time(b) / 20 * 1e3)
    print(f"cta_max={mode} n=2^{lg} quantize {res[0]:.1f} us  update {res[1]:.1f} us", flush=True)
