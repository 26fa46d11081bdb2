"""SGD update time vs tensor size and master mode, CUDA-graph replays (diagnostic)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12334_b200 as F
F.init()
for lg in (20, 22, 24, 26):
    n = 1 << lg
    g = torch.randint(0, 120, (n,), dtype=torch.uint8, device="cuda")
    m = torch.randint(0, 0x3C00, (n,), dtype=torch.int16, device="cuda")
    mom = torch.zeros(n, device="cuda")
    w8 = torch.empty(n, dtype=torch.uint8, device="cuda")
    res = []
    for name, kw in [("rne", dict(master_mode="nearest-even")),
                     ("lfsr", dict(master_mode="stochastic", seed=5)),
                     ("lfsr_w8", dict(master_mode="stochastic", seed=5, w_e5m2=w8)),
                     ("ctr", dict(master_mode="stochastic", bits="counter", seed=5))]:
        fn = lambda: F.sgd_momentum_update(g, "fp8", m, mom, lr=0.1, mu=0.9, scale=8192.0, **kw)
        for _ in range(3): fn()
        st = torch.cuda.Stream(); torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            for _ in range(20): fn()
        gr.replay(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); gr.replay(); b.record(); torch.cuda.synchronize()
        us = a.elapsed_time(b) / 20 * 1e3
        res.append(f"{name} {us:.1f} us ({n * 13 / us / 1e6:.2f} TB/s)")
    print(f"n=2^{lg}: " + " | ".join(res), flush=True)
