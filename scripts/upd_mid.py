import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12334_b200 as F
F.init()
for n in (9*4096, 144*4096, 256*4096, 400*4096, 576*4096, 592*4096, 700*4096, 1024*4096):
    g = torch.randint(0, 120, (n,), dtype=torch.uint8, device="cuda")
    m = torch.randint(0, 0x3C00, (n,), dtype=torch.int16, device="cuda")
    mom = torch.zeros(n, device="cuda"); w8 = torch.empty(n, dtype=torch.uint8, device="cuda")
    fn = lambda: F.sgd_momentum_update(g, "fp8", m, mom, lr=0.1, mu=0.9, scale=8192.0, master_mode="stochastic", seed=5, w_e5m2=w8)
    for _ in range(3): fn()
    st = torch.cuda.Stream(); torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        for _ in range(20): fn()
    gr.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); gr.replay(); b.record(); torch.cuda.synchronize()
    print(f"blocks={n//4096:5d}  {a.elapsed_time(b)/20*1e3:6.1f} us", flush=True)
