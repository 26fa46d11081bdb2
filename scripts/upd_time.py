"""Time the SGD update modes over 2^28 parameters (GB/s of algorithmic bytes; diagnostic)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12334_b200 as F
F.init()
n = 1 << 28
grad = torch.randint(0, 120, (n,), dtype=torch.uint8, device="cuda")
master = torch.randint(0, 0x3C00, (n,), dtype=torch.int16, device="cuda")
mom = torch.zeros(n, dtype=torch.float32, device="cuda")
w8 = torch.empty(n, dtype=torch.uint8, device="cuda")
res = []
for md, kw, bpe in [("lfsr", dict(master_mode="stochastic", bits="lfsr", seed=1), 13),
                    ("lfsr_w8", dict(master_mode="stochastic", bits="lfsr", seed=1, w_e5m2=w8), 14),
                    ("rne", dict(master_mode="nearest-even"), 13),
                    ("counter", dict(master_mode="stochastic", bits="counter", seed=1), 13),
                    ("counter_w8", dict(master_mode="stochastic", bits="counter", seed=1, w_e5m2=w8), 14),
                    ("rne_w8", dict(master_mode="nearest-even", w_e5m2=w8), 14)]:
    for _ in range(3):
        F.sgd_momentum_update(grad, "fp8", master, mom, lr=1e-4, mu=0.9, scale=8192.0, **kw)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(10):
        F.sgd_momentum_update(grad, "fp8", master, mom, lr=1e-4, mu=0.9, scale=8192.0, **kw)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    res.append(f"{md} {ms:.4f} ms {n * bpe / ms / 1e6:.0f} GB/s")
print(os.environ.get("FP8B_UPD_VARIANT", "0"), " | ".join(res))
