"""One SGD update launch per mode over 2^28 parameters (ncu target, diagnostic)."""
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
modes = sys.argv[1:] or ["rne", "lfsr", "counter_w8", "counter"]
for md in modes:
    kw = {"rne": dict(master_mode="nearest-even"), "lfsr": dict(master_mode="stochastic", seed=1),
          "counter_w8": dict(master_mode="stochastic", bits="counter", seed=1, w_e5m2=w8),
          "counter": dict(master_mode="stochastic", bits="counter", seed=1),
          "rne_w8": dict(master_mode="nearest-even", w_e5m2=w8)}[md]
    for _ in range(2):
        F.sgd_momentum_update(grad, "fp8", master, mom, lr=1e-4, mu=0.9, scale=8192.0, **kw)
torch.cuda.synchronize()
