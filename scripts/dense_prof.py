"""Config-1 Dense step launches (for an ncu launch list; diagnostic)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12334_b200 as F
F.init()
B, I, O_ = 512, 1024, 1024
x = torch.empty(B * I, dtype=torch.float32, device="cuda")
w = torch.empty(I * O_, dtype=torch.float32, device="cuda")
e = torch.empty(B * O_, dtype=torch.float32, device="cuda")
F.fill_synthetic(x, "normal", 0, 1.0)
F.fill_synthetic(w, "normal", 1, 1.0 / 32.0)
F.fill_synthetic(e, "normal", 2, 0.01 * 8192.0)
sc = F.LossScaler("dynamic-backoff", 8192.0, min_threshold_schedule=[(0, 8192.0)])
L = F.DenseLayer(w.reshape(I, O_), batch=B, lr=0.1, mu=0.9, scaler=sc, engine="tensor",
                 master_mode="stochastic", seed=1)
for it in range(3):
    L.step(x, e, it)
torch.cuda.synchronize()
print("ok")
