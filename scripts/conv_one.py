"""Run one conv pass a few times (for ncu): conv_one.py C F HW K kind [q]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12334_b200 as F  # noqa: E402

F.init()
c, f, hw, k = (int(v) for v in sys.argv[1:5])
kind, q = sys.argv[5], len(sys.argv) > 6
nb, pad = 256, k // 2
P = nb * hw * hw
xs = torch.empty(P * c, device="cuda"); F.fill_synthetic(xs, "halfnormal", 11, 1.0)
ws = torch.empty(f * k * k * c, device="cuda"); F.fill_synthetic(ws, "normal", 12, (2.0 / (k * k * c)) ** 0.5)
es = torch.empty(P * f, device="cuda"); F.fill_synthetic(es, "normal", 13, 1e-5 * 8192.0)
X = F.quantize(xs).reshaped([nb, hw, hw, c]); W = F.quantize(ws).reshaped([f, k, k, c])
E = F.quantize(es).reshaped([nb, hw, hw, f])
kw = dict(layout="nhwc", engine="tensor")
if q:
    kw.update(out_fmt="fp8", want_y=False)
for _ in range(3):
    if kind == "fprop":
        F.conv2d(X, W, 1, pad, **kw)
    elif kind == "dgrad":
        F.conv2d_backward_data(E, W, 1, pad, hw, hw, **kw)
    else:
        F.conv2d_backward_weights(X, E, k, k, 1, pad, **kw)
torch.cuda.synchronize()
print("ok")
