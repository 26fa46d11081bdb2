"""Time each piece of a config-4 layer step (iteration helper)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1905_12334_b200 as F  # noqa: E402

F.init()
nb, c, f, hw, k = 256, int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
pad = k // 2
P = nb * hw * hw
xs = torch.empty(P * c, device="cuda"); F.fill_synthetic(xs, "halfnormal", 11, 1.0)
ws = torch.empty(f * k * k * c, device="cuda"); F.fill_synthetic(ws, "normal", 12, (2.0 / (k * k * c)) ** 0.5)
es = torch.empty(P * f, device="cuda"); F.fill_synthetic(es, "normal", 13, 1e-5 * 8192.0)
X = F.quantize(xs).reshaped([nb, hw, hw, c]); W = F.quantize(ws).reshaped([f, k, k, c])
E = F.quantize(es).reshaped([nb, hw, hw, f])
master = F.quantize(ws, "fp16").codes
mom = torch.zeros(f * k * k * c, device="cuda")
sc = F.LossScaler("dynamic-backoff", 8192.0, min_threshold_schedule=[(0, 8192.0)])
bwd = F.Counters()
qdw = F.quantize(torch.zeros(f * k * k * c, device="cuda")).codes
pieces = {
    "fprop_f32": lambda: F.conv2d(X, W, 1, pad, layout="nhwc", engine="tensor"),
    "fprop_q": lambda: F.conv2d(X, W, 1, pad, layout="nhwc", engine="tensor", out_fmt="fp8", want_y=False),
    "fprop_f32_and_q": lambda: F.conv2d(X, W, 1, pad, layout="nhwc", engine="tensor", out_fmt="fp8"),
    "dgrad_f32": lambda: F.conv2d_backward_data(E, W, 1, pad, hw, hw, layout="nhwc", engine="tensor"),
    "dgrad_q": lambda: F.conv2d_backward_data(E, W, 1, pad, hw, hw, layout="nhwc", engine="tensor",
                                              out_fmt="fp8", out_counters=bwd, want_y=False),
    "wgrad_f32": lambda: F.conv2d_backward_weights(X, E, k, k, 1, pad, layout="nhwc", engine="tensor"),
    "wgrad_q": lambda: F.conv2d_backward_weights(X, E, k, k, 1, pad, layout="nhwc", engine="tensor",
                                                 out_fmt="fp8", out_counters=bwd, want_y=False),
    "update": lambda: F.sgd_momentum_update(qdw, "fp8", master, mom, lr=0.1, mu=0.9, scaler=sc,
                                            skip_counters=bwd, master_mode="stochastic", seed=5,
                                            w_e5m2=W.codes),
    "scaler": lambda: sc.step_async(True, 0, counters=bwd),
}
for name, fn in pieces.items():
    print(f"{name:18s} {bench._graph_ms(fn, 5) * 1000:9.1f} us", flush=True)
