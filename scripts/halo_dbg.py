"""Time the halo conv kernel under FP8B_CONV_HALO_DBG knobs (diagnostic)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12334_b200 as F
F.init()
c, f, hw, k = (int(v) for v in sys.argv[1:5])
nb, pad = 256, k // 2
P = nb * hw * hw
xs = torch.empty(P * c, device="cuda"); F.fill_synthetic(xs, "halfnormal", 11, 1.0)
ws = torch.empty(f * k * k * c, device="cuda"); F.fill_synthetic(ws, "normal", 12, (2.0 / (k * k * c)) ** 0.5)
X = F.quantize(xs).reshaped([nb, hw, hw, c]); W = F.quantize(ws).reshaped([f, k, k, c])
for q in (False, True):
    for dbg in ("0", "4", "7"):
        os.environ["FP8B_CONV_HALO_DBG"] = dbg.split("s")[0]
        os.environ["FP8B_CONV_HALO_STAGES"] = dbg.split("s")[1] if "s" in dbg else "4"
        kw = dict(layout="nhwc", engine="tensor")
        if q: kw.update(out_fmt="fp8", want_y=False)
        for _ in range(3): F.conv2d(X, W, 1, pad, **kw)
        st = torch.cuda.Stream()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(10): F.conv2d(X, W, 1, pad, stream=st, **kw)
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): g.replay()
        e1.record(); torch.cuda.synchronize()
        print(f"{c}x{f}@{hw} k{k} {'q' if q else 'f32'} dbg={dbg} {e0.elapsed_time(e1)/50*1e3:.1f} us (graph)", flush=True)
