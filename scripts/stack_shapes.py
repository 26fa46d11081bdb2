"""Per-shape timing of the config-5 linear stack GEMMs (E5M2 out, the stack's
layouts), NB=1 vs NB=2 (diagnostic)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12334_b200 as F
from paper_1905_12334_b200.stack import transformer_base_layers

T = int(os.environ.get("T", str(1 << 20)))
F.init()
layers = transformer_base_layers()
shapes = {}
for _, i, o in layers:
    shapes[(i, o)] = shapes.get((i, o), 0) + 1
buf = torch.randint(0, 0x3C, (T * 32000 + 4096,), dtype=torch.uint8, device="cuda")
buf2 = torch.randint(0, 0x3C, (T * 2048 + 4096,), dtype=torch.uint8, device="cuda")
w = torch.randint(0, 0x3C, (2048 * 32000,), dtype=torch.uint8, device="cuda")
out = torch.empty(T * 32000, dtype=torch.uint8, device="cuda")


def t(fn, reps=3):
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


tot = {}
for nb in os.environ.get("NBS", "1,2").split(","):
    os.environ["FP8B_GEMM_NB"] = nb
    total = 0.0
    for (i, o), cnt in shapes.items():
        x = buf2[: T * i]
        e = buf[: T * o]
        W = w[: i * o]
        kw = dict(want_c=False, out_fmt="fp8")
        fp = t(lambda: F.gemm_codes(x, W, T, o, i, "fp8", a_major="k", b_major="n", out_codes=out[: T * o], **kw))
        dg = t(lambda: F.gemm_codes(e, W, T, i, o, "fp8", a_major="k", b_major="k", out_codes=out[: T * i], **kw))
        wg = t(lambda: F.gemm_codes(x, e, i, o, T, "fp8", a_major="m", b_major="n", out_codes=out[: i * o], **kw))
        fl = 2.0 * T * i * o
        print(f"NB={nb} {i}x{o} x{cnt}: fprop {fp:.3f} ms ({fl/fp/1e9:.0f} TF/s)  dgrad {dg:.3f} ({fl/dg/1e9:.0f})  wgrad {wg:.3f} ({fl/wg/1e9:.0f})", flush=True)
        total += cnt * (fp + dg + wg)
    print(f"NB={nb} total GEMM ms per step: {total:.1f}", flush=True)
