"""Config-5 generator wgrad dW[512, 32000] = X^T E over T tokens under env
variants (diagnostic): python scripts/wgrad_gen.py 'NB=2' 'NB=1,SPLITK=8' ..."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12334_b200 as F

T = int(os.environ.get("T", str(1 << 20)))
F.init()
x = torch.randint(0, 0x3C, (T * 512,), dtype=torch.uint8, device="cuda")
e = torch.randint(0, 0x3C, (T * 32000,), dtype=torch.uint8, device="cuda")
out = torch.empty(512 * 32000, dtype=torch.uint8, device="cuda")
for spec in sys.argv[1:] or [""]:
    env = dict(kv.split("=") for kv in spec.split(",") if kv)
    for k, v in env.items():
        os.environ["FP8B_GEMM_" + k] = v
    fn = lambda: F.gemm_codes(x, e, 512, 32000, T, "fp8", a_major="m", b_major="n",  # noqa: E731
                              want_c=False, out_fmt="fp8", out_codes=out)
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(3):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{spec or 'default':24s} {ms:7.3f} ms  {2.0 * T * 512 * 32000 / ms / 1e9:6.0f} TF/s", flush=True)
    for k in env:
        os.environ.pop("FP8B_GEMM_" + k, None)
