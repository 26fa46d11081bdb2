"""Run one hot-path kernel a few times on the bench-size input (for ncu -k filters).

    python scripts/prof.py {rne|lfsr|fp16ctr|upd_rne|upd_lfsr|gemm|gemm_e5m2} [reps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12334_b200 as F  # noqa: E402


def main():
    what = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    F.init()
    n = 1 << 28
    if what in ("rne", "lfsr", "fp16ctr"):
        x = torch.empty(n, dtype=torch.float32, device="cuda")
        F.fill_synthetic(x, "config2", 0, 0.01)
        out8 = torch.empty(n, dtype=torch.uint8, device="cuda")
        out16 = torch.empty(n, dtype=torch.int16, device="cuda")
        for _ in range(reps):
            if what == "rne":
                F.quantize(x, "fp8", out=out8)
            elif what == "lfsr":
                F.quantize(x, "fp8", "stochastic", 1, out=out8)
            else:
                F.quantize(x, "fp16", "stochastic", 1, bits="counter", out=out16)
    elif what.startswith("upd"):
        grad = torch.randint(0, 120, (n,), dtype=torch.uint8, device="cuda")
        master = torch.randint(0, 0x3C00, (n,), dtype=torch.int16, device="cuda")
        mom = torch.zeros(n, dtype=torch.float32, device="cuda")
        kw = dict(master_mode="nearest-even") if what == "upd_rne" else dict(master_mode="stochastic", seed=1)
        for _ in range(reps):
            F.sgd_momentum_update(grad, "fp8", master, mom, lr=1e-4, mu=0.9, scale=8192.0, **kw)
    else:
        m = nn = k = 8192
        x = torch.empty(m * k + k * nn, dtype=torch.float32, device="cuda")
        F.fill_synthetic(x, "normal", 3, 1.0)
        qa = F.quantize(x[: m * k]).codes
        qb = F.quantize(x[m * k:]).codes
        for _ in range(reps):
            if what == "gemm":
                F.gemm_codes(qa, qb, m, nn, k, "fp8")
            else:
                F.gemm_codes(qa, qb, m, nn, k, "fp8", want_c=False, out_fmt="fp8")
    torch.cuda.synchronize()
    print("ok", what)


if __name__ == "__main__":
    main()
