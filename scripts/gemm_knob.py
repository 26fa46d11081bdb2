"""Interleaved timing of the fused-E5M2-output GEMM under environment knobs that
the launcher reads on every call. Usage:
  python scripts/gemm_knob.py KNOB=v1,v2,... MxNxK[:bk] ...   (value '-' = unset)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12334_b200 as F  # noqa: E402


def main():
    knob, vals = sys.argv[1].split("=")
    vals = vals.split(",")
    F.init()
    for spec in sys.argv[2:]:
        shape, _, bmaj = spec.partition(":")
        m, n, k = (int(v) for v in shape.split("x"))
        x = torch.empty(m * k + k * n, dtype=torch.float32, device="cuda")
        F.fill_synthetic(x, "normal", 3, 1.0)
        qa = F.quantize(x[: m * k]).codes
        qb = F.quantize(x[m * k:]).codes
        cq = torch.empty(m * n, dtype=torch.uint8, device="cuda")
        res = {v: [] for v in vals}
        sums = {}
        for rep in range(3):
            for v in vals:
                if v == "-":
                    os.environ.pop(knob, None)
                else:
                    os.environ[knob] = v
                kw = dict(want_c=False, out_fmt="fp8", out_codes=cq, b_major="k" if bmaj == "bk" else "n")
                for _ in range(3):
                    F.gemm_codes(qa, qb, m, n, k, "fp8", **kw)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                for _ in range(10):
                    F.gemm_codes(qa, qb, m, n, k, "fp8", **kw)
                e1.record()
                torch.cuda.synchronize()
                res[v].append(round(e0.elapsed_time(e1) * 100, 1))  # us per call
                s = int(cq[:: 997].to(torch.int64).sum().item())
                assert sums.setdefault("s", s) == s, (spec, v)
        os.environ.pop(knob, None)
        for v in vals:
            print(f"{spec:28s} {knob}={v:6s} {res[v]} us")


if __name__ == "__main__":
    main()
