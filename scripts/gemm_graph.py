"""Device time per fused-E5M2-output GEMM as CUDA-graph replays (no host launch
overhead). Usage: python scripts/gemm_graph.py MxNxK[:bk][:am] ... (bk: B stored [N,K]; am: A stored [K,M])"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1905_12334_b200 as F  # noqa: E402

F.init()
for spec in sys.argv[1:]:
    shape, _, bmaj = spec.partition(":")
    amaj = "m" if "am" in bmaj else "k"
    m, n, k = (int(v) for v in shape.split("x"))
    x = torch.empty(m * k + k * n, dtype=torch.float32, device="cuda")
    F.fill_synthetic(x, "normal", 3, 1.0)
    qa = F.quantize(x[: m * k]).codes
    qb = F.quantize(x[m * k:]).codes
    cq = torch.empty(m * n, dtype=torch.uint8, device="cuda")
    kw = dict(want_c=False, out_fmt="fp8", out_codes=cq, b_major="k" if "bk" in bmaj else "n", a_major=amaj)
    ms = bench._graph_ms(lambda: F.gemm_codes(qa, qb, m, n, k, "fp8", **kw), 20)
    print(f"{spec:26s} {ms * 1000:8.1f} us  {2.0 * m * n * k / ms / 1e9:8.1f} TFLOP/s")
