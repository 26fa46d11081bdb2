import os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import bench
import paper_1905_12334_b200 as F
F.init()
x = torch.zeros(4096, device="cuda"); out = torch.empty(4096, dtype=torch.uint8, device="cuda")
print("stream_probe 4096 elems:", round(bench._graph_ms(lambda: F.stream_probe(x, out, 1), 20) * 1000, 2), "us per node")
print("quantize 4096 elems   :", round(bench._graph_ms(lambda: F.quantize(x, "fp8", out=out), 20) * 1000, 2), "us per node")
a = torch.zeros(256 * 128, dtype=torch.uint8, device="cuda"); b = torch.zeros(128 * 256, dtype=torch.uint8, device="cuda")
cq = torch.empty(256 * 256, dtype=torch.uint8, device="cuda")
print("gemm 256x256x128      :", round(bench._graph_ms(lambda: F.gemm_codes(a, b, 256, 256, 128, "fp8", want_c=False, out_fmt="fp8", out_codes=cq), 20) * 1000, 2), "us per node")
a1 = torch.zeros(128 * 128, dtype=torch.uint8, device="cuda")
cq1 = torch.empty(128 * 256, dtype=torch.uint8, device="cuda")
print("gemm 128x256x128 (1SM):", round(bench._graph_ms(lambda: F.gemm_codes(a1, b, 128, 256, 128, "fp8", want_c=False, out_fmt="fp8", out_codes=cq1), 20) * 1000, 2), "us per node")
