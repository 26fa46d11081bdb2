#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python -m pytest tests/test_gemm_gpu.py -q -x -k "tensor_engine_tolerance" > gpurun_out/gemm_first.log 2>&1; rc=$?; echo "gemm-first rc=$rc"; tail -3 gpurun_out/gemm_first.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_step_gpu.py -q -rf > gpurun_out/gemm_tests.log 2>&1; echo "gemm-tests rc=$?"; tail -3 gpurun_out/gemm_tests.log
for v in 0 1; do
FP8B_GEMM_2SM=$v timeout 300 python - > gpurun_out/gemm_bench_$v.log 2>&1 <<'PY'
import torch, sys
sys.path.insert(0, '.')
import paper_1905_12334_b200 as F
F.init()
for (m, n, k) in [(8192, 8192, 8192), (16384, 16384, 16384), (16384, 1024, 16384), (4096, 4096, 4096), (2048, 2048, 2048)]:
    x = torch.empty(m * k + k * n, dtype=torch.float32, device="cuda")
    F.fill_synthetic(x, "normal", 3, 1.0)
    qa = F.quantize(x[: m * k]).codes; qb = F.quantize(x[m * k:]).codes
    del x
    c = torch.empty((m, n), dtype=torch.float32, device="cuda")
    cq = torch.empty(m * n, dtype=torch.uint8, device="cuda")
    for label, kw in [("f32", dict(c=c)), ("e5m2", dict(want_c=False, out_fmt="fp8", out_codes=cq))]:
        for _ in range(3): F.gemm_codes(qa, qb, m, n, k, "fp8", **kw)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record()
        reps = 10
        for _ in range(reps): F.gemm_codes(qa, qb, m, n, k, "fp8", **kw)
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        print(f"{m}x{n}x{k} {label} {ms:.3f} ms {2*m*n*k/ms/1e9:.1f} TF/s", flush=True)
    del qa, qb, c, cq; torch.cuda.empty_cache()
PY
echo "bench2sm=$v rc=$?"; cat gpurun_out/gemm_bench_$v.log
done
