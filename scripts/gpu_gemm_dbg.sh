#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x -rf > gpurun_out/gemm_tests.log 2>&1; echo "gemm-tests rc=$?"; tail -3 gpurun_out/gemm_tests.log
for d in 0 1 2; do
FP8B_GEMM_DBG=$d timeout 120 python scripts/gemm_bench.py --shapes 8192x8192x8192 --outs f32 > gpurun_out/gemm_dbg_$d.log 2>&1; echo "dbg=$d"; cat gpurun_out/gemm_dbg_$d.log
done
timeout 120 python scripts/gemm_bench.py --shapes 512x2048x1048576 2048x512x1048576 512x1536x1048576 16384x1024x16384 > gpurun_out/gemm_splitk.log 2>&1; cat gpurun_out/gemm_splitk.log
FP8B_GEMM_SPLITK=1 timeout 120 python scripts/gemm_bench.py --shapes 512x2048x1048576 16384x1024x16384 >> gpurun_out/gemm_splitk.log 2>&1; cat gpurun_out/gemm_splitk.log
