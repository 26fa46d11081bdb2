#!/bin/bash
# stream-K: parity tests, then the DP / SK / NB sweep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_streamk_gpu.py -q -x -rf > gpurun_out/sk_tests.log 2>&1; echo "sk tests rc=$?"
tail -5 gpurun_out/sk_tests.log
export SK_SHAPES=${SK_SHAPES:-4096x4096x4096,16384x1024x16384,6144x6144x6144,2048x2048x2048}
timeout 600 python scripts/sk_sweep.py "dp1=FP8B_GEMM_SK:0,FP8B_GEMM_NB:1" "dp2=FP8B_GEMM_SK:0,FP8B_GEMM_NB:2" \
   "sk1=FP8B_GEMM_SK:1,FP8B_GEMM_NB:1" "sk2=FP8B_GEMM_SK:1,FP8B_GEMM_NB:2" "auto=" > gpurun_out/sk_sweep.log 2>&1; echo "sweep rc=$?"
cat gpurun_out/sk_sweep.log
