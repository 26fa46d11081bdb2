#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_step_gpu.py tests/test_stack_gpu.py tests/test_dp_gpu.py tests/test_conv_gpu.py -q -x -rf > gpurun_out/tests_gemm.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/tests_gemm.log
timeout 300 python scripts/gemm_bench.py --shapes 8192x8192x8192 16384x1024x16384 4096x4096x4096 512x2048x1048576 > gpurun_out/gemm_bench_full.log 2>&1; cat gpurun_out/gemm_bench_full.log
timeout 300 python scripts/gemm_ab.py nb1=FP8B_GEMM_NB:1 auto= > gpurun_out/ab_auto.log 2>&1; cat gpurun_out/ab_auto.log
