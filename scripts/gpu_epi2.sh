#!/bin/bash
# GEMM epilogue A/B: two-chunk TMEM loads + early accumulator release (default)
# vs the one-chunk late-release loop (FP8B_GEMM_DBG=1024); parity first.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_step_gpu.py tests/test_stack_gpu.py -q -x -rf > gpurun_out/epi2_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/epi2_tests.log
for d in 0 1024; do
FP8B_GEMM_DBG=$d timeout 200 python scripts/gemm_clock.py --shapes 8192x8192x8192 16384x1024x16384 --cublas 0 --seconds 0.5 > gpurun_out/epi2_clock_$d.log 2>&1; echo "dbg=$d"; cat gpurun_out/epi2_clock_$d.log
done
timeout 300 python scripts/stack_shapes.py > gpurun_out/epi2_stack.log 2>&1; cat gpurun_out/epi2_stack.log
FP8B_GEMM_DBG=1024 timeout 300 python scripts/stack_shapes.py > gpurun_out/epi2_stack_old.log 2>&1; cat gpurun_out/epi2_stack_old.log
