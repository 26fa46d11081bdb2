#!/bin/bash
# Warp-uniform MMA issuer: parity, then ncu cycles (8192^3, 4096^3, short K) and interleaved wall clock.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_step_gpu.py tests/test_stack_gpu.py -q -x -rf > gpurun_out/mma1_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/mma1_tests.log
source <(sed -n '/^M=/,/^}/p' scripts/gpu_diag7.sh)
run q8192 "ours_q 8192"
run f8192 "ours 8192"
run q8192_noepi "ours_q 8192" FP8B_GEMM_DBG=4
run q8192_4x2 "ours_q 8192" FP8B_GEMM_EPI=4x2
run q4096 "ours_q 4096"
run shortk "ours_q 65536 8192 512"
timeout 300 python scripts/gemm_ab.py q=q:1 f=FP8B_GEMM_EPI:8x2 q42=q:1,FP8B_GEMM_EPI:4x2 > gpurun_out/mma1_ab.log 2>&1; cat gpurun_out/mma1_ab.log
