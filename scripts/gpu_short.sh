#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_step_gpu.py tests/test_stack_gpu.py tests/test_conv_gpu.py -q -x -rf > gpurun_out/tests_short.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/tests_short.log
FP8B_GEMM_EPI=8x2 timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x -k "tensor or splitk or large" > gpurun_out/tests_ew8.log 2>&1; echo "ew8 tests rc=$?"; tail -2 gpurun_out/tests_ew8.log
NBS=1 timeout 300 python scripts/stack_shapes.py > gpurun_out/stack_shapes2.log 2>&1; cat gpurun_out/stack_shapes2.log
FP8B_GEMM_EPI=4x2 NBS=1 timeout 300 python scripts/stack_shapes.py > gpurun_out/stack_shapes3.log 2>&1; cat gpurun_out/stack_shapes3.log
