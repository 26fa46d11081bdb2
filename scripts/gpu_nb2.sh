#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
FP8B_GEMM_NB=2 timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x -k "tensor" > gpurun_out/nb2_tests.log 2>&1; echo "nb2 tests rc=$?"; tail -3 gpurun_out/nb2_tests.log
FP8B_GEMM_NB=2 timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x -k "splitk or large" > gpurun_out/nb2_tests2.log 2>&1; echo "nb2 tests2 rc=$?"; tail -3 gpurun_out/nb2_tests2.log
AB_ARGS="nb1=FP8B_GEMM_NB:1 nb2=FP8B_GEMM_NB:2" timeout 300 python scripts/gemm_ab.py nb1=FP8B_GEMM_NB:1 nb2=FP8B_GEMM_NB:2 > gpurun_out/ab_nb.log 2>&1; cat gpurun_out/ab_nb.log
