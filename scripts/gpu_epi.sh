#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in 8x1 8x2; do
FP8B_GEMM_EPI=$v FP8B_GEMM_NB=2 timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x -k "tensor or splitk or large" > gpurun_out/epi_$v.log 2>&1; echo "$v tests rc=$?"; tail -2 gpurun_out/epi_$v.log
done
timeout 300 python scripts/gemm_ab.py e4x2=FP8B_GEMM_EPI:4x2 e8x1=FP8B_GEMM_EPI:8x1 e8x2=FP8B_GEMM_EPI:8x2 > gpurun_out/ab_epi.log 2>&1; cat gpurun_out/ab_epi.log
