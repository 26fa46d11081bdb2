#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/gemm_clock.py --shapes 8192x8192x8192 16384x1024x16384 > gpurun_out/gemm_clock.log 2>&1; echo "rc=$?"
FP8B_GEMM_2SM=0 timeout 120 python scripts/gemm_clock.py --shapes 8192x8192x8192 --cublas 0 >> gpurun_out/gemm_clock.log 2>&1; echo "rc=$?"
cat gpurun_out/gemm_clock.log
