#!/bin/bash
# A-stationary short-K GEMM (config-5 FFN-in fprop shape): full ncu capture with source.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc2 -c 1 -o gpurun_out/gemm_ast -f python scripts/gemm_one.py ours_q 1048576 2048 512 > gpurun_out/ncu_ast.log 2>&1; echo "rc=$?"
# FP8B_GEMM_AST=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc2 -c 1 -o gpurun_out/gemm_noast -f python scripts/gemm_one.py ours_q 1048576 2048 512 > gpurun_out/ncu_noast.log 2>&1; echo "rc=$?"
