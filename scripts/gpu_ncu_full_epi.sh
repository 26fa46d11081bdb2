#!/bin/bash
# Full ncu captures (source-level stall sampling) of the 2-SM GEMM, E5M2 output.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
FP8B_GEMM_EPI=8x1 timeout 400 ncu --set full --import-source on --clock-control none -k regex:gemm_tc2 -c 1 -o gpurun_out/gemm_q_8x1 -f python scripts/gemm_one.py ours_q > gpurun_out/ncu_full_8x1.log 2>&1; echo "8x1 rc=$?"
FP8B_GEMM_EPI=4x2 FP8B_GEMM_DBG=1024 timeout 400 ncu --set full --import-source on --clock-control none -k regex:gemm_tc2 -c 1 -o gpurun_out/gemm_q_4x2old -f python scripts/gemm_one.py ours_q > gpurun_out/ncu_full_4x2old.log 2>&1; echo "4x2old rc=$?"
ls -la gpurun_out/*.ncu-rep
