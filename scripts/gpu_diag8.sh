#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
source <(sed -n '/^M=/,/^}/p' scripts/gpu_diag7.sh)
run q_alu "ours_q 8192" FP8B_GEMM_DBG=4096
run q_alu23 "ours_q 8192" FP8B_GEMM_DBG=12288
run q_alu_4x2 "ours_q 8192" FP8B_GEMM_DBG=4096 FP8B_GEMM_EPI=4x2
run q_alu23_4x2 "ours_q 8192" FP8B_GEMM_DBG=12288 FP8B_GEMM_EPI=4x2
