#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
source <(sed -n '/^M=/,/^}/p' scripts/gpu_diag7.sh)
run q_alu "ours_q 8192" FP8B_GEMM_DBG=4096
run q_alu_sp0 "ours_q 8192" FP8B_GEMM_DBG=20480
run q_alu_sp1 "ours_q 8192" FP8B_GEMM_DBG=36864
run q_alu_sp01 "ours_q 8192" FP8B_GEMM_DBG=12288
