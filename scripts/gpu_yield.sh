#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
source <(sed -n '/^M=/,/^}/p' scripts/gpu_diag7.sh)
run q8192 "ours_q 8192"
run q8192_y1 "ours_q 8192" FP8B_GEMM_DBG=131072
run q8192_yall "ours_q 8192" FP8B_GEMM_DBG=983040
run shortk "ours_q 65536 8192 512"
run shortk_y1 "ours_q 65536 8192 512" FP8B_GEMM_DBG=131072
