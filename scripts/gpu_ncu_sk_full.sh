#!/bin/bash
# ncu --set full of the stream-K hybrid kernel (diagnostic)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SH=${SH:-16384 1024 16384}
FP8B_GEMM_SK=1 FP8B_GEMM_NB=2 python scripts/gemm_one.py ours_q $SH > /dev/null 2>&1 && \
FP8B_GEMM_SK=1 FP8B_GEMM_NB=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc2 --launch-skip 2 --launch-count 1 -o gpurun_out/sk2_full -f python scripts/gemm_one.py ours_q $SH > gpurun_out/sk2_full.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/sk2_full.log
