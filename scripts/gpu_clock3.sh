#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for d in 4 6 2 0; do
FP8B_GEMM_DBG=$d timeout 120 python scripts/gemm_clock.py --shapes 8192x8192x8192 --cublas 0 --seconds 0.3 > gpurun_out/clock3_dbg_$d.log 2>&1; echo "dbg=$d"; cat gpurun_out/clock3_dbg_$d.log
done
