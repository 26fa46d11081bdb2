#!/bin/bash
# Sustained GEMM clock / power / FLOP-per-clock: NB=1, NB=2, cuBLASLt (diagnostic).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for nb in 2 1; do
FP8B_GEMM_NB=$nb timeout 200 python scripts/gemm_clock.py --shapes 8192x8192x8192 --cublas $((nb==1)) --seconds 2 > gpurun_out/clock_nb$nb.log 2>&1; echo "nb=$nb"; cat gpurun_out/clock_nb$nb.log
done
