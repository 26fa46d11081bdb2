#!/bin/bash
# Short-K GEMM (epilogue-bound, config-5 fprop-like): full ncu capture with source.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 400 ncu --set full --import-source on --clock-control none -k regex:gemm_tc2 -c 1 -o gpurun_out/gemm_shortk -f python scripts/gemm_one.py ours_q 65536 8192 512 > gpurun_out/ncu_shortk.log 2>&1; echo "rc=$?"
timeout 200 ncu --metrics gpu__time_duration.sum,gpc__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_tc2 --csv python scripts/gemm_one.py ours_q 4096 > gpurun_out/ncu_4096.csv 2>&1; echo "rc=$?"; grep -v "^==" gpurun_out/ncu_4096.csv | tail -5
