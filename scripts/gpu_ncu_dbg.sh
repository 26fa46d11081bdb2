#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,gpc__cycles_elapsed.max,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed
for d in 0 6 2; do
FP8B_GEMM_DBG=$d timeout 200 ncu --metrics $M --clock-control none -k regex:gemm_tc2 --csv python scripts/gemm_one.py ours > gpurun_out/ncu_dbg_$d.csv 2>&1; echo "dbg=$d rc=$?"
done
timeout 200 ncu --metrics $M --clock-control none --csv python scripts/gemm_one.py cublas > gpurun_out/ncu_cublas.csv 2>&1; echo "cublas rc=$?"
for f in gpurun_out/ncu_dbg_0.csv gpurun_out/ncu_dbg_6.csv gpurun_out/ncu_dbg_2.csv gpurun_out/ncu_cublas.csv; do echo "== $f"; grep -v "^==" $f | python -c "
import csv,sys
for r in csv.DictReader(l for l in sys.stdin if l.startswith('\"')):
    print(r['ID'], r['Kernel Name'][:50], r['Metric Name'], r['Metric Value'])
" | tail -8; done
