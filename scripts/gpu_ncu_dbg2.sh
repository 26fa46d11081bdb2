#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,gpc__cycles_elapsed.max
for d in 14 6; do
FP8B_GEMM_DBG=$d timeout 200 ncu --metrics $M --clock-control none -k regex:gemm_tc2 --csv python scripts/gemm_one.py ours > gpurun_out/ncu2_dbg_$d.csv 2>&1; echo "dbg=$d rc=$?"
grep -v "^==" gpurun_out/ncu2_dbg_$d.csv | python -c "
import csv,sys
for r in csv.DictReader(l for l in sys.stdin if l.startswith('\"')):
    print(r['ID'], r['Metric Name'], r['Metric Value'])
" | tail -4
done
