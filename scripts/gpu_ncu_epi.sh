#!/bin/bash
# ncu per-clock decomposition of the 2-SM GEMM at 8192^3 (diagnostic knobs).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,gpc__cycles_elapsed.max,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum
for d in ${DBGS:-0 6 2 4 2050 2048}; do
FP8B_GEMM_DBG=$d timeout 200 ncu --metrics $M --clock-control none -k regex:gemm_tc2 --csv python scripts/gemm_one.py ours > gpurun_out/ncu_epi_$d.csv 2>&1; echo "dbg=$d rc=$?"
grep -v "^==" gpurun_out/ncu_epi_$d.csv | python -c "
import csv,sys
for r in csv.DictReader(l for l in sys.stdin if l.startswith('\"')):
    print(r['ID'], r['Kernel Name'][:40], r['Metric Name'], r['Metric Value'])
" | tail -6
done
