#!/bin/bash
# ncu metrics: stream-K vs data-parallel, same shape (diagnostic)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SH=${SH:-16384 1024 16384}
M=gpu__time_duration.sum,gpc__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.max.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.min.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second,launch__grid_size,sm__cycles_active.avg,sm__cycles_active.min
for v in "dp2 FP8B_GEMM_SK=0 FP8B_GEMM_NB=2" "sk2 FP8B_GEMM_SK=1 FP8B_GEMM_NB=2" "pk2 FP8B_GEMM_SK=2 FP8B_GEMM_NB=2"; do
  set -- $v; lab=$1; shift
  env "$@" python scripts/gemm_one.py ours_q $SH > /dev/null 2>&1 && \
  env "$@" timeout 200 ncu --metrics $M --clock-control none -k regex:gemm_tc2 --launch-skip 2 --launch-count 1 --csv python scripts/gemm_one.py ours_q $SH > gpurun_out/sk_$lab.csv 2>&1
  echo "== $lab rc=$?"
  grep -v "^==" gpurun_out/sk_$lab.csv | python -c "
import csv,sys
rows=[r for r in csv.DictReader(l for l in sys.stdin if l.startswith('\"'))]
for r in rows: print('  ', r['Metric Name'], r['Metric Value'], r['Metric Unit'])
"
done
