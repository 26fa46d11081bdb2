#!/bin/bash
# Is the 4096^3 / short-K GEMM operand-load bound? (no-MMA and drain-only diagnostics)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,gpc__cycles_elapsed.max,lts__t_bytes.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum
run() {  # label, args, env...
  lab=$1; args=$2; shift 2
  env "$@" timeout 200 ncu --metrics $M --clock-control none -k regex:gemm_tc2 --csv python scripts/gemm_one.py $args > gpurun_out/ncu_d6_$lab.csv 2>&1
  echo "$lab $args $@: $(grep -v '^==' gpurun_out/ncu_d6_$lab.csv | python -c "
import csv,sys
d={}
for r in csv.DictReader(l for l in sys.stdin if l.startswith('\"')): d[r['Metric Name']]=r['Metric Value']
print(' '.join(f'{k.split(\".\")[0].split(\"__\")[-1]}={v}' for k,v in d.items()))
")"
}
for d in 0 1 2048 4; do
run q4096_$d "ours_q 4096" FP8B_GEMM_DBG=$d
run shortk_$d "ours_q 65536 8192 512" FP8B_GEMM_DBG=$d
done
run q4096_nb2 "ours_q 4096" FP8B_GEMM_NB=2
run shortk_nb2 "ours_q 65536 8192 512" FP8B_GEMM_NB=2
run q8192 "ours_q 8192"
