#!/bin/bash
# Does ALU load in the epilogue warps alone (no TMEM, no stores) slow the tensor pipe?
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,gpc__cycles_elapsed.max,smsp__inst_executed.sum
run() {  # label, args, env...
  lab=$1; args=$2; shift 2
  env "$@" timeout 200 ncu --metrics $M --clock-control none -k regex:gemm_tc2 --csv python scripts/gemm_one.py $args > gpurun_out/ncu_d_$lab.csv 2>&1
  echo "$lab $args $@: $(grep -v '^==' gpurun_out/ncu_d_$lab.csv | python -c "
import csv,sys
d={}
for r in csv.DictReader(l for l in sys.stdin if l.startswith('\"')): d[r['Metric Name']]=r['Metric Value']
print(' '.join(f'{k.split(\".\")[0].split(\"__\")[-1]}={v}' for k,v in d.items()))
")"
}
run q_full "ours_q 8192"
run q_noepi "ours_q 8192" FP8B_GEMM_DBG=4
run q_alu "ours_q 8192" FP8B_GEMM_DBG=4096
run q_alu_noload "ours_q 8192" FP8B_GEMM_DBG=4098
run q_noload "ours_q 8192" FP8B_GEMM_DBG=6
