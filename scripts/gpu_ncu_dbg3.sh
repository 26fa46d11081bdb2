#!/bin/bash
# GEMM 8192^3 cycle counts under knob variants (min of 3 ncu runs each)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,gpc__cycles_elapsed.max
run() {  # label, env...
  label=$1; shift
  best=""
  for r in 1 2 3; do
    env "$@" timeout 200 ncu --metrics $M --clock-control none -k regex:gemm_tc2 --csv python scripts/gemm_one.py ours > gpurun_out/ncu3.csv 2>&1
    c=$(grep -v "^==" gpurun_out/ncu3.csv | python -c "
import csv,sys
v=[float(r['Metric Value'].replace(',','')) for r in csv.DictReader(l for l in sys.stdin if l.startswith('\"')) if r['Metric Name']=='gpc__cycles_elapsed.max']
print(int(min(v)))")
    best="$best $c"
  done
  echo "$label: $best"
}
run base FP8B_GEMM_DBG=0
run free FP8B_GEMM_DBG=14
run nold_noepi FP8B_GEMM_DBG=6
run noload FP8B_GEMM_DBG=2
run noepi FP8B_GEMM_DBG=4
run spin_full FP8B_GEMM_DBG=16
run spin_both FP8B_GEMM_DBG=48
run st4 FP8B_GEMM_STAGES=4
run st5 FP8B_GEMM_STAGES=5
