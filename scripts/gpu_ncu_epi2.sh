#!/bin/bash
# ncu cycles of the 2-SM GEMM at 8192^3: epilogue variants (warps x buffers, direct stores).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,gpc__cycles_elapsed.max
run() {  # label, mode, env...
  lab=$1; mode=$2; shift 2
  env "$@" timeout 200 ncu --metrics $M --clock-control none -k regex:gemm_tc2 --csv python scripts/gemm_one.py $mode > gpurun_out/ncu_e2_$lab.csv 2>&1
  echo "$lab $mode $@: $(grep -v '^==' gpurun_out/ncu_e2_$lab.csv | python -c "
import csv,sys
d={}
for r in csv.DictReader(l for l in sys.stdin if l.startswith('\"')): d[r['Metric Name']]=r['Metric Value']
print(d.get('gpc__cycles_elapsed.max'), d.get('gpu__time_duration.sum'), d.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'))
")"
}
run f32_4x2 ours FP8B_GEMM_EPI=4x2
run f32_8x2 ours FP8B_GEMM_EPI=8x2
run f32_8x1 ours FP8B_GEMM_EPI=8x1
run f32_direct ours FP8B_EPI_TMA=0
run q_4x2 ours_q FP8B_GEMM_EPI=4x2
run q_8x2 ours_q FP8B_GEMM_EPI=8x2
run q_direct ours_q FP8B_EPI_TMA=0
run q_drain ours_q FP8B_GEMM_DBG=2048
