#!/bin/bash
# Register-staged E5M2 epilogue: parity, then ncu cycles of the variants, then the config-5 shapes.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_step_gpu.py tests/test_stack_gpu.py -q -x -rf > gpurun_out/epi3_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/epi3_tests.log
FP8B_GEMM_EPI=8x2 timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x -rf > gpurun_out/epi3_tests8.log 2>&1; echo "tests 8x2 rc=$?"; tail -2 gpurun_out/epi3_tests8.log
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,gpc__cycles_elapsed.max
run() {  # label, mode, env...
  lab=$1; mode=$2; shift 2
  env "$@" timeout 200 ncu --metrics $M --clock-control none -k regex:gemm_tc2 --csv python scripts/gemm_one.py $mode > gpurun_out/ncu_e3_$lab.csv 2>&1
  echo "$lab $mode $@: $(grep -v '^==' gpurun_out/ncu_e3_$lab.csv | python -c "
import csv,sys
d={}
for r in csv.DictReader(l for l in sys.stdin if l.startswith('\"')): d[r['Metric Name']]=r['Metric Value']
print(d.get('gpc__cycles_elapsed.max'), d.get('gpu__time_duration.sum'), d.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'))
")"
}
run q_4x2 ours_q FP8B_GEMM_EPI=4x2
run q_8x2 ours_q FP8B_GEMM_EPI=8x2
run q_8x1 ours_q FP8B_GEMM_EPI=8x1
run q_4x2_direct ours_q FP8B_GEMM_EPI=4x2 FP8B_EPI_TMA=0
run q_8x2_direct ours_q FP8B_GEMM_EPI=8x2 FP8B_EPI_TMA=0
run q_4x2_old ours_q FP8B_GEMM_EPI=4x2 FP8B_GEMM_DBG=1024
timeout 300 python scripts/stack_shapes.py > gpurun_out/epi3_stack.log 2>&1; cat gpurun_out/epi3_stack.log | grep -v "^NB=2"
