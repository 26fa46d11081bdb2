#!/bin/bash
# EW=16 (four epilogue warps per TMEM lane quarter) for the shortest K: parity, shapes.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
FP8B_GEMM_EPI=16 FP8B_GEMM_NB=1 timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x -rf > gpurun_out/epi5_tests16.log 2>&1; echo "tests ew16 rc=$?"; tail -3 gpurun_out/epi5_tests16.log
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_step_gpu.py tests/test_stack_gpu.py -q -x -rf > gpurun_out/epi5_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/epi5_tests.log
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,gpc__cycles_elapsed.max
run() {  # label, args, env...
  lab=$1; args=$2; shift 2
  env "$@" timeout 200 ncu --metrics $M --clock-control none -k regex:gemm_tc2 --csv python scripts/gemm_one.py $args > gpurun_out/ncu_e5_$lab.csv 2>&1
  echo "$lab $args $@: $(grep -v '^==' gpurun_out/ncu_e5_$lab.csv | python -c "
import csv,sys
d={}
for r in csv.DictReader(l for l in sys.stdin if l.startswith('\"')): d[r['Metric Name']]=r['Metric Value']
print(d.get('gpc__cycles_elapsed.max'), d.get('gpu__time_duration.sum'), d.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'))
")"
}
run shortk16 "ours_q 65536 8192 512" FP8B_GEMM_EPI=16
run shortk8 "ours_q 65536 8192 512" FP8B_GEMM_EPI=8x2
run shortk16_k1024 "ours_q 65536 8192 1024" FP8B_GEMM_EPI=16
run shortk8_k1024 "ours_q 65536 8192 1024" FP8B_GEMM_EPI=8x2
timeout 300 python scripts/stack_shapes.py > gpurun_out/epi5_stack.log 2>&1; cat gpurun_out/epi5_stack.log | grep -v "^NB=2"
FP8B_GEMM_EPI=16 timeout 300 python scripts/stack_shapes.py > gpurun_out/epi5_stack16.log 2>&1; cat gpurun_out/epi5_stack16.log | grep -v "^NB=2"
