#!/bin/bash
# Rolled, load-pipelined lean E5M2 epilogue: parity, ncu cycles, config-5 shapes, 8192^3 A/B.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_step_gpu.py tests/test_stack_gpu.py tests/test_conv_gpu.py -q -x -rf > gpurun_out/epi4_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/epi4_tests.log
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,gpc__cycles_elapsed.max
run() {  # label, args, env...
  lab=$1; args=$2; shift 2
  env "$@" timeout 200 ncu --metrics $M --clock-control none -k regex:gemm_tc2 --csv python scripts/gemm_one.py $args > gpurun_out/ncu_e4_$lab.csv 2>&1
  echo "$lab $args $@: $(grep -v '^==' gpurun_out/ncu_e4_$lab.csv | python -c "
import csv,sys
d={}
for r in csv.DictReader(l for l in sys.stdin if l.startswith('\"')): d[r['Metric Name']]=r['Metric Value']
print(d.get('gpc__cycles_elapsed.max'), d.get('gpu__time_duration.sum'), d.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'))
")"
}
run shortk "ours_q 65536 8192 512"
run shortk_old "ours_q 65536 8192 512" FP8B_GEMM_DBG=1024
run q8192 "ours_q 8192"
run q4096 "ours_q 4096"
run q4096_nb2 "ours_q 4096" FP8B_GEMM_NB=2
timeout 300 python scripts/stack_shapes.py > gpurun_out/epi4_stack.log 2>&1; cat gpurun_out/epi4_stack.log | grep -v "^NB=2"
timeout 300 python scripts/gemm_ab.py q=q:1 f=FP8B_GEMM_EPI:8x2 > gpurun_out/epi4_ab.log 2>&1; cat gpurun_out/epi4_ab.log
