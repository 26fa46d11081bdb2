#!/bin/bash
# ncu captures of the hot kernels (each command first runs clean without ncu).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for w in ${PROF_WHAT:-lfsr fp16ctr gemm}; do
  case $w in
    rne) K=quant_elem_kernel ;; lfsr) K=quant_lfsr_staged ;; fp16ctr) K=quant_elem_kernel ;;
    upd_rne) K=sgd_elem ;; upd_lfsr) K=sgd_lfsr_staged ;; gemm|gemm_e5m2) K=gemm_tc_kernel ;;
  esac
  timeout 300 python scripts/prof.py $w 3 > gpurun_out/prof_plain_$w.log 2>&1 && \
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
      -o gpurun_out/prof_$w -f python scripts/prof.py $w 3 > gpurun_out/ncu_$w.log 2>&1
  echo "$w rc=$?"
done
# launch list of a short bench run (per-launch device times, cold cache, serialised)
timeout 300 python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bench_small.json 2>&1 && \
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
