#!/bin/bash
# ncu --set full captures of selected hot kernels; each command first runs clean.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for w in ${PROF_WHAT:-lfsr fp16ctr gemm}; do
  case $w in
    rne) K=quant_elem_kernel ;; lfsr) K=quant_lfsr_warp ;; fp16ctr) K=quant_elem_kernel ;;
    upd_rne) K=sgd_elem ;; upd_lfsr) K=sgd_lfsr_warp ;; gemm|gemm_e5m2) K=gemm_tc ;;
  esac
  RUN="python scripts/prof.py $w 3"
  case $w in
    conv3x3) K=conv_tc_kernel; RUN="python scripts/conv_one.py 256 256 14 3 fprop q" ;;
    conv1x1) K=conv_tc_kernel; RUN="python scripts/conv_one.py 64 256 56 1 fprop q" ;;
  esac
  timeout 300 $RUN > gpurun_out/prof_plain_$w.log 2>&1 && \
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
      -o gpurun_out/prof_$w -f $RUN > gpurun_out/ncu_$w.log 2>&1
  echo "$w rc=$?"
done
