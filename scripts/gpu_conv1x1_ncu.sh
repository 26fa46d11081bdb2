#!/bin/bash
# ncu --set full of the HBM-bound 1x1 conv passes at 56x56 (fused E5M2 output)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
cap() {  # name kernel-regex args...
  local name=$1 k=$2; shift 2
  timeout 300 python scripts/conv_one.py "$@" > gpurun_out/plain_$name.log 2>&1 && \
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o gpurun_out/prof_$name -f python scripts/conv_one.py "$@" > gpurun_out/ncu_$name.log 2>&1
  echo "$name rc=$?"
  [ -f gpurun_out/prof_$name.ncu-rep ] || return
  python scripts/summarize_ncu.py report gpurun_out/prof_$name.ncu-rep gpurun_out/ncu_${name}_r02.md > /dev/null 2>&1
  $NCU -i gpurun_out/prof_$name.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$name.csv 2>/dev/null
  python scripts/src_hot.py gpurun_out/src_$name.csv 60 >> gpurun_out/ncu_${name}_r02.md 2>&1
  rm -f gpurun_out/src_$name.csv gpurun_out/prof_$name.ncu-rep
}
cap c1x1_fprop_64_256 "gemm_tc|conv_tc" 64 256 56 1 fprop q
cap c1x1_dgrad_256_64 "conv_tc" 256 64 56 1 dgrad q
cap c1x1_fprop_256_64 "conv_tc" 256 64 56 1 fprop q
