#!/bin/bash
# Round-end ncu evidence: full captures of the hot kernels (each command first
# runs clean without ncu) and the launch list of a short bench run.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
cap() {  # name kernel-regex command...
  local name=$1 k=$2; shift 2
  timeout 300 "$@" > gpurun_out/prof_plain_$name.log 2>&1 && \
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o gpurun_out/prof_$name -f "$@" > gpurun_out/ncu_$name.log 2>&1
  echo "$name rc=$?"
}
cap lfsr quant_lfsr_warp_kernel python scripts/prof.py lfsr 3
cap fp16ctr quant_elem_kernel python scripts/prof.py fp16ctr 3
cap gemm_e5m2 gemm_tc2 python scripts/prof.py gemm_e5m2 3
cap gemm_ast gemm_tc2 python scripts/gemm_one.py ours_q 1048576 2048 512
cap upd_lfsr sgd_lfsr_warp_kernel python scripts/prof.py upd_lfsr 3
bash scripts/gpu_launches.sh
# summaries on the box (the reports themselves exceed gpurun's copy-back limit)
for name in lfsr fp16ctr gemm_e5m2 gemm_ast upd_lfsr; do
  [ -f gpurun_out/prof_$name.ncu-rep ] || continue
  python scripts/summarize_ncu.py report gpurun_out/prof_$name.ncu-rep gpurun_out/ncu_${name}_r01.md > /dev/null 2>&1
  $NCU -i gpurun_out/prof_$name.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$name.csv 2>/dev/null
  python scripts/src_hot.py gpurun_out/src_$name.csv 40 >> gpurun_out/ncu_${name}_r01.md 2>&1
  rm -f gpurun_out/src_$name.csv gpurun_out/prof_$name.ncu-rep
done
python scripts/summarize_ncu.py launches gpurun_out/launches.csv gpurun_out/launches_r01.md > /dev/null 2>&1
echo "summaries rc=$?"
