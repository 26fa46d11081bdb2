#!/bin/bash
# Round-2 ncu evidence: HBM access-mix ceiling, per-piece conv step times, full
# captures of the hot kernels (each command first runs clean without ncu) and the
# launch list of a short bench run.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
./scripts/hbm_ceiling > gpurun_out/hbm_ceiling.txt 2>&1; echo "ceiling rc=$?"
for l in "64 64 56 3" "128 128 28 3" "256 256 14 3" "512 512 7 3" "64 256 56 1" "256 64 56 1" "128 512 28 1" "512 128 28 1" "256 1024 14 1" "1024 256 14 1" "512 2048 7 1" "2048 512 7 1"; do
  echo "== layer C F HW K = $l"; python scripts/conv_pieces.py $l
done > gpurun_out/conv_pieces.txt 2>&1; echo "pieces rc=$?"
cap() {  # name kernel-regex command...
  local name=$1 k=$2; shift 2
  timeout 300 "$@" > gpurun_out/prof_plain_$name.log 2>&1 && \
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o gpurun_out/prof_$name -f "$@" > gpurun_out/ncu_$name.log 2>&1
  echo "$name rc=$?"
}
cap rne quant_elem_kernel python scripts/prof.py rne 3
cap lfsr quant_lfsr_warp_kernel python scripts/prof.py lfsr 3
cap fp16ctr quant_elem_kernel python scripts/prof.py fp16ctr 3
cap gemm_e5m2 gemm_tc2 python scripts/prof.py gemm_e5m2 3
cap upd_lfsr sgd_lfsr_warp_kernel python scripts/prof.py upd_lfsr 3
bash scripts/gpu_launches.sh
for name in rne lfsr fp16ctr gemm_e5m2 upd_lfsr; do
  [ -f gpurun_out/prof_$name.ncu-rep ] || continue
  python scripts/summarize_ncu.py report gpurun_out/prof_$name.ncu-rep gpurun_out/ncu_${name}_r02.md > /dev/null 2>&1
  $NCU -i gpurun_out/prof_$name.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$name.csv 2>/dev/null
  python scripts/src_hot.py gpurun_out/src_$name.csv 40 >> gpurun_out/ncu_${name}_r02.md 2>&1
  rm -f gpurun_out/src_$name.csv gpurun_out/prof_$name.ncu-rep
done
python scripts/summarize_ncu.py launches gpurun_out/launches.csv gpurun_out/launches_r02.md > /dev/null 2>&1
echo "summaries rc=$?"
