#!/bin/bash
# ncu --set full of one command's kernel: gpu_ncu_one.sh NAME KERNEL_REGEX SKIP cmd...
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
name=$1; k=$2; skip=$3; shift 3
timeout 300 "$@" > gpurun_out/plain_$name.log 2>&1 && \
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 \
    -o gpurun_out/prof_$name -f "$@" > gpurun_out/ncu_$name.log 2>&1
echo "$name rc=$?"
[ -f gpurun_out/prof_$name.ncu-rep ] || exit 1
python scripts/summarize_ncu.py report gpurun_out/prof_$name.ncu-rep gpurun_out/ncu_${name}_r02.md > /dev/null 2>&1
$NCU -i gpurun_out/prof_$name.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$name.csv 2>/dev/null
python scripts/src_hot.py gpurun_out/src_$name.csv ${HOT:-60} >> gpurun_out/ncu_${name}_r02.md 2>&1
rm -f gpurun_out/src_$name.csv gpurun_out/prof_$name.ncu-rep
