#!/bin/bash
# ncu source-level executed-count histogram of one kernel: gpu_ncu_hist.sh NAME REGEX SKIP cmd...
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
name=$1; k=$2; skip=$3; shift 3
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 \
    -o gpurun_out/prof_$name -f "$@" > gpurun_out/ncu_$name.log 2>&1
$NCU -i gpurun_out/prof_$name.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$name.csv 2>/dev/null
python scripts/src_hist.py gpurun_out/src_$name.csv ${WANT:-}
[ -n "$LIST" ] && python scripts/src_list.py gpurun_out/src_$name.csv $LIST > gpurun_out/list_$name.txt
rm -f gpurun_out/prof_$name.ncu-rep gpurun_out/src_$name.csv
