#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread
timeout 300 ncu --metrics $M --clock-control none -k regex:sgd --csv python scripts/upd_one.py rne counter counter_w8 rne_w8 lfsr > gpurun_out/ncu_upd.csv 2>&1; echo rc=$?
grep -v "^==" gpurun_out/ncu_upd.csv | python -c "
import csv,sys
for r in csv.DictReader(l for l in sys.stdin if l.startswith('\"')):
    print(r['ID'], r['Kernel Name'][:60], r['Metric Name'], r['Metric Value'])
"
