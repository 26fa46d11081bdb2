#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
M=gpu__time_duration.sum,gpc__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,lts__t_sectors_srcunit_tex.sum,sm__cycles_elapsed.avg.per_second,launch__grid_size,launch__cluster_dim_x
timeout 200 ncu --metrics $M --clock-control none -k regex:gemm_tc2 --csv python scripts/gemm_one.py ours > gpurun_out/cmp_ours.csv 2>&1; echo "ours rc=$?"
timeout 200 ncu --metrics $M --clock-control none -k regex:nvjet --csv python scripts/gemm_one.py cublas > gpurun_out/cmp_cublas.csv 2>&1; echo "cublas rc=$?"
for f in gpurun_out/cmp_ours.csv gpurun_out/cmp_cublas.csv; do echo "== $f"; grep -v "^==" $f | python -c "
import csv,sys
rows=[r for r in csv.DictReader(l for l in sys.stdin if l.startswith('\"'))]
last=rows[-1]['ID']
for r in rows:
    if r['ID']==last: print(r['Metric Name'], r['Metric Value'], r['Metric Unit'])
"; done
