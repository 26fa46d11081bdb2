#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for d in 0 7; do
FP8B_CONV_HALO_DBG=$d python scripts/conv_one.py 64 64 56 3 fprop > /dev/null 2>&1 && \
FP8B_CONV_HALO_DBG=$d timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_active.max,launch__grid_size,launch__block_size,launch__shared_mem_per_block_dynamic --clock-control none --launch-skip 4 --csv python scripts/conv_one.py 64 64 56 3 fprop > gpurun_out/list.csv 2>&1
echo "== dbg $d rc=$?"
grep -v "^==" gpurun_out/list.csv | python -c "
import csv,sys
rows=[r for r in csv.DictReader(l for l in sys.stdin if l.startswith('\"'))]
for r in rows: print('  ', r['ID'], r['Kernel Name'][:50], r['Metric Name'], r['Metric Value'], r['Metric Unit'])
"
done
