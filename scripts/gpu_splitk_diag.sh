#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/splitk_launches.csv python scripts/gemm_bench.py --shapes 512x2048x1048576 --reps 2 > gpurun_out/splitk_ncu.log 2>&1; echo "rc=$?"
python - <<'P'
import csv
rows = list(csv.DictReader(l for l in open('gpurun_out/splitk_launches.csv') if l.startswith('"')))
for r in rows:
    if r.get('Metric Name') == 'gpu__time_duration.sum':
        print(r['Kernel Name'][:60], r['Metric Value'])
P
