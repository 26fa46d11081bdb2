#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/tf_profile.py > gpurun_out/tf_plain.log 2>&1; tail -1 gpurun_out/tf_plain.log | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/tf_profile.py > gpurun_out/tf_launches.csv 2>gpurun_out/tf_ncu.err; echo "ncu rc=$?"
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/tf_launches.csv')) if len(r) > 10]
h=rows[0]; ik=h.index('Kernel Name'); iv=h.index('Metric Value'); ig=h.index('Grid Size') if 'Grid Size' in h else None
data=[(r[ik], float(r[iv])) for r in rows[1:]]
half=len(data)//2
step=data[half:]   # second step
tot=sum(v for _,v in step)
agg=collections.defaultdict(lambda:[0,0.0])
for k,v in step:
    key=k.split('(')[0][:60]
    agg[key][0]+=1; agg[key][1]+=v
print('kernels', len(data), 'step kernels', len(step), 'step ms', tot/1e6)
for k,(n,v) in sorted(agg.items(), key=lambda x:-x[1][1])[:15]: print(f'{v/1e6:9.3f} ms {n:4d}  {k}')
PY
