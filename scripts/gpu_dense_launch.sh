cd $GRAFT_REPO_ROOT
python scripts/dense_prof.py > /dev/null 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv python scripts/dense_prof.py > gpurun_out/dense.csv 2>&1
echo rc=$?
grep -v "^==" gpurun_out/dense.csv | python -c "
import csv,sys
rows=[r for r in csv.DictReader(l for l in sys.stdin if l.startswith('\"'))]
cur=None
for r in rows:
    if r['Metric Name']=='gpu__time_duration.sum': print(r['ID'], r['Kernel Name'][:70], r['Metric Value'], r['Metric Unit'])
    if r['Metric Name']=='launch__grid_size': print('     grid', r['Metric Value'])
" | tail -40
