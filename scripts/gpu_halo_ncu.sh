#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed
for args in "64 64 56 3 fprop" "64 64 56 3 fprop q" "128 128 28 3 fprop q" "64 64 56 3 wgrad" "64 256 56 1 fprop q" "256 64 56 1 fprop q"; do
  python scripts/conv_one.py $args > /dev/null 2>&1 && \
  timeout 300 ncu --metrics $M --clock-control none -k regex:"conv_|splitk" --launch-skip 2 --launch-count 2 --csv python scripts/conv_one.py $args > gpurun_out/cv.csv 2>&1
  echo "== $args rc=$?"
  grep -v "^==" gpurun_out/cv.csv | python -c "
import csv,sys
rows=[r for r in csv.DictReader(l for l in sys.stdin if l.startswith('\"'))]
for r in rows: print('  ', r['Kernel Name'][:60], r['Metric Name'], r['Metric Value'], r['Metric Unit'])
"
done
