#!/bin/bash
# Launch list (per-launch device time + DRAM bytes) of the bench's timed workload,
# after the same command has exited 0 without ncu.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
CMD="python bench.py --steps 3 --warmup 3 --no-extras --no-cpu-baseline --e2e-log2n 20"
$CMD > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err && \
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
