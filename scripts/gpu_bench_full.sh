#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -5 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print(d['value'], d['roofline']['frac'], d['e2e']['value'])
for k in ('gemm','dense_step','gemm_sharded','transformer'): print(k, json.dumps(d.get(k))[:600])
"
