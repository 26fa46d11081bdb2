#!/bin/bash
# quick iteration: selected tests, then optional ncu of selected kernels, then bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest ${TESTS:-tests -m gpu} -q -rf -x > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_iter.log
if [ -n "$PROF_WHAT" ]; then PROF_WHAT="$PROF_WHAT" bash scripts/gpu_prof_only.sh; fi
if [ -z "$NO_BENCH" ]; then timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; fi
