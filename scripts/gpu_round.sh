#!/bin/bash
# One gpurun call: parity tests, smoke, bench (outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 180 python -m pytest tests/test_gemm_gpu.py -q -x -k "tensor_engine_tolerance and 128-256" > gpurun_out/gemm_quick.log 2>&1; echo "gemm-quick rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -rf ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/pytest_gpu.log
