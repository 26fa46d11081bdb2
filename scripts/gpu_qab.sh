#!/bin/bash
# quantizer parity tests, then an interleaved A/B of the config-2 sweep kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m pytest tests/test_quantize_gpu.py tests/test_update_gpu.py -x -q -m gpu > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_q.log
timeout 600 python scripts/quant_ab.py ab/libbase.so paper_1905_12334_b200/libfp8b200.so ${AB_CASES} > gpurun_out/qab.log 2>&1; echo "ab rc=$?"; cat gpurun_out/qab.log
