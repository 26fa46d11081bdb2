#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_conv_halo_gpu.py -q -x > gpurun_out/halo_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/halo_tests.log
python scripts/conv_one.py 64 64 56 3 fprop > /dev/null 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv_halo --launch-skip 2 --launch-count 1 -o gpurun_out/halo_f32 -f python scripts/conv_one.py 64 64 56 3 fprop > gpurun_out/halo_ncu.log 2>&1; echo "ncu rc=$?"
python scripts/conv_one.py 64 64 56 3 fprop q > /dev/null 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv_halo --launch-skip 2 --launch-count 1 -o gpurun_out/halo_q -f python scripts/conv_one.py 64 64 56 3 fprop q >> gpurun_out/halo_ncu.log 2>&1; echo "ncu q rc=$?"
