#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/conv_one.py 64 64 56 3 fprop q > /dev/null 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv_halo --launch-skip 2 --launch-count 1 -o gpurun_out/halo_q3 -f python scripts/conv_one.py 64 64 56 3 fprop q > gpurun_out/halo_ncu.log 2>&1; echo "ncu rc=$?"
