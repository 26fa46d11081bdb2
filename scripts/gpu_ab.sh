#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/gemm_ab.py ${AB_ARGS} > gpurun_out/ab.log 2>&1; echo rc=$?; cat gpurun_out/ab.log
