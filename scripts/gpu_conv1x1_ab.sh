#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L="1x1_64-256@56 1x1_256-64@56 1x1_128-512@28 1x1_512-128@28 1x1_256-1024@14 1x1_1024-256@14 1x1_512-2048@7 1x1_2048-512@7"
for pix in 262144 1000000; do
  echo "== FP8B_CONV_1X1_DGRAD_PIX=$pix"
  FP8B_CONV_1X1_DGRAD_PIX=$pix python scripts/bench_conv.py --only $L | python -c "
import json,sys
d=json.load(sys.stdin)
for k,v in d.items():
    if '@' in k: print(k, {p:v['passes_f32'][p]['ms'] for p in v['passes_f32']}, 'step', v['step']['ms'])
    elif 'all' in k: print(k, v)
"
done
for l in "256 64 56 1" "64 256 56 1"; do echo "== pieces $l"; python scripts/conv_pieces.py $l | grep "_q"; FP8B_CONV_1X1_DGRAD_PIX=1000000 python scripts/conv_pieces.py $l | grep "dgrad_q"; done
