#!/bin/bash
# conv: parity tests, then all-layer timings with the 1x1 GEMM routing on / off
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_conv_halo_gpu.py tests/test_conv_gpu.py -q -x > gpurun_out/conv_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/conv_tests.log
timeout 600 python scripts/bench_conv.py > gpurun_out/conv_on.json 2>&1; echo "on rc=$?"
FP8B_CONV_1X1_GEMM=0 timeout 600 python scripts/bench_conv.py > gpurun_out/conv_off.json 2>&1; echo "off rc=$?"
python - <<'PY'
import json
r={}
for lab in ("on","off"):
    try: r[lab]=json.load(open(f"gpurun_out/conv_{lab}.json"))
    except Exception as e: print(lab, "parse error", open(f"gpurun_out/conv_{lab}.json").read()[-1500:])
for k in r["on"]:
    v=r["on"][k]
    if isinstance(v,dict) and 'passes_f32' in v:
        w=r["off"][k]
        print(f"{k:18s} on {[vv['ms'] for vv in v['passes_f32'].values()]} step {v['step']['ms']}   off {[vv['ms'] for vv in w['passes_f32'].values()]} step {w['step']['ms']}")
for lab in r: print(lab, r[lab].get('all_layers_step'), r[lab].get('all_layers_passes_f32'))
PY
