#!/bin/bash
# halo conv: parity tests, conv timings (halo on / off)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_conv_halo_gpu.py tests/test_conv_gpu.py -q -x > gpurun_out/halo_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/halo_tests.log
timeout 300 python scripts/bench_conv.py --only 3x3_64@56 3x3_128@28 > gpurun_out/halo_conv_on.json 2>&1; echo "bench on rc=$?"
FP8B_CONV_HALO=0 timeout 300 python scripts/bench_conv.py --only 3x3_64@56 3x3_128@28 > gpurun_out/halo_conv_off.json 2>&1; echo "bench off rc=$?"
python - <<'PY'
import json
for lab in ("on","off"):
    try:
        d=json.load(open(f"gpurun_out/halo_conv_{lab}.json"))
    except Exception as e:
        print(lab, "parse error", e); print(open(f"gpurun_out/halo_conv_{lab}.json").read()[-2000:]); continue
    for k,v in d.items():
        if isinstance(v,dict) and 'passes_f32' in v:
            print(lab, k, {kk:vv['ms'] for kk,vv in v['passes_f32'].items()}, 'step', v['step']['ms'])
PY
