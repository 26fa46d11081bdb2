"""Print bench.py's config-4 conv numbers for some layers (iteration helper)."""
import json, os, subprocess, sys
out = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "bench_conv.py"), "--only"] + sys.argv[1:],
                     capture_output=True, text=True).stdout
d = json.loads(out)
for k, v in d.items():
    if isinstance(v, dict) and "passes_f32" in v:
        print(k, {kk: vv["ms"] for kk, vv in v["passes_f32"].items()}, "step", v["step"]["ms"])
