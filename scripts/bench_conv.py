"""Run only bench.py's config-4 conv section (iteration helper)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--conv-batch", type=int, default=256)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--only", nargs="*", default=None)
a = ap.parse_args()
import paper_1905_12334_b200 as F  # noqa: E402
F.init()
print(json.dumps(bench.bench_conv(F, a, reps=a.reps, only=a.only), indent=1))
