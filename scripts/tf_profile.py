"""One config-5 linear-stack step (after one warm-up step) for an ncu launch list (diagnostic)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1905_12334_b200 as F
F.init()
args = argparse.Namespace(tf_tokens=int(os.environ.get("T", str(4096 * 256))), tf_steps=1, tf_warmup=1)
print(bench.bench_transformer(F, args, 1, 0, None))
