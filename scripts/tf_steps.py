import argparse, os, sys
sys.path.insert(0, os.getcwd())
import bench
import paper_1905_12334_b200 as F
F.init()
for s, w in [(2, 1), (5, 2)]:
    args = argparse.Namespace(tf_tokens=4096 * 256, tf_steps=s, tf_warmup=w)
    r = bench.bench_transformer(F, args, 1, 0, None)
    print(s, w, r['ms_per_step'], r['tflops'])
