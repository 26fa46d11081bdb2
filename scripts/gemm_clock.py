"""Sustained GEMM throughput with SM clock / power sampled by NVML every ~5 ms
(iteration helper): how much of the tcgen05 GEMM's gap to nominal is the power
cap, and what each kernel delivers per clock.

    python scripts/gemm_clock.py [--shape 8192x8192x8192] [--seconds 1.5]
"""
import argparse
import os
import statistics
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12334_b200 as F  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", nargs="*", default=["8192x8192x8192"])
ap.add_argument("--seconds", type=float, default=1.5)
ap.add_argument("--cublas", type=int, default=1)
a = ap.parse_args()

import pynvml  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(int(os.environ.get("LOCAL_RANK", "0")))


class Sampler:
    def __enter__(self):
        self.stop = False
        self.s = []
        self.t = threading.Thread(target=self.run, daemon=True)
        self.t.start()
        return self

    def run(self):
        while not self.stop:
            self.s.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                           pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
            time.sleep(0.005)

    def __exit__(self, *e):
        self.stop = True
        self.t.join()

    def summary(self):
        s = self.s[len(self.s) // 4:]  # skip the ramp
        return statistics.median(x[0] for x in s), statistics.median(x[1] for x in s), len(s)


def sustained(fn, flop, label):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fn()
    e1.record()
    torch.cuda.synchronize()
    reps = max(10, int(a.seconds * 1e3 / (e0.elapsed_time(e1) / 5)))
    with Sampler() as smp:
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    mhz, w, ns = smp.summary()
    tf = flop / (ms * 1e-3) / 1e12
    per_clk = tf * 1e12 / (148 * mhz * 1e6)
    print(f"{label:40s} {ms:.4f} ms {tf:7.1f} TF/s  sm {mhz:.0f} MHz  {w:.0f} W  "
          f"{per_clk:7.0f} FLOP/clk/SM ({per_clk / 16384 * 100:.1f}% of 16384)  n={ns}", flush=True)


F.init()
for sh in a.shapes:
    m, n, k = map(int, sh.split("x"))
    x = torch.empty(m * k + k * n, dtype=torch.float32, device="cuda")
    F.fill_synthetic(x, "normal", 3, 1.0)
    qa = F.quantize(x[: m * k]).codes
    qb = F.quantize(x[m * k:]).codes
    c = torch.empty((m, n), dtype=torch.float32, device="cuda")
    cq = torch.empty(m * n, dtype=torch.uint8, device="cuda")
    flop = 2.0 * m * n * k
    sustained(lambda: F.gemm_codes(qa, qb, m, n, k, "fp8", c=c), flop, f"ours {sh} f32")
    sustained(lambda: F.gemm_codes(qa, qb, m, n, k, "fp8", want_c=False, out_fmt="fp8",
                                   out_codes=cq), flop, f"ours {sh} e5m2")
    sustained(lambda: F.gemm_codes(qa, qb, m, n, k, "fp8", b_major="k", c=c), flop,
              f"ours {sh} f32 B K-major")
    if a.cublas:
        a8 = x[: m * k].reshape(m, k).to(torch.float8_e4m3fn)
        b8 = x[m * k:].reshape(n, k).to(torch.float8_e5m2)
        one = torch.ones((), device="cuda")
        sustained(lambda: torch._scaled_mm(a8, b8.t(), scale_a=one, scale_b=one,
                                           out_dtype=torch.bfloat16), flop, f"cublasLt {sh} bf16")
        del a8, b8
    del x, qa, qb, c, cq
    torch.cuda.empty_cache()
