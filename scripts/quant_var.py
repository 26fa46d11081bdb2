"""Interleaved timing of the quant_elem_kernel launch variants (FP8B_QELEM_VAR)
on one box: the library is copied once per variant so each copy latches its own
value of the knob. Usage: python scripts/quant_var.py 0 1 2 3 [case ...]"""
import ctypes
import os
import shutil
import sys
import tempfile

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12334_b200 as F  # noqa: E402
from quant_ab import QCfg  # noqa: E402


def main():
    variants = [a for a in sys.argv[1:] if a.isdigit()]
    only = [a for a in sys.argv[1:] if not a.isdigit()]
    knob = os.environ.get("KNOB", "FP8B_QELEM_VAR")
    src = os.path.join(os.path.dirname(os.path.abspath(F.__file__)), "libfp8b200.so")
    tmp = tempfile.mkdtemp()
    n = 1 << 28
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    F.fill_synthetic(x, "config2", 0, 0.01)
    c8 = torch.empty(n, dtype=torch.uint8, device="cuda")
    c16 = torch.empty(n, dtype=torch.int16, device="cuda")
    cnt = torch.zeros(3, dtype=torch.int64, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    cases = {"e5m2_rne": (0, QCfg(0, 0, 1, 0, 0, 0, None), c8, 5),
             "fp16_sr_counter": (1, QCfg(1, 1, 1, 0, 0, 0, None), c16, 6),
             "e5m2_sr_counter": (0, QCfg(1, 1, 1, 0, 0, 0, None), c8, 5),
             "e5m2_sr_lfsr": (0, QCfg(1, 0, 1, 0, 0, 0, None), c8, 5),
             "fp16_sr_lfsr": (1, QCfg(1, 0, 1, 0, 0, 0, None), c16, 6)}
    if only:
        cases = {k: v for k, v in cases.items() if k in only}

    def call(L, fmt, cfg, out):
        rc = L.fp8b_quantize(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                             ctypes.c_int64(n), fmt, ctypes.byref(cfg),
                             ctypes.c_void_p(cnt.data_ptr()), st)
        assert rc == 0, rc

    libs = []
    for v in variants:
        os.environ[knob] = v
        dst = os.path.join(tmp, f"v{v}.so")
        shutil.copy(src, dst)
        L = ctypes.CDLL(dst, mode=ctypes.RTLD_LOCAL)
        assert L.fp8b_init() == 0
        for fmt, cfg, out, _ in cases.values():  # latch the knob
            call(L, fmt, cfg, out)
        libs.append(L)
    torch.cuda.synchronize()
    ref = {}
    res = {}
    for rep in range(3):
        for name, (fmt, cfg, out, bpe) in cases.items():
            for li, L in enumerate(libs):
                for _ in range(3):
                    call(L, fmt, cfg, out)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                for _ in range(10):
                    call(L, fmt, cfg, out)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / 10
                res.setdefault(name, [[] for _ in libs])[li].append(round(n * bpe / ms / 1e6, 1))
                if rep == 0:  # all variants must produce the same codes
                    h = int(out.view(torch.uint8)[:: 4099].to(torch.int64).sum().item())
                    assert ref.setdefault(name, h) == h, (name, variants[li])
    for name, rows in res.items():
        for v, r in zip(variants, rows):
            print(f"{name:18s} {knob}={v}  {r}  (GB/s)")
    shutil.rmtree(tmp, ignore_errors=True)


if __name__ == "__main__":
    main()
