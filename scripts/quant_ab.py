"""A/B timing of the config-2 sweep kernels between builds of the library
(interleaved on one box). Usage: python scripts/quant_ab.py libA.so libB.so ... [case ...]"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12334_b200 as F  # noqa: E402


class QCfg(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("bits", ctypes.c_int32), ("seed", ctypes.c_uint64),
                ("saturate", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("block_offset", ctypes.c_int64), ("rbits", ctypes.c_void_p)]


def main():
    names = [a for a in sys.argv[1:] if a.endswith(".so")]
    only = [a for a in sys.argv[1:] if not a.endswith(".so")]
    libs = [ctypes.CDLL(os.path.abspath(p), mode=ctypes.RTLD_LOCAL) for p in names]
    for L in libs:
        assert L.fp8b_init() == 0
    n = 1 << 28
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    F.fill_synthetic(x, "config2", 0, 0.01)
    c8 = torch.empty(n, dtype=torch.uint8, device="cuda")
    c16 = torch.empty(n, dtype=torch.int16, device="cuda")
    cnt = torch.zeros(3, dtype=torch.int64, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    cases = {"e5m2_rne": (0, QCfg(0, 0, 1, 0, 0, 0, None), c8, 5),
             "e5m2_sr_lfsr": (0, QCfg(1, 0, 1, 0, 0, 0, None), c8, 5),
             "fp16_sr_counter": (1, QCfg(1, 1, 1, 0, 0, 0, None), c16, 6),
             "fp16_sr_lfsr": (1, QCfg(1, 0, 1, 0, 0, 0, None), c16, 6),
             "e5m2_sr_counter": (0, QCfg(1, 1, 1, 0, 0, 0, None), c8, 5)}
    if only:
        cases = {k: v for k, v in cases.items() if k in only}
    res = {}
    for rep in range(3):
        for name, (fmt, cfg, out, bpe) in cases.items():
            for li, L in enumerate(libs):
                for _ in range(3):
                    L.fp8b_quantize(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                    ctypes.c_int64(n), fmt, ctypes.byref(cfg),
                                    ctypes.c_void_p(cnt.data_ptr()), st)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                for _ in range(10):
                    L.fp8b_quantize(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                    ctypes.c_int64(n), fmt, ctypes.byref(cfg),
                                    ctypes.c_void_p(cnt.data_ptr()), st)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / 10
                res.setdefault(name, [[] for _ in libs])[li].append(round(n * bpe / ms / 1e6, 1))
    for name, rows in res.items():
        for lib, r in zip(names, rows):
            print(f"{name:18s} {os.path.basename(lib):24s} {r}  (GB/s)")


if __name__ == "__main__":
    main()
