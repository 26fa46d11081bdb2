"""Interleaved A/B of the fused-E5M2-output GEMM between builds of the library
(one process, one box). Usage: python scripts/gemm_lib_ab.py libA.so libB.so MxNxK[:bk] ..."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12334_b200 as F  # noqa: E402
from paper_1905_12334_b200 import _lib  # noqa: E402


def main():
    names = [a for a in sys.argv[1:] if a.endswith(".so")]
    specs = [a for a in sys.argv[1:] if not a.endswith(".so")]
    libs = [ctypes.CDLL(os.path.abspath(p), mode=ctypes.RTLD_LOCAL) for p in names]
    for L in libs:
        assert L.fp8b_init() == 0
    F.init()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for spec in specs:
        shape, _, bmaj = spec.partition(":")
        m, n, k = (int(v) for v in shape.split("x"))
        x = torch.empty(m * k + k * n, dtype=torch.float32, device="cuda")
        F.fill_synthetic(x, "normal", 3, 1.0)
        qa = F.quantize(x[: m * k]).codes
        qb = F.quantize(x[m * k:]).codes
        cq = torch.empty(m * n, dtype=torch.uint8, device="cuda")
        args = _lib.GemmArgs(_lib.K_MAJOR, _lib.K_MAJOR if bmaj == "bk" else _lib.MN_MAJOR,
                             _lib.GEMM_TENSOR, 0, None, None, cq.data_ptr(), 0, 0, 1, 0, 0, None)

        def call(L):
            rc = L.fp8b_gemm(ctypes.c_void_p(qa.data_ptr()), ctypes.c_void_p(qb.data_ptr()),
                             ctypes.c_int64(m), ctypes.c_int64(n), ctypes.c_int64(k), 0,
                             ctypes.byref(args), st)
            assert rc == 0, rc

        res = [[] for _ in libs]
        for rep in range(4):
            for li, L in enumerate(libs):
                for _ in range(3):
                    call(L)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                for _ in range(10):
                    call(L)
                e1.record()
                torch.cuda.synchronize()
                res[li].append(round(e0.elapsed_time(e1) * 100, 1))
        for nme, r in zip(names, res):
            print(f"{spec:26s} {os.path.basename(nme):20s} {r} us")


if __name__ == "__main__":
    main()
