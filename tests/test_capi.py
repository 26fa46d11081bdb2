"""CPU: the C-ABI library loads, exports every symbol include/fp8b200.h declares,
its ctypes struct mirrors match the C layout, and its host-side validation
rejects what the reference rejects (these calls fail before any CUDA work)."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(ROOT, "include", "fp8b200.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fp8b_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1905_12334_b200 import _lib
    names = _declared()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(_lib.LIB, n)]
    assert not missing, missing
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_1905_12334_b200", "libfp8b200.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_c():
    from paper_1905_12334_b200 import _lib
    prog = r"""
#include <stdio.h>
#include <stddef.h>
#include "fp8b200.h"
int main(void) {
  printf("%zu %zu %zu %zu\n", sizeof(fp8b_quant_config_t), sizeof(fp8b_gemm_args_t),
         sizeof(fp8b_loss_scaler_t), sizeof(fp8b_sgd_args_t));
  printf("%zu %zu %zu\n", offsetof(fp8b_quant_config_t, rbits),
         offsetof(fp8b_gemm_args_t, cq_counters), offsetof(fp8b_loss_scaler_t, last_scale_after));
  printf("%zu %zu\n", offsetof(fp8b_sgd_args_t, seed), offsetof(fp8b_sgd_args_t, w_counters));
  return 0;
}
"""
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "t.c")
        exe = os.path.join(d, "t")
        open(src, "w").write(prog)
        subprocess.run(["gcc", "-std=c11", "-I", os.path.dirname(HEADER), src, "-o", exe], check=True)
        vals = [int(v) for v in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    want = [C.sizeof(_lib.QuantConfig), C.sizeof(_lib.GemmArgs), C.sizeof(_lib.LossScalerState),
            C.sizeof(_lib.SgdArgs), _lib.QuantConfig.rbits.offset, _lib.GemmArgs.cq_counters.offset,
            _lib.LossScalerState.last_scale_after.offset, _lib.SgdArgs.seed.offset,
            _lib.SgdArgs.w_counters.offset]
    assert vals == want


def test_validation_matches_reference_errors():
    """std::invalid_argument cases of the reference map to FP8B_EINVAL, checked
    on the host before any device work."""
    from paper_1905_12334_b200 import _lib
    L = _lib.LIB
    cfg = _lib.QuantConfig(_lib.SR, _lib.BITS_LFSR, 0, 0, 0, 0, None)
    assert L.fp8b_quantize(None, None, 4, _lib.E5M2, cfg, None, None) == _lib.EINVAL  # tensor.cpp:48
    assert b"seed" in L.fp8b_last_error()
    cfg = _lib.QuantConfig(_lib.RNE, 0, 0, 0, 0, 0, None)
    assert L.fp8b_quantize(None, None, 4, _lib.E5M2, cfg, None, None) == _lib.EINVAL
    cfg = _lib.QuantConfig(7, 0, 1, 0, 0, 0, None)
    assert L.fp8b_quantize(None, None, 4, _lib.E5M2, cfg, None, None) == _lib.EINVAL
    cfg = _lib.QuantConfig(_lib.RNE, 0, 1, 0, 0, 0, None)
    assert L.fp8b_quantize(None, None, 4, 9, cfg, None, None) == _lib.EINVAL
    assert L.fp8b_quantize(None, None, -1, _lib.E5M2, cfg, None, None) == _lib.EINVAL
    cfg = _lib.QuantConfig(_lib.SR, _lib.BITS_SUPPLIED, 1, 0, 0, 0, None)
    assert L.fp8b_quantize(None, None, 4, _lib.E5M2, cfg, None, None) == _lib.EINVAL
    # zero-size calls are no-ops
    cfg = _lib.QuantConfig(_lib.RNE, 0, 1, 0, 0, 0, None)
    assert L.fp8b_quantize(None, None, 0, _lib.E5M2, cfg, None, None) == _lib.OK
    # gemm: format and output checks (kernels.cpp:9-13, 38-44)
    ga = _lib.GemmArgs()
    assert L.fp8b_gemm(None, None, 2, 2, 2, 5, ga, None) == _lib.EINVAL
    assert L.fp8b_gemm(None, None, -2, 2, 2, _lib.E5M2, ga, None) == _lib.EINVAL
    assert L.fp8b_gemm(None, None, 2, 2, 2, _lib.E5M2, ga, None) == _lib.EINVAL  # no output
    # sgd: master SR with zero seed
    sa = _lib.SgdArgs(0.1, 0.9, 0.0, 1.0, None, None, _lib.SR, _lib.BITS_LFSR, 0, 0, None, None,
                      None, 0, 0, None)
    assert L.fp8b_sgd_momentum_update(None, _lib.E5M2, None, None, 4, sa, None) == _lib.EINVAL


@pytest.mark.parametrize("bad", [
    dict(scale=0.0), dict(scale=float("inf")), dict(backoff_factor=1.0), dict(backoff_factor=0.0),
    dict(growth_factor=1.0), dict(growth_interval=0),
    dict(schedule=[(40, 8192.0), (40, 16384.0)]), dict(schedule=[(40, -1.0)]),
])
def test_loss_scaler_option_validation(bad):
    """loss_scaling.cpp:19-38 (pinned by test_loss_scaling.cpp:128-154)."""
    from paper_1905_12334_b200 import _lib
    h = _lib.LossScalerState()
    h.kind = _lib.SCALER_DYNAMIC_BACKOFF
    h.scale = bad.get("scale", 1024.0)
    h.backoff_factor = bad.get("backoff_factor", 0.5)
    h.growth_factor = bad.get("growth_factor", 2.0)
    h.growth_interval = bad.get("growth_interval", 2000)
    sched = bad.get("schedule", [(40, 8192.0), (150, 32768.0)])
    h.n_schedule = len(sched)
    for i, (it, sc) in enumerate(sched):
        h.sched_iter[i], h.sched_scale[i] = it, sc
    dummy = C.create_string_buffer(C.sizeof(h))
    assert _lib.LIB.fp8b_loss_scaler_init(C.addressof(dummy), h, None) == _lib.EINVAL


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1905_12334_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert "import oracle" not in txt and "liboracle" not in txt, fn
                assert "fp8emu_ref" not in txt, fn
