"""GPU: the reference-side C++ drop-in (integration/fp8emu_b200.{hpp,cpp}),
linked beside the UNMODIFIED reference library, returns what the reference
returns through the reference's own types (oracle/_ref/adapter_check, built
by `make -C oracle adapter` in the build container)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
EXE = os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref", "adapter_check")


@pytest.mark.skipif(not os.path.exists(EXE), reason="adapter_check not built (needs /root/reference)")
def test_cpp_dropin_matches_reference():
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.count("PASS") == 7 and "FAIL" not in out.stdout
