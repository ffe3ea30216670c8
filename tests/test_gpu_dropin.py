"""The C++ drop-in: tests/cpp/dropin_parity.cpp drives colosim_gpu.hpp with
the reference's own ModelProfile/GpuProfile/Grid objects and compares against
the unchanged reference headers (maps, 2M composed verdicts per map set,
serving replays sample for sample).  Built here by `make dropin`."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "dropin_parity")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="build/dropin_parity not built (needs /root/reference at build time)")
def test_cpp_dropin_parity():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "PASS" in r.stdout
