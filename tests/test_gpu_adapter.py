"""The drop-in check in C++: the reference's own API (compiled from its sources) side by side with
adapter/aggkin_gpu.hpp over the C ABI (tests/cpp/adapter_parity.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build", "adapter_parity")


def test_adapter_parity(agk):
    if not os.path.exists(BIN):
        pytest.skip("build/adapter_parity not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
