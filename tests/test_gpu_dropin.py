"""Runs the C++ drop-in test (tests/cpp/test_dropin.cpp): the reference's calibrated toy
model served by qarvd::cuda::CudaQuantizedProvider through the reference's run_rollout."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "build", "test_dropin")


def test_dropin_binary(cuda):
    if not os.path.exists(BIN):
        pytest.skip("drop-in binary not built (needs the reference headers at build time)")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(out.stdout[-4000:])
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
    assert "DROPIN PASS" in out.stdout
