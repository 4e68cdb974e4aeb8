"""Runs the C++ drop-in tests (tests/cpp/):
  test_dropin          the reference's calibrated toy model and every qarvd::cuda operator vs the
                       reference on identical inputs (bit-identical unless a stated tolerance)
  test_no_ref_compute  the adapter's whole pipeline linked against poisoned copies of the
                       reference's compute functions (any call aborts): no CPU fallback inside."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BUILD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "build")


def _run(name, marker):
    path = os.path.join(BUILD, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not built (needs the reference headers at build time)")
    out = subprocess.run([path], capture_output=True, text=True, timeout=900)
    print(out.stdout[-6000:])
    assert out.returncode == 0, out.stdout[-6000:] + out.stderr[-2000:]
    assert marker in out.stdout


def test_dropin_binary(cuda):
    _run("test_dropin", "DROPIN PASS")


def test_no_reference_compute_in_adapter(cuda):
    _run("test_no_ref_compute", "NO_REF_COMPUTE PASS")
