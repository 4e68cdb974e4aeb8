"""CPU tests of the drop-in boundary: the C-ABI library loads and exports every symbol the
header declares, the Python binding covers all of them, and the product refuses to run
without a GPU (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2605_21072_b200 as qb
from paper_2605_21072_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qarvd_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qarvd_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    for must in ("qarvd_quantize_act", "qarvd_dual_gemm", "qarvd_prepare_weights",
                 "qarvd_analyze_layers", "qarvd_scale_search", "qarvd_linear_forward_host"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (qarvd_\w+)", out))
    assert set(declared_symbols()) <= exported


def test_python_binding_covers_abi():
    assert set(declared_symbols()) == set(_lib.SIGNATURES)


def test_abi_version_and_no_device_here():
    lib = _lib.load()
    assert lib.qarvd_abi_version() == 1
    if lib.qarvd_device_count() == 0:
        # a compute entry point must fail loudly, never fall back to the CPU
        with pytest.raises(qb.CudaError, match="no CUDA device"):
            _lib.call("qarvd_synth_bf16", ctypes.c_void_p(16), 1, 8, 8, 1, 1.0, None, 0, 1.0, None)


def test_argument_validation_maps_to_reference_exceptions():
    # shape / parameter errors are std::invalid_argument in the reference (engine.cpp:47-50)
    with pytest.raises(qb.InvalidArgument):
        _lib.call("qarvd_dual_gemm", None, 64, None, 64, 4, 4, 48, 0, None, None, None, None, 0, 0,
                  None, 4, None, None, None)
    with pytest.raises(qb.LogicError):
        _lib.call("qarvd_dual_gemm", ctypes.c_void_p(16), 140000, ctypes.c_void_p(16), 140000, 4, 4,
                  140000 - 140000 % 32, 0, ctypes.c_void_p(16), None, ctypes.c_void_p(16), None, 0,
                  0, ctypes.c_void_p(16), 4, None, None, None)
    with pytest.raises(qb.InvalidArgument, match="scale must be positive"):
        _lib.call("qarvd_quantize_act", ctypes.c_void_p(16), 0, 4, 8, 8, None, 8, 1, -1.0, 8,
                  ctypes.c_void_p(16), 8, None, None, None, None)
    with pytest.raises(qb.Unsupported):
        _lib.call("qarvd_quantize_act", ctypes.c_void_p(16), 0, 4, 8, 8, None, 8, 0, 0.0, 12,
                  ctypes.c_void_p(16), 8, None, None, None, None)


def test_sm100a_code_in_library():
    """The shipped .so carries sm_100a SASS with tcgen05 MMA, TMEM loads and TMA."""
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out or "SM100" in out.upper()
    for mnem in ("UTCIMMA", "LDTM", "UTMALDG"):
        assert mnem in out, mnem
