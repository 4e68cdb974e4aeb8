"""ctypes binding of libqarvd_b200.so (the C-ABI declared in include/qarvd_b200.h).

The library is built in-tree (paper_2605_21072_b200/libqarvd_b200.so) by
``__graft_entry__.build()``.  There is no fallback: importing a compute entry
point without the library, or calling it without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int, c_int64, c_uint64, c_void_p, c_char_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QARVD_B200_LIB") or os.path.join(_HERE, "libqarvd_b200.so")  # override: A/B builds

# status codes (qarvd_b200.h)
OK = 0
ERR_INVALID_ARGUMENT = 1
ERR_OUT_OF_RANGE = 2
ERR_LOGIC = 3
ERR_RUNTIME = 4
ERR_CUDA = 5
ERR_UNSUPPORTED = 6

BF16, F32, F64 = 0, 1, 2
ACT_PER_TOKEN, ACT_PER_TENSOR = 0, 1
EPI_NONE, EPI_GELU = 0, 1
MAX_CANDIDATES = 16
MAX_FRAMES = 64


class QarvdError(RuntimeError):
    """Base class; subclasses mirror the reference's C++ exception types."""


class InvalidArgument(QarvdError, ValueError):
    """std::invalid_argument (quant.cpp:59-80, engine.cpp:47-50)."""


class OutOfRange(QarvdError, IndexError):
    """std::out_of_range (engine.cpp:29, dual_scale.cpp:63-64)."""


class LogicError(QarvdError):
    """std::logic_error (engine.cpp:54-55)."""


class CudaError(QarvdError):
    """CUDA / driver failure or no device (no CPU fallback exists)."""


class Unsupported(QarvdError, NotImplementedError):
    """Valid for the reference but outside this build's envelope."""


_EXC = {
    ERR_INVALID_ARGUMENT: InvalidArgument,
    ERR_OUT_OF_RANGE: OutOfRange,
    ERR_LOGIC: LogicError,
    ERR_RUNTIME: QarvdError,
    ERR_CUDA: CudaError,
    ERR_UNSUPPORTED: Unsupported,
}


class OutlierJob(ctypes.Structure):
    _fields_ = [
        ("w", c_void_p),
        ("n", c_int64),
        ("k", c_int64),
        ("ldw", c_int64),
        ("norms", c_void_p),
        ("stats", c_void_p),
        ("counts", c_void_p),
        ("raw_idx", c_void_p),
        ("aligned_idx", c_void_p),
    ]


class SynthDesc(ctypes.Structure):
    _fields_ = [("seed", c_uint64), ("stddev", c_double), ("outlier_cols", c_void_p),
                ("num_outliers", c_int64), ("gamma", c_double)]


class CalibLayer(ctypes.Structure):
    _fields_ = [("index", c_int64), ("n", c_int64), ("k", c_int64), ("rows", c_int64),
                ("w_host", c_void_p), ("w_synth", SynthDesc), ("x_host", c_void_p),
                ("x_synth", POINTER(SynthDesc))]


class SearchJob(ctypes.Structure):
    _fields_ = [
        ("x", c_void_p),
        ("frames", c_int64),
        ("rows", c_int64),
        ("k", c_int64),
        ("ldx", c_int64),
        ("result", c_void_p),
    ]


class CalibConfig(ctypes.Structure):
    """qarvd_calib_config = CalibConfig (calibrate.hpp:16-33); defaults are the reference's."""
    _fields_ = [
        ("iterations", c_int),
        ("batch_size", c_int),
        ("lr_round", c_double),
        ("lr_scale", c_double),
        ("seed", c_uint64),
        ("train_activation_scale", c_int),
        ("zeta", c_double),
        ("gamma_lo", c_double),
        ("reg_lambda", c_double),
        ("beta_start", c_double),
        ("beta_end", c_double),
        ("warmup_frac", c_double),
    ]

    def __init__(self, **kw):
        d = dict(iterations=200, batch_size=4, lr_round=2e-3, lr_scale=4e-5, seed=0,
                 train_activation_scale=1, zeta=1.1, gamma_lo=-0.1, reg_lambda=1e-2,
                 beta_start=10.0, beta_end=2.0, warmup_frac=0.2)
        d.update(kw)
        super().__init__(**d)


class PlannedWeightJob(ctypes.Structure):
    """qarvd_planned_weight_job (include/qarvd_b200.h)."""
    _fields_ = [
        ("w", c_void_p), ("n", c_int64), ("k", c_int64), ("ldw", c_int64),
        ("aligned_idx", c_void_p), ("counts", c_void_p), ("gather", c_void_p), ("gather_cap", c_int64),
        ("plan_info", c_void_p), ("wq", c_void_p), ("ldq", c_int64),
        ("scale_outlier_f64", c_void_p), ("scale_normal_f64", c_void_p),
        ("scale_outlier_f32", c_void_p), ("scale_normal_f32", c_void_p),
    ]


class WeightJob(ctypes.Structure):
    _fields_ = [
        ("w", c_void_p),
        ("n", c_int64),
        ("k", c_int64),
        ("ldw", c_int64),
        ("gather", c_void_p),
        ("k_pad", c_int64),
        ("k_outlier", c_int64),
        ("wq", c_void_p),
        ("ldq", c_int64),
        ("scale_outlier_f64", c_void_p),
        ("scale_normal_f64", c_void_p),
        ("scale_outlier_f32", c_void_p),
        ("scale_normal_f32", c_void_p),
    ]


# (name, restype, argtypes) for every symbol in include/qarvd_b200.h
SIGNATURES = {
    "qarvd_abi_version": (c_int, []),
    "qarvd_last_error": (c_char_p, []),
    "qarvd_device_count": (c_int, []),
    "qarvd_launch_count": (c_uint64, []),
    "qarvd_quantize_act": (
        c_int,
        [c_void_p, c_int, c_int64, c_int64, c_int64, c_void_p, c_int64, c_int, c_double, c_int,
         c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p],
    ),
    "qarvd_prepare_weights": (
        c_int,
        [c_void_p, c_int, c_int64, c_int64, c_int64, c_void_p, c_int64, c_int64, c_int, c_void_p,
         c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    ),
    "qarvd_scale_search_async": (c_int, [c_void_p, c_int, c_void_p, c_int, c_void_p, c_int, c_void_p, c_void_p]),
    "qarvd_prepare_weights_batched": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p]),
    "qarvd_dual_gemm": (
        c_int,
        [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64, c_void_p,
         c_void_p, c_void_p, c_void_p, c_int, c_int, c_void_p, c_int64, c_void_p, c_void_p,
         c_void_p],
    ),
    "qarvd_dual_gemm_rowmax": (
        c_int,
        [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64, c_void_p,
         c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_int64, c_void_p, c_void_p],
    ),
    "qarvd_quantize_act_rowmax": (
        c_int,
        [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int, c_double, c_int, c_void_p, c_int64,
         c_void_p, c_void_p, c_void_p, c_void_p],
    ),
    "qarvd_dual_gemm_pmax_count": (c_int64, [c_int64, c_int64, c_int64]),
    "qarvd_dual_gemm_pmax": (
        c_int,
        [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64, c_void_p,
         c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_int64, c_void_p, c_int64, c_void_p],
    ),
    "qarvd_quantize_act_pmax": (
        c_int,
        [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_int, c_double, c_int, c_void_p,
         c_int64, c_void_p, c_void_p, c_void_p, c_void_p],
    ),
    "qarvd_dual_gemm_f64": (
        c_int,
        [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64, c_void_p,
         c_void_p, c_void_p, c_void_p, c_int64, c_void_p],
    ),
    "qarvd_dual_gemm_f64_slices": (
        c_int,
        [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64, c_void_p,
         c_void_p, c_void_p, c_int, c_void_p, c_int64, c_void_p],
    ),
    "qarvd_linear_create": (
        c_int,
        [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_void_p,
         c_int, c_double, c_int, POINTER(c_void_p)],
    ),
    "qarvd_linear_destroy": (c_int, [c_void_p]),
    "qarvd_linear_forward": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "qarvd_linear_forward_host": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "qarvd_linear_chain_forward_host": (
        c_int, [POINTER(c_void_p), c_int, c_void_p, c_int64, c_void_p, c_void_p]),
    "qarvd_analyze_layers": (
        c_int, [POINTER(OutlierJob), c_int, c_int, c_double, c_double, c_int64, c_void_p]),
    "qarvd_scale_search": (
        c_int,
        [POINTER(SearchJob), c_int, POINTER(c_double), c_int, POINTER(c_double), c_int, c_void_p],
    ),
    "qarvd_weighted_loss_workspace": (c_int64, [c_int64, c_int64, c_int64]),
    "qarvd_prepare_weights_planned": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p]),
    "qarvd_calibrate_layer": (
        c_int, [c_void_p, c_int64, c_int64, c_void_p, c_int, c_void_p, c_void_p, c_double, c_int, c_int,
                c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_char_p, c_void_p,
                c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "qarvd_dual_gemm_quant_workspace_size": (c_int64, [c_int64]),
    "qarvd_dual_gemm_quant": (
        c_int, [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64, c_void_p,
                c_void_p, c_void_p, c_void_p, c_int, c_int, c_double, c_int, c_void_p, c_int64, c_void_p,
                c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
    "qarvd_dual_gemm_workspace_size": (c_int64, [c_int64, c_int64, c_int64, c_int64]),
    "qarvd_dual_gemm_ws": (
        c_int, [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64, c_void_p,
                c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_int64, c_void_p, c_int64, c_void_p]),
    "qarvd_weighted_loss": (
        c_int, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64,
                c_int64, c_int64, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
    "qarvd_quantize_f64": (
        c_int, [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p, ctypes.c_int32, ctypes.c_int32,
                c_void_p, c_void_p, c_void_p, c_void_p]),
    "qarvd_minmax_scale_f64": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_int, c_void_p, c_void_p]),
    "qarvd_percentile_search_f64": (
        c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p]),
    "qarvd_matmul_nt_f64": (
        c_int, [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p]),
    "qarvd_gather_columns": (
        c_int, [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int, c_void_p]),
    "qarvd_dequant_weight_f64": (
        c_int, [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "qarvd_sq_distance_acc_f64": (c_int, [c_void_p, c_void_p, c_int64, c_double, c_void_p, c_int, c_double, c_void_p]),
    "qarvd_zero_point_correct_f64": (
        c_int, [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_int64, c_int64, c_int, ctypes.c_int32,
                c_double, c_void_p, c_void_p, c_void_p]),
    "qarvd_unpack_codes_i4": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_void_p]),
    "qarvd_pack_codes_i8": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_void_p]),
    "qarvd_exp_f64": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "qarvd_adaround_weights": (
        c_int, [c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_int64, c_int64, c_double, c_double, c_int, c_int,
                c_void_p, c_void_p, c_void_p]),
    "qarvd_calib_record_doubles": (c_int64, [c_int64, c_int64, c_int]),
    "qarvd_calibrate_sharded": (
        c_int, [POINTER(CalibLayer), c_int, c_int, c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p, c_int64,
                c_void_p, POINTER(c_double), POINTER(c_int)]),
    "qarvd_probe_int8_peak": (c_int, [c_int, POINTER(c_double), POINTER(c_double), c_void_p]),
    "qarvd_synth_bf16": (
        c_int,
        [c_void_p, c_int64, c_int64, c_int64, c_uint64, c_double, c_void_p, c_int64, c_double,
         c_void_p],
    ),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load the in-tree library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CudaError(
                f"{LIB_PATH} is missing: run __graft_entry__.build() (there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(status: int) -> None:
    if status != OK:
        msg = load().qarvd_last_error().decode(errors="replace")
        raise _EXC.get(status, QarvdError)(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def launch_count() -> int:
    return int(load().qarvd_launch_count())


def probe_int8_peak(iters: int = 20000, stream=None):
    """Dense INT8 tensor-pipe peak measured live (qarvd_probe_int8_peak): (TOPS, ms)."""
    tops, ms = c_double(), c_double()
    call("qarvd_probe_int8_peak", iters, ctypes.byref(tops), ctypes.byref(ms), stream)
    return tops.value, ms.value
