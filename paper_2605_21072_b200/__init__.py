"""paper_2605_21072_b200 — B200-native Q-ARVD quantized-inference + calibration hot path.

The compute lives in ``libqarvd_b200.so`` (hand-written sm_100a CUDA behind the
C-ABI of ``include/qarvd_b200.h``); this package is the host-side mirror of the
reference operator API (``/root/reference/proj/core``) over that ABI, using
torch only for device memory, streams and ``torch.distributed``.
"""
from . import _lib
from ._lib import (BF16, F32, F64, ACT_PER_TOKEN, ACT_PER_TENSOR, EPI_NONE, EPI_GELU,
                   QarvdError, InvalidArgument, OutOfRange, LogicError, CudaError, Unsupported)
from .engine import (DualScalePlan, QuantizedLayer, LinearHandle, build_plan, prepare_weights,
                     kernel_a_quantize_activation, kernel_b_gemm_dequant, quantized_layer_forward)
from .outlier import OutlierReport, analyze_layer, analyze_layers
from .calibrate import (PERCENTILES, weighting_strategy, normalize_alpha, init_scale_percentile_search,
                        scale_search_async, lpt_assign, LayerRecord, allgather_records)

__all__ = [n for n in dir() if not n.startswith("_")]
