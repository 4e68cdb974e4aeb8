"""Host-side mirror of the reference outlier detector (outlier.hpp).

``analyze_layers`` batches ``analyze_layer(name, W, tau, alpha_min, align)``
(outlier.hpp:59-61, outlier.cpp:98-102) over many layers in two kernel
launches (column norms, then per-layer median/MAD/threshold/alignment).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, List, Sequence

import numpy as np
import torch

from . import _lib
from .engine import _dtype_code, _stream

K_MODIFIED_Z_SCORE_FACTOR = 0.6745  # outlier.hpp:13
K_DEFAULT_TAU = 3.5                 # outlier.hpp:14
K_DEFAULT_ALPHA_MIN = 1.2           # outlier.hpp:15
K_DEFAULT_ALIGN = 32                # outlier.hpp:16


@dataclass
class OutlierReport:
    """outlier.hpp:42-55 (norms kept on the device; indices on the host)."""

    layer_name: str
    norms: torch.Tensor
    median: float
    mad: float
    threshold: float
    tau: float
    alpha_min: float
    align: int
    raw_outliers: np.ndarray
    aligned_outliers: np.ndarray

    def has_outliers(self) -> bool:
        return self.raw_outliers.size > 0


class DeviceReports:
    """Raw device outputs of one batched launch (no host synchronisation)."""

    def __init__(self, names, ks, device):
        self.names = list(names)
        self.ks = list(ks)
        total = int(sum(ks))
        L = len(ks)
        self.norms = torch.empty(total, dtype=torch.float64, device=device)
        self.stats = torch.empty((L, 3), dtype=torch.float64, device=device)
        self.counts = torch.empty((L, 2), dtype=torch.int32, device=device)
        self.raw = torch.empty(total, dtype=torch.int32, device=device)
        self.aligned = torch.empty(total, dtype=torch.int32, device=device)
        self.offsets = np.concatenate([[0], np.cumsum(ks)]).astype(np.int64)


def analyze_layers_async(names: Sequence[str], weights: Sequence[torch.Tensor],
                         tau: float = K_DEFAULT_TAU, alpha_min: float = K_DEFAULT_ALPHA_MIN,
                         align: int = K_DEFAULT_ALIGN, out: Optional[DeviceReports] = None) -> DeviceReports:
    """K3 over a batch of layers into device buffers (no host sync).  ``out`` reuses the buffers
    (and the launch table) of an earlier call with the same layers."""
    if out is not None and getattr(out, "_jobs", None) is not None:
        _lib.call("qarvd_analyze_layers", out._jobs, len(weights), _dtype_code(weights[0]), float(tau),
                  float(alpha_min), int(align), _stream())
        out.tau, out.alpha_min, out.align = tau, alpha_min, align
        return out
    if len(weights) == 0:
        raise _lib.InvalidArgument("analyze_layers: no layers")
    dt = {w.dtype for w in weights}
    if len(dt) != 1:
        raise _lib.InvalidArgument("analyze_layers: all weights of one batch need one dtype")
    dev = weights[0].device
    out = DeviceReports(names, [w.shape[1] for w in weights], dev)
    jobs = (_lib.OutlierJob * len(weights))()
    for i, w in enumerate(weights):
        o = int(out.offsets[i])
        jobs[i].w = w.data_ptr()
        jobs[i].n = w.shape[0]
        jobs[i].k = w.shape[1]
        jobs[i].ldw = w.stride(0)
        jobs[i].norms = out.norms.data_ptr() + 8 * o
        jobs[i].stats = out.stats.data_ptr() + 24 * i
        jobs[i].counts = out.counts.data_ptr() + 8 * i
        jobs[i].raw_idx = out.raw.data_ptr() + 4 * o
        jobs[i].aligned_idx = out.aligned.data_ptr() + 4 * o
    _lib.call("qarvd_analyze_layers", jobs, len(weights), _dtype_code(weights[0]), float(tau),
              float(alpha_min), int(align), _stream())
    out.tau, out.alpha_min, out.align = tau, alpha_min, align
    out._jobs = jobs
    return out


def collect_reports(d: DeviceReports) -> List[OutlierReport]:
    stats = d.stats.cpu().numpy()
    counts = d.counts.cpu().numpy()
    raw = d.raw.cpu().numpy()
    aligned = d.aligned.cpu().numpy()
    reps = []
    for i, name in enumerate(d.names):
        o, e = int(d.offsets[i]), int(d.offsets[i + 1])
        reps.append(OutlierReport(
            name, d.norms[o:e], float(stats[i, 0]), float(stats[i, 1]), float(stats[i, 2]),
            d.tau, d.alpha_min, d.align, raw[o:o + counts[i, 0]].astype(np.int64),
            aligned[o:o + counts[i, 1]].astype(np.int64)))
    return reps


def analyze_layers(names: Sequence[str], weights: Sequence[torch.Tensor],
                   tau: float = K_DEFAULT_TAU, alpha_min: float = K_DEFAULT_ALPHA_MIN,
                   align: int = K_DEFAULT_ALIGN) -> List[OutlierReport]:
    return collect_reports(analyze_layers_async(names, weights, tau, alpha_min, align))


def analyze_layer(name: str, w: torch.Tensor, tau: float = K_DEFAULT_TAU,
                  alpha_min: float = K_DEFAULT_ALPHA_MIN,
                  align: int = K_DEFAULT_ALIGN) -> OutlierReport:
    """analyze_layer (outlier.hpp:59-61)."""
    return analyze_layers([name], [w], tau, alpha_min, align)[0]
