"""Host-side mirror of the reference's quantized-linear operator API.

Reference interface (``/root/reference/proj/core/include/qarvd/engine.hpp``):

* ``kernel_a_quantize_activation(x, p)``   engine.hpp:43  -> :func:`kernel_a_quantize_activation`
* ``kernel_b_gemm_dequant(xq, layer)``      engine.hpp:48  -> :func:`kernel_b_gemm_dequant`
* ``permute_activations(x, plan)``          engine.hpp:51  -> folded into K1 via ``plan.gather``
* ``quantized_layer_forward(layer, x, e)``  engine.hpp:60  -> :func:`quantized_layer_forward`
* ``QuantizedLayer``                        engine.hpp:18-30 -> :class:`QuantizedLayer`
* ``DualScalePlan`` / ``build_plan``         dual_scale.hpp:18-41 -> :class:`DualScalePlan`, :func:`build_plan`

Tensors are device-resident torch tensors (torch is the allocator / stream
provider only); every computation runs in libqarvd_b200.so through the C-ABI.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _lib

QMAX8 = 127


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return _lib.BF16
    if t.dtype == torch.float32:
        return _lib.F32
    if t.dtype == torch.float64:
        return _lib.F64
    raise _lib.InvalidArgument(f"unsupported input dtype {t.dtype}")


def _round_up(v: int, m: int) -> int:
    return (v + m - 1) // m * m


@dataclass
class DualScalePlan:
    """Split of a layer's input channels (dual_scale.hpp:18-31).

    ``permutation`` is [sorted outliers | sorted normals] over original column
    ids (dual_scale.cpp:81-83).  ``gather`` is the padded device layout the
    kernels consume: [outliers, -1 pad to a multiple of 32, normals, -1 pad to a
    multiple of 32]; ``k_outlier`` is the padded outlier-slab width and
    ``k_pad`` the padded K.  Zero-code pad columns leave every dot product
    unchanged, so unaligned outlier sets (outlier.cpp:59, :63-66) stay exact.
    """

    layer_name: str
    enabled: bool
    d_in: int
    outlier_indices: np.ndarray
    normal_indices: np.ndarray
    permutation: np.ndarray
    gather: np.ndarray = field(repr=False, default=None)
    k_outlier: int = 0
    k_pad: int = 0

    def outlier_count(self) -> int:
        return int(len(self.outlier_indices))

    def inverse_permutation(self) -> np.ndarray:
        inv = np.empty_like(self.permutation)
        inv[self.permutation] = np.arange(len(self.permutation), dtype=self.permutation.dtype)
        return inv


def build_plan(layer_name: str, d_in: int, aligned_outliers: Sequence[int]) -> DualScalePlan:
    """Column split of build_plan / build_single_scale_plan (dual_scale.cpp:44-90).

    The per-row group scales are computed on the device by
    :func:`prepare_weights` (row_scales_over_columns, dual_scale.cpp:13-24).
    """
    outl = np.asarray(sorted(int(i) for i in aligned_outliers), dtype=np.int64)
    if outl.size and (outl.min() < 0 or outl.max() >= d_in):
        raise _lib.OutOfRange("build_plan: outlier index out of range")
    if outl.size == 0:
        perm = np.arange(d_in, dtype=np.uint32)
        k_pad = _round_up(d_in, 32)
        gather = np.full(k_pad, -1, dtype=np.int32)
        gather[:d_in] = np.arange(d_in, dtype=np.int32)
        return DualScalePlan(layer_name, False, d_in, outl, np.arange(d_in, dtype=np.int64),
                             perm, gather, 0, k_pad)
    mask = np.zeros(d_in, dtype=bool)
    mask[outl] = True
    normals = np.nonzero(~mask)[0].astype(np.int64)
    if normals.size == 0:
        raise _lib.InvalidArgument("build_plan: outlier set would leave no normal channels")
    perm = np.concatenate([outl, normals]).astype(np.uint32)
    k_o = _round_up(outl.size, 32)
    k_pad = k_o + _round_up(normals.size, 32)
    gather = np.full(k_pad, -1, dtype=np.int32)
    gather[: outl.size] = outl
    gather[k_o: k_o + normals.size] = normals
    return DualScalePlan(layer_name, True, d_in, outl, normals, perm, gather, k_o, k_pad)


@dataclass
class QuantizedLayer:
    """Device-resident deployed layer (engine.hpp:18-30).

    ``wq`` holds the pre-permuted int8 codes [out_dim x k_pad]; group scales are
    kept in f64 (the reference's in-memory precision) and f32 (the QARQ on-disk
    precision, engine.cpp:225-233, which the GEMM epilogue uses).
    """

    name: str
    out_dim: int
    in_dim: int
    plan: DualScalePlan
    wq: torch.Tensor
    scale_outlier64: torch.Tensor
    scale_normal64: torch.Tensor
    scale_outlier32: torch.Tensor
    scale_normal32: torch.Tensor
    gather_dev: Optional[torch.Tensor]  # None: inputs already arrive in plan order (pipeline.fold_output_permutation)
    act_granularity: int = _lib.ACT_PER_TOKEN
    act_scale: float = 0.0
    bias: Optional[torch.Tensor] = None
    # asymmetric static activations (QARQ act_symmetric = false, engine.cpp:288-295): codes
    # clamp(rint(x / s) + z, -2^(b-1), 2^(b-1)-1); the zero-point correction of kernel B
    # (engine.cpp:74-83, :95-100) is folded into ``bias`` by qarq.to_device
    act_zero: int = 0

    @property
    def k_pad(self) -> int:
        return self.plan.k_pad

    @property
    def k_outlier(self) -> int:
        return self.plan.k_outlier


def _check_err(err: torch.Tensor, what: str) -> None:
    v = int(err.item())
    if v != 0x7FFFFFFFFFFFFFFF:
        raise _lib.InvalidArgument(f"{what}: non-finite input at flat index {v}")


def prepare_weights(name: str, w: torch.Tensor, plan: DualScalePlan, bits: int = 8,
                    check_finite: bool = True) -> QuantizedLayer:
    """K5: group scales + nearest codes, pre-permuted (dual_scale.cpp:13-114, calibrate.cpp:474-480)."""
    n, k = w.shape
    if k != plan.d_in:
        raise _lib.InvalidArgument("build_plan: report does not match the weight's input width")
    dev = w.device
    gather = torch.from_numpy(plan.gather).to(dev)
    wq = torch.empty((n, plan.k_pad), dtype=torch.int8, device=dev)
    so64 = torch.empty(n, dtype=torch.float64, device=dev)
    sn64 = torch.empty(n, dtype=torch.float64, device=dev)
    so32 = torch.empty(n, dtype=torch.float32, device=dev)
    sn32 = torch.empty(n, dtype=torch.float32, device=dev)
    err = torch.empty(1, dtype=torch.int64, device=dev) if check_finite else None
    _lib.call("qarvd_prepare_weights", w.data_ptr(), _dtype_code(w), n, k, w.stride(0),
              gather.data_ptr(), plan.k_pad, plan.k_outlier, bits, wq.data_ptr(), plan.k_pad,
              so64.data_ptr(), sn64.data_ptr(), so32.data_ptr(), sn32.data_ptr(), _ptr(err),
              _stream())
    if err is not None:
        v = int(err.item())
        if v != 0x7FFFFFFFFFFFFFFF:
            raise _lib.InvalidArgument("fake_quant_dual: non-finite weight element")
    return QuantizedLayer(name, n, k, plan, wq, so64, sn64, so32, sn32, gather)


def prepare_weights_batched(names: Sequence[str], ws: Sequence[torch.Tensor],
                            plans: Sequence[DualScalePlan], bits: int = 8,
                            check_finite: bool = True) -> List[QuantizedLayer]:
    """K5 for many layers in one launch (qarvd_prepare_weights_batched): the plans' gathers go
    to the device in one copy, codes and scales land in one buffer per field (per-layer views).
    Same results as prepare_weights per layer."""
    if not ws:
        return []
    dev = ws[0].device
    dtype = _dtype_code(ws[0])
    for w, plan in zip(ws, plans):
        if w.shape[1] != plan.d_in:
            raise _lib.InvalidArgument("build_plan: report does not match the weight's input width")
        if _dtype_code(w) != dtype:
            raise _lib.InvalidArgument("prepare_weights_batched: weights of one batch share a dtype")
    # gathers: one host concatenation, one H2D (16-byte aligned slices)
    offs, tot = [], 0
    for plan in plans:
        offs.append(tot)
        tot += (plan.k_pad + 3) // 4 * 4
    g_host = np.full(tot, -1, dtype=np.int32)
    for o, plan in zip(offs, plans):
        g_host[o:o + plan.k_pad] = plan.gather
    g_dev = torch.from_numpy(g_host).to(dev)
    # outputs: one buffer per field
    wq_offs, wq_tot, n_offs, n_tot = [], 0, [], 0
    for w, plan in zip(ws, plans):
        wq_offs.append(wq_tot)
        wq_tot += (w.shape[0] * plan.k_pad + 15) // 16 * 16
        n_offs.append(n_tot)
        n_tot += w.shape[0]
    wq_all = torch.empty(wq_tot, dtype=torch.int8, device=dev)
    so64 = torch.empty(n_tot, dtype=torch.float64, device=dev)
    sn64 = torch.empty(n_tot, dtype=torch.float64, device=dev)
    so32 = torch.empty(n_tot, dtype=torch.float32, device=dev)
    sn32 = torch.empty(n_tot, dtype=torch.float32, device=dev)
    jobs = (_lib.WeightJob * len(ws))()
    layers = []
    for i, (name, w, plan) in enumerate(zip(names, ws, plans)):
        n, k = w.shape
        wq = wq_all[wq_offs[i]:wq_offs[i] + n * plan.k_pad].view(n, plan.k_pad)
        sl = slice(n_offs[i], n_offs[i] + n)
        gather = g_dev[offs[i]:offs[i] + plan.k_pad]
        j = jobs[i]
        j.w, j.n, j.k, j.ldw = w.data_ptr(), n, k, w.stride(0)
        j.gather, j.k_pad, j.k_outlier = gather.data_ptr(), plan.k_pad, plan.k_outlier
        j.wq, j.ldq = wq.data_ptr(), plan.k_pad
        j.scale_outlier_f64, j.scale_normal_f64 = so64[sl].data_ptr(), sn64[sl].data_ptr()
        j.scale_outlier_f32, j.scale_normal_f32 = so32[sl].data_ptr(), sn32[sl].data_ptr()
        layers.append(QuantizedLayer(name, n, k, plan, wq, so64[sl], sn64[sl], so32[sl], sn32[sl], gather))
    err = torch.empty(1, dtype=torch.int64, device=dev) if check_finite else None
    _lib.call("qarvd_prepare_weights_batched", jobs, len(ws), dtype, bits, _ptr(err), _stream())
    if err is not None:
        v = int(err.item())
        if v != 0x7FFFFFFFFFFFFFFF:
            raise _lib.InvalidArgument("fake_quant_dual: non-finite weight element")
    return layers


def layer_from_codes(name: str, codes: np.ndarray, scale_outlier: Sequence[float],
                     scale_normal: Sequence[float], plan: DualScalePlan, device="cuda") -> QuantizedLayer:
    """Deploy given integer codes (ORIGINAL column order, e.g. LearnableQuantState::hard_codes,
    calibrate.cpp:163-183) with their per-row group scales: the pre-permute of
    calibrate.cpp:474-480 (wq[r, pos] = codes[r, perm[pos]], zero codes in pad slots)."""
    codes = np.asarray(codes)
    n, k = codes.shape
    if k != plan.d_in:
        raise _lib.InvalidArgument("layer_from_codes: codes do not match the plan's input width")
    if codes.min(initial=0) < -127 or codes.max(initial=0) > 127:
        raise _lib.InvalidArgument("layer_from_codes: codes outside the int8 range")
    g = plan.gather
    wq = np.zeros((n, plan.k_pad), dtype=np.int8)
    valid = g >= 0
    wq[:, valid] = codes[:, g[valid]].astype(np.int8)
    so = np.asarray(scale_outlier if plan.enabled else scale_normal, dtype=np.float64)
    sn = np.asarray(scale_normal, dtype=np.float64)
    t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=device)
    return QuantizedLayer(name, n, k, plan, t(wq, torch.int8), t(so, torch.float64), t(sn, torch.float64),
                          t(so.astype(np.float32), torch.float32), t(sn.astype(np.float32), torch.float32),
                          t(g, torch.int32))


def kernel_a_quantize_activation(x: torch.Tensor, layer_or_plan, granularity: int = _lib.ACT_PER_TOKEN,
                                 static_scale: float = 0.0, bits: int = 8,
                                 check_finite: bool = False):
    """K1 = quantize(permute_activations(x, plan), p) (engine.cpp:32-44, quant.cpp:113-138).

    Returns (xq int8 [m x k_pad], scale_f32 [m], scale_f64 [m]).
    """
    plan = layer_or_plan.plan if isinstance(layer_or_plan, QuantizedLayer) else layer_or_plan
    gather_dev = (layer_or_plan.gather_dev if isinstance(layer_or_plan, QuantizedLayer)
                  else torch.from_numpy(plan.gather).to(x.device))
    m, k = x.shape
    d_in = plan.d_in if gather_dev is not None else plan.k_pad  # folded layer: plan-order input
    if k != d_in:
        raise _lib.InvalidArgument("permute_activations: plan does not match activation width")
    xq = torch.empty((m, plan.k_pad), dtype=torch.int8, device=x.device)
    s32 = torch.empty(m, dtype=torch.float32, device=x.device)
    s64 = torch.empty(m, dtype=torch.float64, device=x.device)
    err = torch.empty(1, dtype=torch.int64, device=x.device) if check_finite else None
    zero = layer_or_plan.act_zero if isinstance(layer_or_plan, QuantizedLayer) else 0
    if zero != 0:
        # asymmetric static params: the exact f64 quantizer (quant.cpp:113-138 with z), then the
        # int8 packing through the plan's gather
        if granularity != _lib.ACT_PER_TENSOR:
            raise _lib.InvalidArgument("quant params: a zero point needs per-tensor static activations")
        sc = torch.full((1,), float(static_scale), dtype=torch.float64, device=x.device)
        zp = torch.full((1,), int(zero), dtype=torch.int32, device=x.device)
        codes = torch.empty((m, k), dtype=torch.int32, device=x.device)
        e = torch.empty(1, dtype=torch.int64, device=x.device)
        x64 = x.double().contiguous()
        _lib.call("qarvd_quantize_f64", x64.data_ptr(), m * k, 1, 1, sc.data_ptr(), zp.data_ptr(),
                  -(1 << (bits - 1)), (1 << (bits - 1)) - 1, codes.data_ptr(), None, e.data_ptr(), _stream())
        bad = torch.zeros(1, dtype=torch.int32, device=x.device)
        g = gather_dev if gather_dev is not None else torch.arange(plan.k_pad, dtype=torch.int32, device=x.device)
        _lib.call("qarvd_pack_codes_i8", codes.data_ptr(), m, k, g.data_ptr(), plan.k_pad, xq.data_ptr(),
                  plan.k_pad, bad.data_ptr(), _stream())
        if int(e.item()) != (1 << 63) - 1:
            raise _lib.InvalidArgument(f"quantize: non-finite input at flat index {int(e.item())}")
        s32.fill_(float(np.float32(static_scale)))
        s64.fill_(float(static_scale))
        return xq, s32, s64
    _lib.call("qarvd_quantize_act", x.data_ptr(), _dtype_code(x), m, k, x.stride(0),
              _ptr(gather_dev), plan.k_pad, granularity, float(static_scale), bits,
              xq.data_ptr(), plan.k_pad, s32.data_ptr(), s64.data_ptr(), _ptr(err), _stream())
    if err is not None:
        _check_err(err, "quantize")
    return xq, s32, s64


def kernel_b_gemm_dequant(xq: torch.Tensor, scale_x: torch.Tensor, layer: QuantizedLayer,
                          out_dtype=torch.bfloat16, epilogue: int = _lib.EPI_NONE,
                          bias: Optional[torch.Tensor] = None, dump_acc: bool = False):
    """K2 (engine.cpp:46-105): dual-slab int8 tensor-core GEMM + fused dequant / bias epilogue.

    Returns y, or (y, acc_outlier, acc_normal) with ``dump_acc``.
    """
    m = xq.shape[0]
    n = layer.out_dim
    y = torch.empty((m, n), dtype=out_dtype, device=xq.device)
    acc_o = torch.zeros((m, n), dtype=torch.int32, device=xq.device) if dump_acc else None
    acc_n = torch.zeros((m, n), dtype=torch.int32, device=xq.device) if dump_acc else None
    b = bias if bias is not None else layer.bias
    _lib.call("qarvd_dual_gemm", xq.data_ptr(), xq.stride(0), layer.wq.data_ptr(),
              layer.wq.stride(0), m, n, layer.k_pad, layer.k_outlier, scale_x.data_ptr(),
              layer.scale_outlier32.data_ptr(), layer.scale_normal32.data_ptr(), _ptr(b), epilogue,
              _lib.BF16 if out_dtype == torch.bfloat16 else _lib.F32, y.data_ptr(), y.stride(0),
              _ptr(acc_o), _ptr(acc_n), _stream())
    if dump_acc:
        return y, acc_o, acc_n
    return y


def quantized_layer_forward(layer: QuantizedLayer, x: torch.Tensor, out_dtype=torch.bfloat16,
                            epilogue: int = _lib.EPI_NONE) -> torch.Tensor:
    """quantized_layer_forward(layer, x, Engine::int_kernels) (engine.cpp:134-142): K1 -> K2."""
    xq, s32, _ = kernel_a_quantize_activation(x, layer, layer.act_granularity, layer.act_scale)
    return kernel_b_gemm_dequant(xq, s32, layer, out_dtype=out_dtype, epilogue=epilogue)


class LinearHandle:
    """qarvd_linear_t: K1 + K2 behind one C-ABI call, incl. the host-buffer entry."""

    def __init__(self, layer: QuantizedLayer, epilogue: int = _lib.EPI_NONE):
        self.layer = layer
        h = _lib.ctypes.c_void_p()
        _lib.call("qarvd_linear_create", layer.wq.data_ptr(), layer.out_dim, layer.k_pad,
                  layer.k_outlier, _ptr(layer.gather_dev), layer.in_dim,
                  layer.scale_outlier32.data_ptr(), layer.scale_normal32.data_ptr(),
                  _ptr(layer.bias), layer.act_granularity, float(layer.act_scale), epilogue,
                  _lib.ctypes.byref(h))
        self.h = h

    def forward(self, x: torch.Tensor, y: Optional[torch.Tensor] = None) -> torch.Tensor:
        m = x.shape[0]
        if y is None:
            y = torch.empty((m, self.layer.out_dim), dtype=torch.bfloat16, device=x.device)
        _lib.call("qarvd_linear_forward", self.h, x.data_ptr(), m, y.data_ptr(), _stream())
        return y

    def forward_host(self, x_host: torch.Tensor, y_host: torch.Tensor) -> torch.Tensor:
        """x_host / y_host: CPU bf16 tensors (pinned for full PCIe bandwidth)."""
        _lib.call("qarvd_linear_forward_host", self.h, x_host.data_ptr(), x_host.shape[0],
                  y_host.data_ptr(), _stream())
        return y_host

    def close(self):
        if self.h:
            _lib.call("qarvd_linear_destroy", self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def chain_forward_host(handles: Sequence[LinearHandle], x_host: torch.Tensor,
                       y_host: torch.Tensor) -> torch.Tensor:
    """qarvd_linear_chain_forward_host: one H2D, K1+K2 per layer, one D2H (synchronous)."""
    arr = (_lib.ctypes.c_void_p * len(handles))(*[h.h for h in handles])
    _lib.call("qarvd_linear_chain_forward_host", arr, len(handles), x_host.data_ptr(),
              x_host.shape[0], y_host.data_ptr(), _stream())
    return y_host


def fuse_siblings(name: str, layers: Sequence[QuantizedLayer]) -> QuantizedLayer:
    """One dual-slab layer for sibling linears that read the same input (e.g. a block's
    self-attention q, k, v), bit-identical per output column to the separate layers.

    The fused K axis is [outlier slab of layer 0 | ... | outlier slab of layer L-1 | all d_in
    columns in original order | pad]: every layer keeps its own outlier columns (and group
    scales) in its own slab, holds zero codes in the other layers' slabs, and zero codes at its
    own outlier columns of the shared normal part.  acc_o / acc_n of each output column are
    therefore the same integer sums as in the separate layer (extra terms are 0 x code), and
    the epilogue is per column.  One K1 (its gather duplicates the slab columns) and one K2
    replace L of each; the K overhead is the sum of the slabs (~6% for three K_o = 32 slabs
    at d_in = 1536)."""
    if not layers:
        raise _lib.InvalidArgument("fuse_siblings: no layers")
    d_in = layers[0].in_dim
    for L in layers:
        if L.in_dim != d_in or L.gather_dev is None:
            raise _lib.InvalidArgument("fuse_siblings: layers must share the input width and carry their gather")
    dev = layers[0].wq.device
    k_o = sum(L.k_outlier for L in layers)
    k_pad = k_o + _round_up(d_in, 32)
    gather = np.full(k_pad, -1, dtype=np.int32)
    off = 0
    for L in layers:
        n_o = L.plan.outlier_count() if L.plan.enabled else 0
        gather[off:off + n_o] = L.plan.gather[:n_o]
        off += L.k_outlier
    gather[k_o:k_o + d_in] = np.arange(d_in, dtype=np.int32)
    n_tot = sum(L.out_dim for L in layers)
    wq = torch.zeros((n_tot, k_pad), dtype=torch.int8, device=dev)
    r0, off = 0, 0
    for L in layers:
        n = L.out_dim
        g = L.plan.gather
        if L.k_outlier:
            wq[r0:r0 + n, off:off + L.k_outlier] = L.wq[:, :L.k_outlier]
        # the layer's normal slab, scattered back to original column order
        pos = np.nonzero(g[L.k_outlier:] >= 0)[0] + L.k_outlier
        cols = torch.as_tensor(k_o + g[pos].astype(np.int64), device=dev)
        wq[r0:r0 + n].index_copy_(1, cols, L.wq[:, torch.as_tensor(pos, device=dev)])
        r0 += n
        off += L.k_outlier
    cat = lambda xs: torch.cat(xs, 0)
    plan = DualScalePlan(name, True, d_in, np.zeros(0, dtype=np.int64), np.arange(d_in, dtype=np.int64),
                         np.arange(d_in, dtype=np.uint32), gather, k_o, k_pad)
    return QuantizedLayer(name, n_tot, d_in, plan, wq, cat([L.scale_outlier64 for L in layers]),
                          cat([L.scale_normal64 for L in layers]), cat([L.scale_outlier32 for L in layers]),
                          cat([L.scale_normal32 for L in layers]), torch.from_numpy(gather).to(dev),
                          layers[0].act_granularity, layers[0].act_scale,
                          None if all(L.bias is None for L in layers) else
                          cat([L.bias if L.bias is not None else torch.zeros(L.out_dim, dtype=torch.float32, device=dev)
                               for L in layers]))
