"""QARQ quantized-model files -> device-resident layers (the format on the left of the path).

Reads the reference's on-disk QuantizedModel (save_quantized_model / load_quantized_model,
/root/reference/proj/core/src/engine.cpp:180-333): magic "QARQ", u16 version 1, u64 header
length, the JSON header, then per layer either bf16 weights (preserved layers) or a QTNS
packed-int tensor of pre-permuted codes (tensor.cpp:155-194, :221-264; 4-bit codes two per
byte, low nibble first), f32 normal-group scales, for dual-scale layers f32 outlier-group
scales and the u32 permutation, then the f32 activation scale and i32 zero point.

``load_qarq`` parses on the host (numpy views of one read); ``to_device`` builds the kernel
layout (engine.build_plan's padded gather from the stored permutation) and uploads codes and
scales once.  The f32 scales are the values the reference itself works with after a load.
"""
from __future__ import annotations

import json
import struct
from dataclasses import dataclass
from typing import List, Optional

import numpy as np
import torch

from . import _lib, engine


@dataclass
class QarqLayer:
    name: str
    out_dim: int
    in_dim: int
    preserved: bool
    bits: int = 8
    codes: Optional[np.ndarray] = None          # int8 [out x in], pre-permuted [outlier | normal]
    scale_normal: Optional[np.ndarray] = None   # f32 [out]
    scale_outlier: Optional[np.ndarray] = None  # f32 [out] (dual-scale layers)
    permutation: Optional[np.ndarray] = None    # u32 [in] (dual-scale layers)
    outlier_count: int = 0
    act_bits: int = 8
    act_symmetric: bool = True
    act_scale: float = 0.0
    act_zero: int = 0
    fp_weight_bf16: Optional[np.ndarray] = None  # uint16 bits [out x in] (preserved layers)
    codes_packed: Optional[np.ndarray] = None    # 4-bit layers: the file's packed bytes (uint8)


def _read_qtns_int(buf: memoryview, pos: int):
    if bytes(buf[pos:pos + 4]) != b"QTNS":
        raise _lib.QarvdError("tensor container: bad magic")
    version, dtype, bits, rank = struct.unpack_from("<HBBB", buf, pos + 4)
    if version != 1:
        raise _lib.QarvdError("tensor container: unsupported version")
    if dtype != 2:
        raise _lib.QarvdError("load_int_tensor: container holds float data")
    pos += 9
    shape = struct.unpack_from("<" + "Q" * rank, buf, pos)
    pos += 8 * rank
    count = int(np.prod(shape)) if rank else 1
    if bits == 4:
        nbytes = (count + 1) // 2
        raw = np.frombuffer(buf, dtype=np.uint8, count=nbytes, offset=pos)
        lo = (raw & 0x0F).astype(np.int8)
        hi = (raw >> 4).astype(np.int8)
        nib = np.empty(2 * nbytes, dtype=np.int8)
        nib[0::2], nib[1::2] = lo, hi
        codes = ((nib << 4).astype(np.int8) >> 4)[:count]  # sign-extend the nibbles
        packed = raw.copy()
    else:
        nbytes = count
        codes = np.frombuffer(buf, dtype=np.int8, count=count, offset=pos).copy()
        packed = None
    return codes.reshape(shape), bits, pos + nbytes, packed


def load_qarq(path: str):
    """(header dict, [QarqLayer]) of a QARQ file, with the reference's checks and messages."""
    with open(path, "rb") as f:
        data = f.read()
    buf = memoryview(data)
    if bytes(buf[:4]) != b"QARQ":
        raise _lib.QarvdError(f"quantized model: bad magic in {path}")
    (version,) = struct.unpack_from("<H", buf, 4)
    if version != 1:
        raise _lib.QarvdError("quantized model: unsupported version")
    (hlen,) = struct.unpack_from("<Q", buf, 6)
    header = json.loads(bytes(buf[14:14 + hlen]).decode())
    pos = 14 + hlen
    layers: List[QarqLayer] = []
    for lj in header["layers"]:
        n, k = int(lj["out_dim"]), int(lj["in_dim"])
        L = QarqLayer(lj["name"], n, k, bool(lj["preserved"]))
        if L.preserved:
            L.fp_weight_bf16 = np.frombuffer(buf, dtype=np.uint16, count=n * k, offset=pos).reshape(n, k).copy()
            pos += 2 * n * k
            layers.append(L)
            continue
        codes, bits, pos, packed = _read_qtns_int(buf, pos)
        if codes.shape != (n, k):
            raise _lib.QarvdError(f"quantized model: weight shape mismatch for {L.name}")
        if bits != int(lj["weight_bits"]):
            raise _lib.QarvdError(f"quantized model: bit-width mismatch for {L.name}")
        L.codes, L.bits, L.codes_packed = codes, bits, packed
        L.scale_normal = np.frombuffer(buf, dtype="<f4", count=n, offset=pos).copy()
        pos += 4 * n
        dual = bool(lj["dual_scale"])
        if dual:
            L.scale_outlier = np.frombuffer(buf, dtype="<f4", count=n, offset=pos).copy()
            pos += 4 * n
            L.permutation = np.frombuffer(buf, dtype="<u4", count=k, offset=pos).copy()
            pos += 4 * k
            L.outlier_count = int(lj["outlier_count"])
        L.act_bits = int(lj["act_bits"])
        L.act_symmetric = bool(lj["act_symmetric"])
        L.act_scale = float(np.frombuffer(buf, dtype="<f4", count=1, offset=pos)[0])
        L.act_zero = int(np.frombuffer(buf, dtype="<i4", count=1, offset=pos + 4)[0])
        pos += 8
        layers.append(L)
    return header, layers


def to_device(L: QarqLayer, device="cuda") -> engine.QuantizedLayer:
    """One QARQ layer as a device QuantizedLayer (per-tensor static activation scale, as the
    reference engine runs it, engine.cpp:57).  Asymmetric activation zero points are outside
    this build's envelope (the reference's own pipeline never writes them)."""
    if L.preserved:
        raise _lib.InvalidArgument(f"kernel_b: layer is preserved, no integer path: {L.name}")
    outl = (np.sort(L.permutation[:L.outlier_count]).astype(np.int64) if L.permutation is not None
            else np.zeros(0, dtype=np.int64))
    plan = engine.build_plan(L.name, L.in_dim, outl)
    if L.permutation is not None and not np.array_equal(plan.permutation, L.permutation):
        raise _lib.QarvdError(f"quantized model: permutation of {L.name} is not [outliers | normals] sorted")
    n_o = len(outl)
    t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=device)
    if L.codes_packed is not None:
        # 4-bit layers: the packed bytes go to the device as stored (half the bytes of int8) and
        # one kernel expands them into the K2 layout (qarvd_unpack_codes_i4)
        idx = np.full(plan.k_pad, -1, dtype=np.int32)
        idx[:n_o] = np.arange(n_o, dtype=np.int32)
        idx[plan.k_outlier:plan.k_outlier + (L.in_dim - n_o)] = np.arange(n_o, L.in_dim, dtype=np.int32)
        wq_dev = torch.empty((L.out_dim, plan.k_pad), dtype=torch.int8, device=device)
        packed_dev, idx_dev = t(L.codes_packed, torch.uint8), t(idx, torch.int32)
        _lib.call("qarvd_unpack_codes_i4", packed_dev.data_ptr(), L.out_dim, L.in_dim, idx_dev.data_ptr(),
                  plan.k_pad, wq_dev.data_ptr(), plan.k_pad, torch.cuda.current_stream().cuda_stream)
    else:
        wq = np.zeros((L.out_dim, plan.k_pad), dtype=np.int8)
        wq[:, :n_o] = L.codes[:, :n_o]
        wq[:, plan.k_outlier:plan.k_outlier + (L.in_dim - n_o)] = L.codes[:, n_o:]
        wq_dev = t(wq, torch.int8)
    sn = L.scale_normal.astype(np.float64)
    so = L.scale_outlier.astype(np.float64) if L.scale_outlier is not None else sn
    layer = engine.QuantizedLayer(L.name, L.out_dim, L.in_dim, plan, wq_dev, t(so, torch.float64),
                                  t(sn, torch.float64), t(so.astype(np.float32), torch.float32),
                                  t(sn.astype(np.float32), torch.float32), t(plan.gather, torch.int32),
                                  _lib.ACT_PER_TENSOR, float(np.float32(L.act_scale)))
    if not L.act_symmetric and L.act_zero != 0:
        # kernel B's zero-point correction (engine.cpp:74-83, :95-100): the per-column integer
        # sums of each group, computed once here (the reference precomputes them "offline"),
        # folded into the epilogue's bias: y = s_x t + (-(z s_x) sum_g s_g[j] colsum_g[j])
        z, s_x = int(L.act_zero), float(np.float32(L.act_scale))
        w64 = layer.wq.to(torch.int64)
        cs_o = w64[:, :plan.k_outlier].sum(1).double()
        cs_n = w64[:, plan.k_outlier:].sum(1).double()
        corr = layer.scale_normal64 * (cs_n + (cs_o if n_o == 0 else 0))
        if n_o > 0:
            corr = layer.scale_outlier64 * cs_o + layer.scale_normal64 * cs_n
        layer.bias = (-(z * s_x) * corr).float().contiguous()
        layer.act_zero = z
    return layer
