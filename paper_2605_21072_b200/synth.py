"""Synthetic Wan-1.3B-shaped layers and activations, generated on the device.

Follows the reference's synthetic-weight recipe (toy_model.cpp:146-166):
Gaussian weights with std 1/sqrt(fan_in), and for every injection whose
pattern matches the layer name a seeded partial Fisher-Yates choice of
``max(1, llround(fraction * d_in))`` input columns scaled by ``gamma``.  The
column choice reproduces the reference PRNG stream exactly
(Prng(mix_seed(mix_seed(seed, li), kInjectSalt)).next_u64(), rng.hpp:11-23);
the Gaussian values come from a counter-based device generator (bf16).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np
import torch

from . import _lib
from .engine import _stream

M64 = (1 << 64) - 1
K_INJECT_SALT = 0x696E6A656374  # "inject", toy_model.cpp:23
K_ACT_SALT = 0x616374           # "act" (this build)

# Wan2.1-1.3B DiT shapes
WAN_DIM = 1536
WAN_FFN = 8960
WAN_BLOCKS = 30
WAN_TEXT_LEN = 512
WAN_TOKENS_PER_FRAME = 1560
WAN_CHUNK_TOKENS = 4680  # one 3-latent-frame chunk
WAN_FRAMES = 21

BLOCK_LAYER_TYPES = ("self_attn.q", "self_attn.k", "self_attn.v", "self_attn.o",
                     "cross_attn.q", "cross_attn.k", "cross_attn.v", "cross_attn.o",
                     "ffn.0", "ffn.2")  # toy_model.cpp:25-27


def splitmix64(state: int) -> Tuple[int, int]:
    """rng.hpp:11-16; returns (new_state, output)."""
    state = (state + 0x9E3779B97F4A7C15) & M64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return state, z ^ (z >> 31)


def mix_seed(a: int, b: int) -> int:
    """rng.hpp:18-23."""
    _, h = splitmix64(a & M64)
    s = h ^ ((b + 0x9E3779B97F4A7C15) & M64)
    _, out = splitmix64(s)
    return out


def pick_outlier_columns(seed: int, layer_index: int, d_in: int, fraction: float) -> np.ndarray:
    """Seeded partial Fisher-Yates of toy_model.cpp:152-166 (returns the chosen columns)."""
    count = max(1, int(np.floor(fraction * d_in + 0.5)))  # llround for positive values
    cols = list(range(d_in))
    state = mix_seed(mix_seed(seed, layer_index), K_INJECT_SALT)
    for i in range(min(count, d_in)):
        state, r = splitmix64(state)
        j = i + r % (d_in - i)
        cols[i], cols[j] = cols[j], cols[i]
    return np.asarray(cols[:count], dtype=np.int64)


@dataclass
class LayerSpec:
    """toy_model.hpp:44-48 plus the synthetic-outlier recipe and the token count it sees."""

    index: int
    name: str
    out_dim: int
    in_dim: int
    tokens: int           # M of one chunk forward
    outlier_fraction: float
    gamma: float

    def weight_bytes(self) -> int:
        return self.out_dim * self.in_dim * 2


def _injection(ltype: str, b: int) -> Tuple[float, float]:
    """Heterogeneous per-type / per-depth outlier pattern (ffn.2 prominent, cross_attn.v smooth,
    PAPER.md:173)."""
    if ltype in ("ffn.0", "ffn.2"):
        return 0.021, 8.0
    if ltype in ("self_attn.q", "self_attn.k", "self_attn.v"):
        return (0.021, 6.0) if b % 2 == 0 else (0.0, 1.0)
    if ltype == "self_attn.o":
        return (0.01, 5.0) if b % 3 == 0 else (0.0, 1.0)
    if ltype == "cross_attn.q":
        return (0.021, 8.0) if b < 10 else (0.0, 1.0)
    if ltype == "cross_attn.k":
        return (0.01, 4.0) if b % 4 == 0 else (0.0, 1.0)
    if ltype == "cross_attn.o":
        return (0.015, 6.0) if b % 2 == 1 else (0.0, 1.0)
    return 0.0, 1.0  # cross_attn.v: smooth


def wan_registry(blocks: int = WAN_BLOCKS, dim: int = WAN_DIM, ffn: int = WAN_FFN,
                 chunk_tokens: int = WAN_CHUNK_TOKENS, text_len: int = WAN_TEXT_LEN) -> List[LayerSpec]:
    specs = []
    li = 0
    for b in range(blocks):
        for t in BLOCK_LAYER_TYPES:
            out_dim, in_dim = dim, dim
            if t == "ffn.0":
                out_dim = ffn
            if t == "ffn.2":
                in_dim = ffn
            tokens = text_len if t in ("cross_attn.k", "cross_attn.v") else chunk_tokens
            frac, gamma = _injection(t, b)
            specs.append(LayerSpec(li, f"block{b}.{t}", out_dim, in_dim, tokens, frac, gamma))
            li += 1
    return specs


def synth_bf16(rows: int, cols: int, seed: int, stddev: float, outlier_cols: Optional[np.ndarray] = None,
               gamma: float = 1.0, device="cuda", out: Optional[torch.Tensor] = None) -> torch.Tensor:
    if out is None:
        out = torch.empty((rows, cols), dtype=torch.bfloat16, device=device)
    oc = None
    if outlier_cols is not None and len(outlier_cols) > 0 and gamma != 1.0:
        oc = torch.as_tensor(np.asarray(outlier_cols, dtype=np.int32), device=out.device)
    _lib.call("qarvd_synth_bf16", out.data_ptr(), rows, cols, out.stride(0), seed & M64,
              float(stddev), None if oc is None else oc.data_ptr(), 0 if oc is None else len(oc),
              float(gamma), _stream())
    return out


def synth_weight(spec: LayerSpec, seed: int = 1, device="cuda", out=None) -> torch.Tensor:
    cols = (pick_outlier_columns(seed, spec.index, spec.in_dim, spec.outlier_fraction)
            if spec.outlier_fraction > 0 else None)
    return synth_bf16(spec.out_dim, spec.in_dim, mix_seed(seed, spec.index),
                      1.0 / np.sqrt(spec.in_dim), cols, spec.gamma, device, out)


def synth_activation(rows: int, k: int, seed: int, frame: int = 0, heavy_fraction: float = 0.005,
                     heavy_gamma: float = 6.0, device="cuda", out=None) -> torch.Tensor:
    """bf16 N(0, s_f^2) activations with seeded heavy channels; s_f = 1 + 0.05*frame."""
    heavy = pick_outlier_columns(seed ^ K_ACT_SALT, 0, k, heavy_fraction)
    return synth_bf16(rows, k, mix_seed(seed ^ K_ACT_SALT, frame + 1), 1.0 + 0.05 * frame,
                      heavy, heavy_gamma, device, out)
