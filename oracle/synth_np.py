"""TEST INFRASTRUCTURE ONLY — numpy inputs for bench.py's reference arm and CPU baselines.

The same recipe as the product's device generator (paper_2605_21072_b200/synth.py, which the
reference arm must not import): Wan-1.3B-shaped bf16-exact weights N(0, 1/fan_in) with the
seeded Fisher-Yates outlier columns of toy_model.cpp:152-166 (rng.hpp streams, bit-exact column
choice) scaled by gamma, and bf16 activations N(0, s_f^2) with seeded heavy channels.  Values are
drawn by numpy, so they are the same distribution and outlier layout, not the device's bit stream.
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
K_INJECT_SALT = 0x696E6A656374  # "inject", toy_model.cpp:23
K_ACT_SALT = 0x616374


def _splitmix64(state):
    state = (state + 0x9E3779B97F4A7C15) & M64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return state, z ^ (z >> 31)


def mix_seed(a, b):
    _, h = _splitmix64(a & M64)
    _, out = _splitmix64(h ^ ((b + 0x9E3779B97F4A7C15) & M64))
    return out


def outlier_columns(seed, layer_index, d_in, fraction):
    count = max(1, int(np.floor(fraction * d_in + 0.5)))
    cols = list(range(d_in))
    state = mix_seed(mix_seed(seed, layer_index), K_INJECT_SALT)
    for i in range(min(count, d_in)):
        state, r = _splitmix64(state)
        j = i + r % (d_in - i)
        cols[i], cols[j] = cols[j], cols[i]
    return np.asarray(cols[:count], dtype=np.int64)


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round to the bf16 grid (RNE, bytes.hpp:40-45), returned as f64."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def weight(out_dim, in_dim, layer_index, seed=1, fraction=0.021, gamma=8.0):
    rng = np.random.default_rng(mix_seed(seed, layer_index))
    w = rng.standard_normal((out_dim, in_dim), dtype=np.float32) / np.float32(np.sqrt(in_dim))
    if fraction > 0:
        w[:, outlier_columns(seed, layer_index, in_dim, fraction)] *= np.float32(gamma)
    return bf16_round(w)


def activation(rows, k, seed, frame=0, heavy_fraction=0.005, heavy_gamma=6.0):
    rng = np.random.default_rng(mix_seed(seed ^ K_ACT_SALT, frame + 1))
    x = rng.standard_normal((rows, k), dtype=np.float32) * np.float32(1.0 + 0.05 * frame)
    x[:, outlier_columns(seed ^ K_ACT_SALT, 0, k, heavy_fraction)] *= np.float32(heavy_gamma)
    return bf16_round(x)
