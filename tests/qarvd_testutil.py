"""Shared helpers for the test-suite (module name chosen to avoid clashing with other
installed `tests` packages)."""
import numpy as np


def rng(seed=0):
    return np.random.default_rng(seed)


def bf16_values(shape, seed=0, scale=1.0, heavy_cols=None, gamma=8.0):
    """Random bf16-representable values (as uint16 bits and f64)."""
    import oracle

    r = np.random.default_rng(seed)
    x = (r.standard_normal(shape) * scale).astype(np.float32)
    if heavy_cols is not None:
        x[..., heavy_cols] *= gamma
    bits = oracle.f32_to_bf16_bits(x)
    return bits, oracle.bf16_bits_to_f64(bits)
