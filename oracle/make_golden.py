"""TEST INFRASTRUCTURE: generate tests/golden/*.npz from the compiled reference
(oracle/_ref/libqarvd_ref.so, i.e. the unmodified reference sources).  Run here,
where /root/reference exists:  python oracle/make_golden.py
The fixtures pin the C restatement even where _ref is unavailable."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def bf16(shape, seed, heavy=None, gamma=8.0, scale=1.0):
    r = np.random.default_rng(seed)
    x = (r.standard_normal(shape) * scale).astype(np.float32)
    if heavy is not None:
        x[..., heavy] *= gamma
    b = oracle.f32_to_bf16_bits(x)
    return b, oracle.bf16_bits_to_f64(b)


def main():
    os.makedirs(OUT, exist_ok=True)
    # quantize (quant.cpp:113-138 via kernel_a_quantize_activation), per-token + static
    _, x = bf16((48, 160), 1, heavy=[5, 99])
    codes, scales = oracle.ref_quantize(x, per_token=True)
    codes_s, _ = oracle.ref_quantize(x, per_token=False, s=0.0173)
    np.savez_compressed(os.path.join(OUT, "quantize.npz"), x=x, codes=codes.astype(np.int8),
                        scales=scales, static_scale=0.0173, codes_static=codes_s.astype(np.int8))
    # kernel_b_gemm_dequant with a dual-scale plan (engine.cpp:46-105)
    r = np.random.default_rng(2)
    m, n, k, no = 16, 24, 128, 32
    xq = r.integers(-127, 128, (m, k)).astype(np.int8)
    wq = r.integers(-127, 128, (n, k)).astype(np.int8)
    so, sn = r.random(n) * 0.01, r.random(n) * 0.002
    sx = np.full(m, 0.0371)
    y = oracle.ref_kernel_b(xq, wq, np.arange(k, dtype=np.uint32), no, True, sx[:1], so, sn)
    np.savez_compressed(os.path.join(OUT, "kernel_b.npz"), xq=xq, wq=wq, n_outlier=no, s_x=sx,
                        s_o=so, s_n=sn, y=y)
    # analyze_layer + build_plan codes (outlier.cpp:98-102, dual_scale.cpp:58-114)
    _, w = bf16((64, 256), 3, heavy=[3, 30, 31, 200], gamma=6.0, scale=1 / 16)
    a = oracle.ref_analyze_layer(w)
    from paper_2605_21072_b200.engine import build_plan

    plan = build_plan("g", 256, a["aligned"])
    bp = oracle.ref_build_plan_codes(w, a["aligned"])
    np.savez_compressed(os.path.join(OUT, "analyze.npz"), w=w, norms=a["norms"], raw=a["raw"],
                        aligned=a["aligned"], threshold=a["threshold"], gather=plan.gather,
                        k_outlier=plan.k_outlier, wq=bp["wq"], s_o=bp["scale_outlier"],
                        s_n=bp["scale_normal"])
    # init_scale_percentile_search (quant.cpp:190-226)
    frames, rows, kk = 21, 12, 128
    xb, x64 = bf16((frames * rows, kk), 4, heavy=list(range(0, kk, 29)))
    best, scale, mse = oracle.ref_percentile_search(x64, frames, rows, kk)
    np.savez_compressed(os.path.join(OUT, "search.npz"), x_bits=xb, frames=frames, rows=rows, k=kk,
                        best_pct=best, scale=scale, mse=mse)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
