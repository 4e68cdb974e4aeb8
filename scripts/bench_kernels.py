"""Per-kernel microbenchmark: K2 at the Wan shapes for each tile width, K1 at the FFN shapes.
Cold L2 (256 MiB flush) before every timed launch; CUDA events on the launching stream."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_21072_b200 as qb  # noqa: E402
from paper_2605_21072_b200 import _lib, engine, synth  # noqa: E402

torch.cuda.set_device(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def make_layer(n, k, n_out, seed):
    spec = synth.LayerSpec(seed, "l", n, k, 4680, n_out / k if n_out else 0.0, 8.0)
    w = synth.synth_weight(spec, seed=seed)
    rep = qb.analyze_layer("l", w)
    plan = engine.build_plan("l", k, rep.aligned_outliers)
    return engine.prepare_weights("l", w, plan)


out = {}
M = int(os.environ.get("M", "4680"))
for name, n, k, no in [("qkv", 1536, 1536, 32), ("ffn0", 8960, 1536, 32), ("ffn2", 1536, 8960, 188)]:
    L = make_layer(n, k, no, seed=hash(name) % 1000)
    x = synth.synth_activation(M, k, seed=3)
    xq, sx, _ = engine.kernel_a_quantize_activation(x, L)
    y = torch.empty((M, n), dtype=torch.bfloat16, device="cuda")
    for cg, bn in ((1, 128), (1, 256), (2, 128), (2, 256)):
        os.environ["QARVD_GEMM_BN"] = str(bn)
        os.environ["QARVD_GEMM_CG"] = str(cg)
        for epi in (qb.EPI_NONE, qb.EPI_GELU):
            f = lambda: _lib.call("qarvd_dual_gemm", xq.data_ptr(), L.k_pad, L.wq.data_ptr(), L.k_pad, M, n,
                                  L.k_pad, L.k_outlier, sx.data_ptr(), L.scale_outlier32.data_ptr(),
                                  L.scale_normal32.data_ptr(), None, epi, qb.BF16, y.data_ptr(), n,
                                  None, None, st)
            ms = timeit(f)
            out[f"gemm_{name}_cg{cg}_bn{bn}_{'gelu' if epi else 'none'}"] = {
                "ms": ms, "tops": 2.0 * M * n * k / (ms * 1e-3) / 1e12}
    os.environ.pop("QARVD_GEMM_BN")
    os.environ.pop("QARVD_GEMM_CG")
    for gran in (qb.ACT_PER_TOKEN, qb.ACT_PER_TENSOR):
        f = lambda: _lib.call("qarvd_quantize_act", x.data_ptr(), qb.BF16, M, k, k, L.gather_dev.data_ptr(),
                              L.k_pad, gran, 0.05, 8, xq.data_ptr(), L.k_pad, sx.data_ptr(), None, None, st)
        ms = timeit(f)
        byt = M * (k * 2 + L.k_pad + 4)
        out[f"quant_{name}_{'token' if gran == 0 else 'static'}"] = {"ms": ms, "gbs": byt / (ms * 1e-3) / 1e9}
    # cuBLAS bf16 at the same shape
    wb = torch.randn(n, k, device="cuda", dtype=torch.bfloat16)
    ms = timeit(lambda: torch.nn.functional.linear(x, wb))
    out[f"cublas_bf16_{name}"] = {"ms": ms, "tflops": 2.0 * M * n * k / (ms * 1e-3) / 1e12}
print(json.dumps(out, indent=1))
