"""Throughput probes of K2 (QARVD_GEMM_DEBUG): full kernel, MMA-only (TMA skipped),
TMA-only (MMA skipped), for each CTA-group / tile width, at the FFN shapes."""
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


def timeit(fn, reps=15, do_flush=True):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if do_flush:
            flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


M = 4680
out = {}
for name, n, k, no in [("qkv", 1536, 1536, 32), ("ffn0", 8960, 1536, 32), ("ffn2", 1536, 8960, 188)]:
    spec = synth.LayerSpec(7, "l", n, k, M, no / k, 8.0)
    w = synth.synth_weight(spec, seed=1)
    plan = engine.build_plan("l", k, qb.analyze_layer("l", w).aligned_outliers)
    L = engine.prepare_weights("l", w, plan)
    x = synth.synth_activation(M, k, seed=3)
    xq, sx, _ = engine.kernel_a_quantize_activation(x, L)
    y = torch.empty((M, n), dtype=torch.bfloat16, device="cuda")
    f = lambda: _lib.call("qarvd_dual_gemm", xq.data_ptr(), L.k_pad, L.wq.data_ptr(), L.k_pad, M, n,
                          L.k_pad, L.k_outlier, sx.data_ptr(), L.scale_outlier32.data_ptr(),
                          L.scale_normal32.data_ptr(), None, 0, qb.BF16, y.data_ptr(), n, None, None, st)
    for cg, bn, ks in ((1, 128, 1), (1, 192, 1), (1, 128, 2), (2, 128, 1), (2, 256, 1), (2, 128, 2),
                       (2, 256, 2)):
        os.environ["QARVD_GEMM_BN"] = str(bn)
        os.environ["QARVD_GEMM_CG"] = str(cg)
        os.environ["QARVD_GEMM_KS"] = str(ks)
        for dbg, tag in ((0, "full"), (2, "mma_only")):
            os.environ["QARVD_GEMM_DEBUG"] = str(dbg)
            for warm in (False,):
                ms = timeit(f, do_flush=not warm)
                out[f"{name}_cg{cg}_bn{bn}_ks{ks}_{tag}{'_warmL2' if warm else ''}"] = round(
                    2.0 * M * n * k / (ms * 1e-3) / 1e12, 1)
        os.environ.pop("QARVD_GEMM_DEBUG")
print(json.dumps(out, indent=1))
