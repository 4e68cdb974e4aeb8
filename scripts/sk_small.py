"""Stream-K K2 at small row counts (the host chain's row chunks): data-parallel vs stream-K over
all SM pairs for the FFN-down shape, 20 launches per CUDA graph, device time per launch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_21072_b200 as qb
from paper_2605_21072_b200 import _lib, engine, synth
n, k, no = 1536, 8960, 188
spec = synth.LayerSpec(7, "l", n, k, 4680, no / k, 8.0)
w = synth.synth_weight(spec, seed=1)
L = engine.prepare_weights("l", w, engine.build_plan("l", k, qb.analyze_layer("l", w).aligned_outliers))
lib = _lib.load()
for m in (256, 584, 1024, 2048):
    xq, sx, _ = engine.kernel_a_quantize_activation(synth.synth_activation(m, k, seed=3), L)
    y0 = torch.empty((m, n), dtype=torch.bfloat16, device="cuda"); y1 = torch.empty_like(y0)
    nb = int(lib.qarvd_dual_gemm_workspace_size(m, n, L.k_pad, L.k_outlier))
    ws = torch.zeros(max(nb, 256) + 256, dtype=torch.uint8, device="cuda")
    st = lambda: torch.cuda.current_stream().cuda_stream
    dp = lambda: _lib.call("qarvd_dual_gemm", xq.data_ptr(), L.k_pad, L.wq.data_ptr(), L.k_pad, m, n, L.k_pad, L.k_outlier,
                           sx.data_ptr(), L.scale_outlier32.data_ptr(), L.scale_normal32.data_ptr(), None, 0, qb.BF16,
                           y0.data_ptr(), n, None, None, st())
    sk = lambda: _lib.call("qarvd_dual_gemm_ws", xq.data_ptr(), L.k_pad, L.wq.data_ptr(), L.k_pad, m, n, L.k_pad,
                           L.k_outlier, sx.data_ptr(), L.scale_outlier32.data_ptr(), L.scale_normal32.data_ptr(), None, 0,
                           y1.data_ptr(), n, ws.data_ptr(), ws.numel(), st())
    res = {}
    for name, f in (("dp", dp), ("sk", sk)):
        f(); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g):
                for _ in range(20):
                    f()
        torch.cuda.synchronize()
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) * 1e3 / 20
    same = torch.equal(y0.view(torch.int16), y1.view(torch.int16))
    print(f"M={m}: workspace {nb} B, data-parallel {res['dp']:.1f} us, stream-K {res['sk']:.1f} us, bit-identical {same}")
