"""K1 diagnostics: per-CTA globaltimer start/end for the two FFN K1 launches (x and U).

Sets QARVD_K1_TRACE to a device buffer before the first K1 launch, runs each K1 of the
folded FFN chain alone (after warm-up), and prints the launch span, CTA start spread,
CTA duration percentiles and the per-SM CTA counts.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

trace = torch.zeros(3 * 8192, dtype=torch.int64, device="cuda")
os.environ["QARVD_K1_TRACE"] = str(trace.data_ptr())

import bench  # noqa: E402
import paper_2605_21072_b200 as qb  # noqa: E402
from paper_2605_21072_b200 import _lib, synth  # noqa: E402
from paper_2605_21072_b200.pipeline import QuantizedChain  # noqa: E402

layers = bench.build_ffn_layers(torch)
chain = QuantizedChain([layers[0][2], layers[1][2]], bench.M_TOKENS, epilogues=[qb.EPI_GELU, qb.EPI_NONE])
chain.x.copy_(synth.synth_activation(bench.M_TOKENS, bench.DIM, seed=7))
for _ in range(3):
    chain.launch()
torch.cuda.synchronize()
st = torch.cuda.current_stream().cuda_stream
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush_rd = torch.ones(64 << 20, dtype=torch.int32, device="cuda")
MODE = os.environ.get("FLUSH", "write")


def do_flush():
    if MODE in ("write", "write+read"):
        flush.fill_(1)
    if MODE == "write+read":
        flush_rd.sum()  # clean reads evict the dirty lines outside the timed region


for i in range(2):
    L = chain.layers[i]
    src = chain._src(i)
    for rep in range(3):
        trace.zero_()
        do_flush()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.call("qarvd_quantize_act", src.data_ptr(), qb.BF16, chain.m, L.in_dim, src.stride(0),
                  None if L.gather_dev is None else L.gather_dev.data_ptr(), L.k_pad,
                  L.act_granularity, float(L.act_scale), 8, chain.xq[i].data_ptr(), L.k_pad,
                  chain.sx[i].data_ptr(), None, None, st)
        e1.record()
        torch.cuda.synchronize()
    t = trace.view(-1, 3).cpu().numpy()
    n = int((t[:, 0] > 0).sum())
    t = t[:n]
    t0 = t[:, 0].min()
    start = (t[:, 0] - t0) / 1e3
    end = (t[:, 1] - t0) / 1e3
    dur = end - start
    sms = np.bincount(t[:, 2].astype(np.int64), minlength=148)
    print(f"[flush={MODE}] K1 layer {i}: k={L.in_dim} gather={L.gather_dev is not None} ctas={n} event={e0.elapsed_time(e1)*1e3:.1f} us "
          f"span={end.max():.1f} us")
    print("  start pct (us):", np.percentile(start, [0, 10, 50, 90, 100]).round(2))
    print("  end   pct (us):", np.percentile(end, [0, 10, 50, 90, 100]).round(2))
    print("  dur   pct (us):", np.percentile(dur, [0, 10, 50, 90, 100]).round(2))
    print("  ctas per SM min/median/max:", sms.min(), int(np.median(sms)), sms.max())
    hist, edges = np.histogram(start, bins=10)
    print("  start histogram:", hist.tolist(), "edges", edges.round(1).tolist())
