"""Which K1(x) CTAs form the tail?  Per-CTA durations (QARVD_K1_TRACE) vs the rows' |x|max."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
trace = torch.zeros(3 * 8192, dtype=torch.int64, device="cuda")
os.environ["QARVD_K1_TRACE"] = str(trace.data_ptr())
import bench
import paper_2605_21072_b200 as qb
from paper_2605_21072_b200 import _lib, synth
layers = bench.build_ffn_layers(torch)
L = layers[0][2]
x = synth.synth_activation(bench.M_TOKENS, bench.DIM, seed=7)
m, k = x.shape
xq = torch.empty((m, L.k_pad), dtype=torch.int8, device="cuda")
sx = torch.empty(m, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
f = lambda: _lib.call("qarvd_quantize_act", x.data_ptr(), qb.BF16, m, k, k, L.gather_dev.data_ptr(), L.k_pad,
                      L.act_granularity, float(L.act_scale), 8, xq.data_ptr(), L.k_pad, sx.data_ptr(), None, None, st)
for _ in range(3): f()
durs = []
for rep in range(5):
    trace.zero_(); torch.cuda.synchronize(); f(); torch.cuda.synchronize()
    t = trace.view(-1, 3).cpu().numpy()[:1170]
    durs.append((t[:, 1] - t[:, 0]) / 1e3)
d = np.median(np.stack(durs), axis=0)
amax_bits = x.view(torch.int16).cpu().numpy().astype(np.uint16) & 0x7fff
rmax = amax_bits.max(axis=1)
pow2 = (rmax & 0x7f) == 0
cta_pow2 = pow2.reshape(-1, 4).any(axis=1)
print("rows with power-of-two |x|max:", int(pow2.sum()), "of", m)
print("CTA duration us: all p50 %.2f p90 %.2f max %.2f" % tuple(np.percentile(d, [50, 90, 100])))
print("CTAs holding a pow2 row: n=%d mean %.2f  | others mean %.2f" % (cta_pow2.sum(), d[cta_pow2].mean(), d[~cta_pow2].mean()))
slow = np.argsort(d)[-10:]
print("10 slowest CTAs:", [(int(c), round(float(d[c]), 2), bool(cta_pow2[c])) for c in slow])
t = trace.view(-1, 3).cpu().numpy()[:1170]
sm = t[:, 2]
st = (t[:, 0] - t[:, 0].min()) / 1e3
en = (t[:, 1] - t[:, 0].min()) / 1e3
print("start spread us:", np.percentile(st, [0, 50, 100]).round(2), " end:", np.percentile(en, [0, 50, 90, 99, 100]).round(2))
per_sm_end = np.zeros(148); per_sm_n = np.zeros(148)
for s_, e_ in zip(sm, en):
    per_sm_end[int(s_)] = max(per_sm_end[int(s_)], e_); per_sm_n[int(s_)] += 1
order = np.argsort(per_sm_end)[::-1][:10]
print("latest-finishing SMs (sm, end us, ctas):", [(int(i), round(float(per_sm_end[i]), 2), int(per_sm_n[i])) for i in order])
print("SM end percentiles:", np.percentile(per_sm_end, [0, 50, 90, 100]).round(2))
# durations by CTA index order (launch order)
d_last = en - st
print("dur by CTA index quartile:", [round(float(np.median(d_last[q * 292:(q + 1) * 292])), 2) for q in range(4)])
