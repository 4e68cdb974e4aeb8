"""Config 3 per-kernel breakdown: the 30-block Wan stack (q/k/v and cross k/v fused, as the bench)
captured sequentially with CUDA event nodes between the kernels, L2 flushed before each replay;
device time and TOPS per layer type for K1 and K2.  Writes a markdown table to stdout."""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_21072_b200.pipeline import wan_stack_chain

torch.cuda.set_device(0)
chain = wan_stack_chain(fuse_qkv=True)
chain.x.normal_()
if chain.ctx is not None:
    chain.ctx.normal_()
g = chain.capture(timed=True)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
acc = None
for _ in range(reps):
    flush.fill_(1)
    g.replay()
    torch.cuda.synchronize()
    t = np.array(chain.kernel_times_ms())
    acc = t if acc is None else acc + t
acc /= reps
rows = defaultdict(lambda: [0.0, 0.0, 0.0, 0])  # type -> [k1 ms, k2 ms, ops, count]
for i, L in enumerate(chain.layers):
    typ = L.name.split(".", 1)[1] if "." in L.name else L.name
    r = rows[typ]
    r[0] += acc[2 * i]
    r[1] += acc[2 * i + 1]
    r[2] += 2.0 * chain.ms[i] * L.out_dim * L.in_dim
    r[3] += 1
tot_k1 = sum(r[0] for r in rows.values())
tot_k2 = sum(r[1] for r in rows.values())
tot_ops = sum(r[2] for r in rows.values())
print(f"Sequential graph (event nodes between kernels cut the PDL overlap), mean of {reps} replays after an L2 flush.\n")
print("| layer type | layers | M x N x K | K1 ms | K2 ms | K2 TOPS | share of the forward |")
print("|---|---|---|---|---|---|---|")
for typ, (k1, k2, ops, n) in rows.items():
    L = next(l for l in chain.layers if l.name.endswith(typ))
    i = chain.layers.index(L)
    print(f"| {typ} | {n} | {chain.ms[i]} x {L.out_dim} x {L.in_dim} | {k1:.3f} | {k2:.3f} | "
          f"{ops / (k2 * 1e-3) / 1e12:.0f} | {(k1 + k2) / (tot_k1 + tot_k2):.1%} |")
print(f"| total | {len(chain.layers)} | | {tot_k1:.3f} | {tot_k2:.3f} | {tot_ops / (tot_k2 * 1e-3) / 1e12:.0f} | "
      f"forward {tot_k1 + tot_k2:.3f} ms = {tot_ops / ((tot_k1 + tot_k2) * 1e-3) / 1e12:.0f} TOPS |")
