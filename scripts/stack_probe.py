"""Per-kernel device times of the config-3 stack (one block shown), from the event-node graph."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_21072_b200 import synth
from paper_2605_21072_b200.pipeline import wan_stack_chain

blocks = int(os.environ.get("BLOCKS", "4"))
ch = wan_stack_chain(blocks=blocks, fuse_rowmax=os.environ.get("FUSE", "0") == "1",
                     fuse_qkv=os.environ.get("FUSEQKV", "0") == "1")
ch.x.copy_(synth.synth_activation(ch.m, 1536, seed=11))
ch.ctx.copy_(synth.synth_activation(512, 1536, seed=13))
g = ch.capture(timed=True)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
kts = []
for _ in range(20):
    flush.fill_(1)
    g.replay()
    torch.cuda.synchronize()
    kts.append(ch.kernel_times_ms())
kt = np.mean(np.asarray(kts[3:]), axis=0) * 1e3
names = synth.BLOCK_LAYER_TYPES
b = blocks - 1
tot = 0
for i, t in enumerate(names if len(ch.layers) == 10 * blocks else []):
    li = b * 10 + i
    L = ch.layers[li]
    print(f"{t:14s} M={ch.ms[li]:5d} {L.in_dim:5d}->{L.out_dim:5d} Ko={L.k_outlier:3d} gather={L.gather_dev is not None!s:5s} "
          f"K1 {kt[2*li]:7.1f} us  K2 {kt[2*li+1]:7.1f} us  ({2*ch.ms[li]*L.in_dim*L.out_dim/kt[2*li+1]/1e6:6.0f} TOPS)")
    tot += kt[2 * li] + kt[2 * li + 1]
print(f"block total {tot:.1f} us; all blocks {kt.sum():.1f} us")
ch.capture(timed=False)
ts = []
for _ in range(10):
    flush.fill_(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ch.replay(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
print(f"plain graph {np.mean(ts[2:])*1e3:.1f} us for {blocks} blocks")

ch.capture(parallel=True)
ts = []
for _ in range(10):
    flush.fill_(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ch.replay(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
print(f"parallel graph {np.mean(ts[2:])*1e3:.1f} us for {blocks} blocks")
