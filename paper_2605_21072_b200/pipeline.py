"""Device-resident chains of quantized linears, replayed as one CUDA graph.

``QuantizedChain`` is the deployment form of a sequence of
``quantized_layer_forward`` calls (engine.cpp:134-142): for each layer K1
(per-token quantize + permutation) then K2 (dual-slab tcgen05 GEMM + fused
epilogue), with every intermediate buffer allocated once.  The whole forward
is captured into a CUDA graph so a step costs one graph launch instead of 2L
host-side kernel launches (the reference runs these as plain C++ calls,
engine.cpp:155-165; on the GPU the launch latency would otherwise exceed the
kernels themselves).
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib
from .engine import QuantizedLayer, _ptr, _stream


def _is_permutation(layer: QuantizedLayer) -> bool:
    """True when the layer's gather lists every input column exactly once (not the case for a
    fused sibling layer, whose gather repeats the outlier columns in their slabs)."""
    g = layer.plan.gather
    v = g[g >= 0]
    return len(v) == layer.in_dim and len(np.unique(v)) == layer.in_dim


def fold_output_permutation(producer: QuantizedLayer,
                            consumer: QuantizedLayer) -> Tuple[QuantizedLayer, QuantizedLayer]:
    """Make ``producer`` emit its outputs directly in ``consumer``'s plan order.

    The consumer's first step, permute_activations(y, plan) (engine.cpp:32-44), only
    reorders y's columns.  Reordering the producer's output channels -- its code rows,
    group scales and bias -- by the consumer's gather yields y already in plan order;
    pad slots get all-zero rows (codes, scales and bias 0), which produce exact zeros
    (GELU(0) = 0), the reference's zero pad columns.  The consumer's K1 then quantizes
    contiguous rows: same codes, same per-token scale (zeros do not move |x|max), and
    no gather.  Returns (producer', consumer'); the originals are left untouched.
    """
    g = consumer.gather_dev
    if g is None:
        return producer, consumer
    if producer.out_dim != consumer.in_dim:
        raise _lib.InvalidArgument("fold_output_permutation: producer width does not match the consumer")
    gl = g.long()
    valid = gl >= 0
    src = gl[valid]
    if src.numel() != consumer.in_dim or not torch.equal(
            torch.sort(src).values, torch.arange(consumer.in_dim, device=src.device)):
        raise _lib.InvalidArgument("fold_output_permutation: plan gather is not a permutation")
    n = consumer.k_pad

    def rows(t: Optional[torch.Tensor]) -> Optional[torch.Tensor]:
        if t is None:
            return None
        out = torch.zeros((n,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        out[valid] = t[src]
        return out

    prod = dataclasses.replace(
        producer, out_dim=n, wq=rows(producer.wq), scale_outlier64=rows(producer.scale_outlier64),
        scale_normal64=rows(producer.scale_normal64), scale_outlier32=rows(producer.scale_outlier32),
        scale_normal32=rows(producer.scale_normal32), bias=rows(producer.bias))
    cons = dataclasses.replace(consumer, in_dim=n, gather_dev=None)
    return prod, cons


class QuantizedChain:
    def __init__(self, layers: Sequence[QuantizedLayer], m: int,
                 epilogues: Optional[Sequence[int]] = None, inputs: Optional[Sequence[int]] = None,
                 fold: bool = True, fuse_rowmax: bool = False, ms: Optional[Sequence[int]] = None,
                 ctx_rows: int = 0, fuse_quant: bool = False):
        """layers[i] consumes the output of layer inputs[i] (-1 = the chain input; default i-1;
        -2 = the context input ``self.ctx`` of ``ctx_rows`` rows, e.g. the text tokens the
        cross-attention k / v projections read).  ``ms[i]`` = rows layer i processes (default m;
        a layer reading a producer must match its rows).

        With ``fold`` every intermediate consumed by exactly one layer is produced in that
        layer's plan order (fold_output_permutation), so its K1 runs without a gather.
        With ``fuse_rowmax`` a folded consumer's per-token |x| max comes from per-row partial
        maxima the producer's GEMM epilogue stores (qarvd_dual_gemm_pmax) and its K1 is a flat
        streaming pass (qarvd_quantize_act_pmax).
        With ``fuse_quant`` a folded per-token consumer of a single producer gets its codes and
        scales straight from the producer's epilogue (qarvd_dual_gemm_quant): the intermediate
        is never stored and the consumer's K1 launch disappears (``self.y`` of such a producer
        stays unwritten).
        ``self.source_ops`` keeps the unfolded shapes for op counting."""
        self.layers = list(layers)
        self.source_layers = list(layers)  # as given (before any output-permutation fold)
        self.m = m
        self.epilogues = list(epilogues) if epilogues is not None else [_lib.EPI_NONE] * len(layers)
        raw_inputs = list(inputs) if inputs is not None else list(range(-1, len(layers) - 1))
        # an input may be a column slice (producer, first column, width) of a producer's output,
        # e.g. the v part of a fused q/k/v layer (engine.fuse_siblings)
        self.inputs = [j[0] if isinstance(j, tuple) else j for j in raw_inputs]
        self.in_cols = [(j[1], j[2]) if isinstance(j, tuple) else None for j in raw_inputs]
        self.raw_inputs = raw_inputs
        self.ms = list(ms) if ms is not None else [m] * len(self.layers)
        for i, j in enumerate(self.inputs):
            want = m if j == -1 else (ctx_rows if j == -2 else self.ms[j])
            if self.ms[i] != want:
                raise _lib.InvalidArgument("QuantizedChain: layer rows do not match its input's rows")
        self.source_ops = float(sum(2.0 * mi * L.out_dim * L.in_dim for mi, L in zip(self.ms, self.layers)))
        if fold:
            for j, i in enumerate(self.inputs):
                if (i >= 0 and self.inputs.count(i) == 1 and self.in_cols[j] is None
                        and self.layers[j].gather_dev is not None and _is_permutation(self.layers[j])):
                    self.layers[i], self.layers[j] = fold_output_permutation(self.layers[i], self.layers[j])
        dev = self.layers[0].wq.device
        # A folded consumer of a single producer gets that producer's per-row |y| max from
        # the producer's epilogue (qarvd_dual_gemm_rowmax) and quantizes with the streaming
        # K1 (qarvd_quantize_act_rowmax), which also resets the buffer for the next step.
        self.rowmax = [None] * len(self.layers)  # indexed by producer
        self.stream_k1 = [False] * len(self.layers)  # indexed by consumer
        if fold:
            for j, i in enumerate(self.inputs):
                L = self.layers[j]
                if (i >= 0 and L.gather_dev is None and self.inputs.count(i) == 1 and fuse_rowmax
                        and self.in_cols[j] is None
                        and L.in_dim >= 512 and L.in_dim % 8 == 0):
                    self.stream_k1[j] = True
                    if L.act_granularity == _lib.ACT_PER_TOKEN:
                        P = self.layers[i]
                        pm = _lib.load().qarvd_dual_gemm_pmax_count(self.ms[i], P.out_dim, P.k_pad)
                        self.rowmax[i] = torch.zeros((self.ms[i], pm), dtype=torch.int32, device=dev)
        # fused consumer K1 (qarvd_dual_gemm_quant): producer i -> consumer j
        self.qz_into = [None] * len(self.layers)  # indexed by producer
        self.qz_from = [None] * len(self.layers)  # indexed by consumer
        self.qz_ws = [None] * len(self.layers)
        if fold and fuse_quant:
            for j, i in enumerate(self.inputs):
                L = self.layers[j]
                if (i >= 0 and not self.stream_k1[j] and self.rowmax[i] is None and L.gather_dev is None
                        and self.inputs.count(i) == 1 and self.in_cols[j] is None
                        and self.layers[i].out_dim % 256 == 0):
                    self.qz_into[i], self.qz_from[j] = j, i
                    nb = int(_lib.load().qarvd_dual_gemm_quant_workspace_size(self.ms[i]))
                    self.qz_ws[i] = torch.zeros(nb, dtype=torch.uint8, device=dev)
        first = {j: i for i, j in reversed(list(enumerate(self.inputs))) if j < 0}
        self.x = torch.empty((m, self.layers[first.get(-1, 0)].in_dim), dtype=torch.bfloat16, device=dev)
        self.ctx = (torch.empty((ctx_rows, self.layers[first[-2]].in_dim), dtype=torch.bfloat16, device=dev)
                    if -2 in first else None)
        # (zero-filled: a fused consumer's pad columns are never written)
        self.xq = [torch.zeros((mi, L.k_pad), dtype=torch.int8, device=dev) for mi, L in zip(self.ms, self.layers)]
        self.sx = [torch.empty(mi, dtype=torch.float32, device=dev) for mi in self.ms]
        self.y = [torch.empty((mi, L.out_dim), dtype=torch.bfloat16, device=dev) for mi, L in zip(self.ms, self.layers)]
        # stream-K workspaces (zero-filled; one per layer so concurrent branches never share)
        self.sk_ws = []
        for mi, L in zip(self.ms, self.layers):
            nb = int(_lib.load().qarvd_dual_gemm_workspace_size(mi, L.out_dim, L.k_pad, L.k_outlier))
            self.sk_ws.append(torch.zeros(nb, dtype=torch.uint8, device=dev) if nb > 0 else None)
        self.graph = None

    def _src(self, i):
        j = self.inputs[i]
        if j == -1:
            return self.x
        if j == -2:
            return self.ctx
        if self.in_cols[i] is not None:
            c0, w = self.in_cols[i]
            return self.y[j][:, c0:c0 + w]
        return self.y[j]

    def launch(self, stream: Optional[int] = None, events: Optional[List] = None):
        """Enqueue K1 + K2 for every layer (2 kernels per layer).  With ``events`` (a list of
        2L+1 timing events) an event is recorded before, between and after the kernels;
        recorded during capture they become graph nodes, so per-kernel device times come
        from the replayed step itself."""
        s = _stream() if stream is None else stream
        if events is not None:
            events[0].record()
        for i in range(len(self.layers)):
            self._enqueue(i, s, events)

    def launch_parallel(self):
        """launch() with the chain's dead-end layers (outputs consumed by no later layer, e.g.
        q / k and the cross-attention k / v of the Wan stack) forked onto two side streams:
        each waits only for its own producer (the context input needs none), so their
        kernels fill the SMs the critical path leaves idle.  Captured into a graph, the
        fork / join become graph edges."""
        main = torch.cuda.current_stream()
        if not hasattr(self, "_side"):
            self._side = [torch.cuda.Stream(device=main.device) for _ in range(2)]
        n = len(self.layers)
        side = {i for i in range(n - 1) if i not in self.inputs}
        wanted = {self.inputs[i] for i in side if self.inputs[i] >= 0}
        start = torch.cuda.Event()
        start.record(main)
        for st in self._side:
            st.wait_event(start)
        after, k = {}, 0
        for i in range(n):
            if i in side:
                st = self._side[k % len(self._side)]
                k += 1
                j = self.inputs[i]
                if j >= 0:
                    st.wait_event(after[j])
                self._enqueue(i, st.cuda_stream)
            else:
                self._enqueue(i, main.cuda_stream)
                if i in wanted:
                    after[i] = torch.cuda.Event()
                    after[i].record(main)
        for st in self._side:
            e = torch.cuda.Event()
            e.record(st)
            main.wait_event(e)

    def _enqueue(self, i: int, s: int, events: Optional[List] = None):
        """K1 + K2 of layer i on stream s."""
        L = self.layers[i]
        src = self._src(i)
        m = self.ms[i]
        if self.qz_from[i] is not None:
            pass  # codes and scales come from the producer's epilogue
        elif self.stream_k1[i]:
            rm = self.rowmax[self.inputs[i]]
            _lib.call("qarvd_quantize_act_pmax", src.data_ptr(), m, L.in_dim, src.stride(0),
                      _ptr(rm), 0 if rm is None else rm.shape[1], L.act_granularity,
                      float(L.act_scale), 8, self.xq[i].data_ptr(), L.k_pad, self.sx[i].data_ptr(),
                      None, None, s)
        else:
            _lib.call("qarvd_quantize_act", src.data_ptr(), _lib.BF16, m, L.in_dim,
                      src.stride(0), _ptr(L.gather_dev), L.k_pad, L.act_granularity,
                      float(L.act_scale), 8, self.xq[i].data_ptr(), L.k_pad, self.sx[i].data_ptr(),
                      None, None, s)
        if events is not None:
            events[2 * i + 1].record()
        if self.qz_into[i] is not None:
            j = self.qz_into[i]
            C = self.layers[j]
            ws = self.qz_ws[i]
            _lib.call("qarvd_dual_gemm_quant", self.xq[i].data_ptr(), L.k_pad, L.wq.data_ptr(), L.k_pad,
                      m, L.out_dim, L.k_pad, L.k_outlier, self.sx[i].data_ptr(),
                      L.scale_outlier32.data_ptr(), L.scale_normal32.data_ptr(), _ptr(L.bias),
                      self.epilogues[i], C.act_granularity, float(C.act_scale), 8, self.xq[j].data_ptr(),
                      C.k_pad, self.sx[j].data_ptr(), None, None, ws.data_ptr(), ws.numel(), s)
        elif self.rowmax[i] is not None:
            _lib.call("qarvd_dual_gemm_pmax", self.xq[i].data_ptr(), L.k_pad, L.wq.data_ptr(),
                      L.k_pad, m, L.out_dim, L.k_pad, L.k_outlier, self.sx[i].data_ptr(),
                      L.scale_outlier32.data_ptr(), L.scale_normal32.data_ptr(), _ptr(L.bias),
                      self.epilogues[i], self.y[i].data_ptr(), L.out_dim, self.rowmax[i].data_ptr(),
                      self.rowmax[i].shape[1], s)
        elif self.sk_ws[i] is not None:
            ws = self.sk_ws[i]
            _lib.call("qarvd_dual_gemm_ws", self.xq[i].data_ptr(), L.k_pad, L.wq.data_ptr(), L.k_pad,
                      m, L.out_dim, L.k_pad, L.k_outlier, self.sx[i].data_ptr(),
                      L.scale_outlier32.data_ptr(), L.scale_normal32.data_ptr(), _ptr(L.bias),
                      self.epilogues[i], self.y[i].data_ptr(), L.out_dim, ws.data_ptr(), ws.numel(), s)
        else:
            _lib.call("qarvd_dual_gemm", self.xq[i].data_ptr(), L.k_pad, L.wq.data_ptr(), L.k_pad,
                      m, L.out_dim, L.k_pad, L.k_outlier, self.sx[i].data_ptr(),
                      L.scale_outlier32.data_ptr(), L.scale_normal32.data_ptr(), _ptr(L.bias),
                      self.epilogues[i], _lib.BF16, self.y[i].data_ptr(), L.out_dim, None, None, s)
        if events is not None:
            events[2 * i + 2].record()

    def capture(self, timed: bool = False, parallel: bool = False):
        """Capture launch() into a CUDA graph (after one eager warm-up launch).  With
        ``timed`` the graph also records per-kernel timing events (``self.events``); with
        ``parallel`` the graph holds launch_parallel()'s side branches."""
        c0 = _lib.launch_count()
        self.launch()
        torch.cuda.synchronize()
        self._launches = _lib.launch_count() - c0  # K1 (+ its deferred tie repair) + K2 per layer
        if parallel:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.launch_parallel()
            torch.cuda.synchronize()
            self.graph = g
            return g
        self.events = ([torch.cuda.Event(enable_timing=True, external=True) for _ in range(2 * len(self.layers) + 1)]
                       if timed else None)  # kept by the caller with the returned graph
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.launch(events=self.events)
        torch.cuda.synchronize()
        self.graph = g
        return g

    def kernel_times_ms(self) -> List[float]:
        """Per-kernel device times [K1, K2] * L of the last replay (timed graphs only)."""
        e = self.events
        return [e[i].elapsed_time(e[i + 1]) for i in range(len(e) - 1)]

    def replay(self):
        if self.graph is None:
            self.capture()
        self.graph.replay()

    @property
    def output(self) -> torch.Tensor:
        return self.y[-1]

    def kernels_per_step(self) -> int:
        """Kernel launches of one step (counted on the eager launch before capture)."""
        return getattr(self, "_launches", 2 * len(self.layers))

    def int_ops(self) -> float:
        """Algorithmic ops of the chain as specified (unfolded shapes, no pad rows)."""
        return self.source_ops


def wan_stack_chain(blocks: int = 30, seed: int = 1, m: Optional[int] = None,
                    text_len: Optional[int] = None, fuse_rowmax: bool = False,
                    fuse_qkv: bool = False, fuse_quant: bool = False) -> "QuantizedChain":
    """BASELINE config 3: every quantized linear of a Wan-1.3B-shaped DiT stack for one chunk.

    Per block (toy_model.cpp:25-27 layer types, Wan2.1 shapes): self_attn.{q,k,v} read the
    block input; self_attn.o reads v's output; cross_attn.q reads o's; cross_attn.{k,v}
    read the 512 text tokens; cross_attn.o reads cross q's; ffn.0 (GELU fused) reads
    cross o's; ffn.2 reads ffn.0's and is the next block's input.  The attention, norm,
    modulation and residual glue between the linears is not on the quantized path (the
    reference's own f64 glue) and is elided: each linear still sees its real
    shape, its own outlier plan (K3 on its synthetic weight) and a real per-token K1.
    With ``fuse_qkv`` the three self-attention projections (and the two cross-attention k / v
    projections of the text tokens) run as one fused dual-slab layer each
    (engine.fuse_siblings: bit-identical per output column); o reads the v columns.
    """
    from . import engine, synth
    from .outlier import analyze_layer

    specs = synth.wan_registry(blocks=blocks)
    m = synth.WAN_CHUNK_TOKENS if m is None else m
    text_len = synth.WAN_TEXT_LEN if text_len is None else text_len
    layers, inputs, epis, ms = [], [], [], []
    block_in = -1
    qkv_types = ("self_attn.q", "self_attn.k", "self_attn.v")
    for b in range(blocks):
        built = {}
        for i, t in enumerate(synth.BLOCK_LAYER_TYPES):
            spec = specs[b * len(synth.BLOCK_LAYER_TYPES) + i]
            w = synth.synth_weight(spec, seed=seed)
            rep = analyze_layer(spec.name, w)
            plan = engine.build_plan(spec.name, spec.in_dim, rep.aligned_outliers)
            built[t] = engine.prepare_weights(spec.name, w, plan)
            del w
        order = list(synth.BLOCK_LAYER_TYPES)
        if fuse_qkv:
            built["self_attn.qkv"] = engine.fuse_siblings(f"block{b}.self_attn.qkv", [built[t] for t in qkv_types])
            built["cross_attn.kv"] = engine.fuse_siblings(f"block{b}.cross_attn.kv",
                                                          [built["cross_attn.k"], built["cross_attn.v"]])
            order = ["self_attn.qkv"] + [t for t in order if t not in qkv_types + ("cross_attn.k", "cross_attn.v")]
            order.insert(order.index("cross_attn.o"), "cross_attn.kv")
        base = len(layers)
        idx = {t: base + i for i, t in enumerate(order)}
        d = synth.WAN_DIM
        src = {"self_attn.q": block_in, "self_attn.k": block_in, "self_attn.v": block_in,
               "self_attn.qkv": block_in,
               "self_attn.o": (idx["self_attn.qkv"], 2 * d, d) if fuse_qkv else idx["self_attn.v"],
               "cross_attn.q": idx["self_attn.o"], "cross_attn.k": -2, "cross_attn.v": -2, "cross_attn.kv": -2,
               "cross_attn.o": idx["cross_attn.q"], "ffn.0": idx["cross_attn.o"], "ffn.2": idx["ffn.0"]}
        for t in order:
            layers.append(built[t])
            inputs.append(src[t])
            epis.append(_lib.EPI_GELU if t == "ffn.0" else _lib.EPI_NONE)
            ms.append(text_len if src[t] == -2 else m)
        block_in = idx["ffn.2"]
    return QuantizedChain(layers, m, epilogues=epis, inputs=inputs, ms=ms, ctx_rows=text_len,
                          fuse_rowmax=fuse_rowmax, fuse_quant=fuse_quant)
