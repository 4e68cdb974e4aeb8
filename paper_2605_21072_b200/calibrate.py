"""Frame-weighted calibration scale search and its layer-sharded driver.

Reference pieces (``/root/reference/proj/core``):

* ``weighting_strategy`` / ``normalize_alpha``   sensitivity.cpp:16-27, :86-112
* ``init_scale_percentile_search``               quant.cpp:185-226
* ``calibrate_model``'s per-layer loop           calibrate.cpp:398-487
  (``parallel_for`` over quantized layers, slot-indexed results, :432-484)

The per-layer unit of ``calibrate_model`` becomes: K3 outlier detection ->
K5 dual-scale weight prep -> K4 frame-weighted activation-scale search, all on
the device.  Across GPUs the layers are split by a deterministic LPT
assignment on algorithmic bytes; each rank runs its layers independently and
one all-gather of packed per-layer records gives every rank the full,
rank-count-invariant result (the reference's thread-count invariance,
threading.hpp:13-14, lifted to GPU count).
"""
from __future__ import annotations

import ctypes
import heapq
import os
from dataclasses import dataclass
from typing import Callable, Dict, List, Optional, Sequence

import numpy as np
import torch

from . import _lib
from .engine import _stream

PERCENTILES = (0.999, 0.9999, 0.99999)  # quant.cpp:185-188
WEIGHTING_KINDS = ("uniform", "heuristic_exp", "reverse", "final_quality")  # sensitivity.hpp:37


def normalize_alpha(raw: Sequence[float]) -> np.ndarray:
    """sensitivity.cpp:16-27 (same f64 op order)."""
    total = 0.0
    for a in raw:
        total += float(a)
    if total <= 0.0:
        return np.full(len(raw), 1.0 / len(raw))
    return np.asarray([float(a) / total for a in raw])


def weighting_strategy(kind: str, n: int, alpha_raw: Optional[Sequence[float]] = None) -> np.ndarray:
    """weighting_strategy (sensitivity.cpp:86-112) for an N-entry profile."""
    if n <= 0:
        raise _lib.InvalidArgument("weighting_strategy: empty profile")
    if kind == "uniform":
        return np.full(n, 1.0 / n)
    if kind == "heuristic_exp":
        w = [2.0 ** -(i + 1) for i in range(n)]
        total = 0.0
        for v in w:
            total += v
        return np.asarray([v / total for v in w])
    if alpha_raw is None or len(alpha_raw) != n:
        raise _lib.InvalidArgument("weighting_strategy: profile required for " + kind)
    a = normalize_alpha(alpha_raw)
    if kind == "reverse":
        return a[::-1].copy()
    if kind == "final_quality":
        return a
    raise _lib.InvalidArgument("unknown weighting kind: " + kind)


@dataclass
class SearchResult:
    """PercentileSearchResult (quant.hpp:72-77) + thresholds and the frame-weighted losses."""

    thresholds: np.ndarray
    scales: np.ndarray
    losses: np.ndarray
    best_index: int
    scale: float
    percentiles: tuple

    @property
    def best_percentile(self) -> float:
        return self.percentiles[self.best_index]


def scale_search_async(xs: Sequence[torch.Tensor], frames: int, frame_weights=None,
                       percentiles=PERCENTILES, bits: int = 8,
                       nonfinite_flag: Optional[torch.Tensor] = None) -> torch.Tensor:
    """K4 over a batch of layers.  xs[i]: bf16 [frames*rows x k].  Returns the device result
    matrix [len(xs), 3*nc+2] (thresholds, scales, losses, best index, best scale)."""
    nc = len(percentiles)
    res = torch.empty((len(xs), 3 * nc + 2), dtype=torch.float64, device=xs[0].device)
    jobs = (_lib.SearchJob * len(xs))()
    for i, x in enumerate(xs):
        if x.dtype != torch.bfloat16:
            raise _lib.InvalidArgument("scale_search: activations must be bf16")
        if x.shape[0] % frames:
            raise _lib.InvalidArgument("scale_search: rows not divisible by the frame count")
        jobs[i].x = x.data_ptr()
        jobs[i].frames = frames
        jobs[i].rows = x.shape[0] // frames
        jobs[i].k = x.shape[1]
        jobs[i].ldx = x.stride(0)
        jobs[i].result = res[i].data_ptr()
    pct = (_lib.ctypes.c_double * nc)(*percentiles)
    w = None
    if frame_weights is not None:
        if len(frame_weights) != frames:
            raise _lib.InvalidArgument("calibrate_model: weight vector length must equal chunk count")
        w = (_lib.ctypes.c_double * frames)(*[float(v) for v in frame_weights])
    if nonfinite_flag is None:  # synchronous: raises on non-finite samples
        _lib.call("qarvd_scale_search", jobs, len(xs), pct, nc, w, bits, _stream())
    else:  # the caller checks nonfinite_flag (int64, -1 = all finite) after its own sync
        _lib.call("qarvd_scale_search_async", jobs, len(xs), pct, nc, w, bits,
                  nonfinite_flag.data_ptr(), _stream())
    return res


def unpack_search(row: np.ndarray, percentiles=PERCENTILES) -> SearchResult:
    nc = len(percentiles)
    return SearchResult(row[:nc].copy(), row[nc:2 * nc].copy(), row[2 * nc:3 * nc].copy(),
                        int(row[3 * nc]), float(row[3 * nc + 1]), tuple(percentiles))


def init_scale_percentile_search(frames: Sequence[torch.Tensor], bits: int = 8,
                                 frame_weights=None) -> SearchResult:
    """init_scale_percentile_search(samples, bits) (quant.cpp:190-226); with ``frame_weights``
    the per-sample MSEs are weighted (Eq. 5 frame weights)."""
    if len(frames) == 0:
        raise _lib.InvalidArgument("percentile search: empty calibration sample list")
    shapes = {tuple(f.shape) for f in frames}
    if len(shapes) != 1:
        raise _lib.Unsupported("scale_search: samples of different shapes")
    x = torch.cat([f.reshape(-1, f.shape[-1]) for f in frames], 0)
    res = scale_search_async([x], len(frames), frame_weights, PERCENTILES, bits)
    return unpack_search(res[0].cpu().numpy())


# ---------------------------------------------------------------------------
# layer sharding (calibrate.cpp:440-484 -> G GPUs)

def lpt_assign(costs: Sequence[float], world: int) -> List[List[int]]:
    """Deterministic longest-processing-time assignment: layers sorted by cost desc
    (ties -> lower index), each to the least-loaded rank (ties -> lower rank).
    Each rank's list is returned in ascending layer order."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    heap = [(0.0, r) for r in range(world)]
    heapq.heapify(heap)
    out: List[List[int]] = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + costs[i], r))
    return [sorted(v) for v in out]


@dataclass
class LayerRecord:
    """Everything the quantized deployment needs from calibration for one layer."""

    index: int
    k_outlier: int            # aligned outlier count (reference K_o)
    outliers: np.ndarray      # aligned outlier indices (ascending)
    act_scale: float          # selected per-tensor activation scale
    best_index: int
    losses: np.ndarray
    scale_outlier: np.ndarray  # f64 [out_dim]
    scale_normal: np.ndarray   # f64 [out_dim]

    def pack(self) -> np.ndarray:
        n = len(self.scale_normal)
        head = [float(self.index), float(n), float(len(self.outliers)), float(len(self.losses)),
                self.act_scale, float(self.best_index)]
        return np.concatenate([np.asarray(head), self.losses, self.scale_outlier,
                               self.scale_normal, self.outliers.astype(np.float64)])

    @staticmethod
    def unpack(buf: np.ndarray, pos: int):
        idx, n, no, nl, act, best = buf[pos:pos + 6]
        n, no, nl = int(n), int(no), int(nl)
        p = pos + 6
        losses = buf[p:p + nl].copy(); p += nl
        so = buf[p:p + n].copy(); p += n
        sn = buf[p:p + n].copy(); p += n
        outl = buf[p:p + no].astype(np.int64); p += no
        return LayerRecord(int(idx), no, outl, float(act), int(best), losses, so, sn), p


def pack_records(records: Sequence[LayerRecord]) -> np.ndarray:
    if not records:
        return np.zeros(0, dtype=np.float64)
    return np.concatenate([r.pack() for r in records])


def unpack_records(buf: np.ndarray) -> List[LayerRecord]:
    out, pos = [], 0
    while pos < len(buf):
        r, pos = LayerRecord.unpack(buf, pos)
        out.append(r)
    return out


def allgather_bytes(payload: np.ndarray, group=None, device=None) -> List[np.ndarray]:
    """One all-gather of a per-rank byte payload (NCCL on GPU, gloo on CPU): the sizes first,
    then the payloads padded to the largest.  Returns every rank's bytes, in rank order."""
    import torch.distributed as dist

    payload = np.ascontiguousarray(payload).view(np.uint8).reshape(-1)
    dev = device if device is not None else torch.device("cpu")
    world = dist.get_world_size(group)
    size = torch.tensor([payload.size], dtype=torch.int64, device=dev)
    sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(sizes, size, group=group)
    sizes = [int(s.item()) for s in sizes]
    cap = max(max(sizes), 8)
    buf = torch.zeros(cap, dtype=torch.uint8, device=dev)
    buf[:payload.size] = torch.from_numpy(payload.copy()).to(dev)
    gathered = torch.empty(world * cap, dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(gathered, buf, group=group)
    g = gathered.cpu().numpy()
    return [g[r * cap: r * cap + sizes[r]].copy() for r in range(world)]


def allgather_records(local: Sequence, group=None, device=None, unpack=None) -> List:
    """All-gather of packed per-layer records (``LayerRecord`` by default; any record with
    ``.index`` and ``.pack()`` plus its ``unpack`` over the concatenated bytes), sorted by
    layer index."""
    unpack = unpack if unpack is not None else (lambda b: unpack_records(b.view(np.float64)))
    payload = (np.concatenate([np.ascontiguousarray(r.pack()).view(np.uint8) for r in local])
               if local else np.zeros(0, dtype=np.uint8))
    recs: List = []
    for b in allgather_bytes(payload, group=group, device=device):
        recs.extend(unpack(b))
    recs.sort(key=lambda r: r.index)
    return recs


def calibrate_model_sharded(costs: Sequence[float], compute: Callable[[List[int]], List],
                            rank: int = 0, world: int = 1, group=None, device=None,
                            unpack=None) -> List:
    """calibrate_model's layer loop (calibrate.cpp:440-484) over `world` ranks.

    ``compute(layer_ids)`` runs this rank's layers (on its GPU) and returns their
    records; one all-gather assembles the full result.  The output is identical
    for every world size (slot-indexed by layer, as the reference's parallel_for).
    ``unpack`` selects the record type (default ``LayerRecord``; ``unpack_calib_records``
    for the AdaRound results of ``calibrate_model_adaround``)."""
    assign = lpt_assign(costs, world)
    local = compute(assign[rank]) if assign[rank] else []
    if world == 1:
        return sorted(local, key=lambda r: r.index)
    return allgather_records(local, group=group, device=device, unpack=unpack)


# ---------------------------------------------------------------------------
# config 4: the per-layer calibration unit on the device, for a shard of the Wan registry

def layer_cost_bytes(spec, frames: int, rows: int) -> float:
    """Algorithmic bytes of one layer's calibration unit: one read of X, one read of W,
    one int8 code write."""
    return float(frames * rows * spec.in_dim * 2 + spec.out_dim * spec.in_dim * 2 +
                 spec.out_dim * spec.in_dim)


class CalibrationShard:
    """Device-resident calibration inputs of this rank's layers and the K3 -> K5 -> K4 unit.

    ``setup()`` materialises W (bf16) and the per-frame activations X (bf16,
    frames x rows tokens) with the counter-based generator, keyed only by
    (seed, layer), so every rank produces the same data for a layer whatever
    the world size.  ``run()`` is the timed calibration step."""

    def __init__(self, specs, layer_ids, frames: int = 21, rows: int = 1560, seed: int = 1,
                 frame_weights=None, device="cuda"):
        self.specs = [specs[i] for i in layer_ids]
        self.ids = list(layer_ids)
        self.frames, self.rows, self.seed = frames, rows, seed
        self.weights = frame_weights
        self.device = device
        self.w, self.x = [], []

    def setup(self):
        from . import synth
        for spec in self.specs:
            self.w.append(synth.synth_weight(spec, seed=self.seed, device=self.device))
            # cross-attn k/v see the 512 text tokens, identical for every frame
            rows = self.rows if spec.tokens != synth.WAN_TEXT_LEN else synth.WAN_TEXT_LEN
            x = torch.empty((self.frames * rows, spec.in_dim), dtype=torch.bfloat16,
                            device=self.device)
            for f in range(self.frames):
                synth.synth_activation(rows, spec.in_dim, seed=synth.mix_seed(self.seed, spec.index),
                                       frame=f, device=self.device, out=x[f * rows:(f + 1) * rows])
            self.x.append(x)
        torch.cuda.synchronize()

    def bytes(self) -> float:
        return float(sum(x.numel() * 2 for x in self.x) + sum(w.numel() * 3 for w in self.w))

    def _prepare_buffers(self):
        """Device buffers and launch tables of the sync-free step (allocated once)."""
        from . import outlier
        dev = self.x[0].device
        L = len(self.specs)
        self._rep = outlier.analyze_layers_async([s.name for s in self.specs], self.w)
        caps = [(s.in_dim + 64 + 15) // 16 * 16 for s in self.specs]
        goff = np.concatenate([[0], np.cumsum(caps)]).astype(np.int64)
        noff = np.concatenate([[0], np.cumsum([s.out_dim for s in self.specs])]).astype(np.int64)
        self._caps, self._noff = caps, noff
        self._gather = torch.empty(int(goff[-1]), dtype=torch.int32, device=dev)
        self._plan_info = torch.empty((L, 2), dtype=torch.int64, device=dev)
        self._wq = [torch.empty((s.out_dim, c), dtype=torch.int8, device=dev) for s, c in zip(self.specs, caps)]
        self._so64 = torch.empty(int(noff[-1]), dtype=torch.float64, device=dev)
        self._sn64 = torch.empty_like(self._so64)
        self._so32 = torch.empty(int(noff[-1]), dtype=torch.float32, device=dev)
        self._sn32 = torch.empty_like(self._so32)
        jobs = (_lib.PlannedWeightJob * L)()
        rep = self._rep
        for i, (spec, w) in enumerate(zip(self.specs, self.w)):
            j = jobs[i]
            o = int(rep.offsets[i])
            j.w, j.n, j.k, j.ldw = w.data_ptr(), w.shape[0], w.shape[1], w.stride(0)
            j.aligned_idx = rep.aligned.data_ptr() + 4 * o
            j.counts = rep.counts.data_ptr() + 8 * i
            j.gather, j.gather_cap = self._gather.data_ptr() + 4 * int(goff[i]), caps[i]
            j.plan_info = self._plan_info.data_ptr() + 16 * i
            j.wq, j.ldq = self._wq[i].data_ptr(), caps[i]
            sl = int(noff[i])
            j.scale_outlier_f64, j.scale_normal_f64 = self._so64.data_ptr() + 8 * sl, self._sn64.data_ptr() + 8 * sl
            j.scale_outlier_f32, j.scale_normal_f32 = self._so32.data_ptr() + 4 * sl, self._sn32.data_ptr() + 4 * sl
        self._jobs = jobs
        groups = {}
        for i, x in enumerate(self.x):
            groups.setdefault(x.shape[0] // self.frames, []).append(i)
        self._groups = groups
        self._side = torch.cuda.Stream(device=dev)
        self._flags = torch.empty(len(groups), dtype=torch.int64, device=dev)

    def run(self) -> List[LayerRecord]:
        """One calibration step, host-sync free until the results come back: K3 -> device plan
        -> K5 on the current stream, K4 (histogram search) on a side stream, one gather of the
        results at the end."""
        from . import outlier
        if not self.specs:
            return []
        if not hasattr(self, "_jobs"):
            self._prepare_buffers()
        main = torch.cuda.current_stream()
        self._side.wait_stream(main)
        if not hasattr(self, "_k4"):  # launch tables of the K4 groups, built once
            nc = len(PERCENTILES)
            self._k4 = []
            for g, (rows, idx) in enumerate(self._groups.items()):
                res = torch.empty((len(idx), 3 * nc + 2), dtype=torch.float64, device=self.x[0].device)
                jobs = (_lib.SearchJob * len(idx))()
                for j, i in enumerate(idx):
                    x = self.x[i]
                    jobs[j].x, jobs[j].frames, jobs[j].rows = x.data_ptr(), self.frames, x.shape[0] // self.frames
                    jobs[j].k, jobs[j].ldx, jobs[j].result = x.shape[1], x.stride(0), res[j].data_ptr()
                pct = (_lib.ctypes.c_double * nc)(*PERCENTILES)
                w = (None if self.weights is None else
                     (_lib.ctypes.c_double * self.frames)(*[float(v) for v in self.weights]))
                self._k4.append((jobs, len(idx), pct, nc, w, res))
        search = {}
        # launch order of the two streams' work (QARVD_CALIB_ORDER=hist_first / k3_first): after
        # round 2's faster K3 / K5, K3 -> plan -> K5 first measures 15.0-15.1 ms per step against
        # 15.5 ms with the histogram pass first
        hist_first = os.environ.get("QARVD_CALIB_ORDER", "k3_first") == "hist_first"

        def k4():
            with torch.cuda.stream(self._side):
                for g, (jobs, nj, pct, nc, w, res) in enumerate(self._k4):
                    _lib.call("qarvd_scale_search_async", jobs, nj, pct, nc, w, 8,
                              self._flags[g:g + 1].data_ptr(), _stream())
                    search[g] = res
        # The K4 histogram pass (one 128 KB-smem CTA per SM, shared-memory-atomic bound) and
        # K3 -> plan -> K5 share the SMs; whichever is enqueued first gets them first
        if hist_first:
            k4()
        rep = outlier.analyze_layers_async([s.name for s in self.specs], self.w, out=self._rep)
        _lib.call("qarvd_prepare_weights_planned", self._jobs, len(self.specs), 8, None, _stream())
        if not hist_first:
            k4()
        main.wait_stream(self._side)
        # results: every field into one pinned host buffer with async copies, one sync
        if not hasattr(self, "_pin"):
            self._pin = {
                "search": [torch.empty(search[g].shape, dtype=search[g].dtype).pin_memory()
                           for g in range(len(self._groups))],
                "flags": torch.empty(self._flags.shape, dtype=torch.int64).pin_memory(),
                "counts": torch.empty(rep.counts.shape, dtype=torch.int32).pin_memory(),
                "aligned": torch.empty(rep.aligned.shape, dtype=torch.int32).pin_memory(),
                "so": torch.empty(self._so64.shape, dtype=torch.float64).pin_memory(),
                "sn": torch.empty(self._sn64.shape, dtype=torch.float64).pin_memory(),
            }
        pin = self._pin
        for g in range(len(self._groups)):
            pin["search"][g].copy_(search[g], non_blocking=True)
        pin["flags"].copy_(self._flags, non_blocking=True)
        pin["counts"].copy_(rep.counts, non_blocking=True)
        pin["aligned"].copy_(rep.aligned, non_blocking=True)
        pin["so"].copy_(self._so64, non_blocking=True)
        pin["sn"].copy_(self._sn64, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        if (pin["flags"].numpy() != -1).any():
            raise _lib.InvalidArgument("quantize: non-finite input in calibration samples")
        search_host = {}
        for g, (rows, idx) in enumerate(self._groups.items()):
            mat = pin["search"][g].numpy()
            for j, i in enumerate(idx):
                search_host[i] = mat[j]
        counts = pin["counts"].numpy()
        aligned = pin["aligned"].numpy()
        so_all = pin["so"].numpy()
        sn_all = pin["sn"].numpy()
        out = []
        nc = len(PERCENTILES)
        for i, spec in enumerate(self.specs):
            r = search_host[i]
            o = int(rep.offsets[i])
            outl = aligned[o:o + counts[i, 1]].astype(np.int64)
            s0, s1 = int(self._noff[i]), int(self._noff[i + 1])
            out.append(LayerRecord(spec.index, len(outl), outl, float(r[3 * nc + 1]), int(r[3 * nc]),
                                   r[2 * nc:3 * nc].copy(), so_all[s0:s1].copy(), sn_all[s0:s1].copy()))
        return out

    def deployed_layers(self):
        """QuantizedLayer views of the last run() (plans rebuilt on the host; not timed)."""
        from . import engine, outlier
        reps = outlier.collect_reports(self._rep)
        info = self._plan_info.cpu().numpy()
        layers = []
        for i, (spec, rep) in enumerate(zip(self.specs, reps)):
            plan = engine.build_plan(spec.name, spec.in_dim, rep.aligned_outliers)
            assert plan.k_outlier == info[i, 0] and plan.k_pad == info[i, 1]
            s0, s1 = int(self._noff[i]), int(self._noff[i + 1])
            layers.append(engine.QuantizedLayer(
                spec.name, spec.out_dim, spec.in_dim, plan, self._wq[i][:, :plan.k_pad].contiguous(),
                self._so64[s0:s1], self._sn64[s0:s1], self._so32[s0:s1], self._sn32[s0:s1],
                torch.from_numpy(plan.gather).to(self._wq[i].device)))
        return layers


def weighted_loss(batch: Sequence, layer, w: torch.Tensor, chunk_weights: Sequence[float],
                  act_scale: float, return_errors: bool = False):
    """Eq. 5 on the GPU: weighted_loss(batch, state, chunk_weights) (calibrate.cpp:201-224).

    ``batch`` holds (x, chunk) pairs: a calibration sample's bf16 activations [rows x k] on the
    device (CalibSample.x, calibrate.hpp:37-41) and its 1-based chunk.  The state is the
    deployable layer (``layer``: plan-order int8 codes and f32 group scales; see
    engine.layer_from_codes for learned codes), its FP weight ``w`` (bf16 [n x k], original
    order) and the per-tensor activation scale (LearnableQuantState::act_params).
    K1 quantizes the stacked samples with the static scale, then one qarvd_weighted_loss call
    evaluates every sample's ||X W^T - FQ(X) What^T||_F^2 and the weighted mean.
    """
    from .engine import kernel_a_quantize_activation
    if len(batch) == 0:
        raise _lib.InvalidArgument("weighted loss: empty batch")
    xs = [x for x, _ in batch]
    chunks = np.asarray([int(c) for _, c in batch], dtype=np.int64)
    rows = np.zeros(len(xs) + 1, dtype=np.int64)
    rows[1:] = np.cumsum([x.shape[0] for x in xs])
    x = xs[0] if len(xs) == 1 else torch.cat(xs, 0)
    x = x.contiguous()
    xq, s32, _ = kernel_a_quantize_activation(x, layer, _lib.ACT_PER_TENSOR, static_scale=float(act_scale))
    m, k = x.shape
    n = layer.out_dim
    cw = np.ascontiguousarray(chunk_weights, dtype=np.float64)
    ws_bytes = int(_lib.load().qarvd_weighted_loss_workspace(m, n, len(xs)))
    ws = torch.empty(max(8, ws_bytes) // 8, dtype=torch.float64, device=x.device)
    err = torch.empty(len(xs), dtype=torch.float64, device=x.device)
    loss = torch.empty(1, dtype=torch.float64, device=x.device)
    _lib.call("qarvd_weighted_loss", x.data_ptr(), x.stride(0), w.data_ptr(), w.stride(0),
              xq.data_ptr(), xq.stride(0), layer.wq.data_ptr(), layer.wq.stride(0), m, n, k,
              layer.k_pad, layer.k_outlier, s32.data_ptr(), layer.scale_outlier32.data_ptr(),
              layer.scale_normal32.data_ptr(), rows.ctypes.data, chunks.ctypes.data, len(xs),
              cw.ctypes.data, len(cw), err.data_ptr(), loss.data_ptr(), ws.data_ptr(), ws_bytes, _stream())
    if return_errors:
        return float(loss.item()), err.cpu().numpy()
    return float(loss.item())


@dataclass
class LayerCalibResult:
    """LayerCalibResult (calibrate.hpp:102-110): learned plan scales, hard codes (original
    column order), the learned per-tensor activation scale, losses and the running-min trace."""

    layer: str
    scale_normal: np.ndarray
    scale_outlier: np.ndarray
    codes: np.ndarray
    act_scale: float
    initial_loss: float
    final_loss: float
    trace: np.ndarray


def calibrate_layer(name: str, w: torch.Tensor, plan, scale_normal: torch.Tensor,
                    scale_outlier: torch.Tensor, act_scale: float, samples: Sequence,
                    chunk_weights: Sequence[float], cfg: Optional["_lib.CalibConfig"] = None,
                    act_bits: int = 8, w_bits: int = 8) -> LayerCalibResult:
    """calibrate_layer (calibrate.cpp:298-396) on the GPU (K7, f64): AdaRound rounding variables,
    learned group and activation scales, frame-weighted Eq. 5 objective, Adam + cosine LR.

    ``w``: the layer's FP weight [n x k] (any float dtype; computed in f64). ``plan``: an
    engine.DualScalePlan; ``scale_normal`` / ``scale_outlier``: its initial per-row group scales
    (e.g. prepare_weights' scale_*64, bit-identical to build_plan). ``samples``: (x [rows x k],
    chunk) pairs (CalibSample, calibrate.hpp:37-41)."""
    cfg = cfg if cfg is not None else _lib.CalibConfig()
    if len(samples) == 0:
        raise _lib.InvalidArgument("calibrate_layer: no calibration samples")
    dev = w.device
    w64 = w.to(torch.float64).contiguous()
    n, k = w64.shape
    x64 = torch.cat([x.to(torch.float64) for x, _ in samples], 0).contiguous()
    rows = np.zeros(len(samples) + 1, dtype=np.int64)
    rows[1:] = np.cumsum([x.shape[0] for x, _ in samples])
    chunks = np.asarray([int(c) for _, c in samples], dtype=np.int64)
    cw = np.ascontiguousarray(chunk_weights, dtype=np.float64)
    mask = np.zeros(k, dtype=np.uint8)
    if plan.enabled:
        mask[np.asarray(plan.outlier_indices, dtype=np.int64)] = 1
    mask_d = torch.from_numpy(mask).to(dev)
    sn = scale_normal.to(torch.float64).contiguous()
    so = scale_outlier.to(torch.float64).contiguous()
    codes = torch.empty((n, k), dtype=torch.int8, device=dev)
    sn_out = torch.empty(n, dtype=torch.float64, device=dev)
    so_out = torch.empty(n, dtype=torch.float64, device=dev)
    scal = torch.empty(3, dtype=torch.float64, device=dev)
    trace = torch.empty(max(1, cfg.iterations), dtype=torch.float64, device=dev)
    _lib.call("qarvd_calibrate_layer", w64.data_ptr(), n, k, mask_d.data_ptr(), int(plan.enabled),
              sn.data_ptr(), so.data_ptr(), float(act_scale), act_bits, w_bits, x64.data_ptr(),
              rows.ctypes.data, chunks.ctypes.data, len(samples), cw.ctypes.data, len(cw),
              ctypes.byref(cfg), name.encode(), codes.data_ptr(), sn_out.data_ptr(), so_out.data_ptr(),
              scal.data_ptr(), trace.data_ptr(), _stream())
    sc = scal.cpu().numpy()
    return LayerCalibResult(name, sn_out.cpu().numpy(), so_out.cpu().numpy(), codes.cpu().numpy(),
                            float(sc[0]), float(sc[1]), float(sc[2]), trace.cpu().numpy()[:cfg.iterations])


# ---------------------------------------------------------------------------
# calibrate_model with AdaRound per layer, sharded over ranks (calibrate.cpp:440-484)

@dataclass
class CalibRecord:
    """One quantized layer's AdaRound result (LayerCalibResult) under its registry slot, as
    it travels in the all-gather: a little-endian byte record
    [i64 index, n, k, trace_len, name_len | f64 act_scale, initial, final | f64 scale_normal[n] |
    f64 scale_outlier[n] | f64 trace | i8 codes[n*k] | name | pad to 8]."""

    index: int
    result: LayerCalibResult

    def pack(self) -> np.ndarray:
        r = self.result
        n, k = r.codes.shape
        name = r.layer.encode()
        head = np.asarray([self.index, n, k, len(r.trace), len(name)], dtype="<i8")
        f = np.concatenate([np.asarray([r.act_scale, r.initial_loss, r.final_loss]),
                            r.scale_normal, r.scale_outlier, r.trace]).astype("<f8")
        body = b"".join([head.tobytes(), f.tobytes(), np.ascontiguousarray(r.codes, dtype=np.int8).tobytes(),
                         name])
        return np.frombuffer(body + b"\0" * (-len(body) % 8), dtype=np.uint8)

    @staticmethod
    def unpack(buf: np.ndarray, pos: int):
        idx, n, k, nt, nl = (int(v) for v in np.frombuffer(buf, dtype="<i8", count=5, offset=pos))
        p = pos + 40
        f = np.frombuffer(buf, dtype="<f8", count=3 + 2 * n + nt, offset=p).copy()
        p += 8 * len(f)
        codes = np.frombuffer(buf, dtype=np.int8, count=n * k, offset=p).reshape(n, k).copy()
        p += n * k
        name = bytes(buf[p:p + nl]).decode()
        p += nl
        p += -(p - pos) % 8
        res = LayerCalibResult(name, f[3:3 + n], f[3 + n:3 + 2 * n], codes, float(f[0]), float(f[1]),
                               float(f[2]), f[3 + 2 * n:])
        return CalibRecord(idx, res), p


def unpack_calib_records(buf: np.ndarray) -> List[CalibRecord]:
    buf = np.ascontiguousarray(buf).view(np.uint8)
    out, pos = [], 0
    while pos < len(buf):
        r, pos = CalibRecord.unpack(buf, pos)
        out.append(r)
    return out


def adaround_cost(n: int, k: int, rows: int, iterations: int) -> float:
    """LPT weight of one layer's AdaRound: its f64 GEMM work, iterations x rows x n x k (the
    forward X.W_soft^T and the weight gradient X^T.E dominate K7)."""
    return float(max(1, iterations)) * rows * n * k


def calibrate_model_adaround(layers: Sequence, samples_of: Callable[[int], Sequence],
                             chunk_weights: Sequence[float], cfg: Optional["_lib.CalibConfig"] = None,
                             rank: int = 0, world: int = 1, group=None, device=None,
                             act_bits: int = 8, w_bits: int = 8,
                             sample_rows: Optional[Sequence[int]] = None) -> List[CalibRecord]:
    """calibrate_model's AdaRound loop (calibrate.cpp:440-484: calibrate_layer per quantized
    layer, independent across layers) over ``world`` GPUs: LPT on ``adaround_cost``, each rank
    runs K7 for its layers, one all-gather of the codes, learned scales and traces.

    ``layers[i]``: (name, w [n x k] device tensor, plan, scale_normal, scale_outlier, act_scale)
    — the inputs of calibrate_layer; ``samples_of(i)``: that layer's (x, chunk) samples on this
    rank's device, called only for this rank's layers; ``sample_rows[i]``: its total sample rows
    for the LPT weights (default: equal).  Identical result for every world size (slot-indexed as the reference's
    parallel_for; K7 is deterministic per layer)."""
    cfg = cfg if cfg is not None else _lib.CalibConfig()
    costs = []
    for i, L in enumerate(layers):
        n, k = L[1].shape
        rows = int(sample_rows[i]) if sample_rows is not None else 1
        costs.append(adaround_cost(n, k, rows, cfg.iterations))

    def compute(ids):
        out = []
        for i in ids:
            name, w, plan, sn, so, act = layers[i]
            out.append(CalibRecord(i, calibrate_layer(name, w, plan, sn, so, act, samples_of(i),
                                                      chunk_weights, cfg, act_bits, w_bits)))
        return out

    return calibrate_model_sharded(costs, compute, rank, world, group=group, device=device,
                                   unpack=unpack_calib_records)


# ---------------------------------------------------------------------------
# the C++ multi-GPU driver (qarvd_calibrate_sharded): the same calibration unit and records,
# one host thread per rank, NCCL all-gather of the packed records

def synth_descriptors(spec, frames: int, rows: int, seed: int = 1):
    """qarvd_calib_layer inputs reproducing CalibrationShard.setup()'s synthetic data exactly
    (synth.synth_weight / synth.synth_activation streams); keeps the host arrays alive."""
    from . import synth
    keep = []

    def desc(seed_, std, cols, gamma):
        d = _lib.SynthDesc()
        d.seed, d.stddev, d.gamma = seed_ & synth.M64, float(std), float(gamma)
        if cols is not None and len(cols) > 0 and gamma != 1.0:
            a = np.ascontiguousarray(cols, dtype=np.int32)
            keep.append(a)
            d.outlier_cols, d.num_outliers = a.ctypes.data, len(a)
        else:
            d.outlier_cols, d.num_outliers = None, 0
        return d

    L = _lib.CalibLayer()
    L.index, L.n, L.k, L.rows = spec.index, spec.out_dim, spec.in_dim, rows
    wcols = (synth.pick_outlier_columns(seed, spec.index, spec.in_dim, spec.outlier_fraction)
             if spec.outlier_fraction > 0 else None)
    L.w_host, L.x_host = None, None
    L.w_synth = desc(synth.mix_seed(seed, spec.index), 1.0 / np.sqrt(spec.in_dim), wcols, spec.gamma)
    s_act = synth.mix_seed(seed, spec.index) ^ synth.K_ACT_SALT
    heavy = synth.pick_outlier_columns(s_act, 0, spec.in_dim, 0.005)
    xs = (_lib.SynthDesc * frames)(*[desc(synth.mix_seed(s_act, f + 1), 1.0 + 0.05 * f, heavy, 6.0)
                                     for f in range(frames)])
    keep.append(xs)
    L.x_synth = xs
    return L, keep


def calibrate_sharded_native(specs, frames: int, rows: int, world: int, devices=None, seed: int = 1,
                             frame_weights=None, percentiles=PERCENTILES):
    """Config 4 through the C++ driver: returns (records sorted by layer, max-over-ranks step ms,
    whether the records crossed NCCL)."""
    from . import synth
    layers = (_lib.CalibLayer * len(specs))()
    keep = []
    cap = 0
    for i, spec in enumerate(specs):
        r = rows if spec.tokens != synth.WAN_TEXT_LEN else synth.WAN_TEXT_LEN
        layers[i], k = synth_descriptors(spec, frames, r, seed)
        keep.append(k)
        cap += int(_lib.load().qarvd_calib_record_doubles(spec.out_dim, spec.in_dim, len(percentiles)))
    devs = np.ascontiguousarray(devices if devices is not None else list(range(world)), dtype=np.int32)
    pct = np.ascontiguousarray(percentiles, dtype=np.float64)
    w = None if frame_weights is None else np.ascontiguousarray(frame_weights, dtype=np.float64)
    recs = np.empty(cap, dtype=np.float64)
    offs = np.empty(len(specs) + 1, dtype=np.int64)
    ms, used = _lib.ctypes.c_double(), _lib.ctypes.c_int()
    _lib.call("qarvd_calibrate_sharded", layers, len(specs), frames, None if w is None else w.ctypes.data,
              pct.ctypes.data, len(pct), world, devs.ctypes.data, recs.ctypes.data, cap, offs.ctypes.data,
              _lib.ctypes.byref(ms), _lib.ctypes.byref(used))
    return unpack_records(recs[:offs[-1]]), ms.value, bool(used.value)
