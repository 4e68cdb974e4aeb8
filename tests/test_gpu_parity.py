"""GPU parity tests: every kernel through the C-ABI vs the CPU oracle (and the compiled
reference where it exists).  Integer outputs (codes, accumulators, indices, selected
scales) are compared bit-exactly; floating outputs as stated per test."""
import numpy as np
import pytest
import torch

import oracle
import paper_2605_21072_b200 as qb
from paper_2605_21072_b200 import engine, calibrate, synth
from qarvd_testutil import bf16_values

pytestmark = pytest.mark.gpu


def to_dev_bf16(bits: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def dev_bits(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def make_plan(k, n_out, seed=0, pad_unaligned=False):
    r = np.random.default_rng(seed)
    outl = np.sort(r.choice(k, size=n_out, replace=False)) if n_out else []
    return engine.build_plan("t", k, outl)


# ---------------------------------------------------------------- K1
@pytest.mark.parametrize("m,k,n_out", [(4680, 1536, 32), (257, 1536, 0), (96, 8960, 192),
                                       (33, 200, 5), (1, 64, 3)])
def test_k1_per_token_bitexact(cuda, m, k, n_out):
    plan = make_plan(k, n_out, seed=m)
    heavy = plan.outlier_indices if n_out else None
    bits, x64 = bf16_values((m, k), seed=k + m, heavy_cols=heavy)
    xq, s32, s64 = engine.kernel_a_quantize_activation(to_dev_bf16(bits), plan, check_finite=True)
    q_ref, s_ref, bad = oracle.quantize_act(x64, plan.gather, per_token=True)
    assert bad < 0
    np.testing.assert_array_equal(xq.cpu().numpy(), q_ref)
    np.testing.assert_array_equal(s64.cpu().numpy(), s_ref)
    np.testing.assert_array_equal(s32.cpu().numpy(), s_ref.astype(np.float32))


def test_k1_ties_and_edges(cuda):
    # rows built so v/s hits exact .5 ties, zeros, max, and an all-zero row
    k = 256
    r = np.random.default_rng(7)
    rows = []
    for i in range(64):
        a = float(2.0 ** r.integers(-6, 6))
        base = np.arange(-k // 2, k // 2, dtype=np.float64) * (a / 127.0) * 0.5
        base[0] = a
        rows.append(base)
    rows.append(np.zeros(k))
    x = np.asarray(rows, dtype=np.float32)
    bits = oracle.f32_to_bf16_bits(x)
    x64 = oracle.bf16_bits_to_f64(bits)
    xq, _, s64 = engine.kernel_a_quantize_activation(to_dev_bf16(bits), engine.build_plan("t", k, []))
    q_ref, s_ref, _ = oracle.quantize_act(x64, None, per_token=True)
    np.testing.assert_array_equal(xq.cpu().numpy()[:, :k], q_ref)
    np.testing.assert_array_equal(s64.cpu().numpy(), s_ref)
    assert s_ref[-1] == np.finfo(np.float64).tiny


def test_k1_static_scale_clamps(cuda):
    bits, x64 = bf16_values((512, 1536), seed=3, scale=4.0)
    plan = make_plan(1536, 32, seed=1)
    s = 0.0123
    xq, s32, _ = engine.kernel_a_quantize_activation(to_dev_bf16(bits), plan, qb.ACT_PER_TENSOR, s)
    q_ref, _, _ = oracle.quantize_act(x64, plan.gather, per_token=False, static_scale=s)
    np.testing.assert_array_equal(xq.cpu().numpy(), q_ref)
    assert (np.abs(q_ref) == 127).any()


def test_k1_f64_input_matches_reference(cuda, ref_lib):
    r = np.random.default_rng(11)
    x64 = r.standard_normal((64, 96)) * 3.0  # not bf16-representable: the f64 path
    codes_ref, scales_ref = oracle.ref_quantize(x64, per_token=True)
    plan = engine.build_plan("t", 96, [])
    xq, _, s64 = engine.kernel_a_quantize_activation(torch.from_numpy(x64).cuda(), plan)
    np.testing.assert_array_equal(xq.cpu().numpy()[:, :96], codes_ref)
    np.testing.assert_array_equal(s64.cpu().numpy(), scales_ref)


def test_k1_nonfinite_reports_first_index(cuda):
    bits, _ = bf16_values((8, 64), seed=5)
    bits[3, 10] = 0x7FC0  # nan
    bits[5, 2] = 0x7F80   # inf
    plan = engine.build_plan("t", 64, [])
    with pytest.raises(qb.InvalidArgument, match="flat index 202"):
        engine.kernel_a_quantize_activation(to_dev_bf16(bits), plan, check_finite=True)


# ---------------------------------------------------------------- K5
@pytest.mark.parametrize("n,k,n_out", [(1536, 1536, 32), (384, 8960, 188), (64, 256, 0), (40, 100, 7)])
def test_k5_weights_bitexact(cuda, n, k, n_out):
    plan = make_plan(k, n_out, seed=n)
    heavy = plan.outlier_indices if n_out else None
    bits, w64 = bf16_values((n, k), seed=n + 1, scale=1.0 / np.sqrt(k), heavy_cols=heavy)
    layer = engine.prepare_weights("t", to_dev_bf16(bits), plan)
    wq_ref, so_ref, sn_ref, bad = oracle.prepare_weights(w64, plan.gather, plan.k_outlier)
    assert bad < 0
    np.testing.assert_array_equal(layer.wq.cpu().numpy(), wq_ref)
    np.testing.assert_array_equal(layer.scale_outlier64.cpu().numpy(), so_ref)
    np.testing.assert_array_equal(layer.scale_normal64.cpu().numpy(), sn_ref)


def test_k5_matches_reference_build_plan(cuda, ref_lib):
    n, k = 96, 256
    plan = make_plan(k, 32, seed=2)
    bits, w64 = bf16_values((n, k), seed=9, heavy_cols=plan.outlier_indices)
    ref = oracle.ref_build_plan_codes(w64, plan.outlier_indices)
    layer = engine.prepare_weights("t", to_dev_bf16(bits), plan)
    np.testing.assert_array_equal(plan.permutation, ref["permutation"])
    np.testing.assert_array_equal(layer.scale_outlier64.cpu().numpy(), ref["scale_outlier"])
    np.testing.assert_array_equal(layer.scale_normal64.cpu().numpy(), ref["scale_normal"])
    np.testing.assert_array_equal(layer.wq.cpu().numpy().astype(np.int32), ref["wq"])


# ---------------------------------------------------------------- K2
def _gemm_case(m, n, k, n_out, seed):
    plan = make_plan(k, n_out, seed=seed)
    heavy = plan.outlier_indices if n_out else None
    wbits, w64 = bf16_values((n, k), seed=seed + 1, scale=1.0 / np.sqrt(k), heavy_cols=heavy)
    xbits, x64 = bf16_values((m, k), seed=seed + 2, heavy_cols=heavy, gamma=4.0)
    layer = engine.prepare_weights("t", to_dev_bf16(wbits), plan)
    xq, s32, s64 = engine.kernel_a_quantize_activation(to_dev_bf16(xbits), layer)
    return plan, layer, xq, s32, s64, w64, x64


@pytest.mark.parametrize("m,n,k,n_out", [
    (4680, 1536, 1536, 32),     # config 1 (self-attn qkv shape)
    (300, 8960, 1536, 32),      # ffn.0 shape, ragged M
    (200, 1536, 8960, 192),     # ffn.2 shape (K_o = 192)
    (130, 256, 256, 0),         # disabled plan: single accumulator
    (77, 96, 160, 5),           # unaligned outliers padded to 32, ragged N
])
def test_k2_accumulators_and_epilogue_bitexact(cuda, m, n, k, n_out):
    plan, layer, xq, s32, s64, _, _ = _gemm_case(m, n, k, n_out, seed=m + n)
    y, acc_o, acc_n = engine.kernel_b_gemm_dequant(xq, s32, layer, dump_acc=True)
    xq_h, wq_h = xq.cpu().numpy(), layer.wq.cpu().numpy()
    _, ao_ref, an_ref = oracle.kernel_b(xq_h, wq_h, plan.k_outlier, s64.cpu().numpy(),
                                        layer.scale_outlier64.cpu().numpy(),
                                        layer.scale_normal64.cpu().numpy(), with_acc=True)
    np.testing.assert_array_equal(acc_o.cpu().numpy(), ao_ref)
    np.testing.assert_array_equal(acc_n.cpu().numpy(), an_ref)
    y_ref = oracle.epilogue_f32(ao_ref, an_ref, plan.k_outlier > 0, s32.cpu().numpy(),
                                layer.scale_outlier32.cpu().numpy(),
                                layer.scale_normal32.cpu().numpy())
    np.testing.assert_array_equal(dev_bits(y), y_ref)


def test_k2_vs_reference_kernel_b_tolerance(cuda, ref_lib):
    """bf16 output vs the reference's own f64 kernel_b_gemm_dequant (per-token rows)."""
    m, n, k = 64, 512, 1536
    plan, layer, xq, s32, s64, w64, x64 = _gemm_case(m, n, k, 32, seed=21)
    ref = oracle.ref_build_plan_codes(w64, plan.outlier_indices)
    xp = oracle.ref_permute(x64, ref["permutation"])
    codes, sx = oracle.ref_quantize(xp, per_token=True)
    np.testing.assert_array_equal(codes, xq.cpu().numpy().astype(np.int32))  # k_pad == k here
    y_ref = oracle.ref_kernel_b(codes, ref["wq"], ref["permutation"], len(plan.outlier_indices),
                                True, sx, ref["scale_outlier"], ref["scale_normal"])
    y, acc_o, acc_n = engine.kernel_b_gemm_dequant(xq, s32, layer, dump_acc=True)
    yd = y.float().cpu().numpy().astype(np.float64)
    so, sn = ref["scale_outlier"], ref["scale_normal"]
    mag = np.abs(sx[:, None] * so[None] * acc_o.cpu().numpy()) + np.abs(sx[:, None] * sn[None] * acc_n.cpu().numpy())
    tol = 2.0 ** -8 * np.abs(y_ref) + 2.0 ** -22 * mag + 1e-30
    assert np.all(np.abs(yd - y_ref) <= tol)


def test_k2_bias_gelu_f32(cuda):
    m, n, k = 256, 384, 512
    plan, layer, xq, s32, s64, _, _ = _gemm_case(m, n, k, 32, seed=5)
    bias = torch.linspace(-1, 1, n, device="cuda", dtype=torch.float32)
    y32, acc_o, acc_n = engine.kernel_b_gemm_dequant(xq, s32, layer, out_dtype=torch.float32,
                                                     bias=bias, dump_acc=True)
    ref32 = oracle.epilogue_f32(acc_o.cpu().numpy(), acc_n.cpu().numpy(), True, s32.cpu().numpy(),
                                layer.scale_outlier32.cpu().numpy(),
                                layer.scale_normal32.cpu().numpy(), bias.cpu().numpy(), out="f32")
    np.testing.assert_array_equal(y32.cpu().numpy(), ref32)
    yg = engine.kernel_b_gemm_dequant(xq, s32, layer, out_dtype=torch.float32, bias=bias,
                                      epilogue=qb.EPI_GELU)
    r = torch.from_numpy(ref32).double()
    gelu = 0.5 * r * (1 + torch.erf(r / np.sqrt(2.0)))
    torch.testing.assert_close(yg.cpu().double(), gelu, rtol=1e-5, atol=1e-6)


def test_linear_handle_device_and_host(cuda):
    m, n, k = 4680, 1536, 1536
    plan, layer, xq, s32, _, _, _ = _gemm_case(m, n, k, 32, seed=3)
    y_ref = engine.kernel_b_gemm_dequant(xq, s32, layer)
    xbits, _ = bf16_values((m, k), seed=3 + 2, heavy_cols=plan.outlier_indices, gamma=4.0)
    x = to_dev_bf16(xbits)
    h = engine.LinearHandle(layer)
    y = h.forward(x)
    torch.cuda.synchronize()
    assert torch.equal(y.view(torch.int16), y_ref.view(torch.int16))
    xh = x.cpu().pin_memory()
    yh = torch.empty((m, n), dtype=torch.bfloat16).pin_memory()
    h.forward_host(xh, yh)
    assert torch.equal(yh.view(torch.int16), y_ref.cpu().view(torch.int16))
    h.close()


# ---------------------------------------------------------------- K3
@pytest.mark.parametrize("n,k,frac,gamma", [(1536, 1536, 0.021, 8.0), (1536, 8960, 0.021, 8.0),
                                            (8960, 1536, 0.021, 8.0), (64, 256, 0.03, 10.0),
                                            (96, 40, 0.1, 5.0), (128, 512, 0.0, 1.0)])
def test_k3_detection_bitexact(cuda, n, k, frac, gamma):
    r = np.random.default_rng(n + k)
    heavy = r.choice(k, size=max(1, int(round(frac * k))), replace=False) if frac else None
    bits, w64 = bf16_values((n, k), seed=k, scale=1.0 / np.sqrt(k), heavy_cols=heavy, gamma=gamma)
    rep = qb.analyze_layer("t", to_dev_bf16(bits))
    o = oracle.analyze_layer(w64)
    np.testing.assert_array_equal(rep.norms.cpu().numpy(), o["norms"])
    assert (rep.median, rep.mad, rep.threshold) == (o["median"], o["mad"], o["threshold"])
    np.testing.assert_array_equal(rep.raw_outliers, o["raw"])
    np.testing.assert_array_equal(rep.aligned_outliers, o["aligned"])


def test_k3_batched_matches_reference(cuda, ref_lib):
    ws, refs = [], []
    for i, (n, k) in enumerate([(64, 256), (128, 96), (32, 1024)]):
        heavy = np.arange(3 + i, k, 37)[: 2 + i]
        bits, w64 = bf16_values((n, k), seed=100 + i, heavy_cols=heavy, gamma=6.0)
        ws.append(to_dev_bf16(bits))
        refs.append(oracle.ref_analyze_layer(w64))
    reps = qb.analyze_layers(["a", "b", "c"], ws)
    for rep, ref in zip(reps, refs):
        np.testing.assert_array_equal(rep.norms.cpu().numpy(), ref["norms"])
        assert (rep.median, rep.mad, rep.threshold) == (ref["median"], ref["mad"], ref["threshold"])
        np.testing.assert_array_equal(rep.raw_outliers, ref["raw"])
        np.testing.assert_array_equal(rep.aligned_outliers, ref["aligned"])


# ---------------------------------------------------------------- K4
@pytest.mark.parametrize("frames,rows,k,kind", [(21, 156, 1536, "heuristic_exp"), (21, 60, 512, "uniform"),
                                                (7, 16, 64, "heuristic_exp"), (3, 5, 40, "uniform")])
def test_k4_search_bitexact_vs_oracle(cuda, frames, rows, k, kind):
    bits, _ = bf16_values((frames * rows, k), seed=frames * k, heavy_cols=np.arange(0, k, 97))
    w = calibrate.weighting_strategy(kind, frames)
    res = calibrate.scale_search_async([to_dev_bf16(bits)], frames, w).cpu().numpy()[0]
    ref = oracle.scale_search_hist(bits, frames, rows, k, weights=w)
    np.testing.assert_array_equal(res, ref)


def test_k4_uniform_limit_equals_reference_percentile_search(cuda, ref_lib):
    frames, rows, k = 21, 40, 1536
    bits, x64 = bf16_values((frames * rows, k), seed=1234, heavy_cols=np.arange(0, k, 97))
    res = calibrate.scale_search_async([to_dev_bf16(bits)], frames, None).cpu().numpy()[0]
    best_pct, scale, mse = oracle.ref_percentile_search(x64, frames, rows, k)
    assert calibrate.PERCENTILES[int(res[9])] == best_pct
    assert res[10] == scale  # bit-identical selected scale
    np.testing.assert_allclose(res[6:9], mse, rtol=1e-12)


def test_k4_batched_layers(cuda):
    frames = 21
    xs, exp = [], []
    w = calibrate.weighting_strategy("heuristic_exp", frames)
    for i, (rows, k) in enumerate([(20, 1536), (20, 8960), (10, 256)]):
        bits, _ = bf16_values((frames * rows, k), seed=i, heavy_cols=np.arange(i, k, 61))
        xs.append(to_dev_bf16(bits))
        exp.append(oracle.scale_search_hist(bits, frames, rows, k, weights=w))
    res = calibrate.scale_search_async(xs, frames, w).cpu().numpy()
    for r, e in zip(res, exp):
        np.testing.assert_array_equal(r, e)


# ---------------------------------------------------------------- synthetic data
def test_synth_weights_outlier_columns_detected(cuda):
    specs = synth.wan_registry(blocks=1)
    spec = [s for s in specs if s.name.endswith("ffn.2")][0]
    w = synth.synth_weight(spec, seed=1)
    rep = qb.analyze_layer(spec.name, w)
    cols = synth.pick_outlier_columns(1, spec.index, spec.in_dim, spec.outlier_fraction)
    assert set(cols.tolist()) <= set(rep.aligned_outliers.tolist())
    assert len(rep.aligned_outliers) == 192


# ---------------------------------------------------------------- K1 without a gather + chain fold
@pytest.mark.parametrize("m,k", [(4680, 8960), (300, 1536), (33, 200), (7, 16384), (5, 2056)])
def test_k1_contiguous_rows_bitexact(cuda, m, k):
    """Identity layout (inputs already in plan order): the no-gather K1 path."""
    bits, x64 = bf16_values((m, k), seed=k + 3 * m, heavy_cols=np.arange(0, k, 97))
    x = to_dev_bf16(bits)
    xq = torch.empty((m, k), dtype=torch.int8, device="cuda")
    s64 = torch.empty(m, dtype=torch.float64, device="cuda")
    qb._lib.call("qarvd_quantize_act", x.data_ptr(), qb.BF16, m, k, k, None, k, qb.ACT_PER_TOKEN,
                 0.0, 8, xq.data_ptr(), k, None, s64.data_ptr(), None, None)
    q_ref, s_ref, _ = oracle.quantize_act(x64, None, per_token=True)
    np.testing.assert_array_equal(xq.cpu().numpy(), q_ref)
    np.testing.assert_array_equal(s64.cpu().numpy(), s_ref)


def test_k1_contiguous_nonfinite_and_static(cuda):
    bits, x64 = bf16_values((16, 1024), seed=17, scale=4.0)
    x = to_dev_bf16(bits)
    xq = torch.empty((16, 1024), dtype=torch.int8, device="cuda")
    s = 0.0123
    qb._lib.call("qarvd_quantize_act", x.data_ptr(), qb.BF16, 16, 1024, 1024, None, 1024,
                 qb.ACT_PER_TENSOR, s, 8, xq.data_ptr(), 1024, None, None, None, None)
    q_ref, _, _ = oracle.quantize_act(x64, None, per_token=False, static_scale=s)
    np.testing.assert_array_equal(xq.cpu().numpy(), q_ref)
    bits[9, 700] = 0x7F80
    bits[12, 5] = 0xFFC0
    err = torch.empty(1, dtype=torch.int64, device="cuda")
    qb._lib.call("qarvd_quantize_act", to_dev_bf16(bits).data_ptr(), qb.BF16, 16, 1024, 1024, None,
                 1024, qb.ACT_PER_TOKEN, 0.0, 8, xq.data_ptr(), 1024, None, None, err.data_ptr(), None)
    torch.cuda.synchronize()
    assert int(err.item()) == 9 * 1024 + 700


@pytest.mark.parametrize("d,f,m,n0,n2", [(256, 640, 300, 32, 13), (1536, 8960, 256, 32, 192),
                                          (96, 200, 33, 5, 0)])
def test_chain_fold_bitexact(cuda, d, f, m, n0, n2):
    """Producing the intermediate in the consumer's plan order (pipeline.fold_output_permutation)
    gives the same codes, scales and final output as permute-then-quantize."""
    from paper_2605_21072_b200.pipeline import QuantizedChain
    p0, p2 = make_plan(d, n0, seed=1), make_plan(f, n2, seed=2)
    w0, _ = bf16_values((f, d), seed=4, scale=1.0 / np.sqrt(d), heavy_cols=p0.outlier_indices if n0 else None)
    w2, _ = bf16_values((d, f), seed=5, scale=1.0 / np.sqrt(f), heavy_cols=p2.outlier_indices if n2 else None)
    L0 = engine.prepare_weights("ffn.0", to_dev_bf16(w0), p0)
    L2 = engine.prepare_weights("ffn.2", to_dev_bf16(w2), p2)
    L0.bias = torch.linspace(-0.5, 0.5, f, device="cuda", dtype=torch.float32)
    xb, _ = bf16_values((m, d), seed=6, heavy_cols=p0.outlier_indices if n0 else None, gamma=4.0)
    outs = []
    for fold, fuse in ((False, False), (True, False), (True, True)):
        ch = QuantizedChain([L0, L2], m, epilogues=[qb.EPI_GELU, qb.EPI_NONE], fold=fold,
                            fuse_rowmax=fuse)
        assert (ch.layers[1].gather_dev is None) == fold
        ch.x.copy_(to_dev_bf16(xb))
        ch.launch()
        torch.cuda.synchronize()
        outs.append((ch.xq[1].clone(), ch.sx[1].clone(), ch.output.clone()))
    (q_a, s_a, y_a) = outs[0]
    for (q_b, s_b, y_b) in outs[1:]:
        assert torch.equal(q_a, q_b)
        assert torch.equal(s_a, s_b)
        assert torch.equal(y_a.view(torch.int16), y_b.view(torch.int16))
    # and the C-ABI host chain over the folded layers agrees
    ch = QuantizedChain([L0, L2], m, epilogues=[qb.EPI_GELU, qb.EPI_NONE], fold=True)
    hs = [engine.LinearHandle(ch.layers[0], qb.EPI_GELU), engine.LinearHandle(ch.layers[1])]
    xh = torch.from_numpy(xb.view(np.int16)).view(torch.bfloat16).pin_memory()
    yh = torch.empty((m, d), dtype=torch.bfloat16).pin_memory()
    engine.chain_forward_host(hs, xh, yh)
    assert torch.equal(yh.view(torch.int16), y_a.cpu().view(torch.int16))
    for h in hs:
        h.close()


@pytest.mark.parametrize("k", [256, 8960])
def test_k1_contiguous_ties(cuda, k):
    """Rows built so v/s lands on exact .5 ties (and an all-zero row) on the no-gather path."""
    r = np.random.default_rng(k)
    rows = []
    for i in range(48):
        a = float(2.0 ** r.integers(-6, 6))
        base = (np.arange(k, dtype=np.float64) % 255 - 127) * (a / 127.0) * 0.5
        base[0] = a
        rows.append(base)
    rows.append(np.zeros(k))
    bits = oracle.f32_to_bf16_bits(np.asarray(rows, dtype=np.float32))
    x64 = oracle.bf16_bits_to_f64(bits)
    m = len(rows)
    x = to_dev_bf16(bits)
    xq = torch.empty((m, k), dtype=torch.int8, device="cuda")
    s64 = torch.empty(m, dtype=torch.float64, device="cuda")
    qb._lib.call("qarvd_quantize_act", x.data_ptr(), qb.BF16, m, k, k, None, k, qb.ACT_PER_TOKEN,
                 0.0, 8, xq.data_ptr(), k, None, s64.data_ptr(), None, None)
    q_ref, s_ref, _ = oracle.quantize_act(x64, None, per_token=True)
    np.testing.assert_array_equal(xq.cpu().numpy(), q_ref)
    np.testing.assert_array_equal(s64.cpu().numpy(), s_ref)


# ---------------------------------------------------------------- chained producer / streaming K1
def _rowmax_bits(y_bf16: torch.Tensor) -> np.ndarray:
    return (dev_bits(y_bf16).astype(np.uint32) & 0x7FFF).max(axis=1)


@pytest.mark.parametrize("m,n,k,n_out,epi", [(300, 8960, 1536, 32, qb.EPI_GELU), (77, 200, 160, 5, qb.EPI_NONE)])
def test_k2_rowmax_matches_output(cuda, m, n, k, n_out, epi):
    """qarvd_dual_gemm_rowmax: same y as qarvd_dual_gemm, plus the per-row max of |bf16 y| bits."""
    plan, layer, xq, s32, s64, _, _ = _gemm_case(m, n, k, n_out, seed=m)
    y_ref = engine.kernel_b_gemm_dequant(xq, s32, layer, epilogue=epi)
    y = torch.empty_like(y_ref)
    rm = torch.zeros(m, dtype=torch.int32, device="cuda")
    for _ in range(2):  # accumulating twice over the same output leaves the max unchanged
        qb._lib.call("qarvd_dual_gemm_rowmax", xq.data_ptr(), layer.k_pad, layer.wq.data_ptr(),
                     layer.k_pad, m, n, layer.k_pad, layer.k_outlier, s32.data_ptr(),
                     layer.scale_outlier32.data_ptr(), layer.scale_normal32.data_ptr(), None, epi,
                     y.data_ptr(), n, rm.data_ptr(), None)
    torch.cuda.synchronize()
    assert torch.equal(y.view(torch.int16), y_ref.view(torch.int16))
    np.testing.assert_array_equal(rm.cpu().numpy().astype(np.uint32), _rowmax_bits(y_ref))


@pytest.mark.parametrize("m,k", [(4680, 8960), (33, 200), (5, 1536)])
def test_k1_stream_rowmax_bitexact(cuda, m, k):
    """qarvd_quantize_act_rowmax == the gather-free qarvd_quantize_act; it resets row_absmax."""
    bits, x64 = bf16_values((m, k), seed=m + k, heavy_cols=np.arange(3, k, 101))
    x = to_dev_bf16(bits)
    rm = torch.from_numpy((bits.astype(np.uint32) & 0x7FFF).max(axis=1).astype(np.int32)).cuda()
    xq = torch.empty((m, k), dtype=torch.int8, device="cuda")
    s64 = torch.empty(m, dtype=torch.float64, device="cuda")
    s32 = torch.empty(m, dtype=torch.float32, device="cuda")
    qb._lib.call("qarvd_quantize_act_rowmax", x.data_ptr(), m, k, k, rm.data_ptr(), qb.ACT_PER_TOKEN,
                 0.0, 8, xq.data_ptr(), k, s32.data_ptr(), s64.data_ptr(), None, None)
    q_ref, s_ref, _ = oracle.quantize_act(x64, None, per_token=True)
    np.testing.assert_array_equal(xq.cpu().numpy(), q_ref)
    np.testing.assert_array_equal(s64.cpu().numpy(), s_ref)
    np.testing.assert_array_equal(s32.cpu().numpy(), s_ref.astype(np.float32))
    assert int(rm.abs().sum().item()) == 0
    # static scale (row_absmax unused)
    s = 0.0123
    qb._lib.call("qarvd_quantize_act_rowmax", x.data_ptr(), m, k, k, None, qb.ACT_PER_TENSOR, s, 8,
                 xq.data_ptr(), k, None, None, None, None)
    q_ref, _, _ = oracle.quantize_act(x64, None, per_token=False, static_scale=s)
    np.testing.assert_array_equal(xq.cpu().numpy(), q_ref)


def test_k1_stream_rowmax_ties_and_nonfinite(cuda):
    k = 256
    r = np.random.default_rng(3)
    rows = []
    for i in range(40):
        a = float(2.0 ** r.integers(-6, 6))
        base = (np.arange(k, dtype=np.float64) % 255 - 127) * (a / 127.0) * 0.5
        base[0] = a
        rows.append(base)
    rows.append(np.zeros(k))
    bits = oracle.f32_to_bf16_bits(np.asarray(rows, dtype=np.float32))
    x64 = oracle.bf16_bits_to_f64(bits)
    m = len(rows)
    rm = torch.from_numpy((bits.astype(np.uint32) & 0x7FFF).max(axis=1).astype(np.int32)).cuda()
    xq = torch.empty((m, k), dtype=torch.int8, device="cuda")
    s64 = torch.empty(m, dtype=torch.float64, device="cuda")
    x = to_dev_bf16(bits)
    qb._lib.call("qarvd_quantize_act_rowmax", x.data_ptr(), m, k, k, rm.data_ptr(), qb.ACT_PER_TOKEN,
                 0.0, 8, xq.data_ptr(), k, None, s64.data_ptr(), None, None)
    q_ref, s_ref, _ = oracle.quantize_act(x64, None, per_token=True)
    np.testing.assert_array_equal(xq.cpu().numpy(), q_ref)
    np.testing.assert_array_equal(s64.cpu().numpy(), s_ref)
    bits[7, 30] = 0x7F80
    bits[9, 3] = 0xFFC0
    rm = torch.from_numpy((bits.astype(np.uint32) & 0x7FFF).max(axis=1).astype(np.int32)).cuda()
    err = torch.empty(1, dtype=torch.int64, device="cuda")
    qb._lib.call("qarvd_quantize_act_rowmax", to_dev_bf16(bits).data_ptr(), m, k, k, rm.data_ptr(),
                 qb.ACT_PER_TOKEN, 0.0, 8, xq.data_ptr(), k, None, None, err.data_ptr(), None)
    torch.cuda.synchronize()
    assert int(err.item()) == 7 * k + 30


def test_host_chain_pipelined_chunks(cuda):
    """qarvd_linear_chain_forward_host splits M into row chunks whose copies overlap the
    compute; the result equals the device-resident chain bit for bit."""
    from paper_2605_21072_b200.pipeline import QuantizedChain
    d, f, m = 256, 640, 3000
    p0, p2 = make_plan(d, 32, seed=3), make_plan(f, 13, seed=4)
    w0, _ = bf16_values((f, d), seed=7, scale=1.0 / np.sqrt(d), heavy_cols=p0.outlier_indices)
    w2, _ = bf16_values((d, f), seed=8, scale=1.0 / np.sqrt(f), heavy_cols=p2.outlier_indices)
    L0 = engine.prepare_weights("ffn.0", to_dev_bf16(w0), p0)
    L2 = engine.prepare_weights("ffn.2", to_dev_bf16(w2), p2)
    xb, _ = bf16_values((m, d), seed=9, heavy_cols=p0.outlier_indices, gamma=4.0)
    ch = QuantizedChain([L0, L2], m, epilogues=[qb.EPI_GELU, qb.EPI_NONE])
    ch.x.copy_(to_dev_bf16(xb))
    ch.launch()
    torch.cuda.synchronize()
    hs = [engine.LinearHandle(ch.layers[0], qb.EPI_GELU), engine.LinearHandle(ch.layers[1])]
    xh = torch.from_numpy(xb.view(np.int16)).view(torch.bfloat16).pin_memory()
    yh = torch.empty((m, d), dtype=torch.bfloat16).pin_memory()
    for _ in range(4):  # eager, then captured into a graph, then replayed
        yh.zero_()
        engine.chain_forward_host(hs, xh, yh)
        assert torch.equal(yh.view(torch.int16), ch.output.cpu().view(torch.int16))
    # new input values through the same (graph-cached) buffers
    xb2, _ = bf16_values((m, d), seed=10, heavy_cols=p0.outlier_indices, gamma=4.0)
    xh.copy_(torch.from_numpy(xb2.view(np.int16)).view(torch.bfloat16))
    ch.x.copy_(to_dev_bf16(xb2))
    ch.launch()
    torch.cuda.synchronize()
    engine.chain_forward_host(hs, xh, yh)
    assert torch.equal(yh.view(torch.int16), ch.output.cpu().view(torch.int16))
    for h in hs:
        h.close()


@pytest.mark.parametrize("m,k", [(4680, 8960), (33, 512), (300, 1536)])
def test_k1_flat_pmax_bitexact(cuda, m, k):
    """qarvd_quantize_act_pmax (row |x| max from partial maxima) == the gather-free K1."""
    bits, x64 = bf16_values((m, k), seed=m + 2 * k, heavy_cols=np.arange(5, k, 89))
    x = to_dev_bf16(bits)
    mag = (bits.astype(np.uint32) & 0x7FFF)
    pm = 7  # arbitrary partition of each row into partials
    parts = np.zeros((m, pm), dtype=np.uint32)
    for p_ in range(pm):
        parts[:, p_] = mag[:, p_::pm].max(axis=1)
    rp = torch.from_numpy(parts.astype(np.int32)).cuda()
    xq = torch.empty((m, k), dtype=torch.int8, device="cuda")
    s64 = torch.empty(m, dtype=torch.float64, device="cuda")
    s32 = torch.empty(m, dtype=torch.float32, device="cuda")
    qb._lib.call("qarvd_quantize_act_pmax", x.data_ptr(), m, k, k, rp.data_ptr(), pm, qb.ACT_PER_TOKEN,
                 0.0, 8, xq.data_ptr(), k, s32.data_ptr(), s64.data_ptr(), None, None)
    q_ref, s_ref, _ = oracle.quantize_act(x64, None, per_token=True)
    np.testing.assert_array_equal(xq.cpu().numpy(), q_ref)
    np.testing.assert_array_equal(s64.cpu().numpy(), s_ref)
    np.testing.assert_array_equal(s32.cpu().numpy(), s_ref.astype(np.float32))
    s = 0.0123
    qb._lib.call("qarvd_quantize_act_pmax", x.data_ptr(), m, k, k, None, 0, qb.ACT_PER_TENSOR, s, 8,
                 xq.data_ptr(), k, None, None, None, None)
    q_ref, _, _ = oracle.quantize_act(x64, None, per_token=False, static_scale=s)
    np.testing.assert_array_equal(xq.cpu().numpy(), q_ref)


def test_k1_flat_pmax_ties_and_nonfinite(cuda):
    k = 1024
    r = np.random.default_rng(5)
    rows = []
    for i in range(40):
        a = float(2.0 ** r.integers(-6, 6))
        base = (np.arange(k, dtype=np.float64) % 255 - 127) * (a / 127.0) * 0.5
        base[0] = a
        rows.append(base)
    rows.append(np.zeros(k))
    bits = oracle.f32_to_bf16_bits(np.asarray(rows, dtype=np.float32))
    x64 = oracle.bf16_bits_to_f64(bits)
    m = len(rows)
    rp = torch.from_numpy((bits.astype(np.uint32) & 0x7FFF).max(axis=1, keepdims=True).astype(np.int32)).cuda()
    xq = torch.empty((m, k), dtype=torch.int8, device="cuda")
    s64 = torch.empty(m, dtype=torch.float64, device="cuda")
    qb._lib.call("qarvd_quantize_act_pmax", to_dev_bf16(bits).data_ptr(), m, k, k, rp.data_ptr(), 1,
                 qb.ACT_PER_TOKEN, 0.0, 8, xq.data_ptr(), k, None, s64.data_ptr(), None, None)
    q_ref, s_ref, _ = oracle.quantize_act(x64, None, per_token=True)
    np.testing.assert_array_equal(xq.cpu().numpy(), q_ref)
    np.testing.assert_array_equal(s64.cpu().numpy(), s_ref)
    bits[7, 30] = 0x7F80
    bits[9, 3] = 0xFFC0
    rp = torch.from_numpy((bits.astype(np.uint32) & 0x7FFF).max(axis=1, keepdims=True).astype(np.int32)).cuda()
    err = torch.empty(1, dtype=torch.int64, device="cuda")
    qb._lib.call("qarvd_quantize_act_pmax", to_dev_bf16(bits).data_ptr(), m, k, k, rp.data_ptr(), 1,
                 qb.ACT_PER_TOKEN, 0.0, 8, xq.data_ptr(), k, None, None, err.data_ptr(), None)
    torch.cuda.synchronize()
    assert int(err.item()) == 7 * k + 30


@pytest.mark.parametrize("m,n,k,n_out,epi", [(300, 8960, 1536, 32, qb.EPI_GELU), (77, 200, 160, 5, qb.EPI_NONE)])
def test_k2_pmax_partials(cuda, m, n, k, n_out, epi):
    """qarvd_dual_gemm_pmax: same y; the row max of its partials is the row max of |bf16 y|."""
    plan, layer, xq, s32, s64, _, _ = _gemm_case(m, n, k, n_out, seed=m + 1)
    y_ref = engine.kernel_b_gemm_dequant(xq, s32, layer, epilogue=epi)
    pm = qb._lib.load().qarvd_dual_gemm_pmax_count(m, n, layer.k_pad)
    y = torch.empty_like(y_ref)
    rp = torch.full((m, pm), -1, dtype=torch.int32, device="cuda")
    qb._lib.call("qarvd_dual_gemm_pmax", xq.data_ptr(), layer.k_pad, layer.wq.data_ptr(), layer.k_pad,
                 m, n, layer.k_pad, layer.k_outlier, s32.data_ptr(), layer.scale_outlier32.data_ptr(),
                 layer.scale_normal32.data_ptr(), None, epi, y.data_ptr(), n, rp.data_ptr(), pm, None)
    torch.cuda.synchronize()
    assert torch.equal(y.view(torch.int16), y_ref.view(torch.int16))
    parts = rp.cpu().numpy().astype(np.uint32)
    assert (parts != 0xFFFFFFFF).all()  # every partial written
    np.testing.assert_array_equal(parts.max(axis=1), _rowmax_bits(y_ref))


def test_k5_batched_matches_per_layer_and_oracle(cuda):
    """qarvd_prepare_weights_batched == qarvd_prepare_weights per layer == oracle, over a
    batch of mixed shapes, ragged outlier sets, a single-scale plan and an all-zero group."""
    shapes = [(384, 8960, 188), (1536, 1536, 32), (96, 256, 0), (200, 1536, 5), (64, 512, 64)]
    ws, plans, refs = [], [], []
    for i, (n, k, no) in enumerate(shapes):
        plan = make_plan(k, no, seed=100 + i)
        bits, w64 = bf16_values((n, k), seed=200 + i, scale=1.0 / np.sqrt(k),
                                heavy_cols=plan.outlier_indices if no else None)
        if i == 4:  # an all-zero outlier group in some rows
            bits[:10, plan.outlier_indices] = 0
            w64 = oracle.bf16_bits_to_f64(bits)
        ws.append(to_dev_bf16(bits))
        plans.append(plan)
        refs.append(oracle.prepare_weights(w64, plan.gather, plan.k_outlier))
    layers = engine.prepare_weights_batched([f"l{i}" for i in range(len(ws))], ws, plans)
    for L, w, plan, (wq_ref, so_ref, sn_ref, bad) in zip(layers, ws, plans, refs):
        assert bad < 0
        np.testing.assert_array_equal(L.wq.cpu().numpy(), wq_ref)
        np.testing.assert_array_equal(L.scale_outlier64.cpu().numpy(), so_ref)
        np.testing.assert_array_equal(L.scale_normal64.cpu().numpy(), sn_ref)
        one = engine.prepare_weights("one", w, plan)
        assert torch.equal(one.wq, L.wq)
        assert torch.equal(one.scale_outlier32, L.scale_outlier32)
        assert torch.equal(one.scale_normal32, L.scale_normal32)


def test_k5_batched_nonfinite(cuda):
    plan = make_plan(512, 32, seed=3)
    bits, _ = bf16_values((40, 512), seed=4)
    bits[11, 7] = 0x7FC0
    with pytest.raises(qb.InvalidArgument, match="non-finite"):
        engine.prepare_weights_batched(["a"], [to_dev_bf16(bits)], [plan])


@pytest.mark.gpu
def test_wan_stack_chain_fold_invariant(cuda):
    """Config 3's stack (multi-consumer block inputs, a context input for cross k/v, per-layer
    rows, GELU on ffn.0) gives bit-identical outputs with and without the permutation folds."""
    from paper_2605_21072_b200 import synth
    from paper_2605_21072_b200.pipeline import QuantizedChain, wan_stack_chain
    ch = wan_stack_chain(blocks=2, m=300, text_len=64)
    assert len(ch.layers) == 20 and ch.ms[5] == 64 and ch.ms[6] == 64
    ref = QuantizedChain(ch.source_layers, ch.m, epilogues=ch.epilogues, inputs=ch.inputs, ms=ch.ms,
                         ctx_rows=64, fold=False)
    x = synth.synth_activation(300, synth.WAN_DIM, seed=3)
    c = synth.synth_activation(64, synth.WAN_DIM, seed=4)
    for chain in (ch, ref):
        chain.x.copy_(x)
        chain.ctx.copy_(c)
        chain.launch()
    torch.cuda.synchronize()
    assert torch.equal(ch.output.view(torch.int16), ref.output.view(torch.int16))
    for i in (0, 1, 5, 6):  # unfolded outputs (q, k of block 0; cross k, v)
        assert torch.equal(ch.y[i].view(torch.int16), ref.y[i].view(torch.int16))
    # graph replay reproduces the eager launch
    ch.capture()
    ch.replay()
    torch.cuda.synchronize()
    assert torch.equal(ch.output.view(torch.int16), ref.output.view(torch.int16))
    assert ch.int_ops() == ref.int_ops()
    # forked side branches (dead-end layers on side streams) reproduce every layer's output
    outs = [y.clone() for y in ch.y]
    for y in ch.y:
        y.zero_()
    ch.capture(parallel=True)
    ch.replay()
    torch.cuda.synchronize()
    for a, b in zip(outs, ch.y):
        assert torch.equal(a.view(torch.int16), b.view(torch.int16))


# ---------------------------------------------------------------- Eq. 5 weighted loss
def _ref_loss_case(n, k, n_out, rows, seed):
    r = np.random.default_rng(seed)
    outl = np.sort(r.choice(k, n_out, replace=False)) if n_out else np.zeros(0, np.int64)
    wb, w = bf16_values((n, k), seed=seed, scale=1.0 / np.sqrt(k), heavy_cols=outl if n_out else None)
    xb, x = bf16_values((sum(rows), k), seed=seed + 1, heavy_cols=outl if n_out else None, gamma=3.0)
    row_off = np.concatenate([[0], np.cumsum(rows)])
    chunks = (np.arange(len(rows)) % 3) + 1
    cw = calibrate.weighting_strategy("heuristic_exp", 3)
    ref = oracle.ref_weighted_loss(w, outl, np.abs(x).max() / 127.0, x, row_off, chunks, cw)
    plan = engine.build_plan("loss", k, outl)
    layer = engine.layer_from_codes("loss", ref["codes"], ref["s_wo"], ref["s_wn"], plan)
    xd = to_dev_bf16(xb)
    batch = [(xd[row_off[i]:row_off[i + 1]], int(chunks[i])) for i in range(len(rows))]
    return ref, layer, to_dev_bf16(wb), batch, cw, (x, w, row_off, chunks)


@pytest.mark.parametrize("n,k,n_out,rows", [(256, 512, 32, (40, 77, 13)), (300, 1536, 64, (200, 129)),
                                            (136, 320, 0, (128,)), (192, 896, 96, (1, 255, 256, 3))])
def test_weighted_loss_vs_reference(cuda, ref_lib, n, k, n_out, rows):
    """The fused tcgen05 Eq. 5 kernel vs the reference's f64 weighted_loss on the same
    reference-initialised LearnableQuantState (codes, group scales and act scale exported by
    the reference).  Tolerance rtol 2e-5: the GPU target is a bf16 x bf16 -> fp32 tensor-core
    product and the prediction uses the f32 copies of the scales (QARQ precision); the
    per-sample errors also match the oracle restatement to the same tolerance."""
    ref, layer, wd, batch, cw, (x, w, row_off, chunks) = _ref_loss_case(n, k, n_out, rows, seed=n + k)
    loss, err = calibrate.weighted_loss(batch, layer, wd, cw, ref["act_scale"], return_errors=True)
    assert np.isclose(loss, ref["loss"], rtol=2e-5, atol=0), (loss, ref["loss"])
    xq, _, _ = oracle.quantize_act(x, None, per_token=False, static_scale=ref["act_scale"])
    _, err_o = oracle.weighted_loss(x, xq, ref["act_scale"], w, ref["codes"], ref["s_wo"], ref["s_wn"],
                                    ref["mask"], row_off, chunks, cw)
    np.testing.assert_allclose(err, err_o, rtol=2e-5)


def test_weighted_loss_exact_zero_and_errors(cuda):
    """W and X on the quantization grids (power-of-two scales) -> every product is exact and
    the loss is exactly 0; the reference's error contract (calibrate.cpp:203, :207-208)."""
    r = np.random.default_rng(5)
    n, k = 256, 640
    codes = r.integers(-40, 41, size=(n, k))
    outl = np.arange(0, k, 20)[:32]
    plan = engine.build_plan("grid", k, outl)
    layer = engine.layer_from_codes("grid", codes, np.full(n, 2.0 ** -6), np.full(n, 2.0 ** -7), plan)
    wv = codes * np.where(np.isin(np.arange(k), outl), 2.0 ** -6, 2.0 ** -7)[None, :]
    xv = r.integers(-20, 21, size=(300, k)) * 2.0 ** -5
    xv[:, 0] = 127 * 2.0 ** -5  # keeps the static scale's codes in range
    wd = to_dev_bf16(oracle.f32_to_bf16_bits(wv.astype(np.float32)))
    xd = to_dev_bf16(oracle.f32_to_bf16_bits(xv.astype(np.float32)))
    loss, err = calibrate.weighted_loss([(xd[:100], 1), (xd[100:], 2)], layer, wd, [0.5, 0.5], 2.0 ** -5,
                                        return_errors=True)
    assert loss == 0.0 and np.all(err == 0.0)
    with pytest.raises(qb.OutOfRange, match="outside the weight vector"):
        calibrate.weighted_loss([(xd[:100], 3)], layer, wd, [0.5, 0.5], 2.0 ** -5)
    with pytest.raises(qb.InvalidArgument, match="empty batch"):
        calibrate.weighted_loss([], layer, wd, [0.5, 0.5], 2.0 ** -5)


def test_weighted_loss_wan_shape_sample_independence(cuda):
    """Full Wan shape (21 frames x 1560 tokens, 1536 -> 1536, K_o = 32): every sample's error
    from one batched call equals (bit-exactly) the same sample evaluated alone, and the loss is
    the chunk-weighted mean of those errors."""
    spec = synth.wan_registry(blocks=1)[0]
    w = synth.synth_weight(spec, seed=1)
    rep = qb.analyze_layer(spec.name, w)
    plan = engine.build_plan(spec.name, spec.in_dim, rep.aligned_outliers)
    layer = engine.prepare_weights(spec.name, w, plan)
    xs = [synth.synth_activation(1560, 1536, seed=3, frame=f) for f in range(21)]
    amax = max(float(x.float().abs().max()) for x in xs)
    cw = calibrate.weighting_strategy("heuristic_exp", 21)
    batch = [(x, f + 1) for f, x in enumerate(xs)]
    loss, err = calibrate.weighted_loss(batch, layer, w, cw, amax / 127.0, return_errors=True)
    assert np.all(err > 0)
    assert np.isclose(loss, float(np.dot(cw, err)) / 21, rtol=1e-14)
    for f in (0, 7, 20):
        _, e1 = calibrate.weighted_loss([batch[f]], layer, w, cw, amax / 127.0, return_errors=True)
        assert e1[0] == err[f]


@pytest.mark.parametrize("m,n,k,n_out", [(4680, 1536, 8960, 188), (3000, 1792, 16384, 60), (4680, 1536, 8960, 0)])
def test_k2_stream_k_bitexact(cuda, m, n, k, n_out, monkeypatch):
    """Stream-K K2 (qarvd_dual_gemm_ws: remainder tiles split along K over all SM pairs, int32
    partials through the workspace) is bit-identical to the data-parallel kernel, on repeated
    launches (self-resetting counters) and after another shape reused the workspace."""
    monkeypatch.setenv("QARVD_GEMM_SK", "1")  # stream-K is opt-in
    lib = qb._lib.load()
    plan = make_plan(k, n_out, seed=3)
    wb, _ = bf16_values((n, k), seed=4, scale=1.0 / np.sqrt(k), heavy_cols=plan.outlier_indices if n_out else None)
    L = engine.prepare_weights("sk", to_dev_bf16(wb), plan)
    xb, _ = bf16_values((m, k), seed=5, heavy_cols=plan.outlier_indices if n_out else None, gamma=4.0)
    xq, s32, _ = engine.kernel_a_quantize_activation(to_dev_bf16(xb), L)
    nb = int(lib.qarvd_dual_gemm_workspace_size(m, n, L.k_pad, L.k_outlier))
    assert nb > 0  # these shapes have a partial last wave and long K
    ws = torch.zeros(nb + 256, dtype=torch.uint8, device="cuda")
    y_dp = torch.empty((m, n), dtype=torch.bfloat16, device="cuda")
    y_sk = torch.empty_like(y_dp)
    qb._lib.call("qarvd_dual_gemm", xq.data_ptr(), L.k_pad, L.wq.data_ptr(), L.k_pad, m, n, L.k_pad,
                 L.k_outlier, s32.data_ptr(), L.scale_outlier32.data_ptr(), L.scale_normal32.data_ptr(),
                 None, qb.EPI_GELU, qb.BF16, y_dp.data_ptr(), n, None, None, None)
    for rep in range(3):
        y_sk.zero_()
        qb._lib.call("qarvd_dual_gemm_ws", xq.data_ptr(), L.k_pad, L.wq.data_ptr(), L.k_pad, m, n, L.k_pad,
                     L.k_outlier, s32.data_ptr(), L.scale_outlier32.data_ptr(), L.scale_normal32.data_ptr(),
                     None, qb.EPI_GELU, y_sk.data_ptr(), n, ws.data_ptr(), ws.numel(), None)
        torch.cuda.synchronize()
        assert torch.equal(y_dp.view(torch.int16), y_sk.view(torch.int16)), rep
    # counters are back to zero after every launch
    assert int(ws[:256].view(torch.int32).abs().sum()) == 0


# ---------------------------------------------------------------- K7 AdaRound calibrate_layer
@pytest.mark.parametrize("n,k,n_out,iters,batch", [(48, 64, 32, 60, 2), (96, 192, 32, 40, 3), (64, 128, 0, 30, 2),
                                                   (45, 100, 8, 20, 3),   # odd N: the DGEMM path
                                                   (38, 200, 0, 20, 4)])  # K off the 32 grid
def test_calibrate_layer_matches_reference(cuda, ref_lib, n, k, n_out, iters, batch):
    """K7 (f64 AdaRound on the GPU) follows the reference calibrate_layer: same sampler, same
    per-element formulas, f64 throughout -> identical hard codes and the learned scales, act
    scale, final loss and running-min trace within 1e-9 relative (cuBLAS DGEMM summation
    order)."""
    r = np.random.default_rng(n + k)
    outl = np.sort(r.choice(k, n_out, replace=False)) if n_out else np.zeros(0, np.int64)
    _, w = bf16_values((n, k), seed=n, scale=1.0 / np.sqrt(k), heavy_cols=outl if n_out else None)
    rows = [20, 13, 31, 8]
    _, x = bf16_values((sum(rows), k), seed=k, heavy_cols=outl if n_out else None, gamma=3.0)
    row_off = np.concatenate([[0], np.cumsum(rows)])
    chunks = np.array([1, 2, 3, 1])
    cw = calibrate.weighting_strategy("heuristic_exp", 3)
    act = float(np.abs(x).max() / 127.0)
    ref = oracle.ref_calibrate_layer(w, outl, act, x, row_off, chunks, cw, iters, batch, 11, "blk3.ffn.2")
    plan = engine.build_plan("blk3.ffn.2", k, outl)
    xd = torch.from_numpy(x).cuda()
    samples = [(xd[row_off[i]:row_off[i + 1]], int(chunks[i])) for i in range(len(rows))]
    cfg = qb._lib.CalibConfig(iterations=iters, batch_size=batch, seed=11)
    res = calibrate.calibrate_layer("blk3.ffn.2", torch.from_numpy(w).cuda(), plan,
                                    torch.from_numpy(ref["init_scale_normal"]).cuda(),
                                    torch.from_numpy(ref["init_scale_outlier"]).cuda(), act, samples, cw, cfg)
    np.testing.assert_array_equal(res.codes.astype(np.int32), ref["codes"])
    np.testing.assert_allclose(res.scale_normal, ref["scale_normal"], rtol=1e-9)
    if n_out:
        np.testing.assert_allclose(res.scale_outlier, ref["scale_outlier"], rtol=1e-9)
    assert np.isclose(res.act_scale, ref["act_scale"], rtol=1e-9)
    # the initial hard loss: V init and h(V) > 0.5 use glibc's exp/log restated bit for bit
    # (libm_ref.cuh), so the nearest-rounding codes are the reference's; only the f64 sums'
    # order (DGEMM vs the reference's sequential k loop) remains
    assert np.isclose(res.initial_loss, ref["initial_loss"], rtol=1e-12)
    assert np.isclose(res.final_loss, ref["final_loss"], rtol=1e-9)
    np.testing.assert_allclose(res.trace, ref["trace"], rtol=1e-9)


@pytest.mark.parametrize("w_bits,act_bits,n_out", [(4, 8, 8), (6, 4, 0), (3, 5, 4)])
def test_calibrate_layer_bit_widths(cuda, ref_lib, w_bits, act_bits, n_out):
    """K7 at other bit widths (W4A8 and narrower: calibrate_layer's weight qmax from the plan's
    weight_bits, the act qmax from its QuantParams): the reference's codes exactly, scales,
    act scale and final loss within 1e-9."""
    n, k = 24, 96
    r = np.random.default_rng(w_bits * 10 + act_bits)
    outl = np.sort(r.choice(k, n_out, replace=False)) if n_out else np.zeros(0, np.int64)
    _, w = bf16_values((n, k), seed=w_bits, scale=1.0 / np.sqrt(k), heavy_cols=outl if n_out else None)
    rows = [15, 22, 9]
    _, x = bf16_values((sum(rows), k), seed=act_bits + 40, heavy_cols=outl if n_out else None, gamma=3.0)
    row_off = np.concatenate([[0], np.cumsum(rows)])
    chunks = np.array([1, 2, 1])
    cw = np.array([1.0, 0.6])
    act = float(np.abs(x).max() / ((1 << (act_bits - 1)) - 1))
    ref = oracle.ref_calibrate_layer(w, outl, act, x, row_off, chunks, cw, 7, 2, 3, "blk1.ffn.0",
                                     w_bits=w_bits, act_bits=act_bits)
    plan = engine.build_plan("blk1.ffn.0", k, outl)
    xd = torch.from_numpy(x).cuda()
    samples = [(xd[row_off[i]:row_off[i + 1]], int(chunks[i])) for i in range(len(rows))]
    res = calibrate.calibrate_layer("blk1.ffn.0", torch.from_numpy(w).cuda(), plan,
                                    torch.from_numpy(ref["init_scale_normal"]).cuda(),
                                    torch.from_numpy(ref["init_scale_outlier"]).cuda(), act, samples, cw,
                                    qb._lib.CalibConfig(iterations=7, batch_size=2, seed=3),
                                    act_bits=act_bits, w_bits=w_bits)
    assert np.abs(res.codes).max() <= (1 << (w_bits - 1)) - 1
    np.testing.assert_array_equal(res.codes.astype(np.int32), ref["codes"])
    # below 8 activation bits x / s_a meets exact .5 ties often (bf16 x, s_a = max|x| / qmax):
    # s_a = exp(log s_a) is glibc's exp bit for bit (libm_ref.cuh), so the x codes agree and
    # every bit width is held to the same 1e-9 as 8 bits
    rtol = 1e-9
    np.testing.assert_allclose(res.scale_normal, ref["scale_normal"], rtol=rtol)
    if n_out:
        np.testing.assert_allclose(res.scale_outlier, ref["scale_outlier"], rtol=rtol)
    assert np.isclose(res.act_scale, ref["act_scale"], rtol=rtol)
    assert np.isclose(res.final_loss, ref["final_loss"], rtol=rtol)


def test_calibrate_layer_errors(cuda):
    plan = engine.build_plan("l", 64, [])
    w = torch.zeros((8, 64), dtype=torch.float64, device="cuda") + 0.1
    s = torch.full((8,), 0.1 / 127, dtype=torch.float64, device="cuda")
    x = torch.ones((4, 64), dtype=torch.float64, device="cuda")
    with pytest.raises(qb.InvalidArgument, match="no calibration samples"):
        calibrate.calibrate_layer("l", w, plan, s, s, 0.01, [], [1.0])
    with pytest.raises(qb.InvalidArgument, match="learning rates must be positive"):
        calibrate.calibrate_layer("l", w, plan, s, s, 0.01, [(x, 1)], [1.0], qb._lib.CalibConfig(lr_round=0.0))
    with pytest.raises(qb.OutOfRange, match="outside the weight vector"):
        calibrate.calibrate_layer("l", w, plan, s, s, 0.01, [(x, 2)], [1.0])


def test_calibrate_model_adaround_matches_reference_layers(cuda, ref_lib):
    """calibrate_model's AdaRound loop through the sharded driver (world 1; world 2 of the same
    records is tests/test_sharding_gloo.py): every slot equals the reference calibrate_layer of
    that layer — codes bit-exact, scales / final loss within 1e-9."""
    specs = [(24, 96, 4, "blk0.attn.q"), (40, 64, 0, "blk0.ffn.0"), (16, 128, 8, "blk0.ffn.2")]
    rows = [17, 9, 22]
    chunks = np.array([1, 2, 2])
    cw = calibrate.weighting_strategy("heuristic_exp", 2)
    cfg = qb._lib.CalibConfig(iterations=6, batch_size=2, seed=5)
    layers, samples, refs = [], [], []
    for li, (n, k, n_out, name) in enumerate(specs):
        r = np.random.default_rng(100 + li)
        outl = np.sort(r.choice(k, n_out, replace=False)) if n_out else np.zeros(0, np.int64)
        _, w = bf16_values((n, k), seed=li + 7, scale=1.0 / np.sqrt(k), heavy_cols=outl if n_out else None)
        _, x = bf16_values((sum(rows), k), seed=li + 70, heavy_cols=outl if n_out else None, gamma=3.0)
        row_off = np.concatenate([[0], np.cumsum(rows)])
        act = float(np.abs(x).max() / 127.0)
        ref = oracle.ref_calibrate_layer(w, outl, act, x, row_off, chunks, cw, 6, 2, 5, name)
        refs.append(ref)
        xd = torch.from_numpy(x).cuda()
        samples.append([(xd[row_off[i]:row_off[i + 1]], int(chunks[i])) for i in range(len(rows))])
        layers.append((name, torch.from_numpy(w).cuda(), engine.build_plan(name, k, outl),
                       torch.from_numpy(ref["init_scale_normal"]).cuda(),
                       torch.from_numpy(ref["init_scale_outlier"]).cuda(), act))
    got = calibrate.calibrate_model_adaround(layers, lambda i: samples[i], cw, cfg,
                                             sample_rows=[sum(rows)] * 3)
    assert [g.index for g in got] == [0, 1, 2]
    for g, ref, (n, k, n_out, name) in zip(got, refs, specs):
        assert g.result.layer == name and g.result.codes.shape == (n, k)
        np.testing.assert_array_equal(g.result.codes.astype(np.int32), ref["codes"])
        np.testing.assert_allclose(g.result.scale_normal, ref["scale_normal"], rtol=1e-9)
        assert np.isclose(g.result.final_loss, ref["final_loss"], rtol=1e-9)
        back = calibrate.unpack_calib_records(g.pack())[0]
        np.testing.assert_array_equal(back.result.codes, g.result.codes)


@pytest.mark.parametrize("m,n,k,n_out,epi", [(4680, 8960, 1536, 32, qb.EPI_GELU), (4680, 1536, 8960, 188, qb.EPI_NONE),
                                             (4680, 1536, 1536, 32, qb.EPI_NONE), (1000, 8960, 1536, 0, qb.EPI_GELU)])
def test_k2_deployed_path_full_shape(cuda, m, n, k, n_out, epi):
    """The deployed K2 path (bf16 TMA-store epilogue holding acc_n in registers, no debug dumps)
    at the full FFN / qkv shapes, on 48 sampled rows: bit-exact vs the oracle's fp32 epilogue
    (same op order) without GELU; with GELU within bf16 rounding of the f64 erf-GELU of the
    oracle's fp32 pre-activation (|err| <= 2^-8 |y| + 1e-6, the A&S erf bound is 3.4e-7)."""
    import math
    plan, layer, xq, s32, s64, _, _ = _gemm_case(m, n, k, n_out, seed=m % 97 + n)
    y = engine.kernel_b_gemm_dequant(xq, s32, layer, epilogue=epi)
    rows = np.sort(np.random.default_rng(m + n).choice(m, 48, replace=False))
    xq_h = xq.cpu().numpy()[rows]
    _, ao, an = oracle.kernel_b(xq_h, layer.wq.cpu().numpy(), plan.k_outlier, s64.cpu().numpy()[rows],
                                layer.scale_outlier64.cpu().numpy(), layer.scale_normal64.cpu().numpy(),
                                with_acc=True)
    yd = dev_bits(y)[rows]
    if epi == qb.EPI_NONE:
        y_ref = oracle.epilogue_f32(ao, an, plan.k_outlier > 0, s32.cpu().numpy()[rows],
                                    layer.scale_outlier32.cpu().numpy(), layer.scale_normal32.cpu().numpy())
        np.testing.assert_array_equal(yd, y_ref)
    else:
        v = oracle.epilogue_f32(ao, an, plan.k_outlier > 0, s32.cpu().numpy()[rows],
                                layer.scale_outlier32.cpu().numpy(), layer.scale_normal32.cpu().numpy(),
                                out="f32").astype(np.float64)
        erf = np.vectorize(math.erf)
        g = 0.5 * v * (1.0 + erf(v / math.sqrt(2.0)))
        yf = (yd.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
        assert np.all(np.abs(yf - g) <= 2.0 ** -8 * np.abs(g) + 1e-6)


def test_calibration_shard_sync_free_matches_per_layer(cuda):
    """CalibrationShard.run (K3 -> device plan -> K5 and K4 without a host round trip) gives
    the same outlier sets, plans, codes and scales as the per-layer host path (analyze_layer ->
    build_plan -> prepare_weights), and the same searched act scale as a per-layer K4 call."""
    specs = synth.wan_registry(blocks=1)
    ids = [0, 3, 6, 8, 9]  # q, o, cross v (512 text tokens), ffn.0, ffn.2
    frames, rows = 3, 40
    wts = calibrate.weighting_strategy("heuristic_exp", frames)
    shard = calibrate.CalibrationShard(specs, ids, frames, rows, frame_weights=wts)
    shard.setup()
    recs = shard.run()
    recs = shard.run()  # second step reuses the buffers (self-contained per step)
    layers = shard.deployed_layers()
    for rec, spec, w, x, L in zip(recs, shard.specs, shard.w, shard.x, layers):
        rep = qb.analyze_layer(spec.name, w)
        np.testing.assert_array_equal(rec.outliers, rep.aligned_outliers)
        plan = engine.build_plan(spec.name, spec.in_dim, rep.aligned_outliers)
        ref = engine.prepare_weights(spec.name, w, plan)
        assert torch.equal(L.wq, ref.wq)
        np.testing.assert_array_equal(rec.scale_outlier, ref.scale_outlier64.cpu().numpy())
        np.testing.assert_array_equal(rec.scale_normal, ref.scale_normal64.cpu().numpy())
        s = calibrate.unpack_search(calibrate.scale_search_async([x], frames, wts).cpu().numpy()[0])
        assert rec.act_scale == s.scale and rec.best_index == s.best_index


# ---------------------------------------------------------------- W4A8 (BitwidthScheme w4a8)
@pytest.mark.parametrize("wbits", [4, 6])
def test_w4a8_weights_and_linear(cuda, ref_lib, wbits):
    """Low-bit weights (the paper's W4A8 setting, BitwidthScheme): K5 at weight_bits = 4 (6)
    gives the reference's build_plan scales (absmax / 7) and codes bit-for-bit; the codes are
    stored as int8 (|code| <= 7) so K2 runs them unchanged -- at these token counts the GEMM is
    tensor-bound and packed int4 storage (tensor.cpp:221-264) would only save weight bytes --
    and its int32 accumulators and bf16 output stay bit-exact vs the oracle."""
    n, k, m = 384, 1536, 700
    plan = make_plan(k, 32, seed=4)
    wb, w64 = bf16_values((n, k), seed=11, scale=1.0 / np.sqrt(k), heavy_cols=plan.outlier_indices)
    ref = oracle.ref_build_plan_codes(w64, plan.outlier_indices, bits=wbits)
    layer = engine.prepare_weights("w4", to_dev_bf16(wb), plan, bits=wbits)
    np.testing.assert_array_equal(layer.scale_outlier64.cpu().numpy(), ref["scale_outlier"])
    np.testing.assert_array_equal(layer.scale_normal64.cpu().numpy(), ref["scale_normal"])
    np.testing.assert_array_equal(layer.wq.cpu().numpy().astype(np.int32), ref["wq"])
    qmax = (1 << (wbits - 1)) - 1
    assert int(layer.wq.abs().max()) <= qmax
    xb, x64 = bf16_values((m, k), seed=12, heavy_cols=plan.outlier_indices, gamma=4.0)
    xq, s32, s64 = engine.kernel_a_quantize_activation(to_dev_bf16(xb), layer)
    y, acc_o, acc_n = engine.kernel_b_gemm_dequant(xq, s32, layer, dump_acc=True)
    _, ao, an = oracle.kernel_b(xq.cpu().numpy(), layer.wq.cpu().numpy(), plan.k_outlier, s64.cpu().numpy(),
                                layer.scale_outlier64.cpu().numpy(), layer.scale_normal64.cpu().numpy(),
                                with_acc=True)
    np.testing.assert_array_equal(acc_o.cpu().numpy(), ao)
    np.testing.assert_array_equal(acc_n.cpu().numpy(), an)
    y_ref = oracle.epilogue_f32(ao, an, True, s32.cpu().numpy(), layer.scale_outlier32.cpu().numpy(),
                                layer.scale_normal32.cpu().numpy())
    np.testing.assert_array_equal(dev_bits(y), y_ref)


def test_bench_json_contract(cuda):
    """bench.py prints one JSON line with the driver's keys (short run, no calibration / stack)."""
    import json
    import subprocess
    import sys
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--steps", "5", "--warmup", "3",
                        "--no-calib", "--no-stack", "--no-cpu-baseline"], capture_output=True, text=True,
                       timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["steps"] == 5 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["value"] > 0
    assert d["gpu_launches"] >= 4 and d["e2e"]["h2d_bytes_per_step"] > 0
    rf = d["roofline"]
    assert rf["bound"] == "tensor" and 0 < rf["frac"] < 1 and rf["unit"] == "TOPS"
    assert "workload" in d["config"]


def test_fused_qkv_bitexact(cuda):
    """engine.fuse_siblings (one dual-slab layer for q, k, v) gives bit-identical outputs per
    column to the three separate layers, alone and inside the config-3 stack."""
    from paper_2605_21072_b200.pipeline import wan_stack_chain
    allspecs = synth.wan_registry(blocks=2)
    specs = [allspecs[0], allspecs[11], allspecs[2]]  # q0, k1, v0: outlier plans and a plain one
    Ls = []
    for spec in specs:
        w = synth.synth_weight(spec, seed=1)
        rep = qb.analyze_layer(spec.name, w)
        Ls.append(engine.prepare_weights(spec.name, w, engine.build_plan(spec.name, spec.in_dim, rep.aligned_outliers)))
    F = engine.fuse_siblings("qkv", Ls)
    x = synth.synth_activation(500, 1536, seed=5)
    xq, s32, _ = engine.kernel_a_quantize_activation(x, F)
    y = engine.kernel_b_gemm_dequant(xq, s32, F)
    for i, L in enumerate(Ls):
        xqi, si, _ = engine.kernel_a_quantize_activation(x, L)
        assert torch.equal(si, s32)
        yi = engine.kernel_b_gemm_dequant(xqi, si, L)
        assert torch.equal(y[:, i * 1536:(i + 1) * 1536].view(torch.int16), yi.view(torch.int16))
    a = wan_stack_chain(blocks=2, m=300, text_len=64)
    b = wan_stack_chain(blocks=2, m=300, text_len=64, fuse_qkv=True)
    xs = synth.synth_activation(300, 1536, seed=3)
    cs = synth.synth_activation(64, 1536, seed=4)
    for ch in (a, b):
        ch.x.copy_(xs)
        ch.ctx.copy_(cs)
        ch.launch()
    torch.cuda.synchronize()
    assert torch.equal(a.output.view(torch.int16), b.output.view(torch.int16))
    assert a.int_ops() == b.int_ops()
    b.capture(parallel=True)
    b.replay()
    torch.cuda.synchronize()
    assert torch.equal(a.output.view(torch.int16), b.output.view(torch.int16))


# ---------------------------------------------------------------- edge cases
@pytest.mark.parametrize("m,n,k,n_out", [(1, 16, 32, 0), (1, 24, 64, 3), (129, 16, 32, 0), (2, 8960, 8960, 188)])
def test_k2_tiny_and_single_row(cuda, m, n, k, n_out):
    """Single rows, N = 16 / 24 (ragged), K = 32 (one MMA step), and a 2-row FFN-down slice:
    accumulators and the bf16 output stay bit-exact."""
    plan, layer, xq, s32, s64, _, _ = _gemm_case(m, n, k, n_out, seed=m + n + k)
    y, acc_o, acc_n = engine.kernel_b_gemm_dequant(xq, s32, layer, dump_acc=True)
    _, ao, an = oracle.kernel_b(xq.cpu().numpy(), layer.wq.cpu().numpy(), plan.k_outlier, s64.cpu().numpy(),
                                layer.scale_outlier64.cpu().numpy(), layer.scale_normal64.cpu().numpy(),
                                with_acc=True)
    np.testing.assert_array_equal(acc_o.cpu().numpy(), ao)
    np.testing.assert_array_equal(acc_n.cpu().numpy(), an)
    y2 = engine.kernel_b_gemm_dequant(xq, s32, layer)  # deployed path (no dumps)
    y_ref = oracle.epilogue_f32(ao, an, plan.k_outlier > 0, s32.cpu().numpy(), layer.scale_outlier32.cpu().numpy(),
                                layer.scale_normal32.cpu().numpy())
    np.testing.assert_array_equal(dev_bits(y2), y_ref)


def test_k1_empty_batch_is_a_noop(cuda):
    plan = make_plan(256, 32, seed=1)
    x = torch.empty((0, 256), dtype=torch.bfloat16, device="cuda")
    xq, s32, s64 = engine.kernel_a_quantize_activation(x, plan)
    assert xq.shape == (0, plan.k_pad) and s32.numel() == 0


def test_weighted_loss_single_row_samples(cuda, ref_lib):
    """Eq. 5 with one-row and 129-row samples (ragged against the 256-row pair tiles)."""
    ref, layer, wd, batch, cw, (x, w, row_off, chunks) = _ref_loss_case(64, 256, 32, (1, 129, 1), seed=77)
    loss, err = calibrate.weighted_loss(batch, layer, wd, cw, ref["act_scale"], return_errors=True)
    assert np.isclose(loss, ref["loss"], rtol=2e-5)


def test_calibrate_layer_zero_iterations_and_large_batch(cuda, ref_lib):
    """iterations = 0 returns the initial (nearest-rounding) state; a batch larger than the
    sample set samples with replacement like the reference."""
    r = np.random.default_rng(3)
    n, k = 32, 64
    outl = np.sort(r.choice(k, 32, replace=False))
    _, w = bf16_values((n, k), seed=5, scale=0.125, heavy_cols=outl)
    _, x = bf16_values((30, k), seed=6, heavy_cols=outl, gamma=3.0)
    row_off = np.array([0, 10, 30])
    chunks = np.array([1, 2])
    cw = calibrate.weighting_strategy("heuristic_exp", 2)
    act = float(np.abs(x).max() / 127.0)
    plan = engine.build_plan("z", k, outl)
    xd = torch.from_numpy(x).cuda()
    samples = [(xd[0:10], 1), (xd[10:30], 2)]
    for iters, batch in ((0, 2), (12, 5)):
        ref = oracle.ref_calibrate_layer(w, outl, act, x, row_off, chunks, cw, iters, batch, 3, "z")
        res = calibrate.calibrate_layer("z", torch.from_numpy(w).cuda(), plan,
                                        torch.from_numpy(ref["init_scale_normal"]).cuda(),
                                        torch.from_numpy(ref["init_scale_outlier"]).cuda(), act, samples, cw,
                                        qb._lib.CalibConfig(iterations=iters, batch_size=batch, seed=3))
        # nearest-rounding init and the hard decisions follow glibc's exp/log bit for bit:
        # identical codes even where w/s sits on an exact .5 tie
        np.testing.assert_array_equal(res.codes.astype(np.int32), ref["codes"])
        np.testing.assert_allclose(res.scale_normal, ref["scale_normal"], rtol=1e-9)
        assert np.isclose(res.final_loss, ref["final_loss"], rtol=1e-9)
        assert len(res.trace) == iters
        if iters == 0:
            assert res.final_loss == res.initial_loss


@pytest.mark.parametrize("wbits", [8, 4])
def test_qarq_loaded_layers_run_on_device(cuda, ref_lib, tmp_path, wbits):
    """A QARQ file written by the reference pipeline, loaded by qarq.load_qarq and uploaded by
    qarq.to_device: K1 codes bit-exact vs the reference quantize with the file's static act
    scale, and the bf16 K2 output within the stated tolerance of kernel_b_gemm_dequant.  At
    W4 the file holds packed 4-bit codes, uploaded packed and expanded on the device
    (qarvd_unpack_codes_i4): the device codes equal the reference loader's exactly."""
    from paper_2605_21072_b200 import qarq
    path = str(tmp_path / "toy.qarq")
    oracle.ref_toy_qarq(path, iterations=4, weight_bits=wbits)
    _, layers = qarq.load_qarq(path)
    checked = 0
    for i, L in enumerate(layers):
        if L.preserved:
            with pytest.raises(qb.InvalidArgument):
                qarq.to_device(L)
            continue
        ref = oracle.ref_qarq_layer(path, i)
        assert L.bits == wbits and (L.codes_packed is not None) == (wbits == 4)
        D = qarq.to_device(L)
        n_o = ref["outlier_count"]
        wq_dev = D.wq.cpu().numpy().astype(np.int32)
        np.testing.assert_array_equal(wq_dev[:, :n_o], ref["wq"][:, :n_o])
        np.testing.assert_array_equal(wq_dev[:, D.k_outlier:D.k_outlier + L.in_dim - n_o], ref["wq"][:, n_o:])
        assert not wq_dev[:, n_o:D.k_outlier].any() and not wq_dev[:, D.k_outlier + L.in_dim - n_o:].any()
        xb, x64 = bf16_values((37, L.in_dim), seed=i, gamma=3.0)
        xq, s32, s64 = engine.kernel_a_quantize_activation(to_dev_bf16(xb), D, qb.ACT_PER_TENSOR,
                                                           static_scale=ref["act_scale"])
        perm = ref["permutation"]
        codes, _ = oracle.ref_quantize(oracle.ref_permute(x64, perm, ref["enabled"]), per_token=False,
                                       s=ref["act_scale"])
        n_o = ref["outlier_count"]
        xq_h = xq.cpu().numpy()
        np.testing.assert_array_equal(xq_h[:, :n_o], codes[:, :n_o])
        np.testing.assert_array_equal(xq_h[:, D.k_outlier:D.k_outlier + L.in_dim - n_o], codes[:, n_o:])
        y_ref = oracle.ref_kernel_b(codes, ref["wq"], perm, n_o, ref["enabled"], np.full(37, ref["act_scale"]),
                                    ref["scale_outlier"], ref["scale_normal"])
        y, acc_o, acc_n = engine.kernel_b_gemm_dequant(xq, s32, D, dump_acc=True)
        mag = (np.abs(ref["act_scale"] * ref["scale_outlier"][None] * acc_o.cpu().numpy()) +
               np.abs(ref["act_scale"] * ref["scale_normal"][None] * acc_n.cpu().numpy()))
        yd = y.float().cpu().numpy().astype(np.float64)
        assert np.all(np.abs(yd - y_ref) <= 2.0 ** -8 * np.abs(y_ref) + 2.0 ** -22 * mag + 1e-30)
        checked += 1
    assert checked > 0


def test_qarq_asymmetric_activations_on_device(cuda, ref_lib, tmp_path):
    """Asymmetric static activations (QARQ act_symmetric = false with a zero point, the loader
    branch engine.cpp:288-295): K1 codes clamp(rint(x / s) + z, -128, 127) bit-exact, and the
    bf16 output against kernel B's f64 formula with the zero-point column-sum correction
    (engine.cpp:86-100, restated here in f64 from the oracle's exact group accumulators)."""
    from paper_2605_21072_b200 import qarq
    path = str(tmp_path / "toy.qarq")
    oracle.ref_toy_qarq(path, iterations=2)
    _, layers = qarq.load_qarq(path)
    checked = 0
    for i, L in enumerate(layers):
        if L.preserved:
            continue
        L.act_symmetric, L.act_zero = False, (-9 if i % 2 else 13)
        D = qarq.to_device(L)
        s_x = float(np.float32(L.act_scale))
        xb, x64 = bf16_values((29, L.in_dim), seed=50 + i, gamma=3.0)
        xq, s32, _ = engine.kernel_a_quantize_activation(to_dev_bf16(xb), D, qb.ACT_PER_TENSOR, static_scale=s_x)
        g = D.plan.gather
        xg = np.where(g[None, :] >= 0, x64[:, np.maximum(g, 0)], 0.0)
        codes = np.where(g[None, :] >= 0, np.clip(np.rint(xg / s_x) + L.act_zero, -128, 127), 0).astype(np.int8)
        np.testing.assert_array_equal(xq.cpu().numpy(), codes)
        y, acc_o, acc_n = engine.kernel_b_gemm_dequant(xq, s32, D, dump_acc=True)
        so, sn = D.scale_outlier64.cpu().numpy(), D.scale_normal64.cpu().numpy()
        w = D.wq.cpu().numpy().astype(np.int64)
        ao, an = acc_o.cpu().numpy().astype(np.float64), acc_n.cpu().numpy().astype(np.float64)
        # engine.cpp:86-100: val = sum_g (s_x s_g) acc_g - (z s_x) sum_g s_g colsum_g
        if D.k_outlier > 0:
            val = (s_x * so)[None] * ao + (s_x * sn)[None] * an
            corr = so * w[:, :D.k_outlier].sum(1) + sn * w[:, D.k_outlier:].sum(1)
        else:
            val = (s_x * sn)[None] * (ao + an)
            corr = sn * w.sum(1)
        y_ref = val - (L.act_zero * s_x) * corr[None]
        mag = np.abs((s_x * so)[None] * ao) + np.abs((s_x * sn)[None] * an) + np.abs(L.act_zero * s_x * corr)[None]
        yd = y.float().cpu().numpy().astype(np.float64)
        assert np.all(np.abs(yd - y_ref) <= 2.0 ** -8 * np.abs(y_ref) + 2.0 ** -22 * mag + 1e-30)
        checked += 1
    assert checked > 0


# ---------------------------------------------------------------- full config shapes
def _bf16_bits(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def _verify_chain_rows(chain, rows, ctx_rows):
    """Every layer of a launched QuantizedChain checked on sampled rows against the oracle:
    the layer's GPU input rows -> oracle K1 (quantize_act with the layer's gather, per-token)
    -> oracle kernel B (exact int32 accumulators, both slabs) -> the fp32 epilogue
    restatement.  K1 codes / scales and the bf16 outputs must be bit-identical; a GELU layer's
    output (MUFU rcp / ex2 in the device GELU) within one bf16 ulp of erf-GELU on the exact
    fp32 pre-activation.  Returns (layers checked, elements compared)."""
    n_el = 0
    for i, L in enumerate(chain.layers):
        src = chain._src(i)
        r = ctx_rows if chain.inputs[i] == -2 else rows
        x_bits = _bf16_bits(src[r])
        x64 = oracle.bf16_bits_to_f64(x_bits)
        g = None if L.gather_dev is None else L.gather_dev.cpu().numpy()
        q, s64, _ = oracle.quantize_act(x64, g, per_token=True)
        np.testing.assert_array_equal(chain.xq[i][r].cpu().numpy(), q, err_msg=f"K1 codes, layer {i} {L.name}")
        np.testing.assert_array_equal(chain.sx[i][r].cpu().numpy(), s64.astype(np.float32),
                                      err_msg=f"K1 scales, layer {i}")
        _, ao, an = oracle.kernel_b(q, L.wq.cpu().numpy(), L.k_outlier, s64, L.scale_outlier64.cpu().numpy(),
                                    L.scale_normal64.cpu().numpy(), with_acc=True)
        bias = None if L.bias is None else L.bias.cpu().numpy()
        got = _bf16_bits(chain.y[i][r])
        if chain.epilogues[i] == qb.EPI_GELU:
            f32 = oracle.epilogue_f32(ao, an, L.k_outlier > 0, s64.astype(np.float32),
                                      L.scale_outlier32.cpu().numpy(), L.scale_normal32.cpu().numpy(), bias, out="f32")
            t = torch.from_numpy(f32).double()
            ref = (0.5 * t * (1 + torch.erf(t / np.sqrt(2.0)))).float()
            got_f = torch.from_numpy(got.view(np.int16)).view(torch.bfloat16).float()
            # one bf16 ulp (2^-7 relative) plus the device GELU's 3.4e-7 absolute error bound
            assert torch.all((got_f - ref).abs() <= 2.0 ** -7 * ref.abs() + 1e-6), f"GELU layer {i}"
        else:
            ref_bits = oracle.epilogue_f32(ao, an, L.k_outlier > 0, s64.astype(np.float32),
                                           L.scale_outlier32.cpu().numpy(), L.scale_normal32.cpu().numpy(), bias)
            np.testing.assert_array_equal(got, ref_bits, err_msg=f"K2 output, layer {i} {L.name}")
        n_el += got.size
    return len(chain.layers), n_el


def test_config3_stack_rows_vs_oracle_chain(cuda):
    """Config 3 at its real shape: the 30-block Wan stack (300 linears, q/k/v and cross k/v
    fused as in bench.py, M = 4680, 512 text tokens), replayed from its parallel CUDA graph;
    64 seeded token rows (and 32 text rows) of every layer vs the oracle chain."""
    from paper_2605_21072_b200.pipeline import wan_stack_chain
    chain = wan_stack_chain(fuse_qkv=True)
    chain.x.copy_(synth.synth_activation(chain.m, synth.WAN_DIM, seed=11))
    chain.ctx.copy_(synth.synth_activation(synth.WAN_TEXT_LEN, synth.WAN_DIM, seed=13))
    chain.capture(parallel=True)
    chain.replay()
    torch.cuda.synchronize()
    r = np.random.default_rng(3)
    rows = torch.from_numpy(np.sort(r.choice(chain.m, 64, replace=False))).cuda()
    ctx_rows = torch.from_numpy(np.sort(r.choice(synth.WAN_TEXT_LEN, 32, replace=False))).cuda()
    n_layers, n_el = _verify_chain_rows(chain, rows, ctx_rows)
    assert n_layers == 30 * 7 and n_el > 64 * 1536 * 200


def test_config5_rollout_step_rows_vs_oracle_chain(cuda):
    """Config 5's batched stack: the 8 rollouts of one GPU batched along M (M = 8 x 4680), one
    denoising step's stack forward; 64 seeded rows spread over the rollouts vs the oracle chain."""
    from paper_2605_21072_b200.pipeline import QuantizedChain, wan_stack_chain
    base = wan_stack_chain(fuse_qkv=True, blocks=6)
    per = 8
    rc = QuantizedChain(base.layers, per * base.m, epilogues=base.epilogues, inputs=base.raw_inputs,
                        ms=[per * mi for mi in base.ms], ctx_rows=per * base.ctx.shape[0])
    del base
    rc.x.copy_(synth.synth_activation(rc.x.shape[0], synth.WAN_DIM, seed=1000, frame=0))
    rc.ctx.copy_(synth.synth_activation(rc.ctx.shape[0], synth.WAN_DIM, seed=17))
    rc.launch_parallel()
    torch.cuda.synchronize()
    r = np.random.default_rng(5)
    rows = torch.from_numpy(np.sort(r.choice(rc.x.shape[0], 64, replace=False))).cuda()
    ctx_rows = torch.from_numpy(np.sort(r.choice(rc.ctx.shape[0], 32, replace=False))).cuda()
    n_layers, _ = _verify_chain_rows(rc, rows, ctx_rows)
    assert n_layers == 6 * 7


@pytest.mark.parametrize("k,seed", [(1536, 1), (8960, 2)])
def test_k4_full_wan_shape_vs_oracle(cuda, k, seed):
    """Config 4 at its real shape: one layer's 21 frames x 1560 tokens (K = 1536, and the
    ffn.2 input width K = 8960: 293 M values), heuristic_exp frame weights; thresholds, scales,
    losses and the selection bit-identical to the oracle's histogram restatement."""
    frames, rows = synth.WAN_FRAMES, synth.WAN_TOKENS_PER_FRAME
    xs = torch.cat([synth.synth_activation(rows, k, seed=seed, frame=f) for f in range(frames)])
    w = calibrate.weighting_strategy("heuristic_exp", frames)
    res = calibrate.scale_search_async([xs], frames, w).cpu().numpy()[0]
    bits = _bf16_bits(xs)
    del xs
    np.testing.assert_array_equal(res, oracle.scale_search_hist(bits, frames, rows, k, weights=w))


def test_k4_full_wan_shape_uniform_vs_reference(cuda, ref_lib):
    """The uniform-weight limit at 21 x 1560 x 1536 against the compiled reference's
    init_scale_percentile_search (pooled full sort, quant.cpp:190-226; ~5 s on one core): same
    percentile, bit-identical scale, candidate MSEs within 1e-12."""
    frames, rows, k = synth.WAN_FRAMES, synth.WAN_TOKENS_PER_FRAME, synth.WAN_DIM
    xs = torch.cat([synth.synth_activation(rows, k, seed=3, frame=f) for f in range(frames)])
    res = calibrate.scale_search_async([xs], frames, None).cpu().numpy()[0]
    x64 = oracle.bf16_bits_to_f64(_bf16_bits(xs))
    del xs
    best_pct, scale, mse = oracle.ref_percentile_search(x64, frames, rows, k)
    assert calibrate.PERCENTILES[int(res[9])] == best_pct
    assert res[10] == scale
    np.testing.assert_allclose(res[6:9], mse, rtol=1e-12)


def test_percentile_search_f64_full_shape_vs_reference(cuda, ref_lib):
    """The drop-in's f64 percentile search (qarvd_percentile_search_f64: device radix select of
    the order statistics + double-double MSEs) on 21 f64 samples of 1560 x 1536 against the
    compiled reference: same percentile, bit-identical scale and thresholds' scales."""
    frames, rows, k = synth.WAN_FRAMES, synth.WAN_TOKENS_PER_FRAME, synth.WAN_DIM
    xs = torch.cat([synth.synth_activation(rows, k, seed=5, frame=f) for f in range(frames)]).double()
    x64 = xs.cpu().numpy()
    offs = (np.arange(frames + 1, dtype=np.int64) * rows * k)
    pct = np.array(calibrate.PERCENTILES, dtype=np.float64)
    res = torch.empty(3 * len(pct) + 2, dtype=torch.float64, device="cuda")
    err = torch.empty(2, dtype=torch.int64, device="cuda")
    qb._lib.call("qarvd_percentile_search_f64", xs.data_ptr(), offs.ctypes.data, frames, pct.ctypes.data, len(pct),
                 8, res.data_ptr(), err.data_ptr(), None)
    res = res.cpu().numpy()
    assert err.cpu().numpy()[0] == -1
    best_pct, scale, mse = oracle.ref_percentile_search(x64, frames, rows, k)
    assert pct[int(res[9])] == best_pct and res[10] == scale
    # the reference sums each sample's 2.4 M squared errors sequentially in f64 (~1e-12 relative
    # rounding at this length); the device sum is double-double, i.e. the exact sum rounded
    np.testing.assert_allclose(res[6:9], mse, rtol=1e-10)


@pytest.mark.parametrize("bn,cg,ks", [(128, 1, 1), (128, 1, 2), (128, 2, 1), (128, 2, 2), (256, 2, 1), (256, 2, 2)])
def test_k2_tile_overrides_bitexact(cuda, monkeypatch, bn, cg, ks):
    """Every tile configuration reachable through QARVD_GEMM_BN / _CG / _KS gives the default
    configuration's bf16 output bit for bit (config 1 and the FFN-down shape)."""
    for n, k, n_out in ((1536, 1536, 32), (1536, 8960, 188)):
        spec = synth.LayerSpec(7, "l", n, k, 4680, n_out / k, 8.0)
        w = synth.synth_weight(spec, seed=1)
        L = engine.prepare_weights("l", w, engine.build_plan("l", k, qb.analyze_layer("l", w).aligned_outliers))
        xq, sx, _ = engine.kernel_a_quantize_activation(synth.synth_activation(1000, k, seed=3), L)
        ref = engine.kernel_b_gemm_dequant(xq, sx, L)
        monkeypatch.setenv("QARVD_GEMM_BN", str(bn))
        monkeypatch.setenv("QARVD_GEMM_CG", str(cg))
        monkeypatch.setenv("QARVD_GEMM_KS", str(ks))
        y = engine.kernel_b_gemm_dequant(xq, sx, L)
        for v in ("QARVD_GEMM_BN", "QARVD_GEMM_CG", "QARVD_GEMM_KS"):
            monkeypatch.delenv(v)
        torch.cuda.synchronize()
        assert torch.equal(y.view(torch.int16), ref.view(torch.int16)), (n, k)


# ---------------------------------------------------------------- K1 bulk-staged variant (opt-in)
@pytest.mark.parametrize("m,k,n_out,gathered", [(4680, 1536, 32, True), (4680, 8960, 0, False),
                                                (257, 1536, 0, True), (300, 2048, 0, False), (33, 200, 5, True)])
def test_k1_bulk_staged_bitexact(cuda, monkeypatch, m, k, n_out, gathered):
    """QARVD_K1_BULK=1 (persistent CTAs, rows staged by cp.async.bulk): same codes and scales as
    the oracle, with and without the plan gather, including tie rows."""
    monkeypatch.setenv("QARVD_K1_BULK", "1")
    plan = make_plan(k, n_out, seed=m + 1)
    bits, x64 = bf16_values((m, k), seed=k + 7 * m, heavy_cols=plan.outlier_indices if n_out else None)
    # a few rows of exact .5 ties
    for i in range(min(m, 8)):
        a = float(2.0 ** (i - 3))
        row = (np.arange(k, dtype=np.float64) % 255 - 127) * (a / 127.0) * 0.5
        row[0] = a
        bits[i] = oracle.f32_to_bf16_bits(row.astype(np.float32))
    x64 = oracle.bf16_bits_to_f64(bits)
    x = to_dev_bf16(bits)
    g = plan.gather if gathered else None
    kout = plan.k_pad if gathered else k
    xq = torch.empty((m, kout), dtype=torch.int8, device="cuda")
    s64 = torch.empty(m, dtype=torch.float64, device="cuda")
    gdev = torch.from_numpy(plan.gather.astype(np.int32)).cuda() if gathered else None
    qb._lib.call("qarvd_quantize_act", x.data_ptr(), qb.BF16, m, k, k, None if gdev is None else gdev.data_ptr(),
                 kout, qb.ACT_PER_TOKEN, 0.0, 8, xq.data_ptr(), kout, None, s64.data_ptr(), None, None)
    q_ref, s_ref, _ = oracle.quantize_act(x64, g, per_token=True)
    np.testing.assert_array_equal(xq.cpu().numpy(), q_ref)
    np.testing.assert_array_equal(s64.cpu().numpy(), s_ref)


# ---------------------------------------------------------------- K2 with the consumer's K1 fused
def _qz_pair(y_codes_ws, m, n, k, ko, gelu, xq, wq, sx, swo, swn, bias, reps=2, static=None):
    """Unfused (qarvd_dual_gemm -> qarvd_quantize_act) and fused (qarvd_dual_gemm_quant) runs;
    static = a per-tensor activation scale (None: per-token)."""
    gran = qb.ACT_PER_TOKEN if static is None else qb.ACT_PER_TENSOR
    sst = 0.0 if static is None else float(static)
    lib = qb._lib
    epi = qb.EPI_GELU if gelu else qb.EPI_NONE
    y = torch.empty((m, n), dtype=torch.bfloat16, device="cuda")
    q_ref = torch.empty((m, n), dtype=torch.int8, device="cuda")
    s_ref = torch.empty(m, dtype=torch.float32, device="cuda")
    d_ref = torch.empty(m, dtype=torch.float64, device="cuda")
    e_ref = torch.empty(1, dtype=torch.int64, device="cuda")
    lib.call("qarvd_dual_gemm", xq.data_ptr(), k, wq.data_ptr(), k, m, n, k, ko, sx.data_ptr(),
             swo.data_ptr(), swn.data_ptr(), None if bias is None else bias.data_ptr(), epi, qb.BF16,
             y.data_ptr(), n, None, None, None)
    lib.call("qarvd_quantize_act", y.data_ptr(), qb.BF16, m, n, n, None, n, gran, sst, 8,
             q_ref.data_ptr(), n, s_ref.data_ptr(), d_ref.data_ptr(), e_ref.data_ptr(), None)
    ws = y_codes_ws
    outs = []
    for _ in range(reps):  # the workspace resets itself between launches
        q = torch.full((m, n), 99, dtype=torch.int8, device="cuda")
        s = torch.empty(m, dtype=torch.float32, device="cuda")
        d = torch.empty(m, dtype=torch.float64, device="cuda")
        e = torch.empty(1, dtype=torch.int64, device="cuda")
        lib.call("qarvd_dual_gemm_quant", xq.data_ptr(), k, wq.data_ptr(), k, m, n, k, ko, sx.data_ptr(),
                 swo.data_ptr(), swn.data_ptr(), None if bias is None else bias.data_ptr(), epi, gran, sst, 8,
                 q.data_ptr(), n, s.data_ptr(), d.data_ptr(), e.data_ptr(), ws.data_ptr(), ws.numel(), None)
        torch.cuda.synchronize()
        outs.append((q, s, d, e))
    # the row-block counters grow by (N tiles x 2 CTAs) per launch, the epoch by one
    nb = (m + 255) // 256
    w64 = ws.view(torch.int64)
    if static is None:
        assert torch.all(w64[m:m + nb] == reps * (n // 256) * 2)
    assert int(w64[m + nb].item()) == reps
    return (q_ref, s_ref, d_ref, e_ref), outs


@pytest.mark.parametrize("static", [None, 0.02])
@pytest.mark.parametrize("m,n,k,ko,gelu,bias", [(4680, 8960, 1536, 32, True, True), (300, 512, 256, 0, False, False),
                                                (1000, 1536, 8960, 192, False, True), (33, 256, 64, 32, True, False)])
def test_k2_fused_quant_bitexact(cuda, m, n, k, ko, gelu, bias, static):
    """qarvd_dual_gemm_quant = qarvd_dual_gemm (bf16) then the per-token K1 on its output: same
    codes, f32 / f64 scales and error index, launch after launch (self-resetting workspace),
    including partial row blocks (m % 256 != 0)."""
    g = torch.Generator(device="cpu").manual_seed(m + n)
    xq = torch.randint(-127, 128, (m, k), generator=g, dtype=torch.int8).cuda()
    wq = torch.randint(-127, 128, (n, k), generator=g, dtype=torch.int8).cuda()
    sx = (torch.rand(m, generator=g) * 0.02 + 1e-3).cuda()
    swo = (torch.rand(n, generator=g) * 1e-3 + 1e-4).cuda()
    swn = (torch.rand(n, generator=g) * 1e-3 + 1e-4).cuda()
    b = (torch.rand(n, generator=g) - 0.5).cuda() if bias else None
    ws = torch.zeros(int(qb._lib.load().qarvd_dual_gemm_quant_workspace_size(m)), dtype=torch.uint8, device="cuda")
    ref, outs = _qz_pair(ws, m, n, k, ko, gelu, xq, wq, sx, swo, swn, b, static=static)
    for q, s, d, e in outs:
        assert torch.equal(q, ref[0])
        assert torch.equal(s.view(torch.int32), ref[1].view(torch.int32))
        assert torch.equal(d.view(torch.int64), ref[2].view(torch.int64))
        assert int(e.item()) == int(ref[3].item()) == 2 ** 63 - 1


@pytest.mark.parametrize("static", [None, 2.0 ** -4])
def test_k2_fused_quant_ties_and_nonfinite(cuda, static):
    """Exact .5 ties (every odd code of half the columns lands on k + 1/2) take the reference's
    division, and a row overflowing to inf reports the same flat index as K1."""
    m, n, k = 512, 512, 512
    g = torch.Generator(device="cpu").manual_seed(5)
    codes = torch.randint(-126, 127, (m, k), generator=g, dtype=torch.int8)
    codes[:, 0] = 127
    xq = codes.cuda()
    wq = torch.eye(n, k, dtype=torch.int8).cuda()  # acc_n = the codes
    c = 2.0 ** -4
    swn = torch.tensor([c if j % 2 == 0 else c / 2 for j in range(n)], dtype=torch.float32).cuda()
    swo = swn.clone()
    sx = torch.ones(m, dtype=torch.float32).cuda()
    sx[77] = 3e38  # y overflows: non-finite row
    ws = torch.zeros(int(qb._lib.load().qarvd_dual_gemm_quant_workspace_size(m)), dtype=torch.uint8, device="cuda")
    ref, outs = _qz_pair(ws, m, n, k, 0, False, xq, wq, sx, swo, swn, None, static=static)
    assert int(ref[3].item()) == 77 * n + 0
    for q, s, d, e in outs:
        assert torch.equal(q, ref[0])
        assert torch.equal(s.view(torch.int32), ref[1].view(torch.int32))
        assert torch.equal(d.view(torch.int64), ref[2].view(torch.int64))
        assert int(e.item()) == int(ref[3].item())
    # the ties are real: odd codes in odd columns halve to k + 1/2 and round half to even
    row = codes[3].numpy().astype(np.int64)
    want = np.where(np.arange(k) % 2 == 1, np.rint(row / 2.0), row)
    np.testing.assert_array_equal(ref[0][3].cpu().numpy().astype(np.int64), want)


@pytest.mark.parametrize("static", [False, True])
def test_chain_fused_quant_bitexact(cuda, static):
    """QuantizedChain(fuse_quant=True) on the Wan FFN: ffn.2's codes, scales and the final output
    equal the unfused folded chain's, replayed from a CUDA graph (per-token and static ffn.2)."""
    from paper_2605_21072_b200.pipeline import QuantizedChain
    d, f, m = 1536, 8960, 4680
    p0, p2 = make_plan(d, 32, seed=1), make_plan(f, 192, seed=2)
    w0, _ = bf16_values((f, d), seed=4, scale=1.0 / np.sqrt(d), heavy_cols=p0.outlier_indices)
    w2, _ = bf16_values((d, f), seed=5, scale=1.0 / np.sqrt(f), heavy_cols=p2.outlier_indices)
    L0 = engine.prepare_weights("ffn.0", to_dev_bf16(w0), p0)
    L2 = engine.prepare_weights("ffn.2", to_dev_bf16(w2), p2)
    L0.bias = torch.linspace(-0.5, 0.5, f, device="cuda", dtype=torch.float32)
    if static:
        L2.act_granularity, L2.act_scale = qb.ACT_PER_TENSOR, 0.01
    xb, _ = bf16_values((m, d), seed=6, heavy_cols=p0.outlier_indices, gamma=4.0)
    outs = []
    for fq in (False, True):
        ch = QuantizedChain([L0, L2], m, epilogues=[qb.EPI_GELU, qb.EPI_NONE], fuse_quant=fq)
        assert (ch.qz_into[0] == 1) == fq
        ch.x.copy_(to_dev_bf16(xb))
        ch.capture()
        for _ in range(3):
            ch.replay()
        torch.cuda.synchronize()
        outs.append((ch.xq[1].clone(), ch.sx[1].clone(), ch.output.clone()))
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][1], outs[1][1])
    assert torch.equal(outs[0][2].view(torch.int16), outs[1][2].view(torch.int16))


@pytest.mark.parametrize("m", [1, 255, 256, 257, 511])
def test_k2_fused_quant_row_block_edges(cuda, m):
    """Row counts at the 256-row block edges (a single row, one short / exact / one over a block):
    the per-token fused quantizer's row-block counting and the partial last block stay exact."""
    n, k, ko = 512, 128, 32
    g = torch.Generator(device="cpu").manual_seed(m)
    xq = torch.randint(-127, 128, (m, k), generator=g, dtype=torch.int8).cuda()
    wq = torch.randint(-127, 128, (n, k), generator=g, dtype=torch.int8).cuda()
    sx = (torch.rand(m, generator=g) * 0.02 + 1e-3).cuda()
    swo = (torch.rand(n, generator=g) * 1e-3 + 1e-4).cuda()
    swn = (torch.rand(n, generator=g) * 1e-3 + 1e-4).cuda()
    b = (torch.rand(n, generator=g) - 0.5).cuda()
    ws = torch.zeros(int(qb._lib.load().qarvd_dual_gemm_quant_workspace_size(m)), dtype=torch.uint8, device="cuda")
    ref, outs = _qz_pair(ws, m, n, k, ko, True, xq, wq, sx, swo, swn, b, reps=3)
    for q, s, d, e in outs:
        assert torch.equal(q, ref[0])
        assert torch.equal(s.view(torch.int32), ref[1].view(torch.int32))
        assert torch.equal(d.view(torch.int64), ref[2].view(torch.int64))


def test_k2_fused_quant_rejects_bad_arguments(cuda):
    """The fused entry validates like the reference: n not a multiple of 256 is outside this
    build's envelope, a missing workspace and a bad static scale are invalid arguments."""
    lib = qb._lib
    m, n, k = 64, 384, 64
    xq = torch.zeros((m, k), dtype=torch.int8, device="cuda")
    wq = torch.zeros((n, k), dtype=torch.int8, device="cuda")
    sx = torch.ones(m, device="cuda")
    sw = torch.ones(n, device="cuda")
    q = torch.empty((m, 512), dtype=torch.int8, device="cuda")
    s = torch.empty(m, device="cuda")
    ws = torch.zeros(int(lib.load().qarvd_dual_gemm_quant_workspace_size(m)), dtype=torch.uint8, device="cuda")
    args = lambda nn, gran, sst, w: (xq.data_ptr(), k, wq.data_ptr(), k, m, nn, k, 0, sx.data_ptr(), sw.data_ptr(),
                                      sw.data_ptr(), None, qb.EPI_NONE, gran, sst, 8, q.data_ptr(), 512, s.data_ptr(),
                                      None, None, w, ws.numel(), None)
    with pytest.raises(qb._lib.Unsupported):
        lib.call("qarvd_dual_gemm_quant", *args(n, qb.ACT_PER_TOKEN, 0.0, ws.data_ptr()))
    with pytest.raises(qb._lib.InvalidArgument):
        lib.call("qarvd_dual_gemm_quant", *args(256, qb.ACT_PER_TOKEN, 0.0, None))
    with pytest.raises(qb._lib.InvalidArgument):
        lib.call("qarvd_dual_gemm_quant", *args(256, qb.ACT_PER_TENSOR, -1.0, ws.data_ptr()))
