"""CPU tests: the oracle restatement pinned against the reference's known-answer examples
(SPEC.md), the committed golden fixtures, and the compiled reference itself (oracle/_ref)."""
import os

import numpy as np
import pytest

import oracle
from qarvd_testutil import bf16_values

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- SPEC.md known answers
def test_kat_quantize_b4():
    # x=[-1, 0.5, 2], symmetric b=4 -> s=2/7, codes [-4, 2, 7]
    x = np.array([[-1.0, 0.5, 2.0]])
    q, s, bad = oracle.quantize_act(x, None, per_token=True, bits=4)
    assert bad < 0 and s[0] == 2.0 / 7.0
    assert q.tolist() == [[-4, 2, 7]]


def test_kat_zero_and_grid_roundtrip():
    s = 0.25
    x = np.array([[0.0, 0.25, -0.5, 31.75, -31.75]])
    q, _, _ = oracle.quantize_act(x, None, per_token=False, static_scale=s)
    np.testing.assert_array_equal(q[0] * s, x[0])


def test_kat_round_half_even():
    for v, e in [(0.5, 0.0), (1.5, 2.0), (2.5, 2.0), (-0.5, -0.0), (-1.5, -2.0), (2.4999, 2.0), (126.5, 126.0)]:
        assert oracle.lib().oracle_round_half_even(v) == e


def test_kat_mad():
    # SPEC.md:176-177
    assert oracle.mad([1, 1, 1, 1, 10]) == (1.0, 0.0)
    assert oracle.mad([1, 2, 3, 4, 5]) == (3.0, 1.0)
    assert oracle.mad([4.0] * 6) == (4.0, 0.0)


def test_kat_detect():
    # SPEC.md:185-187, criterion 3
    d = oracle.analyze_norms([1, 1, 1, 1, 10])
    assert d["raw"].tolist() == [4] and d["threshold"] == 1.2
    assert oracle.analyze_norms([3.0] * 40)["raw"].size == 0


def test_kat_align():
    # |raw|=4, align 32, d_in 256 -> the 32 largest, superset of raw
    r = np.random.default_rng(0)
    v = 1.0 + 0.01 * r.random(256)
    spikes = [7, 50, 100, 200]
    v[spikes] = 10.0
    d = oracle.analyze_norms(v)
    assert d["raw"].tolist() == spikes and len(d["aligned"]) == 32
    assert set(spikes) <= set(d["aligned"].tolist())
    top = np.argsort(-v, kind="stable")[:32]
    assert sorted(top.tolist()) == d["aligned"].tolist()
    # align = 1 -> raw unchanged
    assert oracle.analyze_norms(v, align=1)["aligned"].tolist() == spikes


def test_injection_completeness_and_scale_invariance():
    # SPEC.md:209 / criterion 2: exact recovery for tau in [2.5, 4.5], and scale invariance
    r = np.random.default_rng(1)
    for trial in range(60):
        d_in = [128, 256, 1024][trial % 3]
        gamma = [3.0, 8.0, 10.0][trial % 3]
        v = 1.0 + 0.05 * (r.random(d_in) - 0.5)
        inj = np.sort(r.choice(d_in, size=max(1, int(0.03 * d_in)), replace=False))
        v[inj] *= gamma
        for tau in (2.5, 3.0, 3.5, 4.0, 4.5):
            assert oracle.analyze_norms(v, tau=tau)["raw"].tolist() == inj.tolist()
        assert oracle.analyze_norms(v * 7.25)["raw"].tolist() == inj.tolist()
        smooth = 1.0 + 0.1 * (r.random(d_in) - 0.5)
        assert oracle.analyze_norms(smooth)["raw"].size == 0


def test_weighting_heuristic_exp_sums_to_one():
    w = oracle.weighting(1, None, 21)
    assert abs(w.sum() - 1.0) < 1e-15 and np.all(np.diff(w) < 0)


# ---------------------------------------------------------------- golden fixtures (from oracle/_ref)
def _golden(name):
    p = os.path.join(GOLDEN, name)
    if not os.path.exists(p):
        pytest.skip(f"{name} missing (run oracle/make_golden.py)")
    return np.load(p)


def test_golden_quantize():
    g = _golden("quantize.npz")
    q, s, _ = oracle.quantize_act(g["x"], None, per_token=True)
    np.testing.assert_array_equal(q, g["codes"])
    np.testing.assert_array_equal(s, g["scales"])
    qs, _, _ = oracle.quantize_act(g["x"], None, per_token=False, static_scale=float(g["static_scale"]))
    np.testing.assert_array_equal(qs, g["codes_static"])


def test_golden_kernel_b():
    g = _golden("kernel_b.npz")
    out = oracle.kernel_b(g["xq"], g["wq"], int(g["n_outlier"]), g["s_x"], g["s_o"], g["s_n"])
    np.testing.assert_array_equal(out, g["y"])


def test_golden_analyze_and_plan():
    g = _golden("analyze.npz")
    d = oracle.analyze_layer(g["w"])
    np.testing.assert_array_equal(d["norms"], g["norms"])
    np.testing.assert_array_equal(d["aligned"], g["aligned"])
    np.testing.assert_array_equal(d["raw"], g["raw"])
    assert d["threshold"] == float(g["threshold"])
    wq, so, sn, _ = oracle.prepare_weights(g["w"], g["gather"], int(g["k_outlier"]))
    np.testing.assert_array_equal(wq.astype(np.int32), g["wq"])
    np.testing.assert_array_equal(so, g["s_o"])
    np.testing.assert_array_equal(sn, g["s_n"])


def test_golden_percentile_search():
    g = _golden("search.npz")
    res = oracle.scale_search_hist(g["x_bits"], int(g["frames"]), int(g["rows"]), int(g["k"]))
    assert (0.999, 0.9999, 0.99999)[int(res[9])] == float(g["best_pct"])
    assert res[10] == float(g["scale"])
    np.testing.assert_allclose(res[6:9], g["mse"], rtol=1e-12)


# ---------------------------------------------------------------- oracle vs compiled reference
def test_ref_quantize_random(ref_lib):
    for seed in range(5):
        bits, x64 = bf16_values((64, 200), seed=seed, heavy_cols=[3, 77])
        codes, scales = oracle.ref_quantize(x64, per_token=True)
        q, s, _ = oracle.quantize_act(x64, None, per_token=True)
        np.testing.assert_array_equal(q.astype(np.int32), codes)
        np.testing.assert_array_equal(s, scales)
        r = np.random.default_rng(seed)
        x = r.standard_normal((32, 50)) * 5  # non-bf16 f64 values
        codes, _ = oracle.ref_quantize(x, per_token=False, s=0.03)
        q, _, _ = oracle.quantize_act(x, None, per_token=False, static_scale=0.03)
        np.testing.assert_array_equal(q.astype(np.int32), codes)


def test_ref_kernel_b_random(ref_lib):
    r = np.random.default_rng(3)
    for n_out, enabled in [(32, True), (0, False), (64, True)]:
        m, n, k = 24, 40, 256
        xq = r.integers(-127, 128, (m, k))
        wq = r.integers(-127, 128, (n, k))
        perm = np.arange(k, dtype=np.uint32)
        so, sn = r.random(n) * 0.01, r.random(n) * 0.01
        for sx in (np.array([0.02]), r.random(m) * 0.05):
            y_ref = oracle.ref_kernel_b(xq, wq, perm, n_out, enabled, sx, so, sn)
            y = oracle.kernel_b(xq, wq, n_out if enabled else 0, np.broadcast_to(sx, (m,)), so, sn)
            np.testing.assert_array_equal(y, y_ref)


def test_ref_analyze_random(ref_lib):
    for seed, (n, k, frac) in enumerate([(64, 256, 0.03), (128, 1536, 0.021), (40, 50, 0.1),
                                         (96, 640, 0.0), (32, 96, 0.5)]):
        r = np.random.default_rng(seed)
        heavy = r.choice(k, size=max(1, int(frac * k)), replace=False) if frac else None
        _, w64 = bf16_values((n, k), seed=seed, heavy_cols=heavy, gamma=6.0)
        a = oracle.analyze_layer(w64)
        b = oracle.ref_analyze_layer(w64)
        np.testing.assert_array_equal(a["norms"], b["norms"])
        for key in ("median", "mad", "threshold"):
            assert a[key] == b[key]
        np.testing.assert_array_equal(a["raw"], b["raw"])
        np.testing.assert_array_equal(a["aligned"], b["aligned"])
        # f64 (non-bf16) weights too: separate mul + add, sequential rows
        w = r.standard_normal((n, k))
        np.testing.assert_array_equal(oracle.channel_norms(w), oracle.ref_analyze_layer(w)["norms"])


def test_ref_analyze_norms_ties_and_cap(ref_lib):
    r = np.random.default_rng(9)
    cases = [np.repeat([1.0, 2.0, 5.0], [50, 40, 10]),          # heavy ties at the pivot
             np.concatenate([np.ones(60), np.full(40, 9.0)]),   # cap blocks alignment -> raw
             np.concatenate([np.ones(33), [4.0, 4.0]]),           # d_in < 2*align
             1.0 + r.random(100) * 0.001]
    for v in cases:
        v = r.permutation(v)
        a, b = oracle.analyze_norms(v), oracle.ref_analyze_norms(v)
        for key in ("median", "mad", "threshold"):
            assert a[key] == b[key]
        np.testing.assert_array_equal(a["raw"], b["raw"])
        np.testing.assert_array_equal(a["aligned"], b["aligned"])


def test_ref_build_plan_codes(ref_lib):
    from paper_2605_21072_b200.engine import build_plan

    r = np.random.default_rng(4)
    n, k = 48, 200
    outl = np.sort(r.choice(k, 7, replace=False))  # unaligned: padded to 32 in our layout
    _, w64 = bf16_values((n, k), seed=4, heavy_cols=outl)
    ref = oracle.ref_build_plan_codes(w64, outl)
    plan = build_plan("t", k, outl)
    np.testing.assert_array_equal(plan.permutation, ref["permutation"])
    wq, so, sn, _ = oracle.prepare_weights(w64, plan.gather, plan.k_outlier)
    keep = plan.gather >= 0
    np.testing.assert_array_equal(wq[:, keep].astype(np.int32), ref["wq"])
    np.testing.assert_array_equal(so, ref["scale_outlier"])
    np.testing.assert_array_equal(sn, ref["scale_normal"])
    assert np.all(wq[:, ~keep] == 0)


def test_ref_percentile_search_equals_histogram_form(ref_lib):
    for seed, (frames, rows, k) in enumerate([(21, 20, 256), (7, 16, 64), (3, 9, 40)]):
        bits, x64 = bf16_values((frames * rows, k), seed=seed, heavy_cols=np.arange(0, k, 17))
        best, scale, mse = oracle.ref_percentile_search(x64, frames, rows, k)
        res = oracle.scale_search_hist(bits, frames, rows, k)
        assert (0.999, 0.9999, 0.99999)[int(res[9])] == best
        assert res[10] == scale
        np.testing.assert_array_equal(res[3:6], [s for s in res[3:6]])
        np.testing.assert_allclose(res[6:9], mse, rtol=1e-12)


def test_ref_weighting(ref_lib):
    from paper_2605_21072_b200.calibrate import weighting_strategy

    alpha = np.array([0.7, 0.2, 0.05, 0.03, 0.01, 0.005, 0.005])
    for kind, name in enumerate(["uniform", "heuristic_exp", "reverse", "final_quality"]):
        np.testing.assert_array_equal(weighting_strategy(name, 7, alpha), oracle.ref_weighting(kind, alpha, 7))
        np.testing.assert_array_equal(oracle.weighting(kind, oracle.ref_weighting(3, alpha, 7), 7),
                                      oracle.ref_weighting(kind, alpha, 7))
    np.testing.assert_array_equal(weighting_strategy("heuristic_exp", 21), oracle.ref_weighting(1, None, 21))


def test_ref_toy_injection_columns_match_synth(ref_lib):
    """pick_outlier_columns reproduces the reference's seeded Fisher-Yates (toy_model.cpp:152-166)."""
    from paper_2605_21072_b200.synth import pick_outlier_columns

    # registry index of block0.ffn.2 in the toy model: time_embed=0, block0 types 1..10 -> ffn.2 = 10
    w_inj = oracle.ref_toy_weight("block0.ffn.2", pattern="ffn.2", fraction=0.05, gamma=8.0)
    w_base = oracle.ref_toy_weight("block0.ffn.2")
    ratio = np.abs(w_inj / w_base)
    cols = np.nonzero(np.isclose(ratio, 8.0).all(axis=0))[0]
    mine = np.sort(pick_outlier_columns(1, 10, w_base.shape[1], 0.05))
    np.testing.assert_array_equal(cols, mine)


def test_device_row_scale_formula_is_correctly_rounded():
    """K1 computes s = fl(amax/qmax) as amax*fl(1/qmax) + one fma correction (quantize.cu
    row_s64); exhaustively equal to the division for every bf16 amax and bit width."""
    assert oracle.row_scale_formula_mismatches() == 0


def _loss_case(n, k, n_out, seed, samples=3, rows=5):
    r = np.random.default_rng(seed)
    outl = np.sort(r.choice(k, n_out, replace=False)) if n_out else np.zeros(0, np.int64)
    wb, w = bf16_values((n, k), seed=seed, scale=1.0 / np.sqrt(k), heavy_cols=outl if n_out else None)
    xb, x = bf16_values((samples * rows, k), seed=seed + 1, heavy_cols=outl if n_out else None, gamma=3.0)
    row_off = np.arange(samples + 1) * rows
    chunks = np.array([1, 3, 2][:samples])
    cw = oracle.weighting(1, None, 3)  # heuristic_exp over 3 chunks
    return w, x, outl, row_off, chunks, cw


@pytest.mark.parametrize("n,k,n_out", [(24, 96, 32), (16, 64, 0), (8, 160, 33)])
def test_ref_weighted_loss_equals_restatement(ref_lib, n, k, n_out):
    """Eq. 5 (calibrate.cpp:201-224) on a reference-initialised LearnableQuantState: the plain-C
    restatement reproduces the reference's weighted_loss bit-for-bit."""
    w, x, outl, row_off, chunks, cw = _loss_case(n, k, n_out, seed=n + k)
    act = np.abs(x).max() / 127.0
    ref = oracle.ref_weighted_loss(w, outl, act, x, row_off, chunks, cw)
    xq, _, _ = oracle.quantize_act(x, None, per_token=False, static_scale=ref["act_scale"])
    loss, err = oracle.weighted_loss(x, xq, ref["act_scale"], w, ref["codes"], ref["s_wo"], ref["s_wn"],
                                     ref["mask"], row_off, chunks, cw)
    assert loss == ref["loss"]
    assert loss > 0 and np.all(err > 0)
    assert np.isclose(loss, sum(cw[c - 1] * e for c, e in zip(chunks, err)) / len(chunks), rtol=1e-15)


def test_weighted_loss_errors(ref_lib):
    w, x, outl, row_off, chunks, cw = _loss_case(8, 64, 0, seed=3)
    with pytest.raises(oracle.RefError, match="outside the weight vector"):
        oracle.ref_weighted_loss(w, outl, 0.01, x, row_off, np.array([1, 4, 2]), cw)
    with pytest.raises(IndexError):
        oracle.weighted_loss(x, np.zeros(x.shape, np.int32), 0.01, w, np.zeros(w.shape, np.int32),
                             np.ones(8), np.ones(8), np.zeros(64, np.uint8), row_off, np.array([0, 1, 2]), cw)
    with pytest.raises(oracle.RefError, match="empty batch"):
        oracle.ref_weighted_loss(w, outl, 0.01, x, np.array([0]), np.zeros(0, np.int64), cw)
