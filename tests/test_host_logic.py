"""CPU tests of the host-side logic above the C-ABI: plan layout, synthetic-data recipe,
weighting, LPT layer sharding and the packed all-gather records."""
import numpy as np
import pytest

import paper_2605_21072_b200 as qb
from paper_2605_21072_b200 import calibrate, engine, synth


def test_build_plan_layout_aligned():
    outl = np.arange(0, 1536, 48)[:32]
    p = engine.build_plan("l", 1536, outl)
    assert p.enabled and p.k_outlier == 32 and p.k_pad == 1536
    assert p.permutation[:32].tolist() == sorted(outl.tolist())
    assert sorted(p.permutation.tolist()) == list(range(1536))
    np.testing.assert_array_equal(p.gather[:32], p.permutation[:32])
    np.testing.assert_array_equal(p.gather[32:], p.permutation[32:])
    np.testing.assert_array_equal(p.inverse_permutation()[p.permutation], np.arange(1536))


def test_build_plan_unaligned_pads_both_slabs():
    p = engine.build_plan("l", 100, [3, 50, 99])
    assert p.k_outlier == 32 and p.k_pad == 32 + 128
    assert p.gather[:3].tolist() == [3, 50, 99] and (p.gather[3:32] == -1).all()
    normals = [c for c in range(100) if c not in (3, 50, 99)]
    assert p.gather[32:32 + 97].tolist() == normals and (p.gather[32 + 97:] == -1).all()


def test_build_plan_disabled_and_errors():
    p = engine.build_plan("l", 64, [])
    assert not p.enabled and p.k_outlier == 0 and p.gather.tolist() == list(range(64))
    with pytest.raises(qb.OutOfRange):
        engine.build_plan("l", 64, [64])
    with pytest.raises(qb.InvalidArgument):
        engine.build_plan("l", 4, [0, 1, 2, 3])


def test_wan_registry_shapes():
    specs = synth.wan_registry()
    assert len(specs) == 300
    by = {}
    for s in specs:
        by.setdefault(s.name.split(".", 1)[1], []).append(s)
    assert all(s.out_dim == 8960 and s.in_dim == 1536 for s in by["ffn.0"])
    assert all(s.out_dim == 1536 and s.in_dim == 8960 for s in by["ffn.2"])
    assert all(s.tokens == 512 for s in by["cross_attn.k"] + by["cross_attn.v"])
    assert all(s.outlier_fraction == 0 for s in by["cross_attn.v"])  # smooth
    total = sum(2.0 * s.tokens * s.in_dim * s.out_dim for s in specs)
    assert abs(total / 11.85e12 - 1) < 0.01  # 11.85 T int-ops per chunk


def test_outlier_columns_counts():
    assert len(synth.pick_outlier_columns(1, 9, 1536, 0.021)) == 32
    assert len(synth.pick_outlier_columns(1, 9, 8960, 0.021)) == 188
    c = synth.pick_outlier_columns(5, 3, 64, 0.001)
    assert len(c) == 1 and 0 <= c[0] < 64
    assert len(set(synth.pick_outlier_columns(2, 7, 256, 0.5).tolist())) == 128


def test_mix_seed_reference_constants():
    # splitmix64 from state 0: first output of the reference stream (rng.hpp:11-16)
    st, out = synth.splitmix64(0)
    assert out == 0xE220A8397B1DCDAF
    assert synth.mix_seed(1, 2) != synth.mix_seed(2, 1)


def test_weighting_strategy_contract():
    w = calibrate.weighting_strategy("heuristic_exp", 21)
    assert w[0] > w[1] > w[-1] and abs(w.sum() - 1) < 1e-15
    u = calibrate.weighting_strategy("uniform", 7)
    assert (u == 1 / 7).all()
    a = [0.0] * 5
    np.testing.assert_array_equal(calibrate.weighting_strategy("final_quality", 5, a), np.full(5, 0.2))
    with pytest.raises(qb.InvalidArgument):
        calibrate.weighting_strategy("reverse", 5)


def test_lpt_assignment_deterministic_and_balanced():
    specs = synth.wan_registry()
    costs = [s.weight_bytes() + 21 * 1560 * s.in_dim * 2 for s in specs]
    for world in (1, 2, 4, 8):
        a = calibrate.lpt_assign(costs, world)
        assert sorted(i for r in a for i in r) == list(range(300))
        loads = [sum(costs[i] for i in r) for r in a]
        assert max(loads) / (sum(costs) / world) < 1.02
        assert a == calibrate.lpt_assign(costs, world)


def _fake_record(i, rng):
    n = int(rng.integers(4, 40))
    no = int(rng.integers(0, 5))
    return calibrate.LayerRecord(i, no, np.sort(rng.choice(100, no, replace=False)), rng.random(),
                                 int(rng.integers(0, 3)), rng.random(3), rng.random(n), rng.random(n))


def test_record_pack_roundtrip():
    rng = np.random.default_rng(0)
    recs = [_fake_record(i, rng) for i in range(7)]
    back = calibrate.unpack_records(calibrate.pack_records(recs))
    assert len(back) == 7
    for a, b in zip(recs, back):
        assert a.index == b.index and a.act_scale == b.act_scale and a.best_index == b.best_index
        np.testing.assert_array_equal(a.outliers, b.outliers)
        np.testing.assert_array_equal(a.scale_normal, b.scale_normal)
        np.testing.assert_array_equal(a.scale_outlier, b.scale_outlier)
        np.testing.assert_array_equal(a.losses, b.losses)


def _fake_calib_record(i, rng):
    n, k, nt = int(rng.integers(1, 9)), int(rng.integers(1, 13)), int(rng.integers(0, 6))
    res = calibrate.LayerCalibResult(f"blocks.{i}.attn.q" + "x" * (i % 4), rng.random(n), rng.random(n),
                                     rng.integers(-128, 128, (n, k)).astype(np.int8), rng.random(),
                                     rng.random(), rng.random(), rng.random(nt))
    return calibrate.CalibRecord(i, res)


def test_calib_record_pack_roundtrip():
    rng = np.random.default_rng(1)
    recs = [_fake_calib_record(i, rng) for i in range(9)]
    packed = np.concatenate([r.pack() for r in recs])
    assert packed.dtype == np.uint8 and all(len(r.pack()) % 8 == 0 for r in recs)
    back = calibrate.unpack_calib_records(packed)
    assert len(back) == 9
    for a, b in zip(recs, back):
        ra, rb = a.result, b.result
        assert a.index == b.index and ra.layer == rb.layer
        assert (ra.act_scale, ra.initial_loss, ra.final_loss) == (rb.act_scale, rb.initial_loss, rb.final_loss)
        np.testing.assert_array_equal(ra.codes, rb.codes)
        np.testing.assert_array_equal(ra.scale_normal, rb.scale_normal)
        np.testing.assert_array_equal(ra.scale_outlier, rb.scale_outlier)
        np.testing.assert_array_equal(ra.trace, rb.trace)


def test_adaround_cost_orders_lpt():
    costs = [calibrate.adaround_cost(n, k, r, 100) for n, k, r in ((1536, 8960, 10), (1536, 1536, 10),
                                                                  (8960, 1536, 10), (1536, 1536, 40))]
    assert costs[0] == costs[2] and costs[3] == 4 * costs[1]
    assert calibrate.lpt_assign(costs, 2) == [[0, 3], [1, 2]]


@pytest.fixture(scope="module")
def toy_qarq(tmp_path_factory):
    import oracle
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    path = str(tmp_path_factory.mktemp("qarq") / "toy.qarq")
    n = oracle.ref_toy_qarq(path, iterations=4)
    return path, n


def test_qarq_parser_matches_reference_loader(toy_qarq):
    """qarq.load_qarq reads the reference's own saved model exactly as load_quantized_model
    (engine.cpp:315-333): codes, f32 scales, permutation, act scale, preserved layers."""
    import oracle
    from paper_2605_21072_b200 import qarq
    path, n = toy_qarq
    header, layers = qarq.load_qarq(path)
    assert len(layers) == n == len(header["layers"])
    n_quant = 0
    for i, L in enumerate(layers):
        ref = oracle.ref_qarq_layer(path, i)
        assert L.preserved == ref["preserved"] and (L.out_dim, L.in_dim) == (ref["out_dim"], ref["in_dim"])
        if L.preserved:
            assert L.fp_weight_bf16.shape == (L.out_dim, L.in_dim)
            continue
        n_quant += 1
        np.testing.assert_array_equal(L.codes.astype(np.int32), ref["wq"])
        np.testing.assert_array_equal(L.scale_normal.astype(np.float64), ref["scale_normal"])
        if ref["enabled"]:
            np.testing.assert_array_equal(L.scale_outlier.astype(np.float64), ref["scale_outlier"])
            np.testing.assert_array_equal(L.permutation, ref["permutation"])
            assert L.outlier_count == ref["outlier_count"]
        assert np.float64(np.float32(L.act_scale)) == ref["act_scale"] and L.act_zero == ref["act_zero"]
    assert n_quant > 0


def test_qarq_bad_magic(tmp_path):
    from paper_2605_21072_b200 import qarq, _lib
    p = tmp_path / "bad.qarq"
    p.write_bytes(b"NOPE" + b"\0" * 32)
    with pytest.raises(_lib.QarvdError, match="bad magic"):
        qarq.load_qarq(str(p))
