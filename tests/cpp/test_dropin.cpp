// Drop-in test: the reference's own pipeline (toy model -> calibrate_model -> QuantizedModel)
// and its operators served through qarvd::cuda (libqarvd_b200.so) instead of the reference's CPU
// code, compared with the reference on identical inputs.  Every comparison is exact (bit-identical
// doubles, identical integer codes and index sets) unless a tolerance is stated with its reason.
// Built against the reference headers and oracle/_ref/libqarvd_ref.a (the unmodified reference
// sources); run on a GPU box by tests/test_gpu_dropin.py.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

#include "../../paper_2605_21072_b200/adapter/qarvd_cuda.hpp"
#include "qarvd/calibrate.hpp"
#include "qarvd/dual_scale.hpp"
#include "qarvd/engine.hpp"
#include "qarvd/outlier.hpp"
#include "qarvd/rng.hpp"
#include "qarvd/sensitivity.hpp"
#include "qarvd/threading.hpp"
#include "qarvd/toy_model.hpp"

using namespace qarvd;

static int failures = 0;
#define EXPECT(cond, what)                                        \
  do {                                                            \
    if (!(cond)) {                                                \
      std::printf("FAIL %s (%s:%d)\n", what, __FILE__, __LINE__); \
      ++failures;                                                 \
    }                                                             \
  } while (0)

static Tensor random_tensor(size_t r, size_t c, uint64_t seed, double scale) {
  Prng rng(seed);
  Tensor t({r, c});
  for (size_t i = 0; i < t.size(); ++i) t[i] = rng.gaussian() * scale;
  return t;
}

static bool same_bits(const std::vector<double>& a, const std::vector<double>& b) {
  return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), a.size() * 8) == 0);
}
static bool same_params(const QuantParams& a, const QuantParams& b) {
  return a.bits == b.bits && a.symmetric == b.symmetric && a.granularity == b.granularity &&
         a.channel_axis == b.channel_axis && same_bits(a.scale, b.scale) && a.zero_point == b.zero_point &&
         a.q_min == b.q_min && a.q_max == b.q_max;
}
static bool same_plan(const DualScalePlan& a, const DualScalePlan& b) {
  return a.layer_name == b.layer_name && a.enabled == b.enabled && a.d_in == b.d_in &&
         a.outlier_indices == b.outlier_indices && a.normal_indices == b.normal_indices &&
         a.permutation == b.permutation && same_params(a.params_outlier, b.params_outlier) &&
         same_params(a.params_normal, b.params_normal);
}

template <typename F>
static std::string what_of(F&& f) {
  try {
    f();
  } catch (const std::invalid_argument& e) {
    return std::string("invalid_argument: ") + e.what();
  } catch (const std::out_of_range& e) {
    return std::string("out_of_range: ") + e.what();
  } catch (const std::logic_error& e) {
    return std::string("logic_error: ") + e.what();
  } catch (const std::runtime_error& e) {
    return std::string("runtime_error: ") + e.what();
  }
  return "no exception";
}

int main() {
  ToyModelConfig cfg;  // toy defaults (toy_model.hpp:24-38) + outlier injections
  cfg.injections = {{"ffn.2", 0.05, 8.0}, {"self_attn.q", 0.03, 6.0}};
  const ToyModel model = ToyModel::build(cfg);
  SensitivityProfile prof;
  prof.alpha_raw.assign(cfg.chunks, 1.0);
  prof.alpha_normalized = normalize_alpha(prof.alpha_raw);
  const std::vector<double> w = weighting_strategy(prof, WeightingKind::heuristic_exp);
  ModelCalibOptions opts;
  opts.base.iterations = 8;
  opts.base.batch_size = 2;
  const ModelCalibResult calib = calibrate_model(model, w, opts);
  const QuantizedModel& qm = calib.qmodel;
  std::printf("calibrated %zu layers\n", qm.layers.size());

  // ---- quant.hpp: quantize (every granularity), fake_quant, init_scale_minmax
  {
    const Tensor x = random_tensor(37, 70, 11, 1.7);
    const std::vector<QuantParams> ps = {
        init_scale_minmax(x, 8, Granularity::per_tensor),
        init_scale_minmax(x, 8, Granularity::per_channel, 0),
        init_scale_minmax(x, 6, Granularity::per_channel, 1),
        init_scale_minmax(x, 4, Granularity::per_tensor),
        QuantParams::per_tensor_symmetric(8, 1e-300),  // |v/s| beyond int64: the x86 conversion quirk
    };
    for (size_t i = 0; i < ps.size(); ++i) {
      EXPECT(qarvd::quantize(x, ps[i]).data == qarvd::cuda::quantize(x, ps[i]).data, "quantize codes");
      EXPECT(same_bits(qarvd::fake_quant(x, ps[i]).vec(), qarvd::cuda::fake_quant(x, ps[i]).vec()), "fake_quant");
    }
    QuantParams asym = QuantParams::per_tensor_symmetric(8, 0.013);
    asym.symmetric = false;
    asym.zero_point = {-17};
    asym.q_min = -128;
    asym.q_max = 127;
    EXPECT(qarvd::quantize(x, asym).data == qarvd::cuda::quantize(x, asym).data, "quantize asymmetric");
    for (int bits : {2, 4, 8, 12})
      for (auto [g, ax] : {std::pair{Granularity::per_tensor, 0}, {Granularity::per_channel, 0},
                           {Granularity::per_channel, 1}}) {
        EXPECT(same_params(qarvd::init_scale_minmax(x, bits, g, ax), qarvd::cuda::init_scale_minmax(x, bits, g, ax)),
               "init_scale_minmax");
      }
    Tensor z({3, 5});  // all-zero slices -> DBL_MIN
    EXPECT(same_params(qarvd::init_scale_minmax(z, 8, Granularity::per_channel, 0),
                       qarvd::cuda::init_scale_minmax(z, 8, Granularity::per_channel, 0)),
           "init_scale_minmax zeros");
    Tensor bad = x;
    bad[123] = std::nan("");
    bad[200] = INFINITY;
    EXPECT(what_of([&] { qarvd::quantize(bad, ps[0]); }) == what_of([&] { qarvd::cuda::quantize(bad, ps[0]); }),
           "quantize non-finite message");
    const Tensor xt = random_tensor(70, 37, 12, 1.0);
    EXPECT(what_of([&] { qarvd::quantize(xt, ps[1]); }) == what_of([&] { qarvd::cuda::quantize(xt, ps[1]); }) &&
               what_of([&] { qarvd::cuda::quantize(xt, ps[1]); }).rfind("invalid_argument", 0) == 0,
           "quantize per-channel length mismatch");
    EXPECT(same_params(qarvd::init_scale_minmax(bad, 8, Granularity::per_tensor),
                       qarvd::cuda::init_scale_minmax(bad, 8, Granularity::per_tensor)),
           "init_scale_minmax NaN ignored / inf kept");
  }

  // ---- init_scale_percentile_search on the model's own captures, plus synthetic sample sets
  {
    const std::vector<std::string> names = {"block0.ffn.2", "block1.self_attn.q", "block0.cross_attn.k"};
    const std::vector<CalibSample> cap_ref = collect_calibration(model, {101, 102}, names);
    const std::vector<CalibSample> cap_gpu = qarvd::cuda::collect_calibration(model, {101, 102}, names);
    bool same_cap = cap_ref.size() == cap_gpu.size();
    for (size_t i = 0; same_cap && i < cap_ref.size(); ++i)
      same_cap = cap_ref[i].layer == cap_gpu[i].layer && cap_ref[i].chunk == cap_gpu[i].chunk &&
                 cap_ref[i].x.shape() == cap_gpu[i].x.shape() && same_bits(cap_ref[i].x.vec(), cap_gpu[i].x.vec());
    EXPECT(same_cap, "collect_calibration captures bit-identical");
    size_t n_sets = 0;
    for (const std::string& name : names) {
      std::vector<Tensor> acts;
      for (const CalibSample& c : cap_ref)
        if (c.layer == name) acts.push_back(c.x);
      for (int bits : {8, 6, 4}) {
        const PercentileSearchResult a = qarvd::init_scale_percentile_search(acts, bits);
        const PercentileSearchResult b = qarvd::cuda::init_scale_percentile_search(acts, bits);
        EXPECT(a.best_percentile == b.best_percentile && same_params(a.params, b.params),
               ("percentile search selection " + name).c_str());
        double worst = 0.0;
        for (size_t i = 0; i < a.candidate_mse.size(); ++i)
          worst = std::max(worst, std::fabs(a.candidate_mse[i] - b.candidate_mse[i]) / a.candidate_mse[i]);
        // candidate MSEs: the reference sums sequentially, the device in double-double
        EXPECT(worst <= 1e-12, ("percentile search MSEs within 1e-12 " + name).c_str());
        ++n_sets;
      }
    }
    std::vector<Tensor> syn;
    for (int s = 0; s < 9; ++s) syn.push_back(random_tensor(30 + 7 * s, 96, 500 + s, 0.5 + 0.2 * s));
    const PercentileSearchResult a = qarvd::init_scale_percentile_search(syn, 8);
    const PercentileSearchResult b = qarvd::cuda::init_scale_percentile_search(syn, 8);
    EXPECT(a.best_percentile == b.best_percentile && same_params(a.params, b.params), "percentile search synthetic");
    std::vector<Tensor> one = {Tensor({1, 1}, {-2.5})};
    EXPECT(same_params(qarvd::init_scale_percentile_search(one, 8).params,
                       qarvd::cuda::init_scale_percentile_search(one, 8).params),
           "percentile search single element");
    syn[4][17] = std::nan("");
    EXPECT(what_of([&] { qarvd::init_scale_percentile_search(syn, 8); }) ==
               what_of([&] { qarvd::cuda::init_scale_percentile_search(syn, 8); }),
           "percentile search non-finite message");
    EXPECT(what_of([&] { qarvd::init_scale_percentile_search({}, 8); }) ==
               what_of([&] { qarvd::cuda::init_scale_percentile_search({}, 8); }),
           "percentile search empty");
    std::printf("percentile search: %zu capture sets x bit widths identical\n", n_sets);
  }

  // ---- per-operator parity on every quantized layer (+ plans, products, permutes)
  size_t n_layers = 0;
  for (const auto& l : qm.layers) {
    if (l.preserved) {
      const Tensor x = random_tensor(9, l.in_dim, 5, 1.0);
      EXPECT(same_bits(qarvd::quantized_layer_forward(l, x, Engine::int_kernels).vec(),
                       qarvd::cuda::quantized_layer_forward(l, x, Engine::int_kernels).vec()),
             ("preserved forward " + l.name).c_str());
      continue;
    }
    ++n_layers;
    const Tensor x = random_tensor(24, l.in_dim, 77 + n_layers, 1.5);
    const Tensor xp = qarvd::permute_activations(x, l.plan);
    EXPECT(same_bits(xp.vec(), qarvd::cuda::permute_activations(x, l.plan).vec()), ("permute " + l.name).c_str());
    const IntTensor a_ref = qarvd::kernel_a_quantize_activation(xp, l.act);
    EXPECT(a_ref.data == qarvd::cuda::kernel_a_quantize_activation(xp, l.act).data, ("kernel_a " + l.name).c_str());
    const Tensor b_ref = qarvd::kernel_b_gemm_dequant(a_ref, l);
    EXPECT(same_bits(b_ref.vec(), qarvd::cuda::kernel_b_gemm_dequant(a_ref, l).vec()), ("kernel_b " + l.name).c_str());
    for (Engine e : {Engine::int_kernels, Engine::fakequant_sim})
      EXPECT(same_bits(qarvd::quantized_layer_forward(l, x, e).vec(), qarvd::cuda::quantized_layer_forward(l, x, e).vec()),
             ("layer forward " + l.name).c_str());
    // asymmetric activations: zero-point column-sum correction (engine.cpp:74-100)
    QuantizedLayer la = l;
    la.act.symmetric = false;
    la.act.zero_point = {static_cast<int32_t>(n_layers % 2 ? -9 : 13)};
    la.act.q_min = -128;
    la.act.q_max = 127;
    EXPECT(same_bits(qarvd::quantized_layer_forward(la, x, Engine::int_kernels).vec(),
                     qarvd::cuda::quantized_layer_forward(la, x, Engine::int_kernels).vec()),
           ("layer forward asymmetric " + l.name).c_str());
    const Tensor& W = model.weight(l.name);
    const OutlierReport r_ref = qarvd::analyze_layer(l.name, W);
    const OutlierReport r_gpu = qarvd::cuda::analyze_layer(l.name, W);
    EXPECT(same_bits(r_ref.norms, r_gpu.norms), ("norms " + l.name).c_str());
    EXPECT(r_ref.median == r_gpu.median && r_ref.mad == r_gpu.mad && r_ref.threshold == r_gpu.threshold,
           ("median/mad/threshold " + l.name).c_str());
    EXPECT(r_ref.raw_outliers == r_gpu.raw_outliers && r_ref.aligned_outliers == r_gpu.aligned_outliers,
           ("outlier indices " + l.name).c_str());
    for (int bits : {8, 4})
      EXPECT(same_plan(qarvd::build_plan(W, r_ref, bits), qarvd::cuda::build_plan(W, r_ref, bits)),
             ("build_plan " + l.name).c_str());
    EXPECT(same_plan(qarvd::build_single_scale_plan(l.name, W, 8), qarvd::cuda::build_single_scale_plan(l.name, W, 8)),
           ("build_single_scale_plan " + l.name).c_str());
    EXPECT(same_bits(qarvd::matmul_nt(x, W).vec(), qarvd::cuda::matmul_nt(x, W).vec()), ("matmul_nt " + l.name).c_str());
  }
  std::printf("checked %zu quantized layers\n", n_layers);

  // ---- Eq. 5 weighted_loss (calibrate.cpp:201-224) on reference-initialised states
  {
    size_t n_loss = 0, same = 0;
    for (const auto& l : qm.layers) {
      if (l.preserved) continue;
      const Tensor& W = model.weight(l.name);
      const DualScalePlan plan = build_plan(W, qarvd::analyze_layer(l.name, W), 8);
      std::vector<CalibSample> samples(3);
      std::vector<const CalibSample*> batch;
      for (size_t s = 0; s < samples.size(); ++s) {
        samples[s].layer = l.name;
        samples[s].chunk = s + 1;
        samples[s].x = random_tensor(16 + 7 * s, l.in_dim, 900 + 31 * n_loss + s, 1.0);
        batch.push_back(&samples[s]);
      }
      const QuantParams act = init_scale_minmax(samples[0].x, 8, Granularity::per_tensor, 0);
      const LearnableQuantState st = LearnableQuantState::init(W, plan, act, opts.base);
      const double ref = qarvd::weighted_loss(batch, st, w);
      const double gpu = qarvd::cuda::weighted_loss(batch, st, w);
      same += std::memcmp(&ref, &gpu, 8) == 0;
      ++n_loss;
    }
    std::printf("weighted_loss: %zu / %zu layers bit-identical\n", same, n_loss);
    EXPECT(same == n_loss, "weighted_loss bit-identical");
    const Tensor& W = model.weight(qm.layers[1].name);
    const DualScalePlan plan = build_plan(W, qarvd::analyze_layer("l", W), 8);
    const LearnableQuantState st =
        LearnableQuantState::init(W, plan, QuantParams::per_tensor_symmetric(8, 0.1), opts.base);
    CalibSample s{"l", 9, random_tensor(4, W.cols(), 1, 1.0)};
    EXPECT(what_of([&] { qarvd::cuda::weighted_loss({&s}, st, w); }) ==
               "out_of_range: weighted loss: sample chunk outside the weight vector",
           "weighted_loss chunk out of range -> std::out_of_range with the reference message");
  }

  // ---- calibrate_layer (AdaRound, K7) vs the reference on the model's own captured samples
  {
    const std::vector<std::string> names = {"block0.ffn.2", "block1.self_attn.q"};
    const std::vector<CalibSample> cap = collect_calibration(model, {101, 102}, names);
    for (const std::string& name : names) {
      std::vector<const CalibSample*> ss;
      for (const CalibSample& c : cap)
        if (c.layer == name) ss.push_back(&c);
      const Tensor& W = model.weight(name);
      DualScalePlan plan = build_plan(W, qarvd::analyze_layer(name, W), 8);
      plan.layer_name = name;
      const QuantParams act = init_scale_minmax(ss[0]->x, 8, Granularity::per_tensor, 0);
      for (int iters : {0, 1, 40}) {
        CalibConfig cc = opts.base;
        cc.iterations = iters;
        const LayerCalibResult ref = qarvd::calibrate_layer(W, plan, act, ss, w, cc);
        const LayerCalibResult gpu = qarvd::cuda::calibrate_layer(W, plan, act, ss, w, cc);
        size_t diff = 0;
        for (size_t i = 0; i < ref.codes.data.size(); ++i) diff += ref.codes.data[i] != gpu.codes.data[i];
        double worst = std::fabs(gpu.final_loss - ref.final_loss) / std::fabs(ref.final_loss);
        worst = std::max(worst, std::fabs(gpu.initial_loss - ref.initial_loss) / std::fabs(ref.initial_loss));
        for (size_t r = 0; r < W.rows(); ++r)
          worst = std::max(worst, std::fabs(gpu.plan.params_normal.scale[r] - ref.plan.params_normal.scale[r]) /
                                      ref.plan.params_normal.scale[r]);
        worst = std::max(worst, std::fabs(gpu.act.scale[0] - ref.act.scale[0]) / ref.act.scale[0]);
        std::printf("calibrate_layer %s (%d iterations): %zu code mismatches, final loss %.6e vs %.6e, "
                    "worst rel diff %.3e\n", name.c_str(), iters, diff, gpu.final_loss, ref.final_loss, worst);
        EXPECT(diff == 0, ("calibrate_layer hard codes identical " + name).c_str());
        // learned scales, act scale and losses: the gradients' f64 products run in a different
        // summation order (tensor.cpp's sequential k loop vs blocked device sums), ~1e-15
        // relative per step; the learned activation scale's gradient is a long cancelling sum
        // (calibrate.cpp:293-294) that Adam's normalised step can amplify near zero
        EXPECT(worst <= 1e-6, ("calibrate_layer scales / losses " + name).c_str());
        if (iters == 0) EXPECT(gpu.initial_loss == ref.initial_loss || worst <= 1e-12, "initial loss");
      }
    }
  }

  // ---- calibrate_model with every per-layer step on the GPU vs the reference pipeline, at 1 and 8
  // worker threads (the reference's slot-indexed parallel_for contract, threading.hpp:13-14)
  for (unsigned threads : {1u, 8u}) {
    set_num_threads(threads);
    const ModelCalibResult gcal = qarvd::cuda::calibrate_model(model, w, opts);
    const QuantizedModel& gq = gcal.qmodel;
    size_t same = 0, total = 0, diff_codes = 0, n_codes = 0, same_plans = 0, same_act = 0;
    double worst = 0.0;
    for (size_t li = 0; li < qm.layers.size(); ++li) {
      const QuantizedLayer& a = qm.layers[li];
      const QuantizedLayer& b = gq.layers[li];
      EXPECT(a.preserved == b.preserved && a.name == b.name, "calibrate_model layer set");
      if (a.preserved) {
        EXPECT(same_bits(a.fp_weight.vec(), b.fp_weight.vec()), "calibrate_model preserved bf16 weights");
        continue;
      }
      ++total;
      EXPECT(a.plan.permutation == b.plan.permutation && a.plan.outlier_indices == b.plan.outlier_indices,
             "calibrate_model plans identical");
      same += a.wq.data == b.wq.data;
      for (size_t i = 0; i < a.wq.data.size(); ++i) {
        if (a.wq.data[i] != b.wq.data[i] && diff_codes < 8)
          std::printf("  code mismatch %s [%zu, %zu]: ref %d gpu %d\n", a.name.c_str(), i / a.in_dim, i % a.in_dim,
                      a.wq.data[i], b.wq.data[i]);
        diff_codes += a.wq.data[i] != b.wq.data[i];
      }
      n_codes += a.wq.data.size();
      same_plans += same_bits(a.plan.params_normal.scale, b.plan.params_normal.scale) &&
                    same_bits(a.plan.params_outlier.scale, b.plan.params_outlier.scale);
      same_act += a.act.scale[0] == b.act.scale[0];
      for (size_t r = 0; r < a.out_dim; ++r)
        worst = std::max(worst, std::fabs(a.plan.params_normal.scale[r] - b.plan.params_normal.scale[r]) /
                                    a.plan.params_normal.scale[r]);
      worst = std::max(worst, std::fabs(a.act.scale[0] - b.act.scale[0]) / a.act.scale[0]);
    }
    std::printf("calibrate_model (%u threads): %zu / %zu layers with identical pre-permuted codes (%zu of %zu codes "
                "differ), %zu bit-identical learned scale sets, %zu identical act scales, worst scale rel diff "
                "%.3e\n", threads, same, total, diff_codes, n_codes, same_plans, same_act, worst);
    EXPECT(diff_codes == 0, "calibrate_model codes identical");
    EXPECT(worst <= 1e-6, "calibrate_model learned scales");
  }
  set_num_threads(8);

  // ---- profile_sensitivity: exact providers, identical at 1 and 8 threads
  {
    const BitwidthScheme sch = BitwidthScheme::parse("w8a8");
    const SensitivityProfile a = qarvd::profile_sensitivity(model, sch, {5000, 5001, 5002});
    set_num_threads(1);
    const SensitivityProfile b1 = qarvd::cuda::profile_sensitivity(model, sch, {5000, 5001, 5002});
    set_num_threads(8);
    const SensitivityProfile b8 = qarvd::cuda::profile_sensitivity(model, sch, {5000, 5001, 5002});
    EXPECT(same_bits(a.alpha_raw, b1.alpha_raw) && same_bits(a.alpha_normalized, b1.alpha_normalized),
           "profile_sensitivity alpha bit-identical");
    EXPECT(same_bits(b1.alpha_raw, b8.alpha_raw), "profile_sensitivity thread-count invariant");
    std::printf("profile_sensitivity: %zu chunks, alpha bit-identical %d, 1 vs 8 threads identical %d\n",
                a.alpha_raw.size(), same_bits(a.alpha_raw, b1.alpha_raw), same_bits(b1.alpha_raw, b8.alpha_raw));
  }

  // ---- the seam: run_rollout through the CUDA providers vs the reference engines
  for (uint64_t seed : {5000ull, 5001ull})
    for (Engine e : {Engine::int_kernels, Engine::fakequant_sim}) {
      const Rollout ref = run_quantized(qm, seed, e);
      const Rollout gpu = qarvd::cuda::run_quantized(qm, seed, e);
      bool same = ref.chunks.size() == gpu.chunks.size();
      for (size_t c = 0; same && c < ref.chunks.size(); ++c) same = same_bits(ref.chunks[c].vec(), gpu.chunks[c].vec());
      std::printf("rollout seed %llu engine %s: bit-identical %d\n", static_cast<unsigned long long>(seed),
                  e == Engine::int_kernels ? "int" : "fakequant", same);
      EXPECT(same, "rollout latents bit-identical");
    }
  {
    const QuantMode mode = QuantMode::quantize_only_chunk(2, BitwidthScheme::parse("w4a8"));
    const Rollout a = qarvd::rollout(model, 42, mode, {"block0.ffn.0"});
    const Rollout b = qarvd::cuda::rollout(model, 42, mode, {"block0.ffn.0"});
    bool same = a.chunks.size() == b.chunks.size() && a.captures.size() == b.captures.size();
    for (size_t c = 0; same && c < a.chunks.size(); ++c) same = same_bits(a.chunks[c].vec(), b.chunks[c].vec());
    for (size_t c = 0; same && c < a.captures.size(); ++c) same = same_bits(a.captures[c].x.vec(), b.captures[c].x.vec());
    EXPECT(same, "rollout (MinMax fake-quant w4a8 on chunk 2) bit-identical");
  }

  // ---- concurrent provider use: 8 threads forwarding through one shared provider
  {
    const qarvd::cuda::CudaQuantizedProvider p(qm);
    std::vector<std::string> names;
    for (const auto& l : qm.layers) names.push_back(l.name);
    std::vector<Tensor> outs(names.size() * 4), ref(names.size() * 4);
    auto job = [&](size_t i) {
      const QuantizedLayer& l = qm.layer(names[i % names.size()]);
      outs[i] = p.forward(l.name, random_tensor(5 + i % 7, l.in_dim, 3000 + i, 1.0));
    };
    set_num_threads(1);
    parallel_for(outs.size(), job);
    ref = outs;
    set_num_threads(8);
    parallel_for(outs.size(), job);
    bool same = true;
    for (size_t i = 0; i < outs.size(); ++i) same = same && same_bits(outs[i].vec(), ref[i].vec());
    EXPECT(same, "shared CudaQuantizedProvider: 8 concurrent threads == 1 thread");
  }

  // ---- error convention: same exception types and messages as the reference
  {
    const qarvd::cuda::CudaQuantizedProvider p(qm);
    EXPECT(what_of([&] { p.forward("no_such_layer", Tensor({1, cfg.hidden})); }).rfind("out_of_range", 0) == 0,
           "missing layer -> std::out_of_range");
    for (const auto& l : qm.layers)
      if (l.preserved) {
        const IntTensor codes{{1, l.in_dim}, std::vector<int32_t>(l.in_dim), 8};
        EXPECT(what_of([&] { qarvd::kernel_b_gemm_dequant(codes, l); }) ==
                   what_of([&] { qarvd::cuda::kernel_b_gemm_dequant(codes, l); }),
               "preserved layer -> the reference's std::invalid_argument");
        break;
      }
    Tensor bad = random_tensor(2, qm.layers[1].in_dim, 3, 1.0);
    bad[5] = std::nan("");
    const QuantParams p8 = QuantParams::per_tensor_symmetric(8, 0.1);
    EXPECT(what_of([&] { qarvd::cuda::kernel_a_quantize_activation(bad, p8); }) ==
               "invalid_argument: quantize: non-finite input at flat index 5",
           "non-finite -> std::invalid_argument with the reference message");
    for (const auto& l : qm.layers)
      if (!l.preserved && l.plan.enabled) {
        Tensor bx = random_tensor(3, l.in_dim, 4, 1.0);
        bx[l.in_dim + l.plan.permutation[7]] = INFINITY;
        EXPECT(what_of([&] { qarvd::quantized_layer_forward(l, bx, Engine::int_kernels); }) ==
                   what_of([&] { qarvd::cuda::quantized_layer_forward(l, bx, Engine::int_kernels); }),
               "layer forward non-finite index in permuted order");
        break;
      }
  }

  std::printf(failures ? "DROPIN FAIL %d\n" : "DROPIN PASS\n", failures);
  return failures ? 1 : 0;
}
