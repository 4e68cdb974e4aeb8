// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers around the UNMODIFIED reference functions of
// /root/reference/proj/core (compiled from those sources by oracle/Makefile
// into oracle/_ref/libqarvd_ref.so).  Used to pin the C restatement
// (oracle/qarvd_oracle.c), to generate tests/golden fixtures, and as the
// reference CPU arm of bench.py (`--impl reference`).  Never linked into the
// product library.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "qarvd/calibrate.hpp"
#include "qarvd/dual_scale.hpp"
#include "qarvd/engine.hpp"
#include "qarvd/outlier.hpp"
#include "qarvd/quant.hpp"
#include "qarvd/sensitivity.hpp"
#include "qarvd/tensor.hpp"
#include "qarvd/threading.hpp"
#include "qarvd/toy_model.hpp"

using namespace qarvd;

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = std::string("invalid_argument: ") + e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = std::string("out_of_range: ") + e.what();
    return 2;
  } catch (const std::logic_error& e) {
    g_err = std::string("logic_error: ") + e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = std::string("runtime_error: ") + e.what();
    return 4;
  }
}

Tensor make_tensor(const double* x, int64_t r, int64_t c) {
  return Tensor({static_cast<size_t>(r), static_cast<size_t>(c)},
                std::vector<double>(x, x + r * c));
}

// A QuantizedLayer whose plan reproduces a permutation with `n_outlier` leading entries.
QuantizedLayer make_layer(const int32_t* wq, int64_t n, int64_t k, const uint32_t* perm,
                          int64_t n_outlier, int enabled, const double* s_o, const double* s_n,
                          double s_x) {
  QuantizedLayer l;
  l.name = "shim";
  l.out_dim = static_cast<size_t>(n);
  l.in_dim = static_cast<size_t>(k);
  l.preserved = false;
  l.wq.shape = {static_cast<size_t>(n), static_cast<size_t>(k)};
  l.wq.bits = 8;
  l.wq.data.assign(wq, wq + n * k);
  l.plan.layer_name = "shim";
  l.plan.enabled = enabled != 0;
  l.plan.d_in = static_cast<size_t>(k);
  l.plan.permutation.assign(perm, perm + k);
  if (enabled) {
    l.plan.outlier_indices.assign(perm, perm + n_outlier);
    l.plan.normal_indices.assign(perm + n_outlier, perm + k);
  } else {
    l.plan.normal_indices.assign(perm, perm + k);
  }
  l.plan.params_normal =
      QuantParams::per_channel_symmetric(8, 0, std::vector<double>(s_n, s_n + n));
  l.plan.params_outlier =
      enabled ? QuantParams::per_channel_symmetric(8, 0, std::vector<double>(s_o, s_o + n))
              : l.plan.params_normal;
  l.act = QuantParams::per_tensor_symmetric(8, s_x);
  return l;
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
void ref_set_threads(unsigned n) { set_num_threads(n); }
unsigned ref_num_threads(void) { return num_threads(); }

// quantize(x, p): per_token -> p = init_scale_minmax(x, bits, per_channel, 0); else static s.
int ref_quantize(const double* x, int64_t m, int64_t k, int per_token, double s, int bits,
                 int32_t* codes, double* scales) {
  return guarded([&] {
    const Tensor t = make_tensor(x, m, k);
    const QuantParams p = per_token ? init_scale_minmax(t, bits, Granularity::per_channel, 0)
                                    : QuantParams::per_tensor_symmetric(bits, s);
    const IntTensor q = kernel_a_quantize_activation(t, p);
    std::memcpy(codes, q.data.data(), sizeof(int32_t) * q.data.size());
    if (scales)
      for (int64_t i = 0; i < m; ++i) scales[i] = p.scale_for(per_token ? i : 0);
  });
}

// permute_activations(x, plan) for a plan with the given permutation
int ref_permute(const double* x, int64_t m, int64_t k, const uint32_t* perm, int enabled,
                double* out) {
  return guarded([&] {
    DualScalePlan plan;
    plan.enabled = enabled != 0;
    plan.d_in = static_cast<size_t>(k);
    plan.permutation.assign(perm, perm + k);
    const Tensor o = permute_activations(make_tensor(x, m, k), plan);
    std::memcpy(out, o.data(), sizeof(double) * o.size());
  });
}

// kernel_b_gemm_dequant with a per-row activation scale (rows are independent,
// engine.cpp:86, so the per-token result is kernel B applied row block by row block).
int ref_kernel_b(const int32_t* xq, int64_t m, int64_t k, const int32_t* wq, int64_t n,
                 const uint32_t* perm, int64_t n_outlier, int enabled, const double* s_x,
                 int per_row, const double* s_o, const double* s_n, double* out) {
  return guarded([&] {
    QuantizedLayer base = make_layer(wq, n, k, perm, n_outlier, enabled, s_o, s_n, s_x[0]);
    if (!per_row) {
      IntTensor q;
      q.shape = {static_cast<size_t>(m), static_cast<size_t>(k)};
      q.data.assign(xq, xq + m * k);
      const Tensor y = kernel_b_gemm_dequant(q, base);
      std::memcpy(out, y.data(), sizeof(double) * y.size());
      return;
    }
    parallel_for(static_cast<size_t>(m), [&](size_t i) {
      QuantizedLayer l = base;  // per-row activation scale
      l.act = QuantParams::per_tensor_symmetric(8, s_x[i]);
      IntTensor q;
      q.shape = {1, static_cast<size_t>(k)};
      q.data.assign(xq + i * k, xq + (i + 1) * k);
      const Tensor y = kernel_b_gemm_dequant(q, l);
      std::memcpy(out + i * n, y.data(), sizeof(double) * n);
    });
  });
}

// analyze_layer(name, W, tau, alpha_min, align)
int ref_analyze_layer(const double* w, int64_t n, int64_t k, double tau, double alpha_min,
                      int64_t align, double* norms, double* stats, int64_t* counts, int64_t* raw,
                      int64_t* aligned) {
  return guarded([&] {
    const OutlierReport r =
        analyze_layer("shim", make_tensor(w, n, k), tau, alpha_min, static_cast<size_t>(align));
    std::memcpy(norms, r.norms.data(), sizeof(double) * r.norms.size());
    stats[0] = r.median;
    stats[1] = r.mad;
    stats[2] = r.threshold;
    counts[0] = static_cast<int64_t>(r.raw_outliers.size());
    counts[1] = static_cast<int64_t>(r.aligned_outliers.size());
    for (size_t i = 0; i < r.raw_outliers.size(); ++i) raw[i] = static_cast<int64_t>(r.raw_outliers[i]);
    for (size_t i = 0; i < r.aligned_outliers.size(); ++i)
      aligned[i] = static_cast<int64_t>(r.aligned_outliers[i]);
  });
}

// detect_outliers / align_outliers / mad on a norm vector
int ref_analyze_norms(const double* v, int64_t k, double tau, double alpha_min, int64_t align,
                      double* stats, int64_t* counts, int64_t* raw, int64_t* aligned) {
  return guarded([&] {
    const OutlierReport r = analyze_norms("shim", std::vector<double>(v, v + k), tau, alpha_min,
                                          static_cast<size_t>(align));
    stats[0] = r.median;
    stats[1] = r.mad;
    stats[2] = r.threshold;
    counts[0] = static_cast<int64_t>(r.raw_outliers.size());
    counts[1] = static_cast<int64_t>(r.aligned_outliers.size());
    for (size_t i = 0; i < r.raw_outliers.size(); ++i) raw[i] = static_cast<int64_t>(r.raw_outliers[i]);
    for (size_t i = 0; i < r.aligned_outliers.size(); ++i)
      aligned[i] = static_cast<int64_t>(r.aligned_outliers[i]);
  });
}

// build_plan(W, report with the given aligned outliers) + nearest codes per group,
// pre-permuted [outlier | normal] (calibrate.cpp:474-480).  Codes are produced by
// the reference quantize() on each column group with the plan's per-row params.
int ref_build_plan_codes(const double* w, int64_t n, int64_t k, const int64_t* outliers,
                         int64_t n_out, int bits, double* s_o, double* s_n, uint32_t* perm,
                         int32_t* wq_perm, int* enabled) {
  return guarded([&] {
    const Tensor W = make_tensor(w, n, k);
    OutlierReport rep;
    rep.layer_name = "shim";
    rep.aligned_outliers.assign(outliers, outliers + n_out);
    const DualScalePlan plan = build_plan(W, rep, bits);
    *enabled = plan.enabled ? 1 : 0;
    for (int64_t r = 0; r < n; ++r) {
      s_o[r] = plan.params_outlier.scale[r];
      s_n[r] = plan.params_normal.scale[r];
    }
    std::memcpy(perm, plan.permutation.data(), sizeof(uint32_t) * k);
    const size_t n_o = plan.enabled ? plan.outlier_count() : 0;
    auto group_codes = [&](const std::vector<size_t>& cols, const QuantParams& p, size_t pos0) {
      if (cols.empty()) return;
      Tensor g({static_cast<size_t>(n), cols.size()});
      for (int64_t r = 0; r < n; ++r)
        for (size_t c = 0; c < cols.size(); ++c) g.at(r, c) = W.at(r, cols[c]);
      const IntTensor q = quantize(g, p);
      for (int64_t r = 0; r < n; ++r)
        for (size_t c = 0; c < cols.size(); ++c) wq_perm[r * k + pos0 + c] = q.at(r, c);
    };
    if (plan.enabled) group_codes(plan.outlier_indices, plan.params_outlier, 0);
    group_codes(plan.normal_indices, plan.params_normal, n_o);
  });
}

// init_scale_percentile_search over `frames` samples of [rows x k]
int ref_percentile_search(const double* x, int64_t frames, int64_t rows, int64_t k, int bits,
                          double* best_pct, double* scale, double* cand_mse) {
  return guarded([&] {
    std::vector<Tensor> samples;
    for (int64_t f = 0; f < frames; ++f) samples.push_back(make_tensor(x + f * rows * k, rows, k));
    const PercentileSearchResult r = init_scale_percentile_search(samples, bits);
    *best_pct = r.best_percentile;
    *scale = r.params.scale[0];
    for (size_t c = 0; c < r.candidate_mse.size(); ++c) cand_mse[c] = r.candidate_mse[c];
  });
}

// weighting_strategy(profile, kind) with a profile whose normalized alpha is given
int ref_weighting(int kind, const double* alpha_raw, int64_t n, double* out) {
  return guarded([&] {
    SensitivityProfile prof;
    prof.alpha_raw.assign(alpha_raw, alpha_raw + n);
    prof.alpha_normalized = normalize_alpha(prof.alpha_raw);
    const std::vector<double> w = weighting_strategy(prof, static_cast<WeightingKind>(kind));
    std::memcpy(out, w.data(), sizeof(double) * n);
  });
}

// ToyModel::build (toy_model.cpp:126-170): weight of `layer` with one injection rule
int ref_toy_weight(int64_t blocks, int64_t hidden, uint64_t seed, const char* pattern,
                   double fraction, double gamma, const char* layer, double* out, int64_t* rows,
                   int64_t* cols) {
  return guarded([&] {
    ToyModelConfig cfg;
    cfg.blocks = static_cast<size_t>(blocks);
    cfg.hidden = static_cast<size_t>(hidden);
    cfg.seed = seed;
    if (pattern && pattern[0]) cfg.injections.push_back({pattern, fraction, gamma});
    const ToyModel m = ToyModel::build(cfg);
    const Tensor& w = m.weight(layer);
    *rows = static_cast<int64_t>(w.rows());
    *cols = static_cast<int64_t>(w.cols());
    if (out) std::memcpy(out, w.data(), sizeof(double) * w.size());
  });
}

// round_half_even (quant.hpp:14-20)
double ref_round_half_even(double v) { return round_half_even(v); }

// Timed reference CPU path for one quantized linear:
// permute_activations -> kernel_a_quantize_activation -> kernel_b_gemm_dequant
// (engine.cpp:137-139), row-sharded with the reference parallel_for (rows are
// independent).  Returns seconds; y receives the f64 output.
double ref_time_linear(const double* x, int64_t m, int64_t k, const int32_t* wq, int64_t n,
                       const uint32_t* perm, int64_t n_outlier, int enabled, const double* s_o,
                       const double* s_n, double s_x, int64_t rows_per_task, double* y) {
  double secs = -1.0;
  guarded([&] {
    const QuantizedLayer layer = make_layer(wq, n, k, perm, n_outlier, enabled, s_o, s_n, s_x);
    const Tensor X = make_tensor(x, m, k);
    const size_t tasks = static_cast<size_t>((m + rows_per_task - 1) / rows_per_task);
    const auto t0 = std::chrono::steady_clock::now();
    parallel_for(tasks, [&](size_t t) {
      const int64_t r0 = static_cast<int64_t>(t) * rows_per_task;
      const int64_t r1 = std::min<int64_t>(m, r0 + rows_per_task);
      Tensor xs({static_cast<size_t>(r1 - r0), static_cast<size_t>(k)});
      std::memcpy(xs.data(), X.data() + r0 * k, sizeof(double) * (r1 - r0) * k);
      const Tensor xp = permute_activations(xs, layer.plan);
      const IntTensor xq = kernel_a_quantize_activation(xp, layer.act);
      const Tensor out = kernel_b_gemm_dequant(xq, layer);
      if (y) std::memcpy(y + r0 * n, out.data(), sizeof(double) * out.size());
    });
    secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
  return secs;
}


// Timed reference CPU path for a CHAIN of quantized linears with per-token activation scales
// (the BASELINE workloads): for each row, init_scale_minmax(row, 8, per_channel, axis 0)
// (quant.cpp:161-183) gives the row's scale, then permute_activations -> kernel_a ->
// kernel_b (engine.cpp:137-139) with that scale (kernel B reads act.scale[0], engine.cpp:57,
// so per-token = kernel B row by row), an optional erf-GELU between layers
// (toy_model.cpp:63-67), and the output feeds the next linear.  Row blocks run on the
// reference parallel_for (rows are independent).  layer l: wq [n_l x k_l] pre-permuted int32,
// perm [k_l], scales [n_l]; gelu_after[l] != 0 applies GELU to layer l's output.  Returns
// seconds; y (optional) receives the last layer's f64 output [m x n_last].
struct ChainLayerArgs {
  const int32_t* wq;
  int64_t n, k;
  const uint32_t* perm;
  int64_t n_outlier;
  int enabled;
  const double* s_o;
  const double* s_n;
  int gelu_after;
};
double ref_time_chain_per_token(const double* x, int64_t m, const ChainLayerArgs* layers, int n_layers,
                                int64_t rows_per_task, double* y) {
  double secs = -1.0;
  guarded([&] {
    std::vector<QuantizedLayer> ql;
    for (int l = 0; l < n_layers; ++l)
      ql.push_back(make_layer(layers[l].wq, layers[l].n, layers[l].k, layers[l].perm, layers[l].n_outlier,
                              layers[l].enabled, layers[l].s_o, layers[l].s_n, 1.0));
    const int64_t k0 = layers[0].k, n_last = layers[n_layers - 1].n;
    const size_t tasks = static_cast<size_t>((m + rows_per_task - 1) / rows_per_task);
    const auto t0 = std::chrono::steady_clock::now();
    parallel_for(tasks, [&](size_t t) {
      const int64_t r0 = static_cast<int64_t>(t) * rows_per_task;
      const int64_t r1 = std::min<int64_t>(m, r0 + rows_per_task);
      Tensor cur({static_cast<size_t>(r1 - r0), static_cast<size_t>(k0)});
      std::memcpy(cur.data(), x + r0 * k0, sizeof(double) * (r1 - r0) * k0);
      std::vector<QuantizedLayer> task_layers = ql;  // one copy per task: act is set per row
      for (int l = 0; l < n_layers; ++l) {
        QuantizedLayer& layer = task_layers[static_cast<size_t>(l)];
        const QuantParams per_token = init_scale_minmax(cur, 8, Granularity::per_channel, 0);
        const Tensor xp = permute_activations(cur, layer.plan);
        Tensor out({cur.rows(), layer.out_dim});
        for (size_t i = 0; i < cur.rows(); ++i) {
          Tensor row({1, layer.in_dim});
          std::memcpy(row.data(), xp.data() + i * layer.in_dim, sizeof(double) * layer.in_dim);
          layer.act = QuantParams::per_tensor_symmetric(8, per_token.scale[i]);
          const Tensor o = kernel_b_gemm_dequant(kernel_a_quantize_activation(row, layer.act), layer);
          std::memcpy(out.data() + i * layer.out_dim, o.data(), sizeof(double) * layer.out_dim);
        }
        if (layers[l].gelu_after)
          for (size_t e = 0; e < out.size(); ++e) out[e] = 0.5 * out[e] * (1.0 + std::erf(out[e] / std::sqrt(2.0)));
        cur = std::move(out);
      }
      if (y) std::memcpy(y + r0 * n_last, cur.data(), sizeof(double) * cur.size());
    });
    secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
  return secs;
}

// Timed reference toy rollouts (config 5 at toy scale): run_quantized (engine.cpp:175-178)
// through the reference QuantizedProvider(int) for `n_seeds` prompt seeds of a toy model
// calibrated by the reference calibrate_model (`iterations` AdaRound steps).  Calibration is
// untimed; the seeds run on the reference parallel_for.  Returns seconds for all rollouts.
double ref_time_toy_rollouts(int iterations, int n_seeds) {
  double secs = -1.0;
  guarded([&] {
    ToyModelConfig cfg;
    cfg.injections = {{"ffn.2", 0.05, 8.0}, {"self_attn.q", 0.03, 6.0}};
    const ToyModel model = ToyModel::build(cfg);
    SensitivityProfile prof;
    prof.alpha_raw.assign(cfg.chunks, 1.0);
    prof.alpha_normalized = normalize_alpha(prof.alpha_raw);
    ModelCalibOptions opts;
    opts.base.iterations = iterations;
    const ModelCalibResult calib =
        calibrate_model(model, weighting_strategy(prof, WeightingKind::heuristic_exp), opts);
    std::vector<Rollout> out(static_cast<size_t>(n_seeds));
    const auto t0 = std::chrono::steady_clock::now();
    parallel_for(static_cast<size_t>(n_seeds), [&](size_t s) {
      out[s] = run_quantized(calib.qmodel, 5000 + s, Engine::int_kernels);
    });
    secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
  return secs;
}
}  // extern "C"

// weighted_loss (calibrate.cpp:220-224) on a LearnableQuantState initialised by the reference
// (LearnableQuantState::init with build_plan(W, aligned outliers) and a per-tensor act scale),
// over samples x[row_off[s] .. row_off[s+1]) with 1-based chunks.  Also exports the state's
// deployable quantities: hard codes (original column order), per-row group scales
// weight_scale(r, g) and act_scale(), so the GPU objective can be run on the same state.
extern "C" int ref_weighted_loss(const double* w, int64_t n, int64_t k, const int64_t* outliers,
                                 int64_t n_out, double act_scale, const double* x,
                                 const int64_t* row_off, const int64_t* chunk, int64_t n_samples,
                                 const double* chunk_w, int64_t n_chunks, double* loss,
                                 int32_t* codes, double* s_wo, double* s_wn, double* act_out,
                                 uint8_t* outlier_mask) {
  return guarded([&] {
    const Tensor W = make_tensor(w, n, k);
    OutlierReport rep;
    rep.layer_name = "shim";
    rep.aligned_outliers.assign(outliers, outliers + n_out);
    const DualScalePlan plan = build_plan(W, rep, 8);
    CalibConfig cfg;
    const LearnableQuantState st =
        LearnableQuantState::init(W, plan, QuantParams::per_tensor_symmetric(8, act_scale), cfg);
    std::vector<CalibSample> samples(static_cast<size_t>(n_samples));
    std::vector<const CalibSample*> batch;
    for (int64_t s = 0; s < n_samples; ++s) {
      samples[s].layer = "shim";
      samples[s].chunk = static_cast<size_t>(chunk[s]);
      samples[s].x = make_tensor(x + row_off[s] * k, row_off[s + 1] - row_off[s], k);
      batch.push_back(&samples[s]);
    }
    const std::vector<double> cw(chunk_w, chunk_w + n_chunks);
    *loss = weighted_loss(batch, st, cw);
    const IntTensor hc = st.hard_codes();
    std::memcpy(codes, hc.data.data(), sizeof(int32_t) * n * k);
    for (int64_t r = 0; r < n; ++r) {
      s_wo[r] = st.weight_scale(static_cast<size_t>(r), true);
      s_wn[r] = st.weight_scale(static_cast<size_t>(r), false);
    }
    *act_out = st.act_scale();
    std::memset(outlier_mask, 0, static_cast<size_t>(k));
    if (plan.enabled)
      for (size_t c : plan.outlier_indices) outlier_mask[c] = 1;
  });
}

// calibrate_layer (calibrate.cpp:298-396) with build_plan(W, aligned outliers) and a per-tensor
// act_init; default CalibConfig except iterations / batch size / seed.  Exports the learned
// scales, hard codes, act scale, losses and the trace.
extern "C" int ref_calibrate_layer_bits(const double* w, int64_t n, int64_t k, const int64_t* outliers,
                                        int64_t n_out, double act_scale, const double* x,
                                        const int64_t* row_off, const int64_t* chunk, int64_t n_samples,
                                        const double* chunk_w, int64_t n_chunks, int iterations,
                                        int batch_size, uint64_t seed, const char* name, int32_t* codes,
                                        double* s_n, double* s_o, double* scalars, double* trace,
                                        double* init_s_n, double* init_s_o, int w_bits, int act_bits) {
  return guarded([&] {
    const Tensor W = make_tensor(w, n, k);
    OutlierReport rep;
    rep.layer_name = name;
    rep.aligned_outliers.assign(outliers, outliers + n_out);
    DualScalePlan plan = build_plan(W, rep, w_bits);
    plan.layer_name = name;
    for (int64_t r = 0; r < n; ++r) {
      init_s_n[r] = plan.params_normal.scale[r];
      init_s_o[r] = plan.params_outlier.scale[r];
    }
    CalibConfig cfg;
    cfg.iterations = iterations;
    cfg.batch_size = batch_size;
    cfg.seed = seed;
    std::vector<CalibSample> samples(static_cast<size_t>(n_samples));
    std::vector<const CalibSample*> ptrs;
    for (int64_t s = 0; s < n_samples; ++s) {
      samples[s].layer = name;
      samples[s].chunk = static_cast<size_t>(chunk[s]);
      samples[s].x = make_tensor(x + row_off[s] * k, row_off[s + 1] - row_off[s], k);
      ptrs.push_back(&samples[s]);
    }
    const std::vector<double> cw(chunk_w, chunk_w + n_chunks);
    const LayerCalibResult r = calibrate_layer(W, plan, QuantParams::per_tensor_symmetric(act_bits, act_scale),
                                               ptrs, cw, cfg);
    std::memcpy(codes, r.codes.data.data(), sizeof(int32_t) * n * k);
    for (int64_t i = 0; i < n; ++i) {
      s_n[i] = r.plan.params_normal.scale[i];
      s_o[i] = r.plan.params_outlier.scale[i];
    }
    scalars[0] = r.act.scale[0];
    scalars[1] = r.initial_loss;
    scalars[2] = r.final_loss;
    for (size_t t = 0; t < r.trace.size(); ++t) trace[t] = r.trace[t];
  });
}

extern "C" int ref_calibrate_layer(const double* w, int64_t n, int64_t k, const int64_t* outliers,
                                   int64_t n_out, double act_scale, const double* x,
                                   const int64_t* row_off, const int64_t* chunk, int64_t n_samples,
                                   const double* chunk_w, int64_t n_chunks, int iterations,
                                   int batch_size, uint64_t seed, const char* name, int32_t* codes,
                                   double* s_n, double* s_o, double* scalars, double* trace,
                                   double* init_s_n, double* init_s_o) {
  return ref_calibrate_layer_bits(w, n, k, outliers, n_out, act_scale, x, row_off, chunk, n_samples,
                                  chunk_w, n_chunks, iterations, batch_size, seed, name, codes, s_n, s_o,
                                  scalars, trace, init_s_n, init_s_o, 8, 8);
}

// The reference pipeline's own model file: ToyModel::build (two injections) -> calibrate_model
// (heuristic_exp chunk weights, `iterations` AdaRound steps) -> save_quantized_model(path).
extern "C" int ref_toy_qarq_bits(const char* path, int iterations, int weight_bits, int64_t* n_layers);
extern "C" int ref_toy_qarq(const char* path, int iterations, int64_t* n_layers) {
  return ref_toy_qarq_bits(path, iterations, 8, n_layers);
}
// the same pipeline at another weight bit width (CalibConfig::scheme, e.g. W4A8: the QARQ file
// then holds packed 4-bit codes, tensor.cpp:221-264)
extern "C" int ref_toy_qarq_bits(const char* path, int iterations, int weight_bits, int64_t* n_layers) {
  return guarded([&] {
    ToyModelConfig cfg;
    cfg.injections = {{"ffn.2", 0.05, 8.0}, {"self_attn.q", 0.03, 6.0}};
    const ToyModel model = ToyModel::build(cfg);
    SensitivityProfile prof;
    prof.alpha_raw.assign(cfg.chunks, 1.0);
    prof.alpha_normalized = normalize_alpha(prof.alpha_raw);
    const std::vector<double> w = weighting_strategy(prof, WeightingKind::heuristic_exp);
    ModelCalibOptions opts;
    opts.base.iterations = iterations;
    opts.base.batch_size = 2;
    opts.base.scheme.weight_bits = weight_bits;
    const ModelCalibResult r = calibrate_model(model, w, opts);
    save_quantized_model(path, r.qmodel);
    *n_layers = static_cast<int64_t>(r.qmodel.layers.size());
  });
}

// load_quantized_model(path) layer idx: meta = {preserved, out_dim, in_dim, enabled,
// outlier_count, bits}; arrays sized by the caller from a first call with null arrays.
extern "C" int ref_qarq_layer(const char* path, int64_t idx, int64_t* meta, int32_t* wq, double* s_n,
                              double* s_o, uint32_t* perm, double* act) {
  return guarded([&] {
    const QuantizedModel qm = load_quantized_model(path);
    const QuantizedLayer& l = qm.layers.at(static_cast<size_t>(idx));
    meta[0] = l.preserved;
    meta[1] = static_cast<int64_t>(l.out_dim);
    meta[2] = static_cast<int64_t>(l.in_dim);
    meta[3] = l.preserved ? 0 : l.plan.enabled;
    meta[4] = l.preserved ? 0 : static_cast<int64_t>(l.plan.enabled ? l.plan.outlier_count() : 0);
    meta[5] = l.preserved ? 16 : l.wq.bits;
    if (l.preserved || !wq) return;
    std::memcpy(wq, l.wq.data.data(), sizeof(int32_t) * l.wq.data.size());
    for (size_t r = 0; r < l.out_dim; ++r) {
      s_n[r] = l.plan.params_normal.scale[r];
      s_o[r] = l.plan.params_outlier.scale[r];
    }
    std::memcpy(perm, l.plan.permutation.data(), sizeof(uint32_t) * l.in_dim);
    act[0] = l.act.scale[0];
    act[1] = l.act.zero_point[0];
  });
}
