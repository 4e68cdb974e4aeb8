// Runs the drop-in's whole pipeline with the reference's compute functions poisoned
// (poison_ref_compute.cpp, linked in front of the reference library): calibrate_model, the
// providers through run_rollout, profile_sensitivity and every operator entry must complete
// without touching the reference's CPU implementations.
#include <cstdio>

#include "../../paper_2605_21072_b200/adapter/qarvd_cuda.hpp"
#include "qarvd/rng.hpp"
#include "qarvd/threading.hpp"

using namespace qarvd;

int main() {
  ToyModelConfig cfg;
  cfg.injections = {{"ffn.2", 0.05, 8.0}, {"self_attn.q", 0.03, 6.0}};
  const ToyModel model = ToyModel::build(cfg);
  set_num_threads(4);
  SensitivityProfile prof = qarvd::cuda::profile_sensitivity(model, BitwidthScheme::parse("w8a8"), {5000, 5001});
  const std::vector<double> w = weighting_strategy(prof, WeightingKind::final_quality);
  ModelCalibOptions opts;
  opts.base.iterations = 4;
  opts.base.batch_size = 2;
  const ModelCalibResult calib = qarvd::cuda::calibrate_model(model, w, opts);
  double sink = 0.0;
  for (Engine e : {Engine::int_kernels, Engine::fakequant_sim}) {
    const Rollout r = qarvd::cuda::run_quantized(calib.qmodel, 5000, e);
    sink += r.chunks.back()[0];
  }
  Prng rng(7);
  for (const auto& l : calib.qmodel.layers) {
    Tensor x({6, l.in_dim});
    for (size_t i = 0; i < x.size(); ++i) x[i] = rng.gaussian();
    for (Engine e : {Engine::int_kernels, Engine::fakequant_sim}) sink += qarvd::cuda::quantized_layer_forward(l, x, e)[0];
    if (l.preserved) continue;
    const Tensor& W = model.weight(l.name);
    const OutlierReport rep = qarvd::cuda::analyze_layer(l.name, W);
    const DualScalePlan plan = qarvd::cuda::build_plan(W, rep, 8);
    const Tensor xp = qarvd::cuda::permute_activations(x, plan);
    const IntTensor xq = qarvd::cuda::kernel_a_quantize_activation(xp, l.act);
    sink += qarvd::cuda::kernel_b_gemm_dequant(xq, l)[0];
    sink += qarvd::cuda::fake_quant(x, qarvd::cuda::init_scale_minmax(x, 8, Granularity::per_channel, 0))[0];
    sink += qarvd::cuda::init_scale_percentile_search({x, xp}, 8).params.scale[0];
  }
  std::printf("NO_REF_COMPUTE PASS (checksum %.6e, %zu layers)\n", sink, calib.qmodel.layers.size());
  return 0;
}
