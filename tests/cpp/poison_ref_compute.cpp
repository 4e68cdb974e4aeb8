// Poisoned definitions of the reference's compute functions (quant, outlier, dual_scale, engine,
// calibrate, sensitivity and the built-in providers).  Linked FIRST, with
// --allow-multiple-definition, in front of oracle/_ref/libqarvd_ref.a: every call that would
// reach the reference's CPU implementation of one of them aborts the process instead.
// test_no_ref_compute.cpp then runs the adapter's whole pipeline (qarvd::cuda::calibrate_model,
// the CUDA providers through run_rollout, profile_sensitivity, every operator entry) and must
// finish: the drop-in computes all of it in libqarvd_b200.so.  Only the reference's types, its
// validation helpers and the rollout driver's own f64 glue (rmsnorm / attention / GELU, which calls
// matmul_nt and matmul for the attention scores) remain live.
#include <cstdio>
#include <cstdlib>

#include "qarvd/calibrate.hpp"
#include "qarvd/dual_scale.hpp"
#include "qarvd/engine.hpp"
#include "qarvd/outlier.hpp"
#include "qarvd/quant.hpp"
#include "qarvd/sensitivity.hpp"
#include "qarvd/tensor.hpp"
#include "qarvd/toy_model.hpp"

[[noreturn]] static void poisoned(const char* fn) {
  std::fprintf(stderr, "POISONED reference compute function called: qarvd::%s\n", fn);
  std::fflush(stderr);
  std::abort();
}

namespace qarvd {
IntTensor quantize(const Tensor&, const QuantParams&) { poisoned("quantize"); }
Tensor dequantize(const IntTensor&, const QuantParams&) { poisoned("dequantize"); }
Tensor fake_quant(const Tensor&, const QuantParams&) { poisoned("fake_quant"); }
QuantParams init_scale_minmax(const Tensor&, int, Granularity, size_t) { poisoned("init_scale_minmax"); }
PercentileSearchResult init_scale_percentile_search(const std::vector<Tensor>&, int) {
  poisoned("init_scale_percentile_search");
}
Tensor channel_l2_norms(const Tensor&, size_t) { poisoned("channel_l2_norms"); }
MadResult mad(const std::vector<double>&) { poisoned("mad"); }
std::vector<size_t> detect_outliers(const std::vector<double>&, double, double) { poisoned("detect_outliers"); }
std::vector<size_t> align_outliers(const std::vector<size_t>&, const std::vector<double>&, size_t) {
  poisoned("align_outliers");
}
OutlierReport analyze_layer(const std::string&, const Tensor&, double, double, size_t) { poisoned("analyze_layer"); }
OutlierReport analyze_norms(const std::string&, std::vector<double>, double, double, size_t) {
  poisoned("analyze_norms");
}
DualScalePlan build_plan(const Tensor&, const OutlierReport&, int) { poisoned("build_plan"); }
DualScalePlan build_single_scale_plan(const std::string&, const Tensor&, int) { poisoned("build_single_scale_plan"); }
Tensor fake_quant_dual(const Tensor&, const DualScalePlan&) { poisoned("fake_quant_dual"); }
IntTensor kernel_a_quantize_activation(const Tensor&, const QuantParams&) { poisoned("kernel_a_quantize_activation"); }
Tensor kernel_b_gemm_dequant(const IntTensor&, const QuantizedLayer&) { poisoned("kernel_b_gemm_dequant"); }
Tensor permute_activations(const Tensor&, const DualScalePlan&) { poisoned("permute_activations"); }
Tensor quantized_layer_forward(const QuantizedLayer&, const Tensor&, Engine) { poisoned("quantized_layer_forward"); }
Rollout run_quantized(const QuantizedModel&, uint64_t, Engine) { poisoned("run_quantized"); }
std::vector<CalibSample> collect_calibration(const ToyModel&, const std::vector<uint64_t>&,
                                             const std::vector<std::string>&) {
  poisoned("collect_calibration");
}
LearnableQuantState LearnableQuantState::init(const Tensor&, const DualScalePlan&, const QuantParams&,
                                              const CalibConfig&) {
  poisoned("LearnableQuantState::init");
}
Tensor LearnableQuantState::soft_weight() const { poisoned("LearnableQuantState::soft_weight"); }
Tensor LearnableQuantState::hard_weight() const { poisoned("LearnableQuantState::hard_weight"); }
IntTensor LearnableQuantState::hard_codes() const { poisoned("LearnableQuantState::hard_codes"); }
double weighted_loss(const std::vector<const CalibSample*>&, const LearnableQuantState&, const std::vector<double>&) {
  poisoned("weighted_loss");
}
double soft_weighted_loss(const std::vector<const CalibSample*>&, const LearnableQuantState&,
                          const std::vector<double>&) {
  poisoned("soft_weighted_loss");
}
CalibGradients soft_loss_gradients(const std::vector<const CalibSample*>&, const LearnableQuantState&,
                                   const std::vector<double>&) {
  poisoned("soft_loss_gradients");
}
LayerCalibResult calibrate_layer(const Tensor&, const DualScalePlan&, const QuantParams&,
                                 const std::vector<const CalibSample*>&, const std::vector<double>&,
                                 const CalibConfig&) {
  poisoned("calibrate_layer");
}
ModelCalibResult calibrate_model(const ToyModel&, const std::vector<double>&, const ModelCalibOptions&) {
  poisoned("calibrate_model");
}
SensitivityProfile profile_sensitivity(const ToyModel&, BitwidthScheme, const std::vector<uint64_t>&) {
  poisoned("profile_sensitivity");
}
Tensor FpProvider::forward(const std::string&, const Tensor&) const { poisoned("FpProvider::forward"); }
MinMaxFakeQuantProvider::MinMaxFakeQuantProvider(const ToyModel& model, BitwidthScheme, std::vector<std::string>)
    : model_(model) {
  poisoned("MinMaxFakeQuantProvider");
}
Tensor MinMaxFakeQuantProvider::forward(const std::string&, const Tensor&) const {
  poisoned("MinMaxFakeQuantProvider::forward");
}
Rollout rollout(const ToyModel&, uint64_t, const QuantMode&, const std::vector<std::string>&) { poisoned("rollout"); }
}  // namespace qarvd
