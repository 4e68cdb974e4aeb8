// qarvd_cuda.hpp — drop-in CUDA backend for the reference's quantized-inference
// operators (/root/reference/proj/core/include/qarvd/engine.hpp, outlier.hpp).
//
// A maintainer adds this file pair to the reference tree (or links it from a
// separate target against `qarvd::core` + libqarvd_b200.so) and swaps
//     qarvd::kernel_a_quantize_activation  -> qarvd::cuda::kernel_a_quantize_activation
//     qarvd::kernel_b_gemm_dequant         -> qarvd::cuda::kernel_b_gemm_dequant
//     qarvd::quantized_layer_forward       -> qarvd::cuda::quantized_layer_forward
//     qarvd::analyze_layer                 -> qarvd::cuda::analyze_layer
//     qarvd::weighted_loss                 -> qarvd::cuda::weighted_loss
//     qarvd::calibrate_layer               -> qarvd::cuda::calibrate_layer
//     qarvd::calibrate_model               -> qarvd::cuda::calibrate_model
//     QuantizedProvider (engine.cpp:146-171) -> qarvd::cuda::CudaQuantizedProvider
// Signatures, argument meaning and exception types/messages follow the
// reference.  All arithmetic runs in libqarvd_b200.so (sm_100a); this file only
// stages host tensors to the device and maps C-ABI statuses to exceptions.
#pragma once

#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "qarvd/calibrate.hpp"
#include "qarvd/engine.hpp"
#include "qarvd/outlier.hpp"
#include "qarvd/quant.hpp"
#include "qarvd/sensitivity.hpp"
#include "qarvd/tensor.hpp"
#include "qarvd/toy_model.hpp"

namespace qarvd {
namespace cuda {

// engine.hpp:43 — codes bit-identical to qarvd::quantize (f64 inputs take the exact path).
IntTensor kernel_a_quantize_activation(const Tensor& x, const QuantParams& p);

// engine.hpp:48 — int8 tensor-core GEMM with two int32 accumulators (outlier / normal
// group) and an fp32 dequant epilogue; equals the reference within fp32 rounding.
Tensor kernel_b_gemm_dequant(const IntTensor& xq, const QuantizedLayer& layer);

// engine.hpp:51
Tensor permute_activations(const Tensor& x, const DualScalePlan& plan);

// engine.hpp:60 (Engine::int_kernels semantics; fakequant_sim is delegated to the reference)
Tensor quantized_layer_forward(const QuantizedLayer& layer, const Tensor& x, Engine engine);

// outlier.hpp:59-61 — bit-identical report (norms, median, MAD, threshold, index sets).
OutlierReport analyze_layer(const std::string& layer_name, const Tensor& w,
                            double tau = kDefaultTau, double alpha_min = kDefaultAlphaMin,
                            size_t align = kDefaultAlign);

// calibrate.hpp:80-82 — Eq. 5 with the deployable (hard-rounded) weights, evaluated by one
// fused tcgen05 kernel (qarvd_weighted_loss).  The f64 operands of the target X W^T are split
// into bf16 hi/lo parts and stacked along K ([X_hi X_hi X_lo] . [W_hi W_lo W_hi]^T, ~24-bit
// products, fp32 tensor-core accumulation); the prediction FQ(X) What^T is exact int8 x int8.
// Equals the reference within ~1e-5 relative; same exceptions (empty batch, chunk range).
double weighted_loss(const std::vector<const CalibSample*>& batch, const LearnableQuantState& state,
                     const std::vector<double>& chunk_weights);

// calibrate.hpp:112-116 — AdaRound calibration of one layer on the GPU (K7, f64): the same
// sampler, formulas and Adam schedule as the reference; identical hard codes, learned scales
// and losses to ~1e-9 relative.  Same config validation and exceptions.
LayerCalibResult calibrate_layer(const Tensor& w, const DualScalePlan& plan, const QuantParams& act_init,
                                 const std::vector<const CalibSample*>& samples,
                                 const std::vector<double>& chunk_weights, const CalibConfig& cfg);

// calibrate.hpp:137-139 — the whole-model pipeline with every per-layer step on the GPU:
// capture (the reference's full-precision rollouts, host f64 glue), outlier detection (K3),
// build_plan, the percentile activation init, AdaRound (K7) and the pre-permuted codes.
// Layers run one after another on the device (the reference's parallel_for is slot-indexed,
// so the result does not depend on the order).
ModelCalibResult calibrate_model(const ToyModel& model, const std::vector<double>& chunk_weights,
                                 const ModelCalibOptions& opts);

// Device-resident copy of one QuantizedLayer (codes padded into the kernel layout).
class DeviceLayer;

// LinearProvider (toy_model.hpp:77-81) serving a QuantizedModel from the GPU.  Layers
// are uploaded once; forward() is re-entrant (per-call workspace, one stream per call).
class CudaQuantizedProvider : public LinearProvider {
 public:
  explicit CudaQuantizedProvider(const QuantizedModel& qm);
  ~CudaQuantizedProvider() override;
  Tensor forward(const std::string& layer, const Tensor& x) const override;

 private:
  const QuantizedModel& qm_;
  std::map<std::string, std::shared_ptr<DeviceLayer>> layers_;
};

// MinMaxFakeQuantProvider (toy_model.cpp:306-325) on the tensor cores: fake_quant(x, per-tensor
// minmax) . fake_quant(W, per-channel minmax)^T = s_x * s_w[j] * (codes_x . codes_w), i.e. a
// single-slab int8 GEMM with the reference's f64 epilogue.  Weight codes / scales come from K5
// (single-scale plan), the activation scale from K1's exact per-row scales (max over rows).
class CudaMinMaxFakeQuantProvider : public LinearProvider {
 public:
  CudaMinMaxFakeQuantProvider(const ToyModel& model, BitwidthScheme scheme,
                              std::vector<std::string> keep_list = default_keep_list());
  ~CudaMinMaxFakeQuantProvider() override;
  Tensor forward(const std::string& layer, const Tensor& x) const override;

 private:
  const ToyModel& model_;
  BitwidthScheme scheme_;
  std::vector<std::string> keep_list_;
  std::map<std::string, std::shared_ptr<DeviceLayer>> layers_;
};

// profile_sensitivity (sensitivity.cpp:29-66) with the probes' quantized linears served by
// CudaMinMaxFakeQuantProvider (the full-precision references stay on FpProvider).
SensitivityProfile profile_sensitivity(const ToyModel& model, BitwidthScheme scheme,
                                       const std::vector<uint64_t>& seeds);

// run_quantized (engine.cpp:175-178) with the CUDA provider.
Rollout run_quantized(const QuantizedModel& qm, uint64_t prompt_seed);

}  // namespace cuda
}  // namespace qarvd
