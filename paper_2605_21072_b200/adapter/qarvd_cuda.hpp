// qarvd_cuda.hpp — drop-in CUDA backend for the reference's quantization, inference and
// calibration operators (/root/reference/proj/core/include/qarvd/{quant,dual_scale,engine,
// outlier,calibrate,sensitivity,toy_model,tensor}.hpp).
//
// A maintainer adds this file pair to the reference tree (or links it from a separate target
// against `qarvd::core` + libqarvd_b200.so) and swaps qarvd::X -> qarvd::cuda::X for the
// functions below.  Signatures, argument meaning, results and exception types / messages follow
// the reference; every arithmetic step runs in libqarvd_b200.so (sm_100a).  This file pair only
// stages host tensors, keeps one device context (stream + workspaces) per calling thread, and
// maps C-ABI statuses to exceptions.  From the reference library it uses the types, the
// parameter validation (QuantParams::validate, CalibConfig::validate), and the host drivers that
// call through the LinearProvider seam (run_rollout with its f64 glue, parallel_for,
// latent_mse / normalize_alpha): no reference compute function is called (tests/cpp/
// test_no_ref_compute.cpp links the adapter against poisoned copies of them).
//
// Thread safety: every function and provider method may be called concurrently from any number
// of threads (the reference shares providers across parallel_for workers, sensitivity.cpp:46-52);
// each thread runs on its own stream, results do not depend on the thread count.
#pragma once

#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "qarvd/calibrate.hpp"
#include "qarvd/dual_scale.hpp"
#include "qarvd/engine.hpp"
#include "qarvd/outlier.hpp"
#include "qarvd/quant.hpp"
#include "qarvd/sensitivity.hpp"
#include "qarvd/tensor.hpp"
#include "qarvd/toy_model.hpp"

namespace qarvd {
namespace cuda {

// ---- quant.hpp (bit-identical to the reference's f64 results) ----
// quant.hpp:64 — any granularity / axis / zero point (qarvd_quantize_f64)
IntTensor quantize(const Tensor& x, const QuantParams& p);
// quant.hpp:66
Tensor fake_quant(const Tensor& x, const QuantParams& p);
// quant.hpp:71 (qarvd_minmax_scale_f64)
QuantParams init_scale_minmax(const Tensor& x, int bits, Granularity g, size_t axis = 0);
// quant.hpp:82 — exact order statistics by a device radix select, candidate MSEs in
// double-double (qarvd_percentile_search_f64); same percentile and bit-identical scale
PercentileSearchResult init_scale_percentile_search(const std::vector<Tensor>& samples, int bits);

// ---- dual_scale.hpp (group scales from K5 on the f64 weight) ----
DualScalePlan build_plan(const Tensor& w, const OutlierReport& report, int bits);  // dual_scale.hpp:33
DualScalePlan build_single_scale_plan(const std::string& layer_name, const Tensor& w, int bits);  // :37

// ---- tensor.hpp ----
// tensor.hpp:70 — k-ascending f64 product without FMA (qarvd_matmul_nt_f64), bit-identical
Tensor matmul_nt(const Tensor& a, const Tensor& b);

// ---- engine.hpp ----
// engine.hpp:43 — codes bit-identical to qarvd::quantize
IntTensor kernel_a_quantize_activation(const Tensor& x, const QuantParams& p);
// engine.hpp:48 — int8 tensor-core GEMM (two int32 TMEM accumulators, K2) with the reference's
// f64 epilogue and zero-point correction: bit-identical
Tensor kernel_b_gemm_dequant(const IntTensor& xq, const QuantizedLayer& layer);
// engine.hpp:51 (device gather)
Tensor permute_activations(const Tensor& x, const DualScalePlan& plan);
// engine.hpp:60 — int_kernels: K1 + K2; fakequant_sim and preserved layers: exact f64 products
Tensor quantized_layer_forward(const QuantizedLayer& layer, const Tensor& x, Engine engine);

// ---- outlier.hpp ----
// outlier.hpp:59-61 — bit-identical report (norms, median, MAD, threshold, index sets)
OutlierReport analyze_layer(const std::string& layer_name, const Tensor& w,
                            double tau = kDefaultTau, double alpha_min = kDefaultAlphaMin,
                            size_t align = kDefaultAlign);

// ---- calibrate.hpp ----
// calibrate.hpp:80-82 — Eq. 5 with the deployable (hard-rounded) weights: hard codes, the
// activation fake-quant and both f64 products on the device, bit-identical
double weighted_loss(const std::vector<const CalibSample*>& batch, const LearnableQuantState& state,
                     const std::vector<double>& chunk_weights);
// calibrate.hpp:112-116 — AdaRound calibration of one layer on the GPU (K7, f64): the same
// sampler, formulas, correctly rounded exp/log and Adam schedule as the reference
LayerCalibResult calibrate_layer(const Tensor& w, const DualScalePlan& plan, const QuantParams& act_init,
                                 const std::vector<const CalibSample*>& samples,
                                 const std::vector<double>& chunk_weights, const CalibConfig& cfg);
// calibrate.hpp:45-47 — the full-precision rollouts' linears on the device (CudaFpProvider)
std::vector<CalibSample> collect_calibration(const ToyModel& model, const std::vector<uint64_t>& prompt_seeds,
                                             const std::vector<std::string>& capture_layers);
// calibrate.hpp:137-139 — the whole-model pipeline, every per-layer step on the GPU:
// captures (collect_calibration above), K3, build_plan, the percentile activation init, K7 and the
// pre-permuted codes; the reference's slot-indexed parallel_for over layers, one stream per worker
ModelCalibResult calibrate_model(const ToyModel& model, const std::vector<double>& chunk_weights,
                                 const ModelCalibOptions& opts);

// Device-resident copy of one QuantizedLayer (codes padded into the kernel layout).
class DeviceLayer;

// LinearProvider (toy_model.hpp:77-81) serving a QuantizedModel from the GPU (the reference's
// QuantizedProvider, engine.cpp:146-171).  Layers are uploaded once; forward() is re-entrant.
class CudaQuantizedProvider : public LinearProvider {
 public:
  explicit CudaQuantizedProvider(const QuantizedModel& qm, Engine engine = Engine::int_kernels);
  ~CudaQuantizedProvider() override;
  Tensor forward(const std::string& layer, const Tensor& x) const override;

 private:
  const QuantizedModel& qm_;
  Engine engine_;
  std::map<std::string, std::shared_ptr<DeviceLayer>> layers_;
  std::map<std::string, std::shared_ptr<double>> fp_;  // preserved / fakequant_sim f64 weights
};

// Per-device copies of a provider's f64 weights (created on a device's first use), so one
// provider serves workers on any GPU.
class DeviceWeights {
 public:
  const double* get(const std::string& name, const std::function<std::shared_ptr<double>(int)>& make) const;

 private:
  mutable std::mutex mu_;
  mutable std::map<int, std::map<std::string, std::shared_ptr<double>>> by_device_;
};

// FpProvider (toy_model.hpp:84-91): X W^T with the exact f64 device product.
class CudaFpProvider : public LinearProvider {
 public:
  explicit CudaFpProvider(const ToyModel& model);
  Tensor forward(const std::string& layer, const Tensor& x) const override;

 private:
  const double* weight_on_device(const std::string& layer) const;
  const ToyModel& model_;
  DeviceWeights weights_;
};

// MinMaxFakeQuantProvider (toy_model.cpp:306-325) on the device: cached fake-quantized weights
// (per-row minmax), live per-tensor minmax activations, exact f64 product; bit-identical.
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
  const double* fq_on_device(const std::string& layer) const;
  CudaFpProvider fp_;
  std::map<std::string, std::shared_ptr<double>> fq_home_;  // computed on the constructing device
  DeviceWeights fq_;
};

// profile_sensitivity (sensitivity.cpp:29-66): the reference's slot-indexed parallel_for over
// seeds and (seed, chunk) probes, linears served by CudaFpProvider / CudaMinMaxFakeQuantProvider,
// the tasks spread round-robin over the visible GPUs (QARVD_SENSITIVITY_GPUS caps the count);
// results are identical for any GPU or thread count.
int sensitivity_devices();
SensitivityProfile profile_sensitivity(const ToyModel& model, BitwidthScheme scheme,
                                       const std::vector<uint64_t>& seeds);

// run_quantized (engine.cpp:175-178) and rollout (toy_model.hpp:147-148) with the CUDA providers.
Rollout run_quantized(const QuantizedModel& qm, uint64_t prompt_seed, Engine engine = Engine::int_kernels);
Rollout rollout(const ToyModel& model, uint64_t prompt_seed, const QuantMode& mode,
                const std::vector<std::string>& capture_layers = {});

}  // namespace cuda
}  // namespace qarvd
