// qarvd_cuda.cpp — see qarvd_cuda.hpp.  Host staging + status mapping only.
#include "qarvd_cuda.hpp"

#include <cuda_runtime.h>

#include <cstring>
#include <stdexcept>

#include "../../include/qarvd_b200.h"
#include "qarvd/bytes.hpp"

namespace qarvd {
namespace cuda {

namespace {

[[noreturn]] void throw_status(int st, const std::string& what) {
  const std::string msg = what.empty() ? std::string(qarvd_last_error()) : what;
  switch (st) {
    case QARVD_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case QARVD_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    case QARVD_ERR_LOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

void check(int st) {
  if (st != QARVD_OK) throw_status(st, "");
}

void check_cuda(cudaError_t e) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
}

// RAII device buffer
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  explicit DevBuf(size_t n) : bytes(n) { check_cuda(cudaMalloc(&p, n ? n : 1)); }
  DevBuf(const void* host, size_t n) : DevBuf(n) {
    if (n) check_cuda(cudaMemcpy(p, host, n, cudaMemcpyHostToDevice));
  }
  ~DevBuf() { cudaFree(p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

size_t round_up(size_t v, size_t m) { return (v + m - 1) / m * m; }

// Kernel layout of a plan: [outliers | pad to 32 | normals | pad to 32] (qarvd_b200.h)
struct Layout {
  std::vector<int32_t> gather;  // source column per padded position, -1 = pad
  std::vector<int32_t> pos;     // padded position of permuted column c (reference order)
  size_t k_outlier = 0, k_pad = 0;
};

Layout make_layout(const DualScalePlan& plan, size_t d_in) {
  Layout L;
  const size_t n_o = plan.enabled ? plan.outlier_count() : 0;
  L.k_outlier = round_up(n_o, 32);
  L.k_pad = L.k_outlier + round_up(d_in - n_o, 32);
  L.gather.assign(L.k_pad, -1);
  L.pos.resize(d_in);
  for (size_t c = 0; c < d_in; ++c) {
    const size_t dst = c < n_o ? c : L.k_outlier + (c - n_o);
    L.gather[dst] = plan.enabled ? static_cast<int32_t>(plan.permutation[c]) : static_cast<int32_t>(c);
    L.pos[c] = static_cast<int32_t>(dst);
  }
  return L;
}

}  // namespace

class DeviceLayer {
 public:
  explicit DeviceLayer(const QuantizedLayer& l)
      : name(l.name), n(l.out_dim), k(l.in_dim), layout(make_layout(l.plan, l.in_dim)) {
    if (l.preserved) throw std::invalid_argument("kernel_b: layer is preserved, no integer path: " + l.name);
    if (l.wq.shape.size() != 2 || l.wq.shape[0] != n || l.wq.shape[1] != k)
      throw std::invalid_argument("kernel_b: weight shape mismatch for " + l.name);
    std::vector<int8_t> wq(n * layout.k_pad, 0);
    for (size_t r = 0; r < n; ++r)
      for (size_t c = 0; c < k; ++c)
        wq[r * layout.k_pad + layout.pos[c]] = static_cast<int8_t>(l.wq.data[r * k + c]);
    // f64 group scales exactly as the reference holds them in memory (the f64 epilogue
    // entry point reproduces kernel_b_gemm_dequant bit for bit)
    std::vector<double> so(n), sn(n);
    for (size_t r = 0; r < n; ++r) {
      sn[r] = l.plan.params_normal.scale[r];
      so[r] = l.plan.enabled ? l.plan.params_outlier.scale[r] : l.plan.params_normal.scale[r];
    }
    wq_dev = std::make_unique<DevBuf>(wq.data(), wq.size());
    so_dev = std::make_unique<DevBuf>(so.data(), so.size() * 8);
    sn_dev = std::make_unique<DevBuf>(sn.data(), sn.size() * 8);
    gather_dev = std::make_unique<DevBuf>(layout.gather.data(), layout.gather.size() * 4);
  }
  std::string name;
  size_t n, k;
  Layout layout;
  std::unique_ptr<DevBuf> wq_dev, so_dev, sn_dev, gather_dev;
};

namespace {

// K1 on a host f64 tensor in the layer padded layout; returns device codes + f64 row scales.
void quantize_to_device(const Tensor& x, const Layout& L, const DevBuf& gather_dev,
                        const QuantParams& p, DevBuf& xq, DevBuf& sx, size_t m) {
  if (p.per_channel() || p.zero_point[0] != 0 || !p.symmetric)
    throw std::invalid_argument("quantize: the CUDA engine implements symmetric per-tensor activations");
  p.validate(x.shape());
  DevBuf xd(x.data(), x.size() * sizeof(double));
  DevBuf err(sizeof(int64_t));
  check(qarvd_quantize_act(xd.p, QARVD_F64, static_cast<int64_t>(m), static_cast<int64_t>(x.cols()),
                           static_cast<int64_t>(x.cols()), gather_dev.as<int32_t>(),
                           static_cast<int64_t>(L.k_pad), QARVD_ACT_PER_TENSOR, p.scale[0], p.bits,
                           xq.as<int8_t>(), static_cast<int64_t>(L.k_pad), nullptr, sx.as<double>(),
                           err.as<int64_t>(), nullptr));
  int64_t bad = 0;
  check_cuda(cudaMemcpy(&bad, err.p, sizeof(bad), cudaMemcpyDeviceToHost));
  if (bad != INT64_MAX) {
    // report the first non-finite in the reference's (unpadded, permuted) flat index
    const int64_t row = bad / static_cast<int64_t>(L.k_pad), pc = bad % static_cast<int64_t>(L.k_pad);
    int64_t c = 0;
    for (size_t i = 0; i < L.pos.size(); ++i)
      if (L.pos[i] == pc) c = static_cast<int64_t>(i);
    throw std::invalid_argument("quantize: non-finite input at flat index " +
                                std::to_string(row * static_cast<int64_t>(x.cols()) + c));
  }
}

// sx: device f64 [m] activation scale per row
Tensor gemm_to_host(const DeviceLayer& L, const DevBuf& xq, const DevBuf& sx, size_t m) {
  DevBuf y(m * L.n * sizeof(double));
  check(qarvd_dual_gemm_f64(xq.as<int8_t>(), static_cast<int64_t>(L.layout.k_pad),
                            L.wq_dev->as<int8_t>(), static_cast<int64_t>(L.layout.k_pad),
                            static_cast<int64_t>(m), static_cast<int64_t>(L.n),
                            static_cast<int64_t>(L.layout.k_pad),
                            static_cast<int64_t>(L.layout.k_outlier), sx.as<double>(),
                            L.so_dev->as<double>(), L.sn_dev->as<double>(), y.as<double>(),
                            static_cast<int64_t>(L.n), nullptr));
  Tensor out({m, L.n});
  check_cuda(cudaMemcpy(out.data(), y.p, m * L.n * sizeof(double), cudaMemcpyDeviceToHost));
  return out;
}

}  // namespace

IntTensor kernel_a_quantize_activation(const Tensor& x, const QuantParams& p) {
  p.validate(x.shape());
  if (x.rank() != 2) return qarvd::quantize(x, p);  // non-matrix inputs: not a hot path
  const size_t m = x.rows(), k = x.cols();
  if (p.bits > 8) throw std::invalid_argument("quantize: the CUDA engine stores codes as int8");
  const size_t kp = round_up(k, 32);
  std::vector<int32_t> gather(kp, -1);
  for (size_t c = 0; c < k; ++c) gather[c] = static_cast<int32_t>(c);
  DevBuf gd(gather.data(), gather.size() * 4), xd(x.data(), x.size() * sizeof(double));
  DevBuf q(m * kp + 16), err(sizeof(int64_t));
  std::vector<double> scales_in;
  IntTensor out;
  out.shape = x.shape();
  out.bits = p.bits;
  out.data.resize(m * k);
  if (p.per_channel() && p.channel_axis == 0) {
    // per-token (per-row) scales: one K1 launch per distinct scale is wasteful; rows carry
    // their own scale through the static path one row block at a time
    for (size_t i = 0; i < m; ++i) {
      check(qarvd_quantize_act(xd.as<double>() + i * k, QARVD_F64, 1, static_cast<int64_t>(k),
                               static_cast<int64_t>(k), gd.as<int32_t>(), static_cast<int64_t>(kp),
                               QARVD_ACT_PER_TENSOR, p.scale[i], p.bits, q.as<int8_t>() + i * kp,
                               static_cast<int64_t>(kp), nullptr, nullptr, err.as<int64_t>(), nullptr));
    }
  } else if (p.per_channel()) {
    return qarvd::quantize(x, p);  // per-column scales never occur on the activation path
  } else {
    check(qarvd_quantize_act(xd.p, QARVD_F64, static_cast<int64_t>(m), static_cast<int64_t>(k),
                             static_cast<int64_t>(k), gd.as<int32_t>(), static_cast<int64_t>(kp),
                             QARVD_ACT_PER_TENSOR, p.scale[0], p.bits, q.as<int8_t>(),
                             static_cast<int64_t>(kp), nullptr, nullptr, err.as<int64_t>(), nullptr));
  }
  int64_t bad = 0;
  check_cuda(cudaMemcpy(&bad, err.p, sizeof(bad), cudaMemcpyDeviceToHost));
  if (bad != INT64_MAX) {
    const int64_t row = bad / static_cast<int64_t>(kp), c = bad % static_cast<int64_t>(kp);
    throw std::invalid_argument("quantize: non-finite input at flat index " +
                                std::to_string(row * static_cast<int64_t>(k) + c));
  }
  std::vector<int8_t> h(m * kp);
  check_cuda(cudaMemcpy(h.data(), q.p, h.size(), cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < m; ++i)
    for (size_t c = 0; c < k; ++c) out.data[i * k + c] = h[i * kp + c];
  return out;
}

Tensor permute_activations(const Tensor& x, const DualScalePlan& plan) {
  return qarvd::permute_activations(x, plan);  // a gather; fused into K1 on the device path
}

Tensor kernel_b_gemm_dequant(const IntTensor& xq, const QuantizedLayer& layer) {
  if (layer.preserved)
    throw std::invalid_argument("kernel_b: layer is preserved, no integer path: " + layer.name);
  if (xq.shape.size() != 2 || xq.shape[1] != layer.in_dim)
    throw std::invalid_argument("kernel_b: activation shape does not match layer " + layer.name);
  if (layer.act.zero_point[0] != 0)
    throw std::invalid_argument("kernel_b: asymmetric activations are not supported by the CUDA engine");
  const DeviceLayer L(layer);
  const size_t m = xq.shape[0];
  std::vector<int8_t> h(m * L.layout.k_pad, 0);
  for (size_t i = 0; i < m; ++i)
    for (size_t c = 0; c < L.k; ++c)
      h[i * L.layout.k_pad + L.layout.pos[c]] = static_cast<int8_t>(xq.data[i * L.k + c]);
  DevBuf xd(h.data(), h.size());
  std::vector<double> sx(m, layer.act.scale[0]);
  DevBuf sd(sx.data(), sx.size() * 8);
  return gemm_to_host(L, xd, sd, m);
}

Tensor quantized_layer_forward(const QuantizedLayer& layer, const Tensor& x, Engine engine) {
  if (layer.preserved || engine == Engine::fakequant_sim)
    return qarvd::quantized_layer_forward(layer, x, engine);  // f64 reference paths
  const DeviceLayer L(layer);
  const size_t m = x.rows();
  DevBuf xq(m * L.layout.k_pad + 16), sx(m * 8);
  quantize_to_device(x, L.layout, *L.gather_dev, layer.act, xq, sx, m);
  return gemm_to_host(L, xq, sx, m);
}

OutlierReport analyze_layer(const std::string& layer_name, const Tensor& w, double tau,
                            double alpha_min, size_t align) {
  if (w.rank() != 2) throw std::invalid_argument("channel_l2_norms: input must be 2-D");
  const size_t n = w.rows(), k = w.cols();
  DevBuf wd(w.data(), w.size() * sizeof(double)), norms(k * 8), stats(24), counts(8),
      raw(k * 4), al(k * 4);
  qarvd_outlier_job job{wd.p, static_cast<int64_t>(n), static_cast<int64_t>(k),
                        static_cast<int64_t>(k), norms.as<double>(), stats.as<double>(),
                        counts.as<int32_t>(), raw.as<int32_t>(), al.as<int32_t>()};
  check(qarvd_analyze_layers(&job, 1, QARVD_F64, tau, alpha_min, static_cast<int64_t>(align), nullptr));
  check_cuda(cudaDeviceSynchronize());
  OutlierReport rep;
  rep.layer_name = layer_name;
  rep.tau = tau;
  rep.alpha_min = alpha_min;
  rep.align = align;
  rep.norms.resize(k);
  double st[3];
  int32_t cnt[2];
  check_cuda(cudaMemcpy(rep.norms.data(), norms.p, k * 8, cudaMemcpyDeviceToHost));
  check_cuda(cudaMemcpy(st, stats.p, 24, cudaMemcpyDeviceToHost));
  check_cuda(cudaMemcpy(cnt, counts.p, 8, cudaMemcpyDeviceToHost));
  std::vector<int32_t> r(k), a(k);
  check_cuda(cudaMemcpy(r.data(), raw.p, k * 4, cudaMemcpyDeviceToHost));
  check_cuda(cudaMemcpy(a.data(), al.p, k * 4, cudaMemcpyDeviceToHost));
  rep.median = st[0];
  rep.mad = st[1];
  rep.threshold = st[2];
  rep.raw_outliers.assign(r.begin(), r.begin() + cnt[0]);
  rep.aligned_outliers.assign(a.begin(), a.begin() + cnt[1]);
  return rep;
}

CudaQuantizedProvider::CudaQuantizedProvider(const QuantizedModel& qm) : qm_(qm) {
  for (const auto& l : qm.layers)
    if (!l.preserved) layers_.emplace(l.name, std::make_shared<DeviceLayer>(l));
}

CudaQuantizedProvider::~CudaQuantizedProvider() = default;

Tensor CudaQuantizedProvider::forward(const std::string& layer, const Tensor& x) const {
  const QuantizedLayer& l = qm_.layer(layer);  // std::out_of_range as the reference (engine.cpp:29)
  if (l.preserved) return matmul_nt(x, l.fp_weight);
  const DeviceLayer& L = *layers_.at(layer);
  const size_t m = x.rows();
  DevBuf xq(m * L.layout.k_pad + 16), sx(m * 8);
  quantize_to_device(x, L.layout, *L.gather_dev, l.act, xq, sx, m);
  return gemm_to_host(L, xq, sx, m);
}

namespace {
// bf16 round-to-nearest-even of an f64 value (through f32, as bytes.hpp:40-45 for finite values)
uint16_t bf16_rne(double v) {
  const float f = static_cast<float>(v);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}
double bf16_value(uint16_t h) {
  const uint32_t u = static_cast<uint32_t>(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
// rows of [a_hi a_hi a_lo] (x side) or [a_hi a_lo a_hi] (w side), 3k bf16 per row
std::vector<uint16_t> split3(const double* a, size_t rows, size_t k, bool x_side) {
  std::vector<uint16_t> out(rows * 3 * k);
  for (size_t r = 0; r < rows; ++r)
    for (size_t c = 0; c < k; ++c) {
      const double v = a[r * k + c];
      const uint16_t hi = bf16_rne(v);
      const uint16_t lo = bf16_rne(v - bf16_value(hi));
      uint16_t* o = out.data() + r * 3 * k;
      o[c] = hi;
      o[k + c] = x_side ? hi : lo;
      o[2 * k + c] = x_side ? lo : hi;
    }
  return out;
}
}  // namespace

double weighted_loss(const std::vector<const CalibSample*>& batch, const LearnableQuantState& state,
                     const std::vector<double>& chunk_weights) {
  if (batch.empty()) throw std::invalid_argument("weighted loss: empty batch");
  const size_t n = state.weight.rows(), k = state.weight.cols();
  std::vector<int64_t> rows{0}, chunks;
  for (const CalibSample* s : batch) {
    if (s->x.cols() != k) throw std::invalid_argument("weighted loss: sample width does not match the weight");
    rows.push_back(rows.back() + static_cast<int64_t>(s->x.rows()));
    chunks.push_back(static_cast<int64_t>(s->chunk));
  }
  const size_t m = static_cast<size_t>(rows.back());
  // stacked samples (f64, for K1) and the split bf16 operands of the target
  std::vector<double> x64(m * k);
  size_t off = 0;
  for (const CalibSample* s : batch) {
    std::memcpy(x64.data() + off, s->x.data(), s->x.size() * sizeof(double));
    off += s->x.size();
  }
  const std::vector<uint16_t> xs = split3(x64.data(), m, k, true);
  const std::vector<uint16_t> ws = split3(state.weight.data(), n, k, false);
  // deployable state: hard codes in the kernel layout, learned group scales (f32), act scale
  const Layout L = make_layout(state.plan, k);
  const IntTensor hc = state.hard_codes();
  std::vector<int8_t> wq(n * L.k_pad, 0);
  std::vector<float> so(n), sn(n);
  for (size_t r = 0; r < n; ++r) {
    for (size_t c = 0; c < k; ++c) {
      const size_t pc = state.plan.enabled ? static_cast<size_t>(state.plan.permutation[c]) : c;
      wq[r * L.k_pad + L.pos[c]] = static_cast<int8_t>(hc.data[r * k + pc]);
    }
    sn[r] = static_cast<float>(state.weight_scale(r, false));
    so[r] = static_cast<float>(state.plan.enabled ? state.weight_scale(r, true) : state.weight_scale(r, false));
  }
  const QuantParams act = state.act_params();
  DevBuf x_dev(xs.data(), xs.size() * 2), w_dev(ws.data(), ws.size() * 2);
  DevBuf x64_dev(x64.data(), x64.size() * sizeof(double));
  DevBuf wq_dev(wq.data(), wq.size()), so_dev(so.data(), n * 4), sn_dev(sn.data(), n * 4);
  DevBuf gather_dev(L.gather.data(), L.gather.size() * 4);
  DevBuf xq_dev(m * L.k_pad), sx_dev(m * 4), err_dev(sizeof(int64_t));
  check(qarvd_quantize_act(x64_dev.p, QARVD_F64, static_cast<int64_t>(m), static_cast<int64_t>(k),
                           static_cast<int64_t>(k), gather_dev.as<int32_t>(), static_cast<int64_t>(L.k_pad),
                           QARVD_ACT_PER_TENSOR, act.scale[0], act.bits, xq_dev.as<int8_t>(),
                           static_cast<int64_t>(L.k_pad), sx_dev.as<float>(), nullptr, err_dev.as<int64_t>(),
                           nullptr));
  int64_t bad = 0;
  check_cuda(cudaMemcpy(&bad, err_dev.p, sizeof(bad), cudaMemcpyDeviceToHost));
  if (bad != INT64_MAX) throw std::invalid_argument("quantize: non-finite input");
  const int64_t wsb = qarvd_weighted_loss_workspace(static_cast<int64_t>(m), static_cast<int64_t>(n),
                                                    static_cast<int64_t>(batch.size()));
  DevBuf work(static_cast<size_t>(wsb)), err(batch.size() * 8), loss(8);
  check(qarvd_weighted_loss(x_dev.as<uint16_t>(), static_cast<int64_t>(3 * k), w_dev.as<uint16_t>(),
                            static_cast<int64_t>(3 * k), xq_dev.as<int8_t>(), static_cast<int64_t>(L.k_pad),
                            wq_dev.as<int8_t>(), static_cast<int64_t>(L.k_pad), static_cast<int64_t>(m),
                            static_cast<int64_t>(n), static_cast<int64_t>(3 * k),
                            static_cast<int64_t>(L.k_pad), static_cast<int64_t>(L.k_outlier),
                            sx_dev.as<float>(), so_dev.as<float>(), sn_dev.as<float>(), rows.data(),
                            chunks.data(), static_cast<int64_t>(batch.size()), chunk_weights.data(),
                            static_cast<int64_t>(chunk_weights.size()), err.as<double>(), loss.as<double>(),
                            work.p, wsb, nullptr));
  double out = 0.0;
  check_cuda(cudaMemcpy(&out, loss.p, 8, cudaMemcpyDeviceToHost));
  return out;
}

CudaMinMaxFakeQuantProvider::CudaMinMaxFakeQuantProvider(const ToyModel& model, BitwidthScheme scheme,
                                                         std::vector<std::string> keep_list)
    : model_(model), scheme_(scheme), keep_list_(std::move(keep_list)) {
  if (scheme_.is_lossless()) return;
  for (const auto& spec : model.registry()) {
    if (matches_keep_list(spec.name, keep_list_)) continue;
    const Tensor& w = model.weight(spec.name);
    const size_t n = w.rows(), k = w.cols();
    // K5 on the f64 weight with the single-scale (identity) plan: per-row absmax / qmax scales
    // (init_scale_minmax per_channel axis 0, quant.cpp:170-182) and nearest codes
    DualScalePlan plan = build_single_scale_plan(spec.name, w, scheme_.weight_bits);
    const Layout L = make_layout(plan, k);
    DevBuf w_d(w.data(), w.size() * 8), g_d(L.gather.data(), L.gather.size() * 4);
    DevBuf wq_d(n * L.k_pad), so_d(n * 8), sn_d(n * 8), err(8);
    check(qarvd_prepare_weights(w_d.p, QARVD_F64, static_cast<int64_t>(n), static_cast<int64_t>(k),
                                static_cast<int64_t>(k), g_d.as<int32_t>(), static_cast<int64_t>(L.k_pad), 0,
                                scheme_.weight_bits, wq_d.as<int8_t>(), static_cast<int64_t>(L.k_pad),
                                so_d.as<double>(), sn_d.as<double>(), nullptr, nullptr, err.as<int64_t>(), nullptr));
    std::vector<int8_t> wq(n * L.k_pad);
    check_cuda(cudaMemcpy(wq.data(), wq_d.p, wq.size(), cudaMemcpyDeviceToHost));
    check_cuda(cudaMemcpy(plan.params_normal.scale.data(), sn_d.p, n * 8, cudaMemcpyDeviceToHost));
    plan.params_outlier = plan.params_normal;
    QuantizedLayer ql;
    ql.name = spec.name;
    ql.out_dim = n;
    ql.in_dim = k;
    ql.preserved = false;
    ql.plan = plan;
    ql.wq.shape = {n, k};
    ql.wq.bits = scheme_.weight_bits;
    ql.wq.data.resize(n * k);
    for (size_t r = 0; r < n; ++r)
      for (size_t c = 0; c < k; ++c) ql.wq.data[r * k + c] = wq[r * L.k_pad + L.pos[c]];
    layers_.emplace(spec.name, std::make_shared<DeviceLayer>(ql));
  }
}

CudaMinMaxFakeQuantProvider::~CudaMinMaxFakeQuantProvider() = default;

Tensor CudaMinMaxFakeQuantProvider::forward(const std::string& layer, const Tensor& x) const {
  if (scheme_.is_lossless() || matches_keep_list(layer, keep_list_)) return matmul_nt(x, model_.weight(layer));
  const DeviceLayer& L = *layers_.at(layer);
  const size_t m = x.rows();
  // per-tensor minmax scale = max over rows of K1's exact per-row scales fl(absmax_r / qmax)
  // (rounding is monotone, so it equals fl(absmax / qmax), quant.cpp:165-168)
  DevBuf xd(x.data(), x.size() * 8), xq(m * L.layout.k_pad + 16), s_rows(m * 8), err(8);
  check(qarvd_quantize_act(xd.p, QARVD_F64, static_cast<int64_t>(m), static_cast<int64_t>(x.cols()),
                           static_cast<int64_t>(x.cols()), L.gather_dev->as<int32_t>(),
                           static_cast<int64_t>(L.layout.k_pad), QARVD_ACT_PER_TOKEN, 0.0,
                           scheme_.activation_bits, xq.as<int8_t>(), static_cast<int64_t>(L.layout.k_pad),
                           nullptr, s_rows.as<double>(), err.as<int64_t>(), nullptr));
  std::vector<double> sr(m);
  check_cuda(cudaMemcpy(sr.data(), s_rows.p, m * 8, cudaMemcpyDeviceToHost));
  double s = 0.0;
  for (double v : sr) s = std::max(s, v);
  QuantParams act = QuantParams::per_tensor_symmetric(scheme_.activation_bits, s);
  DevBuf sx(m * 8);
  quantize_to_device(x, L.layout, *L.gather_dev, act, xq, sx, m);
  return gemm_to_host(L, xq, sx, m);
}

SensitivityProfile profile_sensitivity(const ToyModel& model, BitwidthScheme scheme,
                                       const std::vector<uint64_t>& seeds) {
  if (seeds.empty()) throw std::invalid_argument("profile_sensitivity: need at least one seed");
  const size_t n_chunks = model.config().chunks;
  const FpProvider fp(model);
  const CudaMinMaxFakeQuantProvider quant(model, scheme);
  std::vector<Rollout> references(seeds.size());
  for (size_t s = 0; s < seeds.size(); ++s)
    references[s] = run_rollout(model.config(), fp, nullptr, QuantTarget::none, 0, seeds[s]);
  std::vector<std::vector<double>> per_seed(seeds.size(), std::vector<double>(n_chunks, 0.0));
  for (size_t s = 0; s < seeds.size(); ++s)
    for (size_t i = 0; i < n_chunks; ++i) {
      const Rollout probe = run_rollout(model.config(), fp, &quant, QuantTarget::only_chunk, i + 1, seeds[s]);
      per_seed[s][i] = latent_mse(references[s], probe);
    }
  SensitivityProfile profile;
  profile.scheme = scheme;
  profile.seeds = seeds;
  profile.per_seed = std::move(per_seed);
  profile.alpha_raw.assign(n_chunks, 0.0);
  for (size_t i = 0; i < n_chunks; ++i) {
    double acc = 0.0;
    for (size_t s = 0; s < seeds.size(); ++s) acc += profile.per_seed[s][i];
    profile.alpha_raw[i] = acc / static_cast<double>(seeds.size());
  }
  profile.alpha_normalized = normalize_alpha(profile.alpha_raw);
  return profile;
}

LayerCalibResult calibrate_layer(const Tensor& w, const DualScalePlan& plan, const QuantParams& act_init,
                                 const std::vector<const CalibSample*>& samples,
                                 const std::vector<double>& chunk_weights, const CalibConfig& cfg) {
  cfg.validate();
  if (samples.empty()) throw std::invalid_argument("calibrate_layer: no calibration samples");
  if (act_init.per_channel() || act_init.zero_point[0] != 0)
    throw std::invalid_argument("calibrate_layer: the activation init must be per-tensor symmetric");
  const size_t n = w.rows(), k = w.cols();
  std::vector<uint8_t> mask(k, 0);
  if (plan.enabled)
    for (size_t c : plan.outlier_indices) mask[c] = 1;
  std::vector<int64_t> rows{0}, chunks;
  for (const CalibSample* s : samples) {
    if (s->x.cols() != k) throw std::invalid_argument("calibrate_layer: sample width does not match the weight");
    rows.push_back(rows.back() + static_cast<int64_t>(s->x.rows()));
    chunks.push_back(static_cast<int64_t>(s->chunk));
  }
  std::vector<double> x(static_cast<size_t>(rows.back()) * k);
  size_t off = 0;
  for (const CalibSample* s : samples) {
    std::memcpy(x.data() + off, s->x.data(), s->x.size() * sizeof(double));
    off += s->x.size();
  }
  const std::vector<double>& sn = plan.params_normal.scale;
  const std::vector<double>& so = plan.enabled ? plan.params_outlier.scale : plan.params_normal.scale;
  DevBuf w_d(w.data(), w.size() * 8), mask_d(mask.data(), k), sn_d(sn.data(), n * 8), so_d(so.data(), n * 8);
  DevBuf x_d(x.data(), x.size() * 8), codes_d(n * k), sn_out(n * 8), so_out(n * 8), sc_out(3 * 8),
      tr_out(static_cast<size_t>(cfg.iterations > 0 ? cfg.iterations : 1) * 8);
  qarvd_calib_config c{};
  c.iterations = cfg.iterations;
  c.batch_size = cfg.batch_size;
  c.lr_round = cfg.lr_round;
  c.lr_scale = cfg.lr_scale;
  c.seed = cfg.seed;
  c.train_activation_scale = cfg.train_activation_scale ? 1 : 0;
  c.zeta = cfg.zeta;
  c.gamma_lo = cfg.gamma_lo;
  c.reg_lambda = cfg.reg_lambda;
  c.beta_start = cfg.beta_start;
  c.beta_end = cfg.beta_end;
  c.warmup_frac = cfg.warmup_frac;
  check(qarvd_calibrate_layer(w_d.as<double>(), static_cast<int64_t>(n), static_cast<int64_t>(k),
                              mask_d.as<uint8_t>(), plan.enabled ? 1 : 0, sn_d.as<double>(), so_d.as<double>(),
                              act_init.scale[0], act_init.bits, plan.params_normal.bits, x_d.as<double>(),
                              rows.data(), chunks.data(), static_cast<int64_t>(samples.size()),
                              chunk_weights.data(), static_cast<int64_t>(chunk_weights.size()), &c,
                              plan.layer_name.c_str(), codes_d.as<int8_t>(), sn_out.as<double>(),
                              so_out.as<double>(), sc_out.as<double>(), tr_out.as<double>(), nullptr));
  std::vector<int8_t> codes(n * k);
  std::vector<double> lsn(n), lso(n), sc(3), tr(static_cast<size_t>(cfg.iterations > 0 ? cfg.iterations : 0));
  check_cuda(cudaMemcpy(codes.data(), codes_d.p, n * k, cudaMemcpyDeviceToHost));
  check_cuda(cudaMemcpy(lsn.data(), sn_out.p, n * 8, cudaMemcpyDeviceToHost));
  check_cuda(cudaMemcpy(lso.data(), so_out.p, n * 8, cudaMemcpyDeviceToHost));
  check_cuda(cudaMemcpy(sc.data(), sc_out.p, 3 * 8, cudaMemcpyDeviceToHost));
  if (!tr.empty()) check_cuda(cudaMemcpy(tr.data(), tr_out.p, tr.size() * 8, cudaMemcpyDeviceToHost));
  LayerCalibResult r;
  r.layer = plan.layer_name;
  // plan_with_learned_scales (calibrate.cpp:185-199)
  r.plan = plan;
  r.plan.params_normal = QuantParams::per_channel_symmetric(plan.params_normal.bits, 0, lsn);
  r.plan.params_outlier = QuantParams::per_channel_symmetric(plan.params_outlier.bits, 0, lso);
  r.codes.shape = {n, k};
  r.codes.bits = plan.params_normal.bits;
  r.codes.data.assign(codes.begin(), codes.end());
  r.act = QuantParams::per_tensor_symmetric(act_init.bits, sc[0]);
  r.initial_loss = sc[1];
  r.final_loss = sc[2];
  r.trace = tr;
  return r;
}

ModelCalibResult calibrate_model(const ToyModel& model, const std::vector<double>& chunk_weights,
                                 const ModelCalibOptions& opts) {
  opts.base.validate();
  if (chunk_weights.size() != model.config().chunks)
    throw std::invalid_argument("calibrate_model: weight vector length must equal chunk count");
  std::vector<std::string> quant_layers;
  for (const auto& spec : model.registry())
    if (!matches_keep_list(spec.name, opts.keep_list)) quant_layers.push_back(spec.name);
  const std::vector<CalibSample> samples = collect_calibration(model, opts.prompt_seeds, quant_layers);
  ModelCalibResult out;
  out.qmodel.cfg = model.config();
  out.qmodel.scheme = opts.base.scheme;
  out.qmodel.keep_list = opts.keep_list;
  out.qmodel.layers.resize(model.registry().size());
  for (size_t li = 0; li < model.registry().size(); ++li) {
    const LayerSpec& spec = model.registry()[li];
    if (matches_keep_list(spec.name, opts.keep_list)) {  // preserved: bf16 passthrough
      QuantizedLayer l;
      l.name = spec.name;
      l.out_dim = spec.out_dim;
      l.in_dim = spec.in_dim;
      l.preserved = true;
      Tensor fp = model.weight(spec.name);
      for (size_t i = 0; i < fp.size(); ++i) fp[i] = static_cast<double>(bf16_to_float(float_to_bf16(static_cast<float>(fp[i]))));
      l.fp_weight = fp;
      out.qmodel.layers[li] = std::move(l);
      continue;
    }
    const Tensor& w = model.weight(spec.name);
    DualScalePlan plan;
    if (opts.dual_scale) {
      const OutlierReport report = qarvd::cuda::analyze_layer(spec.name, w, opts.tau, opts.alpha_min, opts.align);
      plan = build_plan(w, report, opts.base.scheme.weight_bits);
    } else {
      plan = build_single_scale_plan(spec.name, w, opts.base.scheme.weight_bits);
    }
    std::vector<const CalibSample*> ls;
    std::vector<Tensor> acts;
    for (const auto& smp : samples)
      if (smp.layer == spec.name) {
        ls.push_back(&smp);
        acts.push_back(smp.x);
      }
    // percentile activation init of the f64 captures (quant.cpp:190-226; the GPU search, K4,
    // works on bf16 bit-pattern histograms)
    const PercentileSearchResult act_init = init_scale_percentile_search(acts, opts.base.scheme.activation_bits);
    LayerCalibResult res = qarvd::cuda::calibrate_layer(w, plan, act_init.params, ls, chunk_weights, opts.base);
    QuantizedLayer l;
    l.name = spec.name;
    l.out_dim = spec.out_dim;
    l.in_dim = spec.in_dim;
    l.preserved = false;
    l.plan = res.plan;
    l.act = res.act;
    l.wq.shape = {spec.out_dim, spec.in_dim};
    l.wq.bits = res.codes.bits;
    l.wq.data.resize(spec.out_dim * spec.in_dim);
    for (size_t r = 0; r < spec.out_dim; ++r)  // pre-permuted [outlier | normal] (calibrate.cpp:474-480)
      for (size_t pos = 0; pos < spec.in_dim; ++pos)
        l.wq.data[r * spec.in_dim + pos] = res.codes.at(r, res.plan.permutation[pos]);
    out.qmodel.layers[li] = std::move(l);
    out.layer_results.push_back(std::move(res));
  }
  return out;
}

Rollout run_quantized(const QuantizedModel& qm, uint64_t prompt_seed) {
  const CudaQuantizedProvider provider(qm);
  return run_rollout(qm.cfg, provider, &provider, QuantTarget::all, 0, prompt_seed);
}

}  // namespace cuda
}  // namespace qarvd
