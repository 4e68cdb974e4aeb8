// qarvd_cuda.cpp — see qarvd_cuda.hpp.  Host staging, per-thread device contexts and status
// mapping only: every arithmetic step runs in libqarvd_b200.so.  The reference library is linked
// for its types, its parameter validation (QuantParams::validate, CalibConfig::validate) and its
// host drivers (run_rollout, parallel_for); none of its compute functions is called from here
// (tests/cpp/test_no_ref_compute.cpp links this file against poisoned copies of them).
#include "qarvd_cuda.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <cstring>
#include <limits>
#include <stdexcept>

#include "../../include/qarvd_b200.h"
#include "qarvd/bytes.hpp"
#include "qarvd/threading.hpp"

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

size_t round_up(size_t v, size_t m) { return (v + m - 1) / m * m; }

// ---- per-thread execution contexts ----------------------------------------------------
// Providers are shared const across the reference's parallel_for workers (sensitivity.cpp:46-52,
// calibrate.cpp:440), so every call runs on its own thread's context: a non-blocking stream and
// grow-only device workspaces.  Contexts live in a process-wide pool; a thread takes one on its
// first call and returns it when it exits, so the short-lived parallel_for workers reuse the
// streams and buffers instead of creating and freeing them per call.
struct Context {
  int device = -1;
  cudaStream_t stream = nullptr;
  std::vector<std::pair<void*, size_t>> slots;

  // grow-only workspace `slot` of at least `bytes` (contents undefined)
  template <typename T = void>
  T* ws(size_t slot, size_t bytes) {
    if (slots.size() <= slot) slots.resize(slot + 1, {nullptr, 0});
    auto& s = slots[slot];
    if (s.second < bytes) {
      if (s.first) {
        check_cuda(cudaStreamSynchronize(stream));
        check_cuda(cudaFree(s.first));
        s.first = nullptr;
        s.second = 0;
      }
      const size_t cap = std::max<size_t>(round_up(bytes, 256), 4096);
      check_cuda(cudaMalloc(&s.first, cap));
      s.second = cap;
    }
    return static_cast<T*>(s.first);
  }
  void sync() { check_cuda(cudaStreamSynchronize(stream)); }
};

class ContextPool {
 public:
  Context* acquire(int device) {
    {
      std::lock_guard<std::mutex> lock(mu_);
      for (size_t i = 0; i < free_.size(); ++i)
        if (free_[i]->device == device) {
          Context* c = free_[i];
          free_.erase(free_.begin() + static_cast<std::ptrdiff_t>(i));
          return c;
        }
    }
    auto* c = new Context();
    c->device = device;
    check_cuda(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    return c;
  }
  void release(Context* c) {
    std::lock_guard<std::mutex> lock(mu_);
    free_.push_back(c);
  }

 private:
  std::mutex mu_;
  std::vector<Context*> free_;  // process lifetime: never destroyed (streams outlive threads)
};
ContextPool& pool() {
  static auto* p = new ContextPool();
  return *p;
}
struct ContextHolder {
  Context* c = nullptr;
  ~ContextHolder() {
    if (c) pool().release(c);
  }
};
Context& ctx() {
  thread_local ContextHolder h;
  int dev = 0;
  check_cuda(cudaGetDevice(&dev));
  if (!h.c || h.c->device != dev) {
    if (h.c) pool().release(h.c);
    h.c = pool().acquire(dev);
  }
  return *h.c;
}

// workspace slots (one call never uses a slot twice)
enum Slot : size_t {
  kX, kX2, kXq, kSx, kY, kY2, kW, kW2, kCodes, kScales, kScales2, kIdx, kErr, kMisc, kMisc2, kMisc3,
  kLoss0, kLoss1, kLayerWq, kLayerSo, kLayerSn, kLayerGather,
};

void h2d(Context& c, void* dst, const void* src, size_t bytes) {
  if (bytes) check_cuda(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c.stream));
}
void d2h(Context& c, void* dst, const void* src, size_t bytes) {
  if (bytes) check_cuda(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c.stream));
}
template <typename T>
T* upload(Context& c, size_t slot, const T* host, size_t count) {
  T* d = c.ws<T>(slot, count * sizeof(T));
  h2d(c, d, host, count * sizeof(T));
  return d;
}

// Kernel layout of a plan: [outliers | pad to 32 | normals | pad to 32] (qarvd_b200.h).
struct Layout {
  std::vector<int32_t> gather;  // original column per padded position (x -> xq, K1), -1 = pad
  std::vector<int32_t> pack;    // plan position per padded position (pre-permuted codes), -1 = pad
  std::vector<int32_t> pos;     // padded position of plan position c
  size_t n_outlier = 0, k_outlier = 0, k_pad = 0;
};

Layout make_layout(const DualScalePlan& plan, size_t d_in) {
  Layout L;
  L.n_outlier = plan.enabled ? plan.outlier_count() : 0;
  L.k_outlier = round_up(L.n_outlier, 32);
  L.k_pad = L.k_outlier + round_up(d_in - L.n_outlier, 32);
  L.gather.assign(L.k_pad, -1);
  L.pack.assign(L.k_pad, -1);
  L.pos.resize(d_in);
  for (size_t c = 0; c < d_in; ++c) {
    const size_t dst = c < L.n_outlier ? c : L.k_outlier + (c - L.n_outlier);
    L.gather[dst] = plan.enabled ? static_cast<int32_t>(plan.permutation[c]) : static_cast<int32_t>(c);
    L.pack[dst] = static_cast<int32_t>(c);
    L.pos[c] = static_cast<int32_t>(dst);
  }
  return L;
}

// the reference's flat index of a non-finite element found at padded position `bad`
int64_t unpadded_index(int64_t bad, const Layout& L, size_t k) {
  const int64_t row = bad / static_cast<int64_t>(L.k_pad), pc = bad % static_cast<int64_t>(L.k_pad);
  int64_t c = 0;
  for (size_t i = 0; i < L.pos.size(); ++i)
    if (L.pos[i] == pc) c = static_cast<int64_t>(i);
  return row * static_cast<int64_t>(k) + c;
}

std::string nonfinite_msg(int64_t i) { return "quantize: non-finite input at flat index " + std::to_string(i); }

}  // namespace

// Device-resident copy of one QuantizedLayer: padded int8 codes, f64 group scales, the K1 gather.
// Owned by a provider (uploaded once), or transient: a free function's per-call copy lives in the
// calling thread's grow-only workspace slots, so steady-state calls allocate nothing.
class DeviceLayer {
 public:
  explicit DeviceLayer(const QuantizedLayer& l, bool transient = false)
      : name(l.name), n(l.out_dim), k(l.in_dim), layout(make_layout(l.plan, l.in_dim)), owned(!transient) {
    if (l.preserved) throw std::invalid_argument("kernel_b: layer is preserved, no integer path: " + l.name);
    if (l.wq.shape.size() != 2 || l.wq.shape[0] != n || l.wq.shape[1] != k)
      throw std::invalid_argument("kernel_b: weight shape mismatch for " + l.name);
    if (l.wq.bits > 8) throw std::invalid_argument("kernel_b: the CUDA engine stores codes as int8");
    Context& c = ctx();
    if (owned) {
      check_cuda(cudaMalloc(&wq, n * layout.k_pad));
      check_cuda(cudaMalloc(&so, n * 8));
      check_cuda(cudaMalloc(&sn, n * 8));
      check_cuda(cudaMalloc(&gather, layout.k_pad * 4));
    } else {
      wq = c.ws<int8_t>(kLayerWq, n * layout.k_pad);
      so = c.ws<double>(kLayerSo, n * 8);
      sn = c.ws<double>(kLayerSn, n * 8);
      gather = c.ws<int32_t>(kLayerGather, layout.k_pad * 4);
    }
    const int32_t* codes = upload(c, kCodes, l.wq.data.data(), n * k);
    const int32_t* pack = upload(c, kIdx, layout.pack.data(), layout.k_pad);
    int* bad = c.ws<int>(kErr, sizeof(int));
    check_cuda(cudaMemsetAsync(bad, 0, sizeof(int), c.stream));
    check(qarvd_pack_codes_i8(codes, static_cast<int64_t>(n), static_cast<int64_t>(k), pack,
                              static_cast<int64_t>(layout.k_pad), wq, static_cast<int64_t>(layout.k_pad), bad,
                              c.stream));
    // f64 group scales exactly as the reference holds them in memory (the f64 epilogue
    // reproduces kernel_b_gemm_dequant bit for bit)
    h2d(c, sn, l.plan.params_normal.scale.data(), n * 8);
    h2d(c, so, (l.plan.enabled ? l.plan.params_outlier.scale : l.plan.params_normal.scale).data(), n * 8);
    h2d(c, gather, layout.gather.data(), layout.k_pad * 4);
    int hbad = 0;
    d2h(c, &hbad, bad, sizeof(int));
    c.sync();
    if (hbad) throw std::invalid_argument("kernel_b: the CUDA engine stores codes as int8");
  }
  ~DeviceLayer() {
    if (!owned) return;
    cudaFree(wq);
    cudaFree(so);
    cudaFree(sn);
    cudaFree(gather);
  }
  DeviceLayer(const DeviceLayer&) = delete;
  DeviceLayer& operator=(const DeviceLayer&) = delete;

  std::string name;
  size_t n, k;
  Layout layout;
  int8_t* wq = nullptr;
  double* so = nullptr;
  double* sn = nullptr;
  int32_t* gather = nullptr;
  bool owned;
};

namespace {

// kernel B (K2 tensor-core int32 accumulators + the reference's f64 epilogue, engine.cpp:86-100)
// on device codes xq [m x k_pad] in the layer layout -> host f64 [m x n]
Tensor gemm_to_host(Context& c, const DeviceLayer& L, const QuantParams& act, const int8_t* xq, size_t m) {
  const double s_x = act.scale[0];
  const int32_t z_x = act.zero_point.empty() ? 0 : act.zero_point[0];
  double* sx = c.ws<double>(kSx, m * 8);
  {
    std::vector<double> h(m, s_x);
    h2d(c, sx, h.data(), m * 8);
    c.sync();  // h is a local
  }
  double* y = c.ws<double>(kY, m * L.n * 8);
  check(qarvd_dual_gemm_f64(xq, static_cast<int64_t>(L.layout.k_pad), L.wq, static_cast<int64_t>(L.layout.k_pad),
                            static_cast<int64_t>(m), static_cast<int64_t>(L.n), static_cast<int64_t>(L.layout.k_pad),
                            static_cast<int64_t>(L.layout.k_outlier), sx, L.so, L.sn, y, static_cast<int64_t>(L.n),
                            c.stream));
  if (z_x != 0)
    check(qarvd_zero_point_correct_f64(y, static_cast<int64_t>(L.n), static_cast<int64_t>(m),
                                       static_cast<int64_t>(L.n), L.wq, static_cast<int64_t>(L.layout.k_pad),
                                       static_cast<int64_t>(L.layout.k_pad), static_cast<int64_t>(L.layout.k_outlier),
                                       L.layout.n_outlier > 0 ? 2 : 1, z_x, s_x, L.so, L.sn, c.stream));
  Tensor out({m, L.n});
  d2h(c, out.data(), y, m * L.n * 8);
  c.sync();
  return out;
}

// kernel A on a host activation (original column order) into the layer layout: per-tensor symmetric
// params take K1 (f64 input, exact path, gather fused); any other params (asymmetric zero point) the
// generic exact quantizer followed by the int8 packing
int8_t* quantize_to_layout(Context& c, const DeviceLayer& L, const Tensor& x, const QuantParams& p) {
  if (x.rank() != 2 || x.cols() != L.k)
    throw std::invalid_argument("permute_activations: plan does not match activation width");
  p.validate(x.shape());
  if (p.per_channel()) throw std::invalid_argument("kernel_b: per-tensor activation params expected");
  if (p.bits > 8 || p.q_min < -128 || p.q_max > 127)
    throw std::invalid_argument("quantize: the CUDA engine stores codes as int8");
  const size_t m = x.rows();
  const double* xd = upload(c, kX, x.data(), x.size());
  int8_t* xq = c.ws<int8_t>(kXq, m * L.layout.k_pad + 16);
  int64_t* err = c.ws<int64_t>(kErr, 8);
  int64_t bad = INT64_MAX;
  if (p.symmetric && p.zero_point[0] == 0) {
    check(qarvd_quantize_act(xd, QARVD_F64, static_cast<int64_t>(m), static_cast<int64_t>(L.k),
                             static_cast<int64_t>(L.k), L.gather, static_cast<int64_t>(L.layout.k_pad),
                             QARVD_ACT_PER_TENSOR, p.scale[0], p.bits, xq, static_cast<int64_t>(L.layout.k_pad),
                             nullptr, nullptr, err, c.stream));
    d2h(c, &bad, err, 8);
    c.sync();
    if (bad != INT64_MAX) throw std::invalid_argument(nonfinite_msg(unpadded_index(bad, L.layout, L.k)));
    return xq;
  }
  // quantize(permute(x)) = permute(quantize(x)) for per-tensor params: codes in original order,
  // then packed through the K1 gather (original column per padded position)
  double* sd = upload(c, kScales, p.scale.data(), 1);
  int32_t* zd = upload(c, kMisc, p.zero_point.data(), 1);
  int32_t* codes = c.ws<int32_t>(kCodes, m * L.k * 4);
  check(qarvd_quantize_f64(xd, static_cast<int64_t>(m * L.k), 1, 1, sd, zd, p.q_min, p.q_max, codes, nullptr, err,
                           c.stream));
  int* pbad = c.ws<int>(kMisc2, sizeof(int));
  check_cuda(cudaMemsetAsync(pbad, 0, sizeof(int), c.stream));
  check(qarvd_pack_codes_i8(codes, static_cast<int64_t>(m), static_cast<int64_t>(L.k), L.gather,
                            static_cast<int64_t>(L.layout.k_pad), xq, static_cast<int64_t>(L.layout.k_pad), pbad,
                            c.stream));
  d2h(c, &bad, err, 8);
  c.sync();
  if (bad != INT64_MAX) {
    // the reference quantizes the permuted tensor: report the first bad element in that order
    const size_t k = L.k;
    std::vector<double> row(k);
    const int64_t r = bad / static_cast<int64_t>(k);
    std::memcpy(row.data(), x.data() + r * k, k * 8);
    int64_t first = bad;
    for (size_t cpos = 0; cpos < k; ++cpos) {
      const size_t orig = L.layout.gather[L.layout.pos[cpos]];
      if (!std::isfinite(row[orig])) {
        first = r * static_cast<int64_t>(k) + static_cast<int64_t>(cpos);
        break;
      }
    }
    throw std::invalid_argument(nonfinite_msg(first));
  }
  return xq;
}

// LearnableQuantState on the device (what / codes and act scale); returns device pointers in slots
struct DeviceState {
  double* w = nullptr;       // [n x k]
  double* what = nullptr;    // hard weights [n x k]
  int8_t* codes = nullptr;   // hard codes [n x k] (optional)
  double* act_scale = nullptr;  // [1] exp(log_act_scale)
};
DeviceState upload_state(Context& c, const LearnableQuantState& st, bool want_codes) {
  const size_t n = st.weight.rows(), k = st.weight.cols();
  DeviceState d;
  d.w = upload(c, kW, st.weight.data(), n * k);
  const double* v = upload(c, kW2, st.v.data(), n * k);
  std::vector<uint8_t> mask(k, 0);
  if (st.plan.enabled)
    for (size_t col : st.plan.outlier_indices) mask[col] = 1;
  std::vector<double> log_s(2 * n + 1);
  for (size_t r = 0; r < n; ++r) {
    log_s[r] = st.log_scale_normal[r];
    log_s[n + r] = st.plan.enabled ? st.log_scale_outlier[r] : st.log_scale_normal[r];
  }
  log_s[2 * n] = st.log_act_scale;
  double* ls = upload(c, kScales2, log_s.data(), log_s.size());
  const uint8_t* md = upload(c, kMisc3, mask.data(), k);
  d.what = c.ws<double>(kY2, n * k * 8);
  if (want_codes) d.codes = c.ws<int8_t>(kMisc, n * k);
  check(qarvd_adaround_weights(d.w, v, md, st.plan.enabled ? 1 : 0, ls, static_cast<int64_t>(n),
                               static_cast<int64_t>(k), st.zeta, st.gamma_lo, st.plan.params_normal.bits, 1, d.what,
                               d.codes, c.stream));
  d.act_scale = c.ws<double>(kMisc2, 8);
  check(qarvd_exp_f64(ls + 2 * n, d.act_scale, 1, c.stream));
  c.sync();  // the host vectors above go out of scope
  return d;
}

}  // namespace

// ---- quant.hpp -------------------------------------------------------------------------

IntTensor quantize(const Tensor& x, const QuantParams& p) {
  p.validate(x.shape());
  Context& c = ctx();
  size_t extent = 1, inner = 1;
  if (p.per_channel()) {
    extent = x.shape()[p.channel_axis];
    for (size_t a = p.channel_axis + 1; a < x.shape().size(); ++a) inner *= x.shape()[a];
  }
  IntTensor out;
  out.shape = x.shape();
  out.bits = p.bits;
  out.data.resize(x.size());
  if (x.size() == 0) return out;
  const double* xd = upload(c, kX, x.data(), x.size());
  const double* sd = upload(c, kScales, p.scale.data(), p.scale.size());
  const int32_t* zd = upload(c, kMisc, p.zero_point.data(), p.zero_point.size());
  int32_t* codes = c.ws<int32_t>(kCodes, x.size() * 4);
  int64_t* err = c.ws<int64_t>(kErr, 8);
  check(qarvd_quantize_f64(xd, static_cast<int64_t>(x.size()), static_cast<int64_t>(inner),
                           static_cast<int64_t>(extent), sd, zd, p.q_min, p.q_max, codes, nullptr, err, c.stream));
  int64_t bad = INT64_MAX;
  d2h(c, &bad, err, 8);
  d2h(c, out.data.data(), codes, x.size() * 4);
  c.sync();
  if (bad != INT64_MAX) throw std::invalid_argument(nonfinite_msg(bad));
  return out;
}

Tensor fake_quant(const Tensor& x, const QuantParams& p) {
  p.validate(x.shape());
  Context& c = ctx();
  size_t extent = 1, inner = 1;
  if (p.per_channel()) {
    extent = x.shape()[p.channel_axis];
    for (size_t a = p.channel_axis + 1; a < x.shape().size(); ++a) inner *= x.shape()[a];
  }
  Tensor out(x.shape());
  if (x.size() == 0) return out;
  const double* xd = upload(c, kX, x.data(), x.size());
  const double* sd = upload(c, kScales, p.scale.data(), p.scale.size());
  const int32_t* zd = upload(c, kMisc, p.zero_point.data(), p.zero_point.size());
  double* deq = c.ws<double>(kY, x.size() * 8);
  int64_t* err = c.ws<int64_t>(kErr, 8);
  check(qarvd_quantize_f64(xd, static_cast<int64_t>(x.size()), static_cast<int64_t>(inner),
                           static_cast<int64_t>(extent), sd, zd, p.q_min, p.q_max, nullptr, deq, err, c.stream));
  int64_t bad = INT64_MAX;
  d2h(c, &bad, err, 8);
  d2h(c, out.data(), deq, x.size() * 8);
  c.sync();
  if (bad != INT64_MAX) throw std::invalid_argument(nonfinite_msg(bad));
  return out;
}

QuantParams init_scale_minmax(const Tensor& x, int bits, Granularity g, size_t axis) {
  if (bits < 2 || bits > 30)
    throw std::invalid_argument("bit width out of supported range [2,30]: " + std::to_string(bits));
  size_t extent = 1, inner = 1;
  if (g == Granularity::per_channel) {
    if (axis >= x.shape().size()) throw std::invalid_argument("init_scale_minmax: axis out of range");
    extent = x.shape()[axis];
    for (size_t a = axis + 1; a < x.shape().size(); ++a) inner *= x.shape()[a];
  }
  Context& c = ctx();
  const double* xd = upload(c, kX, x.data(), x.size());
  double* sd = c.ws<double>(kScales, extent * 8);
  check(qarvd_minmax_scale_f64(xd, static_cast<int64_t>(x.size()), static_cast<int64_t>(inner),
                               static_cast<int64_t>(extent), bits, sd, c.stream));
  std::vector<double> scales(extent);
  d2h(c, scales.data(), sd, extent * 8);
  c.sync();
  if (g == Granularity::per_tensor) return QuantParams::per_tensor_symmetric(bits, scales[0]);
  return QuantParams::per_channel_symmetric(bits, axis, std::move(scales));
}

PercentileSearchResult init_scale_percentile_search(const std::vector<Tensor>& samples, int bits) {
  if (bits < 2 || bits > 30)
    throw std::invalid_argument("bit width out of supported range [2,30]: " + std::to_string(bits));
  if (samples.empty()) throw std::invalid_argument("percentile search: empty calibration sample list");
  Context& c = ctx();
  std::vector<int64_t> offsets{0};
  for (const Tensor& s : samples) offsets.push_back(offsets.back() + static_cast<int64_t>(s.size()));
  if (offsets.back() == 0) throw std::invalid_argument("quantile of empty vector");
  double* xd = c.ws<double>(kX, static_cast<size_t>(offsets.back()) * 8);
  for (size_t i = 0; i < samples.size(); ++i) h2d(c, xd + offsets[i], samples[i].data(), samples[i].size() * 8);
  const std::vector<double>& pct = PercentileSearchResult::percentiles();
  const int nc = static_cast<int>(pct.size());
  double* res = c.ws<double>(kY, (3 * pct.size() + 2) * 8);
  int64_t* err = c.ws<int64_t>(kErr, 16);
  check(qarvd_percentile_search_f64(xd, offsets.data(), static_cast<int64_t>(samples.size()), pct.data(), nc, bits,
                                    res, err, c.stream));
  std::vector<double> r(3 * pct.size() + 2);
  int64_t e[2];
  d2h(c, r.data(), res, r.size() * 8);
  d2h(c, e, err, 16);
  c.sync();
  // the reference's first failure in its loop order: candidate 0's scale is validated before any
  // element is read, then the first sample holding a non-finite value throws (quant.cpp:114-129)
  if (!(r[nc] > 0.0) || !std::isfinite(r[nc]))
    throw std::invalid_argument("quant params: scale must be positive and finite");
  if (e[0] >= 0) throw std::invalid_argument(nonfinite_msg(e[1]));
  PercentileSearchResult out;
  out.candidate_mse.assign(r.begin() + 2 * nc, r.begin() + 3 * nc);
  const int best = static_cast<int>(r[3 * nc]);
  out.best_percentile = pct[best];
  out.params = QuantParams::per_tensor_symmetric(bits, r[3 * nc + 1]);
  return out;
}

// ---- dual_scale.hpp --------------------------------------------------------------------

namespace {
// row_scales_over_columns (dual_scale.cpp:13-24) for both groups of a plan, through K5 on the f64
// weight (its scales are the reference's absmax / qmax, DBL_MIN for empty or all-zero groups)
void group_scales(const Tensor& w, const DualScalePlan& plan, int bits, std::vector<double>& so,
                  std::vector<double>& sn) {
  if (bits < 2 || bits > 8) throw std::invalid_argument("build_plan: the CUDA engine supports 2..8-bit weights");
  const size_t n = w.rows(), k = w.cols();
  Context& c = ctx();
  const Layout L = make_layout(plan, k);
  const double* wd = upload(c, kW, w.data(), n * k);
  const int32_t* gd = upload(c, kIdx, L.gather.data(), L.k_pad);
  int8_t* wq = c.ws<int8_t>(kCodes, n * L.k_pad);
  double* so_d = c.ws<double>(kScales, n * 8);
  double* sn_d = c.ws<double>(kScales2, n * 8);
  int64_t* err = c.ws<int64_t>(kErr, 8);
  check(qarvd_prepare_weights(wd, QARVD_F64, static_cast<int64_t>(n), static_cast<int64_t>(k),
                              static_cast<int64_t>(k), gd, static_cast<int64_t>(L.k_pad),
                              static_cast<int64_t>(L.k_outlier), bits, wq, static_cast<int64_t>(L.k_pad), so_d, sn_d,
                              nullptr, nullptr, err, c.stream));
  so.resize(n);
  sn.resize(n);
  d2h(c, so.data(), so_d, n * 8);
  d2h(c, sn.data(), sn_d, n * 8);
  c.sync();
}
}  // namespace

DualScalePlan build_single_scale_plan(const std::string& layer_name, const Tensor& w, int bits) {
  if (w.rank() != 2) throw std::invalid_argument("build_plan: weight must be 2-D");
  DualScalePlan plan;
  plan.layer_name = layer_name;
  plan.enabled = false;
  plan.d_in = w.cols();
  plan.normal_indices.resize(plan.d_in);
  plan.permutation.resize(plan.d_in);
  for (size_t i = 0; i < plan.d_in; ++i) {
    plan.normal_indices[i] = i;
    plan.permutation[i] = static_cast<uint32_t>(i);
  }
  std::vector<double> so, sn;
  group_scales(w, plan, bits, so, sn);
  plan.params_normal = QuantParams::per_channel_symmetric(bits, 0, std::move(sn));
  plan.params_outlier = plan.params_normal;
  return plan;
}

DualScalePlan build_plan(const Tensor& w, const OutlierReport& report, int bits) {
  if (w.rank() != 2) throw std::invalid_argument("build_plan: weight must be 2-D");
  const size_t d_in = w.cols();
  if (!report.norms.empty() && report.norms.size() != d_in)
    throw std::invalid_argument("build_plan: report does not match the weight's input width");
  for (size_t idx : report.aligned_outliers)
    if (idx >= d_in) throw std::out_of_range("build_plan: outlier index out of range");
  if (report.aligned_outliers.empty()) return qarvd::cuda::build_single_scale_plan(report.layer_name, w, bits);
  DualScalePlan plan;
  plan.layer_name = report.layer_name;
  plan.enabled = true;
  plan.d_in = d_in;
  plan.outlier_indices = report.aligned_outliers;
  std::vector<uint8_t> is_out(d_in, 0);
  for (size_t cidx : plan.outlier_indices) is_out[cidx] = 1;
  for (size_t cidx = 0; cidx < d_in; ++cidx)
    if (!is_out[cidx]) plan.normal_indices.push_back(cidx);
  if (plan.normal_indices.empty())
    throw std::invalid_argument("build_plan: outlier set would leave no normal channels");
  for (size_t cidx : plan.outlier_indices) plan.permutation.push_back(static_cast<uint32_t>(cidx));
  for (size_t cidx : plan.normal_indices) plan.permutation.push_back(static_cast<uint32_t>(cidx));
  std::vector<double> so, sn;
  group_scales(w, plan, bits, so, sn);
  plan.params_outlier = QuantParams::per_channel_symmetric(bits, 0, std::move(so));
  plan.params_normal = QuantParams::per_channel_symmetric(bits, 0, std::move(sn));
  return plan;
}

// ---- tensor.hpp ------------------------------------------------------------------------

Tensor matmul_nt(const Tensor& a, const Tensor& b) {
  if (a.rank() != 2 || b.rank() != 2) throw std::invalid_argument("matmul_nt: inputs must be 2-D");
  if (a.cols() != b.cols()) throw std::invalid_argument("matmul_nt: shape mismatch");
  Context& c = ctx();
  const size_t m = a.rows(), k = a.cols(), n = b.rows();
  Tensor out({m, n});
  if (m == 0 || n == 0) return out;
  const double* ad = upload(c, kX, a.data(), m * k);
  const double* bd = upload(c, kW, b.data(), n * k);
  double* cd = c.ws<double>(kY, m * n * 8);
  check(qarvd_matmul_nt_f64(ad, static_cast<int64_t>(m), static_cast<int64_t>(k), static_cast<int64_t>(k), bd,
                            static_cast<int64_t>(n), static_cast<int64_t>(k), cd, static_cast<int64_t>(n), c.stream));
  d2h(c, out.data(), cd, m * n * 8);
  c.sync();
  return out;
}

// ---- engine.hpp ------------------------------------------------------------------------

IntTensor kernel_a_quantize_activation(const Tensor& x, const QuantParams& p) { return qarvd::cuda::quantize(x, p); }

Tensor permute_activations(const Tensor& x, const DualScalePlan& plan) {
  if (!plan.enabled) return x;
  if (x.cols() != plan.permutation.size())
    throw std::invalid_argument("permute_activations: plan does not match activation width");
  Context& c = ctx();
  const size_t m = x.rows(), k = x.cols();
  std::vector<int32_t> idx(plan.permutation.begin(), plan.permutation.end());
  const double* xd = upload(c, kX, x.data(), m * k);
  const int32_t* id = upload(c, kIdx, idx.data(), k);
  double* out_d = c.ws<double>(kY, m * k * 8);
  check(qarvd_gather_columns(xd, static_cast<int64_t>(m), static_cast<int64_t>(k), id, static_cast<int64_t>(k), out_d,
                             static_cast<int64_t>(k), 8, c.stream));
  Tensor out({m, k});
  d2h(c, out.data(), out_d, m * k * 8);
  c.sync();
  return out;
}

Tensor kernel_b_gemm_dequant(const IntTensor& xq, const QuantizedLayer& layer) {
  if (layer.preserved)
    throw std::invalid_argument("kernel_b: layer is preserved, no integer path: " + layer.name);
  if (xq.shape.size() != 2 || xq.shape[1] != layer.in_dim)
    throw std::invalid_argument("kernel_b: activation shape does not match layer " + layer.name);
  const DeviceLayer L(layer, /*transient=*/true);
  Context& c = ctx();
  const size_t m = xq.shape[0];
  const int32_t* codes = upload(c, kCodes, xq.data.data(), m * L.k);
  const int32_t* pack = upload(c, kIdx, L.layout.pack.data(), L.layout.k_pad);
  int8_t* xd = c.ws<int8_t>(kXq, m * L.layout.k_pad + 16);
  int* bad = c.ws<int>(kErr, sizeof(int));
  check_cuda(cudaMemsetAsync(bad, 0, sizeof(int), c.stream));
  check(qarvd_pack_codes_i8(codes, static_cast<int64_t>(m), static_cast<int64_t>(L.k), pack,
                            static_cast<int64_t>(L.layout.k_pad), xd, static_cast<int64_t>(L.layout.k_pad), bad,
                            c.stream));
  int hbad = 0;
  d2h(c, &hbad, bad, sizeof(int));
  c.sync();
  if (hbad) throw std::invalid_argument("kernel_b: the CUDA engine stores codes as int8");
  return gemm_to_host(c, L, layer.act, xd, m);
}

namespace {
Tensor fakequant_forward(Context& c, const Tensor& x, const QuantParams& act, const double* w_dev, size_t n) {
  // matmul_nt(fake_quant(x, act), W_deq) (engine.cpp:141)
  act.validate(x.shape());
  if (act.per_channel()) throw std::invalid_argument("kernel_b: per-tensor activation params expected");
  const size_t m = x.rows(), k = x.cols();
  const double* xd = upload(c, kX, x.data(), m * k);
  const double* sd = upload(c, kScales, act.scale.data(), 1);
  const int32_t* zd = upload(c, kMisc, act.zero_point.data(), 1);
  double* xhat = c.ws<double>(kX2, m * k * 8);
  int64_t* err = c.ws<int64_t>(kErr, 8);
  check(qarvd_quantize_f64(xd, static_cast<int64_t>(m * k), 1, 1, sd, zd, act.q_min, act.q_max, nullptr, xhat, err,
                           c.stream));
  double* y = c.ws<double>(kY, m * n * 8);
  check(qarvd_matmul_nt_f64(xhat, static_cast<int64_t>(m), static_cast<int64_t>(k), static_cast<int64_t>(k), w_dev,
                            static_cast<int64_t>(n), static_cast<int64_t>(k), y, static_cast<int64_t>(n), c.stream));
  int64_t bad = INT64_MAX;
  d2h(c, &bad, err, 8);
  Tensor out({m, n});
  d2h(c, out.data(), y, m * n * 8);
  c.sync();
  if (bad != INT64_MAX) throw std::invalid_argument(nonfinite_msg(bad));
  return out;
}

// dequantized_weight_original_order (engine.cpp:117-130) into device slot `slot`
double* dequant_weight(Context& c, const QuantizedLayer& l, size_t slot) {
  const size_t n = l.out_dim, k = l.in_dim;
  const int32_t* wq = upload(c, kCodes, l.wq.data.data(), n * k);
  const uint32_t* perm = l.plan.enabled ? upload(c, kIdx, l.plan.permutation.data(), k) : nullptr;
  const double* sn = upload(c, kScales, l.plan.params_normal.scale.data(), n);
  const double* so = l.plan.enabled ? upload(c, kScales2, l.plan.params_outlier.scale.data(), n) : sn;
  double* w = c.ws<double>(slot, n * k * 8);
  check(qarvd_dequant_weight_f64(wq, static_cast<int64_t>(n), static_cast<int64_t>(k), perm,
                                 static_cast<int64_t>(l.plan.enabled ? l.plan.outlier_count() : 0), so, sn, w,
                                 c.stream));
  return w;
}
}  // namespace

Tensor quantized_layer_forward(const QuantizedLayer& layer, const Tensor& x, Engine engine) {
  if (layer.preserved) return qarvd::cuda::matmul_nt(x, layer.fp_weight);
  Context& c = ctx();
  if (engine == Engine::fakequant_sim) {
    const double* w = dequant_weight(c, layer, kW);
    return fakequant_forward(c, x, layer.act, w, layer.out_dim);
  }
  const DeviceLayer L(layer, /*transient=*/true);
  const int8_t* xq = quantize_to_layout(c, L, x, layer.act);
  return gemm_to_host(c, L, layer.act, xq, x.rows());
}

// ---- outlier.hpp -----------------------------------------------------------------------

OutlierReport analyze_layer(const std::string& layer_name, const Tensor& w, double tau, double alpha_min,
                            size_t align) {
  if (w.rank() != 2) throw std::invalid_argument("channel_l2_norms: input must be 2-D");
  const size_t n = w.rows(), k = w.cols();
  Context& c = ctx();
  const double* wd = upload(c, kW, w.data(), n * k);
  double* norms = c.ws<double>(kY, k * 8);
  double* stats = c.ws<double>(kScales, 24);
  int32_t* counts = c.ws<int32_t>(kMisc, 8);
  int32_t* raw = c.ws<int32_t>(kIdx, k * 4);
  int32_t* al = c.ws<int32_t>(kCodes, k * 4);
  qarvd_outlier_job job{wd, static_cast<int64_t>(n), static_cast<int64_t>(k), static_cast<int64_t>(k), norms,
                        stats, counts, raw, al};
  check(qarvd_analyze_layers(&job, 1, QARVD_F64, tau, alpha_min, static_cast<int64_t>(align), c.stream));
  OutlierReport rep;
  rep.layer_name = layer_name;
  rep.tau = tau;
  rep.alpha_min = alpha_min;
  rep.align = align;
  rep.norms.resize(k);
  double st[3];
  int32_t cnt[2];
  std::vector<int32_t> r(k), a(k);
  d2h(c, rep.norms.data(), norms, k * 8);
  d2h(c, st, stats, 24);
  d2h(c, cnt, counts, 8);
  d2h(c, r.data(), raw, k * 4);
  d2h(c, a.data(), al, k * 4);
  c.sync();
  rep.median = st[0];
  rep.mad = st[1];
  rep.threshold = st[2];
  rep.raw_outliers.assign(r.begin(), r.begin() + cnt[0]);
  rep.aligned_outliers.assign(a.begin(), a.begin() + cnt[1]);
  return rep;
}

// ---- providers ------------------------------------------------------------------------

CudaQuantizedProvider::CudaQuantizedProvider(const QuantizedModel& qm, Engine engine) : qm_(qm), engine_(engine) {
  Context& c = ctx();
  for (const auto& l : qm.layers) {
    if (l.preserved) {
      // preserved layers: matmul_nt(x, fp_weight) (engine.cpp:158) on the device
      double* w = nullptr;
      check_cuda(cudaMalloc(&w, l.fp_weight.size() * 8));
      h2d(c, w, l.fp_weight.data(), l.fp_weight.size() * 8);
      fp_.emplace(l.name, std::shared_ptr<double>(w, [](double* p) { cudaFree(p); }));
    } else if (engine == Engine::fakequant_sim) {
      const double* wdq = dequant_weight(c, l, kW);
      double* w = nullptr;
      check_cuda(cudaMalloc(&w, l.out_dim * l.in_dim * 8));
      check_cuda(cudaMemcpyAsync(w, wdq, l.out_dim * l.in_dim * 8, cudaMemcpyDeviceToDevice, c.stream));
      fp_.emplace(l.name, std::shared_ptr<double>(w, [](double* p) { cudaFree(p); }));
    } else {
      layers_.emplace(l.name, std::make_shared<DeviceLayer>(l));
    }
  }
  c.sync();
}

CudaQuantizedProvider::~CudaQuantizedProvider() = default;

namespace {
Tensor fp_forward(Context& c, const Tensor& x, const double* w_dev, size_t n) {
  if (x.rank() != 2) throw std::invalid_argument("matmul_nt: inputs must be 2-D");
  const size_t m = x.rows(), k = x.cols();
  const double* xd = upload(c, kX, x.data(), m * k);
  double* y = c.ws<double>(kY, m * n * 8);
  check(qarvd_matmul_nt_f64(xd, static_cast<int64_t>(m), static_cast<int64_t>(k), static_cast<int64_t>(k), w_dev,
                            static_cast<int64_t>(n), static_cast<int64_t>(k), y, static_cast<int64_t>(n), c.stream));
  Tensor out({m, n});
  d2h(c, out.data(), y, m * n * 8);
  c.sync();
  return out;
}
}  // namespace

Tensor CudaQuantizedProvider::forward(const std::string& layer, const Tensor& x) const {
  const QuantizedLayer& l = qm_.layer(layer);  // std::out_of_range as the reference (engine.cpp:29)
  Context& c = ctx();
  if (l.preserved) {
    if (x.cols() != l.in_dim) throw std::invalid_argument("matmul_nt: shape mismatch");
    return fp_forward(c, x, fp_.at(layer).get(), l.out_dim);
  }
  if (engine_ == Engine::fakequant_sim) return fakequant_forward(c, x, l.act, fp_.at(layer).get(), l.out_dim);
  const DeviceLayer& L = *layers_.at(layer);
  const int8_t* xq = quantize_to_layout(c, L, x, l.act);
  return gemm_to_host(c, L, l.act, xq, x.rows());
}

namespace {
// device copy of `bytes` from `src` (any device or host) on device `dev`
std::shared_ptr<double> copy_to_device(int dev, const void* src, size_t bytes, bool src_on_device) {
  int cur = 0;
  check_cuda(cudaGetDevice(&cur));
  check_cuda(cudaSetDevice(dev));
  double* d = nullptr;
  check_cuda(cudaMalloc(&d, bytes));
  check_cuda(cudaMemcpy(d, src, bytes, src_on_device ? cudaMemcpyDefault : cudaMemcpyHostToDevice));
  check_cuda(cudaSetDevice(cur));
  return std::shared_ptr<double>(d, [dev](double* p) {
    int c = 0;
    cudaGetDevice(&c);
    cudaSetDevice(dev);
    cudaFree(p);
    cudaSetDevice(c);
  });
}
}  // namespace

const double* DeviceWeights::get(const std::string& name, const std::function<std::shared_ptr<double>(int)>& make) const {
  int dev = 0;
  check_cuda(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu_);
  auto& per = by_device_[dev];
  auto it = per.find(name);
  if (it == per.end()) it = per.emplace(name, make(dev)).first;
  return it->second.get();
}

CudaFpProvider::CudaFpProvider(const ToyModel& model) : model_(model) {
  for (const auto& spec : model.registry()) weight_on_device(spec.name);  // upload to the current device
}

const double* CudaFpProvider::weight_on_device(const std::string& layer) const {
  return weights_.get(layer, [&](int dev) {
    const Tensor& w = model_.weight(layer);
    return copy_to_device(dev, w.data(), w.size() * 8, false);
  });
}

Tensor CudaFpProvider::forward(const std::string& layer, const Tensor& x) const {
  const Tensor& w = model_.weight(layer);  // the reference's lookup and exception
  if (x.rank() != 2 || x.cols() != w.cols()) throw std::invalid_argument("matmul_nt: shape mismatch");
  return fp_forward(ctx(), x, weight_on_device(layer), w.rows());
}

CudaMinMaxFakeQuantProvider::CudaMinMaxFakeQuantProvider(const ToyModel& model, BitwidthScheme scheme,
                                                         std::vector<std::string> keep_list)
    : model_(model), scheme_(scheme), keep_list_(std::move(keep_list)), fp_(model) {
  if (scheme_.is_lossless()) return;
  Context& c = ctx();
  for (const auto& spec : model.registry()) {
    if (matches_keep_list(spec.name, keep_list_)) continue;
    // fake_quant(w, init_scale_minmax(w, wb, per_channel, 0)) (toy_model.cpp:312-315), cached
    const Tensor& w = model.weight(spec.name);
    const size_t n = w.rows(), k = w.cols();
    const double* wd = upload(c, kW, w.data(), n * k);
    double* sd = c.ws<double>(kScales, n * 8);
    check(qarvd_minmax_scale_f64(wd, static_cast<int64_t>(n * k), static_cast<int64_t>(k), static_cast<int64_t>(n),
                                 scheme_.weight_bits, sd, c.stream));
    double* fq = nullptr;
    check_cuda(cudaMalloc(&fq, n * k * 8));
    int64_t* err = c.ws<int64_t>(kErr, 8);
    const int32_t qmax = QuantParams::symmetric_max(scheme_.weight_bits);
    check(qarvd_quantize_f64(wd, static_cast<int64_t>(n * k), static_cast<int64_t>(k), static_cast<int64_t>(n), sd,
                             nullptr, -qmax, qmax, nullptr, fq, err, c.stream));
    int64_t bad = INT64_MAX;
    d2h(c, &bad, err, 8);
    c.sync();
    if (bad != INT64_MAX) {
      cudaFree(fq);
      throw std::invalid_argument(nonfinite_msg(bad));
    }
    int dev = 0;
    check_cuda(cudaGetDevice(&dev));
    std::shared_ptr<double> owned(fq, [](double* p) { cudaFree(p); });
    fq_home_.emplace(spec.name, owned);
    fq_.get(spec.name, [&](int) { return owned; });
  }
}

const double* CudaMinMaxFakeQuantProvider::fq_on_device(const std::string& layer) const {
  // other devices get a copy of the cached fake-quantized weights (computed once, above)
  return fq_.get(layer, [&](int dev) {
    const Tensor& w = model_.weight(layer);
    return copy_to_device(dev, fq_home_.at(layer).get(), w.size() * 8, true);
  });
}

CudaMinMaxFakeQuantProvider::~CudaMinMaxFakeQuantProvider() = default;

Tensor CudaMinMaxFakeQuantProvider::forward(const std::string& layer, const Tensor& x) const {
  if (scheme_.is_lossless() || matches_keep_list(layer, keep_list_)) return fp_.forward(layer, x);
  const Tensor& w = model_.weight(layer);
  if (x.rank() != 2 || x.cols() != w.cols()) throw std::invalid_argument("matmul_nt: shape mismatch");
  // live per-tensor minmax activation params (toy_model.cpp:321-323), all on the device
  Context& c = ctx();
  const size_t m = x.rows(), k = x.cols(), n = w.rows();
  const double* xd = upload(c, kX, x.data(), m * k);
  double* sd = c.ws<double>(kScales, 8);
  check(qarvd_minmax_scale_f64(xd, static_cast<int64_t>(m * k), 1, 1, scheme_.activation_bits, sd, c.stream));
  double* xhat = c.ws<double>(kX2, m * k * 8);
  int64_t* err = c.ws<int64_t>(kErr, 8);
  const int32_t qmax = QuantParams::symmetric_max(scheme_.activation_bits);
  check(qarvd_quantize_f64(xd, static_cast<int64_t>(m * k), 1, 1, sd, nullptr, -qmax, qmax, nullptr, xhat, err,
                           c.stream));
  double* y = c.ws<double>(kY, m * n * 8);
  check(qarvd_matmul_nt_f64(xhat, static_cast<int64_t>(m), static_cast<int64_t>(k), static_cast<int64_t>(k),
                            fq_on_device(layer), static_cast<int64_t>(n), static_cast<int64_t>(k), y,
                            static_cast<int64_t>(n), c.stream));
  int64_t bad = INT64_MAX;
  double s = 0.0;
  d2h(c, &bad, err, 8);
  d2h(c, &s, sd, 8);
  Tensor out({m, n});
  d2h(c, out.data(), y, m * n * 8);
  c.sync();
  if (!(s > 0.0) || !std::isfinite(s)) throw std::invalid_argument("quant params: scale must be positive and finite");
  if (bad != INT64_MAX) throw std::invalid_argument(nonfinite_msg(bad));
  return out;
}

// ---- rollouts ---------------------------------------------------------------------------

Rollout run_quantized(const QuantizedModel& qm, uint64_t prompt_seed, Engine engine) {
  const CudaQuantizedProvider provider(qm, engine);
  return run_rollout(qm.cfg, provider, &provider, QuantTarget::all, 0, prompt_seed);
}

Rollout rollout(const ToyModel& model, uint64_t prompt_seed, const QuantMode& mode,
                const std::vector<std::string>& capture_layers) {
  const CudaFpProvider fp(model);
  if (mode.target == QuantTarget::none)
    return run_rollout(model.config(), fp, nullptr, mode.target, mode.chunk, prompt_seed, capture_layers);
  const CudaMinMaxFakeQuantProvider quant(model, mode.scheme, mode.keep_list);
  return run_rollout(model.config(), fp, &quant, mode.target, mode.chunk, prompt_seed, capture_layers);
}

std::vector<CalibSample> collect_calibration(const ToyModel& model, const std::vector<uint64_t>& prompt_seeds,
                                             const std::vector<std::string>& capture_layers) {
  if (prompt_seeds.empty()) throw std::invalid_argument("collect_calibration: need at least one prompt seed");
  for (const auto& name : capture_layers)
    if (!model.has_layer(name)) throw std::out_of_range("collect_calibration: layer not in registry: " + name);
  const CudaFpProvider fp(model);
  std::vector<std::vector<CalibSample>> per_prompt(prompt_seeds.size());
  parallel_for(prompt_seeds.size(), [&](size_t p) {
    Rollout r = run_rollout(model.config(), fp, nullptr, QuantTarget::none, 0, prompt_seeds[p], capture_layers);
    per_prompt[p].reserve(r.captures.size());
    for (auto& cap : r.captures) per_prompt[p].push_back({cap.layer, cap.chunk, std::move(cap.x)});
  });
  std::vector<CalibSample> samples;
  for (auto& batch : per_prompt)
    for (auto& s : batch) samples.push_back(std::move(s));
  return samples;
}

int sensitivity_devices() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1) n = 1;
  if (const char* e = getenv("QARVD_SENSITIVITY_GPUS")) {
    const int v = atoi(e);
    if (v >= 1 && v < n) n = v;
  }
  return n;
}

SensitivityProfile profile_sensitivity(const ToyModel& model, BitwidthScheme scheme,
                                       const std::vector<uint64_t>& seeds) {
  if (seeds.empty()) throw std::invalid_argument("profile_sensitivity: need at least one seed");
  const size_t n_chunks = model.config().chunks;
  const CudaFpProvider fp(model);
  const CudaMinMaxFakeQuantProvider quant(model, scheme);
  // sensitivity.cpp:37-52: references per seed, then every (seed, chunk) probe, each slot written
  // by exactly one worker (the providers are shared across workers; each worker thread has its
  // own device context)
  // data-parallel over GPUs: task t runs on device t % G (every worker thread has a device
  // context per GPU; the providers keep one weight copy per device)
  int home = 0;
  check_cuda(cudaGetDevice(&home));
  const int gpus = sensitivity_devices();
  auto on_device = [&](size_t task) { check_cuda(cudaSetDevice(static_cast<int>((home + task) % gpus))); };
  std::vector<Rollout> references(seeds.size());
  parallel_for(seeds.size(), [&](size_t s) {
    on_device(s);
    references[s] = run_rollout(model.config(), fp, nullptr, QuantTarget::none, 0, seeds[s]);
  });
  std::vector<std::vector<double>> per_seed(seeds.size(), std::vector<double>(n_chunks, 0.0));
  parallel_for(seeds.size() * n_chunks, [&](size_t task) {
    on_device(task);
    const size_t s = task / n_chunks, i = task % n_chunks;
    const Rollout probe = run_rollout(model.config(), fp, &quant, QuantTarget::only_chunk, i + 1, seeds[s]);
    per_seed[s][i] = latent_mse(references[s], probe);
  });
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

// ---- calibrate.hpp ----------------------------------------------------------------------

double weighted_loss(const std::vector<const CalibSample*>& batch, const LearnableQuantState& state,
                     const std::vector<double>& chunk_weights) {
  // weighted_recon_loss(batch, state, w, state.hard_weight()) (calibrate.cpp:201-224): per sample
  // target = X W^T and pred = FQ(X) What^T as exact f64 products, total += w_chunk ||target - pred||^2
  if (batch.empty()) throw std::invalid_argument("weighted loss: empty batch");
  Context& c = ctx();
  const size_t n = state.weight.rows(), k = state.weight.cols();
  const DeviceState d = upload_state(c, state, false);
  double* total = c.ws<double>(kLoss0, 8);
  int64_t* err = c.ws<int64_t>(kErr, 8);
  const int32_t qmax = QuantParams::symmetric_max(state.act_bits);
  int64_t bad_sample = -1, bad_index = 0;
  for (size_t b = 0; b < batch.size(); ++b) {
    const CalibSample* s = batch[b];
    if (s->chunk < 1 || s->chunk > chunk_weights.size())
      throw std::out_of_range("weighted loss: sample chunk outside the weight vector");
    if (s->x.rank() != 2 || s->x.cols() != k) throw std::invalid_argument("matmul_nt: shape mismatch");
    const size_t m = s->x.rows();
    const double* xd = upload(c, kX, s->x.data(), m * k);
    double* tgt = c.ws<double>(kY, m * n * 8);
    double* xhat = c.ws<double>(kX2, m * k * 8);
    double* pred = c.ws<double>(kLoss1, m * n * 8);
    check(qarvd_matmul_nt_f64(xd, static_cast<int64_t>(m), static_cast<int64_t>(k), static_cast<int64_t>(k), d.w,
                              static_cast<int64_t>(n), static_cast<int64_t>(k), tgt, static_cast<int64_t>(n), c.stream));
    check(qarvd_quantize_f64(xd, static_cast<int64_t>(m * k), 1, 1, d.act_scale, nullptr, -qmax, qmax, nullptr, xhat,
                             err, c.stream));
    check(qarvd_matmul_nt_f64(xhat, static_cast<int64_t>(m), static_cast<int64_t>(k), static_cast<int64_t>(k), d.what,
                              static_cast<int64_t>(n), static_cast<int64_t>(k), pred, static_cast<int64_t>(n),
                              c.stream));
    check(qarvd_sq_distance_acc_f64(tgt, pred, static_cast<int64_t>(m * n), chunk_weights[s->chunk - 1], total,
                                    b > 0 ? 1 : 0, b + 1 == batch.size() ? static_cast<double>(batch.size()) : 0.0,
                                    c.stream));
    int64_t bad = INT64_MAX;
    d2h(c, &bad, err, 8);
    c.sync();  // the per-sample buffers are reused by the next sample
    if (bad != INT64_MAX && bad_sample < 0) {
      bad_sample = static_cast<int64_t>(b);
      bad_index = bad;
      break;
    }
  }
  if (bad_sample >= 0) throw std::invalid_argument(nonfinite_msg(bad_index));
  double out = 0.0;
  d2h(c, &out, total, 8);
  c.sync();
  return out;
}

LayerCalibResult calibrate_layer(const Tensor& w, const DualScalePlan& plan, const QuantParams& act_init,
                                 const std::vector<const CalibSample*>& samples,
                                 const std::vector<double>& chunk_weights, const CalibConfig& cfg) {
  cfg.validate();
  if (samples.empty()) throw std::invalid_argument("calibrate_layer: no calibration samples");
  if (act_init.per_channel() || act_init.zero_point[0] != 0)
    throw std::invalid_argument("calibrate_layer: the activation init must be per-tensor symmetric");
  Context& c = ctx();
  const size_t n = w.rows(), k = w.cols();
  std::vector<uint8_t> mask(k, 0);
  if (plan.enabled)
    for (size_t col : plan.outlier_indices) mask[col] = 1;
  std::vector<int64_t> rows{0}, chunks;
  for (const CalibSample* s : samples) {
    if (s->x.cols() != k) throw std::invalid_argument("calibrate_layer: sample width does not match the weight");
    rows.push_back(rows.back() + static_cast<int64_t>(s->x.rows()));
    chunks.push_back(static_cast<int64_t>(s->chunk));
  }
  const std::vector<double>& sn = plan.params_normal.scale;
  const std::vector<double>& so = plan.enabled ? plan.params_outlier.scale : plan.params_normal.scale;
  const double* w_d = upload(c, kW, w.data(), n * k);
  const uint8_t* mask_d = upload(c, kMisc, mask.data(), k);
  const double* sn_d = upload(c, kScales, sn.data(), n);
  const double* so_d = upload(c, kScales2, so.data(), n);
  double* x_d = c.ws<double>(kX, static_cast<size_t>(rows.back()) * k * 8);
  for (size_t i = 0; i < samples.size(); ++i)
    h2d(c, x_d + rows[i] * static_cast<int64_t>(k), samples[i]->x.data(), samples[i]->x.size() * 8);
  int8_t* codes_d = c.ws<int8_t>(kCodes, n * k);
  double* sn_out = c.ws<double>(kY, n * 8);
  double* so_out = c.ws<double>(kY2, n * 8);
  double* sc_out = c.ws<double>(kMisc2, 3 * 8);
  const size_t iters = static_cast<size_t>(cfg.iterations > 0 ? cfg.iterations : 0);
  double* tr_out = c.ws<double>(kMisc3, std::max<size_t>(iters, 1) * 8);
  qarvd_calib_config cc{};
  cc.iterations = cfg.iterations;
  cc.batch_size = cfg.batch_size;
  cc.lr_round = cfg.lr_round;
  cc.lr_scale = cfg.lr_scale;
  cc.seed = cfg.seed;
  cc.train_activation_scale = cfg.train_activation_scale ? 1 : 0;
  cc.zeta = cfg.zeta;
  cc.gamma_lo = cfg.gamma_lo;
  cc.reg_lambda = cfg.reg_lambda;
  cc.beta_start = cfg.beta_start;
  cc.beta_end = cfg.beta_end;
  cc.warmup_frac = cfg.warmup_frac;
  check(qarvd_calibrate_layer(w_d, static_cast<int64_t>(n), static_cast<int64_t>(k), mask_d, plan.enabled ? 1 : 0,
                              sn_d, so_d, act_init.scale[0], act_init.bits, plan.params_normal.bits, x_d, rows.data(),
                              chunks.data(), static_cast<int64_t>(samples.size()), chunk_weights.data(),
                              static_cast<int64_t>(chunk_weights.size()), &cc, plan.layer_name.c_str(), codes_d,
                              sn_out, so_out, sc_out, tr_out, c.stream));
  std::vector<int8_t> codes(n * k);
  std::vector<double> lsn(n), lso(n), sc(3), tr(iters);
  d2h(c, codes.data(), codes_d, n * k);
  d2h(c, lsn.data(), sn_out, n * 8);
  d2h(c, lso.data(), so_out, n * 8);
  d2h(c, sc.data(), sc_out, 3 * 8);
  d2h(c, tr.data(), tr_out, iters * 8);
  c.sync();
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
  const std::vector<CalibSample> samples = qarvd::cuda::collect_calibration(model, opts.prompt_seeds, quant_layers);
  ModelCalibResult out;
  out.qmodel.cfg = model.config();
  out.qmodel.scheme = opts.base.scheme;
  out.qmodel.keep_list = opts.keep_list;
  out.qmodel.layers.resize(model.registry().size());
  out.layer_results.resize(quant_layers.size());
  std::vector<size_t> registry_slot;
  for (size_t li = 0; li < model.registry().size(); ++li) {
    const LayerSpec& spec = model.registry()[li];
    if (!matches_keep_list(spec.name, opts.keep_list)) {
      registry_slot.push_back(li);
      continue;
    }
    // preserved: bf16 passthrough (calibrate.cpp:419-430)
    QuantizedLayer l;
    l.name = spec.name;
    l.out_dim = spec.out_dim;
    l.in_dim = spec.in_dim;
    l.preserved = true;
    Tensor fp = model.weight(spec.name);
    for (size_t i = 0; i < fp.size(); ++i) fp[i] = static_cast<double>(bf16_to_float(float_to_bf16(static_cast<float>(fp[i]))));
    l.fp_weight = fp;
    out.qmodel.layers[li] = std::move(l);
  }
  // the reference's slot-indexed parallel_for over layers (calibrate.cpp:440-484); each worker
  // runs its layers on its own stream: K3 -> plan (K5 scales) -> percentile init -> K7 -> pre-permute
  parallel_for(quant_layers.size(), [&](size_t qi) {
    const LayerSpec& spec = model.registry()[registry_slot[qi]];
    const Tensor& w = model.weight(spec.name);
    DualScalePlan plan;
    if (opts.dual_scale) {
      const OutlierReport report = qarvd::cuda::analyze_layer(spec.name, w, opts.tau, opts.alpha_min, opts.align);
      plan = qarvd::cuda::build_plan(w, report, opts.base.scheme.weight_bits);
    } else {
      plan = qarvd::cuda::build_single_scale_plan(spec.name, w, opts.base.scheme.weight_bits);
    }
    std::vector<const CalibSample*> ls;
    std::vector<Tensor> acts;
    for (const auto& smp : samples)
      if (smp.layer == spec.name) {
        ls.push_back(&smp);
        acts.push_back(smp.x);
      }
    const PercentileSearchResult act_init =
        qarvd::cuda::init_scale_percentile_search(acts, opts.base.scheme.activation_bits);
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
    // pre-permuted [outlier | normal] codes (calibrate.cpp:474-480) through the device gather
    {
      Context& c = ctx();
      const size_t n = spec.out_dim, k = spec.in_dim;
      const int32_t* cd = upload(c, kCodes, res.codes.data.data(), n * k);
      std::vector<int32_t> idx(res.plan.permutation.begin(), res.plan.permutation.end());
      const int32_t* id = upload(c, kIdx, idx.data(), k);
      int32_t* pd = c.ws<int32_t>(kY, n * k * 4);
      check(qarvd_gather_columns(cd, static_cast<int64_t>(n), static_cast<int64_t>(k), id, static_cast<int64_t>(k),
                                 pd, static_cast<int64_t>(k), 4, c.stream));
      l.wq.data.resize(n * k);
      d2h(c, l.wq.data.data(), pd, n * k * 4);
      c.sync();
    }
    out.qmodel.layers[registry_slot[qi]] = std::move(l);
    out.layer_results[qi] = std::move(res);
  });
  return out;
}

}  // namespace cuda
}  // namespace qarvd
