// K7 — AdaRound calibration of one layer on the GPU (f64), the reference's calibrator.
//
// Replaces calibrate_layer (/root/reference/proj/core/src/calibrate.cpp:298-396) with its
// state LearnableQuantState (calibrate.cpp:77-199) and gradients soft_loss_gradients
// (calibrate.cpp:232-296): learned rounding variables V with the rectified sigmoid
// h(V) = clip(sigmoid(V)(zeta - gamma) + gamma, 0, 1), learned per-row log group scales and
// a learned log activation scale, trained with the frame-weighted Eq. 5 objective
// (1/B) sum_s w[chunk_s] ||X_s W^T - FQ(X_s) What^T||^2, the corner-pushing regulariser
// after warm-up, and bias-corrected Adam with a cosine-annealed learning rate.
//
// Everything stays f64-accurate like the reference, so the trajectory follows it to rounding:
// the per-iteration products (prediction X^ What^T - target, dL/dWhat = D^T X^) run on the int8
// tensor cores as exact integer slice products (K2 with its f64 epilogue, Ozaki-style: see
// kOzSlices), each over the batch's samples stacked along the rows (QARVD_K7_OZAKI=0 takes
// cuBLAS DGEMM instead; the one-time target product X W^T stays a DGEMM); the reference's third
// product dL/dX^ = D What only feeds the act-scale gradient, which equals <What, dL/dWhat>;
// every elementwise step,
// reduction and Adam update is a kernel here with the reference's per-element formula, and
// every reduction runs in a fixed order (deterministic).  The target X_s W^T is computed
// once per sample (W is fixed during calibration).  The host only replays the reference's
// batch sampler (Prng(mix_seed(seed, fnv1a(layer)))) and enqueues launches; losses,
// divergence and results stay on the device until the end.
#include <cublas_v2.h>

#include <map>

#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "crmath.cuh"
#include "libm_ref.cuh"

namespace qarvd_b200 {
namespace {

// ---- host restatement of rng.hpp (splitmix64, mix_seed, fnv1a) ------------------------
uint64_t splitmix64_h(uint64_t& s) {
  uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
uint64_t mix_seed_h(uint64_t a, uint64_t b) {
  uint64_t s = a;
  const uint64_t h = splitmix64_h(s);
  s = h ^ (b + 0x9e3779b97f4a7c15ULL);
  return splitmix64_h(s);
}
uint64_t fnv1a_h(const char* d, size_t n) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (size_t i = 0; i < n; ++i) {
    h ^= static_cast<unsigned char>(d[i]);
    h *= 0x100000001b3ULL;
  }
  return h;
}

constexpr int kT = 256;
inline unsigned blocks_for(int64_t n) {
  const int64_t b = (n + kT - 1) / kT;
  return static_cast<unsigned>(b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16);
}

// sigmoid (calibrate.cpp:18) with the reference's own exp (libm_ref.cuh: glibc's algorithm, bit for bit)
__device__ __forceinline__ double sigmoid_d(double x) { return 1.0 / (1.0 + libm::exp(-x)); }
__device__ __forceinline__ double clampd(double v, double lo, double hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}
// 1.5 * 2^52: for |x| < 2^51, x + kRoundMagic rounds x to an integer (round-half-even, as rint) whose
// two's complement sits in the low word, and (x + kRoundMagic) - kRoundMagic == rint(x) exactly
constexpr double kRoundMagic = 6755399441055744.0;

// weight_scale(r, outlier_group) = exp(log scale) (calibrate.cpp:117-119); log_s = [normal n | outlier n]
__device__ __forceinline__ double wscale(const double* log_s, int64_t n, int64_t r, bool outl) {
  return libm::exp(outl ? log_s[n + r] : log_s[r]);
}

// LearnableQuantState::init V (calibrate.cpp:96-114): h(V) = frac(w/s), clamped to [1e-4, 1-1e-4]
__global__ void init_v_kernel(const double* w, const uint8_t* mask, int enabled, const double* s_n,
                              const double* s_o, int64_t n, int64_t k, double zeta, double gamma,
                              double* v) {
  const double span = zeta - gamma;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n * k;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / k, c = i - r * k;
    const double s = (enabled && mask[c]) ? s_o[r] : s_n[r];
    const double ratio = w[i] / s;
    double frac = ratio - floor(ratio);
    frac = clampd(frac, 1e-4, 1.0 - 1e-4);
    const double p = (frac - gamma) / span;
    v[i] = libm::log(p / (1.0 - p));
  }
}

// soft weights (calibrate.cpp:245-266): what = s*clip(floor(w/s) + h(V)), the clipped code and
// dh/dV (0 where the pre-activation or the code clips).  hard = 1: h -> [h > 0.5] (hard_weight,
// calibrate.cpp:159-161), codes_out = int8 codes (hard_codes, calibrate.cpp:163-183).
__global__ void weights_kernel(const double* w, const double* v, const uint8_t* mask, int enabled,
                               const double* log_s, int64_t n, int64_t k, double zeta, double gamma,
                               int qmin, int qmax, int hard, double* what, double* code,
                               double* dhdv, int8_t* codes_out) {
  const double span = zeta - gamma;
  // one CTA per weight row: the row's two group scales are computed once
  const int64_t r = blockIdx.x;
  const double s_n = wscale(log_s, n, r, false), s_o = wscale(log_s, n, r, true);
  for (int64_t c = threadIdx.x; c < k; c += blockDim.x) {
    const int64_t i = r * k + c;
    const bool outl = enabled && mask[c];
    const double s = outl ? s_o : s_n;
    const double sig = sigmoid_d(v[i]);
    const double pre = sig * span + gamma;
    const double h = clampd(pre, 0.0, 1.0);
    const double u = floor(w[i] / s) + (hard ? (h > 0.5 ? 1.0 : 0.0) : h);
    const double cl = clampd(u, static_cast<double>(qmin), static_cast<double>(qmax));
    what[i] = s * cl;
    if (code) code[i] = cl;
    if (dhdv) {
      const bool inside_code = u > static_cast<double>(qmin) && u < static_cast<double>(qmax);
      const bool inside_h = pre > 0.0 && pre < 1.0;
      dhdv[i] = (inside_code && inside_h) ? span * sig * (1.0 - sig) : 0.0;
    }
    if (codes_out) codes_out[i] = static_cast<int8_t>(cl);
  }
}

// fake_quant(x, act) (quant.cpp:113-159, per-tensor symmetric, s = exp(log_sa)): xhat = code * s
// in f64; a non-finite input sets *bad (the reference throws)
__global__ void xhat_kernel(const double* x, int64_t count, const double* log_sa, int qmax,
                            double* xhat, int* bad) {
  const double s = libm::exp(*log_sa);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double xv = x[i];
    if (!isfinite(xv)) {
      *bad = 1;
      xhat[i] = 0.0;
      continue;
    }
    const double q = clampd(rint(xv / s), -static_cast<double>(qmax), static_cast<double>(qmax));
    xhat[i] = q * s;
  }
}

// fixed-order block sums: block p of the grid reduces the contiguous range p of [0, count)
// (four independent accumulators per thread, then a shuffle tree) -> partial[p]
constexpr int kRedBlocks = 296;
constexpr int kMaxGroup = 16;  // samples stacked into one GEMM
__device__ __forceinline__ double block_sum(double acc) {
  __shared__ double red[kT / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kT / 32; ++w) t += red[w];
  return t;
}
// partial[p] = sum a[i]*b[i] over block p's range (b = nullptr: a[i]^2); with sub, a[i] is
// first replaced by a[i] - sub[i]; with rescale the range is written back as a[i] * scale
// (sub or rescale: written back whenever either is set)
__global__ void __launch_bounds__(kT) dot_partial_kernel(double* a, const double* b, int64_t count,
                                                          int rescale, double scale, double* partial,
                                                          const double* sub = nullptr) {
  const int64_t per = (count + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * per, hi = lo + per < count ? lo + per : count;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int64_t i = lo + threadIdx.x;
  for (; i + 3 * kT < hi; i += 4 * kT) {
    double v0 = a[i], v1 = a[i + kT], v2 = a[i + 2 * kT], v3 = a[i + 3 * kT];
    if (sub) v0 -= sub[i], v1 -= sub[i + kT], v2 -= sub[i + 2 * kT], v3 -= sub[i + 3 * kT];
    if (b) {
      a0 += v0 * b[i], a1 += v1 * b[i + kT], a2 += v2 * b[i + 2 * kT], a3 += v3 * b[i + 3 * kT];
    } else {
      a0 += v0 * v0, a1 += v1 * v1, a2 += v2 * v2, a3 += v3 * v3;
    }
    if (rescale) a[i] = v0 * scale, a[i + kT] = v1 * scale, a[i + 2 * kT] = v2 * scale, a[i + 3 * kT] = v3 * scale;
    else if (sub) a[i] = v0, a[i + kT] = v1, a[i + 2 * kT] = v2, a[i + 3 * kT] = v3;
  }
  for (; i < hi; i += kT) {
    const double v0 = sub ? a[i] - sub[i] : a[i];
    a0 += b ? v0 * b[i] : v0 * v0;
    if (rescale) a[i] = v0 * scale;
    else if (sub) a[i] = v0;
  }
  const double t = block_sum((a0 + a1) + (a2 + a3));
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
}
struct GroupWeights {
  double w[kMaxGroup];
};
// *acc (+)= sum_g wt.w[g] * (sum of partial[g*per ..][per]) in a fixed order (per <= kRedBlocks):
// warp g sums group g (all of its loads issued before the adds), thread 0 combines the groups
// in order; with log_sa the total is multiplied by exp(*log_sa) (act grad).  Launch with
// kMaxGroup * 32 threads.
__global__ void __launch_bounds__(kMaxGroup * 32) dot_final_kernel(const double* partial, int groups,
                                                                  GroupWeights wt, const double* log_sa,
                                                                  int accumulate, double* acc,
                                                                  int per = kRedBlocks) {
  constexpr int kPer = (kRedBlocks + 31) / 32;
  __shared__ double gsum[kMaxGroup];
  const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (g < groups) {
    double v[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int i = lane + 32 * j;
      v[j] = i < per ? partial[g * per + i] : 0.0;
    }
    double sum = 0.0;
#pragma unroll
    for (int j = 0; j < kPer; ++j) sum += v[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, o);
    if (lane == 0) gsum[g] = sum;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  double total = 0.0;
  for (int i = 0; i < groups; ++i) total += wt.w[i] * gsum[i];
  if (log_sa) total *= libm::exp(*log_sa);
  *acc = accumulate ? *acc + total : total;
}

// per-iteration loss bookkeeping: loss = acc / B; best = min(best, loss) -> trace[t];
// the first non-finite iteration is recorded (the reference throws at it)
__global__ void trace_kernel(const double* acc, double inv_b, double* best, double* trace, int t,
                             int* diverged_at) {
  const double loss = *acc * inv_b;
  if (!isfinite(loss) && *diverged_at < 0) *diverged_at = t;
  const double b = *best < loss ? *best : loss;
  *best = b;
  trace[t] = b;
}

// gradients (calibrate.cpp:276-289, :345-362): v_grad = gW*s*dh_dv (+ regulariser), per-row
// log-scale grads sum_c gW*s*code split by group; one CTA per row, fixed-order reduction
__global__ void __launch_bounds__(kT) grad_kernel(const double* gw, const double* v, const double* code,
                                                  const double* dhdv, const uint8_t* mask, int enabled,
                                                  const double* log_s, int64_t n, int64_t k, int reg_on,
                                                  double reg_lambda, double beta, double zeta, double gamma,
                                                  double* vgrad, double* sgrad) {
  const int64_t r = blockIdx.x;
  double gn = 0.0, go = 0.0;
  const double span = zeta - gamma;
  const double s_n = wscale(log_s, n, r, false), s_o = wscale(log_s, n, r, true);
  for (int64_t c = threadIdx.x; c < k; c += kT) {
    const int64_t i = r * k + c;
    const bool outl = enabled && mask[c];
    const double s = outl ? s_o : s_n;
    const double gwe = gw[i];
    double g = gwe * s * dhdv[i];
    if (reg_on) {
      const double sig = sigmoid_d(v[i]);
      const double pre = sig * span + gamma;
      const double h = clampd(pre, 0.0, 1.0);
      const double centered = 2.0 * h - 1.0;
      const double mag = fabs(centered);
      const double dreg_dh = -2.0 * beta * libm::pow(mag > 1e-12 ? mag : 1e-12, beta - 1.0) *
                             (centered >= 0 ? 1.0 : -1.0);
      const double dh_dv = (pre > 0.0 && pre < 1.0) ? span * sig * (1.0 - sig) : 0.0;
      g += reg_lambda * dreg_dh * dh_dv;
    }
    vgrad[i] = g;
    const double gs = gwe * s * code[i];
    if (outl) go += gs;
    else gn += gs;
  }
  __shared__ double rn[kT], ro[kT];
  rn[threadIdx.x] = gn;
  ro[threadIdx.x] = go;
  __syncthreads();
  for (int s = kT / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      rn[threadIdx.x] += rn[threadIdx.x + s];
      ro[threadIdx.x] += ro[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    sgrad[r] = rn[0];
    sgrad[n + r] = enabled ? ro[0] : 0.0;  // calibrate.cpp:374
  }
}

// AdamBuffer::step (calibrate.cpp:27-40); c1 / c2 = 1 - b^t from the host (std::pow)
__global__ void adam_kernel(double* p, const double* g, double* m, double* v, int64_t count, double lr,
                            double c1, double c2) {
  constexpr double b1 = 0.9, b2 = 0.999, eps = 1e-8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    m[i] = b1 * m[i] + (1.0 - b1) * g[i];
    v[i] = b2 * v[i] + (1.0 - b2) * g[i] * g[i];
    p[i] -= lr * (m[i] / c1) / (sqrt(v[i] / c2) + eps);
  }
}

__global__ void log_kernel(const double* a, double* out, int64_t count) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = libm::log(a[i]);
}
__global__ void exp_kernel(const double* a, double* out, int64_t count) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = libm::exp(a[i]);
}
__global__ void loss_kernel(const double* acc, double inv, double* out) { *out = *acc * inv; }
__global__ void set_scalars_kernel(double* log_sa, double act_scale, double* best, int* diverged,
                                   int* bad) {
  *log_sa = libm::log(act_scale);
  *best = INFINITY;
  *diverged = -1;
  *bad = 0;
}

const char* cublas_msg(cublasStatus_t s) {
  switch (s) {
    case CUBLAS_STATUS_NOT_INITIALIZED: return "not initialized";
    case CUBLAS_STATUS_ALLOC_FAILED: return "alloc failed";
    case CUBLAS_STATUS_INVALID_VALUE: return "invalid value";
    case CUBLAS_STATUS_EXECUTION_FAILED: return "execution failed";
    default: return "error";
  }
}
#define QARVD_CUBLAS_TRY(expr)                                                           \
  do {                                                                                   \
    cublasStatus_t _s = (expr);                                                          \
    if (_s != CUBLAS_STATUS_SUCCESS)                                                     \
      QARVD_FAIL(QARVD_ERR_CUDA, std::string("cuBLAS: ") + cublas_msg(_s) + " at " +     \
                                     __FILE__ + ":" + std::to_string(__LINE__));         \
  } while (0)


// ---- the two f64 products on the int8 tensor cores (Ozaki-style exact slices) ---------------
// P = X^ What^T and dL/dWhat = D'^T X^ run as K2 (tcgen05 kind::i8, exact int32 accumulators)
// over integer slices, recombined in f64:
//   X^ = s_a * code_x exactly (act codes, |code| <= 127);
//   What[j, c] = s_g(j) * u[j, c], u = clip(floor(w/s) + h) split into kOzSlices int8 slices
//     u = q0 + q1 2^-7 + q2 2^-14 + ...  (q0 = rint(u), later slices rint of the scaled residual,
//     |q_t| <= 64): the representation error is <= 2^-(7 kOzSlices - 6) absolute;
//   D'[:, j] = 2^E_j d, |d| < 1 (E_j from the column's max |D'|), d = sum_t r_t 2^(-6 - 7t).
// Each slice product is exact (|acc| < 2^31 for k <= 132K act columns / 264K batch rows), the
// group scales (outlier / normal) ride in K2's dual-slab f64 epilogue, and the slices are summed
// smallest first in K2's epilogue (qarvd_dual_gemm_f64_slices: the slices of one product are
// consecutive output columns).  kOzSlices = 8 carries 7 + 7*7 = 56 bits of u and 6 + 7*7 = 55 bits
// of d: both f64 operands are represented exactly, so the products are exact integer sums and
// the only roundings are the f64 epilogue's (scale products and the slice sum) -- tighter than
// the reference's own f64 matmul.
constexpr int kOzSlices = 8;

// the samples stacked into one group: stacked rows [off[j], off[j+1]) are rows [src[j], ...) of
// the sample arrays; coef[j] = 2 w_j / B, the gradient's row scale of sample j
struct GroupRows {
  int64_t off[kMaxGroup + 1];
  int64_t src[kMaxGroup];
  double coef[kMaxGroup];
  int count;
};
__device__ __forceinline__ int group_of(const GroupRows& g, int64_t r) {
  int j = 0;
  while (j + 1 < g.count && r >= g.off[j + 1]) ++j;
  return j;
}

// clamp(rint(x / s)) (quant.cpp:132-135) without a division on the common path: t = x * (1/s) is
// within |x/s| 2^-52 < 2^-37 of x / s while |t| <= qmax + 1 <= 2^15 (beyond that every path clamps
// to the same code, so t is clamped there first), so rint(t) is the reference's code unless t is
// within 2^-30 of a rounding boundary, where the exact quotient decides
__device__ __forceinline__ int act_code(double xv, double rinv, double s, int qmax, double lim) {
  double t = xv * rinv;
  t = t > lim ? lim : (t < -lim ? -lim : t);
  const double qm = t + kRoundMagic;
  int q = __double2loint(qm);
  if (fabs(t - (qm - kRoundMagic)) > 0.5 - 0x1p-30) q = __double2int_rn(__ddiv_rn(xv, s));
  return max(-qmax, min(qmax, q));
}

// the act codes of a whole group in one pass over 64 x 64 tiles: cx [stacked rows x ldq] in the
// K2 column order (GEMM1's A operand) and, when bt != NULL, the transpose bt[pos[c] * kb + row]
// (GEMM2's B operand, K-major over the stacked rows; rows in [rows_g, kb) are zero)
__global__ void __launch_bounds__(256) act_codes_group_kernel(const double* __restrict__ x, int64_t k, GroupRows g,
                                                               int64_t rows_g, int64_t kb, const int32_t* pos,
                                                               int64_t ldq, const double* log_sa, int qmax,
                                                               int8_t* __restrict__ cx, int8_t* __restrict__ bt,
                                                               int* bad) {
  __shared__ int8_t tile[64][64 + 4];
  __shared__ double s_sr[2];  // s = exp(log s_a) and 1 / s, once per CTA (glibc exp restated)
  if (threadIdx.x == 64) {
    const double sv = libm::exp(*log_sa);
    s_sr[0] = sv;
    s_sr[1] = 1.0 / sv;
  }
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 64, c0 = static_cast<int64_t>(blockIdx.x) * 64;
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  __shared__ const double* rowp[64];  // source row of each tile row (NULL past the group)
  if (threadIdx.x < 64) {
    const int64_t row = r0 + threadIdx.x;
    const double* p = nullptr;
    if (row < rows_g) {
      const int j = group_of(g, row);
      p = x + (g.src[j] + row - g.off[j]) * k;
    }
    rowp[threadIdx.x] = p;
  }
  __syncthreads();
  const double s = s_sr[0], rinv = s_sr[1];
  const double lim = static_cast<double>(qmax) + 1.0;
  const int64_t c = c0 + tx;
  const bool col_ok = c < k;
  double xv[16];  // all 16 loads in flight before any store
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const double* p = rowp[ty + 4 * u];
    xv[u] = (p && col_ok) ? p[c] : 0.0;
  }
  bool finite = true;
  int8_t* cxc = cx + (col_ok ? pos[c] : 0) + (r0 + ty) * ldq;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int rr = ty + 4 * u;
    int q = 0;
    if (rowp[rr] && col_ok) {
      if (isfinite(xv[u])) q = act_code(xv[u], rinv, s, qmax, lim);
      else finite = false;
      cxc[4 * u * ldq] = static_cast<int8_t>(q);
    }
    tile[rr][tx] = static_cast<int8_t>(q);
  }
  if (!finite) *bad = 1;
  if (!bt) return;
  __syncthreads();
  for (int it = threadIdx.x; it < 64 * 16; it += 256) {  // 4 consecutive rows per store
    const int cc = it >> 4, rg = (it & 15) * 4;
    const int64_t c = c0 + cc, row = r0 + rg;
    if (c >= k || row >= kb) continue;  // kb % 32 == 0: all four rows are < kb
    const uint32_t w = static_cast<uint8_t>(tile[rg][cc]) | static_cast<uint32_t>(static_cast<uint8_t>(tile[rg + 1][cc])) << 8 |
                       static_cast<uint32_t>(static_cast<uint8_t>(tile[rg + 2][cc])) << 16 |
                       static_cast<uint32_t>(static_cast<uint8_t>(tile[rg + 3][cc])) << 24;
    *reinterpret_cast<uint32_t*>(bt + static_cast<int64_t>(pos[c]) * kb + row) = w;
  }
}

// D_b = P_b - T_b over a whole group (calibrate.cpp:279-280): per (sample, row chunk, column
// block) CTA the partial ||D||^2 -> partial[j * per + chunk * gridDim.x + blockIdx.x] (fixed
// order); with grads, D is rescaled in place to D' = coef_j D and the column maxima |D'| are
// folded into cmax (as bits: non-negative doubles order like their bit patterns).  Two adjacent
// columns per thread (n even) so rows are read as 16-byte pairs.
__global__ void __launch_bounds__(kT) resid_kernel(double* __restrict__ d, const double* __restrict__ target,
                                                    int64_t n, GroupRows g,
                                                    int chunks, int grads, double* partial, int per,
                                                    unsigned long long* cmax) {
  const int j = blockIdx.y / chunks, ch = blockIdx.y - j * chunks;
  const int64_t rows = g.off[j + 1] - g.off[j];
  const int64_t per_ch = (rows + chunks - 1) / chunks;
  const int64_t lo = ch * per_ch, hi = lo + per_ch < rows ? lo + per_ch : rows;
  const int64_t c = 2 * (static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x);
  const double coef = g.coef[j];
  double a0 = 0.0, a1 = 0.0, m0 = 0.0, m1 = 0.0;
  if (c < n) {
    const bool two = c + 1 < n;
    double* dp = d + (g.off[j] + lo) * n + c;
    const double* tp = target + (g.src[j] + lo) * n + c;
    if ((n & 1) == 0) {
#pragma unroll 4
      for (int64_t r = lo; r < hi; ++r, dp += n, tp += n) {
        const double2 pv = *reinterpret_cast<const double2*>(dp);
        const double2 tv = *reinterpret_cast<const double2*>(tp);
        const double v0 = pv.x - tv.x, v1 = pv.y - tv.y;
        a0 += v0 * v0;
        a1 += v1 * v1;
        if (grads) {
          const double e0 = v0 * coef, e1 = v1 * coef;
          *reinterpret_cast<double2*>(dp) = make_double2(e0, e1);
          m0 = fmax(m0, fabs(e0));
          m1 = fmax(m1, fabs(e1));
        }
      }
    } else {
      for (int64_t r = lo; r < hi; ++r, dp += n, tp += n) {
        const double v0 = dp[0] - tp[0], v1 = two ? dp[1] - tp[1] : 0.0;
        a0 += v0 * v0;
        a1 += v1 * v1;
        if (grads) {
          dp[0] = v0 * coef;
          m0 = fmax(m0, fabs(v0 * coef));
          if (two) {
            dp[1] = v1 * coef;
            m1 = fmax(m1, fabs(v1 * coef));
          }
        }
      }
    }
    if (grads && cmax) {
      atomicMax(cmax + c, static_cast<unsigned long long>(__double_as_longlong(m0)));
      if (two) atomicMax(cmax + c + 1, static_cast<unsigned long long>(__double_as_longlong(m1)));
    }
  }
  const double t = block_sum(a0 + a1);
  if (threadIdx.x == 0) partial[j * per + ch * gridDim.x + blockIdx.x] = t;
}

// the slices of u = What / s_g (the clipped soft code) in the K2 layout: slice t of row r at row
// r * kOzSlices + t
__global__ void w_slices_kernel(const double* code, int64_t n, int64_t k, const int32_t* pos, int64_t ldq,
                                int8_t* wsl) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n * k;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / k, c = i - r * k;
    double rem = code[i];
    int8_t* out = wsl + (r * kOzSlices) * ldq + pos[c];
#pragma unroll
    for (int t = 0; t < kOzSlices; ++t) {
      if (t > 0) rem *= 128.0;  // exact; |rem| <= 0.5 before the scaling
      const double qm = rem + kRoundMagic;
      out[t * ldq] = static_cast<int8_t>(__double2loint(qm));
      rem -= qm - kRoundMagic;  // exact
    }
  }
}

// per-run scales of the forward product: so / sn of row j = s_g(j) (slice t's 2^-7t is applied
// by the GEMM epilogue), and the act scale per stacked row
__global__ void oz_scales_kernel(const double* log_s, int64_t n, int enabled, const double* log_sa,
                                 int64_t rows, double* so_sl, double* sn_sl, double* sx_rows) {
  const double sa = libm::exp(*log_sa);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n || i < rows;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (i < n) {
      sn_sl[i] = libm::exp(log_s[i]);
      so_sl[i] = libm::exp(enabled ? log_s[n + i] : log_s[i]);
    }
    if (i < rows) sx_rows[i] = sa;
  }
}

// D' slices transposed for the gradient product: B[(j kOzSlices + t), i] = r_t(i, j) (K-major over
// the batch rows).  Tiles of 128 rows x 32 columns through shared memory: the loads are 256-byte
// row segments (lane = column), the stores 128-byte runs of one (column, slice) row (4 rows per
// lane); the column's 2^-E_j is formed once per thread.
constexpr int kDsRows = 128;
__global__ void __launch_bounds__(256) d_slices_t_kernel(const double* d, int64_t rows, int64_t n,
                                                         const unsigned long long* mx, int64_t lda, int8_t* a) {
  __shared__ __align__(4) int8_t tile[kOzSlices][32][kDsRows + 4];
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * kDsRows, j0 = static_cast<int64_t>(blockIdx.y) * 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;  // 8 warps x 16 rows
  const int64_t j = j0 + lane;
  double f = 0.0;  // 2^-E_j: m in [2^(E-1), 2^E), so D' f is in (-1, 1)
  if (j < n) {
    const double m = __longlong_as_double(static_cast<long long>(mx[j]));
    int e = 0;
    if (m > 0.0) {
      frexp(m, &e);
      f = ldexp(1.0, -e);
    }
  }
  double dv[kDsRows / 8];  // the warp's 16 rows, all loads in flight first
#pragma unroll
  for (int u = 0; u < kDsRows / 8; ++u) {
    const int64_t i = i0 + warp + 8 * u;
    dv[u] = (i < rows && j < n) ? d[i * n + j] : 0.0;
  }
#pragma unroll
  for (int u = 0; u < kDsRows / 8; ++u) {
    const int r = warp + 8 * u;
    double rem = dv[u] * f * 64.0;
#pragma unroll
    for (int t = 0; t < kOzSlices; ++t) {
      if (t > 0) rem *= 128.0;
      const double qm = rem + kRoundMagic;  // rint(rem) in the low word, no conversion unit
      tile[t][lane][r] = static_cast<int8_t>(__double2loint(qm));
      rem -= qm - kRoundMagic;
    }
  }
  __syncthreads();
  // lda % 32 == 0 and i0 % 128 == 0: a lane's 4 rows are all inside or all outside [0, lda)
  const int64_t i = i0 + 4 * lane;
  if (i >= lda) return;
  for (int p = warp; p < 32 * kOzSlices; p += 8) {
    const int jj = p / kOzSlices, t = p - jj * kOzSlices;
    if (j0 + jj >= n) break;
    *reinterpret_cast<uint32_t*>(a + ((j0 + jj) * kOzSlices + t) * lda + i) =
        *reinterpret_cast<const uint32_t*>(&tile[t][jj][4 * lane]);
  }
}

// the gradient product's per-run column scales 2^(E_j - 6) (slice t's 2^-7t is applied by the
// GEMM epilogue) and its row scale s_a (rows: the act columns)
__global__ void oz_grad_scales_kernel(const unsigned long long* mx, int64_t n, const double* log_sa, int64_t kp,
                                      double* scol, double* srow) {
  const double sa = libm::exp(*log_sa);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n || i < kp;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (i < n) {
      const double m = __longlong_as_double(static_cast<long long>(mx[i]));
      int e = 0;
      if (m > 0.0) frexp(m, &e);
      scol[i] = m > 0.0 ? ldexp(1.0, e - 6) : 0.0;
    }
    if (i < kp) srow[i] = sa;
  }
}

// gw[j, c] (+)= Gt[pos[c], j]: the slice-summed product back to [n x k], original column order
__global__ void oz_combine_grad_kernel(const double* gt, int64_t n, int64_t k, const int32_t* pos,
                                       int accumulate, double* gw) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n * k;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = i / k, c = i - j * k;
    const double v = gt[static_cast<int64_t>(pos[c]) * n + j];
    gw[i] = accumulate ? gw[i] + v : v;
  }
}

struct DevArena {
  std::vector<void*> ptrs;
  cudaStream_t s;
  explicit DevArena(cudaStream_t st) : s(st) {}
  ~DevArena() {
    for (void* p : ptrs) cudaFreeAsync(p, s);
  }
  template <typename T>
  T* get(int64_t count) {
    void* p = nullptr;
    if (cudaMallocAsync(&p, static_cast<size_t>(count > 0 ? count : 1) * sizeof(T), s) != cudaSuccess)
      return nullptr;
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
};

}  // namespace
}  // namespace qarvd_b200

using namespace qarvd_b200;

extern "C" int qarvd_calibrate_layer(const double* w, int64_t n, int64_t k, const uint8_t* outlier_mask,
                                     int plan_enabled, const double* scale_normal_init,
                                     const double* scale_outlier_init, double act_scale_init,
                                     int act_bits, int w_bits, const double* x,
                                     const int64_t* sample_rows, const int64_t* sample_chunk,
                                     int64_t n_samples, const double* chunk_weights, int64_t n_chunks,
                                     const qarvd_calib_config* cfg, const char* layer_name,
                                     int8_t* codes, double* scale_normal_out, double* scale_outlier_out,
                                     double* scalars_out, double* trace_out, void* stream) {
  clear_error();
  if (!cfg) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "calib config: null");
  // CalibConfig::validate (calibrate.cpp:45-52)
  if (cfg->iterations < 0) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "calib config: iterations must be >= 0");
  if (cfg->batch_size < 1) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "calib config: batch size must be >= 1");
  if (!(cfg->lr_round > 0.0) || !(cfg->lr_scale > 0.0))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "calib config: learning rates must be positive");
  if (!(cfg->zeta > 1.0) || !(cfg->gamma_lo < 0.0))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "calib config: rectified sigmoid needs zeta > 1 > 0 > gamma");
  if (n_samples <= 0) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "calibrate_layer: no calibration samples");
  if (n <= 0 || k <= 0 || !w || !x || !outlier_mask || !scale_normal_init || !sample_rows ||
      !sample_chunk || !chunk_weights || !codes || !scale_normal_out || !scale_outlier_out ||
      !scalars_out || (plan_enabled && !scale_outlier_init))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "calibrate_layer: null pointer or empty shape");
  if (act_bits < 2 || act_bits > 8 || w_bits < 2 || w_bits > 8)
    QARVD_FAIL(QARVD_ERR_UNSUPPORTED, "calibrate_layer: bit widths outside [2, 8]");
  if (!(act_scale_init > 0.0) || !std::isfinite(act_scale_init))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "quant params: scale must be positive and finite");
  for (int64_t s = 0; s < n_samples; ++s) {
    if (sample_rows[s + 1] <= sample_rows[s])
      QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "calibrate_layer: empty or unordered sample rows");
    if (sample_chunk[s] < 1 || sample_chunk[s] > n_chunks)
      QARVD_FAIL(QARVD_ERR_OUT_OF_RANGE, "weighted loss: sample chunk outside the weight vector");
  }
  if (sample_rows[0] != 0) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "calibrate_layer: sample rows must start at 0");
  if (int st = require_device()) return st;
  cudaStream_t s = as_stream(stream);

  // cuBLAS handles are bound to the device current at creation: one per (thread, device)
  static thread_local std::map<int, cublasHandle_t> handles;
  int dev = 0;
  QARVD_CUDA_TRY(cudaGetDevice(&dev));
  cublasHandle_t& handle = handles[dev];
  if (!handle) QARVD_CUBLAS_TRY(cublasCreate(&handle));
  QARVD_CUBLAS_TRY(cublasSetStream(handle, s));
  QARVD_CUBLAS_TRY(cublasSetPointerMode(handle, CUBLAS_POINTER_MODE_HOST));

  const int64_t nk = n * k, m_all = sample_rows[n_samples];
  int64_t max_rows = 0;
  for (int64_t i = 0; i < n_samples; ++i) {
    const int64_t r = sample_rows[i + 1] - sample_rows[i];
    max_rows = r > max_rows ? r : max_rows;
  }
  const int wq_max = (1 << (w_bits - 1)) - 1, aq_max = (1 << (act_bits - 1)) - 1;
  const double zeta = cfg->zeta, gamma = cfg->gamma_lo;

  DevArena A(s);
  double* v = A.get<double>(nk);
  double* mv = A.get<double>(nk);
  double* vv = A.get<double>(nk);
  double* what = A.get<double>(nk);
  double* code = A.get<double>(nk);
  double* dhdv = A.get<double>(nk);
  double* gw = A.get<double>(nk);
  double* log_s = A.get<double>(2 * n);
  double* ms = A.get<double>(2 * n);
  double* vs = A.get<double>(2 * n);
  double* sgrad = A.get<double>(2 * n);
  double* target = A.get<double>(m_all * n);
  // samples are stacked G at a time (rows <= cap_rows) so each product is one GEMM
  const int64_t G = cfg->batch_size < kMaxGroup ? cfg->batch_size : kMaxGroup;
  const int64_t cap_rows = G * max_rows;
  double* d = A.get<double>(cap_rows * n);
  // per-iteration products on the int8 tensor cores (QARVD_K7_OZAKI=0: cuBLAS DGEMM, A/B)
  // the slice products stack kOzSlices = 8 digit rows per output row: K2 needs 8n % 16 == 0, so
  // an odd out_dim takes the DGEMM path
  const bool ozaki = !(getenv("QARVD_K7_OZAKI") && getenv("QARVD_K7_OZAKI")[0] == '0') && (n % 2 == 0);
  double* xhat = ozaki ? nullptr : A.get<double>(cap_rows * k);
  // K2 layout of the plan: [outlier columns | pad to 32 | normal columns | pad to 32]
  std::vector<int32_t> pos_h(static_cast<size_t>(k));
  int64_t k_o_pad = 0, k_pad = 0;
  {
    std::vector<uint8_t> mask_h(static_cast<size_t>(k));
    QARVD_CUDA_TRY(cudaMemcpyAsync(mask_h.data(), outlier_mask, static_cast<size_t>(k), cudaMemcpyDeviceToHost, s));
    QARVD_CUDA_TRY(cudaStreamSynchronize(s));
    int64_t no = 0;
    for (int64_t c = 0; c < k; ++c) no += (plan_enabled && mask_h[c]) ? 1 : 0;
    k_o_pad = (no + 31) / 32 * 32;
    k_pad = k_o_pad + (k - no + 31) / 32 * 32;
    int64_t io = 0, in = 0;
    for (int64_t c = 0; c < k; ++c)
      pos_h[c] = static_cast<int32_t>((plan_enabled && mask_h[c]) ? io++ : k_o_pad + in++);
  }
  const int64_t tn = kOzSlices * n, kb_cap = (cap_rows + 31) / 32 * 32;
  int32_t* ozpos = ozaki ? A.get<int32_t>(k) : nullptr;
  int8_t* cx = ozaki ? A.get<int8_t>(kb_cap * k_pad) : nullptr;
  int8_t* wsl = ozaki ? A.get<int8_t>(tn * k_pad) : nullptr;
  double* so_sl = ozaki ? A.get<double>(tn) : nullptr;
  double* sn_sl = ozaki ? A.get<double>(tn) : nullptr;
  double* sx_rows = ozaki ? A.get<double>(kb_cap) : nullptr;
  unsigned long long* cmax = ozaki ? A.get<unsigned long long>(n) : nullptr;
  int8_t* amat = ozaki ? A.get<int8_t>(tn * kb_cap) : nullptr;
  int8_t* bmat = ozaki ? A.get<int8_t>(k_pad * kb_cap) : nullptr;
  double* sx_a = ozaki ? A.get<double>(tn) : nullptr;
  double* srow_a = ozaki ? A.get<double>(k_pad) : nullptr;
  double* gsl = ozaki ? A.get<double>(k_pad * n) : nullptr;
  if (ozaki && (!ozpos || !cx || !wsl || !so_sl || !sn_sl || !sx_rows || !cmax || !amat || !bmat || !sx_a ||
                !srow_a || !gsl))
    QARVD_FAIL(QARVD_ERR_CUDA, "calibrate_layer: device allocation failed");
  if (ozaki) {
    QARVD_CUDA_TRY(cudaMemcpyAsync(ozpos, pos_h.data(), static_cast<size_t>(k) * 4, cudaMemcpyHostToDevice, s));
    QARVD_CUDA_TRY(cudaMemsetAsync(cx, 0, static_cast<size_t>(kb_cap * k_pad), s));   // pad columns stay 0
    QARVD_CUDA_TRY(cudaMemsetAsync(wsl, 0, static_cast<size_t>(tn * k_pad), s));
    QARVD_CUDA_TRY(cudaMemsetAsync(bmat, 0, static_cast<size_t>(k_pad * kb_cap), s));  // pad rows stay 0
  }
  double* partial = A.get<double>(kMaxGroup * kRedBlocks);
  // scalars: [0] log_sa [1] m_a [2] v_a [3] g_a [4] loss acc [5] best
  double* sc = A.get<double>(8);
  int* flags = A.get<int>(2);  // [0] diverged_at, [1] non-finite input
  if (!v || !mv || !vv || !what || !code || !dhdv || !gw || !log_s || !ms || !vs || !sgrad || !target ||
      !d || (!ozaki && !xhat) || !partial || !sc || !flags)
    QARVD_FAIL(QARVD_ERR_CUDA, "calibrate_layer: device allocation failed");
  QARVD_CUDA_TRY(cudaMemsetAsync(mv, 0, nk * 8, s));
  QARVD_CUDA_TRY(cudaMemsetAsync(vv, 0, nk * 8, s));
  QARVD_CUDA_TRY(cudaMemsetAsync(ms, 0, 2 * n * 8, s));
  QARVD_CUDA_TRY(cudaMemsetAsync(vs, 0, 2 * n * 8, s));
  QARVD_CUDA_TRY(cudaMemsetAsync(sc, 0, 8 * 8, s));
  set_scalars_kernel<<<1, 1, 0, s>>>(sc + 0, act_scale_init, sc + 5, flags, flags + 1);
  // LearnableQuantState::init (calibrate.cpp:77-115)
  const double* s_o_init = plan_enabled ? scale_outlier_init : scale_normal_init;
  log_kernel<<<blocks_for(n), kT, 0, s>>>(scale_normal_init, log_s, n);
  log_kernel<<<blocks_for(n), kT, 0, s>>>(s_o_init, log_s + n, n);
  init_v_kernel<<<blocks_for(nk), kT, 0, s>>>(w, outlier_mask, plan_enabled, scale_normal_init, s_o_init,
                                             n, k, zeta, gamma, v);
  count_launch(4);
  QARVD_LAUNCH_CHECK();
  // targets X_s W^T for every sample, once (row-major [rows x n] = col-major W^T-op GEMM)
  const double one = 1.0, zero = 0.0;
  QARVD_CUBLAS_TRY(cublasDgemm(handle, CUBLAS_OP_T, CUBLAS_OP_N, static_cast<int>(n), static_cast<int>(m_all),
                               static_cast<int>(k), &one, w, static_cast<int>(k), x, static_cast<int>(k), &zero,
                               target, static_cast<int>(n)));

  std::vector<double> wsamp(static_cast<size_t>(n_samples));
  for (int64_t i = 0; i < n_samples; ++i) wsamp[i] = chunk_weights[sample_chunk[i] - 1];

  // one pass of the objective over `list` with the current weights in `what`:
  // sc[4] = sum_b w_b ||D_b||^2; with grads: gw = sum_b coeff_b D_b^T X^_b, sc[3] = act-scale
  // grad.  Up to G consecutive samples are stacked along the rows, so D = X^ What^T - T and
  // dL/dWhat = D'^T X^ are one GEMM each per group, with D' = coeff_b D_b (rows rescaled in
  // place once ||D_b||^2 is read).
  auto objective = [&](const std::vector<int64_t>& list, bool grads) -> int {
    const double inv_b = 1.0 / static_cast<double>(list.size());
    size_t pos = 0;
    for (int gi = 0; pos < list.size(); ++gi) {
      size_t end = pos;
      int64_t rows_g = 0;
      while (end < list.size() && static_cast<int64_t>(end - pos) < G) {
        const int64_t r = sample_rows[list[end] + 1] - sample_rows[list[end]];
        if (rows_g + r > cap_rows) break;
        rows_g += r;
        ++end;
      }
      GroupWeights wl{};
      GroupRows gr{};
      gr.count = static_cast<int>(end - pos);
      for (size_t j = pos; j < end; ++j) {
        const int64_t si = list[j], jj = static_cast<int64_t>(j - pos);
        gr.src[jj] = sample_rows[si];
        gr.off[jj + 1] = gr.off[jj] + sample_rows[si + 1] - sample_rows[si];
        gr.coef[jj] = 2.0 * wsamp[si] * inv_b;
        wl.w[jj] = wsamp[si];
      }
      const int64_t kb = (rows_g + 31) / 32 * 32;
      if (ozaki) {
        // P = s_a code_x . What^T as kOzSlices exact int8 products (K2, f64 epilogue carries the
        // group scales and the slice weights), summed smallest slice first; the act codes of
        // the whole group in one pass, with their transpose for the gradient product
        act_codes_group_kernel<<<dim3(static_cast<unsigned>((k + 63) / 64),
                                      static_cast<unsigned>(((grads ? kb : rows_g) + 63) / 64)),
                                 256, 0, s>>>(x, k, gr, rows_g, kb, ozpos, k_pad, sc + 0, aq_max, cx,
                                              grads ? bmat : nullptr, flags + 1);
        oz_scales_kernel<<<blocks_for(tn > rows_g ? tn : rows_g), kT, 0, s>>>(log_s, n, plan_enabled, sc + 0, rows_g,
                                                                           so_sl, sn_sl, sx_rows);
        count_launch(2);
        if (int st = qarvd_dual_gemm_f64_slices(cx, k_pad, wsl, k_pad, rows_g, tn, k_pad, k_o_pad, sx_rows, so_sl,
                                                sn_sl, kOzSlices, d, n, s))
          return st;
      } else {
        for (size_t j = pos, off = 0; j < end; ++j) {
          const int64_t si = list[j], r0 = sample_rows[si], rows = sample_rows[si + 1] - r0;
          xhat_kernel<<<blocks_for(rows * k), kT, 0, s>>>(x + r0 * k, rows * k, sc + 0, aq_max, xhat + off * k,
                                                         flags + 1);
          off += rows;
        }
        // P = X^ What^T   [rows_g x n]; D = P - T is formed by the reduction below
        QARVD_CUBLAS_TRY(cublasDgemm(handle, CUBLAS_OP_T, CUBLAS_OP_N, static_cast<int>(n), static_cast<int>(rows_g),
                                     static_cast<int>(k), &one, what, static_cast<int>(k), xhat,
                                     static_cast<int>(k), &zero, d, static_cast<int>(n)));
      }
      // D_b = P_b - T_b (calibrate.cpp:279-280), ||D_b||^2, and D_b *= coeff_b for the gradient
      // (with the column maxima of D' for its slices), one pass over the group
      const bool colmax = grads && ozaki;
      if (colmax) QARVD_CUDA_TRY(cudaMemsetAsync(cmax, 0, static_cast<size_t>(n) * 8, s));
      const int gx = static_cast<int>((n + 2 * kT - 1) / (2 * kT));
      const int chunks = std::max(1, kRedBlocks / gx);
      resid_kernel<<<dim3(static_cast<unsigned>(gx), static_cast<unsigned>(chunks * gr.count)), kT, 0, s>>>(
          d, target, n, gr, chunks, grads ? 1 : 0, partial, chunks * gx, colmax ? cmax : nullptr);
      dot_final_kernel<<<1, kMaxGroup * 32, 0, s>>>(partial, gr.count, wl, nullptr, gi > 0, sc + 4, chunks * gx);
      count_launch(2);
      if (grads && ozaki) {
        // dL/dWhat (+)= D'^T X^ = s_a D'^T code_x: D' split per column (2^E_j x int8 slices, K-major
        // over the batch rows), code_x^T from the act-code pass, one K2 over all slices,
        // recombined per column
        d_slices_t_kernel<<<dim3(static_cast<unsigned>((kb + kDsRows - 1) / kDsRows), static_cast<unsigned>((n + 31) / 32)), 256, 0, s>>>(
            d, rows_g, n, cmax, kb, amat);
        oz_grad_scales_kernel<<<blocks_for(tn > k_pad ? tn : k_pad), kT, 0, s>>>(cmax, n, sc + 0, k_pad, sx_a, srow_a);
        count_launch(2);
        // Gt [k_pad x n] = s_a code_x^T . D' (act columns as rows, the D' slices as columns)
        if (int st = qarvd_dual_gemm_f64_slices(bmat, kb, amat, kb, k_pad, tn, kb, 0, srow_a, nullptr, sx_a,
                                                kOzSlices, gsl, n, s))
          return st;
        oz_combine_grad_kernel<<<blocks_for(nk), kT, 0, s>>>(gsl, n, k, ozpos, gi > 0 ? 1 : 0, gw);
        count_launch(1);
      } else if (grads) {
        // dL/dWhat (+)= D'^T X^   [n x k]
        QARVD_CUBLAS_TRY(cublasDgemm(handle, CUBLAS_OP_N, CUBLAS_OP_T, static_cast<int>(k), static_cast<int>(n),
                                     static_cast<int>(rows_g), &one, xhat, static_cast<int>(k), d,
                                     static_cast<int>(n), gi > 0 ? &one : &zero, gw, static_cast<int>(k)));
        count_launch(1);
      }
      pos = end;
    }
    if (grads && cfg->train_activation_scale) {
      // act-scale grad sum_b coeff_b sum (D_b What) * s_a * code_x (calibrate.cpp:300-304)
      // = <What, sum_b coeff_b D_b^T X^_b> = <What, gw>, since X^ = s_a code_x: the dL/dX^
      // product is never formed
      GroupWeights unit{};
      unit.w[0] = 1.0;
      dot_partial_kernel<<<kRedBlocks, kT, 0, s>>>(what, gw, nk, 0, 0.0, partial);
      dot_final_kernel<<<1, kMaxGroup * 32, 0, s>>>(partial, 1, unit, nullptr, 0, sc + 3);
      count_launch(2);
    }
    QARVD_LAUNCH_CHECK();
    return QARVD_OK;
  };
  std::vector<int64_t> all(static_cast<size_t>(n_samples));
  for (int64_t i = 0; i < n_samples; ++i) all[i] = i;

  // initial hard loss (calibrate.cpp:320)
  // the int8 slices of the clipped codes that What = s_g * code is built from (Ozaki products)
  auto slice_weights = [&]() {
    if (!ozaki) return;
    w_slices_kernel<<<blocks_for(nk), kT, 0, s>>>(code, n, k, ozpos, k_pad, wsl);
    count_launch();
  };
  weights_kernel<<<static_cast<unsigned>(n), kT, 0, s>>>(w, v, outlier_mask, plan_enabled, log_s, n, k, zeta, gamma,
                                              -wq_max, wq_max, 1, what, ozaki ? code : nullptr, nullptr, nullptr);
  count_launch();
  slice_weights();
  if (int st = objective(all, false)) return st;
  loss_kernel<<<1, 1, 0, s>>>(sc + 4, 1.0 / static_cast<double>(n_samples), scalars_out + 1);  // initial
  count_launch();

  uint64_t st_rng = mix_seed_h(cfg->seed, fnv1a_h(layer_name ? layer_name : "", layer_name ? std::strlen(layer_name) : 0));
  const int iters = cfg->iterations;
  const int warmup = static_cast<int>(cfg->warmup_frac * static_cast<double>(iters));
  std::vector<int64_t> batch(static_cast<size_t>(cfg->batch_size));
  for (int t = 0; t < iters; ++t) {
    for (int b = 0; b < cfg->batch_size; ++b)
      batch[b] = static_cast<int64_t>(splitmix64_h(st_rng) % static_cast<uint64_t>(n_samples));
    weights_kernel<<<static_cast<unsigned>(n), kT, 0, s>>>(w, v, outlier_mask, plan_enabled, log_s, n, k, zeta, gamma,
                                                -wq_max, wq_max, 0, what, code, dhdv, nullptr);
    count_launch();
    slice_weights();
    if (int st = objective(batch, true)) return st;
    trace_kernel<<<1, 1, 0, s>>>(sc + 4, 1.0 / static_cast<double>(batch.size()), sc + 5,
                                 trace_out ? trace_out : sc + 7, trace_out ? t : 0, flags);
    const bool reg_on = t >= warmup && cfg->reg_lambda > 0.0;
    const double frac = iters > 1 ? static_cast<double>(t) / static_cast<double>(iters - 1) : 1.0;
    const double beta = cfg->beta_start + (cfg->beta_end - cfg->beta_start) * frac;
    grad_kernel<<<static_cast<unsigned>(n), kT, 0, s>>>(gw, v, code, dhdv, outlier_mask, plan_enabled, log_s,
                                                       n, k, reg_on ? 1 : 0, cfg->reg_lambda, beta, zeta,
                                                       gamma, gw, sgrad);
    const double anneal = 0.5 * (1.0 + std::cos(M_PI * static_cast<double>(t) / static_cast<double>(iters)));
    const double c1 = 1.0 - std::pow(0.9, t + 1), c2 = 1.0 - std::pow(0.999, t + 1);
    adam_kernel<<<blocks_for(nk), kT, 0, s>>>(v, gw, mv, vv, nk, cfg->lr_round * anneal, c1, c2);
    adam_kernel<<<blocks_for(2 * n), kT, 0, s>>>(log_s, sgrad, ms, vs, 2 * n, cfg->lr_scale * anneal, c1, c2);
    if (cfg->train_activation_scale)
      adam_kernel<<<1, 32, 0, s>>>(sc + 0, sc + 3, sc + 1, sc + 2, 1, cfg->lr_scale * anneal, c1, c2);
    count_launch(5);
    QARVD_LAUNCH_CHECK();
  }

  // final hard loss, hard codes, learned scales and act scale (calibrate.cpp:391-395)
  weights_kernel<<<static_cast<unsigned>(n), kT, 0, s>>>(w, v, outlier_mask, plan_enabled, log_s, n, k, zeta, gamma,
                                              -wq_max, wq_max, 1, what, ozaki ? code : nullptr, nullptr, codes);
  count_launch();
  slice_weights();
  if (int st = objective(all, false)) return st;
  loss_kernel<<<1, 1, 0, s>>>(sc + 4, 1.0 / static_cast<double>(n_samples), scalars_out + 2);  // final
  exp_kernel<<<blocks_for(n), kT, 0, s>>>(log_s, scale_normal_out, n);
  exp_kernel<<<blocks_for(n), kT, 0, s>>>(log_s + n, scale_outlier_out, n);
  exp_kernel<<<1, 32, 0, s>>>(sc + 0, scalars_out, 1);  // scalars_out[0] = act scale
  count_launch(4);
  QARVD_LAUNCH_CHECK();
  int fl[2] = {0, 0};
  QARVD_CUDA_TRY(cudaMemcpyAsync(fl, flags, sizeof(fl), cudaMemcpyDeviceToHost, s));
  QARVD_CUDA_TRY(cudaStreamSynchronize(s));
  if (fl[1]) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "quantize: non-finite input");
  if (fl[0] >= 0)
    QARVD_FAIL(QARVD_ERR_RUNTIME, "calibration diverged for layer " + std::string(layer_name ? layer_name : "") +
                                      " at iteration " + std::to_string(fl[0]));
  return QARVD_OK;
}

extern "C" int qarvd_adaround_weights(const double* w, const double* v, const uint8_t* outlier_mask,
                                      int plan_enabled, const double* log_scale, int64_t n, int64_t k,
                                      double zeta, double gamma_lo, int w_bits, int hard, double* what,
                                      int8_t* codes, void* stream) {
  clear_error();
  if (n < 0 || k < 0 || w_bits < 2 || w_bits > 8 || (n * k > 0 && (!w || !v || !outlier_mask || !log_scale)))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "qarvd_adaround_weights: invalid argument");
  if (int st = require_device()) return st;
  if (n * k == 0) return QARVD_OK;
  double* scratch = nullptr;
  cudaStream_t s = as_stream(stream);
  if (!what) {
    QARVD_CUDA_TRY(cudaMallocAsync(&scratch, static_cast<size_t>(n * k) * sizeof(double), s));
    what = scratch;
  }
  const int qmax = (1 << (w_bits - 1)) - 1;
  weights_kernel<<<static_cast<unsigned>(n), kT, 0, s>>>(w, v, outlier_mask, plan_enabled, log_scale, n, k, zeta, gamma_lo,
                                                  -qmax, qmax, hard ? 1 : 0, what, nullptr, nullptr, codes);
  count_launch();
  if (scratch) cudaFreeAsync(scratch, s);
  QARVD_LAUNCH_CHECK();
  return QARVD_OK;
}
