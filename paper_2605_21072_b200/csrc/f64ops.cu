// Exact f64 restatements, on the device, of the reference's generic operators that sit next to
// the hot path and that the C++ drop-in (adapter/qarvd_cuda.cpp) must serve without the
// reference's CPU code:
//
//   qarvd_quantize_f64          quantize / dequantize / fake_quant   quant.cpp:113-159
//   qarvd_minmax_scale_f64      init_scale_minmax                    quant.cpp:161-183
//   qarvd_percentile_search_f64 init_scale_percentile_search         quant.cpp:20-28, :185-226
//   qarvd_matmul_nt_f64         matmul_nt (k-ascending, no FMA)      tensor.cpp:82-105
//   qarvd_gather_columns        permute_activations / the pre-permute engine.cpp:36-44,
//                                                                    calibrate.cpp:474-480
//   qarvd_dequant_weight_f64    dequantized_weight_original_order    engine.cpp:117-130
//
// Every floating operation is the reference's operation with an explicit round-to-nearest
// intrinsic (the reference build has no FMA), so results are bit-identical to the f64 CPU code.
// The percentile search replaces the reference's full std::sort of the pooled |x| by an exact
// MSB-first radix select of only the order statistics the three quantiles need (|x| bit
// patterns order like the values), and its per-sample squared errors by double-double sums
// (the reference's sequential sum differs from the exact sum by its own rounding error only).
#include <climits>
#include <vector>

#include "common.cuh"
#include "crmath.cuh"
#include "libm_ref.cuh"

namespace qarvd_b200 {
namespace {

constexpr int kT = 256;
inline unsigned grid_for(int64_t n, int per_thread = 1) {
  const int64_t b = (n + static_cast<int64_t>(kT) * per_thread - 1) / (static_cast<int64_t>(kT) * per_thread);
  return static_cast<unsigned>(b < 1 ? 1 : (b > kNumSMs * 16 ? kNumSMs * 16 : b));
}

__global__ void set_i64_kernel(int64_t* p, int64_t v, int count) {
  if (threadIdx.x < count) p[threadIdx.x] = v;
}

// static_cast<int64_t>(double) as the reference's x86-64 build executes it (cvttsd2si): values
// outside the int64 range (and NaN) become INT64_MIN, which the clamp then sends to q_min.
__device__ __forceinline__ int64_t cvtt_i64(double t) {
  return (t > -9223372036854775808.0 && t < 9223372036854775808.0) ? static_cast<int64_t>(t)
                                                                   : INT64_MIN;
}

// quantize (quant.cpp:113-138): code = clamp(rhe(v / s) + z, q_min, q_max); round_half_even
// (quant.hpp:14-20) is rint in the default rounding mode; optional dequantize (:140-155).
__global__ void quantize_f64_kernel(const double* __restrict__ x, int64_t count, int64_t inner,
                                    int64_t extent, const double* __restrict__ scales,
                                    const int32_t* __restrict__ zps, int32_t q_min, int32_t q_max,
                                    int32_t* __restrict__ codes, double* __restrict__ deq,
                                    unsigned long long* err) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double v = x[i];
    if (!isfinite(v)) {
      atomicMin(err, static_cast<unsigned long long>(i));
      continue;
    }
    const int64_t ch = extent > 1 ? (i / inner) % extent : 0;
    const double s = scales[ch];
    const int64_t z = zps ? zps[ch] : 0;
    // + zero point with two's-complement wrap-around, as the x86-64 build executes it
    int64_t code = static_cast<int64_t>(static_cast<uint64_t>(cvtt_i64(rint(__ddiv_rn(v, s)))) +
                                        static_cast<uint64_t>(z));
    code = code < q_min ? q_min : (code > q_max ? q_max : code);
    if (codes) codes[i] = static_cast<int32_t>(code);
    if (deq) deq[i] = __dmul_rn(static_cast<double>(static_cast<int32_t>(code) - static_cast<int32_t>(z)), s);
  }
}

// init_scale_minmax (quant.cpp:161-183): per slice absmax via the |x| bit patterns (monotone for
// non-negative doubles); NaN never wins std::max(absmax, NaN) (the comparison is false).
__global__ void absmax_f64_kernel(const double* __restrict__ x, int64_t count, int64_t inner,
                                  int64_t extent, unsigned long long* __restrict__ amax) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double a = fabs(x[i]);
    if (isnan(a) || a == 0.0) continue;
    const int64_t ch = extent > 1 ? (i / inner) % extent : 0;
    atomicMax(amax + ch, static_cast<unsigned long long>(__double_as_longlong(a)));
  }
}
__global__ void minmax_finish_kernel(double* scales, int64_t extent, double qmax) {
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < extent;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double a = __longlong_as_double(reinterpret_cast<const long long*>(scales)[c]);
    scales[c] = a > 0.0 ? __ddiv_rn(a, qmax) : DBL_MIN;
  }
}

// matmul_nt (tensor.cpp:82-105): c(i,j) = sum_k a(i,k) b(j,k), accumulated from 0.0 in ascending
// k with a separate rounding per multiply and add.  32x32 output tile per 256 threads (4
// outputs per thread), 32-wide k slabs staged in shared memory; each output keeps its own
// sequential sum, so the tiling never changes the order.
constexpr int kMmTile = 32;
__global__ void __launch_bounds__(kT) matmul_nt_f64_kernel(const double* __restrict__ a, int64_t m, int64_t k,
                                                           int64_t lda, const double* __restrict__ b, int64_t n,
                                                           int64_t ldb, double* __restrict__ c, int64_t ldc) {
  __shared__ double as[kMmTile][kMmTile + 1], bs[kMmTile][kMmTile + 1];
  const int64_t i0 = static_cast<int64_t>(blockIdx.y) * kMmTile, j0 = static_cast<int64_t>(blockIdx.x) * kMmTile;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // ty in [0, 8): rows ty, ty+8, ty+16, ty+24
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t k0 = 0; k0 < k; k0 += kMmTile) {
    for (int r = ty; r < kMmTile; r += 8) {
      const int64_t ii = i0 + r, jj = j0 + r, kk = k0 + tx;
      as[r][tx] = (ii < m && kk < k) ? a[ii * lda + kk] : 0.0;
      bs[r][tx] = (jj < n && kk < k) ? b[jj * ldb + kk] : 0.0;
    }
    __syncthreads();
    const int kn = k - k0 < kMmTile ? static_cast<int>(k - k0) : kMmTile;
    for (int q = 0; q < kn; ++q) {
      const double bv = bs[tx][q];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] = __dadd_rn(acc[u], __dmul_rn(as[ty + 8 * u][q], bv));
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t ii = i0 + ty + 8 * u, jj = j0 + tx;
    if (ii < m && jj < n) c[ii * ldc + jj] = acc[u];
  }
}

// out[r, c] = idx[c] >= 0 ? in[r, idx[c]] : 0
template <typename T>
__global__ void gather_cols_kernel(const T* __restrict__ in, int64_t rows, int64_t ld_in,
                                   const int32_t* __restrict__ idx, int64_t cols, T* __restrict__ out,
                                   int64_t ld_out) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    const int32_t src = idx[c];
    out[r * ld_out + c] = src >= 0 ? in[r * ld_in + src] : T(0);
  }
}

// dequantized_weight_original_order (engine.cpp:117-130)
__global__ void dequant_weight_kernel(const int32_t* __restrict__ wq, int64_t n, int64_t k,
                                      const uint32_t* __restrict__ perm, int64_t n_outlier,
                                      const double* __restrict__ s_o, const double* __restrict__ s_n,
                                      double* __restrict__ w) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n * k;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = i / k, pos = i - j * k;
    const int64_t orig = perm ? perm[pos] : pos;
    const double s = pos < n_outlier ? s_o[j] : s_n[j];
    w[j * k + orig] = __dmul_rn(static_cast<double>(wq[i]), s);
  }
}

// ---- percentile search -------------------------------------------------------------------
constexpr int kMaxTargets = 2 * QARVD_MAX_CANDIDATES;
struct SelectState {
  unsigned long long prefix[kMaxTargets];
  unsigned long long rank[kMaxTargets];  // remaining rank within the prefix's bucket
};

// one MSB-first 8-bit radix pass over the pooled |x| keys for every target order statistic
__global__ void __launch_bounds__(kT) radix_pass_kernel(const double* __restrict__ x, int64_t count,
                                                        const SelectState* __restrict__ st, int targets,
                                                        int shift, unsigned long long* __restrict__ hist) {
  extern __shared__ unsigned int sh[];  // [targets][256]
  for (int i = threadIdx.x; i < targets * 256; i += kT) sh[i] = 0;
  __syncthreads();
  unsigned long long pre[kMaxTargets];
  for (int t = 0; t < targets; ++t) pre[t] = st->prefix[t];
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const unsigned long long key = static_cast<unsigned long long>(__double_as_longlong(x[i])) & 0x7fffffffffffffffULL;
    const unsigned digit = static_cast<unsigned>(key >> shift) & 255u;
    for (int t = 0; t < targets; ++t)
      if (shift == 56 || ((key ^ pre[t]) >> (shift + 8)) == 0) atomicAdd(&sh[t * 256 + digit], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < targets * 256; i += kT)
    if (sh[i]) atomicAdd(hist + i, static_cast<unsigned long long>(sh[i]));
}
// one warp per target: the digit whose cumulative count passes the remaining rank
__global__ void radix_select_kernel(SelectState* st, int targets, int shift, unsigned long long* hist) {
  const int t = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (t >= targets) return;
  if (lane == 0) {
    unsigned long long r = st->rank[t], cum = 0;
    int d = 0;
    for (; d < 255; ++d) {
      const unsigned long long h = hist[t * 256 + d];
      if (cum + h > r) break;
      cum += h;
    }
    st->rank[t] = r - cum;
    st->prefix[t] |= static_cast<unsigned long long>(d) << shift;
  }
  __syncwarp();
  for (int i = lane; i < 256; i += 32) hist[t * 256 + i] = 0;
}

struct CandDesc {
  double pct[QARVD_MAX_CANDIDATES];
  int t_lo[QARVD_MAX_CANDIDATES], t_hi[QARVD_MAX_CANDIDATES];  // target slots (t_hi < 0: no interpolation)
};
// thresholds (interpolated_quantile, quant.cpp:20-28) and candidate scales (:203-206)
__global__ void thresholds_kernel(const SelectState* st, CandDesc cd, int nc, unsigned long long n, double qmax,
                                  double* result) {
  if (threadIdx.x != 0) return;
  for (int c = 0; c < nc; ++c) {
    const double lo_v = __longlong_as_double(static_cast<long long>(st->prefix[cd.t_lo[c]]));
    double thr = lo_v;
    if (cd.t_hi[c] >= 0) {
      const double h = __dmul_rn(cd.pct[c], static_cast<double>(n - 1));
      const unsigned long long lo = static_cast<unsigned long long>(h);
      const double frac = __dsub_rn(h, static_cast<double>(lo));
      const double hi_v = __longlong_as_double(static_cast<long long>(st->prefix[cd.t_hi[c]]));
      thr = __dadd_rn(lo_v, __dmul_rn(frac, __dsub_rn(hi_v, lo_v)));
    }
    result[c] = thr;
    result[nc + c] = thr > 0.0 ? __ddiv_rn(thr, qmax) : DBL_MIN;
  }
}

struct MseBlock {
  int64_t sample, begin, end;  // element range [begin, end) of the pooled array
};
// per (block, candidate): double-double sum of (x - fake_quant(x))^2 over the block's range;
// non-finite elements record their in-sample index (the reference throws there)
__global__ void __launch_bounds__(kT) mse_partial_kernel(const double* __restrict__ x,
                                                         const MseBlock* __restrict__ blocks,
                                                         const int64_t* __restrict__ sample_begin,
                                                         const double* __restrict__ result, int nc, double qmax,
                                                         double* __restrict__ partial,
                                                         unsigned long long* __restrict__ nonfinite) {
  const MseBlock b = blocks[blockIdx.x];
  double s[QARVD_MAX_CANDIDATES];
  crm::dd acc[QARVD_MAX_CANDIDATES];
  for (int c = 0; c < nc; ++c) {
    s[c] = result[nc + c];
    acc[c] = {0.0, 0.0};
  }
  for (int64_t i = b.begin + threadIdx.x; i < b.end; i += kT) {
    const double v = x[i];
    if (!isfinite(v)) {
      atomicMin(nonfinite + b.sample, static_cast<unsigned long long>(i - sample_begin[b.sample]));
      continue;
    }
    for (int c = 0; c < nc; ++c) {
      int64_t code = cvtt_i64(rint(__ddiv_rn(v, s[c])));
      code = code < -static_cast<int64_t>(qmax) ? -static_cast<int64_t>(qmax)
                                                : (code > static_cast<int64_t>(qmax) ? static_cast<int64_t>(qmax) : code);
      const double d = __dsub_rn(v, __dmul_rn(static_cast<double>(code), s[c]));
      acc[c] = crm::dd_add(acc[c], crm::two_prod(d, d));
    }
  }
  __shared__ double red_hi[kT], red_lo[kT];
  for (int c = 0; c < nc; ++c) {
    red_hi[threadIdx.x] = acc[c].hi;
    red_lo[threadIdx.x] = acc[c].lo;
    __syncthreads();
    for (int w = kT / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w) {
        const crm::dd r = crm::dd_add({red_hi[threadIdx.x], red_lo[threadIdx.x]},
                                      {red_hi[threadIdx.x + w], red_lo[threadIdx.x + w]});
        red_hi[threadIdx.x] = r.hi;
        red_lo[threadIdx.x] = r.lo;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      partial[(static_cast<int64_t>(blockIdx.x) * nc + c) * 2] = red_hi[0];
      partial[(static_cast<int64_t>(blockIdx.x) * nc + c) * 2 + 1] = red_lo[0];
    }
    __syncthreads();
  }
}
// candidate MSEs (quant.cpp:208-224): mse = (sum_s frob_s / size_s) / S in sample order; argmin
// with <= (ties to the larger percentile); result = {thr[nc], scale[nc], mse[nc], best, scale}
__global__ void mse_final_kernel(const double* partial, const int64_t* block_first, const int64_t* sizes,
                                 int64_t n_samples, int nc, double* result) {
  if (threadIdx.x != 0) return;
  double best = INFINITY;
  int best_c = 0;
  for (int c = 0; c < nc; ++c) {
    double mse_sum = 0.0;
    for (int64_t s = 0; s < n_samples; ++s) {
      crm::dd t = {0.0, 0.0};
      for (int64_t bl = block_first[s]; bl < block_first[s + 1]; ++bl)
        t = crm::dd_add(t, {partial[(bl * nc + c) * 2], partial[(bl * nc + c) * 2 + 1]});
      mse_sum = __dadd_rn(mse_sum, __ddiv_rn(t.hi, static_cast<double>(sizes[s])));
    }
    const double mse = __ddiv_rn(mse_sum, static_cast<double>(n_samples));
    result[2 * nc + c] = mse;
    if (mse <= best) {
      best = mse;
      best_c = c;
    }
  }
  result[3 * nc] = static_cast<double>(best_c);
  result[3 * nc + 1] = result[nc + best_c];
}

// ---- small helpers of the drop-in's f64 paths ----------------------------------------------
// *total = (accumulate ? *total : 0) + weight * sum_i (a_i - b_i)^2, the sum sequential in i
// (frobenius_sq_distance, tensor.cpp:116-126; weighted_recon_loss, calibrate.cpp:206-214);
// divide_by > 0 then divides the total (the batch mean, calibrate.cpp:215).
__global__ void sq_distance_acc_kernel(const double* a, const double* b, int64_t count, double weight,
                                       double* total, int accumulate, double divide_by) {
  if (threadIdx.x != 0) return;
  double acc = 0.0;
  for (int64_t i = 0; i < count; ++i) {
    const double d = __dsub_rn(a[i], b[i]);
    acc = __dadd_rn(acc, __dmul_rn(d, d));
  }
  double t = __dadd_rn(accumulate ? *total : 0.0, __dmul_rn(weight, acc));
  if (divide_by > 0.0) t = __ddiv_rn(t, divide_by);
  *total = t;
}

// zero-point correction of kernel B (engine.cpp:74-83, :95-100): per output column the integer
// column sums of each group, corr = sum_g s_g[j] * colsum_g[j] (outlier group first), then
// y[i, j] -= (z_x * s_x) * corr.  One warp per column.
__global__ void zero_point_correct_kernel(double* y, int64_t ldy, int64_t m, int64_t n, const int8_t* wq,
                                          int64_t ldw, int64_t k, int64_t k_outlier, int groups, int32_t z_x,
                                          double s_x, const double* s_wo, const double* s_wn) {
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= n) return;
  long long cs_o = 0, cs_n = 0;
  for (int64_t c = lane; c < k; c += 32) {
    const int v = wq[j * ldw + c];
    if (c < k_outlier) cs_o += v;
    else cs_n += v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cs_o += __shfl_xor_sync(0xffffffffu, cs_o, o);
    cs_n += __shfl_xor_sync(0xffffffffu, cs_n, o);
  }
  double corr = 0.0;
  if (groups == 2) corr = __dadd_rn(corr, __dmul_rn(s_wo[j], static_cast<double>(cs_o)));
  corr = __dadd_rn(corr, __dmul_rn(s_wn[j], static_cast<double>(groups == 2 ? cs_n : cs_n + cs_o)));
  const double sub = __dmul_rn(__dmul_rn(static_cast<double>(z_x), s_x), corr);
  for (int64_t i = lane; i < m; i += 32) y[i * ldy + j] = __dsub_rn(y[i * ldy + j], sub);
}

// out[r, c] = idx[c] >= 0 ? (int8) in[r, idx[c]] : 0; a code outside int8 sets *bad
__global__ void pack_codes_kernel(const int32_t* __restrict__ in, int64_t rows, int64_t ld_in,
                                  const int32_t* __restrict__ idx, int64_t cols, int8_t* __restrict__ out,
                                  int64_t ld_out, int* bad) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    const int32_t src = idx[c];
    const int32_t v = src >= 0 ? in[r * ld_in + src] : 0;
    if (v < -128 || v > 127) *bad = 1;
    out[r * ld_out + c] = static_cast<int8_t>(v);
  }
}

// packed 4-bit codes (tensor.cpp:221-264 storage: two per byte, low nibble first, over the flat
// [rows x k_src] tensor) -> int8 kernel layout through the column map
__global__ void unpack_i4_kernel(const uint8_t* __restrict__ packed, int64_t rows, int64_t k_src,
                                 const int32_t* __restrict__ idx, int64_t cols, int8_t* __restrict__ out,
                                 int64_t ld_out) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    const int32_t src = idx[c];
    int8_t v = 0;
    if (src >= 0) {
      const int64_t f = r * k_src + src;
      const uint8_t b = packed[f >> 1];
      const uint8_t nib = (f & 1) ? (b >> 4) : (b & 0x0fu);
      v = static_cast<int8_t>(static_cast<int8_t>(nib << 4) >> 4);  // sign-extend
    }
    out[r * ld_out + c] = v;
  }
}

__global__ void cr_exp_kernel(const double* in, double* out, int64_t count) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = libm::exp(in[i]);
}

struct Arena {
  std::vector<void*> ptrs;
  cudaStream_t s;
  explicit Arena(cudaStream_t st) : s(st) {}
  ~Arena() {
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

extern "C" {

int qarvd_quantize_f64(const double* x, int64_t count, int64_t inner, int64_t extent,
                       const double* scales, const int32_t* zero_points, int32_t q_min,
                       int32_t q_max, int32_t* codes, double* dequant, int64_t* err_index,
                       void* stream) {
  clear_error();
  if (count < 0 || inner < 1 || extent < 1 || !scales || (count > 0 && !x) || q_min > q_max)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "qarvd_quantize_f64: invalid argument");
  if (int st = require_device()) return st;
  cudaStream_t s = as_stream(stream);
  if (err_index) {
    set_i64_kernel<<<1, 32, 0, s>>>(err_index, INT64_MAX, 1);
    count_launch();
  }
  if (count == 0) return QARVD_OK;
  quantize_f64_kernel<<<grid_for(count, 4), kT, 0, s>>>(
      x, count, inner, extent, scales, zero_points, q_min, q_max, codes, dequant,
      reinterpret_cast<unsigned long long*>(err_index));
  count_launch();
  QARVD_LAUNCH_CHECK();
  return QARVD_OK;
}

int qarvd_minmax_scale_f64(const double* x, int64_t count, int64_t inner, int64_t extent, int bits,
                           double* scales, void* stream) {
  clear_error();
  if (bits < 2 || bits > 30)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "bit width out of supported range [2,30]: " + std::to_string(bits));
  if (count < 0 || inner < 1 || extent < 1 || !scales || (count > 0 && !x))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "qarvd_minmax_scale_f64: invalid argument");
  if (int st = require_device()) return st;
  cudaStream_t s = as_stream(stream);
  QARVD_CUDA_TRY(cudaMemsetAsync(scales, 0, static_cast<size_t>(extent) * sizeof(double), s));
  if (count > 0) {
    absmax_f64_kernel<<<grid_for(count, 4), kT, 0, s>>>(x, count, inner, extent,
                                                        reinterpret_cast<unsigned long long*>(scales));
    count_launch();
  }
  minmax_finish_kernel<<<grid_for(extent), kT, 0, s>>>(scales, extent,
                                                       static_cast<double>((1 << (bits - 1)) - 1));
  count_launch();
  QARVD_LAUNCH_CHECK();
  return QARVD_OK;
}

int qarvd_matmul_nt_f64(const double* a, int64_t m, int64_t k, int64_t lda, const double* b, int64_t n,
                        int64_t ldb, double* c, int64_t ldc, void* stream) {
  clear_error();
  if (m < 0 || n < 0 || k < 0 || (m > 0 && n > 0 && (!c || ldc < n)) ||
      (m > 0 && k > 0 && (!a || lda < k)) || (n > 0 && k > 0 && (!b || ldb < k)))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "qarvd_matmul_nt_f64: invalid argument");
  if (int st = require_device()) return st;
  if (m == 0 || n == 0) return QARVD_OK;
  const dim3 grid(static_cast<unsigned>((n + kMmTile - 1) / kMmTile), static_cast<unsigned>((m + kMmTile - 1) / kMmTile));
  if (grid.y > 65535) QARVD_FAIL(QARVD_ERR_UNSUPPORTED, "qarvd_matmul_nt_f64: m too large");
  matmul_nt_f64_kernel<<<grid, kT, 0, as_stream(stream)>>>(a, m, k, lda, b, n, ldb, c, ldc);
  count_launch();
  QARVD_LAUNCH_CHECK();
  return QARVD_OK;
}

int qarvd_gather_columns(const void* in, int64_t rows, int64_t ld_in, const int32_t* idx,
                         int64_t out_cols, void* out, int64_t ld_out, int elem_bytes, void* stream) {
  clear_error();
  if (rows < 0 || out_cols < 0 || !idx || !in || !out || ld_out < out_cols ||
      (elem_bytes != 1 && elem_bytes != 2 && elem_bytes != 4 && elem_bytes != 8))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "qarvd_gather_columns: invalid argument");
  if (int st = require_device()) return st;
  if (rows == 0 || out_cols == 0) return QARVD_OK;
  cudaStream_t s = as_stream(stream);
  const unsigned g = grid_for(rows * out_cols, 4);
  switch (elem_bytes) {
    case 1: gather_cols_kernel<int8_t><<<g, kT, 0, s>>>(static_cast<const int8_t*>(in), rows, ld_in, idx, out_cols, static_cast<int8_t*>(out), ld_out); break;
    case 2: gather_cols_kernel<uint16_t><<<g, kT, 0, s>>>(static_cast<const uint16_t*>(in), rows, ld_in, idx, out_cols, static_cast<uint16_t*>(out), ld_out); break;
    case 4: gather_cols_kernel<int32_t><<<g, kT, 0, s>>>(static_cast<const int32_t*>(in), rows, ld_in, idx, out_cols, static_cast<int32_t*>(out), ld_out); break;
    default: gather_cols_kernel<double><<<g, kT, 0, s>>>(static_cast<const double*>(in), rows, ld_in, idx, out_cols, static_cast<double*>(out), ld_out); break;
  }
  count_launch();
  QARVD_LAUNCH_CHECK();
  return QARVD_OK;
}

int qarvd_dequant_weight_f64(const int32_t* wq, int64_t n, int64_t k, const uint32_t* perm,
                             int64_t n_outlier, const double* scale_outlier, const double* scale_normal,
                             double* w_out, void* stream) {
  clear_error();
  if (n < 0 || k < 0 || n_outlier < 0 || n_outlier > k || !scale_normal || (n_outlier > 0 && !scale_outlier) ||
      (n * k > 0 && (!wq || !w_out)))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "qarvd_dequant_weight_f64: invalid argument");
  if (int st = require_device()) return st;
  if (n * k == 0) return QARVD_OK;
  dequant_weight_kernel<<<grid_for(n * k, 4), kT, 0, as_stream(stream)>>>(wq, n, k, perm, n_outlier, scale_outlier,
                                                                          scale_normal, w_out);
  count_launch();
  QARVD_LAUNCH_CHECK();
  return QARVD_OK;
}

int qarvd_percentile_search_f64(const double* x, const int64_t* sample_offsets, int64_t n_samples,
                                const double* percentiles, int num_cand, int bits, double* result,
                                int64_t* err, void* stream) {
  clear_error();
  if (bits < 2 || bits > 30)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "bit width out of supported range [2,30]: " + std::to_string(bits));
  if (n_samples <= 0) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "percentile search: empty calibration sample list");
  if (!sample_offsets || !percentiles || !result || !err || num_cand < 1 || num_cand > QARVD_MAX_CANDIDATES ||
      sample_offsets[0] != 0)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "qarvd_percentile_search_f64: invalid argument");
  for (int64_t i = 0; i < n_samples; ++i)
    if (sample_offsets[i + 1] < sample_offsets[i])
      QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "qarvd_percentile_search_f64: unordered sample offsets");
  const int64_t total = sample_offsets[n_samples];
  if (total == 0) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "quantile of empty vector");
  if (!x) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "qarvd_percentile_search_f64: invalid argument");
  if (int st = require_device()) return st;
  cudaStream_t s = as_stream(stream);
  const double qmax = static_cast<double>((1 << (bits - 1)) - 1);

  // the order statistics each candidate needs (interpolated_quantile, quant.cpp:20-28)
  CandDesc cd{};
  std::vector<unsigned long long> ranks;
  auto slot = [&](unsigned long long r) {
    for (size_t i = 0; i < ranks.size(); ++i)
      if (ranks[i] == r) return static_cast<int>(i);
    ranks.push_back(r);
    return static_cast<int>(ranks.size() - 1);
  };
  const unsigned long long n = static_cast<unsigned long long>(total);
  for (int c = 0; c < num_cand; ++c) {
    cd.pct[c] = percentiles[c];
    if (n == 1) {
      cd.t_lo[c] = slot(0);
      cd.t_hi[c] = -1;
      continue;
    }
    const double h = percentiles[c] * static_cast<double>(n - 1);
    const unsigned long long lo = static_cast<unsigned long long>(h);
    if (lo + 1 >= n) {
      cd.t_lo[c] = slot(n - 1);
      cd.t_hi[c] = -1;
    } else {
      cd.t_lo[c] = slot(lo);
      cd.t_hi[c] = slot(lo + 1);
    }
  }
  const int targets = static_cast<int>(ranks.size());
  SelectState init{};
  for (int t = 0; t < targets; ++t) init.rank[t] = ranks[t];

  // per-sample MSE blocks of <= 16 elements per thread
  constexpr int64_t kChunk = static_cast<int64_t>(kT) * 16;
  std::vector<MseBlock> blocks;
  std::vector<int64_t> block_first(static_cast<size_t>(n_samples) + 1), sizes(static_cast<size_t>(n_samples));
  for (int64_t i = 0; i < n_samples; ++i) {
    block_first[i] = static_cast<int64_t>(blocks.size());
    sizes[i] = sample_offsets[i + 1] - sample_offsets[i];
    for (int64_t b = sample_offsets[i]; b < sample_offsets[i + 1]; b += kChunk)
      blocks.push_back({i, b, b + kChunk < sample_offsets[i + 1] ? b + kChunk : sample_offsets[i + 1]});
  }
  block_first[n_samples] = static_cast<int64_t>(blocks.size());

  Arena A(s);
  SelectState* st_d = A.get<SelectState>(1);
  unsigned long long* hist = A.get<unsigned long long>(kMaxTargets * 256);
  MseBlock* blocks_d = A.get<MseBlock>(static_cast<int64_t>(blocks.size()));
  int64_t* first_d = A.get<int64_t>(n_samples + 1);
  int64_t* sizes_d = A.get<int64_t>(n_samples);
  int64_t* begin_d = A.get<int64_t>(n_samples + 1);
  double* partial = A.get<double>(static_cast<int64_t>(blocks.size()) * num_cand * 2);
  unsigned long long* nonfinite = A.get<unsigned long long>(n_samples);
  if (!st_d || !hist || !blocks_d || !first_d || !sizes_d || !begin_d || !partial || !nonfinite)
    QARVD_FAIL(QARVD_ERR_CUDA, "percentile search: device allocation failed");
  QARVD_CUDA_TRY(cudaMemcpyAsync(st_d, &init, sizeof(init), cudaMemcpyHostToDevice, s));
  QARVD_CUDA_TRY(cudaMemsetAsync(hist, 0, kMaxTargets * 256 * sizeof(unsigned long long), s));
  QARVD_CUDA_TRY(cudaMemcpyAsync(blocks_d, blocks.data(), blocks.size() * sizeof(MseBlock), cudaMemcpyHostToDevice, s));
  QARVD_CUDA_TRY(cudaMemcpyAsync(first_d, block_first.data(), block_first.size() * 8, cudaMemcpyHostToDevice, s));
  QARVD_CUDA_TRY(cudaMemcpyAsync(sizes_d, sizes.data(), sizes.size() * 8, cudaMemcpyHostToDevice, s));
  QARVD_CUDA_TRY(cudaMemcpyAsync(begin_d, sample_offsets, static_cast<size_t>(n_samples + 1) * 8,
                                 cudaMemcpyHostToDevice, s));
  QARVD_CUDA_TRY(cudaMemsetAsync(nonfinite, 0xff, static_cast<size_t>(n_samples) * 8, s));
  const size_t smem = static_cast<size_t>(targets) * 256 * sizeof(unsigned int);
  for (int shift = 56; shift >= 0; shift -= 8) {
    radix_pass_kernel<<<grid_for(total, 8), kT, smem, s>>>(x, total, st_d, targets, shift, hist);
    radix_select_kernel<<<1, targets * 32, 0, s>>>(st_d, targets, shift, hist);
    count_launch(2);
  }
  thresholds_kernel<<<1, 32, 0, s>>>(st_d, cd, num_cand, n, qmax, result);
  mse_partial_kernel<<<static_cast<unsigned>(blocks.size()), kT, 0, s>>>(x, blocks_d, begin_d, result, num_cand, qmax,
                                                                         partial, nonfinite);
  mse_final_kernel<<<1, 32, 0, s>>>(partial, first_d, sizes_d, n_samples, num_cand, result);
  count_launch(3);
  QARVD_LAUNCH_CHECK();
  // first sample (in order) holding a non-finite value, and its flat index (quant.cpp:128-129)
  std::vector<unsigned long long> nf(static_cast<size_t>(n_samples));
  QARVD_CUDA_TRY(cudaMemcpyAsync(nf.data(), nonfinite, nf.size() * 8, cudaMemcpyDeviceToHost, s));
  QARVD_CUDA_TRY(cudaStreamSynchronize(s));
  int64_t e[2] = {-1, -1};
  for (int64_t i = 0; i < n_samples; ++i)
    if (nf[i] != ~0ULL) {
      e[0] = i;
      e[1] = static_cast<int64_t>(nf[i]);
      break;
    }
  QARVD_CUDA_TRY(cudaMemcpyAsync(err, e, sizeof(e), cudaMemcpyHostToDevice, s));
  QARVD_CUDA_TRY(cudaStreamSynchronize(s));
  return QARVD_OK;
}

int qarvd_sq_distance_acc_f64(const double* a, const double* b, int64_t count, double weight, double* total,
                              int accumulate, double divide_by, void* stream) {
  clear_error();
  if (count < 0 || !total || (count > 0 && (!a || !b)))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "qarvd_sq_distance_acc_f64: invalid argument");
  if (int st = require_device()) return st;
  sq_distance_acc_kernel<<<1, 32, 0, as_stream(stream)>>>(a, b, count, weight, total, accumulate, divide_by);
  count_launch();
  QARVD_LAUNCH_CHECK();
  return QARVD_OK;
}

int qarvd_zero_point_correct_f64(double* y, int64_t ldy, int64_t m, int64_t n, const int8_t* wq, int64_t ldw,
                                 int64_t k, int64_t k_outlier, int groups, int32_t z_x, double s_x,
                                 const double* s_wo, const double* s_wn, void* stream) {
  clear_error();
  if (m < 0 || n < 0 || k < 0 || !y || !wq || !s_wn || (groups == 2 && !s_wo) || (groups != 1 && groups != 2) ||
      k_outlier < 0 || k_outlier > k || ldy < n || ldw < k)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "qarvd_zero_point_correct_f64: invalid argument");
  if (int st = require_device()) return st;
  if (m == 0 || n == 0 || z_x == 0) return QARVD_OK;
  zero_point_correct_kernel<<<static_cast<unsigned>((n + 7) / 8), 256, 0, as_stream(stream)>>>(
      y, ldy, m, n, wq, ldw, k, k_outlier, groups, z_x, s_x, s_wo, s_wn);
  count_launch();
  QARVD_LAUNCH_CHECK();
  return QARVD_OK;
}

int qarvd_pack_codes_i8(const int32_t* in, int64_t rows, int64_t ld_in, const int32_t* idx, int64_t out_cols,
                        int8_t* out, int64_t ld_out, int* bad, void* stream) {
  clear_error();
  if (rows < 0 || out_cols < 0 || !in || !idx || !out || !bad || ld_out < out_cols)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "qarvd_pack_codes_i8: invalid argument");
  if (int st = require_device()) return st;
  if (rows == 0 || out_cols == 0) return QARVD_OK;
  pack_codes_kernel<<<grid_for(rows * out_cols, 4), kT, 0, as_stream(stream)>>>(in, rows, ld_in, idx, out_cols,
                                                                                out, ld_out, bad);
  count_launch();
  QARVD_LAUNCH_CHECK();
  return QARVD_OK;
}

int qarvd_unpack_codes_i4(const uint8_t* packed, int64_t rows, int64_t k_src, const int32_t* idx,
                          int64_t out_cols, int8_t* out, int64_t ld_out, void* stream) {
  clear_error();
  if (rows < 0 || k_src < 0 || out_cols < 0 || ld_out < out_cols || (rows * out_cols > 0 && (!idx || !out)) ||
      (rows * k_src > 0 && !packed))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "qarvd_unpack_codes_i4: invalid argument");
  if (int st = require_device()) return st;
  if (rows == 0 || out_cols == 0) return QARVD_OK;
  unpack_i4_kernel<<<grid_for(rows * out_cols, 4), kT, 0, as_stream(stream)>>>(packed, rows, k_src, idx, out_cols,
                                                                               out, ld_out);
  count_launch();
  QARVD_LAUNCH_CHECK();
  return QARVD_OK;
}

int qarvd_exp_f64(const double* in, double* out, int64_t count, void* stream) {
  clear_error();
  if (count < 0 || (count > 0 && (!in || !out))) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "qarvd_exp_f64: invalid argument");
  if (int st = require_device()) return st;
  if (count == 0) return QARVD_OK;
  cr_exp_kernel<<<grid_for(count), kT, 0, as_stream(stream)>>>(in, out, count);
  count_launch();
  QARVD_LAUNCH_CHECK();
  return QARVD_OK;
}

}  // extern "C"
