// K3 — per-layer outlier detection, batched over layers.
//
// Reference: analyze_layer (outlier.cpp:98-102) =
//   channel_l2_norms(W, 1)            tensor.cpp:132-150  (f64, rows summed in order i = 0..n-1)
//   mad / sorted_median               outlier.cpp:13-18, :30-38
//   threshold = max(med + (tau/0.6745)*MAD, alpha*med)   outlier.cpp:46-47 / :91-92
//   raw = {j : v_j > threshold}       outlier.cpp:48-51
//   align_outliers                    outlier.cpp:54-78
// Every floating operation below is the reference's operation with explicit
// round-to-nearest intrinsics (no FMA contraction), so norms, median, MAD,
// threshold and both index sets are bit-identical to the f64 CPU code.
//
// Kernel 1 (HBM-bound): one thread owns 2 adjacent columns (kNormCols; one 4-byte bf16
// load per row, a warp covers 128 contiguous bytes of a row) and accumulates the two
// column sums sequentially over the rows, exactly the reference order, with 8 rows of
// loads (kNormRows) in flight before they are added in order.
// For bf16/f32 inputs w*w is exact in f64, so the sum is the only rounding.
// Kernel 2 (tiny): one 1024-thread CTA per layer takes the medians and the alignment pivot by
// exact radix selection over the norms' bit patterns (no sort) and runs the selection /
// alignment.  The norm jobs run longest columns first (their sequential sums are the
// kernel's critical path) with 32 rows of loads in flight on columns of >= 4096 rows.
#include <algorithm>
#include <climits>
#include <vector>

#include "common.cuh"

namespace qarvd_b200 {
namespace {

constexpr int kNormThreads = 256;
constexpr int kSelThreads = 1024;
constexpr int kMaxSelK = 16384;

struct NormJobDev {
  const void* w;
  int64_t n, k, ldw;
  double* norms;
  int64_t col_groups;   // ceil(k / 8)
  int64_t group_begin;  // prefix over jobs
};

template <typename T>
__device__ __forceinline__ double sq(T v) {
  const double d = InType<T>::to_double(v);
  return __dmul_rn(d, d);
}

// grid-stride over the concatenated 2-column groups of all jobs.  Each column's sum stays
// sequential over rows (tensor.cpp:138-140, bit-exact); parallelism comes from many threads
// (two columns each) and from issuing 8 rows of loads before adding them in order.
constexpr int kNormCols = 2;
constexpr int kNormRows = 8;

template <typename T>
struct Pair;
template <>
struct Pair<uint16_t> {
  using V = uint32_t;
  __device__ static void split(V v, uint16_t& a, uint16_t& b) {
    a = static_cast<uint16_t>(v & 0xffffu);
    b = static_cast<uint16_t>(v >> 16);
  }
};
template <>
struct Pair<float> {
  using V = float2;
  __device__ static void split(V v, float& a, float& b) {
    a = v.x;
    b = v.y;
  }
};
template <>
struct Pair<double> {
  using V = double2;
  __device__ static void split(V v, double& a, double& b) {
    a = v.x;
    b = v.y;
  }
};

template <typename T>
__global__ void __launch_bounds__(kNormThreads)
    column_norms_kernel(const NormJobDev* __restrict__ jobs, int num_jobs, int64_t total_groups) {
  using PV = typename Pair<T>::V;
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < total_groups;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int lo = 0, hi = num_jobs - 1;  // the last job whose first group is <= g
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (jobs[mid].group_begin <= g) lo = mid;
      else hi = mid - 1;
    }
    const NormJobDev job = jobs[lo];
    const int64_t c0 = (g - job.group_begin) * kNormCols;
    const T* w = static_cast<const T*>(job.w);
    double a0 = 0.0, a1 = 0.0;
    const bool pair = (c0 + 2 <= job.k) && ((job.ldw & 1) == 0) &&
                      ((reinterpret_cast<uintptr_t>(w) & (sizeof(PV) - 1)) == 0);
    if (pair) {
      const T* base = w + c0;
      int64_t i = 0;
      if (job.n >= 4096) {  // long chains: 4x the loads in flight (the chain is latency-bound)
        for (; i + 4 * kNormRows <= job.n; i += 4 * kNormRows) {
          PV d[4 * kNormRows];
#pragma unroll
          for (int u = 0; u < 4 * kNormRows; ++u) d[u] = __ldg(reinterpret_cast<const PV*>(base + (i + u) * job.ldw));
#pragma unroll
          for (int u = 0; u < 4 * kNormRows; ++u) {
            T e0, e1;
            Pair<T>::split(d[u], e0, e1);
            a0 = __dadd_rn(a0, sq<T>(e0));
            a1 = __dadd_rn(a1, sq<T>(e1));
          }
        }
      }
      for (; i + kNormRows <= job.n; i += kNormRows) {
        PV d[kNormRows];
#pragma unroll
        for (int u = 0; u < kNormRows; ++u) d[u] = __ldg(reinterpret_cast<const PV*>(base + (i + u) * job.ldw));
#pragma unroll
        for (int u = 0; u < kNormRows; ++u) {
          T e0, e1;
          Pair<T>::split(d[u], e0, e1);
          a0 = __dadd_rn(a0, sq<T>(e0));
          a1 = __dadd_rn(a1, sq<T>(e1));
        }
      }
      for (; i < job.n; ++i) {
        T e0, e1;
        Pair<T>::split(__ldg(reinterpret_cast<const PV*>(base + i * job.ldw)), e0, e1);
        a0 = __dadd_rn(a0, sq<T>(e0));
        a1 = __dadd_rn(a1, sq<T>(e1));
      }
    } else {
      const bool two = c0 + 1 < job.k;
      for (int64_t i = 0; i < job.n; ++i) {
        const T* row = w + i * job.ldw + c0;
        a0 = __dadd_rn(a0, sq<T>(row[0]));
        if (two) a1 = __dadd_rn(a1, sq<T>(row[1]));
      }
    }
    job.norms[c0] = __dsqrt_rn(a0);
    if (c0 + 1 < job.k) job.norms[c0 + 1] = __dsqrt_rn(a1);
  }
}

// ---- selection -------------------------------------------------------------
// The r-th smallest (0-based) of k keys key(i) (order-preserving u64 images of non-negative
// doubles): MSB-first radix select, 8 bits per pass, a 256-bin shared histogram of the keys
// that match the prefix so far, one warp scans it.  Exact, no sort (the previous bitonic sorts
// of P = 2048 / 16384 keys took ~25 / 60 us per layer).
template <typename KeyFn>
__device__ unsigned long long radix_select(int k, KeyFn key, unsigned long long r, uint32_t* hist,
                                           unsigned long long* s_pick) {
  unsigned long long prefix = 0, mask = 0;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
      const unsigned long long x = key(i);
      if ((x & mask) == prefix) atomicAdd(&hist[(x >> shift) & 0xffu], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      uint32_t c[8], tot = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c[j] = hist[lane * 8 + j];
        tot += c[j];
      }
      uint32_t incl = tot;  // inclusive prefix over lanes
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      unsigned long long before = incl - tot;
      const bool mine = before <= r && r < before + tot;
      if (mine) {
        int b = lane * 8;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (before + c[j] > r) break;
          before += c[j];
          ++b;
        }
        s_pick[0] = static_cast<unsigned long long>(b);
        s_pick[1] = before;
      }
    }
    __syncthreads();
    const unsigned long long b = s_pick[0], before = s_pick[1];
    __syncthreads();
    prefix |= b << shift;
    mask |= 0xffull << shift;
    r -= before;
  }
  return prefix;
}

// sorted_median (outlier.cpp:13-18) of k keys via selection
template <typename KeyFn>
__device__ double median_select(int k, KeyFn key, uint32_t* hist, unsigned long long* s_pick) {
  const unsigned long long hi = radix_select(k, key, static_cast<unsigned long long>(k / 2), hist, s_pick);
  if (k & 1) return __longlong_as_double(static_cast<long long>(hi));
  const unsigned long long lo = radix_select(k, key, static_cast<unsigned long long>(k / 2 - 1), hist, s_pick);
  return __dmul_rn(0.5, __dadd_rn(__longlong_as_double(static_cast<long long>(lo)),
                                  __longlong_as_double(static_cast<long long>(hi))));
}

// block-wide ordered compaction: writes indices i (ascending) with pred(i) true
template <typename Pred>
__device__ int compact_indices(int k, Pred pred, int32_t* out, int* warp_tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int base = 0;
  for (int c0 = 0; c0 < k; c0 += blockDim.x) {
    const int i = c0 + threadIdx.x;
    const bool f = (i < k) && pred(i);
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) warp_tot[warp] = __popc(bal);
    __syncthreads();
    int off = 0, tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      if (w < warp) off += warp_tot[w];
      tot += warp_tot[w];
    }
    if (f) out[base + off + __popc(bal & ((1u << lane) - 1u))] = i;
    base += tot;
    __syncthreads();
  }
  return base;
}

struct SelJobDev {
  int64_t k;
  const double* norms;
  double* stats;
  int32_t* counts;
  int32_t* raw_idx;
  int32_t* aligned_idx;
};

__global__ void __launch_bounds__(kSelThreads)
    select_outliers_kernel(const SelJobDev* __restrict__ jobs, double tau, double alpha_min,
                           int64_t align) {
  extern __shared__ unsigned long long sbuf[];  // scratch: the norms' keys, then int32 indices
  __shared__ int warp_tot[32];
  __shared__ double s_val[4];
  __shared__ uint32_t s_hist[256];
  __shared__ unsigned long long s_pick[2];
  const SelJobDev job = jobs[blockIdx.x];
  const int k = static_cast<int>(job.k);
  const double* v = job.norms;
  for (int i = threadIdx.x; i < k; i += blockDim.x)
    sbuf[i] = static_cast<unsigned long long>(__double_as_longlong(v[i]));
  __syncthreads();
  const unsigned long long* keys = sbuf;

  // median of norms (norms are non-negative: their bit patterns order like the values)
  const double med = median_select(k, [&](int i) { return keys[i]; }, s_hist, s_pick);

  // MAD = median |v - med|   (outlier.cpp:35-36)
  const double mad_sel = median_select(
      k,
      [&](int i) {
        return static_cast<unsigned long long>(
            __double_as_longlong(fabs(__dsub_rn(__longlong_as_double(static_cast<long long>(keys[i])), med))));
      },
      s_hist, s_pick);
  if (threadIdx.x == 0) {
    const double mad = mad_sel;
    const double zc = __ddiv_rn(tau, 0.6745);  // kModifiedZScoreFactor (outlier.hpp:13)
    const double a = __dadd_rn(med, __dmul_rn(zc, mad));
    const double b = __dmul_rn(alpha_min, med);
    s_val[1] = mad;
    s_val[2] = (a < b) ? b : a;  // std::max
  }
  __syncthreads();
  const double thr = s_val[2];

  // raw outliers, ascending (outlier.cpp:48-51)
  const int R = compact_indices(k, [&](int i) { return v[i] > thr; }, job.raw_idx, warp_tot);

  // align_outliers (outlier.cpp:54-78)
  int A;
  const int64_t al = align;
  bool use_raw = (R == 0) || (k < 2 * al);
  int64_t target = ((R + al - 1) / al) * al;
  if (!use_raw) {
    const int64_t cap = k - al;
    if (target > cap) {
      target = (cap / al) * al;
      if (target < R) use_raw = true;
    }
  }
  if (R == 0) {
    A = 0;
  } else if (use_raw) {
    for (int i = threadIdx.x; i < R; i += blockDim.x) job.aligned_idx[i] = job.raw_idx[i];
    A = R;
  } else {
    // the `target` largest norms, ties -> lower index: pivot value = target-th largest
    const unsigned long long pivot = radix_select(
        k, [&](int i) { return keys[i]; }, static_cast<unsigned long long>(k - target), s_hist, s_pick);
    // count strictly greater, then take equal ones in index order
    const double pv = __longlong_as_double(static_cast<long long>(pivot));
    int greater = 0;
    for (int i = threadIdx.x; i < k; i += blockDim.x) greater += keys[i] > pivot ? 1 : 0;
    greater = __reduce_add_sync(0xffffffffu, greater);
    if ((threadIdx.x & 31) == 0) warp_tot[threadIdx.x >> 5] = greater;
    __syncthreads();
    if (threadIdx.x == 0) {
      int g = 0;
      for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) g += warp_tot[w];
      warp_tot[0] = static_cast<int>(target) - g;  // equal ones to take
    }
    __syncthreads();
    const int need_eq = warp_tot[0];
    __syncthreads();
    // rank of each equal element among equals (index order) via compaction into scratch after
    // the keys (k u64 keys, then k int32 indices)
    int32_t* eq_idx = reinterpret_cast<int32_t*>(sbuf + k);
    const int n_eq = compact_indices(k, [&](int i) { return v[i] == pv; }, eq_idx, warp_tot);
    (void)n_eq;
    // mark: greater, or one of the first need_eq equals
    // (eq_idx is ascending; membership test by binary search)
    A = compact_indices(
        k,
        [&](int i) {
          const double x = v[i];
          if (x > pv) return true;
          if (x != pv) return false;
          int lo = 0, hi = need_eq;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (eq_idx[mid] < i) lo = mid + 1;
            else hi = mid;
          }
          return lo < need_eq && eq_idx[lo] == i;
        },
        job.aligned_idx, warp_tot);
  }
  if (threadIdx.x == 0) {
    job.stats[0] = med;
    job.stats[1] = s_val[1];
    job.stats[2] = thr;
    job.counts[0] = R;
    job.counts[1] = A;
  }
}

}  // namespace
}  // namespace qarvd_b200

using namespace qarvd_b200;

extern "C" int qarvd_analyze_layers(const qarvd_outlier_job* jobs, int num_jobs, int w_dtype,
                                    double tau, double alpha_min, int64_t align, void* stream) {
  clear_error();
  if (num_jobs < 0 || (num_jobs > 0 && !jobs))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "analyze_layers: invalid job list");
  if (!(tau > 0.0)) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "detect_outliers: tau must be positive");
  if (!(alpha_min > 1.0))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "detect_outliers: alpha_min must exceed 1");
  if (align == 0) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "align_outliers: align must be >= 1");
  if (w_dtype != QARVD_BF16 && w_dtype != QARVD_F32 && w_dtype != QARVD_F64)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "analyze_layers: unknown dtype");
  if (num_jobs == 0) return QARVD_OK;
  std::vector<NormJobDev> nj(num_jobs);
  std::vector<SelJobDev> sj(num_jobs);
  int64_t groups = 0;
  int64_t max_k = 0;
  for (int i = 0; i < num_jobs; ++i) {
    const qarvd_outlier_job& J = jobs[i];
    if (J.k <= 0) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "mad: empty vector");
    if (J.n <= 0 || J.ldw < J.k || !J.w || !J.norms || !J.stats || !J.counts || !J.raw_idx ||
        !J.aligned_idx)
      QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "analyze_layers: invalid job " + std::to_string(i));
    if (J.k > kMaxSelK)
      QARVD_FAIL(QARVD_ERR_UNSUPPORTED, "analyze_layers: d_in above 16384 is not supported");
    nj[i] = NormJobDev{J.w, J.n, J.k, J.ldw, J.norms, (J.k + kNormCols - 1) / kNormCols, 0};
    sj[i] = SelJobDev{J.k, J.norms, J.stats, J.counts, J.raw_idx, J.aligned_idx};
    if (J.k > max_k) max_k = J.k;
  }
  // the longest column chains (most rows) first: their sequential sums set the kernel's
  // critical path (e.g. the 8960-row FFN-up layers), so they start in the first wave and the
  // short columns fill in around them (order of the norm jobs does not change any result)
  std::stable_sort(nj.begin(), nj.end(), [](const NormJobDev& a, const NormJobDev& b) { return a.n > b.n; });
  for (int i = 0; i < num_jobs; ++i) {
    nj[i].group_begin = groups;
    groups += nj[i].col_groups;
  }
  if (int st = require_device()) return st;
  cudaStream_t s = as_stream(stream);
  void* dev = nullptr;
  const size_t bytes = num_jobs * (sizeof(NormJobDev) + sizeof(SelJobDev));
  QARVD_CUDA_TRY(cudaMallocAsync(&dev, bytes, s));
  NormJobDev* d_nj = static_cast<NormJobDev*>(dev);
  SelJobDev* d_sj = reinterpret_cast<SelJobDev*>(d_nj + num_jobs);
  QARVD_CUDA_TRY(cudaMemcpyAsync(d_nj, nj.data(), num_jobs * sizeof(NormJobDev),
                                 cudaMemcpyHostToDevice, s));
  QARVD_CUDA_TRY(cudaMemcpyAsync(d_sj, sj.data(), num_jobs * sizeof(SelJobDev),
                                 cudaMemcpyHostToDevice, s));
  const int64_t blocks_needed = (groups + kNormThreads - 1) / kNormThreads;
  const int grid = static_cast<int>(blocks_needed < kNumSMs * 16 ? blocks_needed : kNumSMs * 16);
  static const cudaError_t carve = [] {
    cudaError_t e = prefer_max_shared(column_norms_kernel<uint16_t>);
    if (e == cudaSuccess) e = prefer_max_shared(column_norms_kernel<float>);
    if (e == cudaSuccess) e = prefer_max_shared(column_norms_kernel<double>);
    return e;
  }();
  QARVD_CUDA_TRY(carve);
  if (w_dtype == QARVD_BF16)
    column_norms_kernel<uint16_t><<<grid, kNormThreads, 0, s>>>(d_nj, num_jobs, groups);
  else if (w_dtype == QARVD_F32)
    column_norms_kernel<float><<<grid, kNormThreads, 0, s>>>(d_nj, num_jobs, groups);
  else
    column_norms_kernel<double><<<grid, kNormThreads, 0, s>>>(d_nj, num_jobs, groups);
  count_launch();
  QARVD_LAUNCH_CHECK();
  const size_t smem = static_cast<size_t>(max_k) * (sizeof(unsigned long long) + sizeof(int32_t));
  QARVD_CUDA_TRY(set_smem_attrs(select_outliers_kernel, kMaxSelK * static_cast<int>(sizeof(unsigned long long) + sizeof(int32_t))));
  select_outliers_kernel<<<num_jobs, kSelThreads, smem, s>>>(d_sj, tau, alpha_min, align);
  count_launch();
  QARVD_LAUNCH_CHECK();
  QARVD_CUDA_TRY(cudaFreeAsync(dev, s));
  return QARVD_OK;
}
