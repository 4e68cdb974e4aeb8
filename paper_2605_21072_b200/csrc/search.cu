// K4 — frame-weighted calibration scale search, batched over layers.
//
// Reference: init_scale_percentile_search (quant.cpp:190-226) pools |x| of
// all calibration samples, sorts it (quant.cpp:201), takes the candidate
// thresholds as interpolated quantiles (quant.cpp:20-28) for
// p in {0.999, 0.9999, 0.99999} (quant.cpp:185-188), scores each candidate by
// the mean per-sample fake-quant MSE (quant.cpp:208-217) and keeps the argmin
// with ties to the larger percentile (quant.cpp:219).  This build scores each
// frame's MSE with the frame weights of weighting_strategy
// (sensitivity.cpp:86-112), the Eq. 5 frame weighting applied to the
// activation-scale search.
//
// One pass over X: per (layer, frame) 2^15-bin histograms of the bf16 |x|
// bit patterns (exact integer counts).  Symmetric fake-quant error depends
// only on |x| (quant.hpp:14-20 is odd-symmetric), so every order statistic and
// every per-frame squared error is a function of the histograms:
//   thr_c  = exact order statistics of the pooled histogram, interpolated as quant.cpp:23-27
//   mse_f  = (sum_b cnt_f[b] * e_c(v_b)) / n_f,  e_c(v) = (v - s_c*clamp(rint(v/s_c)))^2
// The bin sum runs in a fixed canonical order (128 blocks of 256 bins, each
// block summed in ascending bin order, then the block partials in ascending
// order); oracle/qarvd_oracle.c restates exactly that order, so losses and the
// selected scale are bit-identical to the oracle and agree with the
// reference's element-order sums to ~1e-13 relative.
#include <vector>

#include "common.cuh"

namespace qarvd_b200 {
namespace {

constexpr int kBins = 32768;         // |bf16| bit patterns 0x0000..0x7fff
constexpr int kFiniteBins = 0x7f80;  // >= 0x7f80 is inf / nan
constexpr int kHistThreads = 512;
constexpr int kBlockBins = 256;
constexpr int kNumBlocks = kBins / kBlockBins;  // 128
constexpr int kEvalThreads = 512;
constexpr int kEvalGroup = 4;  // blocks whose squared errors are staged together

struct HistUnit {
  const uint16_t* x;  // first row of the unit
  int64_t rows, k, ldx;
  uint32_t* hist;     // [kBins] histogram of this (layer, frame)
  unsigned long long* err;
};

// Persistent: one CTA per SM walks a contiguous range of the units (sorted by layer, frame), so
// after the grid is dispatched the K3 -> K5 kernels queued behind it get the SM resources and the
// HBM bandwidth the histogram pass leaves (its shared-memory atomics, not HBM, bound it); the
// shared histogram is flushed to the unit's global histogram only when the target changes.
__global__ void __launch_bounds__(kHistThreads)
    hist_kernel(const HistUnit* __restrict__ units, int num_units) {
  extern __shared__ uint32_t sh[];
  const int per = (num_units + gridDim.x - 1) / gridDim.x;
  const int u0 = blockIdx.x * per, u1 = min(num_units, u0 + per);
  if (u0 >= u1) return;
  for (int i = threadIdx.x; i < kBins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  bool bad = false;
  auto count8 = [&](const uint4 d) {
    const uint32_t w[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const uint32_t lo = w[h] & 0x7fffu, hi = (w[h] >> 16) & 0x7fffu;
      bad |= (lo >= kFiniteBins) | (hi >= kFiniteBins);
      atomicAdd(&sh[lo], 1u);
      atomicAdd(&sh[hi], 1u);
    }
  };
  for (int ui = u0; ui < u1; ++ui) {
    const HistUnit u = units[ui];
    const bool vec = ((u.k & 7) == 0) && ((u.ldx & 7) == 0) &&
                     ((reinterpret_cast<uintptr_t>(u.x) & 15) == 0);
    if (vec && u.ldx == u.k) {
      // contiguous rows: one flat stream of 16-byte chunks (no per-chunk row division)
      const uint4* p = reinterpret_cast<const uint4*>(u.x);
      const int64_t total = u.rows * (u.k >> 3);
      int64_t t = threadIdx.x;
      for (; t + 3 * blockDim.x < total; t += 4 * blockDim.x) {
        const uint4 d0 = __ldg(p + t), d1 = __ldg(p + t + blockDim.x), d2 = __ldg(p + t + 2 * blockDim.x),
                    d3 = __ldg(p + t + 3 * blockDim.x);
        count8(d0);
        count8(d1);
        count8(d2);
        count8(d3);
      }
      for (; t < total; t += blockDim.x) count8(__ldg(p + t));
    } else if (vec) {
      const int vpr = static_cast<int>(u.k >> 3);  // uint4 per row
      for (int64_t r = 0; r < u.rows; ++r) {
        const uint4* p = reinterpret_cast<const uint4*>(u.x + r * u.ldx);
        for (int v = threadIdx.x; v < vpr; v += blockDim.x) count8(__ldg(p + v));
      }
    } else {
      const int64_t total = u.rows * u.k;
      for (int64_t t = threadIdx.x; t < total; t += blockDim.x) {
        const int64_t r = t / u.k, c = t - r * u.k;
        const uint32_t b = u.x[r * u.ldx + c] & 0x7fffu;
        bad |= b >= kFiniteBins;
        atomicAdd(&sh[b], 1u);
      }
    }
    if (bad && u.err) atomicMin(u.err, 0ull);
    bad = false;
    if (ui + 1 == u1 || units[ui + 1].hist != u.hist) {  // target changes: flush and clear
      __syncthreads();
      for (int i = threadIdx.x; i < kBins; i += blockDim.x) {
        const uint32_t c = sh[i];
        if (c) {
          atomicAdd(&u.hist[i], c);
          sh[i] = 0;
        }
      }
      __syncthreads();
    }
  }
}

struct EvalJob {
  const uint32_t* hist;  // [frames][kBins]
  int64_t frames;
  int64_t per_frame;     // elements per frame (rows * k)
  double* result;        // [3*nc + 2]
};

struct EvalConst {
  double pct[QARVD_MAX_CANDIDATES];
  double w[QARVD_MAX_FRAMES];
  int nc;
  int qmax;
  int equal_weights;
  double wsum;
};

__device__ __forceinline__ double bin_value(int b) {
  return static_cast<double>(__uint_as_float(static_cast<uint32_t>(b) << 16));
}

// squared fake-quant error of |x| = v at scale s (quant.cpp:132-135, :151, tensor.cpp:121-123)
__device__ __forceinline__ double fq_err(double v, double s, int qmax) {
  double q = rint(__ddiv_rn(v, s));
  if (q > qmax) q = qmax;
  const double d = __dsub_rn(v, __dmul_rn(q, s));
  return __dmul_rn(d, d);
}

__global__ void __launch_bounds__(kEvalThreads)
    eval_kernel(const EvalJob* __restrict__ jobs, const EvalConst cst) {
  extern __shared__ unsigned char smem_eval[];
  uint32_t* pooled = reinterpret_cast<uint32_t*>(smem_eval);                 // [kBins]
  uint32_t* blk_tot = pooled + kBins;                                        // [kNumBlocks]
  double* part = reinterpret_cast<double*>(blk_tot + kNumBlocks);            // [frames][nc][kNumBlocks]
  __shared__ double s_thr[QARVD_MAX_CANDIDATES], s_scale[QARVD_MAX_CANDIDATES];
  __shared__ unsigned long long s_rank[2 * QARVD_MAX_CANDIDATES];
  __shared__ int s_bin[2 * QARVD_MAX_CANDIDATES];
  __shared__ double s_mse[QARVD_MAX_FRAMES * QARVD_MAX_CANDIDATES];

  const EvalJob job = jobs[blockIdx.x];
  const int F = static_cast<int>(job.frames);
  const int nc = cst.nc;

  // 1. pooled histogram (exact integers)
  for (int b = threadIdx.x; b < kBins; b += blockDim.x) {
    uint32_t s = 0;
    for (int f = 0; f < F; ++f) s += job.hist[static_cast<int64_t>(f) * kBins + b];
    pooled[b] = s;
  }
  __syncthreads();
  // block totals for the rank search
  for (int blk = threadIdx.x; blk < kNumBlocks; blk += blockDim.x) {
    uint32_t s = 0;
    for (int b = 0; b < kBlockBins; ++b) s += pooled[blk * kBlockBins + b];
    blk_tot[blk] = s;
  }
  __syncthreads();

  // 2. candidate thresholds = interpolated quantiles (quant.cpp:20-28)
  const unsigned long long n = static_cast<unsigned long long>(job.per_frame) * F;
  if (threadIdx.x < 2 * nc) {
    const int c = threadIdx.x >> 1;
    const double h = __dmul_rn(cst.pct[c], static_cast<double>(n - 1));
    const unsigned long long lo = static_cast<unsigned long long>(h);
    unsigned long long rank = (threadIdx.x & 1) ? lo + 1 : lo;
    if (rank >= n) rank = n - 1;
    s_rank[threadIdx.x] = rank;
    // bin holding the rank-th smallest |x|
    unsigned long long cum = 0;
    int blk = 0;
    while (blk < kNumBlocks && cum + blk_tot[blk] <= rank) cum += blk_tot[blk++];
    int b = blk * kBlockBins;
    while (cum + pooled[b] <= rank) cum += pooled[b++];
    s_bin[threadIdx.x] = b;
  }
  __syncthreads();
  if (threadIdx.x < nc) {
    const int c = threadIdx.x;
    double thr;
    if (n == 1) {
      thr = bin_value(s_bin[2 * c]);
    } else {
      const double h = __dmul_rn(cst.pct[c], static_cast<double>(n - 1));
      const unsigned long long lo = static_cast<unsigned long long>(h);
      if (lo + 1 >= n) {
        thr = bin_value(s_bin[2 * c + 1]);  // sorted.back()
      } else {
        const double frac = __dsub_rn(h, static_cast<double>(lo));
        const double a = bin_value(s_bin[2 * c]), b = bin_value(s_bin[2 * c + 1]);
        thr = __dadd_rn(a, __dmul_rn(frac, __dsub_rn(b, a)));
      }
    }
    s_thr[c] = thr;
    s_scale[c] = thr > 0.0 ? __ddiv_rn(thr, static_cast<double>(cst.qmax)) : DBL_MIN;
  }
  __syncthreads();

  // 3. per (frame, candidate, block): the block's bins summed in ascending order (the canonical
  //    order; zero counts add +0.0 and are skipped).  Blocks go in groups of kEvalGroup: the
  //    group's squared errors e_c(v_b) are computed once into shared memory, then one thread per
  //    (frame, candidate, block) chain streams its frame's counts of that block.
  double* e_sm = reinterpret_cast<double*>(part + static_cast<size_t>(F) * nc * kNumBlocks);
  const int chains = F * nc * kEvalGroup;
  for (int g0 = 0; g0 < kNumBlocks; g0 += kEvalGroup) {
    for (int i = threadIdx.x; i < nc * kEvalGroup * kBlockBins; i += blockDim.x) {
      const int c = i / (kEvalGroup * kBlockBins), r = i - c * (kEvalGroup * kBlockBins);
      const int b = g0 * kBlockBins + r;
      e_sm[i] = pooled[b] ? fq_err(bin_value(b), s_scale[c], cst.qmax) : 0.0;
    }
    __syncthreads();
    for (int ch = threadIdx.x; ch < chains; ch += blockDim.x) {
      const int gb = ch % kEvalGroup, fc = ch / kEvalGroup;
      const int f = fc / nc, c = fc - f * nc;
      const int blk = g0 + gb;
      double acc = 0.0;
      if (blk_tot[blk]) {
        const uint32_t* h = job.hist + static_cast<int64_t>(f) * kBins + blk * kBlockBins;
        const double* e = e_sm + (c * kEvalGroup + gb) * kBlockBins;
        for (int b = 0; b < kBlockBins; ++b) {
          const uint32_t cnt = __ldg(h + b);
          if (cnt) acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(cnt), e[b]));
        }
      }
      part[(f * nc + c) * kNumBlocks + blk] = acc;
    }
    __syncthreads();
  }
  // 4. per (frame, candidate): sum the block partials in order, / n_f
  for (int item = threadIdx.x; item < F * nc; item += blockDim.x) {
    double t = 0.0;
    for (int blk = 0; blk < kNumBlocks; ++blk) t = __dadd_rn(t, part[item * kNumBlocks + blk]);
    s_mse[item] = __ddiv_rn(t, static_cast<double>(job.per_frame));
  }
  __syncthreads();
  // 5. weighted loss per candidate and the argmin (ties -> later candidate, quant.cpp:219)
  if (threadIdx.x == 0) {
    double best = __longlong_as_double(0x7ff0000000000000ll);
    int best_c = 0;
    for (int c = 0; c < nc; ++c) {
      double loss;
      if (cst.equal_weights) {
        double sum = 0.0;
        for (int f = 0; f < F; ++f) sum = __dadd_rn(sum, s_mse[f * nc + c]);
        loss = __ddiv_rn(sum, static_cast<double>(F));
      } else {
        double sum = 0.0;
        for (int f = 0; f < F; ++f) sum = __dadd_rn(sum, __dmul_rn(cst.w[f], s_mse[f * nc + c]));
        loss = __ddiv_rn(sum, cst.wsum);
      }
      job.result[c] = s_thr[c];
      job.result[nc + c] = s_scale[c];
      job.result[2 * nc + c] = loss;
      if (loss <= best) {
        best = loss;
        best_c = c;
      }
    }
    job.result[3 * nc] = static_cast<double>(best_c);
    job.result[3 * nc + 1] = s_scale[best_c];
  }
}

}  // namespace
}  // namespace qarvd_b200

using namespace qarvd_b200;

namespace qarvd_b200 {
namespace {
int scale_search_impl(const qarvd_search_job* jobs, int num_jobs, const double* percentiles,
                      int num_cand, const double* frame_weights, int bits, void* stream,
                      unsigned long long* err_out);
}  // namespace
}  // namespace qarvd_b200

extern "C" int qarvd_scale_search(const qarvd_search_job* jobs, int num_jobs,
                                  const double* percentiles, int num_cand,
                                  const double* frame_weights, int bits, void* stream) {
  return qarvd_b200::scale_search_impl(jobs, num_jobs, percentiles, num_cand, frame_weights, bits,
                                       stream, nullptr);
}

extern "C" int qarvd_scale_search_async(const qarvd_search_job* jobs, int num_jobs,
                                        const double* percentiles, int num_cand,
                                        const double* frame_weights, int bits,
                                        uint64_t* nonfinite_flag_dev, void* stream) {
  if (!nonfinite_flag_dev) {
    qarvd_b200::clear_error();
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "scale_search_async: null non-finite flag");
  }
  return qarvd_b200::scale_search_impl(jobs, num_jobs, percentiles, num_cand, frame_weights, bits,
                                       stream, reinterpret_cast<unsigned long long*>(nonfinite_flag_dev));
}

namespace qarvd_b200 {
namespace {
int scale_search_impl(const qarvd_search_job* jobs, int num_jobs, const double* percentiles,
                      int num_cand, const double* frame_weights, int bits, void* stream,
                      unsigned long long* err_out) {
  clear_error();
  if (num_jobs < 0 || (num_jobs > 0 && !jobs))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "scale_search: invalid job list");
  if (num_cand < 1 || num_cand > QARVD_MAX_CANDIDATES || !percentiles)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "scale_search: 1..16 candidate percentiles required");
  if (bits < 2 || bits > 30)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT,
               "bit width out of supported range [2,30]: " + std::to_string(bits));
  if (num_jobs == 0) return QARVD_OK;
  const int64_t F = jobs[0].frames;
  if (F < 1 || F > QARVD_MAX_FRAMES)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "percentile search: empty calibration sample list");
  EvalConst cst{};
  for (int c = 0; c < num_cand; ++c) {
    if (!(percentiles[c] >= 0.0 && percentiles[c] <= 1.0))
      QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "scale_search: percentile outside [0,1]");
    cst.pct[c] = percentiles[c];
  }
  cst.nc = num_cand;
  cst.qmax = (1 << (bits - 1)) - 1;
  cst.equal_weights = 1;
  cst.wsum = 0.0;
  for (int f = 0; f < F; ++f) {
    const double w = frame_weights ? frame_weights[f] : 1.0;
    if (!(w >= 0.0) || !(w <= DBL_MAX))
      QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "scale_search: frame weights must be finite and >= 0");
    cst.w[f] = w;
    cst.wsum += w;  // sequential, as the oracle
    if (frame_weights && w != frame_weights[0]) cst.equal_weights = 0;
  }
  if (!(cst.wsum > 0.0)) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "scale_search: frame weights sum to 0");

  std::vector<HistUnit> units;
  std::vector<EvalJob> ejobs(num_jobs);
  const int64_t target_elems = 1 << 20;
  for (int j = 0; j < num_jobs; ++j) {
    const qarvd_search_job& J = jobs[j];
    if (J.frames != F)
      QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "scale_search: all jobs in a batch need the same frame count");
    if (!J.x || !J.result || J.rows <= 0 || J.k <= 0 || J.ldx < J.k)
      QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "scale_search: invalid job " + std::to_string(j));
    if (static_cast<double>(J.rows) * J.k * F >= 4294967296.0)
      QARVD_FAIL(QARVD_ERR_UNSUPPORTED, "scale_search: more than 2^32 elements in one layer");
    ejobs[j] = EvalJob{nullptr, F, J.rows * J.k, J.result};
  }
  if (int st = require_device()) return st;
  cudaStream_t s = as_stream(stream);

  // workspace: histograms [jobs][F][kBins] u32 + error word + job tables
  const size_t hist_bytes = static_cast<size_t>(num_jobs) * F * kBins * sizeof(uint32_t);
  void* ws = nullptr;
  QARVD_CUDA_TRY(cudaMallocAsync(&ws, hist_bytes + 64, s));
  uint32_t* hist = static_cast<uint32_t*>(ws);
  unsigned long long* err =
      reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + hist_bytes);
  QARVD_CUDA_TRY(cudaMemsetAsync(ws, 0, hist_bytes, s));
  QARVD_CUDA_TRY(cudaMemsetAsync(err, 0xff, sizeof(unsigned long long), s));
  for (int j = 0; j < num_jobs; ++j) {
    const qarvd_search_job& J = jobs[j];
    ejobs[j].hist = hist + static_cast<size_t>(j) * F * kBins;
    const int64_t rows_per_unit = std::max<int64_t>(1, target_elems / J.k);
    for (int64_t f = 0; f < F; ++f) {
      for (int64_t r0 = 0; r0 < J.rows; r0 += rows_per_unit) {
        HistUnit u;
        u.x = J.x + (f * J.rows + r0) * J.ldx;
        u.rows = std::min<int64_t>(rows_per_unit, J.rows - r0);
        u.k = J.k;
        u.ldx = J.ldx;
        u.hist = hist + (static_cast<size_t>(j) * F + f) * kBins;
        u.err = err;
        units.push_back(u);
      }
    }
  }
  void* tables = nullptr;
  const size_t tbytes = units.size() * sizeof(HistUnit) + ejobs.size() * sizeof(EvalJob);
  QARVD_CUDA_TRY(cudaMallocAsync(&tables, tbytes, s));
  HistUnit* d_units = static_cast<HistUnit*>(tables);
  EvalJob* d_jobs = reinterpret_cast<EvalJob*>(d_units + units.size());
  QARVD_CUDA_TRY(cudaMemcpyAsync(d_units, units.data(), units.size() * sizeof(HistUnit),
                                 cudaMemcpyHostToDevice, s));
  QARVD_CUDA_TRY(cudaMemcpyAsync(d_jobs, ejobs.data(), ejobs.size() * sizeof(EvalJob),
                                 cudaMemcpyHostToDevice, s));

  const int hist_smem = kBins * sizeof(uint32_t);
  QARVD_CUDA_TRY(
      set_smem_attrs(hist_kernel, hist_smem));
  // persistent grid: one CTA per SM (128 KB of shared memory each)
  const int hist_grid = static_cast<int>(std::min<size_t>(units.size(), static_cast<size_t>(kNumSMs)));
  hist_kernel<<<hist_grid, kHistThreads, hist_smem, s>>>(d_units, static_cast<int>(units.size()));
  count_launch();
  QARVD_LAUNCH_CHECK();

  const size_t eval_smem = kBins * sizeof(uint32_t) + kNumBlocks * sizeof(uint32_t) +
                           static_cast<size_t>(F) * num_cand * kNumBlocks * sizeof(double) +
                           static_cast<size_t>(num_cand) * kEvalGroup * kBlockBins * sizeof(double);
  if (eval_smem > 227 * 1024)
    QARVD_FAIL(QARVD_ERR_UNSUPPORTED, "scale_search: frames x candidates too large for one CTA");
  QARVD_CUDA_TRY(set_smem_attrs(eval_kernel, static_cast<int>(eval_smem)));
  eval_kernel<<<num_jobs, kEvalThreads, eval_smem, s>>>(d_jobs, cst);
  count_launch();
  QARVD_LAUNCH_CHECK();

  // non-finite input check (reference: quantize throws on non-finite, quant.cpp:128-129)
  if (err_out) {  // async variant: the caller checks the flag (~0 = all finite) later
    QARVD_CUDA_TRY(cudaMemcpyAsync(err_out, err, sizeof(unsigned long long), cudaMemcpyDeviceToDevice, s));
    QARVD_CUDA_TRY(cudaFreeAsync(tables, s));
    QARVD_CUDA_TRY(cudaFreeAsync(ws, s));
    return QARVD_OK;
  }
  unsigned long long h_err = ~0ull;
  QARVD_CUDA_TRY(cudaMemcpyAsync(&h_err, err, sizeof(h_err), cudaMemcpyDeviceToHost, s));
  QARVD_CUDA_TRY(cudaFreeAsync(tables, s));
  QARVD_CUDA_TRY(cudaFreeAsync(ws, s));
  QARVD_CUDA_TRY(cudaStreamSynchronize(s));
  if (h_err != ~0ull)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "quantize: non-finite input in calibration samples");
  return QARVD_OK;
}
}  // namespace
}  // namespace qarvd_b200
