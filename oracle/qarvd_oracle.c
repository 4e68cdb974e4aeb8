/*
 * qarvd_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Plain-C restatement of the Q-ARVD reference hot path
 * (/root/reference/proj/core/src), compiled with -ffp-contract=off so every
 * f64 expression rounds exactly like the reference's Release build (which has
 * no FMA instructions).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library.
 *
 * Pinned against: the compiled reference itself (oracle/_ref/libqarvd_ref.so,
 * built from the reference sources by oracle/Makefile) and the SPEC.md
 * known-answer examples; see tests/test_oracle_*.py and tests/golden/.
 *
 * Additions beyond the reference (documented in DESIGN.md): per-token
 * activation scales, an optional bias (D2), the fp32 epilogue
 * restatement of the GPU kernel, and the histogram form of the frame-weighted
 * scale search (D5) in its canonical summation order.
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ---- scalar helpers ------------------------------------------------------ */

/* round_half_even, quant.hpp:14-20 */
double oracle_round_half_even(double v) {
  const double fl = floor(v);
  const double diff = v - fl;
  if (diff > 0.5) return fl + 1.0;
  if (diff < 0.5) return fl;
  return (fmod(fl, 2.0) == 0.0) ? fl : fl + 1.0;
}

/* code = clamp(round_half_even(v / s), -qmax, qmax), quant.cpp:130-135 */
static int32_t code_of(double v, double s, int qmax) {
  const double q = oracle_round_half_even(v / s);
  if (q > (double)qmax) return qmax;
  if (q < -(double)qmax) return -qmax;
  return (int32_t)q;
}

/* bf16 <-> float, bytes.hpp:40-52 */
uint16_t oracle_float_to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  const uint32_t rounding = 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)((u + rounding) >> 16);
}
float oracle_bf16_to_float(uint16_t h) {
  const uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* ---- K1: permute + quantize (engine.cpp:32-44, quant.cpp:113-138, :161-183) --
 * x f64 [m x k]; gather[k_out] source column or -1 (NULL = identity).
 * per_token: scale_i = max_c |x_ic| / qmax (init_scale_minmax axis 0), DBL_MIN if 0.
 * else: static scale for every row.  Returns -1, or the first flat index
 * (row * k_out + c, gathered coordinates) with a non-finite value. */
int64_t oracle_quantize_act(const double* x, int64_t m, int64_t k, const int32_t* gather,
                            int64_t k_out, int per_token, double static_scale, int bits,
                            int8_t* q, double* scales) {
  const int qmax = (1 << (bits - 1)) - 1;
  int64_t first_bad = -1;
  for (int64_t i = 0; i < m && first_bad < 0; ++i)
    for (int64_t c = 0; c < k_out; ++c) {
      const int32_t src = gather ? gather[c] : (int32_t)c;
      if (src >= 0 && !isfinite(x[i * k + src])) {
        first_bad = i * k_out + c;
        break;
      }
    }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    const double* xr = x + i * k;
    double s = static_scale;
    if (per_token) {
      double absmax = 0.0;
      for (int64_t c = 0; c < k; ++c) {
        const double a = fabs(xr[c]);
        absmax = absmax < a ? a : absmax; /* std::max(absmax, |x|) */
      }
      s = absmax > 0.0 ? absmax / (double)qmax : DBL_MIN;
    }
    if (scales) scales[i] = s;
    for (int64_t c = 0; c < k_out; ++c) {
      const int32_t src = gather ? gather[c] : (int32_t)c;
      q[i * k_out + c] =
          (src < 0 || !isfinite(xr[src])) ? 0 : (int8_t)code_of(xr[src], s, qmax);
    }
  }
  return first_bad;
}

/* ---- K5: dual-scale weight prep (dual_scale.cpp:13-24, :58-114; calibrate.cpp:474-480) --
 * Group scales per output row over gathered columns [0, k_o) and [k_o, k_pad);
 * codes pre-permuted, pads 0.  k_o == 0: single-scale plan, s_o = s_n. */
int64_t oracle_prepare_weights(const double* w, int64_t n, int64_t k, const int32_t* gather,
                               int64_t k_pad, int64_t k_o, int bits, int8_t* wq, double* s_o,
                               double* s_n) {
  const int qmax = (1 << (bits - 1)) - 1;
  int64_t first_bad = -1;
  for (int64_t r = 0; r < n && first_bad < 0; ++r)
    for (int64_t c = 0; c < k_pad; ++c) {
      const int32_t src = gather ? gather[c] : (int32_t)c;
      if (src >= 0 && !isfinite(w[r * k + src])) {
        first_bad = r * k_pad + c;
        break;
      }
    }
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < n; ++r) {
    const double* wr = w + r * k;
    double ao = 0.0, an = 0.0;
    for (int64_t c = 0; c < k_pad; ++c) {
      const int32_t src = gather ? gather[c] : (int32_t)c;
      if (src < 0) continue;
      const double a = fabs(wr[src]);
      if (c < k_o) ao = ao < a ? a : ao;
      else an = an < a ? a : an;
    }
    const double sn = an > 0.0 ? an / (double)qmax : DBL_MIN;
    const double so = k_o > 0 ? (ao > 0.0 ? ao / (double)qmax : DBL_MIN) : sn;
    if (s_o) s_o[r] = so;
    if (s_n) s_n[r] = sn;
    for (int64_t c = 0; c < k_pad; ++c) {
      const int32_t src = gather ? gather[c] : (int32_t)c;
      wq[r * k_pad + c] = src < 0 ? 0 : (int8_t)code_of(wr[src], c < k_o ? so : sn, qmax);
    }
  }
  return first_bad;
}

/* ---- K2 reference: kernel_b_gemm_dequant (engine.cpp:46-105) ----------------
 * exact int64 group dots, then val = sum_g (s_x*s_w[g][j]) * acc_g, outlier
 * group first; per-row s_x (rows are independent, engine.cpp:86).  Optional
 * int32 dumps of the two group accumulators. */
void oracle_kernel_b(const int8_t* xq, const int8_t* wq, int64_t m, int64_t n, int64_t k,
                     int64_t k_o, const double* s_x, const double* s_o, const double* s_n,
                     double* out, int32_t* acc_o, int32_t* acc_n) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    const int8_t* xr = xq + i * k;
    for (int64_t j = 0; j < n; ++j) {
      const int8_t* wr = wq + j * k;
      int64_t ao = 0, an = 0;
      for (int64_t c = 0; c < k_o; ++c) ao += (int64_t)xr[c] * (int64_t)wr[c];
      for (int64_t c = k_o; c < k; ++c) an += (int64_t)xr[c] * (int64_t)wr[c];
      double val = 0.0;
      if (k_o > 0) val += (s_x[i] * s_o[j]) * (double)ao;
      val += (s_x[i] * s_n[j]) * (double)an;
      if (out) out[i * n + j] = val;
      if (acc_o) acc_o[i * n + j] = (int32_t)ao;
      if (acc_n) acc_n[i * n + j] = (int32_t)an;
    }
  }
}

/* ---- fp32 restatement of the GPU epilogue (dual_gemm.cu), bit-exact --------
 * t = s_o*float(acc_o); t = fmaf(s_n, float(acc_n), t)   (k_o > 0)
 * t = s_n*float(acc_n)                                   (k_o == 0)
 * y = bias ? fmaf(s_x, t, bias) : s_x*t;  -> bf16 RNE (out_bf16) or f32. */
void oracle_epilogue_f32(const int32_t* acc_o, const int32_t* acc_n, int64_t m, int64_t n,
                         int has_outlier, const float* s_x, const float* s_o, const float* s_n,
                         const float* bias, uint16_t* out_bf16, float* out_f32) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      const float an = (float)acc_n[i * n + j];
      float t;
      if (has_outlier) t = fmaf(s_n[j], an, s_o[j] * (float)acc_o[i * n + j]);
      else t = s_n[j] * an;
      const float y = bias ? fmaf(s_x[i], t, bias[j]) : s_x[i] * t;
      if (out_bf16) out_bf16[i * n + j] = oracle_float_to_bf16(y);
      if (out_f32) out_f32[i * n + j] = y;
    }
}

/* ---- K3: outlier detection ---------------------------------------------------
 * channel_l2_norms(W, 1), tensor.cpp:132-150: rows summed in order, mul + add */
void oracle_channel_norms(const double* w, int64_t n, int64_t k, double* norms) {
  for (int64_t j = 0; j < k; ++j) norms[j] = 0.0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < k; ++j) {
      const double p = w[i * k + j] * w[i * k + j];
      norms[j] = norms[j] + p;
    }
  for (int64_t j = 0; j < k; ++j) norms[j] = sqrt(norms[j]);
}

static int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* sorted_median + mad, outlier.cpp:13-18, :30-38 */
void oracle_mad(const double* v, int64_t n, double* median, double* mad) {
  double* tmp = (double*)malloc(sizeof(double) * (size_t)n);
  memcpy(tmp, v, sizeof(double) * (size_t)n);
  qsort(tmp, (size_t)n, sizeof(double), cmp_double);
  const double med = (n % 2 == 1) ? tmp[n / 2] : 0.5 * (tmp[n / 2 - 1] + tmp[n / 2]);
  for (int64_t i = 0; i < n; ++i) tmp[i] = fabs(v[i] - med);
  qsort(tmp, (size_t)n, sizeof(double), cmp_double);
  *mad = (n % 2 == 1) ? tmp[n / 2] : 0.5 * (tmp[n / 2 - 1] + tmp[n / 2]);
  *median = med;
  free(tmp);
}

static const double* g_sort_norms;
/* stable order: norm descending, index ascending (outlier.cpp:67-70) */
static int cmp_desc_idx(const void* a, const void* b) {
  const int64_t i = *(const int64_t*)a, j = *(const int64_t*)b;
  const double x = g_sort_norms[i], y = g_sort_norms[j];
  if (x != y) return x > y ? -1 : 1;
  return (i > j) - (i < j);
}
static int cmp_i64(const void* a, const void* b) {
  const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

/* analyze_norms (outlier.cpp:80-96) = mad -> threshold -> detect (:40-52) -> align (:54-78).
 * stats = {median, mad, threshold}; counts = {|raw|, |aligned|}. Not thread-safe. */
void oracle_analyze_norms(const double* norms, int64_t k, double tau, double alpha_min,
                          int64_t align, double* stats, int64_t* counts, int64_t* raw,
                          int64_t* aligned) {
  double med, mad;
  oracle_mad(norms, k, &med, &mad);
  const double a = med + (tau / 0.6745) * mad;
  const double b = alpha_min * med;
  const double thr = a < b ? b : a;
  int64_t R = 0;
  for (int64_t i = 0; i < k; ++i)
    if (norms[i] > thr) raw[R++] = i;
  int64_t A;
  if (R == 0) {
    A = 0;
  } else if (k < 2 * align) {
    memcpy(aligned, raw, sizeof(int64_t) * (size_t)R);
    A = R;
  } else {
    int64_t target = ((R + align - 1) / align) * align;
    const int64_t cap = k - align;
    int use_raw = 0;
    if (target > cap) {
      target = (cap / align) * align;
      if (target < R) use_raw = 1;
    }
    if (use_raw) {
      memcpy(aligned, raw, sizeof(int64_t) * (size_t)R);
      A = R;
    } else {
      int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
      for (int64_t i = 0; i < k; ++i) order[i] = i;
      g_sort_norms = norms;
      qsort(order, (size_t)k, sizeof(int64_t), cmp_desc_idx); /* total order => stable */
      memcpy(aligned, order, sizeof(int64_t) * (size_t)target);
      qsort(aligned, (size_t)target, sizeof(int64_t), cmp_i64);
      A = target;
      free(order);
    }
  }
  stats[0] = med;
  stats[1] = mad;
  stats[2] = thr;
  counts[0] = R;
  counts[1] = A;
}

/* ---- K4: frame-weighted scale search, histogram form (search.cu) ------------
 * x: bf16 bits [frames*rows x k].  result[3*nc+2] = thresholds, scales, losses,
 * best index, best scale.  Canonical summation order: 128 blocks x 256 bins,
 * ascending inside a block, then block partials ascending.  Equal weights (or
 * weights == NULL) use (1/S) * sum_f mse_f exactly as quant.cpp:216-217. */
#define K4_BINS 32768
#define K4_BLOCK 256
#define K4_NBLK (K4_BINS / K4_BLOCK)

static double bin_value(int b) { return (double)oracle_bf16_to_float((uint16_t)b); }

static double fq_err(double v, double s, int qmax) {
  double q = oracle_round_half_even(v / s);
  if (q > (double)qmax) q = (double)qmax;
  const double d = v - q * s;
  return d * d;
}

int oracle_scale_search_hist(const uint16_t* x, int64_t frames, int64_t rows, int64_t k,
                             const double* pct, int nc, const double* weights, int bits,
                             double* result) {
  const int qmax = (1 << (bits - 1)) - 1;
  const int64_t per_frame = rows * k;
  uint32_t* hist = (uint32_t*)calloc((size_t)frames * K4_BINS, sizeof(uint32_t));
  uint64_t* pooled = (uint64_t*)calloc(K4_BINS, sizeof(uint64_t));
  if (!hist || !pooled) return -1;
  for (int64_t f = 0; f < frames; ++f)
    for (int64_t e = 0; e < per_frame; ++e) {
      const uint16_t b = x[f * per_frame + e] & 0x7fffu;
      if (b >= 0x7f80u) {
        free(hist);
        free(pooled);
        return 1; /* non-finite */
      }
      hist[f * K4_BINS + b]++;
    }
  for (int64_t f = 0; f < frames; ++f)
    for (int b = 0; b < K4_BINS; ++b) pooled[b] += hist[f * K4_BINS + b];
  const uint64_t n = (uint64_t)per_frame * (uint64_t)frames;

  /* order statistic of rank r (0-based) -> bin value */
  double* thr = result;
  double* scale = result + nc;
  double* loss = result + 2 * nc;
  for (int c = 0; c < nc; ++c) {
    double t;
    uint64_t ranks[2];
    const double h = pct[c] * (double)(n - 1);
    const uint64_t lo = (uint64_t)h;
    ranks[0] = lo;
    ranks[1] = lo + 1 < n ? lo + 1 : n - 1;
    double vals[2];
    for (int r = 0; r < 2; ++r) {
      uint64_t cum = 0;
      int b = 0;
      while (cum + pooled[b] <= ranks[r]) cum += pooled[b++];
      vals[r] = bin_value(b);
    }
    if (n == 1) t = vals[0];
    else if (lo + 1 >= n) t = vals[1];
    else {
      const double frac = h - (double)lo;
      t = vals[0] + frac * (vals[1] - vals[0]);
    }
    thr[c] = t;
    scale[c] = t > 0.0 ? t / (double)qmax : DBL_MIN;
  }
  int equal = 1;
  double wsum = 0.0;
  for (int64_t f = 0; f < frames; ++f) {
    const double w = weights ? weights[f] : 1.0;
    wsum += w;
    if (weights && w != weights[0]) equal = 0;
  }
  double* mse = (double*)malloc(sizeof(double) * (size_t)(frames * nc));
  for (int c = 0; c < nc; ++c)
    for (int64_t f = 0; f < frames; ++f) {
      double total = 0.0;
      for (int blk = 0; blk < K4_NBLK; ++blk) {
        double part = 0.0;
        for (int b = blk * K4_BLOCK; b < (blk + 1) * K4_BLOCK; ++b) {
          if (!pooled[b]) continue;
          const double e = fq_err(bin_value(b), scale[c], qmax);
          part = part + (double)hist[f * K4_BINS + b] * e;
        }
        total = total + part;
      }
      mse[f * nc + c] = total / (double)per_frame;
    }
  double best = INFINITY;
  int best_c = 0;
  for (int c = 0; c < nc; ++c) {
    double sum = 0.0;
    if (equal) {
      for (int64_t f = 0; f < frames; ++f) sum = sum + mse[f * nc + c];
      loss[c] = sum / (double)frames;
    } else {
      for (int64_t f = 0; f < frames; ++f) sum = sum + weights[f] * mse[f * nc + c];
      loss[c] = sum / wsum;
    }
    if (loss[c] <= best) {
      best = loss[c];
      best_c = c;
    }
  }
  result[3 * nc] = (double)best_c;
  result[3 * nc + 1] = scale[best_c];
  free(mse);
  free(hist);
  free(pooled);
  return 0;
}

/* ---- frame weights, weighting_strategy (sensitivity.cpp:86-112) -------------
 * kind: 0 uniform, 1 heuristic_exp, 2 reverse, 3 final_quality; alpha = normalized profile */
void oracle_weighting(int kind, const double* alpha, int64_t n, double* w) {
  if (kind == 0) {
    for (int64_t i = 0; i < n; ++i) w[i] = 1.0 / (double)n;
  } else if (kind == 1) {
    double total = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      w[i] = pow(2.0, -(double)(i + 1));
      total += w[i];
    }
    for (int64_t i = 0; i < n; ++i) w[i] /= total;
  } else if (kind == 2) {
    for (int64_t i = 0; i < n; ++i) w[i] = alpha[n - 1 - i];
  } else {
    for (int64_t i = 0; i < n; ++i) w[i] = alpha[i];
  }
}

/* normalize_alpha, sensitivity.cpp:16-27 */
void oracle_normalize_alpha(const double* raw, int64_t n, double* out) {
  double total = 0.0;
  for (int64_t i = 0; i < n; ++i) total += raw[i];
  for (int64_t i = 0; i < n; ++i) out[i] = total <= 0.0 ? 1.0 / (double)n : raw[i] / total;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Check of the device's row-scale formula (quantize.cu row_s64): for every positive
 * finite bf16 amax and every qmax of 2..8 bits, y = amax * fl(1/qmax) corrected by one
 * fma equals the correctly rounded fl(amax / qmax) of quant.cpp:168-181.  Returns the
 * number of mismatches (0). */
int64_t oracle_row_scale_formula_mismatches(void) {
  int64_t bad = 0;
  for (int b = 2; b <= 8; ++b) {
    const double q = (double)((1 << (b - 1)) - 1);
    const double rq = 1.0 / q;
    for (uint32_t h = 1; h < 0x7f80u; ++h) {
      const uint32_t u = h << 16;
      float f;
      memcpy(&f, &u, 4);
      const double a = (double)f;
      const double y = a * rq;
      const double y2 = fma(fma(-y, q, a), rq, y);
      if (y2 != a / q) ++bad;
    }
  }
  return bad;
}

/* ---- Eq. 5 frame-weighted reconstruction loss ------------------------------
 * weighted_recon_loss (calibrate.cpp:201-216) with the deployable weights:
 *   (1/B) sum_s w[chunk_s - 1] * || X_s W^T - FQ(X_s) What^T ||_F^2
 * target = matmul_nt(X, W) (tensor.cpp:82-105: c(i,j) += a(i,k) * b(k,j), k ascending
 * from 0.0); FQ(X) = (q - 0) * s_x (quant.cpp:140-159, per-tensor act params);
 * What = s_g(row) * code (calibrate.cpp:128-147, hard rounding); the squared distance
 * accumulates row-major (tensor.cpp:116-126).  x [m x k] stacks the samples (rows
 * row_off[s] .. row_off[s+1]); codes / w are in ORIGINAL column order; xq are the
 * activation codes (row-major [m x k], original order); s_wo / s_wn per output row,
 * outlier_mask[c] = 1 for outlier columns.  err[s] receives each sample's distance.
 * Returns 0, or 1 for an empty batch, 2 for a chunk outside [1, n_chunks]. */
int oracle_weighted_loss(const double* x, const int32_t* xq, double s_x, const double* w,
                         const int32_t* codes, const double* s_wo, const double* s_wn,
                         const uint8_t* outlier_mask, int64_t m, int64_t n, int64_t k,
                         const int64_t* row_off, const int64_t* chunk, int64_t n_samples,
                         const double* chunk_w, int64_t n_chunks, double* err, double* loss) {
  if (n_samples <= 0) return 1;
  (void)m;
  double* what = (double*)malloc(sizeof(double) * (size_t)(n * k));
  double* t = (double*)malloc(sizeof(double) * (size_t)n);
  double* p = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t j = 0; j < n; ++j)
    for (int64_t c = 0; c < k; ++c)
      what[j * k + c] = (outlier_mask[c] ? s_wo[j] : s_wn[j]) * (double)codes[j * k + c];
  double total = 0.0;
  int st = 0;
  for (int64_t s = 0; s < n_samples && !st; ++s) {
    if (chunk[s] < 1 || chunk[s] > n_chunks) { st = 2; break; }
    double acc = 0.0;
    for (int64_t i = row_off[s]; i < row_off[s + 1]; ++i) {
      for (int64_t j = 0; j < n; ++j) { t[j] = 0.0; p[j] = 0.0; }
      for (int64_t c = 0; c < k; ++c) {
        const double av = x[i * k + c];
        const double fq = (double)xq[i * k + c] * s_x;
        for (int64_t j = 0; j < n; ++j) {
          t[j] += av * w[j * k + c];
          p[j] += fq * what[j * k + c];
        }
      }
      for (int64_t j = 0; j < n; ++j) {
        const double d = t[j] - p[j];
        acc += d * d;
      }
    }
    err[s] = acc;
    total += chunk_w[chunk[s] - 1] * acc;
  }
  if (!st) *loss = total / (double)n_samples;
  free(what);
  free(t);
  free(p);
  return st;
}
