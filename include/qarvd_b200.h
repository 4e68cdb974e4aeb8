/*
 * qarvd_b200.h — C-ABI of the B200-native Q-ARVD quantized-inference and
 * calibration hot path (libqarvd_b200.so).
 *
 * Every entry point replaces one operator of the reference C++ core
 * (/root/reference/proj/core); the citation above each declaration names the
 * reference interface it stands in for.  The reference works on host f64
 * std::vector tensors and throws C++ exceptions; this ABI works on DEVICE
 * pointers + sizes + a cudaStream_t (passed as void*) and returns an int
 * status plus a thread-local message (qarvd_last_error).  The C++ adapter in
 * paper_2605_21072_b200/adapter/ maps statuses back onto the reference's
 * exception types (std::invalid_argument, std::out_of_range, std::logic_error,
 * std::runtime_error) with the reference's message prefixes.
 *
 * Layout conventions (identical to the reference, tensor.hpp:67-70):
 *   activations X  row-major [m x k]   (ld = elements between rows)
 *   weights     W  row-major [n x k]   (both GEMM operands are K-major)
 *   permuted / padded K axis: `gather[c]` = source column of output column c,
 *   or -1 for a zero pad column.  A dual-scale plan's permutation
 *   [outlier | normal] (dual_scale.cpp:81-83) becomes
 *   gather = [outliers..., (-1 pad to a multiple of 32)..., normals..., (-1 pad)]
 *   and k_outlier is the padded outlier-slab width (a multiple of 32).
 *
 * No torch types cross this boundary.  No CPU fallback exists behind it: when
 * no CUDA device is present every compute entry point returns
 * QARVD_ERR_CUDA.
 */
#ifndef QARVD_B200_H
#define QARVD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QARVD_B200_ABI_VERSION 1

/* ---- status codes (mapped to the reference's exception types) ---------- */
enum {
  QARVD_OK = 0,
  QARVD_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument (quant.cpp:59-80, engine.cpp:47-50) */
  QARVD_ERR_OUT_OF_RANGE = 2,     /* std::out_of_range (engine.cpp:29, dual_scale.cpp:63-64)  */
  QARVD_ERR_LOGIC = 3,            /* std::logic_error (engine.cpp:54-55)                      */
  QARVD_ERR_RUNTIME = 4,          /* std::runtime_error                                      */
  QARVD_ERR_CUDA = 5,             /* CUDA / driver failure, or no device                     */
  QARVD_ERR_UNSUPPORTED = 6       /* valid for the reference, outside this build's envelope  */
};

/* element types for X / W inputs and GEMM outputs */
enum { QARVD_BF16 = 0, QARVD_F32 = 1, QARVD_F64 = 2 };

/* activation quantizer granularity */
enum {
  QARVD_ACT_PER_TOKEN = 0,  /* init_scale_minmax(x, b, per_channel, axis 0) (quant.cpp:170-182) */
  QARVD_ACT_PER_TENSOR = 1  /* QuantParams::per_tensor_symmetric(b, s), static (engine.cpp:57)   */
};

/* GEMM epilogue options (bit flags) */
enum {
  QARVD_EPI_NONE = 0,
  QARVD_EPI_GELU = 1 /* y = gelu_erf(y) after dequant + bias (toy_model.cpp:62-66 uses the erf form) */
};

int qarvd_abi_version(void);
/* Thread-local message of the last failing call on this thread ("" if none). */
const char* qarvd_last_error(void);
/* Number of CUDA devices visible (0 on a CPU-only host). Never fails. */
int qarvd_device_count(void);
/* Kernel launches issued by this library since load (all threads). */
uint64_t qarvd_launch_count(void);

/* ---- K1: activation quantization fused with the dual-scale permutation --
 * Replaces  kernel_a_quantize_activation(permute_activations(x, plan), p)
 *           engine.hpp:43 / engine.cpp:32-44, numeric contract quant.cpp:113-138.
 * x       : device [m x k] (ldx), dtype QARVD_BF16 | QARVD_F32 | QARVD_F64.
 * gather  : device int32 [k_out] source column per output column (-1 = zero);
 *           NULL = identity (k_out must equal k).
 * granularity: QARVD_ACT_PER_TOKEN (scale = rowmax|x| / qmax, computed here)
 *           or QARVD_ACT_PER_TENSOR (scale = static_scale, validated > 0 finite).
 * bits    : 2..8, symmetric range +-(2^(bits-1)-1) (quant.hpp:36).
 * xq      : device int8 [m x k_out] (ldq), codes in gathered order.
 * scale_f32 / scale_f64 : device [m] per-row scale (per-tensor: replicated);
 *           either may be NULL.  All-zero rows get DBL_MIN / 0.0f (quant.cpp:164).
 * err_index: device int64[1] or NULL.  Receives the smallest flat index
 *           (row*k_out + c, gathered coordinates) holding a non-finite input,
 *           or INT64_MAX.  The reference throws
 *           "quantize: non-finite input at flat index N" (quant.cpp:128-129);
 *           the adapter reproduces that from this value.
 * Codes are bit-identical to round_half_even(v / s) in f64 (quant.hpp:14-20).
 */
int qarvd_quantize_act(const void* x, int x_dtype, int64_t m, int64_t k, int64_t ldx,
                       const int32_t* gather, int64_t k_out, int granularity,
                       double static_scale, int bits, int8_t* xq, int64_t ldq,
                       float* scale_f32, double* scale_f64, int64_t* err_index,
                       void* stream);

/* K1 for bf16 rows already in plan order (identity gather, k_out = k) whose |x| max is
 * known: per-token with row_absmax from the producer (qarvd_dual_gemm_rowmax), or a
 * static per-tensor scale (row_absmax unused, may be NULL).  Same codes, scales and
 * error reporting as qarvd_quantize_act(x, QARVD_BF16, m, k, ldx, NULL, k, ...);
 * per-token rows reset their row_absmax entry to 0.  k, ldx, ldq multiples of 8. */
int qarvd_quantize_act_rowmax(const uint16_t* x, int64_t m, int64_t k, int64_t ldx,
                              uint32_t* row_absmax, int granularity, double static_scale,
                              int bits, int8_t* xq, int64_t ldq, float* scale_f32,
                              double* scale_f64, int64_t* err_index, void* stream);

/* K1 for bf16 rows in plan order (identity gather, k_out = k, k >= 512) whose |x| max
 * comes from a producer's partial maxima: row_pmax [m x pm_count] as written by
 * qarvd_dual_gemm_pmax (per-token), or a static per-tensor scale (row_pmax unused).  Same
 * codes, scales and error reporting as qarvd_quantize_act(x, QARVD_BF16, m, k, ldx, NULL,
 * k, ...); a flat streaming pass (no per-row synchronisation, nothing to reset). */
int qarvd_quantize_act_pmax(const uint16_t* x, int64_t m, int64_t k, int64_t ldx,
                            const uint32_t* row_pmax, int64_t pm_count, int granularity,
                            double static_scale, int bits, int8_t* xq, int64_t ldq,
                            float* scale_f32, double* scale_f64, int64_t* err_index, void* stream);

/* ---- K5: dual-scale weight preparation ----------------------------------
 * Replaces  build_plan scales (dual_scale.cpp:13-24, :58-90) +
 *           nearest-rounding codes of fake_quant_dual (dual_scale.cpp:92-114) +
 *           the pre-permute of calibrate.cpp:474-480.
 * w       : device [n x k] (ldw), dtype as above.
 * gather  : device int32 [k_pad] (see header comment); NULL = identity.
 * k_outlier: outlier-slab width in gathered coordinates (0 = single-scale plan,
 *           build_single_scale_plan dual_scale.cpp:44-56).
 * wq      : device int8 [n x k_pad] (ldq) pre-permuted codes.
 * scale_*_f64 / _f32 : device [n] per-row group scales (absmax/qmax, DBL_MIN
 *           when the group is all zero); any may be NULL.  For k_outlier == 0
 *           the outlier scales equal the normal ones (dual_scale.cpp:55).
 * err_index: as for qarvd_quantize_act (reference: "fake_quant_dual: non-finite
 *           weight element").
 */
int qarvd_prepare_weights(const void* w, int w_dtype, int64_t n, int64_t k, int64_t ldw,
                          const int32_t* gather, int64_t k_pad, int64_t k_outlier, int bits,
                          int8_t* wq, int64_t ldq, double* scale_outlier_f64,
                          double* scale_normal_f64, float* scale_outlier_f32,
                          float* scale_normal_f32, int64_t* err_index, void* stream);

/* K5 batched over layers (one launch for a whole calibration step).  Each job is one
 * qarvd_prepare_weights call's arguments; all jobs share w_dtype and bits.  bf16 jobs
 * with k <= 12288 run in one batched kernel, others take the per-layer kernel.
 * err_index: min over jobs of the first non-finite index (as for prepare_weights), or NULL. */
typedef struct qarvd_weight_job {
  const void* w;              /* device [n x k] (ldw) weights                          */
  int64_t n, k, ldw;
  const int32_t* gather;      /* device int32 [k_pad] plan gather                      */
  int64_t k_pad, k_outlier;
  int8_t* wq;                 /* out device int8 [n x k_pad] (ldq)                     */
  int64_t ldq;
  double* scale_outlier_f64;  /* out device [n] each; any may be NULL                  */
  double* scale_normal_f64;
  float* scale_outlier_f32;
  float* scale_normal_f32;
} qarvd_weight_job;
int qarvd_prepare_weights_batched(const qarvd_weight_job* jobs, int num_jobs, int w_dtype,
                                  int bits, int64_t* err_index, void* stream);

/* K3 -> plan -> K5 without a host round trip: the plan's column split (build_plan,
 * dual_scale.cpp:44-90) is built on the device from K3's aligned outlier set, then the batched
 * K5 reads it.  bf16 weights, rows of <= 10240 values.
 *   aligned_idx / counts: qarvd_analyze_layers outputs (counts[1] = |aligned|)
 *   gather: out device int32 [gather_cap >= k + 64]; plan_info: out device int64 {k_outlier, k_pad}
 *   wq: out [n x ldq], ldq >= k + 64 (only the first k_pad columns of each row are written). */
typedef struct qarvd_planned_weight_job {
  const void* w;
  int64_t n, k, ldw;
  const int32_t* aligned_idx;
  const int32_t* counts;
  int32_t* gather;
  int64_t gather_cap;
  int64_t* plan_info;
  int8_t* wq;
  int64_t ldq;
  double* scale_outlier_f64;
  double* scale_normal_f64;
  float* scale_outlier_f32;
  float* scale_normal_f32;
} qarvd_planned_weight_job;
int qarvd_prepare_weights_planned(const qarvd_planned_weight_job* jobs, int num_jobs, int bits,
                                  int64_t* err_index, void* stream);

/* ---- K2: dual-scale W8A8 GEMM + dequant + bias epilogue ------------------
 * Replaces  kernel_b_gemm_dequant(xq, layer)  engine.hpp:48 / engine.cpp:46-105
 * (symmetric activations; the reference's zero-point correction, engine.cpp:95-100,
 * is returned as QARVD_ERR_UNSUPPORTED by the adapter).
 * xq [m x k] (ldq), wq [n x k] (ldw): int8 codes, both already in
 *           [outlier | normal] order.  k % 32 == 0, k_outlier % 32 == 0,
 *           0 <= k_outlier < k, ldq/ldw multiples of 16, pointers 16-B aligned.
 *           k <= 132104 keeps the int32 accumulators exact (127*127*k < 2^31).
 * Two int32 tensor-memory accumulators per tile:
 *           acc_o = sum_{c <  k_outlier} xq[i,c]*wq[j,c]
 *           acc_n = sum_{c >= k_outlier} xq[i,c]*wq[j,c]
 * Epilogue (fp32, this exact op order):
 *           t = s_wo[j]*float(acc_o);  t = fmaf(s_wn[j], float(acc_n), t);
 *           y = bias ? fmaf(s_x[i], t, bias[j]) : s_x[i]*t;  [gelu]; round to out dtype (RNE).
 * scale_x : device f32 [m];  scale_w_outlier / scale_w_normal : device f32 [n].
 * bias    : device f32 [n] or NULL (reference parity: NULL).
 * y       : device [m x n] (ldy), out_dtype QARVD_BF16 or QARVD_F32.
 * acc_outlier / acc_normal : device int32 [m x n] debug dumps or NULL.
 */
int qarvd_dual_gemm(const int8_t* xq, int64_t ldq, const int8_t* wq, int64_t ldw, int64_t m,
                    int64_t n, int64_t k, int64_t k_outlier, const float* scale_x,
                    const float* scale_w_outlier, const float* scale_w_normal, const float* bias,
                    int epilogue, int out_dtype, void* y, int64_t ldy, int32_t* acc_outlier,
                    int32_t* acc_normal, void* stream);

/* K2 for a chained producer: bf16 y as qarvd_dual_gemm, plus
 *   row_absmax[i] = max(row_absmax[i], max_j (bf16 bits of y[i,j]) & 0x7fff)
 * (the per-token |y| max the next layer's K1 needs, reduced in the epilogue instead of
 * re-reading y).  row_absmax: device uint32 [m], zero before the first step; the
 * consumer's qarvd_quantize_act_rowmax resets it.  No reference counterpart: the fusion
 * of engine.cpp:134-142 (layer i output) with quant.cpp:170-182 (layer i+1 scales). */
int qarvd_dual_gemm_rowmax(const int8_t* xq, int64_t ldq, const int8_t* wq, int64_t ldw, int64_t m,
                           int64_t n, int64_t k, int64_t k_outlier, const float* scale_x,
                           const float* scale_w_outlier, const float* scale_w_normal,
                           const float* bias, int epilogue, uint16_t* y, int64_t ldy,
                           uint32_t* row_absmax, void* stream);

/* K2 for a chained producer, plain-store variant: bf16 y as qarvd_dual_gemm, plus
 *   row_pmax[i * pm_count + p] = max over output columns of tile/epilogue-warp p of
 *                                (bf16 bits of y[i, j]) & 0x7fff,
 * pm_count = qarvd_dual_gemm_pmax_count(m, n, k) partials per row, rewritten every call. */
/* Stream-K variant of qarvd_dual_gemm for bf16 outputs: when the last wave of 256 x 256 pair
 * tiles is partial and K is long, the remainder tiles are split along K over all SM pairs
 * (int32 partial sums of the normal slab exchanged through `workspace`, exact).  Results are
 * bit-identical to qarvd_dual_gemm.  workspace: device, 256-byte aligned, ZERO-FILLED once
 * before first use (its counters reset themselves), >= qarvd_dual_gemm_workspace_size bytes
 * (0 = this shape runs data-parallel; the call then ignores the workspace).  One workspace
 * per concurrently running call. */
int64_t qarvd_dual_gemm_workspace_size(int64_t m, int64_t n, int64_t k, int64_t k_outlier);
int qarvd_dual_gemm_ws(const int8_t* xq, int64_t ldq, const int8_t* wq, int64_t ldw, int64_t m,
                       int64_t n, int64_t k, int64_t k_outlier, const float* scale_x,
                       const float* scale_w_outlier, const float* scale_w_normal, const float* bias,
                       int epilogue, uint16_t* y, int64_t ldy, void* workspace,
                       int64_t workspace_bytes, void* stream);
int64_t qarvd_dual_gemm_pmax_count(int64_t m, int64_t n, int64_t k);
int qarvd_dual_gemm_pmax(const int8_t* xq, int64_t ldq, const int8_t* wq, int64_t ldw, int64_t m,
                         int64_t n, int64_t k, int64_t k_outlier, const float* scale_x,
                         const float* scale_w_outlier, const float* scale_w_normal,
                         const float* bias, int epilogue, uint16_t* y, int64_t ldy,
                         uint32_t* row_pmax, int64_t pm_count, void* stream);

/* K2 of a chained producer with its consumer's per-token K1 fused into the epilogue:
 *   quantized_layer_forward(layer_b, quantized_layer_forward(layer_a, x)) without the
 *   intermediate ever reaching memory (engine.cpp:134-142 twice; kernel_a on kernel_b's output).
 * y = act(s_x (s_wo acc_o + s_wn acc_n) + b) is rounded to bf16 exactly as qarvd_dual_gemm
 * writes it, and each row is quantized as
 *   qarvd_quantize_act(y, QARVD_BF16, m, n, n, NULL, n, granularity, static_scale, bits,
 *                      q, ldq_out, scale_f32, scale_f64, err_index, stream)
 * would (per-token: the row max waits for the row's other N tiles; per-tensor static: the codes
 * come straight from the epilogue registers): same codes (columns 0..n-1 of each row; columns n..ldq_out-1 untouched), same scales,
 * same non-finite reporting (flat index row * ldq_out + c).  The consumer's input channels must
 * be in this layer's output order (no gather; pipeline.fold_output_permutation does that).
 * n % 256 == 0; q rows 16-byte aligned.  workspace: device, 16-byte aligned, ZERO-FILLED once
 * before first use, >= qarvd_dual_gemm_quant_workspace_size(m) bytes, one per concurrently
 * running call; it needs no reset between calls (per-launch epochs, counters only grow), but a
 * launch that fails midway leaves it invalid (zero it again).  QARVD_ERR_UNSUPPORTED when the persistent grid cannot be
 * co-resident on this device (the caller then runs qarvd_dual_gemm + qarvd_quantize_act). */
int64_t qarvd_dual_gemm_quant_workspace_size(int64_t m);
int qarvd_dual_gemm_quant(const int8_t* xq, int64_t ldq, const int8_t* wq, int64_t ldw, int64_t m,
                          int64_t n, int64_t k, int64_t k_outlier, const float* scale_x,
                          const float* scale_w_outlier, const float* scale_w_normal,
                          const float* bias, int epilogue, int granularity, double static_scale,
                          int bits, int8_t* q, int64_t ldq_out,
                          float* scale_f32, double* scale_f64, int64_t* err_index,
                          void* workspace, int64_t workspace_bytes, void* stream);

/* K2 with the reference's exact f64 epilogue (engine.cpp:86-94: val = 0; val += (s_x*s_wo[j])*acc_o;
 * val += (s_x*s_wn[j])*acc_n) on f64 scales -> f64 y.  Bit-identical to kernel_b_gemm_dequant
 * for symmetric activations; used by the C++ drop-in adapter (toy / reference-parity path). */
int qarvd_dual_gemm_f64(const int8_t* xq, int64_t ldq, const int8_t* wq, int64_t ldw, int64_t m,
                        int64_t n, int64_t k, int64_t k_outlier, const double* scale_x,
                        const double* scale_w_outlier, const double* scale_w_normal, double* y,
                        int64_t ldy, void* stream);

/* K2 with the f64 epilogue whose output columns come in runs of `slices` (2, 4, 8 or 16)
 * consecutive products, slice t of a run weighted 2^-7t, recombined into one f64 column:
 *   y[i, j] = (s_x[i] * s_wo[j]) * V_o(i, j) + (s_x[i] * s_wn[j]) * V_n(i, j)   (no FMA),
 *   V(i, j) = sum_t 2^-7t acc(i, j*slices + t),
 * where groups of four slices combine exactly in int64 and the groups add in f64, smallest
 * first.  With int8 slices of a wider operand (t-th slice = t-th 7-bit digit) stacked along N
 * this is an exact integer product recombined in f64 (K7's Ozaki-style products).  The scales
 * are per run: s_wo / s_wn have n / slices entries.  n % 16 == 0; y is [m x n / slices] (ldy). */
int qarvd_dual_gemm_f64_slices(const int8_t* xq, int64_t ldq, const int8_t* wq, int64_t ldw, int64_t m,
                               int64_t n, int64_t k, int64_t k_outlier, const double* scale_x,
                               const double* scale_w_outlier, const double* scale_w_normal, int slices,
                               double* y, int64_t ldy, void* stream);

/* ---- K1+K2: one quantized linear, host buffers (end-to-end entry) --------
 * Replaces  quantized_layer_forward(layer, x, Engine::int_kernels)
 *           engine.hpp:60 / engine.cpp:134-142 (per-token or static activations).
 * Host x (bf16 bits [m x k]) -> H2D -> K1 -> K2 -> D2H -> host y (bf16 [m x n]).
 * The device-resident layer (codes, scales, gather) comes from
 * qarvd_linear_create; workspace for activations is owned by the handle.
 */
typedef struct qarvd_linear* qarvd_linear_t;
int qarvd_linear_create(const int8_t* wq_dev, int64_t n, int64_t k_pad, int64_t k_outlier,
                        const int32_t* gather_dev, int64_t k_in, const float* scale_w_outlier_dev,
                        const float* scale_w_normal_dev, const float* bias_dev, int granularity,
                        double static_scale, int epilogue, qarvd_linear_t* out);
int qarvd_linear_destroy(qarvd_linear_t layer);
/* device-pointer forward (x bf16 [m x k_in] -> y bf16 [m x n]) */
int qarvd_linear_forward(qarvd_linear_t layer, const uint16_t* x_dev, int64_t m, uint16_t* y_dev,
                         void* stream);
/* host-buffer forward: copies in, runs K1+K2, copies out, synchronizes */
int qarvd_linear_forward_host(qarvd_linear_t layer, const uint16_t* x_host, int64_t m,
                              uint16_t* y_host, void* stream);

/* chained host-buffer forward through several linears (e.g. FFN up -> down):
 * one H2D of x, K1+K2 per layer on the device, one D2H of the last output.
 * layers[i].n must equal layers[i+1].k_in. */
int qarvd_linear_chain_forward_host(const qarvd_linear_t* layers, int num_layers,
                                    const uint16_t* x_host, int64_t m, uint16_t* y_host,
                                    void* stream);

/* ---- K3: per-layer outlier detection (batched over layers) ---------------
 * Replaces  analyze_layer(name, W, tau, alpha_min, align)  outlier.hpp:59-61,
 *           i.e. channel_l2_norms(W, 1) (tensor.cpp:132-150) -> mad (outlier.cpp:30-38)
 *           -> detect_outliers (outlier.cpp:40-52) -> align_outliers (outlier.cpp:54-78).
 * All outputs are device pointers; bit-exact with the reference's f64 results.
 */
typedef struct qarvd_outlier_job {
  const void* w;       /* device [n x k] (ldw) weight, dtype given to the call   */
  int64_t n, k, ldw;
  double* norms;       /* out [k]  channel L2 norms                              */
  double* stats;       /* out [3]  median, mad, threshold                        */
  int32_t* counts;     /* out [2]  |raw|, |aligned|                              */
  int32_t* raw_idx;    /* out [k]  raw outlier indices, ascending                */
  int32_t* aligned_idx;/* out [k]  aligned outlier indices, ascending            */
} qarvd_outlier_job;
int qarvd_analyze_layers(const qarvd_outlier_job* jobs, int num_jobs, int w_dtype, double tau,
                         double alpha_min, int64_t align, void* stream);

/* ---- K4: frame-weighted calibration scale search (batched over layers) ---
 * Replaces  init_scale_percentile_search(samples, bits)  quant.hpp:78-82 /
 *           quant.cpp:190-226, generalised with frame weights from
 *           weighting_strategy (sensitivity.cpp:86-112):
 *   L(c) = sum_f w_f * mse_f(c) / sum_f w_f,  mse_f(c) = ||X_f - FQ_{s_c}(X_f)||^2 / |X_f|
 *   (all w_f equal reduces to, and is evaluated as, (1/S) sum_f mse_f = quant.cpp:216).
 * X of one layer is `frames` consecutive row blocks of `rows` rows, [frames*rows x k] bf16.
 * Candidate thresholds are exact order statistics of the pooled |x| (quant.cpp:20-28),
 * argmin with ties to the larger percentile (quant.cpp:219).
 */
#define QARVD_MAX_CANDIDATES 16
#define QARVD_MAX_FRAMES 64
typedef struct qarvd_search_job {
  const uint16_t* x;   /* device bf16 [frames*rows x k] (ldx)                     */
  int64_t frames, rows, k, ldx;
  double* result;      /* out device f64 [3*num_cand + 2]:
                          thresholds[c], scales[c], losses[c], best_index, best_scale */
} qarvd_search_job;
int qarvd_scale_search(const qarvd_search_job* jobs, int num_jobs, const double* percentiles,
                       int num_cand, const double* frame_weights, int bits, void* stream);
/* Same, without the host synchronisation: the non-finite check lands in *nonfinite_flag_dev
 * (device uint64; all ones = every sample finite) for the caller to read later. */
int qarvd_scale_search_async(const qarvd_search_job* jobs, int num_jobs,
                             const double* percentiles, int num_cand,
                             const double* frame_weights, int bits, uint64_t* nonfinite_flag_dev,
                             void* stream);

/* ---- Eq. 5: frame-weighted output-space reconstruction loss ---------------
 * Replaces  weighted_loss(batch, state, chunk_weights)  calibrate.hpp:80-82 /
 *           calibrate.cpp:201-224:
 *   loss = (1/B) sum_s chunk_weights[chunk_s - 1] * || X_s W^T - FQ(X_s) What^T ||_F^2
 * One tcgen05 kernel per call: X W^T (bf16 x bf16 -> f32 TMEM) and the two int8 slabs of
 * xq . wq^T (int32 TMEM) per 128 x 128 tile, squared difference reduced in the epilogue;
 * neither product is written to memory.
 *   x  device bf16 [m x k] (ldx): the B samples stacked, sample s = rows
 *      sample_rows[s] .. sample_rows[s+1] (HOST int64 [B+1], sample_rows[B] = m)
 *   w  device bf16 [n x k] (ldw): the FP weight, same column order as x
 *   xq / wq  device int8 codes [m x k_pad] / [n x k_pad] in plan order (K1 / K5 outputs),
 *      k_outlier leading outlier-slab columns; scale_x f32 [m], scale_w_* f32 [n]
 *   sample_chunk  HOST int64 [B], 1-based; chunk_weights HOST f64 [n_chunks]
 *   sample_err  out device f64 [B]; loss  out device f64 [1]
 *   workspace   device, >= qarvd_weighted_loss_workspace(m, n, B) bytes, 8-byte aligned
 * Errors as the reference: empty batch -> INVALID_ARGUMENT, a chunk outside [1, n_chunks]
 * -> OUT_OF_RANGE ("sample chunk outside the weight vector", calibrate.cpp:207-208).
 */
int64_t qarvd_weighted_loss_workspace(int64_t m, int64_t n, int64_t n_samples);
int qarvd_weighted_loss(const uint16_t* x, int64_t ldx, const uint16_t* w, int64_t ldw,
                        const int8_t* xq, int64_t ldq, const int8_t* wq, int64_t ldwq, int64_t m,
                        int64_t n, int64_t k, int64_t k_pad, int64_t k_outlier,
                        const float* scale_x, const float* scale_w_outlier,
                        const float* scale_w_normal, const int64_t* sample_rows,
                        const int64_t* sample_chunk, int64_t n_samples,
                        const double* chunk_weights, int64_t n_chunks, double* sample_err,
                        double* loss, void* workspace, int64_t workspace_bytes, void* stream);

/* ---- K7: AdaRound layer calibration (f64, the reference's calibrator) ------
 * Replaces  calibrate_layer(w, plan, act_init, samples, chunk_weights, cfg)  calibrate.hpp:112-116
 *           (calibrate.cpp:298-396, LearnableQuantState calibrate.cpp:77-199,
 *           soft_loss_gradients calibrate.cpp:232-296).
 * All tensors are f64 device arrays: w [n x k]; outlier_mask u8 [k] (1 = outlier column of the
 * plan); the plan's initial group scales [n] (scale_outlier_init ignored when !plan_enabled);
 * x = the samples stacked [rows x k], sample s = rows sample_rows[s] .. sample_rows[s+1]
 * (HOST int64 [S+1]); sample_chunk HOST int64 [S] (1-based); chunk_weights HOST f64.
 * layer_name seeds the batch sampler exactly as the reference (mix_seed(seed, fnv1a(name))).
 * Outputs (device): codes int8 [n x k] original column order (hard_codes), learned scales [n],
 * scalars_out f64 [3] = {act scale, initial hard loss, final hard loss}, trace_out f64
 * [iterations] running-min batch loss (may be NULL).  Divergence -> QARVD_ERR_RUNTIME with the
 * reference message; invalid configs -> the reference's CalibConfig::validate messages.
 */
typedef struct qarvd_calib_config {
  int iterations, batch_size;
  double lr_round, lr_scale;
  uint64_t seed;
  int train_activation_scale;
  double zeta, gamma_lo, reg_lambda, beta_start, beta_end, warmup_frac;
} qarvd_calib_config;
int qarvd_calibrate_layer(const double* w, int64_t n, int64_t k, const uint8_t* outlier_mask,
                          int plan_enabled, const double* scale_normal_init,
                          const double* scale_outlier_init, double act_scale_init, int act_bits,
                          int w_bits, const double* x, const int64_t* sample_rows,
                          const int64_t* sample_chunk, int64_t n_samples,
                          const double* chunk_weights, int64_t n_chunks,
                          const qarvd_calib_config* cfg, const char* layer_name, int8_t* codes,
                          double* scale_normal_out, double* scale_outlier_out, double* scalars_out,
                          double* trace_out, void* stream);

/* ---- exact f64 restatements of the reference's generic operators ---------
 * The C++ drop-in (adapter/) serves these reference functions from the device, bit-identical
 * to the reference's f64 CPU code (no FMA, the reference's op order).  All pointers are
 * device pointers unless marked HOST.
 *
 * Replaces  quantize / dequantize / fake_quant  quant.hpp:64-66 / quant.cpp:113-159.
 * Element i uses channel ch = (i / inner) % extent (extent = 1: per-tensor).  codes (int32, the
 * IntTensor storage) and dequant (f64: (code - z) * s) may each be NULL.  zero_points NULL = 0.
 * err_index: int64[1], receives the smallest flat index of a non-finite x (or INT64_MAX); the
 * reference throws "quantize: non-finite input at flat index N" (quant.cpp:128-129). */
int qarvd_quantize_f64(const double* x, int64_t count, int64_t inner, int64_t extent,
                       const double* scales, const int32_t* zero_points, int32_t q_min,
                       int32_t q_max, int32_t* codes, double* dequant, int64_t* err_index,
                       void* stream);
/* Replaces  init_scale_minmax(x, bits, g, axis)  quant.hpp:71 / quant.cpp:161-183:
 * scales[extent] = absmax over each slice / (2^(bits-1)-1), DBL_MIN for all-zero slices. */
int qarvd_minmax_scale_f64(const double* x, int64_t count, int64_t inner, int64_t extent, int bits,
                           double* scales, void* stream);
/* Replaces  init_scale_percentile_search(samples, bits)  quant.hpp:82 / quant.cpp:185-226.
 * x: the samples concatenated; sample_offsets HOST int64 [n_samples + 1]; percentiles HOST
 * [num_cand] (the reference's {0.999, 0.9999, 0.99999}).  Exact order statistics of the pooled
 * |x| by radix select; per-sample squared errors summed in double-double.
 * result: f64 [3*num_cand + 2] = thresholds, scales, candidate MSEs, best index, best scale.
 * err: int64 [2] = {first sample holding a non-finite value, its flat index} or {-1, -1}
 * (the reference throws "quantize: non-finite input at flat index N" there).  Synchronizes. */
int qarvd_percentile_search_f64(const double* x, const int64_t* sample_offsets, int64_t n_samples,
                                const double* percentiles, int num_cand, int bits, double* result,
                                int64_t* err, void* stream);
/* Replaces  matmul_nt(a, b)  tensor.hpp:70 / tensor.cpp:82-105: c[m x n] = a[m x k] b[n x k]^T,
 * each output summed from 0.0 in ascending k with separate multiply and add roundings. */
int qarvd_matmul_nt_f64(const double* a, int64_t m, int64_t k, int64_t lda, const double* b, int64_t n,
                        int64_t ldb, double* c, int64_t ldc, void* stream);
/* Replaces  permute_activations  engine.cpp:36-44 and the code pre-permute calibrate.cpp:474-480:
 * out[r, c] = idx[c] >= 0 ? in[r, idx[c]] : 0 for elements of elem_bytes (1, 2, 4 or 8). */
int qarvd_gather_columns(const void* in, int64_t rows, int64_t ld_in, const int32_t* idx,
                         int64_t out_cols, void* out, int64_t ld_out, int elem_bytes, void* stream);
/* Replaces  dequantized_weight_original_order  engine.cpp:117-130 (the fakequant_sim weights):
 * w_out[j, perm[pos]] = wq[j, pos] * (pos < n_outlier ? s_o[j] : s_n[j]); perm NULL = identity. */
int qarvd_dequant_weight_f64(const int32_t* wq, int64_t n, int64_t k, const uint32_t* perm,
                             int64_t n_outlier, const double* scale_outlier, const double* scale_normal,
                             double* w_out, void* stream);

/* *total = (accumulate ? *total : 0) + weight * sum_i (a_i - b_i)^2 with the sum sequential in i
 * (frobenius_sq_distance tensor.cpp:116-126 inside weighted_recon_loss calibrate.cpp:206-214);
 * divide_by > 0 then divides the total (the batch mean, calibrate.cpp:215).  total: device f64[1]. */
int qarvd_sq_distance_acc_f64(const double* a, const double* b, int64_t count, double weight, double* total,
                              int accumulate, double divide_by, void* stream);
/* Kernel B's zero-point correction (engine.cpp:74-83, :95-100) applied to an f64 output of
 * qarvd_dual_gemm_f64: y[i, j] -= (z_x * s_x) * sum_g s_g[j] * colsum_g[j], colsum over the
 * group's columns of wq (groups = 2: [0, k_outlier) outlier then normal; 1: one group). */
int qarvd_zero_point_correct_f64(double* y, int64_t ldy, int64_t m, int64_t n, const int8_t* wq, int64_t ldw,
                                 int64_t k, int64_t k_outlier, int groups, int32_t z_x, double s_x,
                                 const double* s_wo, const double* s_wn, void* stream);
/* int32 codes (IntTensor storage) -> int8 kernel layout: out[r, c] = idx[c] >= 0 ? in[r, idx[c]] : 0;
 * *bad (device int) is set to 1 when a code is outside [-128, 127]. */
int qarvd_pack_codes_i8(const int32_t* in, int64_t rows, int64_t ld_in, const int32_t* idx, int64_t out_cols,
                        int8_t* out, int64_t ld_out, int* bad, void* stream);
/* Packed 4-bit codes as the reference stores them (tensor.cpp:221-264, save_int_tensor /
 * load_int_tensor: two per byte, low nibble first, over the flat [rows x k_src] tensor) ->
 * int8 kernel layout on the device: out[r, c] = idx[c] >= 0 ? sext(nibble(r * k_src + idx[c])) : 0.
 * The W4A8 weights travel and sit in HBM packed until this one expansion (QARQ loader). */
int qarvd_unpack_codes_i4(const uint8_t* packed, int64_t rows, int64_t k_src, const int32_t* idx,
                          int64_t out_cols, int8_t* out, int64_t ld_out, void* stream);
/* out[i] = exp(in[i]) exactly as the reference's std::exp (glibc's algorithm restated, libm_ref.cuh). */
int qarvd_exp_f64(const double* in, double* out, int64_t count, void* stream);
/* LearnableQuantState soft / hard weights and hard codes (calibrate.cpp:138-183):
 * what = s * clamp(floor(w / s) + r, -qmax, qmax) with r = h(V) (hard = 0) or [h(V) > 0.5]
 * (hard = 1), s = exp(log_scale[group row]) (log_scale = [normal n | outlier n]); codes (int8,
 * original column order) written when non-NULL and hard; what may be NULL. */
int qarvd_adaround_weights(const double* w, const double* v, const uint8_t* outlier_mask,
                           int plan_enabled, const double* log_scale, int64_t n, int64_t k,
                           double zeta, double gamma_lo, int w_bits, int hard, double* what,
                           int8_t* codes, void* stream);

/* ---- multi-GPU calibration driver (C++ host, one thread per rank) ---------
 * Replaces  calibrate_model's slot-indexed parallel_for over layers  calibrate.cpp:440-484,
 * sharded over GPUs: a deterministic LPT split of the layers by algorithmic bytes (ties ->
 * lower layer index, lower rank), each rank's share calibrated on devices[rank] with no host
 * round trip -- K3 (analyze) -> device plan + K5 (weights) on one stream, K4 (frame-weighted
 * percentile search, quant.cpp:185-226 + sensitivity.cpp:86-112 weights) on another -- then ONE
 * ncclAllGather of the packed per-layer records over NVLink (communicator over the ranks'
 * devices; when ranks share a device -- a single-GPU emulation of G ranks -- the records are
 * gathered through host memory and *used_nccl is 0).  Results do not depend on `world`.
 * A layer's inputs are host bf16 buffers or, when NULL, generated on the owning GPU by the
 * counter-based synthetic generator (qarvd_synth_bf16) from its descriptors, so no input
 * crosses PCIe.  records: f64, one record per layer in layer order:
 *   [index, n, n_outliers, num_cand, act_scale, best_index, losses[num_cand],
 *    scale_outlier[n], scale_normal[n], outliers[n_outliers]]
 * (qarvd_calib_record_doubles gives a record's length); record_offsets [num_layers + 1].
 * step_ms: max over ranks of the device time of the calibration unit (inputs resident). */
typedef struct qarvd_synth_desc {
  uint64_t seed;
  double stddev;
  const int32_t* outlier_cols; /* HOST int32 [num_outliers] */
  int64_t num_outliers;
  double gamma;
} qarvd_synth_desc;
typedef struct qarvd_calib_layer {
  int64_t index;                   /* registry index (the record key)                        */
  int64_t n, k, rows;              /* W [n x k]; X = frames consecutive blocks of rows x k    */
  const uint16_t* w_host;          /* HOST bf16 [n x k], or NULL: generated from w_synth      */
  qarvd_synth_desc w_synth;
  const uint16_t* x_host;          /* HOST bf16 [frames*rows x k], or NULL: frame f generated */
  const qarvd_synth_desc* x_synth; /*   from x_synth[f] (HOST array of frames descriptors)    */
} qarvd_calib_layer;
int64_t qarvd_calib_record_doubles(int64_t n, int64_t n_outliers, int num_cand);
int qarvd_calibrate_sharded(const qarvd_calib_layer* layers, int num_layers, int frames,
                            const double* frame_weights, const double* percentiles, int num_cand,
                            int world, const int* devices, double* records, int64_t records_cap,
                            int64_t* record_offsets, double* step_ms, int* used_nccl);

/* ---- measurement -----------------------------------------------------------
 * Dense INT8 tensor-pipe peak at the clocks this board holds under tensor load: back-to-back
 * tcgen05.mma kind::i8 M128xN256xK32 on every SM from shared memory (no memory traffic), timed
 * with CUDA events over `iters` x 4 MMAs per SM (after a short warm-up launch).  Synchronizes. */
int qarvd_probe_int8_peak(int iters, double* tops_out, double* ms_out, void* stream);

/* ---- synthetic Wan-shaped data (counter-based, deterministic on device) --
 * Follows the reference recipe toy_model.cpp:146-166: Gaussian-like / sqrt(fan_in)
 * weights with a seeded set of input columns scaled by gamma.  Values are
 * generated directly as bf16.  outlier_cols: device int32 [num_outliers] or NULL.
 */
int qarvd_synth_bf16(uint16_t* out, int64_t rows, int64_t cols, int64_t ld, uint64_t seed,
                     double stddev, const int32_t* outlier_cols, int64_t num_outliers,
                     double gamma, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* QARVD_B200_H */
