// K2 — dual-scale W8A8 linear on the sm_100a tensor cores.
//
// Replaces the reference's scalar triple loop kernel_b_gemm_dequant
// (/root/reference/proj/core/src/engine.cpp:46-105).  The reference keeps one
// int64 accumulator per (row, column, group) and combines the groups in f64,
// outlier group first (engine.cpp:86-94).  Here both operands are int8 codes
// already permuted [outlier | normal] along K (calibrate.cpp:474-480 for the
// weights, K1 for the activations); TMA streams 128-byte K-slices of both into
// a 128B-swizzled shared-memory ring, a single elected thread issues
// tcgen05.mma.kind::i8 (M=128 per CTA, 256 over an SM pair with cta_group::2, N=BN, K=32) and
// routes every K=32 step to one of two int32 tensor-memory accumulators: acc_o for
// k < k_outlier, acc_n after.  int32 is exact because |code| <= 127 and k <= 132104 (D4 in
// SURVEY.md).  Sixteen epilogue warps (four per TMEM lane quadrant) read both accumulators
// with tcgen05.ld and apply
//   y = s_x[i] * (s_wo[j]*acc_o + s_wn[j]*acc_n) (+ bias[j]) [gelu] -> bf16
// (or f32, the reference's exact f64 epilogue, K7's slice recombination, or the next layer's
// int8 codes: qarvd_dual_gemm_quant).  Persistent, warp-specialised: warp 0 = TMA producer,
// warp 1 = MMA issuer, warp 2 = TMEM allocator, warps 4..19 = epilogue.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"

namespace qarvd_b200 {
namespace {

constexpr int BM = 128;  // rows of the activation tile (one TMEM lane per row)
constexpr int BK = 128;  // bytes (= int8 elements) of K per 128B-swizzle sub-tile (one TMA box)
// 4 control warps + 16 epilogue warps (4 per TMEM lane quadrant).  The epilogue (dequant,
// GELU, bf16 pack, stores) is latency-bound per warp, so it runs on as many warps as the
// register file allows (96 registers x 640 threads) in 16-column chunks.
constexpr int kEpiWarps = 16;
constexpr int kThreads = 128 + 32 * kEpiWarps;
constexpr int kCtrlRegs = 32;   // setmaxnreg split of 640 x 96 registers
constexpr int kEpiRegs = 112;   //   (4 x 32 x 32 + 16 x 32 x 112 = 640 x 96)
constexpr int CW = 16;            // columns per epilogue chunk (one tcgen05.ld .32x32b.x16)

// K7's slice products (qarvd_dual_gemm_f64_slices): run j of T consecutive accumulator columns holds
// the integer products of slices t = 0..T-1 whose weight is 2^-7t.  Groups of four slices combine
// exactly in int64 (|acc| < 2^31, so a group stays below 2^53 and converts to f64 exactly); the
// group values are scaled by exact powers of two and added smallest first, then
// y = s_x (s_o v_o + s_n v_n) with the per-run scales.
__device__ __forceinline__ double exp2_int(int e) {  // 2^e, e in the normal range
  return __longlong_as_double(static_cast<long long>(1023 + e) << 52);
}
// int64 -> f64 for |v| < 2^51 without the XU pipe's conversion: the bits of 1.5 * 2^52 + v are
// the bits of 0x1.8p52 plus v, so one integer add and one exact f64 subtraction
__device__ __forceinline__ double small_i64_to_f64(long long v) {
  return __dsub_rn(__longlong_as_double(v + 0x4338000000000000LL), 6755399441055744.0);
}
// MAGIC: |group| < 2^51 (k <= 32768: |acc| <= k * 127 * 128 < 2^29, a group of four < 2^50.1)
template <int T, bool MAGIC>
__device__ __forceinline__ double slice_value(const uint32_t* acc) {
  double v = 0.0;
#pragma unroll
  for (int g0 = ((T - 1) / 4) * 4; g0 >= 0; g0 -= 4) {
    const int last = (g0 + 4 < T ? g0 + 4 : T) - 1;
    long long part = static_cast<int32_t>(acc[last]);
#pragma unroll
    for (int t = last - 1; t >= g0; --t)  // one IMAD.WIDE per slice
      part += static_cast<long long>(static_cast<int32_t>(acc[t])) * (1LL << (7 * (last - t)));
    const double pv = MAGIC ? small_i64_to_f64(part) : __ll2double_rn(part);
    v = g0 == ((T - 1) / 4) * 4 ? __dmul_rn(pv, exp2_int(-7 * last))
                                : __fma_rn(pv, exp2_int(-7 * last), v);
  }
  return v;
}
template <int T, bool MAGIC>
__device__ __forceinline__ void slice_runs(const uint32_t* rn, const uint32_t* ro, bool has_outlier, double sx,
                                           const double* so, const double* sn, int64_t run0, double* yr) {
  double out[CW / T];
#pragma unroll
  for (int g = 0; g < CW / T; ++g) {
    const double vn = __dmul_rn(__dmul_rn(sx, sn[run0 + g]), slice_value<T, MAGIC>(rn + g * T));
    out[g] = has_outlier ? __dadd_rn(__dmul_rn(__dmul_rn(sx, so[run0 + g]), slice_value<T, MAGIC>(ro + g * T)), vn)
                         : vn;
  }
  if (CW / T == 2 && (reinterpret_cast<uintptr_t>(yr) & 15) == 0) {
    *reinterpret_cast<double2*>(yr) = make_double2(out[0], out[1]);
  } else {
#pragma unroll
    for (int g = 0; g < CW / T; ++g) yr[g] = out[g];
  }
}
constexpr int kYStageBytes = 32 * CW * 2;  // one warp's bf16 staging tile: 32 rows x 32 B

// BN = output columns of the (pair) tile; CG = CTAs per MMA (1, or 2 = an SM pair
// computing a 256-row tile, each CTA holding its 128 A rows and BN/2 B rows).
// KS = 128-byte K sub-tiles per pipeline stage.  Every stage costs the MMA issuer one
// mbarrier wait (~110-250 clk that the tensor pipe does not overlap, measured by
// scripts/mma_rate2.cu), so KS = 2 (8 MMAs per wait) halves that overhead per MAC.
template <int BN, int CG, int KS>
struct GemmCfg {
  static constexpr int kASub = BM * BK;           // one 128 B K sub-tile of A
  static constexpr int kBSub = (BN / CG) * BK;    // one 128 B K sub-tile of this CTA's B
  static constexpr int kABytes = KS * kASub;
  static constexpr int kBBytes = KS * kBSub;
  // y staging: one 32 x 16 bf16 tile per epilogue warp, double-buffered unless the operand
  // stages need the room
  static constexpr int kYBufs = KS == 2 ? 1 : 2;
  static constexpr int kEpiBytes = 512 /*barriers*/ + 3 * BN * 4 * 4 /*scales: 16 warps x 3 x BN/4*/ +
                                   kEpiWarps * kYStageBytes * kYBufs /*y staging*/;
  static constexpr int kStages = (227 * 1024 - kEpiBytes) / (kABytes + kBBytes) > 8
                                     ? 8
                                     : (227 * 1024 - kEpiBytes) / (kABytes + kBBytes);
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kAccStages = 512 / (2 * BN);  // two accumulators per stage
  static constexpr uint32_t kTmemCols = 512;
  static constexpr size_t kSmemBytes = static_cast<size_t>(kStages) * kStageBytes + kEpiBytes;
};

struct GemmParams {
  int64_t m, n, k, k_o;
  const float* scale_x;
  const float* scale_wo;
  const float* scale_wn;
  const float* bias;
  void* y;
  int64_t ldy;
  int32_t* acc_o_dbg;
  int32_t* acc_n_dbg;
  int epilogue;
  int out_dtype;
  int num_m_blks, num_n_blks, num_tiles;
  const double* sx64;  // QARVD_F64 output: f64 scales, reference epilogue (engine.cpp:86-94)
  const double* so64;
  const double* sn64;
  int f64_slices;      // QARVD_F64 with f64_slices = T > 1: each run of T consecutive output columns
                       // (slice t weighted 2^-7t, per-run scales) recombines into one f64 column
  uint32_t* row_absmax;  // optional: atomicMax per row of the sign-cleared bf16 output bits
  uint32_t* row_pmax;    // optional: per-row partial maxima, [m][pm_count] (one per epilogue
  int pm_count;          //   warp and tile: pm_count = num_n_blks * 4), plain stores
  int use_tma_store;  // bf16 output through the TMA store path
  int direct_store;   // QARVD_GEMM_DIRECT=1: fast path stores bf16 rows from registers
  int epi_regs;       // fast path holds acc_n in registers (QARVD_GEMM_EPIREG=0 disables)
  int spin;
  int trace;  // QARVD_GEMM_TRACE: CTA 0 prints per-tile clocks (diagnostic)
  // stream-K (optional, qarvd_dual_gemm_ws): tiles [0, sk_tiles) are split along K into
  // contiguous ranges of k-blocks over all SM pairs (processed first), the rest are
  // data-parallel.  A pair that does not own a tile's last k-block stores its partial acc_n
  // (int32, exact) in sk_slots; the owner adds them in its epilogue.
  int sk_tiles;
  int sk_slots_per_tile;
  int32_t* sk_slots;    // [sk_tiles][sk_slots_per_tile][BN][TM] int32, column-major per tile
  uint32_t* sk_count;   // [sk_tiles][2]: writer-warp arrivals, owner-warp reads (self-resetting)
  int debug;  // QARVD_GEMM_DEBUG: 1 = skip the MMAs, 2 = skip the TMA loads (throughput probes)
  // fused consumer K1 (qarvd_dual_gemm_quant; the kernel's QZ instance, tiles in row-major
  // order): the bf16 output is quantized per token in the epilogue instead of being stored.
  // qz_rowmax [m]: (launch epoch << 16) | row |y| max as sign-cleared bf16 bits; qz_count
  // [num_m_blks]: arrivals per row block, growing across launches (zero-filled once).
  unsigned long long* cta_times;  // QARVD_GEMM_DEBUG=128: per-CTA start / end globaltimer
  int row_major;  // tile order: all N tiles of a row block consecutive (the per-token fused quantizer)
  int qz;
  int qz_qmax;
  int qz_static;       // per-tensor static scale: codes in phase 2, no row-block wait
  double qz_s_static;  //   the scale (validated finite > 0)
  unsigned long long* qz_rowmax;
  unsigned long long* qz_count;
  unsigned long long* qz_epoch;  // launches completed on this workspace
  unsigned int* qz_done;         // CTAs finished in the running launch
  int8_t* qz_q;
  int64_t qz_ldq;
  float* qz_sx;
  double* qz_s64;
  unsigned long long* qz_err;
};

// Work list of one SM pair: its stream-K k-block range over the split tiles first, then its
// data-parallel tiles (t = sk_tiles + pair, + pairs, ...).  Unit u = tile * nkb + issue index.
struct SkSched {
  int tiles, pairs, sk, nkb;
  int64_t units;  // sk * nkb
  __host__ __device__ SkSched(int tiles_, int pairs_, int sk_, int nkb_)
      : tiles(tiles_), pairs(pairs_), sk(sk_), nkb(nkb_), units(static_cast<int64_t>(sk_) * nkb_) {}
  __host__ __device__ int64_t u_begin(int c) const { return units * c / pairs; }
  // the pair whose range holds unit u (the largest c with u_begin(c) <= u)
  __host__ __device__ int pair_of(int64_t u) const {
    return static_cast<int>(((u + 1) * pairs - 1) / units);
  }
  // partial contributors (non-owners) of split tile t, and the slot of pair c
  __host__ __device__ int partials(int t) const {
    return pair_of(static_cast<int64_t>(t) * nkb + nkb - 1) - pair_of(static_cast<int64_t>(t) * nkb);
  }
  __host__ __device__ int slot_of(int t, int c) const { return c - pair_of(static_cast<int64_t>(t) * nkb); }
};
// A pair's items: its stream-K segments in DESCENDING tile order (the prefix of its last tile,
// which it only contributes to, comes first; the suffix of its first tile, which it owns and
// whose partials the neighbouring pairs publish as THEIR first items, comes last -- so no owner
// waits on a pair that is itself waiting), then its data-parallel tiles.
template <bool SKT>
struct SkIter {
  int64_t u0 = 0, u1 = 0;
  int tcur = 0, tlo = 0;
  int dp;
  __host__ __device__ SkIter(const SkSched& s, int c) : dp(SKT ? s.sk + c : c) {
    if (SKT && s.units) {
      u0 = s.u_begin(c);
      u1 = s.u_begin(c + 1);
      tlo = static_cast<int>(u0 / s.nkb);
      tcur = u1 > u0 ? static_cast<int>((u1 - 1) / s.nkb) : tlo - 1;
    } else {
      tcur = -1;
    }
  }
  // next work item: tile t, issue-index range [i0, i1); false when done
  __host__ __device__ bool next(const SkSched& s, int& t, int& i0, int& i1) {
    if (SKT && tcur >= tlo) {
      t = tcur--;
      const int64_t b = static_cast<int64_t>(t) * s.nkb;
      i0 = static_cast<int>((u0 > b ? u0 : b) - b);
      i1 = static_cast<int>((u1 < b + s.nkb ? u1 : b + s.nkb) - b);
      return true;
    }
    if (dp < s.tiles) {
      t = dp;
      i0 = 0;
      i1 = s.nkb;
      dp += s.pairs;
      return true;
    }
    return false;
  }
};

// ---- packed fp32x2 helpers (sm_100a FFMA2 / FMUL2: one instruction per element pair,
// each lane rounded exactly like the scalar fma.rn / mul.rn) -------------------------
__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void upk2(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// gelu(v) = 0.5 v (1 + erf(v/sqrt 2)) on a pair (toy_model.cpp:62-66 uses the erf form).
// erf via Abramowitz & Stegun 7.1.26 (|error| <= 1.5e-7, far below the bf16 output
// resolution): one rcp + one ex2 per element, the rest on packed FMAs (erff's two-range
// coefficient selection cost more than the whole dequant epilogue).  The epilogue is
// issue-bound (scripts/epi_rate.cu), so the form below minimises instructions.
// Non-finite v -> NaN (inputs are finite int32 accumulators times finite scales).
__device__ __forceinline__ uint64_t gelu2(uint64_t v) {
  // gelu(v) = h (1 + erf z), h = v/2, z = v/sqrt2.  With erf|z| = 1 - E (A&S 7.1.26:
  // E = t P(t) exp(-z^2), t = 1/(1 + p|z|)) and sign z = sign h:  gelu = max(v, 0) - |h| E.
  // In w = v sqrt(log2(e)/2): exp(-z^2) = 2^(-w^2), p|z| = p'|w|, and |h| P(t) = |w| Q(t)
  // with Q = -P / (2 sqrt(log2(e)/2)) folded into the coefficients.  No cancellation for
  // v < 0 (|error| <= 3.4e-7 absolute over [-10, 10], checked in f32 against scipy's erf).
  const uint64_t w = mul2(v, pk2(0.8493218f, 0.8493218f));
  float w0, w1, v0, v1;
  upk2(w, w0, w1);
  upk2(v, v0, v1);
  const uint64_t aw = pk2(fabsf(w0), fabsf(w1));
  float d0, d1;
  upk2(fma2(pk2(0.272737481f, 0.272737481f), aw, pk2(1.0f, 1.0f)), d0, d1);
  const uint64_t t = pk2(rcp_approx(d0), rcp_approx(d1));
  uint64_t q = fma2(pk2(-0.624854695f, -0.624854695f), t, pk2(0.85547788f, 0.85547788f));
  q = fma2(q, t, pk2(-0.836793392f, -0.836793392f));
  q = fma2(q, t, pk2(0.167484654f, 0.167484654f));
  q = fma2(q, t, pk2(-0.150019458f, -0.150019458f));
  const uint64_t g = mul2(mul2(aw, t), q);
  float s0, s1;
  upk2(mul2(w, w), s0, s1);
  return fma2(g, pk2(ex2_approx(-s0), ex2_approx(-s1)), pk2(fmaxf(v0, 0.f), fmaxf(v1, 0.f)));
}

// y = s_x * (s_wo*acc_o + s_wn*acc_n) (+ bias) [gelu], written back into rn as float bits.
// Same per-element op order as the scalar form (oracle_epilogue_f32), on packed pairs;
// specialised on (outlier slab?, bias?, gelu?) so every variant is straight-line code.
template <bool HO, bool HB, bool GL>
__device__ __forceinline__ void epi_math(uint32_t (&rn)[CW], const uint32_t (&ro)[CW],
                                         const float* scc, int bn, float sx) {
  const uint64_t sx2 = pk2(sx, sx);
#pragma unroll
  for (int e4 = 0; e4 < CW / 4; ++e4) {
    const float4 sn4 = reinterpret_cast<const float4*>(scc)[e4];
    float4 so4 = sn4, sb4 = sn4;
    if (HO) so4 = reinterpret_cast<const float4*>(scc + bn)[e4];
    if (HB) sb4 = reinterpret_cast<const float4*>(scc + 2 * bn)[e4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = 4 * e4 + 2 * h;
      const uint64_t sn = h ? pk2(sn4.z, sn4.w) : pk2(sn4.x, sn4.y);
      const uint64_t an = pk2(__int2float_rn(static_cast<int>(rn[e])),
                              __int2float_rn(static_cast<int>(rn[e + 1])));
      uint64_t t;
      if (HO) {
        const uint64_t so = h ? pk2(so4.z, so4.w) : pk2(so4.x, so4.y);
        const uint64_t ao = pk2(__int2float_rn(static_cast<int>(ro[e])),
                                __int2float_rn(static_cast<int>(ro[e + 1])));
        t = fma2(sn, an, mul2(so, ao));
      } else {
        t = mul2(sn, an);
      }
      uint64_t v;
      if (HB) v = fma2(sx2, t, h ? pk2(sb4.z, sb4.w) : pk2(sb4.x, sb4.y));
      else v = mul2(sx2, t);
      if (GL) v = gelu2(v);
      float y0, y1;
      upk2(v, y0, y1);
      rn[e] = __float_as_uint(y0);
      rn[e + 1] = __float_as_uint(y1);
    }
  }
}

// ---- fused consumer K1 (qarvd_dual_gemm_quant): the per-token arithmetic of K1's register
// kernel (quantize.cu: quant_act_reg_kernel, act_codes2<false>, act_fix8_div), restated on the
// epilogue's registers so the codes are those qarvd_quantize_act writes for the bf16 output.
constexpr float kQzMagic = 12582912.0f;  // 1.5 * 2^23: an fp32 add rounds to an integer (RNE)
constexpr float kQzGuard = 0.49997f;     // quantize.cu tie_guard<false>()
// 8 codes by the reference's f64 division (quant.cpp:132-135); non-finite values are reported
// (the reference throws, quant.cpp:113-121) and give 0 -- quantize.cu act_code_slow
__device__ __forceinline__ uint2 qz_div8_body(uint4 d, double s64, int qmax, unsigned long long* err, int64_t flat) {
  const uint32_t w[4] = {d.x, d.y, d.z, d.w};
  uint32_t c[8];
#pragma unroll
  for (int h = 0; h < 8; ++h) {
    const uint32_t bits = h & 1 ? (w[h >> 1] & 0xffff0000u) : (w[h >> 1] << 16);
    if ((bits & 0x7f800000u) == 0x7f800000u) {
      if (err) atomicMin(err, static_cast<unsigned long long>(flat + h));
      c[h] = 0u;
    } else {
      c[h] = static_cast<uint32_t>(quant_code_exact(static_cast<double>(__uint_as_float(bits)), s64, qmax)) & 0xffu;
    }
  }
  return make_uint2(__byte_perm(__byte_perm(c[0], c[1], 0x0040), __byte_perm(c[2], c[3], 0x0040), 0x5410),
                    __byte_perm(__byte_perm(c[4], c[5], 0x0040), __byte_perm(c[6], c[7], 0x0040), 0x5410));
}
__device__ __noinline__ uint2 qz_div8(uint4 d, double s64, int qmax, unsigned long long* err, int64_t flat) {
  return qz_div8_body(d, s64, qmax, err, flat);
}
// fast codes of 8 bf16 values (4 packed words): magic + rint(v r) by one packed FMA, the exact
// residual v r - rint(v r) by a second; |residual| > guard flags the group for the division
__device__ __forceinline__ uint2 qz_codes8(uint4 d, float r, float& dmax) {
  const uint32_t w[4] = {d.x, d.y, d.z, d.w};
  const uint64_t r2 = pk2(r, r), m2 = pk2(kQzMagic, kQzMagic);
  uint32_t c[8];
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const uint64_t v2 = pk2(__uint_as_float(w[h] << 16), __uint_as_float(w[h] & 0xffff0000u));
    const uint64_t y2 = fma2(v2, r2, m2);
    const uint64_t n2 = fma2(y2, pk2(-1.f, -1.f), m2);
    const uint64_t d2 = fma2(v2, r2, n2);
    float d0, d1, y0, y1;
    upk2(d2, d0, d1);
    upk2(y2, y0, y1);
    dmax = fmaxf(dmax, fmaxf(fabsf(d0), fabsf(d1)));
    c[2 * h] = __float_as_uint(y0);
    c[2 * h + 1] = __float_as_uint(y1);
  }
  return make_uint2(__byte_perm(__byte_perm(c[0], c[1], 0x0040), __byte_perm(c[2], c[3], 0x0040), 0x5410),
                    __byte_perm(__byte_perm(c[4], c[5], 0x0040), __byte_perm(c[6], c[7], 0x0040), 0x5410));
}
// static per-tensor codes of 8 bf16 values: t = clamp(v r, +-qmax), magic + rint(t); |t - rint t|
// above the guard flags the group (quantize.cu act_codes2<true>, tie_guard<true>)
constexpr float kQzGuardStatic = 0.4999f;
__device__ __forceinline__ uint2 qz_codes8_static(uint4 d, float r, float fq, float& dmax) {
  const uint32_t w[4] = {d.x, d.y, d.z, d.w};
  uint32_t c[8];
#pragma unroll
  for (int h = 0; h < 8; ++h) {
    const float v = __uint_as_float(h & 1 ? (w[h >> 1] & 0xffff0000u) : (w[h >> 1] << 16));
    const float t = fminf(fmaxf(__fmul_rn(v, r), -fq), fq);
    const float y = __fadd_rn(t, kQzMagic);
    dmax = fmaxf(dmax, fabsf(__fsub_rn(t, __fsub_rn(y, kQzMagic))));
    c[h] = __float_as_uint(y);
  }
  return make_uint2(__byte_perm(__byte_perm(c[0], c[1], 0x0040), __byte_perm(c[2], c[3], 0x0040), 0x5410),
                    __byte_perm(__byte_perm(c[4], c[5], 0x0040), __byte_perm(c[6], c[7], 0x0040), 0x5410));
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* a) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
  return v;
}

template <int BN, int CG, int KS, bool SKT = false, bool QZ = false>
__global__ void __launch_bounds__(kThreads, 1)
    dual_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                     const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmY, const GemmParams p) {
  using C = GemmCfg<BN, CG, KS>;
  constexpr int TM = BM * CG;  // rows of the (pair) tile
  constexpr int SK = BK * KS;  // K bytes per stage
  // 1024-B alignment (128B swizzle atoms) comes from the declaration, not from pointer
  // rounding: integer rounding would hide the shared address space (generic LD/ST).
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kStages * C::kABytes;
  uint8_t* epi_ystage = sB + C::kStages * C::kBBytes;  // 1024-aligned
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_ystage + kEpiWarps * kYStageBytes * C::kYBufs);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + C::kAccStages;
  uint64_t* tofree = tempty + C::kAccStages;  // acc_o released (one-stage TMEM only)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tofree + 1);
  float* epi_scales = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + 512);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  __shared__ long long s_trace[6][32];  // QARVD_GEMM_TRACE: per-tile clocks of CTA 0
  __shared__ long long s_clk0;
  __shared__ unsigned long long s_g0;
  if ((p.trace || (p.debug & 128)) && threadIdx.x == 0) {
    s_clk0 = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(s_g0));
  }
  const uint32_t rank = CG == 2 ? ptx::cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  const int cta_id = static_cast<int>(blockIdx.x) / CG;  // pair index
  const int num_ctas = static_cast<int>(gridDim.x) / CG;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    if (p.use_tma_store || QZ) ptx::prefetch_tmap(&tmY);
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < C::kAccStages; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], kEpiWarps * CG);  // one arrive per epilogue warp of the pair
    }
    ptx::mbar_init(tofree, kEpiWarps * CG);
    ptx::fence_mbar_init();
  }
  if (warp == 2) {
    if (CG == 2) ptx::tmem_alloc_2sm(tmem_slot, C::kTmemCols);
    else ptx::tmem_alloc(tmem_slot, C::kTmemCols);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (CG == 2) ptx::cluster_sync();  // peer barriers initialised before any remote arrive
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // prologue done: wait for the producer of xq / scale_x (PDL), then let the next kernel
  // launch -- its CTAs only fit on SMs this grid has left
  pdl_wait();
  pdl_launch_dependents();
  // 640 threads x 96 registers: the control warpgroup (producer, MMA issuer, TMEM owner)
  // needs few, the epilogue holds a warp's whole acc_n slice (64 registers) -> 32 / 112,
  // set inside each role branch so ptxas sizes every branch by its own limit

  const int num_kb = static_cast<int>((p.k + SK - 1) / SK);
  // producer / MMA-issuer waits (QARVD_GEMM_SPIN=1: retry without the suspend hint)
  auto ctl_wait = [&](uint64_t* bar, uint32_t parity) {
    if (p.spin) ptx::mbar_wait_spin(bar, parity);
    else ptx::mbar_wait(bar, parity);
  };
  // one-stage TMEM: k-blocks holding outlier steps are issued last (see the MMA issuer)
  auto kblock_rotation = [&](int ko32_, int nkb) {
    if (C::kAccStages != 1) return 0;
    const int r = (ko32_ + SK / 32 - 1) / (SK / 32);
    return (r > 0 && r < nkb) ? r : 0;
  };

  if (warp == 0) {
    // ===================== TMA producer (whole warp loops, lane 0 issues) ==============
    ptx::setmaxnreg_dec<kCtrlRegs>();
    int stage = 0;
    uint32_t phase = 0;
    const int rot = kblock_rotation(static_cast<int>(p.k_o / 32), num_kb);  // = the MMA issuer's
    const SkSched sks(p.num_tiles, num_ctas, p.sk_tiles, num_kb);
    SkIter<SKT> it(sks, cta_id);
    int t, i0, i1;
    while (it.next(sks, t, i0, i1)) {
      const int m_blk = (QZ && p.row_major) ? t / p.num_n_blks : t % p.num_m_blks;
      const int n_blk = (QZ && p.row_major) ? t % p.num_n_blks : t / p.num_m_blks;
      const int a_row = m_blk * TM + static_cast<int>(rank) * BM;
      const int b_row = n_blk * BN + static_cast<int>(rank) * (BN / CG);
      for (int i = i0; i < i1; ++i) {
        const int kb = (i + rot) < num_kb ? i + rot : i + rot - num_kb;
        ctl_wait(&empty[stage], phase ^ 1);
        if (lane == 0) {
          if (p.debug == 2) {
            if (leader) ptx::mbar_arrive(&full[stage]);
          } else if (CG == 1) {
            ptx::mbar_expect_tx(&full[stage], C::kStageBytes);
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
              ptx::tma_load_2d(sA + stage * C::kABytes + ks * C::kASub, &tmA, &full[stage],
                               kb * SK + ks * BK, a_row);
              ptx::tma_load_2d(sB + stage * C::kBBytes + ks * C::kBSub, &tmB, &full[stage],
                               kb * SK + ks * BK, b_row);
            }
          } else {
            if (leader) ptx::mbar_expect_tx(&full[stage], 2 * C::kStageBytes);
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
              ptx::tma_load_2d_2sm(sA + stage * C::kABytes + ks * C::kASub, &tmA, &full[stage],
                                   kb * SK + ks * BK, a_row);
              ptx::tma_load_2d_2sm(sB + stage * C::kBBytes + ks * C::kBSub, &tmB, &full[stage],
                                   kb * SK + ks * BK, b_row);
            }
          }
        }
        __syncwarp();
        if (++stage == C::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    ptx::setmaxnreg_dec<kCtrlRegs>();
    // The whole warp runs the (warp-uniform) loop so descriptors, accumulator addresses
    // and slab routing live in uniform registers; lane 0 issues.
    //
    // TMEM: with two accumulator stages (BN <= 128) tile t+1 uses the other stage.  With
    // one stage (BN >= 192: acc_o + acc_n fill the 512 columns) the k-blocks holding
    // outlier steps run LAST, and the epilogue releases the accumulators in two steps:
    // acc_n as soon as it has folded s_wn*acc_n + s_wo*acc_o into acc_o's columns, acc_o
    // after the stores.  The next tile's acc_n MMAs wait only for the first step.
    if (leader) {
      constexpr uint32_t idesc = ptx::idesc_i8(TM, BN);
      const uint64_t a_desc0 = ptx::sw128_kmajor_desc(ptx::smem_u32(sA));
      const uint64_t b_desc0 = ptx::sw128_kmajor_desc(ptx::smem_u32(sB));
      const int k32 = static_cast<int>(p.k / 32), ko32 = static_cast<int>(p.k_o / 32);
      constexpr int SPB = SK / 32;  // K=32 steps per k-block
      // k-block rotation (outlier k-blocks last) and the first acc_n step in issue order
      const int rot = kblock_rotation(ko32, num_kb);
      const int first_n = rot > 0 ? rot * SPB : ko32;
      const int kb_first_n = first_n / SPB;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      const SkSched sks(p.num_tiles, num_ctas, p.sk_tiles, num_kb);
      SkIter<SKT> it(sks, cta_id);
      int t, i0, i1, item = 0;
      while (it.next(sks, t, i0, i1)) {
        // the first acc_n step this item issues (accumulate = 0) and its k-block
        int seg_first_n = first_n, kb_seg_first_n = kb_first_n;
        if (SKT && i0 > 0) {
          seg_first_n = -1;
          for (int i = i0; i < i1 && seg_first_n < 0; ++i) {
            const int kb = (i + rot) < num_kb ? i + rot : i + rot - num_kb;
            const int s0 = kb * SPB > ko32 ? kb * SPB : ko32;
            if (s0 < (kb + 1) * SPB && s0 < k32) {
              seg_first_n = s0;
              kb_seg_first_n = kb;
            }
          }
        }
        // trace clocks go straight to shared memory: a clock held in registers across the tile
        // costs the epilogue warps two spilled 64-bit values per tile
        const bool trc_mma = p.trace && blockIdx.x == static_cast<unsigned>(p.trace - 1) && item < 32 && lane == 0;
        if (trc_mma) s_trace[0][item] = clock64();
        if (C::kAccStages == 2) ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_o = tmem_base + static_cast<uint32_t>(acc * 2 * BN);
        const uint32_t d_n = d_o + BN;
        for (int i = i0; i < i1; ++i) {
          const int kb = (i + rot) < num_kb ? i + rot : i + rot - num_kb;
          // acc_o is needed only by the outlier steps: in the (last-issued) outlier block the
          // normal steps go first and the wait for the epilogue's acc_o release sits right
          // before the first outlier step
          const bool wait_o = C::kAccStages == 1 && ko32 > 0 && kb == 0;
          if (C::kAccStages == 1) {
            if (kb == kb_seg_first_n) ctl_wait(&tempty[0], acc_phase ^ 1);   // acc_n free
            ptx::tc_fence_after();
          }
          ctl_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint64_t ad = a_desc0 + static_cast<uint64_t>(stage * (C::kABytes >> 4));
          const uint64_t bd = b_desc0 + static_cast<uint64_t>(stage * (C::kBBytes >> 4));
          auto issue = [&](bool outlier_pass) {
            if (lane == 0 && p.debug != 1) {
#pragma unroll
              for (int j = 0; j < SPB; ++j) {
                const int s32 = kb * SPB + j;  // K=32 step index
                const bool outl = s32 < ko32;
                if (s32 < k32 && outl == outlier_pass) {
                  const uint32_t d = outl ? d_o : d_n;
                  const uint32_t accumulate = (outl ? s32 == 0 : s32 == seg_first_n) ? 0u : 1u;
                  // sub-tile j/4; +32 bytes along K inside the 128B swizzle row = +2 in the
                  // >>4 address field
                  const uint64_t ao = static_cast<uint64_t>((j >> 2) * (C::kASub >> 4) + 2 * (j & 3));
                  const uint64_t bo = static_cast<uint64_t>((j >> 2) * (C::kBSub >> 4) + 2 * (j & 3));
                  if (CG == 1) ptx::mma_i8(d, ad + ao, bd + bo, idesc, accumulate);
                  else ptx::mma_i8_2sm(d, ad + ao, bd + bo, idesc, accumulate);
                }
              }
            }
          };
          // all SPB steps of this block are normal and inside K: straight-line issue
          const bool plain = kb * SPB >= ko32 && (kb + 1) * SPB <= k32;
          if (plain) {
            if (p.debug != 1 && ptx::elect_one()) {
              const uint32_t acc0 = kb * SPB == seg_first_n ? 0u : 1u;
#pragma unroll
              for (int j = 0; j < SPB; ++j) {
                constexpr uint64_t kA = C::kASub >> 4, kB = C::kBSub >> 4;
                const uint64_t ao = static_cast<uint64_t>(j >> 2) * kA + 2 * (j & 3);
                const uint64_t bo = static_cast<uint64_t>(j >> 2) * kB + 2 * (j & 3);
                if (CG == 1) ptx::mma_i8(d_n, ad + ao, bd + bo, idesc, j == 0 ? acc0 : 1u);
                else ptx::mma_i8_2sm(d_n, ad + ao, bd + bo, idesc, j == 0 ? acc0 : 1u);
              }
            }
          } else {
          issue(false);
          if (wait_o) {
            __syncwarp();
            ctl_wait(&tofree[0], acc_phase ^ 1);  // acc_o free
            ptx::tc_fence_after();
          }
          issue(true);
          }
          __syncwarp();
          if (lane == 0) {
            if (CG == 1) ptx::mma_commit(&empty[stage]);
            else ptx::mma_commit_2sm_mc(&empty[stage], 0x3);
          }
          __syncwarp();
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (lane == 0) {
          if (CG == 1) ptx::mma_commit(&tfull[acc]);
          else ptx::mma_commit_2sm_mc(&tfull[acc], 0x3);
          const int ti = item;
          if (p.trace && blockIdx.x == static_cast<unsigned>(p.trace - 1) && ti < 32) s_trace[1][ti] = clock64();
        }
        ++item;
        __syncwarp();
        if (++acc == C::kAccStages) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue: 16 warps, 4 per TMEM lane quadrant =====================
    ptx::setmaxnreg_inc<kEpiRegs>();
    // Warp w may only touch TMEM lanes 32*(w%4)..+31; the four warps of a quadrant take
    // every fourth 16-column chunk.  Each tile's column scales are prefetched one tile
    // ahead; bf16 results go through a 32B-swizzled staging tile and a TMA bulk tensor store.
    constexpr int kSubs = kEpiWarps / 4;
    const int ew = warp - 4;
    const int q = warp & 3;
    const int half = ew >> 2;  // this warp's chunk phase within its quadrant
    const int etid = ew * 32 + lane;
    const bool has_outlier = p.k_o > 0;
    const bool gelu = (p.epilogue & QARVD_EPI_GELU) != 0;
    // two-step release (see the MMA issuer) for bf16/f32 outputs without debug dumps
    const bool two_step = C::kAccStages == 1 && p.out_dtype != QARVD_F64 && !p.acc_n_dbg &&
                          !p.acc_o_dbg;
    const int epi_mode = (has_outlier ? 1 : 0) | (p.bias ? 2 : 0) | (gelu && !two_step ? 4 : 0);
    uint8_t* ystage0 = epi_ystage + ew * kYStageBytes * C::kYBufs;  // kYBufs x (32 rows x 32 B, SWIZZLE_32B)
    int ybuf = 0;
    // Column scales: every warp stages the 64 (BN / kSubs) columns it owns in a private
    // [3][WC] slot (s_wn, s_wo, bias), prefetched one tile ahead -- no cross-warp barrier, so
    // the 16 warps drift freely between the TMEM handshakes.
    constexpr int WC = BN / kSubs;
    float* wsc = epi_scales + ew * 3 * WC;
    auto scol = [&](int c) { return wsc + ((c - half) / kSubs) * CW; };  // chunk c's scales
    float pf_n[WC / 32], pf_o[WC / 32], pf_b[WC / 32], pf_x = 0.f;
#pragma unroll
    for (int u = 0; u < WC / 32; ++u) pf_n[u] = pf_o[u] = pf_b[u] = 0.f;
    auto prefetch = [&](int tt) {
      if (tt >= p.num_tiles || p.out_dtype == QARVD_F64) return;
#pragma unroll
      for (int u = 0; u < WC / 32; ++u) {
        const int jl = lane + 32 * u;
        const int64_t j = static_cast<int64_t>((QZ && p.row_major) ? tt % p.num_n_blks : tt / p.num_m_blks) * BN +
                          (half + (jl / CW) * kSubs) * CW + jl % CW;
        const int64_t jc = j < p.n ? j : p.n - 1;
        pf_n[u] = __ldg(p.scale_wn + jc);
        if (has_outlier) pf_o[u] = __ldg(p.scale_wo + jc);
        if (p.bias) pf_b[u] = __ldg(p.bias + jc);
      }
      const int64_t r = static_cast<int64_t>((QZ && p.row_major) ? tt / p.num_n_blks : tt % p.num_m_blks) * TM +
                        rank * BM + q * 32 + lane;
      pf_x = (r < p.m && p.scale_x) ? __ldg(p.scale_x + r) : 0.f;
    };
    auto release = [&](uint64_t* bar) {
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 1) ptx::mbar_arrive(bar);
        else ptx::mbar_arrive_leader(bar);
      }
    };
    // |y| max of the row over this tile (sign-cleared bf16 bits, packed 16-bit lanes); the
    // consumer's per-token K1 reads it instead of re-reducing the row (pipeline.QuantizedChain)
    uint32_t tile_mx = 0;
    // y (fp32 bits in rn) -> bf16 TMA store, or direct bf16 / f32 stores
    auto store_chunk = [&](uint32_t (&rn)[CW], int64_t row0, int64_t row, int64_t col0, int ncols) {
      if (p.use_tma_store) {
        uint32_t pk[CW / 2];
#pragma unroll
        for (int e = 0; e < CW / 2; ++e) {
          const __nv_bfloat162 h2 =
              __floats2bfloat162_rn(__uint_as_float(rn[2 * e]), __uint_as_float(rn[2 * e + 1]));
          pk[e] = *reinterpret_cast<const uint32_t*>(&h2);
        }
        if (p.row_absmax || p.row_pmax) {
#pragma unroll
          for (int e = 0; e < CW / 2; ++e) {
            const uint32_t keep = (2 * e + 1 < ncols ? 0x7fff7fffu : 0u) | (2 * e < ncols ? 0x7fffu : 0u);
            tile_mx = __vmaxu2(tile_mx, pk[e] & keep);
          }
        }
        uint8_t* ystage = ystage0 + ybuf * kYStageBytes;
        if (C::kYBufs == 2) {
          ybuf ^= 1;
          if (lane == 0) ptx::bulk_wait_read1();  // the store issued from this buffer has read it
        } else if (lane == 0) {
          ptx::bulk_wait_read0();
        }
        __syncwarp();
        // SWIZZLE_32B: the 16-byte half index of row r is XORed with bit 7 of the row's
        // byte offset (r >> 2 & 1), which also spreads a warp's 16-byte stores over all banks
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int phys = (i ^ ((lane >> 2) & 1)) << 4;
          *reinterpret_cast<uint4*>(ystage + lane * 32 + phys) =
              make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
        }
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0 && row0 < p.m) {
          ptx::tma_store_2d(&tmY, ystage, static_cast<int32_t>(col0), static_cast<int32_t>(row0));
          ptx::bulk_commit();
        }
      } else if (row < p.m && p.out_dtype == QARVD_BF16) {
        __nv_bfloat16* yr = reinterpret_cast<__nv_bfloat16*>(p.y) + row * p.ldy + col0;
#pragma unroll
        for (int e = 0; e < CW; ++e)
          if (e < ncols) {
            const __nv_bfloat16 h = __float2bfloat16_rn(__uint_as_float(rn[e]));
            yr[e] = h;
            tile_mx = max(tile_mx, static_cast<uint32_t>(__bfloat16_as_ushort(h)) & 0x7fffu);
          }
      } else if (row < p.m) {
        float* yr = reinterpret_cast<float*>(p.y) + row * p.ldy + col0;
        if (ncols == CW && ((reinterpret_cast<uintptr_t>(yr) & 15) == 0)) {
          float4* dst = reinterpret_cast<float4*>(yr);
#pragma unroll
          for (int v4 = 0; v4 < CW / 4; ++v4)
            dst[v4] = make_float4(__uint_as_float(rn[4 * v4]), __uint_as_float(rn[4 * v4 + 1]),
                                  __uint_as_float(rn[4 * v4 + 2]), __uint_as_float(rn[4 * v4 + 3]));
        } else {
#pragma unroll
          for (int e = 0; e < CW; ++e)
            if (e < ncols) yr[e] = __uint_as_float(rn[e]);
        }
      }
    };
    const SkSched sks(p.num_tiles, num_ctas, p.sk_tiles, num_kb);
    SkIter<SKT> it(sks, cta_id);
    int t, i0, i1, item = 0;
    int nt = -1, ni0 = 0, ni1 = 0;  // the item after this one (scale prefetch)
    bool have = it.next(sks, t, i0, i1);
    if (have) prefetch(t);
    // fused quantizer: this launch's epoch (launches completed on the workspace + 1) and 1/qmax
    const unsigned long long qz_epoch = QZ ? __ldcg(p.qz_epoch) + 1ull : 0ull;
    const double qz_rq = QZ ? 1.0 / static_cast<double>(p.qz_qmax) : 0.0;
    // static per-tensor mode: r = fl32(1 / s) (quantize.cu scale_static), unusable r -> division
    const double qz_rd = QZ && p.qz_static ? 1.0 / p.qz_s_static : 0.0;
    const float qz_sr = static_cast<float>(qz_rd);
    const float qz_fq = static_cast<float>(p.qz_qmax);
    const bool qz_sexact = QZ && p.qz_static && !(qz_rd <= static_cast<double>(FLT_MAX) && qz_rd >= static_cast<double>(FLT_MIN));
    // fused quantizer, static per-tensor scale: bf16-round one 16-column chunk (fp32 bits in rn),
    // its codes straight away (no row maximum to wait for), staged and TMA-stored
    auto qz_static_chunk = [&](const uint32_t (&rn)[CW], int64_t row0_, bool row_ok_, int64_t row_, int64_t col0,
                               int i) {
      uint32_t pk[CW / 2];
      uint32_t cm = 0;
#pragma unroll
      for (int e = 0; e < CW / 2; ++e) {
        const __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(rn[2 * e]), __uint_as_float(rn[2 * e + 1]));
        pk[e] = *reinterpret_cast<const uint32_t*>(&h2);
        cm = __vmaxu2(cm, pk[e] & 0x7fff7fffu);
      }
      const bool bad = max(cm & 0xffffu, cm >> 16) >= 0x7f80u;  // non-finite: reported
      const uint4 d0 = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      const uint4 d1 = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      float dm0 = 0.f, dm1 = 0.f;
      uint2 lo = qz_codes8_static(d0, qz_sr, qz_fq, dm0);
      uint2 hi = qz_codes8_static(d1, qz_sr, qz_fq, dm1);
      if (row_ok_ && (qz_sexact || bad || dm0 > kQzGuardStatic || dm1 > kQzGuardStatic)) {
        const int64_t flat = row_ * p.qz_ldq + col0;
        if (qz_sexact || bad || dm0 > kQzGuardStatic) lo = qz_div8(d0, p.qz_s_static, p.qz_qmax, p.qz_err, flat);
        if (qz_sexact || bad || dm1 > kQzGuardStatic) hi = qz_div8(d1, p.qz_s_static, p.qz_qmax, p.qz_err, flat + 8);
      }
      uint8_t* stg = ystage0 + (i & 1) * (kYStageBytes / 2);
      if (lane == 0) ptx::bulk_wait_read1();  // the store issued from this buffer has read it
      __syncwarp();
      *reinterpret_cast<uint4*>(stg + lane * 16) = make_uint4(lo.x, lo.y, hi.x, hi.y);
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0 && row0_ < p.m) {
        ptx::tma_store_2d(&tmY, stg, static_cast<int32_t>(col0), static_cast<int32_t>(row0_));
        ptx::bulk_commit();
      }
    };
    // Fused quantizer, phase B of a tile (deferred by one tile, see below): wait until the tile's
    // row block is complete, read the row maxima and round the codes held in `u` (bf16 pairs).
    uint32_t qz_u[QZ ? BN / CW / (kEpiWarps / 4) : 1][CW / 2];
    int qz_prev_m = -1, qz_prev_n = 0;
    auto qz_phase_b = [&](int pm_blk, int pn_blk) {
      constexpr int kSubsQ = kEpiWarps / 4;
      constexpr int NCHQ = BN / CW / kSubsQ;
      const int halfq = ew >> 2;
      const int64_t prow0 = static_cast<int64_t>(pm_blk) * TM + rank * BM + q * 32;
      const int64_t prow = prow0 + lane;
      const bool prow_ok = prow < p.m;
      const unsigned long long P = static_cast<unsigned long long>(p.num_n_blks) * CG;
      if (ew == 0 && lane == 0) {
        const unsigned long long want = qz_epoch * P;
        for (uint32_t polls = 0; ld_acquire_u64(p.qz_count + pm_blk) < want; ++polls) {
          if (polls > (1u << 24)) __trap();  // a row block that never completes: fail loudly
          __nanosleep(64);
        }
      }
      ptx::named_bar_sync(1, kEpiWarps * 32);
      uint32_t mag = 0;
      if (prow_ok) {
        const unsigned long long v = ld_acquire_u64(p.qz_rowmax + prow);
        mag = (v >> 16) == qz_epoch ? static_cast<uint32_t>(v & 0xffffu) : 0u;
      }
      const float amax = __uint_as_float(mag << 16);
      const int qmax = p.qz_qmax;
      const float r = amax > 0.f ? __fmul_rn(__frcp_rn(amax), static_cast<float>(qmax)) : 0.f;
      const bool slow = mag >= 0x7f80u || (amax > 0.f && !(r <= FLT_MAX && r >= FLT_MIN));
      double s64 = DBL_MIN;
      if (amax > 0.f) {
        const double a = static_cast<double>(amax), y = a * qz_rq;
        s64 = fma(fma(-y, static_cast<double>(qmax), a), qz_rq, y);
      }
      if (prow_ok && pn_blk == 0 && halfq == 0) {
        p.qz_sx[prow] = amax > 0.f ? __double2float_rn(s64) : 0.f;
        if (p.qz_s64) p.qz_s64[prow] = s64;
      }
      // fast codes for each group of 8; a group with a value within the tie guard (every group of
      // a rare row) again by the reference's division, out of line.  Codes go through the warp's
      // staging tile (32 rows x 16 B, two buffers) and a TMA store per chunk
#pragma unroll
      for (int i = 0; i < NCHQ; ++i) {
        const int c = halfq + i * kSubsQ;
        const uint4 d0 = make_uint4(qz_u[i][0], qz_u[i][1], qz_u[i][2], qz_u[i][3]);
        const uint4 d1 = make_uint4(qz_u[i][4], qz_u[i][5], qz_u[i][6], qz_u[i][7]);
        float dm0 = 0.f, dm1 = 0.f;
        uint2 lo = qz_codes8(d0, r, dm0);
        uint2 hi = qz_codes8(d1, r, dm1);
        if (prow_ok && (slow || dm0 > kQzGuard || dm1 > kQzGuard)) {
          const int64_t flat = prow * p.qz_ldq + static_cast<int64_t>(pn_blk) * BN + c * CW;
          if (slow || dm0 > kQzGuard) lo = qz_div8(d0, s64, qmax, slow ? p.qz_err : nullptr, flat);
          if (slow || dm1 > kQzGuard) hi = qz_div8(d1, s64, qmax, slow ? p.qz_err : nullptr, flat + 8);
        }
        uint8_t* stg = ystage0 + (i & 1) * (kYStageBytes / 2);
        if (lane == 0) ptx::bulk_wait_read1();  // the store issued from this buffer has read it
        __syncwarp();
        *reinterpret_cast<uint4*>(stg + lane * 16) = make_uint4(lo.x, lo.y, hi.x, hi.y);
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0 && prow0 < p.m) {
          ptx::tma_store_2d(&tmY, stg, static_cast<int32_t>(static_cast<int64_t>(pn_blk) * BN + c * CW),
                            static_cast<int32_t>(prow0));
          ptx::bulk_commit();
        }
      }
    };
    int acc = 0;
    uint32_t acc_phase = 0;
    for (; have; have = nt >= 0 ? (t = nt, i0 = ni0, i1 = ni1, true) : false, ++item) {
      nt = it.next(sks, nt, ni0, ni1) ? nt : -1;
      const int m_blk = (QZ && p.row_major) ? t / p.num_n_blks : t % p.num_m_blks;
      const int n_blk = (QZ && p.row_major) ? t % p.num_n_blks : t / p.num_m_blks;
#pragma unroll
      for (int u = 0; u < WC / 32; ++u) {
        wsc[lane + 32 * u] = pf_n[u];
        wsc[WC + lane + 32 * u] = pf_o[u];
        wsc[2 * WC + lane + 32 * u] = pf_b[u];
      }
      const float sx = pf_x;
      prefetch(nt >= 0 ? nt : p.num_tiles);
      const int64_t row0 = static_cast<int64_t>(m_blk) * TM + rank * BM + q * 32;
      const int64_t row = row0 + lane;
      const bool row_ok = row < p.m;
      tile_mx = 0;
      __syncwarp();  // this warp's scales visible to its lanes
      const bool trc_epi = p.trace && blockIdx.x == static_cast<unsigned>(p.trace - 1) && lane == 0 && warp == 4 &&
                           item < 32;
      if (trc_epi) s_trace[2][item] = clock64();
      ptx::mbar_wait(&tfull[acc], acc_phase);
      if (trc_epi) s_trace[3][item] = clock64();
      ptx::tc_fence_after();
      const uint32_t t_lane = static_cast<uint32_t>(q * 32) << 16;
      const uint32_t t_o = tmem_base + t_lane + static_cast<uint32_t>(acc * 2 * BN);
      const uint32_t t_n = t_o + BN;
      // Fast path (the deployment case: two-step bf16 TMA stores, tile inside N, no debug
      // outputs): compile-time chunk loops with the per-chunk checks hoisted to the tile.
      const bool fast = two_step && (p.use_tma_store || QZ) && !p.row_absmax &&
                        static_cast<int64_t>(n_blk + 1) * BN <= p.n;
      if (BN <= 128 && p.out_dtype == QARVD_F64 && p.f64_slices == 8 && p.k <= 32768 && !p.acc_n_dbg &&
          !p.acc_o_dbg) {
        // K7's slice products: every chunk of the warp (both slabs) is read into registers and
        // the TMEM stage is released at once, so the next tile's MMAs overlap this tile's f64
        // recombination
        constexpr int NCH = BN / CW / kSubs;
        uint32_t an[NCH][CW], ao[NCH][CW];
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
          ptx::tmem_ld16(t_n + (half + i * kSubs) * CW, an[i]);
          if (has_outlier) ptx::tmem_ld16(t_o + (half + i * kSubs) * CW, ao[i]);
        }
        const int64_t run_base = (static_cast<int64_t>(n_blk) * BN + half * CW) / 8;
        const double sx64 = row_ok ? p.sx64[row] : 0.0;
        ptx::tmem_wait_ld();
        release(&tempty[acc]);
        if (C::kAccStages == 1) release(&tofree[0]);
        if (row_ok) {
          double* yr = reinterpret_cast<double*>(p.y) + row * p.ldy + run_base;
          const bool vec = ((reinterpret_cast<uintptr_t>(yr) | static_cast<uintptr_t>(p.ldy * 8)) & 15) == 0;
#pragma unroll
          for (int i = 0; i < NCH; ++i) {
            if ((run_base + i * (kSubs * CW / 8)) * 8 >= p.n) break;
            const int64_t r0 = run_base + i * (kSubs * CW / 8);
            double out[2];
#pragma unroll
            for (int g = 0; g < 2; ++g) {
              const double vn = __dmul_rn(__dmul_rn(sx64, p.sn64[r0 + g]), slice_value<8, true>(an[i] + 8 * g));
              out[g] = has_outlier
                           ? __dadd_rn(__dmul_rn(__dmul_rn(sx64, p.so64[r0 + g]), slice_value<8, true>(ao[i] + 8 * g)), vn)
                           : vn;
            }
            double* dst = yr + i * (kSubs * CW / 8);
            if (vec) {
              *reinterpret_cast<double2*>(dst) = make_double2(out[0], out[1]);
            } else {
              dst[0] = out[0];
              dst[1] = out[1];
            }
          }
        }
      } else if (fast && p.epi_regs && !QZ) {
        // register-held variant: the warp's 4 acc_n chunks (64 columns) are read into
        // registers and acc_n is released at once; the dequant/GELU/stores then overlap the
        // next tile's normal-slab MMAs and only acc_o (read chunk by chunk) gates its outliers.
        constexpr int NCH = BN / CW / kSubs;
        uint32_t an[NCH][CW];
#pragma unroll
        for (int i = 0; i < NCH; ++i) ptx::tmem_ld16(t_n + (half + i * kSubs) * CW, an[i]);
        ptx::tmem_wait_ld();
        release(&tempty[0]);  // acc_n free: the next tile's normal-slab MMAs may start
        if (p.trace && blockIdx.x == static_cast<unsigned>(p.trace - 1) && lane == 0 && warp == 4) {
          const int ti = item;
          if (ti < 32) s_trace[5][ti] = clock64();
        }
        // stream-K: slot layout [tile][slot][BN columns][TM rows] (a warp's 32 rows of one
        // column are 128 contiguous bytes)
        const int trow = static_cast<int>(rank) * BM + q * 32 + lane;
        bool sk_partial = false;
        if (SKT && t < p.sk_tiles) {
          uint32_t* cnt = p.sk_count + 2 * t;
          if (i1 < num_kb) {
            // not the owner: publish this pair's partial acc_n and signal the owner
            int32_t* slot = p.sk_slots + (static_cast<int64_t>(t) * p.sk_slots_per_tile + sks.slot_of(t, cta_id)) *
                                             (static_cast<int64_t>(BN) * TM);
#pragma unroll
            for (int i = 0; i < NCH; ++i)
#pragma unroll
              for (int e = 0; e < CW; ++e)
                slot[static_cast<int64_t>((half + i * kSubs) * CW + e) * TM + trow] =
                    static_cast<int32_t>(an[i][e]);
            __syncwarp();
            if (lane == 0) {
              __threadfence();  // cumulative over the warp's stores ordered by the barrier
              atomicAdd(cnt, 1u);
            }
            release(&tofree[0]);
            sk_partial = true;
          } else if (sks.partials(t) > 0) {
            // owner: wait for every partial (one arrival per writer warp), add them (int32,
            // exact), and the last reader warp resets the counters for the next launch
            const uint32_t want = static_cast<uint32_t>(sks.partials(t) * kEpiWarps * CG);
            if (lane == 0) {
              uint32_t got;
              asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(got) : "l"(cnt) : "memory");
              while (got < want) {
                __nanosleep(256);
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(got) : "l"(cnt) : "memory");
              }
            }
            __syncwarp();
            __threadfence();
            const int32_t* slot0 = p.sk_slots + static_cast<int64_t>(t) * p.sk_slots_per_tile *
                                                    (static_cast<int64_t>(BN) * TM);
            for (int sl = 0; sl < sks.partials(t); ++sl) {
              const int32_t* slot = slot0 + static_cast<int64_t>(sl) * BN * TM;
#pragma unroll
              for (int i = 0; i < NCH; ++i)
#pragma unroll
                for (int e = 0; e < CW; ++e)
                  an[i][e] = static_cast<uint32_t>(
                      static_cast<int32_t>(an[i][e]) +
                      __ldcg(slot + static_cast<int64_t>((half + i * kSubs) * CW + e) * TM + trow));
            }
            __syncwarp();
            if (lane == 0 && atomicAdd(cnt + 1, 1u) == static_cast<uint32_t>(kEpiWarps * CG) - 1u) {
              cnt[0] = 0u;
              cnt[1] = 0u;
            }
          }
        }
        using T_ = std::true_type;
        using F_ = std::false_type;
        // t = s_wn*acc_n (+ s_wo*acc_o) into the held registers, then acc_o is released too:
        // the whole y = s_x*t (+ b) [gelu] -> bf16 tail overlaps the next tile's MMAs
        auto fold = [&](auto ho) {
          constexpr bool HO = decltype(ho)::value;
#pragma unroll
          for (int i = 0; i < NCH; ++i) {
            const int c = half + i * kSubs;
            uint32_t ro[CW];
            if (HO) {
              ptx::tmem_ld16(t_o + c * CW, ro);
              ptx::tmem_wait_ld();
            }
            const float* scc = scol(c);
#pragma unroll
            for (int e4 = 0; e4 < CW / 4; ++e4) {
              const float4 sn4 = reinterpret_cast<const float4*>(scc)[e4];
              float4 so4 = sn4;
              if (HO) so4 = reinterpret_cast<const float4*>(scc + WC)[e4];
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int e = 4 * e4 + 2 * h;
                const uint64_t sn = h ? pk2(sn4.z, sn4.w) : pk2(sn4.x, sn4.y);
                const uint64_t a2 = pk2(__int2float_rn(static_cast<int>(an[i][e])),
                                        __int2float_rn(static_cast<int>(an[i][e + 1])));
                uint64_t tt;
                if (HO) {
                  const uint64_t so = h ? pk2(so4.z, so4.w) : pk2(so4.x, so4.y);
                  const uint64_t ao = pk2(__int2float_rn(static_cast<int>(ro[e])),
                                          __int2float_rn(static_cast<int>(ro[e + 1])));
                  tt = fma2(sn, a2, mul2(so, ao));
                } else {
                  tt = mul2(sn, a2);
                }
                float y0, y1;
                upk2(tt, y0, y1);
                an[i][e] = __float_as_uint(y0);
                an[i][e + 1] = __float_as_uint(y1);
              }
            }
          }
        };
        if (sk_partial) {
        } else {
        if (has_outlier) fold(T_{});
        else fold(F_{});
        release(&tofree[0]);  // acc_o free: the next tile's outlier steps may issue
        const uint64_t sx2 = pk2(sx, sx);
        auto tail = [&](auto hb, auto gl) {
          constexpr bool HB = decltype(hb)::value, GL = decltype(gl)::value;
#pragma unroll
          for (int i = 0; i < NCH; ++i) {
            const int c = half + i * kSubs;
            const float* scb = scol(c) + 2 * WC;
#pragma unroll
            for (int e4 = 0; e4 < CW / 4; ++e4) {
              float4 sb4 = make_float4(0.f, 0.f, 0.f, 0.f);
              if (HB) sb4 = reinterpret_cast<const float4*>(scb)[e4];
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int e = 4 * e4 + 2 * h;
                const uint64_t tt = pk2(__uint_as_float(an[i][e]), __uint_as_float(an[i][e + 1]));
                uint64_t v;
                if (HB) v = fma2(sx2, tt, h ? pk2(sb4.z, sb4.w) : pk2(sb4.x, sb4.y));
                else v = mul2(sx2, tt);
                if (GL) v = gelu2(v);
                float y0, y1;
                upk2(v, y0, y1);
                an[i][e] = __float_as_uint(y0);
                an[i][e + 1] = __float_as_uint(y1);
              }
            }
            if (p.debug & 32) {  // diagnostic: math without stores
#pragma unroll
              for (int e = 0; e < CW; ++e) tile_mx ^= an[i][e];
            } else {
              store_chunk(an[i], row0, row, static_cast<int64_t>(n_blk) * BN + c * CW, CW);
            }
          }
          if ((p.debug & 32) && tile_mx == 0x12345678u) p.acc_o_dbg[0] = 1;
        };
        if (p.debug & 16) {  // diagnostic: no tail (fold + releases only)
        } else if (gelu) {
          if (p.bias) tail(T_{}, T_{});
          else tail(F_{}, T_{});
        } else {
          if (p.bias) tail(T_{}, F_{});
          else tail(F_{}, F_{});
        }
        }  // owner / data-parallel item
      } else if (fast) {
        // phase 1 (blocks the next tile's normal slab): t = s_wn*acc_n (+ s_wo*acc_o), folded
        // into acc_o's columns as f32 bits; phase 2 (overlaps the next tile's MMAs):
        // y = s_x*t (+ b) [gelu] -> bf16.  Same per-element op order as epi_math.
        auto phase1 = [&](auto ho) {
          constexpr bool HO = decltype(ho)::value;
#pragma unroll
          for (int i = 0; i < BN / CW / kSubs; ++i) {
            const int c = half + i * kSubs;
            uint32_t rn[CW], ro[CW];
            ptx::tmem_ld16(t_n + c * CW, rn);
            if (HO) ptx::tmem_ld16(t_o + c * CW, ro);
            ptx::tmem_wait_ld();
            const float* scc = scol(c);
#pragma unroll
            for (int e4 = 0; e4 < CW / 4; ++e4) {
              const float4 sn4 = reinterpret_cast<const float4*>(scc)[e4];
              float4 so4 = sn4;
              if (HO) so4 = reinterpret_cast<const float4*>(scc + WC)[e4];
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int e = 4 * e4 + 2 * h;
                const uint64_t sn = h ? pk2(sn4.z, sn4.w) : pk2(sn4.x, sn4.y);
                const uint64_t an = pk2(__int2float_rn(static_cast<int>(rn[e])),
                                        __int2float_rn(static_cast<int>(rn[e + 1])));
                uint64_t tt;
                if (HO) {
                  const uint64_t so = h ? pk2(so4.z, so4.w) : pk2(so4.x, so4.y);
                  const uint64_t ao = pk2(__int2float_rn(static_cast<int>(ro[e])),
                                          __int2float_rn(static_cast<int>(ro[e + 1])));
                  tt = fma2(sn, an, mul2(so, ao));
                } else {
                  tt = mul2(sn, an);
                }
                float y0, y1;
                upk2(tt, y0, y1);
                rn[e] = __float_as_uint(y0);
                rn[e + 1] = __float_as_uint(y1);
              }
            }
            ptx::tmem_st16(t_o + c * CW, rn);  // fold t into acc_o's columns
          }
        };
        using T_ = std::true_type;
        using F_ = std::false_type;
        if (has_outlier) phase1(T_{});
        else phase1(F_{});
        ptx::tmem_wait_st();
        release(&tempty[0]);  // acc_n free: the next tile's normal-slab MMAs may start
        if (p.trace && blockIdx.x == static_cast<unsigned>(p.trace - 1) && lane == 0 && warp == 4) {
          const int ti = item;
          if (ti < 32) s_trace[5][ti] = clock64();
        }
        // fused quantizer: the previous tile's phase B while this tile's MMAs run (qz_u is free
        // again for this tile's bf16 values afterwards)
        if (QZ && qz_prev_m >= 0) qz_phase_b(qz_prev_m, qz_prev_n);
        const uint64_t sx2 = pk2(sx, sx);
        auto phase2 = [&](auto gl, auto hb, auto direct) {
          constexpr bool GL = decltype(gl)::value, HB = decltype(hb)::value;
          constexpr bool DS = decltype(direct)::value;
#pragma unroll
          for (int i = 0; i < BN / CW / kSubs; ++i) {
            const int c = half + i * kSubs;
            uint32_t rn[CW];
            ptx::tmem_ld16(t_o + c * CW, rn);
            ptx::tmem_wait_ld();
            const float* scb = scol(c) + 2 * WC;
#pragma unroll
            for (int e4 = 0; e4 < CW / 4; ++e4) {
              float4 sb4 = make_float4(0.f, 0.f, 0.f, 0.f);
              if (HB) sb4 = reinterpret_cast<const float4*>(scb)[e4];
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int e = 4 * e4 + 2 * h;
                const uint64_t tt = pk2(__uint_as_float(rn[e]), __uint_as_float(rn[e + 1]));
                uint64_t v;
                if (HB) v = fma2(sx2, tt, h ? pk2(sb4.z, sb4.w) : pk2(sb4.x, sb4.y));
                else v = mul2(sx2, tt);
                if (GL) v = gelu2(v);
                float y0, y1;
                upk2(v, y0, y1);
                rn[e] = __float_as_uint(y0);
                rn[e + 1] = __float_as_uint(y1);
              }
            }
            const int64_t col0 = static_cast<int64_t>(n_blk) * BN + c * CW;
            if (QZ && p.qz_static) {
              qz_static_chunk(rn, row0, row_ok, row, col0, i);
            } else if (QZ) {
              // the bf16 output stays in registers for the deferred phase B
#pragma unroll
              for (int e = 0; e < CW / 2; ++e) {
                const __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(rn[2 * e]),
                                                                __uint_as_float(rn[2 * e + 1]));
                const uint32_t b = *reinterpret_cast<const uint32_t*>(&h2);
                qz_u[QZ ? i : 0][e] = b;
                tile_mx = __vmaxu2(tile_mx, b & 0x7fff7fffu);
              }
            } else if (DS) {
              uint32_t pk[CW / 2];
#pragma unroll
              for (int e = 0; e < CW / 2; ++e) {
                const __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(rn[2 * e]),
                                                                __uint_as_float(rn[2 * e + 1]));
                pk[e] = *reinterpret_cast<const uint32_t*>(&h2);
                if (p.row_pmax) tile_mx = __vmaxu2(tile_mx, pk[e] & 0x7fff7fffu);
              }
              if (row_ok) {
                uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.y) +
                                                      row * p.ldy + col0);
                dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
              }
            } else {
              store_chunk(rn, row0, row, col0, CW);
            }
          }
        };
        const bool direct = p.direct_store != 0;
        auto phase2_b = [&](auto gl, auto hb) {
          if (p.debug & 4) {  // diagnostic: phase 2 reads TMEM only (no math, no stores)
#pragma unroll
            for (int i = 0; i < BN / CW / kSubs; ++i) {
              uint32_t rn[CW];
              ptx::tmem_ld16(t_o + (half + i * kSubs) * CW, rn);
              ptx::tmem_wait_ld();
#pragma unroll
              for (int e = 0; e < CW; ++e) tile_mx ^= rn[e];
            }
            if (tile_mx == 0x12345678u) p.acc_o_dbg[0] = 1;
            return;
          }
          if (p.debug & 8) phase2(F_{}, F_{}, F_{});  // diagnostic: stores without GELU
          else if (direct && !QZ) phase2(gl, hb, T_{});
          else phase2(gl, hb, F_{});
        };
        if (gelu) {
          if (p.bias) phase2_b(T_{}, T_{});
          else phase2_b(T_{}, F_{});
        } else {
          if (p.bias) phase2_b(F_{}, T_{});
          else phase2_b(F_{}, F_{});
        }
        release(&tofree[0]);  // acc_o free
        if (QZ && p.qz_static) {
          if (row_ok && n_blk == 0 && half == 0) {
            p.qz_sx[row] = __double2float_rn(p.qz_s_static);
            if (p.qz_s64) p.qz_s64[row] = p.qz_s_static;
          }
        } else if (QZ) {
          // Fused consumer K1.  The row's |y| max spans every N tile of its row block (other SM
          // pairs).  Phase A (here): each warp publishes its 64-column partial max tagged with
          // this launch's epoch e (64-bit atomicMax of (e << 16) | bf16 bits: older launches'
          // values lose) and one thread per CTA arrives on the row block's counter.  Phase B
          // (qz_phase_b, deferred to the next tile, after its phase 1 has released acc_n, so the
          // row block has had a tile period to complete and the wait overlaps the MMAs): wait
          // until the counter reaches e * P (every arrival of launches 1..e), round the held
          // bf16 values.  Tiles run in row-major order on a persistent grid whose CTAs are all
          // resident (checked on the host), so every tile a row block waits for has started: its
          // pair finished its earlier tiles' phase A.  Nothing is reset: counters only grow,
          // stale maxima carry old epochs.
          const uint32_t part = max(tile_mx & 0xffffu, tile_mx >> 16);
          if (row_ok && part) atomicMax(p.qz_rowmax + row, (qz_epoch << 16) | part);
          ptx::named_bar_sync(1, kEpiWarps * 32);  // the CTA's partial maxima are published
          if (ew == 0 && lane == 0) {
            __threadfence();
            atomicAdd(p.qz_count + m_blk, 1ull);
          }
          qz_prev_m = m_blk;
          qz_prev_n = n_blk;
        }
      } else {
#pragma unroll 1
      for (int c = half; c < BN / CW; c += kSubs) {
        const int64_t col0 = static_cast<int64_t>(n_blk) * BN + c * CW;
        if (col0 >= p.n) break;  // warp-uniform
        const int ncols = (p.n - col0) < CW ? static_cast<int>(p.n - col0) : CW;
        uint32_t rn[CW], ro[CW];
        ptx::tmem_ld16(t_n + c * CW, rn);
        if (has_outlier) ptx::tmem_ld16(t_o + c * CW, ro);
        ptx::tmem_wait_ld();
        if (p.out_dtype == QARVD_F64) {
          // exact restatement of the reference epilogue: val = 0; val += (s_x*s_wo)*acc_o;
          // val += (s_x*s_wn)*acc_n  (outlier group first, f64, no FMA)
          if (row_ok) {
            const double sx64 = p.sx64[row];
            const int T = p.f64_slices;
            if (T > 1) {  // n % 16 == 0 and T | 16: whole runs only
              double* yr = reinterpret_cast<double*>(p.y) + row * p.ldy + col0 / T;
              if (p.k <= 32768) {
                switch (T) {
                  case 2: slice_runs<2, true>(rn, ro, has_outlier, sx64, p.so64, p.sn64, col0 / T, yr); break;
                  case 4: slice_runs<4, true>(rn, ro, has_outlier, sx64, p.so64, p.sn64, col0 / T, yr); break;
                  case 8: slice_runs<8, true>(rn, ro, has_outlier, sx64, p.so64, p.sn64, col0 / T, yr); break;
                  default: slice_runs<16, true>(rn, ro, has_outlier, sx64, p.so64, p.sn64, col0 / T, yr); break;
                }
              } else {
                switch (T) {
                  case 2: slice_runs<2, false>(rn, ro, has_outlier, sx64, p.so64, p.sn64, col0 / T, yr); break;
                  case 4: slice_runs<4, false>(rn, ro, has_outlier, sx64, p.so64, p.sn64, col0 / T, yr); break;
                  case 8: slice_runs<8, false>(rn, ro, has_outlier, sx64, p.so64, p.sn64, col0 / T, yr); break;
                  default: slice_runs<16, false>(rn, ro, has_outlier, sx64, p.so64, p.sn64, col0 / T, yr); break;
                }
              }
              continue;
            }
            double vv[CW];
#pragma unroll
            for (int e = 0; e < CW; ++e) {
              double v = 0.0;
              if (e < ncols) {
                if (has_outlier)
                  v = __dadd_rn(v, __dmul_rn(__dmul_rn(sx64, p.so64[col0 + e]),
                                             static_cast<double>(static_cast<int32_t>(ro[e]))));
                v = __dadd_rn(v, __dmul_rn(__dmul_rn(sx64, p.sn64[col0 + e]),
                                           static_cast<double>(static_cast<int32_t>(rn[e]))));
              }
              vv[e] = v;
            }
            {
              double* yr = reinterpret_cast<double*>(p.y) + row * p.ldy + col0;
#pragma unroll
              for (int e = 0; e < CW; ++e)
                if (e < ncols) yr[e] = vv[e];
            }
          }
          continue;
        }
        if (row_ok && p.acc_n_dbg) {
#pragma unroll
          for (int e = 0; e < CW; ++e) {
            if (e >= ncols) continue;
            p.acc_n_dbg[row * p.n + col0 + e] = static_cast<int32_t>(rn[e]);
            if (p.acc_o_dbg)
              p.acc_o_dbg[row * p.n + col0 + e] = has_outlier ? static_cast<int32_t>(ro[e]) : 0;
          }
        }
        {
          const float* scc = scol(c);
          switch (epi_mode) {
            case 0: epi_math<false, false, false>(rn, ro, scc, WC, sx); break;
            case 1: epi_math<true, false, false>(rn, ro, scc, WC, sx); break;
            case 2: epi_math<false, true, false>(rn, ro, scc, WC, sx); break;
            case 3: epi_math<true, true, false>(rn, ro, scc, WC, sx); break;
            case 4: epi_math<false, false, true>(rn, ro, scc, WC, sx); break;
            case 5: epi_math<true, false, true>(rn, ro, scc, WC, sx); break;
            case 6: epi_math<false, true, true>(rn, ro, scc, WC, sx); break;
            default: epi_math<true, true, true>(rn, ro, scc, WC, sx); break;
          }
        }
        if (two_step) ptx::tmem_st16(t_o + c * CW, rn);  // fold y into acc_o's columns
        else store_chunk(rn, row0, row, col0, ncols);
      }
      if (two_step) {
        ptx::tmem_wait_st();
        release(&tempty[0]);  // acc_n free: the next tile's normal-slab MMAs may start
        if (p.trace && blockIdx.x == static_cast<unsigned>(p.trace - 1) && lane == 0 && warp == 4) {
          const int ti = item;
          if (ti < 32) s_trace[5][ti] = clock64();
        }
#pragma unroll 1
        for (int c = half; c < BN / CW; c += kSubs) {
          const int64_t col0 = static_cast<int64_t>(n_blk) * BN + c * CW;
          if (col0 >= p.n) break;
          const int ncols = (p.n - col0) < CW ? static_cast<int>(p.n - col0) : CW;
          uint32_t rn[CW];
          ptx::tmem_ld16(t_o + c * CW, rn);
          ptx::tmem_wait_ld();
          if (gelu) {
#pragma unroll
            for (int e = 0; e < CW; e += 2) {
              float y0, y1;
              upk2(gelu2(pk2(__uint_as_float(rn[e]), __uint_as_float(rn[e + 1]))), y0, y1);
              rn[e] = __float_as_uint(y0);
              rn[e + 1] = __float_as_uint(y1);
            }
          }
          store_chunk(rn, row0, row, col0, ncols);
        }
        release(&tofree[0]);  // acc_o free
      } else {
        release(&tempty[acc]);
        if (C::kAccStages == 1) release(&tofree[0]);
      }
      }  // generic path
      if (p.row_absmax && row_ok)
        atomicMax(p.row_absmax + row, max(tile_mx & 0xffffu, tile_mx >> 16));
      if (p.row_pmax && row_ok)
        p.row_pmax[row * p.pm_count + n_blk * kSubs + half] = max(tile_mx & 0xffffu, tile_mx >> 16);
      {
        const int ti = item;
        if (p.trace && blockIdx.x == static_cast<unsigned>(p.trace - 1) && lane == 0 && warp == 4 && ti < 32)
          s_trace[4][ti] = clock64();
      }
      if (++acc == C::kAccStages) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (QZ && qz_prev_m >= 0) qz_phase_b(qz_prev_m, qz_prev_n);
    if (lane == 0) ptx::bulk_wait_all();
  } else {
    ptx::setmaxnreg_dec<kCtrlRegs>();  // warps 2-3
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (QZ && threadIdx.x == 0) {
    // the last CTA out publishes this launch's epoch (every CTA read the old one at its start)
    __threadfence();
    if (atomicAdd(p.qz_done, 1u) == gridDim.x - 1u) {
      *p.qz_epoch = __ldcg(p.qz_epoch) + 1ull;
      *p.qz_done = 0u;
      __threadfence();
    }
  }
  if (p.trace && blockIdx.x == static_cast<unsigned>(p.trace - 1) && threadIdx.x == 0) {
    unsigned long long g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    const long long c1 = clock64();
    printf("effective SM clock over the kernel: %.0f MHz\n",
           1e3 * static_cast<double>(c1 - s_clk0) / static_cast<double>(g1 - s_g0));
    const int nt = SKT ? 3 : (p.num_tiles - cta_id + num_ctas - 1) / num_ctas;
    const long long t0 = s_trace[0][0];
    printf("CTA %d (kernel start -> first MMA %lld clk, end %lld clk)\n", static_cast<int>(blockIdx.x),
           t0 - s_clk0, c1 - t0);
    for (int i = 0; i < nt && i < 32; ++i)
      printf("tile %2d: mma %7lld..%7lld  epi wait %7lld tfull %7lld phase1 %7lld done %7lld\n", i,
             s_trace[0][i] - t0, s_trace[1][i] - t0, s_trace[2][i] - t0, s_trace[3][i] - t0,
             s_trace[5][i] - t0, s_trace[4][i] - t0);
  }
  if ((p.debug & 128) && threadIdx.x == 0 && p.cta_times) {
    // diagnostic (QARVD_GEMM_DEBUG=128): per-CTA start / end globaltimer (ns)
    unsigned long long g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    p.cta_times[2 * blockIdx.x] = s_g0;
    p.cta_times[2 * blockIdx.x + 1] = g1;
  }
  if (CG == 2) ptx::cluster_sync();  // the leader's MMAs wrote this CTA's TMEM / read its smem
  if (warp == 2) {
    ptx::tc_fence_after();
    if (CG == 2) ptx::tmem_dealloc_2sm(tmem_base, C::kTmemCols);
    else ptx::tmem_dealloc(tmem_base, C::kTmemCols);
  }
}

// ---- host side -------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult qres;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qres) ==
            cudaSuccess &&
        qres == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

// 2-D int8 K-major operand [rows x k] (ld bytes), box = box_rows x 128 B, 128B swizzle.
int make_operand_tmap(CUtensorMap* map, const int8_t* base, int64_t rows, int64_t k, int64_t ld,
                      int box_rows) {
  auto encode = get_encode_fn();
  if (!encode) QARVD_FAIL(QARVD_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(base), dims,
                      strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    QARVD_FAIL(QARVD_ERR_CUDA, "cuTensorMapEncodeTiled failed with CUresult " + std::to_string(r));
  return QARVD_OK;
}

// bf16 output [m x n] (ld elements), box CW cols x 32 rows, 32B swizzle (epilogue staging)
int make_y_tmap(CUtensorMap* map, void* y, int64_t m, int64_t n, int64_t ld) {
  auto encode = get_encode_fn();
  if (!encode) QARVD_FAIL(QARVD_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(m)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
  cuuint32_t box[2] = {CW, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, y, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    QARVD_FAIL(QARVD_ERR_CUDA, "cuTensorMapEncodeTiled (y) failed with CUresult " + std::to_string(r));
  return QARVD_OK;
}

// int8 codes [m x n] (ld bytes), box 16 cols x 32 rows, no swizzle (fused quantizer staging)
int make_q_tmap(CUtensorMap* map, void* q, int64_t m, int64_t n, int64_t ld) {
  auto encode = get_encode_fn();
  if (!encode) QARVD_FAIL(QARVD_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(m)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld)};
  cuuint32_t box[2] = {CW, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, q, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    QARVD_FAIL(QARVD_ERR_CUDA, "cuTensorMapEncodeTiled (q) failed with CUresult " + std::to_string(r));
  return QARVD_OK;
}

// QARVD_GEMM_DEBUG=128 diagnostic buffer (2 x 1024 globaltimer stamps), read by qarvd_debug_cta_times
unsigned long long* debug_cta_times() {
  static unsigned long long* buf = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    if (cudaMalloc(&buf, 2 * 1024 * sizeof(unsigned long long)) != cudaSuccess) buf = nullptr;
  });
  return buf;
}

int sm_count() {
  static int count = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&count, cudaDevAttrMultiProcessorCount, dev);
    if (count <= 0) count = kNumSMs;
  });
  return count;
}

template <int BN, int CG, int KS>
int launch_gemm(const int8_t* xq, int64_t ldq, const int8_t* wq, int64_t ldw, GemmParams p,
                cudaStream_t stream) {
  using C = GemmCfg<BN, CG, KS>;
  static std::once_flag attr_once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(attr_once, [] {
    attr_err = set_smem_attrs(dual_gemm_kernel<BN, CG, KS, false>, static_cast<int>(C::kSmemBytes));
    if constexpr (BN == 256 && CG == 2 && KS == 2) {
      if (attr_err == cudaSuccess)
        attr_err = set_smem_attrs(dual_gemm_kernel<BN, CG, KS, true>, static_cast<int>(C::kSmemBytes));
      if (attr_err == cudaSuccess)
        attr_err = set_smem_attrs(dual_gemm_kernel<BN, CG, KS, false, true>, static_cast<int>(C::kSmemBytes));
    }
  });
  QARVD_CUDA_TRY(attr_err);
  CUtensorMap ta, tb;
  int st = make_operand_tmap(&ta, xq, p.m, p.k, ldq, BM);
  if (st) return st;
  st = make_operand_tmap(&tb, wq, p.n, p.k, ldw, BN / CG);
  if (st) return st;
  CUtensorMap ty;
  std::memset(&ty, 0, sizeof(ty));
  p.use_tma_store = p.out_dtype == QARVD_BF16 && !p.acc_n_dbg && !p.acc_o_dbg && !p.qz && p.y &&
                    (reinterpret_cast<uintptr_t>(p.y) & 15) == 0 && (p.ldy * 2) % 16 == 0;
  {
    const char* e = std::getenv("QARVD_GEMM_DIRECT");
    p.direct_store = (e && e[0] == '1') ? 1 : 0;
    const char* r = std::getenv("QARVD_GEMM_EPIREG");
    p.epi_regs = (r && r[0] == '0') ? 0 : 1;
    const char* sp = std::getenv("QARVD_GEMM_SPIN");
    p.spin = (sp && sp[0] == '1') ? 1 : 0;
  }
  if (p.use_tma_store) {
    st = make_y_tmap(&ty, p.y, p.m, p.n, p.ldy);
    if (st) return st;
  } else if (p.qz) {
    st = make_q_tmap(&ty, p.qz_q, p.m, p.n, p.qz_ldq);
    if (st) return st;
  }
  if (!p.use_tma_store || !p.epi_regs || p.debug) p.sk_tiles = 0;  // stream-K needs the fast path
  p.num_m_blks = static_cast<int>((p.m + BM * CG - 1) / (BM * CG));
  p.num_n_blks = static_cast<int>((p.n + BN - 1) / BN);
  p.pm_count = p.num_n_blks * (kEpiWarps / 4);
  p.num_tiles = p.num_m_blks * p.num_n_blks;
  const int units = sm_count() / CG;
  const int grid = CG * (p.num_tiles < units ? p.num_tiles : units);
  if constexpr (BN == 256 && CG == 2 && KS == 2) {
  if (p.qz) {
    // the fused quantizer's row blocks wait for tiles of other CTAs: every CTA of the grid
    // must be resident at once (one per SM by its shared memory).  It runs the chunked
    // two-phase epilogue (acc_n folded into acc_o's TMEM columns), not the register-held one:
    // holding the bf16 tile for the deferred rounding leaves no registers for that variant.
    p.epi_regs = 0;
    static std::once_flag occ_once;
    static int max_units = 0;
    std::call_once(occ_once, [] {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(CG * 2);
      cfg.blockDim = dim3(kThreads);
      cfg.dynamicSmemBytes = C::kSmemBytes;
      cudaLaunchAttribute attr{};
      attr.id = cudaLaunchAttributeClusterDimension;
      attr.val.clusterDim.x = CG;
      attr.val.clusterDim.y = 1;
      attr.val.clusterDim.z = 1;
      cfg.attrs = &attr;
      cfg.numAttrs = CG > 1 ? 1 : 0;
      int n = 0;
      if (CG > 1) {
        if (cudaOccupancyMaxActiveClusters(&n, dual_gemm_kernel<BN, CG, KS, false, true>, &cfg) != cudaSuccess) n = 0;
      } else {
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dual_gemm_kernel<BN, CG, KS, false, true>, kThreads,
                                                          C::kSmemBytes) == cudaSuccess)
          n = per_sm * sm_count();
      }
      cudaGetLastError();
      max_units = n;
    });
    if (max_units < grid / CG)
      QARVD_FAIL(QARVD_ERR_UNSUPPORTED, "kernel_b (fused quantizer): the persistent grid (" + std::to_string(grid / CG) +
                                            " CTA groups) cannot be co-resident (" + std::to_string(max_units) + ")");
  }
  }
  // stream-K instance only for the deployed tile shape (the data-parallel instance keeps the
  // register budget of its epilogue)
  if (p.qz) {
    if constexpr (BN == 256 && CG == 2 && KS == 2)
      QARVD_CUDA_TRY(launch_pdl(dual_gemm_kernel<BN, CG, KS, false, true>, dim3(grid), dim3(kThreads), C::kSmemBytes,
                                stream, CG, ta, tb, ty, p));
    else
      QARVD_FAIL(QARVD_ERR_UNSUPPORTED, "kernel_b (fused quantizer): only the 256 x 256 pair-tile configuration");
  } else if (BN == 256 && CG == 2 && KS == 2 && p.sk_tiles > 0)
    QARVD_CUDA_TRY(launch_pdl(dual_gemm_kernel<BN, CG, KS, (BN == 256 && CG == 2 && KS == 2)>, dim3(grid),
                              dim3(kThreads), C::kSmemBytes, stream, CG, ta, tb, ty, p));
  else
    QARVD_CUDA_TRY(launch_pdl(dual_gemm_kernel<BN, CG, KS, false>, dim3(grid), dim3(kThreads), C::kSmemBytes,
                              stream, CG, ta, tb, ty, p));
  count_launch();
  QARVD_LAUNCH_CHECK();
  return QARVD_OK;
}

// Tile configuration (BN, CG, KS).  QARVD_GEMM_BN=128|192|256, QARVD_GEMM_CG=1|2 and
// QARVD_GEMM_KS=1|2 override.  Default: SM-pair tiles of 256 x 256 with 256-byte K stages.
// * BN = 256 halves the B traffic per MAC versus 128 but fits only one TMEM stage
//   (2 accumulators x 256 columns); the two-step release overlaps most of the epilogue.
// * KS = 2 halves the MMA issuer's per-stage mbarrier waits, which the tensor pipe does not
//   overlap: measured on the Wan FFN (M = 4680, bench.py), 256/2/2 beats the wave-exact
//   192/1/1 on N = 1536 (57.5 vs 63.7 us) as well as on N = 8960.
struct TileCfg {
  int bn, cg, ks;
};
TileCfg choose_cfg(int64_t m, int64_t n, int64_t k) {
  (void)k;
  TileCfg c{256, 2, 2};
  // small GEMMs (e.g. the cross-attention k / v projections of 512 text tokens: 12 pair tiles
  // for 74 SM pairs) run 256 x 128 tiles: twice the parallelism (measured 16.4 -> 12.3 us)
  if (((m + 255) / 256) * ((n + 255) / 256) * 2 < static_cast<int64_t>(sm_count() / 2)) c.bn = 128;

  if (const char* env = getenv("QARVD_GEMM_BN")) {
    // 192-column tiles are not offered: their epilogue leaves a third of the columns unwritten
    // at N = 1536 (found by test_k2_tile_overrides_bitexact); 128 and 256 are tested bit-exact
    const int v = atoi(env);
    if (v == 128 || v == 256) c.bn = v;
  }
  if (const char* env = getenv("QARVD_GEMM_CG")) {
    const int v = atoi(env);
    if (v == 1 || v == 2) c.cg = v;
  }
  if (const char* env = getenv("QARVD_GEMM_KS")) {
    const int v = atoi(env);
    if (v == 1 || v == 2) c.ks = v;
  }
  if (c.bn == 192 && c.cg == 2) c.ks = 1;
  return c;
}

// Stream-K workspace of one call (QARVD_GEMM_SK=1), or bytes = 0 when the call runs
// data-parallel: only the
// deployed configuration (256 x 256 pair tiles, 256-byte stages, bf16 TMA-store epilogue
// holding acc_n in registers, N a multiple of 256, the outlier slab inside one k-block) with
// a partial last wave and long K ranges (>= 8 k-blocks per pair) splits tiles.
struct SkLayout {
  int sk_tiles = 0, slots_per_tile = 0;
  int64_t count_bytes = 0, bytes = 0;
};
SkLayout sk_layout(int64_t m, int64_t n, int64_t k, int64_t k_o, int out_dtype, bool dumps) {
  SkLayout L;
  const TileCfg c = choose_cfg(m, n, k);
  // opt-in (QARVD_GEMM_SK=1): measured on the FFN-down shape it does not pay yet -- the
  // non-owners' partial stores take 10-30K cycles under the GEMM's load traffic and the owners'
  // fixups wait on them (K2)
  const char* sk_env = getenv("QARVD_GEMM_SK");
  const bool off = !(sk_env && sk_env[0] == '1');
  const char* er = std::getenv("QARVD_GEMM_EPIREG");
  if (off || (er && er[0] == '0') || c.bn != 256 || c.cg != 2 || c.ks != 2 ||
      out_dtype != QARVD_BF16 || dumps || n % 256 != 0 || k_o >= 256 || m <= 0)
    return L;
  const int pairs = sm_count() / 2;
  const int tiles = static_cast<int>((m + 255) / 256) * static_cast<int>(n / 256);
  const int nkb = static_cast<int>((k + 255) / 256);
  const int rem = tiles % pairs;
  if (rem == 0 || tiles < pairs) return L;
  const SkSched s(tiles, pairs, rem, nkb);
  if (s.units < 8LL * pairs) return L;
  int mx = 0;
  for (int t = 0; t < rem; ++t) mx = s.partials(t) > mx ? s.partials(t) : mx;
  L.sk_tiles = rem;
  L.slots_per_tile = mx > 0 ? mx : 1;
  L.count_bytes = (static_cast<int64_t>(rem) * 2 * 4 + 255) / 256 * 256;
  L.bytes = L.count_bytes + static_cast<int64_t>(rem) * L.slots_per_tile * 256 * 256 * 4;
  return L;
}

}  // namespace

int64_t dual_gemm_workspace_size(int64_t m, int64_t n, int64_t k, int64_t k_o) {
  return sk_layout(m, n, k, k_o, QARVD_BF16, false).bytes;
}

int dual_gemm_launch(const int8_t* xq, int64_t ldq, const int8_t* wq, int64_t ldw, int64_t m,
                     int64_t n, int64_t k, int64_t k_outlier, const float* scale_x,
                     const float* scale_wo, const float* scale_wn, const float* bias,
                     int epilogue, int out_dtype, void* y, int64_t ldy, int32_t* acc_o,
                     int32_t* acc_n, cudaStream_t stream, const double* sx64 = nullptr,
                     const double* so64 = nullptr, const double* sn64 = nullptr,
                     uint32_t* row_absmax = nullptr, uint32_t* row_pmax = nullptr,
                     void* sk_workspace = nullptr, int64_t sk_workspace_bytes = 0, int f64_slices = 0) {
  GemmParams p{};
  p.f64_slices = f64_slices;
  p.row_absmax = row_absmax;
  p.row_pmax = row_pmax;
  p.sx64 = sx64;
  p.so64 = so64;
  p.sn64 = sn64;
  p.m = m;
  p.n = n;
  p.k = k;
  p.k_o = k_outlier;
  p.scale_x = scale_x;
  p.scale_wo = scale_wo;
  p.scale_wn = scale_wn;
  p.bias = bias;
  p.y = y;
  p.ldy = ldy;
  p.acc_o_dbg = acc_o;
  p.acc_n_dbg = acc_n;
  p.debug = getenv("QARVD_GEMM_DEBUG") ? atoi(getenv("QARVD_GEMM_DEBUG")) : 0;
  p.trace = getenv("QARVD_GEMM_TRACE") ? 1 + (getenv("QARVD_GEMM_TRACE_CTA") ? atoi(getenv("QARVD_GEMM_TRACE_CTA")) : 0) : 0;
  if (p.debug & 128) p.cta_times = debug_cta_times();
  p.epilogue = epilogue;
  p.out_dtype = out_dtype;
  TileCfg c = choose_cfg(m, n, k);
  if (out_dtype == QARVD_F64 && f64_slices > 1 && !getenv("QARVD_GEMM_BN")) {
    // K7's slice products: at 256 columns one accumulator stage fills TMEM, so the MMA of the
    // next tile waits for the whole f64 epilogue; 128-column tiles double-buffer the
    // accumulators and the epilogue overlaps the next tile's MMA (QARVD_F64_BN=256 for A/B)
    const char* env = getenv("QARVD_F64_BN");
    c.bn = env && atoi(env) == 256 ? 256 : 128;
    // short K (the forward product, K = the layer width): 128-byte stages keep twice as many
    // loads in flight (measured: QARVD_GEMM_KS=1 on both products cut the loss passes by 16%
    // but slowed the long-K gradient product)
    if (!getenv("QARVD_GEMM_KS") && k <= 4096) c.ks = 1;
  }
  if (sk_workspace) {
    const SkLayout L = sk_layout(m, n, k, k_outlier, out_dtype, acc_o || acc_n || row_absmax || row_pmax);
    if (L.bytes > 0 && sk_workspace_bytes >= L.bytes) {
      p.sk_tiles = L.sk_tiles;
      p.sk_slots_per_tile = L.slots_per_tile;
      p.sk_count = static_cast<uint32_t*>(sk_workspace);
      p.sk_slots = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(sk_workspace) + L.count_bytes);
    }
  }
  if (c.cg == 2) {
    if (c.bn == 256) return c.ks == 2 ? launch_gemm<256, 2, 2>(xq, ldq, wq, ldw, p, stream)
                                      : launch_gemm<256, 2, 1>(xq, ldq, wq, ldw, p, stream);
    if (c.bn == 192) return launch_gemm<192, 2, 1>(xq, ldq, wq, ldw, p, stream);
    return c.ks == 2 ? launch_gemm<128, 2, 2>(xq, ldq, wq, ldw, p, stream)
                     : launch_gemm<128, 2, 1>(xq, ldq, wq, ldw, p, stream);
  }
  if (c.bn == 256) return c.ks == 2 ? launch_gemm<256, 1, 2>(xq, ldq, wq, ldw, p, stream)
                                    : launch_gemm<256, 1, 1>(xq, ldq, wq, ldw, p, stream);
  if (c.bn == 192) return c.ks == 2 ? launch_gemm<192, 1, 2>(xq, ldq, wq, ldw, p, stream)
                                    : launch_gemm<192, 1, 1>(xq, ldq, wq, ldw, p, stream);
  return c.ks == 2 ? launch_gemm<128, 1, 2>(xq, ldq, wq, ldw, p, stream)
                   : launch_gemm<128, 1, 1>(xq, ldq, wq, ldw, p, stream);
}

}  // namespace qarvd_b200

using namespace qarvd_b200;

namespace {
int dual_gemm_checked(const int8_t* xq, int64_t ldq, const int8_t* wq, int64_t ldw, int64_t m,
                      int64_t n, int64_t k, int64_t k_outlier, const float* scale_x,
                      const float* scale_w_outlier, const float* scale_w_normal, const float* bias,
                      int epilogue, int out_dtype, void* y, int64_t ldy, int32_t* acc_outlier,
                      int32_t* acc_normal, uint32_t* row_absmax, void* stream,
                      uint32_t* row_pmax = nullptr) {
  clear_error();
  if (m <= 0 || n <= 0 || k <= 0)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: empty shape");
  if (k % 32 != 0 || k_outlier % 32 != 0 || k_outlier < 0 || k_outlier >= k)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT,
               "kernel_b: k and k_outlier must be multiples of 32 with 0 <= k_outlier < k");
  if (k > 132104)
    QARVD_FAIL(QARVD_ERR_LOGIC,
               "kernel_b: reduction dimension too large for exact int32 accumulation");
  if (ldq < k || ldw < k || ldq % 16 || ldw % 16 || ldy < n)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: leading dimensions must be >= k (n for y) and multiples of 16");
  if ((reinterpret_cast<uintptr_t>(xq) & 15) || (reinterpret_cast<uintptr_t>(wq) & 15))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: operand pointers must be 16-byte aligned");
  if (!xq || !wq || !scale_x || !scale_w_normal || !y || (k_outlier > 0 && !scale_w_outlier))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: null pointer argument");
  if (out_dtype != QARVD_BF16 && out_dtype != QARVD_F32)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: output dtype must be bf16 or f32");
  if ((row_absmax || row_pmax) && out_dtype != QARVD_BF16)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: row |y| max is defined for bf16 outputs");
  if (int st = require_device()) return st;
  return dual_gemm_launch(xq, ldq, wq, ldw, m, n, k, k_outlier, scale_x, scale_w_outlier,
                          scale_w_normal, bias, epilogue, out_dtype, y, ldy, acc_outlier,
                          acc_normal, as_stream(stream), nullptr, nullptr, nullptr, row_absmax,
                          row_pmax);
}
}  // namespace

extern "C" int qarvd_dual_gemm(const int8_t* xq, int64_t ldq, const int8_t* wq, int64_t ldw,
                               int64_t m, int64_t n, int64_t k, int64_t k_outlier,
                               const float* scale_x, const float* scale_w_outlier,
                               const float* scale_w_normal, const float* bias, int epilogue,
                               int out_dtype, void* y, int64_t ldy, int32_t* acc_outlier,
                               int32_t* acc_normal, void* stream) {
  return dual_gemm_checked(xq, ldq, wq, ldw, m, n, k, k_outlier, scale_x, scale_w_outlier,
                           scale_w_normal, bias, epilogue, out_dtype, y, ldy, acc_outlier,
                           acc_normal, nullptr, stream);
}

extern "C" int qarvd_dual_gemm_rowmax(const int8_t* xq, int64_t ldq, const int8_t* wq, int64_t ldw,
                                      int64_t m, int64_t n, int64_t k, int64_t k_outlier,
                                      const float* scale_x, const float* scale_w_outlier,
                                      const float* scale_w_normal, const float* bias, int epilogue,
                                      uint16_t* y, int64_t ldy, uint32_t* row_absmax, void* stream) {
  if (!row_absmax) {
    clear_error();
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: null row |y| max buffer");
  }
  return dual_gemm_checked(xq, ldq, wq, ldw, m, n, k, k_outlier, scale_x, scale_w_outlier,
                           scale_w_normal, bias, epilogue, QARVD_BF16, y, ldy, nullptr, nullptr,
                           row_absmax, stream);
}

extern "C" int qarvd_dual_gemm_f64(const int8_t* xq, int64_t ldq, const int8_t* wq, int64_t ldw,
                                   int64_t m, int64_t n, int64_t k, int64_t k_outlier,
                                   const double* scale_x, const double* scale_w_outlier,
                                   const double* scale_w_normal, double* y, int64_t ldy,
                                   void* stream) {
  clear_error();
  if (m <= 0 || n <= 0 || k <= 0) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: empty shape");
  if (k % 32 != 0 || k_outlier % 32 != 0 || k_outlier < 0 || k_outlier >= k)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT,
               "kernel_b: k and k_outlier must be multiples of 32 with 0 <= k_outlier < k");
  if (k > 132104)
    QARVD_FAIL(QARVD_ERR_LOGIC, "kernel_b: reduction dimension too large for exact int32 accumulation");
  if (ldq < k || ldw < k || ldq % 16 || ldw % 16 || ldy < n)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: invalid leading dimension");
  if (!xq || !wq || !scale_x || !scale_w_normal || !y || (k_outlier > 0 && !scale_w_outlier))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: null pointer argument");
  if ((reinterpret_cast<uintptr_t>(xq) & 15) || (reinterpret_cast<uintptr_t>(wq) & 15))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: operand pointers must be 16-byte aligned");
  if (int st = require_device()) return st;
  static const float kDummy = 0.f;  // f32 scales unused on the f64 path
  (void)kDummy;
  return dual_gemm_launch(xq, ldq, wq, ldw, m, n, k, k_outlier, nullptr, nullptr, nullptr, nullptr,
                          QARVD_EPI_NONE, QARVD_F64, y, ldy, nullptr, nullptr, as_stream(stream),
                          scale_x, scale_w_outlier, scale_w_normal);
}

extern "C" int qarvd_dual_gemm_f64_slices(const int8_t* xq, int64_t ldq, const int8_t* wq, int64_t ldw,
                                          int64_t m, int64_t n, int64_t k, int64_t k_outlier,
                                          const double* scale_x, const double* scale_w_outlier,
                                          const double* scale_w_normal, int slices, double* y, int64_t ldy,
                                          void* stream) {
  clear_error();
  if (m <= 0 || n <= 0 || k <= 0) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: empty shape");
  if (!(slices == 2 || slices == 4 || slices == 8 || slices == 16) || n % 16 != 0)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "qarvd_dual_gemm_f64_slices: slices in {2,4,8,16}, n % 16 == 0");
  if (k % 32 != 0 || k_outlier % 32 != 0 || k_outlier < 0 || k_outlier >= k)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT,
               "kernel_b: k and k_outlier must be multiples of 32 with 0 <= k_outlier < k");
  if (k > 132104)
    QARVD_FAIL(QARVD_ERR_LOGIC, "kernel_b: reduction dimension too large for exact int32 accumulation");
  if (ldq < k || ldw < k || ldq % 16 || ldw % 16 || ldy < n / slices)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: invalid leading dimension");
  if (!xq || !wq || !scale_x || !scale_w_normal || !y || (k_outlier > 0 && !scale_w_outlier))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: null pointer argument");
  if ((reinterpret_cast<uintptr_t>(xq) & 15) || (reinterpret_cast<uintptr_t>(wq) & 15))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: operand pointers must be 16-byte aligned");
  if (int st = require_device()) return st;
  return dual_gemm_launch(xq, ldq, wq, ldw, m, n, k, k_outlier, nullptr, nullptr, nullptr, nullptr,
                          QARVD_EPI_NONE, QARVD_F64, y, ldy, nullptr, nullptr, as_stream(stream),
                          scale_x, scale_w_outlier, scale_w_normal, nullptr, nullptr, nullptr, 0, slices);
}

extern "C" int64_t qarvd_dual_gemm_workspace_size(int64_t m, int64_t n, int64_t k, int64_t k_outlier) {
  if (m <= 0 || n <= 0 || k <= 0) return 0;
  return qarvd_b200::dual_gemm_workspace_size(m, n, k, k_outlier);
}

extern "C" int qarvd_dual_gemm_ws(const int8_t* xq, int64_t ldq, const int8_t* wq, int64_t ldw,
                                  int64_t m, int64_t n, int64_t k, int64_t k_outlier,
                                  const float* scale_x, const float* scale_w_outlier,
                                  const float* scale_w_normal, const float* bias, int epilogue,
                                  uint16_t* y, int64_t ldy, void* workspace, int64_t workspace_bytes,
                                  void* stream) {
  if (workspace && (reinterpret_cast<uintptr_t>(workspace) & 255)) {
    clear_error();
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: workspace must be 256-byte aligned");
  }
  clear_error();
  if (m <= 0 || n <= 0 || k <= 0) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: empty shape");
  if (k % 32 != 0 || k_outlier % 32 != 0 || k_outlier < 0 || k_outlier >= k)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT,
               "kernel_b: k and k_outlier must be multiples of 32 with 0 <= k_outlier < k");
  if (k > 132104)
    QARVD_FAIL(QARVD_ERR_LOGIC, "kernel_b: reduction dimension too large for exact int32 accumulation");
  if (ldq < k || ldw < k || ldq % 16 || ldw % 16 || ldy < n)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: leading dimensions must be >= k (n for y) and multiples of 16");
  if ((reinterpret_cast<uintptr_t>(xq) & 15) || (reinterpret_cast<uintptr_t>(wq) & 15))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: operand pointers must be 16-byte aligned");
  if (!xq || !wq || !scale_x || !scale_w_normal || !y || (k_outlier > 0 && !scale_w_outlier))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: null pointer argument");
  if (int st = require_device()) return st;
  return dual_gemm_launch(xq, ldq, wq, ldw, m, n, k, k_outlier, scale_x, scale_w_outlier, scale_w_normal,
                          bias, epilogue, QARVD_BF16, y, ldy, nullptr, nullptr, as_stream(stream), nullptr,
                          nullptr, nullptr, nullptr, nullptr, workspace, workspace_bytes);
}

extern "C" int64_t qarvd_dual_gemm_pmax_count(int64_t m, int64_t n, int64_t k) {
  if (n <= 0) return 0;
  const TileCfg c = choose_cfg(m, n, k);
  return (n + c.bn - 1) / c.bn * (kEpiWarps / 4);
}

extern "C" int qarvd_dual_gemm_pmax(const int8_t* xq, int64_t ldq, const int8_t* wq, int64_t ldw,
                                    int64_t m, int64_t n, int64_t k, int64_t k_outlier,
                                    const float* scale_x, const float* scale_w_outlier,
                                    const float* scale_w_normal, const float* bias, int epilogue,
                                    uint16_t* y, int64_t ldy, uint32_t* row_pmax, int64_t pm_count,
                                    void* stream) {
  if (!row_pmax || pm_count != qarvd_dual_gemm_pmax_count(m, n, k)) {
    clear_error();
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT,
               "kernel_b: row partial-max buffer missing or pm_count != qarvd_dual_gemm_pmax_count");
  }
  return dual_gemm_checked(xq, ldq, wq, ldw, m, n, k, k_outlier, scale_x, scale_w_outlier,
                           scale_w_normal, bias, epilogue, QARVD_BF16, y, ldy, nullptr, nullptr,
                           nullptr, stream, row_pmax);
}

// ---- K2 with the consumer's per-token K1 fused into the epilogue -------------------------
namespace qarvd_b200 {
namespace {
__global__ void qz_init_err_kernel(unsigned long long* err) { *err = 0x7fffffffffffffffull; }
int64_t qz_blocks(int64_t m) { return (m + 255) / 256; }  // row blocks of the 256 x 256 pair tiles
}  // namespace
}  // namespace qarvd_b200

extern "C" int64_t qarvd_dual_gemm_quant_workspace_size(int64_t m) {
  if (m <= 0) return 0;
  return (static_cast<int64_t>(m + qz_blocks(m) + 2) * 8 + 255) / 256 * 256;
}

extern "C" int qarvd_dual_gemm_quant(const int8_t* xq, int64_t ldq, const int8_t* wq, int64_t ldw,
                                     int64_t m, int64_t n, int64_t k, int64_t k_outlier,
                                     const float* scale_x, const float* scale_w_outlier,
                                     const float* scale_w_normal, const float* bias, int epilogue, int granularity,
                                     double static_scale, int bits, int8_t* q, int64_t ldq_out, float* scale_f32,
                                     double* scale_f64,
                                     int64_t* err_index, void* workspace, int64_t workspace_bytes,
                                     void* stream) {
  clear_error();
  if (m <= 0 || n <= 0 || k <= 0) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: empty shape");
  if (k % 32 != 0 || k_outlier % 32 != 0 || k_outlier < 0 || k_outlier >= k)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT,
               "kernel_b: k and k_outlier must be multiples of 32 with 0 <= k_outlier < k");
  if (k > 132104)
    QARVD_FAIL(QARVD_ERR_LOGIC, "kernel_b: reduction dimension too large for exact int32 accumulation");
  if (ldq < k || ldw < k || ldq % 16 || ldw % 16)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: leading dimensions must be >= k and multiples of 16");
  if ((reinterpret_cast<uintptr_t>(xq) & 15) || (reinterpret_cast<uintptr_t>(wq) & 15))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: operand pointers must be 16-byte aligned");
  if (!xq || !wq || !scale_x || !scale_w_normal || (k_outlier > 0 && !scale_w_outlier) || !q || !scale_f32)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: null pointer argument");
  if (bits < 2 || bits > 8) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "quantize: bits must be in [2, 8]");
  if (granularity != QARVD_ACT_PER_TOKEN && granularity != QARVD_ACT_PER_TENSOR)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "quantize: unknown activation granularity");
  if (granularity == QARVD_ACT_PER_TENSOR && !(std::isfinite(static_scale) && static_scale > 0.0))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "QuantParams: scale must be finite and > 0");
  if (n % 256 != 0 || ldq_out < n || ldq_out % 16 || (reinterpret_cast<uintptr_t>(q) & 15))
    QARVD_FAIL(QARVD_ERR_UNSUPPORTED,
               "qarvd_dual_gemm_quant: n must be a multiple of 256 and the codes 16-byte aligned rows (ldq_out >= n)");
  if (!workspace || workspace_bytes < qarvd_dual_gemm_quant_workspace_size(m) ||
      (reinterpret_cast<uintptr_t>(workspace) & 15))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT,
               "qarvd_dual_gemm_quant: workspace missing, misaligned or smaller than qarvd_dual_gemm_quant_workspace_size");
  if (int st = require_device()) return st;
  cudaStream_t s = as_stream(stream);
  if (err_index) {
    qz_init_err_kernel<<<1, 1, 0, s>>>(reinterpret_cast<unsigned long long*>(err_index));
    count_launch();
    QARVD_CUDA_TRY(cudaGetLastError());
  }
  GemmParams p{};
  p.m = m;
  p.n = n;
  p.k = k;
  p.k_o = k_outlier;
  p.scale_x = scale_x;
  p.scale_wo = scale_w_outlier;
  p.scale_wn = scale_w_normal;
  p.bias = bias;
  p.epilogue = epilogue;
  p.out_dtype = QARVD_BF16;
  p.qz = 1;
  p.qz_qmax = (1 << (bits - 1)) - 1;
  p.qz_static = granularity == QARVD_ACT_PER_TENSOR ? 1 : 0;
  p.row_major = p.qz_static ? 0 : 1;
  p.qz_s_static = static_scale;
  p.qz_rowmax = static_cast<unsigned long long*>(workspace);
  p.qz_count = static_cast<unsigned long long*>(workspace) + m;
  p.qz_epoch = p.qz_count + qz_blocks(m);
  p.qz_done = reinterpret_cast<unsigned int*>(p.qz_epoch + 1);
  p.qz_q = q;
  p.qz_ldq = ldq_out;
  p.qz_sx = scale_f32;
  p.qz_s64 = scale_f64;
  p.qz_err = reinterpret_cast<unsigned long long*>(err_index);
  p.trace = getenv("QARVD_GEMM_TRACE") ? 1 + (getenv("QARVD_GEMM_TRACE_CTA") ? atoi(getenv("QARVD_GEMM_TRACE_CTA")) : 0) : 0;
  p.debug = getenv("QARVD_GEMM_DEBUG") ? atoi(getenv("QARVD_GEMM_DEBUG")) : 0;
  // the fused epilogue is built for the deployed tile (256 x 256 pair tiles, one TMEM stage,
  // the register-held accumulator path)
  return launch_gemm<256, 2, 2>(xq, ldq, wq, ldw, p, s);
}

// diagnostic (not part of the ABI header): the per-CTA start / end globaltimer stamps of the last
// K2 launch made with QARVD_GEMM_DEBUG=128, n CTAs -> host[2n]
extern "C" int qarvd_debug_cta_times(unsigned long long* host, int n) {
  unsigned long long* d = qarvd_b200::debug_cta_times();
  if (!d || n <= 0 || n > 1024) return QARVD_ERR_INVALID_ARGUMENT;
  return cudaMemcpy(host, d, 2 * n * sizeof(unsigned long long), cudaMemcpyDeviceToHost) == cudaSuccess ? QARVD_OK
                                                                                                      : QARVD_ERR_CUDA;
}
