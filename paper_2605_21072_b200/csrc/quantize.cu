// K1 (activation quantization fused with the dual-scale permutation) and
// K5 (dual-scale weight preparation): both are one HBM-bound pass of
// "row absmax -> scale -> round-half-even codes in gathered order".
//
// Reference semantics:
//   K1 = quantize(permute_activations(x, plan), p)   engine.cpp:32-44, quant.cpp:113-138
//        with p per-token = init_scale_minmax(x, b, per_channel, 0) (quant.cpp:170-182)
//        or per-tensor static p (engine.cpp:57).
//   K5 = row_scales_over_columns over the outlier and normal column groups
//        (dual_scale.cpp:13-24, :58-90) + nearest codes as in fake_quant_dual
//        (dual_scale.cpp:92-114), stored pre-permuted (calibrate.cpp:474-480).
//
// Layout: bf16 rows are staged once into shared memory with 16-byte coalesced
// loads (one warp per row), the row absmax is a warp-shuffle reduction, and
// each lane then emits 16 consecutive output codes (one 16-byte store) by
// gathering through `gather` from the shared-memory copy.
#include <cuda_bf16.h>

#include <climits>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "ptx.cuh"

namespace qarvd_b200 {
namespace {

enum Mode { kActPerToken = 0, kActStatic = 1, kWeightDual = 2 };

constexpr int kWarpsPerCta = 4;
constexpr int kMaxSmemK = 16384;  // bf16 elements staged per warp (32 KB)

__device__ __forceinline__ void record_error(unsigned long long* err, int64_t flat) {
  if (err) atomicMin(err, static_cast<unsigned long long>(flat));
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Scale of one group from its absmax a (exact bf16 value as float):
// s64 = a / qmax in f64 (quant.cpp:168/181), DBL_MIN for a == 0 (quant.cpp:164);
// r32 = qmax / a in fp32 for the fast path; exact = r32 unusable (not normal).
struct GroupScale {
  double s64;
  float s32;
  float r32;
  bool exact;
};
__device__ __forceinline__ GroupScale scale_from_absmax(float a, int qmax) {
  GroupScale g;
  if (a > 0.f) {
    g.s64 = __ddiv_rn(static_cast<double>(a), static_cast<double>(qmax));
    g.s32 = __double2float_rn(g.s64);
    g.r32 = __fdiv_rn(static_cast<float>(qmax), a);
    g.exact = !(g.r32 <= FLT_MAX && g.r32 >= FLT_MIN);
  } else {
    g.s64 = DBL_MIN;
    g.s32 = 0.f;  // all codes are 0; the epilogue product is 0 either way
    g.r32 = 0.f;
    g.exact = false;
  }
  return g;
}
__device__ __forceinline__ GroupScale scale_static(double s64) {
  GroupScale g;
  g.s64 = s64;
  g.s32 = __double2float_rn(s64);
  const double r = 1.0 / s64;
  g.r32 = __double2float_rn(r);
  g.exact = !(r <= static_cast<double>(FLT_MAX) && r >= static_cast<double>(FLT_MIN));
  return g;
}

__device__ __forceinline__ int code_of(float v, const GroupScale& g, int qmax) {
  if (g.exact) return quant_code_exact(static_cast<double>(v), g.s64, qmax);
  return quant_code_fast(v, g.r32, g.s64, qmax);
}

// ---------------------------------------------------------------------------
// bf16 fast kernel: one warp per row, row staged in shared memory.
template <int MODE>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
    quant_rows_bf16_kernel(const uint16_t* __restrict__ x, int64_t m, int64_t k, int64_t ldx,
                           const int32_t* __restrict__ gather, int64_t k_out, int64_t k_o,
                           double static_scale, int qmax, int8_t* __restrict__ q, int64_t ldq,
                           float* __restrict__ s32_o, double* __restrict__ s64_o,
                           float* __restrict__ s32_n, double* __restrict__ s64_n,
                           unsigned long long* err) {
  extern __shared__ uint4 smem_rows[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t kstride = (k + 7) & ~int64_t(7);
  uint16_t* row_s = reinterpret_cast<uint16_t*>(smem_rows) + warp * kstride;
  const bool vec_in = ((ldx & 7) == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  const bool vec_out = ((ldq & 15) == 0) && ((reinterpret_cast<uintptr_t>(q) & 15) == 0) &&
                       (gather == nullptr || (reinterpret_cast<uintptr_t>(gather) & 15) == 0);

  for (int64_t row = static_cast<int64_t>(blockIdx.x) * kWarpsPerCta + warp; row < m;
       row += static_cast<int64_t>(gridDim.x) * kWarpsPerCta) {
    const uint16_t* xr = x + row * ldx;
    float amax = 0.f;
    bool bad = false;
    // ---- stage the row (16-byte coalesced loads) and take |x| max ----
    if (vec_in) {
      const int64_t nvec = k >> 3;
      for (int64_t v = lane; v < nvec; v += 32) {
        const uint4 d = __ldg(reinterpret_cast<const uint4*>(xr) + v);
        reinterpret_cast<uint4*>(row_s)[v] = d;
        const uint32_t w[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const uint16_t lo = static_cast<uint16_t>(w[h] & 0xffffu);
          const uint16_t hi = static_cast<uint16_t>(w[h] >> 16);
          bad |= !InType<uint16_t>::finite(lo) || !InType<uint16_t>::finite(hi);
          amax = fmaxf(amax, fabsf(bf16_bits_to_float(lo)));
          amax = fmaxf(amax, fabsf(bf16_bits_to_float(hi)));
        }
      }
      for (int64_t c = (nvec << 3) + lane; c < k; c += 32) {
        const uint16_t h = xr[c];
        row_s[c] = h;
        bad |= !InType<uint16_t>::finite(h);
        amax = fmaxf(amax, fabsf(bf16_bits_to_float(h)));
      }
    } else {
      for (int64_t c = lane; c < k; c += 32) {
        const uint16_t h = xr[c];
        row_s[c] = h;
        bad |= !InType<uint16_t>::finite(h);
        amax = fmaxf(amax, fabsf(bf16_bits_to_float(h)));
      }
    }
    __syncwarp();

    // ---- scales ----
    GroupScale g_o, g_n;
    if (MODE == kActPerToken) {
      g_n = scale_from_absmax(warp_max(amax), qmax);
      g_o = g_n;
      if (lane == 0) {
        if (s32_n) s32_n[row] = g_n.s32;
        if (s64_n) s64_n[row] = g_n.s64;
      }
    } else if (MODE == kActStatic) {
      g_n = scale_static(static_scale);
      g_o = g_n;
      if (lane == 0) {
        if (s32_n) s32_n[row] = g_n.s32;
        if (s64_n) s64_n[row] = g_n.s64;
      }
    } else {
      // group absmax over the gathered columns: [0, k_o) outlier, [k_o, k_out) normal
      float ao = 0.f, an = 0.f;
      for (int64_t c = lane; c < k_out; c += 32) {
        const int32_t src = gather ? __ldg(gather + c) : static_cast<int32_t>(c);
        if (src < 0) continue;
        const float v = fabsf(bf16_bits_to_float(row_s[src]));
        if (c < k_o) ao = fmaxf(ao, v);
        else an = fmaxf(an, v);
      }
      g_n = scale_from_absmax(warp_max(an), qmax);
      g_o = k_o > 0 ? scale_from_absmax(warp_max(ao), qmax) : g_n;
      if (lane == 0) {
        if (s32_n) s32_n[row] = g_n.s32;
        if (s64_n) s64_n[row] = g_n.s64;
        if (s32_o) s32_o[row] = g_o.s32;
        if (s64_o) s64_o[row] = g_o.s64;
      }
    }
    bad = __any_sync(0xffffffffu, bad);

    // ---- codes, 16 per lane per iteration ----
    int8_t* qr = q + row * ldq;
    for (int64_t c0 = static_cast<int64_t>(lane) * 16; c0 < k_out; c0 += 32 * 16) {
      int32_t src[16];
      if (gather && vec_out && c0 + 16 <= k_out) {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int4 gi = __ldg(reinterpret_cast<const int4*>(gather + c0) + v);
          src[4 * v] = gi.x;
          src[4 * v + 1] = gi.y;
          src[4 * v + 2] = gi.z;
          src[4 * v + 3] = gi.w;
        }
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int64_t c = c0 + e;
          src[e] = c < k_out ? (gather ? __ldg(gather + c) : static_cast<int32_t>(c)) : -1;
        }
      }
      uint32_t packed[4] = {0, 0, 0, 0};
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        int code = 0;
        if (src[e] >= 0) {
          const uint16_t h = row_s[src[e]];
          if (bad && !InType<uint16_t>::finite(h)) record_error(err, row * k_out + c0 + e);
          const bool outl = (MODE == kWeightDual) && (c0 + e < k_o);
          code = code_of(bf16_bits_to_float(h), outl ? g_o : g_n, qmax);
        }
        packed[e >> 2] |= (static_cast<uint32_t>(code) & 0xffu) << (8 * (e & 3));
      }
      if (vec_out && c0 + 16 <= k_out) {
        *reinterpret_cast<uint4*>(qr + c0) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
      } else {
        for (int e = 0; e < 16 && c0 + e < k_out; ++e)
          qr[c0 + e] = static_cast<int8_t>((packed[e >> 2] >> (8 * (e & 3))) & 0xffu);
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// K1 fast path (bf16 activations, per-token or static scale).
//
// One team of T threads owns one row.  It loads the row with coalesced 16-byte
// loads straight into registers (at most kK1Vec chunks of 8 values per thread),
// reduces |x|max across the team and emits the codes:
//   * no permutation (the producer already wrote the row in plan order, see
//     pipeline.QuantizedChain): codes come from the registers, 8 per chunk,
//     written back as one 8-byte store;
//   * with a permutation: the row is also copied to a per-team shared-memory
//     buffer (plus 8 zero sentinels that pad slots read) and every thread
//     gathers 16 codes per step through the plan's index table.
// Teams never wait on one another, so each SM keeps many rows in flight.
//
// Rounding: t = v * (qmax/absmax) in fp32 (packed f32x2 FMAs), q = t rounded by
// the 1.5*2^23 magic add.  |t - v/s| < 3.1e-5 for |t| <= 254, so q equals the
// reference's f64 round_half_even(v/s) (quant.cpp:123-131) unless t lies within
// 1e-4 of a half-integer; the exact residual d = v*r - q (one fma) flags those
// (~0.04% of chunks), which are recomputed with the f64 division.
constexpr int kK1Vec = 8;
// Residual above which the f64 path decides.  Per-token: t = v*r32 with the product exact
// (fma) and r32 = fl(fl(1/amax) * qmax) within 2^-23 of qmax/amax, so |t - v/s64| <= |t| *
// 2^-23 <= 1.6e-5 for |t| <= 127: guard 3e-5.  Static: the product is rounded as well and
// clamped, |t - v/s64| <= |t| * 2^-23 <= 3.1e-5 for |t| <= 254: guard 1e-4.
template <bool kStatic>
__device__ __forceinline__ constexpr float tie_guard() { return kStatic ? 0.4999f : 0.49997f; }
constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: an fp32 add rounds to an integer (RNE)

__device__ __noinline__ int act_code_exact(float v, double s64, int qmax) {
  return quant_code_exact(static_cast<double>(v), s64, qmax);
}

__device__ __forceinline__ uint32_t pack4(uint32_t b0, uint32_t b1, uint32_t b2, uint32_t b3) {
  return __byte_perm(__byte_perm(b0, b1, 0x0040), __byte_perm(b2, b3, 0x0040), 0x5410);
}
__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void upk2(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

struct ActScale {
  float r;      // fp32 reciprocal qmax/absmax (or 1/s for a static scale)
  float fq;     // qmax as float (static clamp)
  bool exact;   // r is unusable: every code takes the f64 division
  double s64;   // f64 scale, valid where exact/rare paths need it
};

// Fast codes of two bf16 values (packed in w); code words carry the code in their
// low byte.  |residual| is folded into dmax (> 0.4999 => the chunk is redone exactly).
template <bool kStatic>
__device__ __forceinline__ void act_codes2(float lo, float hi, const ActScale& sc, uint32_t& c0,
                                           uint32_t& c1, float& dmax) {
  if (kStatic) {
    const float t0 = fminf(fmaxf(__fmul_rn(lo, sc.r), -sc.fq), sc.fq);
    const float t1 = fminf(fmaxf(__fmul_rn(hi, sc.r), -sc.fq), sc.fq);
    const float y0 = __fadd_rn(t0, kMagic), y1 = __fadd_rn(t1, kMagic);
    dmax = fmaxf(dmax, fmaxf(fabsf(__fsub_rn(t0, __fsub_rn(y0, kMagic))),
                             fabsf(__fsub_rn(t1, __fsub_rn(y1, kMagic)))));
    c0 = __float_as_uint(y0);
    c1 = __float_as_uint(y1);
  } else {
    const uint64_t v2 = pk2(lo, hi), r2 = pk2(sc.r, sc.r), m2 = pk2(kMagic, kMagic);
    const uint64_t y2 = ffma2(v2, r2, m2);                // magic + rint(v*r)
    const uint64_t n2 = ffma2(y2, pk2(-1.f, -1.f), m2);  // -rint(v*r), exact
    const uint64_t d2 = ffma2(v2, r2, n2);                // v*r - rint(v*r), one rounding
    float d0, d1, y0, y1;
    upk2(d2, d0, d1);
    upk2(y2, y0, y1);
    dmax = fmaxf(dmax, fmaxf(fabsf(d0), fabsf(d1)));
    c0 = __float_as_uint(y0);
    c1 = __float_as_uint(y1);
  }
}

// Slow code of one value: non-finite inputs are reported (the reference throws,
// quant.cpp:113-121) and give 0; everything else takes the exact f64 division.
__device__ __forceinline__ uint32_t act_code_slow(uint16_t h, double s64, int qmax,
                                                  unsigned long long* err, int64_t flat) {
  if ((h & 0x7f80u) == 0x7f80u) {
    record_error(err, flat);
    return 0u;
  }
  return static_cast<uint32_t>(act_code_exact(bf16_bits_to_float(h), s64, qmax));
}

// Patch the codes of one flagged chunk (N values, bf16 bits hv): values within the tie guard
// take the exact f64 division (`rescan` / kExact are kept for the callers' interface).
template <bool kStatic, int N, bool kExact>
__device__ __forceinline__ void act_fix_chunk(const uint16_t* hv, uint32_t* c, const ActScale& sc,
                                              double s64, int qmax, bool& rescan) {
#pragma unroll
  for (int e = 0; e < N; ++e) {
    const float v = __uint_as_float(static_cast<uint32_t>(hv[e]) << 16);
    bool divide = false;
    // a value within the guard takes the reference's own arithmetic, rint(v / s) in f64 (round 2:
    // deciding it by the f64 boundary analysis of act_code_tie first was slower -- K1 at
    // 4680 x 1536 18.4 -> 14.3 us with the division, its one-row-per-warp critical path shorter)
    if (kStatic) {
      const float t = fminf(fmaxf(__fmul_rn(v, sc.r), -sc.fq), sc.fq);
      divide = fabsf(__fsub_rn(t, rintf(t))) > tie_guard<true>();
    } else {
      const float t = __fmul_rn(v, sc.r);
      const float d = __fmaf_rn(v, sc.r, -rintf(t));
      divide = fabsf(d) > tie_guard<false>();
    }
    if (divide) c[e] = static_cast<uint32_t>(act_code_exact(v, s64, qmax)) & 0xffu;
    (void)rescan;
  }
}

// Persistent teams: team g of the grid quantizes rows g, g + G, g + 2G, ... (G teams in
// total).  Each team keeps S row slots in shared memory filled by 1-D TMA bulk copies (one
// instruction per row; per-thread loads through L1 cap the bytes in flight per SM and left
// HBM at ~2 TB/s), so rows j+1 .. j+S-1 stream in while row j is rounded.  Teams are either
// four independent warps per CTA (rows of <= 2048 values; lane 0 refills its own slots) or
// one CTA of W consumer warps -- the count that splits the row's 16-byte chunks evenly --
// plus a producer warp that refills slots as the consumers release them (full/empty
// mbarriers).  A one-CTA team combines its per-warp |x| maxima through mbarriers one row
// ahead: each warp publishes row j+1's partial maximum before rounding row j, so no
// CTA-wide barrier sits on the row loop (4 partial buffers: a warp runs at most three rows
// ahead of the slowest reader).  The permutation, when present, is staged once per CTA as an
// int16 table (pad -> k, the zero sentinel column of every row slot).
constexpr int kK1Parts = 4;

// Out-of-line repair of the chunks a thread flagged in its streaming loop (bit i = its
// i-th chunk / step): recompute the fast codes, decide the values within the tie guard
// exactly (act_fix_chunk), then values only the f64 division decides, and store again.
// Kept out of the loop so the hot path stays a short straight-line body.
template <bool kStatic, bool kGather>
__device__ __noinline__ void act_fix_flagged(const uint16_t* srow, const int16_t* gidx,
                                             int8_t* qr, int tt, int T, uint32_t flagged,
                                             ActScale sc, double s64, int qmax) {
  constexpr int N = kGather ? 4 : 8;
  while (flagged) {
    const int i = __ffs(flagged) - 1;
    flagged &= flagged - 1;
    const int c0 = (tt + i * T) * N;
    uint16_t hv[N];
    uint32_t c[N];
    float dmax = 0.f;
#pragma unroll
    for (int e = 0; e < N; ++e) hv[e] = srow[kGather ? gidx[c0 + e] : c0 + e];
#pragma unroll
    for (int e = 0; e < N; e += 2)
      act_codes2<kStatic>(__uint_as_float(static_cast<uint32_t>(hv[e]) << 16),
                          __uint_as_float(static_cast<uint32_t>(hv[e + 1]) << 16), sc, c[e],
                          c[e + 1], dmax);
    bool rescan = false;
    act_fix_chunk<kStatic, N, false>(hv, c, sc, s64, qmax, rescan);
    if (rescan) act_fix_chunk<kStatic, N, true>(hv, c, sc, s64, qmax, rescan);
#pragma unroll
    for (int e = 0; e < N; ++e) qr[c0 + e] = static_cast<int8_t>(c[e]);
  }
}

template <int S, int W, bool kWarpTeams>
struct K1Shape {
  static constexpr int kTeams = kWarpTeams ? 4 : 1;
  static constexpr int kConsumers = kWarpTeams ? 32 : 32 * W;  // rounding threads per team
  static constexpr int kThreads = kWarpTeams ? 128 : 32 * (W + 1);
  static constexpr int kMinBlocks = kWarpTeams ? 8 : (1024 / kThreads > 0 ? 1024 / kThreads : 1);
};

// kRowMax (one-CTA teams, no gather): |x|max comes from row_absmax (written by the
// producing GEMM's epilogue) instead of a reduction, so consumer warps never wait on one
// another; the producer warp resets each row's entry once every consumer released it.
template <int S, int W, bool kStatic, bool kGather, bool kWarpTeams, bool kRowMax = false>
__global__ void __launch_bounds__(K1Shape<S, W, kWarpTeams>::kThreads,
                                  K1Shape<S, W, kWarpTeams>::kMinBlocks)
    quant_act_rows_kernel(const uint16_t* __restrict__ x, int64_t m, int k, int64_t ldx,
                          const int32_t* __restrict__ gather, int k_out, double static_scale,
                          int qmax, double rqmax, int8_t* __restrict__ q, int64_t ldq,
                          float* __restrict__ s32_out, double* __restrict__ s64_out,
                          unsigned long long* __restrict__ err,
                          unsigned long long* __restrict__ trace, int dbg,
                          uint32_t* __restrict__ row_absmax) {
  static_assert(!kRowMax || (!kWarpTeams && !kGather && !kStatic),
                "row_absmax mode: per-token, one-CTA teams, no gather");
  using Sh = K1Shape<S, W, kWarpTeams>;
  constexpr int kTeams = Sh::kTeams;
  constexpr int T = Sh::kConsumers;
  extern __shared__ __align__(128) uint16_t k1_smem[];
  __shared__ uint32_t part[kK1Parts][kWarpTeams ? 1 : W];
  __shared__ __align__(8) uint64_t pbar[kK1Parts];
  __shared__ __align__(8) uint64_t full[kTeams][S];
  __shared__ __align__(8) uint64_t empty[S];
  if (trace && threadIdx.x == 0) {  // diagnostics (QARVD_K1_TRACE): CTA start time and SM
    unsigned long long t;
    uint32_t smid;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    trace[3 * blockIdx.x] = t;
    trace[3 * blockIdx.x + 2] = smid;
  }
  const int team = kWarpTeams ? static_cast<int>(threadIdx.x >> 5) : 0;
  const int tt = kWarpTeams ? static_cast<int>(threadIdx.x & 31) : static_cast<int>(threadIdx.x);
  const int warp = tt >> 5, lane = threadIdx.x & 31;
  const int nvec = k >> 3;
  const int row_stride = (k + 8 + 63) & ~63;  // + 8 zero sentinels; 128-byte aligned slots
  const uint32_t row_bytes = static_cast<uint32_t>(k) * 2u;
  uint16_t* slots = k1_smem + team * S * row_stride;
  int16_t* gidx = reinterpret_cast<int16_t*>(k1_smem + kTeams * S * row_stride);
  const int64_t step = static_cast<int64_t>(gridDim.x) * kTeams;
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * kTeams + team;
  const int nrows = row0 < m ? static_cast<int>((m - 1 - row0) / step + 1) : 0;

  auto load_row = [&](int j) {  // one lane: stream row j of this team into its slot
    const int s = j % S;
    ptx::mbar_expect_tx(&full[team][s], row_bytes);
    ptx::bulk_load_1d(slots + s * row_stride, x + (row0 + static_cast<int64_t>(j) * step) * ldx,
                      row_bytes, &full[team][s]);
  };
  auto wait_full = [&](int j) {
    ptx::mbar_wait_spin(&full[team][j % S], static_cast<uint32_t>((j / S) & 1));
  };
  // |x| max of this thread's chunks as packed 16-bit max of the sign-cleared bf16 bits
  // (non-finite values are exactly the magnitudes >= 0x7f80), reduced over the warp
  auto warp_part_max = [&](int slot) -> uint32_t {
    const uint16_t* srow = slots + slot * row_stride;
    uint32_t mx = 0;
#pragma unroll 4
    for (int vi = tt; vi < nvec; vi += T) {
      const uint4 d = *reinterpret_cast<const uint4*>(srow + vi * 8);
      mx = __vmaxu2(mx, __vmaxu2(__vmaxu2(d.x & 0x7fff7fffu, d.y & 0x7fff7fffu),
                                 __vmaxu2(d.z & 0x7fff7fffu, d.w & 0x7fff7fffu)));
    }
    return __reduce_max_sync(0xffffffffu, max(mx & 0xffffu, mx >> 16));
  };
  auto publish = [&](int j) {  // this warp's partial max of row j (landed)
    const uint32_t pm = warp_part_max(j % S);
    if (lane == 0) part[j % kK1Parts][warp] = pm;
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&pbar[j % kK1Parts]);
  };

  if (threadIdx.x == 0) {
    for (int t = 0; t < kTeams; ++t)
      for (int s = 0; s < S; ++s) ptx::mbar_init(&full[t][s], 1);
    for (int s = 0; s < S; ++s) ptx::mbar_init(&empty[s], W);
    for (int b = 0; b < kK1Parts; ++b) ptx::mbar_init(&pbar[b], W);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();  // x is written by the previous kernel of the chain
  pdl_launch_dependents();
  // the first rows stream in while the permutation table is staged
  const bool producer = kWarpTeams ? lane == 0 : (warp == W && lane == 0);
  if (producer)
    for (int j = 0; j < S && j < nrows; ++j) load_row(j);
  if (kGather) {  // k_out % 16 == 0 and gather 16-byte aligned (launch_rows)
#pragma unroll 4
    for (int c4 = threadIdx.x; c4 < (k_out >> 2); c4 += blockDim.x) {
      const int4 g = __ldg(reinterpret_cast<const int4*>(gather) + c4);
      const uint32_t lo = static_cast<uint16_t>(g.x < 0 ? k : g.x) |
                          (static_cast<uint32_t>(g.y < 0 ? k : g.y) << 16);
      const uint32_t hi = static_cast<uint16_t>(g.z < 0 ? k : g.z) |
                          (static_cast<uint32_t>(g.w < 0 ? k : g.w) << 16);
      reinterpret_cast<uint2*>(gidx)[c4] = make_uint2(lo, hi);
    }
  }
  if (tt < 8) {
#pragma unroll
    for (int s = 0; s < S; ++s) slots[s * row_stride + k + tt] = 0;
  }
  __syncthreads();

  if (!kWarpTeams && warp == W) {
    // producer warp: refill each slot once all consumer warps released it
    if (lane == 0) {
      for (int j = S; j < nrows; ++j) {
        ptx::mbar_wait_spin(&empty[j % S], static_cast<uint32_t>((j / S - 1) & 1));
        if (kRowMax) row_absmax[row0 + static_cast<int64_t>(j - S) * step] = 0u;
        load_row(j);
      }
      if (kRowMax)  // the last rows' entries, once their slots are released
        for (int j = nrows > S ? nrows - S : 0; j < nrows; ++j) {
          ptx::mbar_wait_spin(&empty[j % S], static_cast<uint32_t>((j / S) & 1));
          row_absmax[row0 + static_cast<int64_t>(j) * step] = 0u;
        }
    }
  } else {
    if (!kWarpTeams && !kRowMax && nrows > 0) {
      wait_full(0);
      publish(0);
    }
    for (int j = 0; j < nrows; ++j) {
      const int64_t row = row0 + static_cast<int64_t>(j) * step;
      const int slot = j % S;
      const uint16_t* srow = slots + slot * row_stride;
      uint32_t mag;
      if (kWarpTeams) {
        wait_full(j);
        mag = warp_part_max(slot);
      } else if (kRowMax) {
        mag = kStatic ? 0u : __ldcg(row_absmax + row);
        wait_full(j);
      } else {
        if (j + 1 < nrows) {
          wait_full(j + 1);
          publish(j + 1);
        }
        ptx::mbar_wait_spin(&pbar[j % kK1Parts], static_cast<uint32_t>((j / kK1Parts) & 1));
        mag = 0;
#pragma unroll
        for (int w = 0; w < (kWarpTeams ? 1 : W); ++w) mag = max(mag, part[j % kK1Parts][w]);
      }

      const bool row_bad = mag >= 0x7f80u;
      const float amax = __uint_as_float(mag << 16);
      ActScale sc;
      sc.fq = static_cast<float>(qmax);
      if (kStatic) {
        const GroupScale g = scale_static(static_scale);
        sc.r = g.r32;
        sc.exact = g.exact;
        sc.s64 = static_scale;
      } else {
        // r = fl(fl(1/amax) * qmax): within 2^-23 of qmax/amax, inside the tie guard's margin
        sc.r = amax > 0.f ? __fmul_rn(__frcp_rn(amax), static_cast<float>(qmax)) : 0.f;
        sc.exact = amax > 0.f && !(sc.r <= FLT_MAX && sc.r >= FLT_MIN);
        sc.s64 = 0.0;
      }
      // s64 = fl64(amax / qmax) (quant.cpp:168-181) as y = amax * fl64(1/qmax) plus one fma
      // correction -- equal to the correctly rounded quotient for every bf16 amax and every
      // qmax of 2..8 bits (checked exhaustively, tests/test_oracle.py)
      auto row_s64 = [&]() -> double {
        if (kStatic) return static_scale;
        if (!(amax > 0.f)) return DBL_MIN;
        const double a = static_cast<double>(amax), y = a * rqmax;
        return fma(fma(-y, static_cast<double>(qmax), a), rqmax, y);
      };
      if (tt == T - 1) {
        const double s = row_s64();
        if (s32_out) s32_out[row] = (kStatic || amax > 0.f) ? __double2float_rn(s) : 0.f;
        if (s64_out) s64_out[row] = s;
      }
      int8_t* qr = q + row * ldq;
      auto src_of = [&](int c) -> int { return kGather ? gidx[c] : c; };

      if (dbg & 1) {
        // diagnostics: no codes
      } else if (row_bad || sc.exact) {
        // rare rows: a non-finite input (reported; the reference throws) or an unusable
        // fp32 reciprocal -- every code takes the exact path
        const double s64 = row_s64();
        for (int c = tt; c < k_out; c += T)
          qr[c] = static_cast<int8_t>(act_code_slow(srow[src_of(c)], s64, qmax, err, row * k_out + c));
      } else {
        // Fast codes.  A chunk holding a value within the tie guard sets its bit in
        // `flagged` and is repaired after the loop (act_fix_flagged).
        const double s64 = row_s64();
        uint32_t flagged = 0;
        if (!kGather) {
          int i = 0;
#pragma unroll 2
          for (int vi = tt; vi < nvec; vi += T, ++i) {
            const uint4 d = *reinterpret_cast<const uint4*>(srow + vi * 8);
            const uint32_t w[4] = {d.x, d.y, d.z, d.w};
            uint32_t c[8];
            float dmax = 0.f;
            if (dbg & 4) {  // diagnostics: trivial codes (isolates the rounding math)
#pragma unroll
              for (int h = 0; h < 4; ++h) {
                c[2 * h] = w[h] >> 8;
                c[2 * h + 1] = w[h] >> 24;
              }
            } else {
#pragma unroll
            for (int h = 0; h < 4; ++h)
              act_codes2<kStatic>(__uint_as_float(w[h] << 16), __uint_as_float(w[h] & 0xffff0000u),
                                  sc, c[2 * h], c[2 * h + 1], dmax);
            }
            flagged |= static_cast<uint32_t>(dmax > tie_guard<kStatic>()) << i;
            const uint2 st = make_uint2(pack4(c[0], c[1], c[2], c[3]), pack4(c[4], c[5], c[6], c[7]));
            if (!(dbg & 2) || st.x == 0x12345678u) *reinterpret_cast<uint2*>(qr + vi * 8) = st;
          }
        } else {
          // 4 consecutive codes per lane per step: neighbouring lanes read shared memory
          // 8 bytes apart (at most 2-way bank conflicts for a near-contiguous gather) and
          // write one coalesced 4-byte word each
          int i = 0;
#pragma unroll 4
          for (int c0 = tt * 4; c0 < k_out; c0 += T * 4, ++i) {
            const uint2 gp = *reinterpret_cast<const uint2*>(gidx + c0);
            const uint16_t hv[4] = {srow[gp.x & 0xffffu], srow[gp.x >> 16], srow[gp.y & 0xffffu],
                                    srow[gp.y >> 16]};
            uint32_t c[4];
            float dmax = 0.f;
            act_codes2<kStatic>(__uint_as_float(static_cast<uint32_t>(hv[0]) << 16),
                                __uint_as_float(static_cast<uint32_t>(hv[1]) << 16), sc, c[0], c[1], dmax);
            act_codes2<kStatic>(__uint_as_float(static_cast<uint32_t>(hv[2]) << 16),
                                __uint_as_float(static_cast<uint32_t>(hv[3]) << 16), sc, c[2], c[3], dmax);
            flagged |= static_cast<uint32_t>(dmax > tie_guard<kStatic>()) << i;
            *reinterpret_cast<uint32_t*>(qr + c0) = pack4(c[0], c[1], c[2], c[3]);
          }
        }
        if (flagged) act_fix_flagged<kStatic, kGather>(srow, gidx, qr, tt, T, flagged, sc, s64, qmax);
      }
      // release the slot: the team's lane 0 (warp teams) or the producer warp refills it
      __syncwarp();
      if (kWarpTeams) {
        if (lane == 0 && j + S < nrows) load_row(j + S);
      } else if (lane == 0) {
        ptx::mbar_arrive(&empty[slot]);
      }
    }
  }
  if (trace) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      trace[3 * blockIdx.x + 1] = t;
    }
  }
}

// ---------------------------------------------------------------------------
// Streaming K1 for rows already in plan order whose |x|max is known: per-token rows whose
// producer GEMM wrote row_absmax in its epilogue (qarvd_dual_gemm_rowmax; the chain folds
// the permutation into that producer, pipeline.QuantizedChain), or a static scale.  Every
// 16-byte chunk is then independent: one CTA per row (grid-stride), threads stride over the
// row's chunks, no barrier between load and store.  A per-token row's row_absmax entry is
// reset to 0 once the row is done, ready for the producer's next step.
template <bool kStatic>
__device__ __noinline__ void act_fix_flagged_global(const uint16_t* xr, int8_t* qr, int tid, int nthr,
                                                    uint32_t flagged, ActScale sc, double s64,
                                                    int qmax) {
  while (flagged) {
    const int i = __ffs(flagged) - 1;
    flagged &= flagged - 1;
    const int c0 = (tid + i * nthr) * 8;
    uint16_t hv[8];
    uint32_t c[8];
    float dmax = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) hv[e] = xr[c0 + e];
#pragma unroll
    for (int e = 0; e < 8; e += 2)
      act_codes2<kStatic>(__uint_as_float(static_cast<uint32_t>(hv[e]) << 16),
                          __uint_as_float(static_cast<uint32_t>(hv[e + 1]) << 16), sc, c[e],
                          c[e + 1], dmax);
    bool rescan = false;
    act_fix_chunk<kStatic, 8, false>(hv, c, sc, s64, qmax, rescan);
    if (rescan) act_fix_chunk<kStatic, 8, true>(hv, c, sc, s64, qmax, rescan);
#pragma unroll
    for (int e = 0; e < 8; ++e) qr[c0 + e] = static_cast<int8_t>(c[e]);
  }
}

constexpr int kStreamThreads = 256;

template <bool kStatic>
__global__ void __launch_bounds__(kStreamThreads, 4)
    quant_act_stream_kernel(const uint16_t* __restrict__ x, int64_t m, int k, int64_t ldx,
                            uint32_t* __restrict__ row_absmax, double static_scale, int qmax,
                            double rqmax, int8_t* __restrict__ q, int64_t ldq,
                            float* __restrict__ s32_out, double* __restrict__ s64_out,
                            unsigned long long* __restrict__ err) {
  const int nvec = k >> 3;
  const int tid = threadIdx.x;
  pdl_wait();
  pdl_launch_dependents();
  for (int64_t row = blockIdx.x; row < m; row += gridDim.x) {
    const uint32_t mag = kStatic ? 0u : __ldcg(row_absmax + row);
    const bool row_bad = mag >= 0x7f80u;
    const float amax = __uint_as_float(mag << 16);
    ActScale sc;
    sc.fq = static_cast<float>(qmax);
    if (kStatic) {
      const GroupScale g = scale_static(static_scale);
      sc.r = g.r32;
      sc.exact = g.exact;
      sc.s64 = static_scale;
    } else {
      sc.r = amax > 0.f ? __fmul_rn(__frcp_rn(amax), static_cast<float>(qmax)) : 0.f;
      sc.exact = amax > 0.f && !(sc.r <= FLT_MAX && sc.r >= FLT_MIN);
      sc.s64 = 0.0;
    }
    double s64;
    if (kStatic) {
      s64 = static_scale;
    } else if (!(amax > 0.f)) {
      s64 = DBL_MIN;
    } else {  // fl64(amax / qmax), see quant_act_rows_kernel
      const double a = static_cast<double>(amax), y = a * rqmax;
      s64 = fma(fma(-y, static_cast<double>(qmax), a), rqmax, y);
    }
    if (tid == 0) {
      if (s32_out) s32_out[row] = (kStatic || amax > 0.f) ? __double2float_rn(s64) : 0.f;
      if (s64_out) s64_out[row] = s64;
    }
    const uint16_t* xr = x + row * ldx;
    int8_t* qr = q + row * ldq;
    if (row_bad || sc.exact) {
      // a non-finite input (reported; the reference throws) or an unusable fp32 reciprocal
      for (int c = tid; c < k; c += kStreamThreads) {
        const uint16_t h = xr[c];
        // a static-scale row has no |x|max: its non-finite values surface here per value
        qr[c] = static_cast<int8_t>(act_code_slow(h, s64, qmax, err, row * k + c));
      }
    } else {
      uint32_t flagged = 0;
      int i = 0;
#pragma unroll 4
      for (int vi = tid; vi < nvec; vi += kStreamThreads, ++i) {
        const uint4 d = ldg_stream(reinterpret_cast<const uint4*>(xr) + vi);
        const uint32_t w[4] = {d.x, d.y, d.z, d.w};
        uint32_t c[8];
        float dmax = 0.f;
        if (kStatic) {  // no |x|max: non-finite values are caught per chunk
          const uint32_t mx = __vmaxu2(__vmaxu2(w[0] & 0x7fff7fffu, w[1] & 0x7fff7fffu),
                                       __vmaxu2(w[2] & 0x7fff7fffu, w[3] & 0x7fff7fffu));
          if (max(mx & 0xffffu, mx >> 16) >= 0x7f80u) dmax = 1.f;
        }
#pragma unroll
        for (int h = 0; h < 4; ++h)
          act_codes2<kStatic>(__uint_as_float(w[h] << 16), __uint_as_float(w[h] & 0xffff0000u), sc,
                              c[2 * h], c[2 * h + 1], dmax);
        flagged |= static_cast<uint32_t>(dmax > tie_guard<kStatic>()) << i;
        *reinterpret_cast<uint2*>(qr + vi * 8) =
            make_uint2(pack4(c[0], c[1], c[2], c[3]), pack4(c[4], c[5], c[6], c[7]));
      }
      if (flagged) {
        if (kStatic) {  // flagged static chunks: exact per value (also reports non-finite ones)
          while (flagged) {
            const int b = __ffs(flagged) - 1;
            flagged &= flagged - 1;
            const int c0 = (tid + b * kStreamThreads) * 8;
            for (int e = 0; e < 8; ++e)
              qr[c0 + e] = static_cast<int8_t>(act_code_slow(xr[c0 + e], s64, qmax, err, row * k + c0 + e));
          }
        } else {
          act_fix_flagged_global<kStatic>(xr, qr, tid, kStreamThreads, flagged, sc, s64, qmax);
        }
      }
    }
    if (!kStatic) {
      __syncthreads();  // every thread has read row_absmax[row]
      if (tid == 0) row_absmax[row] = 0u;
    }
  }
}

// ---------------------------------------------------------------------------
// Flat K1 for rows already in plan order whose |x|max is known from the producer GEMM's
// per-row partial maxima (qarvd_dual_gemm_pmax: one per epilogue warp and 256-column tile,
// row-major [m][pm_count], rewritten every step -- nothing to reset), or a static scale.
// The M x K/8 16-byte chunks are split into spans of 1024 consecutive chunks, one span per
// CTA (256 threads x 4 chunks): every thread issues its four loads first, the CTA folds the
// partial maxima of the <= 18 rows its span touches (k >= 512) in shared memory, then rounds
// and stores.  No row-level synchronisation, so loads, rounding and stores of neighbouring
// CTAs overlap like a plain elementwise kernel (the structure that reaches the HBM floor in
// scripts/stream_probe.cu).
constexpr int kFlatThreads = 256;
constexpr int kFlatChunks = 4;
constexpr int kFlatSpan = kFlatThreads * kFlatChunks;
constexpr int kFlatMaxRows = 18;

// repair of one flagged chunk (values within the tie guard / only the division decides)
template <bool kStatic>
__device__ __noinline__ void act_fix_one_chunk(const uint16_t* xs, int8_t* qs, ActScale sc,
                                               double s64, int qmax, unsigned long long* err,
                                               int64_t flat) {
  uint16_t hv[8];
  uint32_t c[8];
  float dmax = 0.f;
  bool bad = false;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    hv[e] = xs[e];
    bad |= (hv[e] & 0x7f80u) == 0x7f80u;
  }
  if (kStatic && bad) {  // a static scale has no |x|max: non-finite values surface per value
#pragma unroll
    for (int e = 0; e < 8; ++e) qs[e] = static_cast<int8_t>(act_code_slow(hv[e], s64, qmax, err, flat + e));
    return;
  }
#pragma unroll
  for (int e = 0; e < 8; e += 2)
    act_codes2<kStatic>(__uint_as_float(static_cast<uint32_t>(hv[e]) << 16),
                        __uint_as_float(static_cast<uint32_t>(hv[e + 1]) << 16), sc, c[e], c[e + 1], dmax);
  bool rescan = false;
  act_fix_chunk<kStatic, 8, false>(hv, c, sc, s64, qmax, rescan);
  if (rescan) act_fix_chunk<kStatic, 8, true>(hv, c, sc, s64, qmax, rescan);
#pragma unroll
  for (int e = 0; e < 8; ++e) qs[e] = static_cast<int8_t>(c[e]);
}

template <bool kStatic>
__global__ void __launch_bounds__(kFlatThreads, 5)
    quant_act_flat_kernel(const uint16_t* __restrict__ x, int64_t m, int k, int64_t ldx,
                          const uint32_t* __restrict__ row_pmax, int pm_count, double static_scale,
                          int qmax, double rqmax, int8_t* __restrict__ q, int64_t ldq,
                          float* __restrict__ s32_out, double* __restrict__ s64_out,
                          unsigned long long* __restrict__ err) {
  __shared__ uint32_t s_mag[kFlatMaxRows];
  __shared__ float s_r[kFlatMaxRows];
  __shared__ double s_s64[kFlatMaxRows];
  __shared__ int s_slow[kFlatMaxRows];
  const int nvec = k >> 3;
  const int tid = threadIdx.x;
  const int64_t total = m * nvec;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * kFlatSpan;
  const int64_t ra = c0 / nvec;                         // first row of the span
  const int base0 = static_cast<int>(c0 - ra * nvec);  // its first chunk within that row
  const int span = static_cast<int>(total - c0 < kFlatSpan ? total - c0 : kFlatSpan);
  const int nr = (base0 + span - 1) / nvec + 1;        // rows touched (<= kFlatMaxRows)
  if (tid < kFlatMaxRows) s_mag[tid] = 0u;
  pdl_wait();
  pdl_launch_dependents();

  // ---- issue the loads (row / column of each chunk by stepping, no per-chunk division)
  uint4 d[kFlatChunks];
  int rl[kFlatChunks], col[kFlatChunks];
  {
    int local = base0 + tid;
    int r = local / nvec;
    int cc = local - r * nvec;
#pragma unroll
    for (int i = 0; i < kFlatChunks; ++i) {
      rl[i] = r;
      col[i] = cc;
      if (tid + i * kFlatThreads < span)
        d[i] = ldg_stream(reinterpret_cast<const uint4*>(x + (ra + r) * ldx) + cc);
      cc += kFlatThreads;
      while (cc >= nvec) {
        cc -= nvec;
        ++r;
      }
    }
  }
  __syncthreads();  // s_mag cleared
  if (!kStatic) {
    for (int rr = 0; rr < nr; ++rr) {
      const uint32_t* pr = row_pmax + (ra + rr) * pm_count;
      uint32_t mx = 0;
      for (int j = tid; j < pm_count; j += kFlatThreads) mx = max(mx, __ldcg(pr + j));
      mx = __reduce_max_sync(0xffffffffu, mx);
      if ((tid & 31) == 0 && mx) atomicMax(&s_mag[rr], mx);
    }
    __syncthreads();
  }
  if (tid < nr) {
    const int64_t row = ra + tid;
    const uint32_t mag = kStatic ? 0u : s_mag[tid];
    const float amax = __uint_as_float(mag << 16);
    double s64;
    float r;
    bool slow;
    if (kStatic) {
      const GroupScale g = scale_static(static_scale);
      r = g.r32;
      slow = g.exact;
      s64 = static_scale;
    } else {
      r = amax > 0.f ? __fmul_rn(__frcp_rn(amax), static_cast<float>(qmax)) : 0.f;
      slow = mag >= 0x7f80u || (amax > 0.f && !(r <= FLT_MAX && r >= FLT_MIN));
      if (!(amax > 0.f)) {
        s64 = DBL_MIN;
      } else {  // fl64(amax / qmax), see quant_act_rows_kernel
        const double a = static_cast<double>(amax), y = a * rqmax;
        s64 = fma(fma(-y, static_cast<double>(qmax), a), rqmax, y);
      }
    }
    s_r[tid] = r;
    s_s64[tid] = s64;
    s_slow[tid] = slow ? 1 : 0;
    if (row * nvec >= c0) {  // this span holds the row's first chunk: it writes the scales
      if (s32_out) s32_out[row] = (kStatic || amax > 0.f) ? __double2float_rn(s64) : 0.f;
      if (s64_out) s64_out[row] = s64;
    }
  }
  __syncthreads();

  ActScale sc;
  sc.fq = static_cast<float>(qmax);
  sc.exact = false;
  sc.s64 = 0.0;
  uint32_t flagged = 0;
#pragma unroll
  for (int i = 0; i < kFlatChunks; ++i) {
    if (tid + i * kFlatThreads >= span) continue;
    const int rr = rl[i];
    const int64_t row = ra + rr;
    int8_t* qs = q + row * ldq + col[i] * 8;
    sc.r = s_r[rr];
    const uint32_t w[4] = {d[i].x, d[i].y, d[i].z, d[i].w};
    uint32_t c[8];
    float dmax = 0.f;
    if (kStatic) {  // no |x|max: non-finite values are caught per chunk
      const uint32_t mx = __vmaxu2(__vmaxu2(w[0] & 0x7fff7fffu, w[1] & 0x7fff7fffu),
                                   __vmaxu2(w[2] & 0x7fff7fffu, w[3] & 0x7fff7fffu));
      if (max(mx & 0xffffu, mx >> 16) >= 0x7f80u) dmax = 1.f;
    }
#pragma unroll
    for (int h = 0; h < 4; ++h)
      act_codes2<kStatic>(__uint_as_float(w[h] << 16), __uint_as_float(w[h] & 0xffff0000u), sc,
                          c[2 * h], c[2 * h + 1], dmax);
    if (s_slow[rr] || dmax > tie_guard<kStatic>()) flagged |= 1u << i;
    *reinterpret_cast<uint2*>(qs) = make_uint2(pack4(c[0], c[1], c[2], c[3]), pack4(c[4], c[5], c[6], c[7]));
  }
  while (flagged) {  // (rare) out of line: ties, slow rows, non-finite values
    const int i = __ffs(flagged) - 1;
    flagged &= flagged - 1;
    const int rr = rl[i];
    const int64_t row = ra + rr;
    const uint16_t* xs = x + row * ldx + col[i] * 8;
    int8_t* qs = q + row * ldq + col[i] * 8;
    if (s_slow[rr]) {
      for (int e = 0; e < 8; ++e)
        qs[e] = static_cast<int8_t>(act_code_slow(xs[e], s_s64[rr], qmax, err, row * k + col[i] * 8 + e));
    } else {
      ActScale sf = sc;
      sf.r = s_r[rr];
      act_fix_one_chunk<kStatic>(xs, qs, sf, s_s64[rr], qmax, err, row * k + col[i] * 8);
    }
  }
}

// ---------------------------------------------------------------------------
// K5 batched over layers (calibration: every layer's weights in one launch).  One warp team
// per row: the row streams into shared memory by a 1-D bulk copy, pass 1 takes the
// outlier- and normal-group |w| maxima through the layer's int16 gather table, pass 2
// emits the codes of each group with its scale (same exact rounding and tie handling as
// K1), four per lane per step.  grid.y = layer; each CTA stages its layer's table.
struct WeightJobDev {
  const uint16_t* w;
  int64_t n, k, ldw;
  const int32_t* gather;
  int64_t k_pad, k_o;     // or, with plan_info, upper bounds (the device plan decides)
  const int64_t* plan_info;  // optional device {k_outlier, k_pad} (qarvd_prepare_weights_planned)
  int8_t* wq;
  int64_t ldq;
  double* so64;
  double* sn64;
  float* so32;
  float* sn32;
};
constexpr int kWTeams = 8;

template <bool dummy = false>
__device__ __noinline__ void wq_fix_chunk(const uint16_t* hv, uint32_t* c, ActScale sc, double s64, int qmax) {
  bool rescan = false;
  act_fix_chunk<false, 4, false>(hv, c, sc, s64, qmax, rescan);
  if (rescan) act_fix_chunk<false, 4, true>(hv, c, sc, s64, qmax, rescan);
}

// TW warps per row (1 for rows of <= 2048 values, 8 for the wide rows: one warp per 8960-wide
// row kept 4-5 warps per SM busy), TEAMS row teams per CTA.  Pass 1 takes the two group maxima
// from the contiguous row (16-byte reads) with an outlier-column bitmask instead of the gather.
template <int TW, int TEAMS>
__global__ void __launch_bounds__(32 * TW * TEAMS)
    prep_weights_batched_kernel(const WeightJobDev* __restrict__ jobs, int qmax, double rqmax,
                                unsigned long long* __restrict__ err) {
  constexpr int T = 32 * TW;
  extern __shared__ __align__(128) uint16_t wsm[];
  __shared__ __align__(8) uint64_t full[TEAMS][2];
  __shared__ uint32_t red[TEAMS][TW][2];
  const WeightJobDev J = jobs[blockIdx.y];
  const int team = static_cast<int>(threadIdx.x) / T, tt = static_cast<int>(threadIdx.x) % T;
  const int lane = threadIdx.x & 31, warp = tt >> 5;
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * TEAMS + team;
  if (static_cast<int64_t>(blockIdx.x) * TEAMS >= J.n) return;  // CTA-uniform
  pdl_wait();  // the plan kernel (qarvd_prepare_weights_planned) writes gather / plan_info
  const int k = static_cast<int>(J.k);
  const int k_pad = static_cast<int>(J.plan_info ? J.plan_info[1] : J.k_pad);
  const int k_o = static_cast<int>(J.plan_info ? J.plan_info[0] : J.k_o);
  const int row_stride = (k + 8 + 63) & ~63;
  // two row slots per team: row j+1 streams in while row j is rounded
  uint16_t* slots = wsm + team * 2 * row_stride;
  int16_t* gidx = reinterpret_cast<int16_t*>(wsm + TEAMS * 2 * row_stride);
  uint32_t* omask = reinterpret_cast<uint32_t*>(wsm + TEAMS * 2 * row_stride + ((J.k_pad + 7) & ~int64_t(7)));
  const int mask_words = (k + 31) >> 5;
  const int64_t step = static_cast<int64_t>(gridDim.x) * TEAMS;
  const uint32_t row_bytes = static_cast<uint32_t>(k) * 2u;
  if (threadIdx.x < 2 * TEAMS) ptx::mbar_init(&full[threadIdx.x >> 1][threadIdx.x & 1], 1);
  ptx::fence_mbar_init();
  for (int i = threadIdx.x; i < mask_words; i += blockDim.x) omask[i] = 0u;
  __syncthreads();
  auto load = [&](int sl, int64_t row) {
    ptx::mbar_expect_tx(&full[team][sl], row_bytes);
    ptx::bulk_load_1d(slots + sl * row_stride, J.w + row * J.ldw, row_bytes, &full[team][sl]);
  };
  if (tt == 0) {
    if (row0 < J.n) load(0, row0);
    if (row0 + step < J.n) load(1, row0 + step);
  }
  for (int c4 = threadIdx.x; c4 < (k_pad >> 2); c4 += blockDim.x) {
    const int4 g = __ldg(reinterpret_cast<const int4*>(J.gather) + c4);
    const uint32_t lo = static_cast<uint16_t>(g.x < 0 ? k : g.x) | (static_cast<uint32_t>(g.y < 0 ? k : g.y) << 16);
    const uint32_t hi = static_cast<uint16_t>(g.z < 0 ? k : g.z) | (static_cast<uint32_t>(g.w < 0 ? k : g.w) << 16);
    reinterpret_cast<uint2*>(gidx)[c4] = make_uint2(lo, hi);
  }
  for (int p = threadIdx.x; p < k_o; p += blockDim.x) {  // the outlier slab's columns
    const int g = __ldg(J.gather + p);
    if (g >= 0 && g < k) atomicOr(&omask[g >> 5], 1u << (g & 31));
  }
  if (tt < 8) {
    slots[k + tt] = 0;
    slots[row_stride + k + tt] = 0;
  }
  __syncthreads();

  const int nv = k >> 3;
  const uint4* const slot4[2] = {reinterpret_cast<const uint4*>(slots), reinterpret_cast<const uint4*>(slots + row_stride)};
  int j = 0;
  for (int64_t row = row0; row < J.n; row += step, ++j) {
    const uint16_t* srow = slots + (j & 1) * row_stride;
    ptx::mbar_wait_spin(&full[team][j & 1], static_cast<uint32_t>((j >> 1) & 1));
    // ---- pass 1: group maxima over the contiguous row (sign-cleared bf16 bits)
    uint32_t mo = 0, mn = 0;
    const uint4* s4 = slot4[j & 1];
    for (int c8 = tt; c8 < nv; c8 += T) {
      const uint4 d = s4[c8];
      const uint32_t mb = (omask[c8 >> 2] >> ((c8 & 3) * 8)) & 0xffu;
      if (mb == 0u) {
        const uint32_t m2 = __vmaxu2(__vmaxu2(d.x & 0x7fff7fffu, d.y & 0x7fff7fffu),
                                     __vmaxu2(d.z & 0x7fff7fffu, d.w & 0x7fff7fffu));
        mn = max(mn, max(m2 & 0xffffu, m2 >> 16));
      } else {
        const uint32_t w[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const uint32_t lo = w[h] & 0x7fffu, hi = (w[h] >> 16) & 0x7fffu;
          const bool olo = (mb >> (2 * h)) & 1u, ohi = (mb >> (2 * h + 1)) & 1u;
          mo = max(mo, olo ? lo : 0u);
          mn = max(mn, olo ? 0u : lo);
          mo = max(mo, ohi ? hi : 0u);
          mn = max(mn, ohi ? 0u : hi);
        }
      }
    }
    for (int c = nv * 8 + tt; c < k; c += T) {  // k % 8 tail
      const uint32_t v = srow[c] & 0x7fffu;
      if ((omask[c >> 5] >> (c & 31)) & 1u) mo = max(mo, v);
      else mn = max(mn, v);
    }
    mo = __reduce_max_sync(0xffffffffu, mo);
    mn = __reduce_max_sync(0xffffffffu, mn);
    if (TW > 1) {
      if (lane == 0) {
        red[team][warp][0] = mo;
        red[team][warp][1] = mn;
      }
      __syncthreads();
#pragma unroll
      for (int w = 0; w < TW; ++w) {
        mo = max(mo, red[team][w][0]);
        mn = max(mn, red[team][w][1]);
      }
    }
    const bool bad = mo >= 0x7f80u || mn >= 0x7f80u;
    ActScale so, sn;
    double so64, sn64;
    auto group = [&](uint32_t mg, ActScale& sc, double& s64) {
      const float amax = __uint_as_float(mg << 16);
      sc.fq = static_cast<float>(qmax);
      sc.s64 = 0.0;
      sc.r = amax > 0.f ? __fmul_rn(__frcp_rn(amax), static_cast<float>(qmax)) : 0.f;
      sc.exact = amax > 0.f && !(sc.r <= FLT_MAX && sc.r >= FLT_MIN);
      if (!(amax > 0.f)) {
        s64 = DBL_MIN;  // dual_scale.cpp:13-24 (all-zero group)
      } else {  // fl64(amax / qmax), see quant_act_rows_kernel
        const double a = static_cast<double>(amax), y = a * rqmax;
        s64 = fma(fma(-y, static_cast<double>(qmax), a), rqmax, y);
      }
    };
    group(mn, sn, sn64);
    if (k_o > 0) group(mo, so, so64);
    else {
      so = sn;
      so64 = sn64;  // single-scale plan: outlier scale = normal scale (dual_scale.cpp:55)
    }
    if (tt == 0) {
      if (J.so64) J.so64[row] = so64;
      if (J.sn64) J.sn64[row] = sn64;
      if (J.so32) J.so32[row] = so64 == DBL_MIN ? 0.f : __double2float_rn(so64);
      if (J.sn32) J.sn32[row] = sn64 == DBL_MIN ? 0.f : __double2float_rn(sn64);
    }
    int8_t* qr = J.wq + row * J.ldq;
    // ---- pass 2: codes in plan order through the gather, four per lane per step
    for (int c0 = tt * 4; c0 < k_pad; c0 += 4 * T) {
      const uint2 gp = *reinterpret_cast<const uint2*>(gidx + c0);
      const uint16_t hv[4] = {srow[gp.x & 0xffffu], srow[gp.x >> 16], srow[gp.y & 0xffffu], srow[gp.y >> 16]};
      const bool outl = c0 < k_o;
      const ActScale& sc = outl ? so : sn;
      const double s64 = outl ? so64 : sn64;
      uint32_t c[4];
      if (bad || sc.exact) {
        for (int e = 0; e < 4; ++e) {
          const int g = gidx[c0 + e];
          c[e] = (g >= k) ? 0u : act_code_slow(hv[e], s64, qmax, err, row * k_pad + c0 + e);
        }
      } else {
        float dmax = 0.f;
        act_codes2<false>(__uint_as_float(static_cast<uint32_t>(hv[0]) << 16),
                          __uint_as_float(static_cast<uint32_t>(hv[1]) << 16), sc, c[0], c[1], dmax);
        act_codes2<false>(__uint_as_float(static_cast<uint32_t>(hv[2]) << 16),
                          __uint_as_float(static_cast<uint32_t>(hv[3]) << 16), sc, c[2], c[3], dmax);
        if (dmax > tie_guard<false>()) wq_fix_chunk(hv, c, sc, s64, qmax);
      }
      *reinterpret_cast<uint32_t*>(qr + c0) = pack4(c[0], c[1], c[2], c[3]);
    }
    if (TW > 1) __syncthreads();  // the slot (and red) is free once the whole team is done
    else __syncwarp();
    if (tt == 0 && row + 2 * step < J.n) load(j & 1, row + 2 * step);
  }
}

// ---------------------------------------------------------------------------
// Generic kernel (f32 / f64 inputs, or rows too wide for shared memory):
// one warp per row, reads straight from global memory; f64 inputs always take
// the exact division (reference f64 semantics, no bf16 assumption).
template <int MODE, typename T>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
    quant_rows_generic_kernel(const T* __restrict__ x, int64_t m, int64_t k, int64_t ldx,
                              const int32_t* __restrict__ gather, int64_t k_out, int64_t k_o,
                              double static_scale, int qmax, int8_t* __restrict__ q, int64_t ldq,
                              float* __restrict__ s32_o, double* __restrict__ s64_o,
                              float* __restrict__ s32_n, double* __restrict__ s64_n,
                              unsigned long long* err) {
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t row = static_cast<int64_t>(blockIdx.x) * kWarpsPerCta + warp; row < m;
       row += static_cast<int64_t>(gridDim.x) * kWarpsPerCta) {
    const T* xr = x + row * ldx;
    double s_o64, s_n64;
    if (MODE == kActStatic) {
      s_o64 = s_n64 = static_scale;
    } else {
      double ao = 0.0, an = 0.0;
      for (int64_t c = lane; c < k_out; c += 32) {
        const int32_t src = gather ? __ldg(gather + c) : static_cast<int32_t>(c);
        if (src < 0) continue;
        const double v = fabs(InType<T>::to_double(xr[src]));
        if (!(v <= DBL_MAX)) continue;  // non-finite: reported below
        if (MODE == kWeightDual && c < k_o) ao = fmax(ao, v);
        else an = fmax(an, v);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        ao = fmax(ao, __shfl_xor_sync(0xffffffffu, ao, o));
        an = fmax(an, __shfl_xor_sync(0xffffffffu, an, o));
      }
      s_n64 = an > 0.0 ? __ddiv_rn(an, static_cast<double>(qmax)) : DBL_MIN;
      s_o64 = (MODE == kWeightDual && k_o > 0)
                  ? (ao > 0.0 ? __ddiv_rn(ao, static_cast<double>(qmax)) : DBL_MIN)
                  : s_n64;
    }
    if (lane == 0) {
      if (s32_n) s32_n[row] = s_n64 == DBL_MIN ? 0.f : __double2float_rn(s_n64);
      if (s64_n) s64_n[row] = s_n64;
      if (MODE == kWeightDual) {
        if (s32_o) s32_o[row] = s_o64 == DBL_MIN ? 0.f : __double2float_rn(s_o64);
        if (s64_o) s64_o[row] = s_o64;
      }
    }
    int8_t* qr = q + row * ldq;
    for (int64_t c = lane; c < k_out; c += 32) {
      const int32_t src = gather ? __ldg(gather + c) : static_cast<int32_t>(c);
      int code = 0;
      if (src >= 0) {
        const T v = xr[src];
        if (!InType<T>::finite(v)) {
          record_error(err, row * k_out + c);
        } else {
          const double s = (MODE == kWeightDual && c < k_o) ? s_o64 : s_n64;
          code = quant_code_exact(InType<T>::to_double(v), s, qmax);
        }
      }
      qr[c] = static_cast<int8_t>(code);
    }
  }
}

__global__ void init_err_kernel(unsigned long long* err) { *err = 0x7fffffffffffffffull; }

int grid_for_rows(int64_t m) {
  const int64_t ctas = (m + kWarpsPerCta - 1) / kWarpsPerCta;
  const int64_t cap = static_cast<int64_t>(kNumSMs) * 16;
  return static_cast<int>(ctas < cap ? ctas : cap);
}

template <int S, int W, bool kStatic, bool kGather, bool kWarpTeams>
int launch_act_rows_t(const uint16_t* x, int64_t m, int k, int64_t ldx, const int32_t* gather,
                      int k_out, double static_scale, int qmax, int8_t* q, int64_t ldq, float* s32,
                      double* s64, unsigned long long* err, cudaStream_t stream) {
  constexpr int kTeams = K1Shape<S, W, kWarpTeams>::kTeams;
  constexpr int kThreads = K1Shape<S, W, kWarpTeams>::kThreads;
  auto kern = quant_act_rows_kernel<S, W, kStatic, kGather, kWarpTeams>;
  static std::once_flag once;
  static cudaError_t attr = cudaSuccess;
  std::call_once(once, [&] { attr = set_smem_attrs(kern, 110 * 1024); });
  QARVD_CUDA_TRY(attr);
  const size_t smem = static_cast<size_t>(kTeams) * S * ((k + 8 + 63) & ~63) * 2 +
                      (kGather ? static_cast<size_t>((k_out + 7) & ~7) * 2 : 0);
  // persistent grid: as many CTAs as fit on the GPU (cached per shared-memory size)
  static thread_local size_t cached_smem = 0;
  static thread_local int cached_blocks = 0;
  if (cached_smem != smem) {
    int nb = 0;
    QARVD_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kThreads, smem));
    cached_smem = smem;
    cached_blocks = nb > 0 ? nb : 1;
  }
  const int64_t need = (m + kTeams - 1) / kTeams;
  const int64_t cap = static_cast<int64_t>(kNumSMs) * cached_blocks;
  const int64_t grid = need < cap ? need : cap;
  // QARVD_K1_TRACE=<device address>: per-CTA (start, end, smid) globaltimer trace (diagnostics)
  static unsigned long long* trace = [] {
    const char* e = getenv("QARVD_K1_TRACE");
    return e ? reinterpret_cast<unsigned long long*>(strtoull(e, nullptr, 0)) : nullptr;
  }();
  static const int dbg = getenv("QARVD_K1_DEBUG") ? atoi(getenv("QARVD_K1_DEBUG")) : 0;
  QARVD_CUDA_TRY(launch_pdl(kern, dim3(static_cast<unsigned>(grid)), dim3(kThreads), smem, stream, 1, x, m,
                            k, ldx, gather, k_out, static_scale, qmax, 1.0 / static_cast<double>(qmax), q,
                            ldq, s32, s64, err, trace, dbg, static_cast<uint32_t*>(nullptr)));
  return QARVD_OK;
}

// Team shape for a row of nvec 16-byte chunks: four one-warp teams per CTA for rows of up
// to 256 chunks, else one CTA of 4..8 warps, the count that splits the chunks most evenly
// (ties: more warps), e.g. 1120 chunks (K = 8960) -> 7 warps x 5 chunks per thread.
inline int k1_team_warps(int nvec) {
  if (nvec <= 256) return 1;
  int best_w = 8, best_waste = 1 << 30;
  for (int w = 8; w >= 4; --w) {
    const int per = (nvec + 32 * w - 1) / (32 * w);
    const int waste = per * 32 * w - nvec;
    if (waste < best_waste) {
      best_waste = waste;
      best_w = w;
    }
  }
  return best_w;
}

template <int W>
int launch_act_rowmax_ring(const uint16_t* x, int64_t m, int k, int64_t ldx, uint32_t* row_absmax,
                           int qmax, int8_t* q, int64_t ldq, float* s32, double* s64,
                           unsigned long long* err, cudaStream_t stream) {
  constexpr int S = 4;
  constexpr int kThreads = K1Shape<S, W, false>::kThreads;
  auto kern = quant_act_rows_kernel<S, W, false, false, false, true>;
  static std::once_flag once;
  static cudaError_t attr = cudaSuccess;
  std::call_once(once, [&] { attr = set_smem_attrs(kern, 110 * 1024); });
  QARVD_CUDA_TRY(attr);
  const size_t smem = static_cast<size_t>(S) * ((k + 8 + 63) & ~63) * 2;
  static thread_local size_t cached_smem = 0;
  static thread_local int cached_blocks = 0;
  if (cached_smem != smem) {
    int nb = 0;
    QARVD_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kThreads, smem));
    cached_smem = smem;
    cached_blocks = nb > 0 ? nb : 1;
  }
  const int64_t cap = static_cast<int64_t>(kNumSMs) * cached_blocks;
  const int64_t grid = m < cap ? m : cap;
  static const int dbg = getenv("QARVD_K1_DEBUG") ? atoi(getenv("QARVD_K1_DEBUG")) : 0;
  QARVD_CUDA_TRY(launch_pdl(kern, dim3(static_cast<unsigned>(grid)), dim3(kThreads), smem, stream, 1, x, m,
                            k, ldx, static_cast<const int32_t*>(nullptr), k, 0.0, qmax,
                            1.0 / static_cast<double>(qmax), q, ldq, s32, s64, err,
                            static_cast<unsigned long long*>(nullptr), dbg, row_absmax));
  return QARVD_OK;
}

int launch_act_rowmax(const uint16_t* x, int64_t m, int k, int64_t ldx, uint32_t* row_absmax,
                      int qmax, int8_t* q, int64_t ldq, float* s32, double* s64,
                      unsigned long long* err, cudaStream_t stream) {
  switch (k1_team_warps(k / 8)) {
    case 4: return launch_act_rowmax_ring<4>(x, m, k, ldx, row_absmax, qmax, q, ldq, s32, s64, err, stream);
    case 5: return launch_act_rowmax_ring<5>(x, m, k, ldx, row_absmax, qmax, q, ldq, s32, s64, err, stream);
    case 6: return launch_act_rowmax_ring<6>(x, m, k, ldx, row_absmax, qmax, q, ldq, s32, s64, err, stream);
    case 7: return launch_act_rowmax_ring<7>(x, m, k, ldx, row_absmax, qmax, q, ldq, s32, s64, err, stream);
    case 8: return launch_act_rowmax_ring<8>(x, m, k, ldx, row_absmax, qmax, q, ldq, s32, s64, err, stream);
  }
  QARVD_FAIL(QARVD_ERR_LOGIC, "unsupported K1 team size");
}

template <bool kStatic, bool kGather>
int launch_act_rows_g(const uint16_t* x, int64_t m, int k, int64_t ldx, const int32_t* gather,
                      int k_out, double static_scale, int qmax, int8_t* q, int64_t ldq, float* s32,
                      double* s64, unsigned long long* err, cudaStream_t stream) {
  // warp teams: one slot (a 1-row-per-team grid keeps 8 CTAs per SM resident, so every row
  // of a 4680-token step gets its own team in one wave); CTA teams: three
  int w = k1_team_warps(k / 8), slots = w == 1 ? 1 : 3;
  // diagnostics: QARVD_K1_SHAPE=<warps>x<slots> overrides the team shape of one-CTA teams
  static const char* shape = getenv("QARVD_K1_SHAPE");
  if (shape) sscanf(shape, "%dx%d", &w, &slots);
  const int key = w * 10 + slots;
  switch (key) {
#define QARVD_K1_CASE(WW, SS, TEAMS)                                                              \
  case WW * 10 + SS:                                                                              \
    return launch_act_rows_t<SS, WW, kStatic, kGather, TEAMS>(x, m, k, ldx, gather, k_out,       \
                                                              static_scale, qmax, q, ldq, s32,   \
                                                              s64, err, stream);
    QARVD_K1_CASE(1, 1, true)
    QARVD_K1_CASE(1, 2, true)
    QARVD_K1_CASE(2, 2, false)
    QARVD_K1_CASE(2, 3, false)
    QARVD_K1_CASE(4, 2, false)
    QARVD_K1_CASE(4, 3, false)
    QARVD_K1_CASE(5, 3, false)
    QARVD_K1_CASE(6, 3, false)
    QARVD_K1_CASE(7, 2, false)
    QARVD_K1_CASE(7, 3, false)
    QARVD_K1_CASE(8, 3, false)
#undef QARVD_K1_CASE
  }
  QARVD_FAIL(QARVD_ERR_LOGIC, "unsupported K1 team shape");
}


// ---------------------------------------------------------------------------
// K1, register-resident variant (the default for bf16 rows whose 16-byte chunks split evenly
// over the team): a team (one warp for rows of <= 2048 values, four teams per CTA; else one CTA
// of W warps) owns one row and every thread issues all of its V chunk loads at once
// (ld.global.nc, no L1 allocation), so the whole step's rows are in flight together; the
// |x| max is a packed 16-bit max over the registers (+ one shared-memory exchange for W > 1),
// and the codes come straight from the registers (plan-order rows) or from a per-team
// shared-memory copy through the plan's gather (read as int32 through L1).  One launch per
// step, no producer warp, no per-row barriers: the previous slot-ring kernel spent half its
// SM cycles waiting (ncu: 48% SMSP active, long_scoreboard) on a 1-row-per-team grid.
template <int V, int W, bool kStatic, bool kGather>
__device__ __noinline__ uint2 act_fix8_reg(uint4 d, ActScale sc, double s64, int qmax);
template <bool kStatic>
__device__ __noinline__ uint32_t act_fix4_reg(uint2 hv2, ActScale sc, double s64, int qmax);

// the 8 codes of a flagged chunk by the reference's own arithmetic, rint(v / s) in f64 then the
// clamp (quant.cpp:132-135): shorter than the tie analysis (act_fix8_reg), which on a
// one-row-per-warp launch lengthened the critical path of the ~half of the warps that hold a tie
__device__ __noinline__ uint2 act_fix8_div(uint4 d, double s64, int qmax) {
  const uint32_t w[4] = {d.x, d.y, d.z, d.w};
  uint32_t c[8];
#pragma unroll
  for (int h = 0; h < 8; ++h) {
    const uint32_t bits = h & 1 ? (w[h >> 1] & 0xffff0000u) : (w[h >> 1] << 16);
    c[h] = static_cast<uint32_t>(quant_code_exact(static_cast<double>(__uint_as_float(bits)), s64, qmax)) & 0xffu;
  }
  return make_uint2(pack4(c[0], c[1], c[2], c[3]), pack4(c[4], c[5], c[6], c[7]));
}

constexpr unsigned int kK1RepairCap = 512;  // near-tie chunks queued per CTA for the shared repair

// the gathered twin: plan positions c = tt, tt + T, ... < k_out through the int16 table
__device__ __noinline__ void act_slow_row_g(const uint16_t* xr, const int16_t* gidx, int k, int k_out, int8_t* qr,
                                            int tt, int T, double s64, int qmax, unsigned long long* err,
                                            int64_t flat0) {
  for (int c = tt; c < k_out; c += T) {
    const int g = gidx[c];
    qr[c] = g >= k ? static_cast<int8_t>(0) : static_cast<int8_t>(act_code_slow(xr[g], s64, qmax, err, flat0 + c));
  }
}

// every code of a rare row by the exact division (non-finite values reported), plan-order rows:
// this thread's chunks (tt + i T) * 8, i < V
__device__ __noinline__ void act_slow_row(const uint16_t* xr, int k, int8_t* qr, int tt, int T, int V, double s64,
                                          int qmax, unsigned long long* err, int64_t flat0) {
  for (int i = 0; i < V; ++i) {
    const int c0 = (tt + i * T) * 8;
    if (c0 >= k) break;
    for (int h = 0; h < 8; ++h)
      qr[c0 + h] = static_cast<int8_t>(act_code_slow(xr[c0 + h], s64, qmax, err, flat0 + c0 + h));
  }
}

template <int V, int W, bool kStatic, bool kGather>
__global__ void __launch_bounds__(W == 1 ? 256 : 32 * W, W == 1 ? 4 : (1152 / (32 * W) > 0 ? 1152 / (32 * W) : 1))
    quant_act_reg_kernel(const uint16_t* __restrict__ x, int64_t m, int k, int64_t ldx,
                         const int32_t* __restrict__ gather, int k_out, double static_scale, int qmax,
                         double rqmax, int8_t* __restrict__ q, int64_t ldq, float* __restrict__ s32_out,
                         double* __restrict__ s64_out, unsigned long long* __restrict__ err) {
  constexpr int kTeams = W == 1 ? 8 : 1;
  constexpr int T = 32 * W;
  extern __shared__ __align__(16) uint16_t k1r_smem[];
  __shared__ uint32_t wmax[W];
  const int row_stride = (k + 8 + 63) & ~63;
  const int team = W == 1 ? static_cast<int>(threadIdx.x >> 5) : 0;
  const int tt = W == 1 ? static_cast<int>(threadIdx.x & 31) : static_cast<int>(threadIdx.x);
  const int lane = threadIdx.x & 31, warp = tt >> 5;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * kTeams + team;
  // the plan's gather as an int16 table, staged once per CTA (pad -> k: the zero sentinel of
  // every row copy); read through L1 per row it cost more bytes than the row itself
  int16_t* gidx = reinterpret_cast<int16_t*>(k1r_smem + kTeams * row_stride);
  // runs[j]: the first source column of output chunk j (8 columns) when the chunk copies 8
  // consecutive source columns (a plan keeps the normal columns in order, so almost every chunk
  // does), else -1.  Such a chunk is gathered by two funnel shifts of three aligned words.
  int16_t* runs = gidx + ((k_out + 7) & ~7);
  if (kGather) {
    for (int c8 = threadIdx.x; c8 < (k_out >> 3); c8 += blockDim.x) {
      const int4 ga = __ldg(reinterpret_cast<const int4*>(gather) + 2 * c8);
      const int4 gb = __ldg(reinterpret_cast<const int4*>(gather) + 2 * c8 + 1);
      const int g[8] = {ga.x, ga.y, ga.z, ga.w, gb.x, gb.y, gb.z, gb.w};
      uint32_t w[4];
#pragma unroll
      for (int h = 0; h < 4; ++h)
        w[h] = static_cast<uint16_t>(g[2 * h] < 0 ? k : g[2 * h]) |
               (static_cast<uint32_t>(g[2 * h + 1] < 0 ? k : g[2 * h + 1]) << 16);
      reinterpret_cast<uint4*>(gidx)[c8] = make_uint4(w[0], w[1], w[2], w[3]);
      bool run = g[0] >= 0 && g[0] + 7 < k;
#pragma unroll
      for (int h = 1; h < 8; ++h) run = run && g[h] == g[0] + h;
      runs[c8] = static_cast<int16_t>(run ? g[0] : -1);
    }
  }
  __shared__ unsigned int s_nfix;
  __shared__ unsigned int s_fix[kK1RepairCap];  // (team << 16) | (tt << 4) | chunk
  __shared__ double s_s64[kTeams];
  if (threadIdx.x == 0) s_nfix = 0u;
  pdl_wait();  // x is written by the previous kernel of the chain
  pdl_launch_dependents();
  uint4 d[V];
  const bool live = row < m;  // W > 1: one team per CTA, the whole CTA shares it
  if (live) {
    const uint4* xr = reinterpret_cast<const uint4*>(x + row * ldx);
#pragma unroll
    for (int i = 0; i < V; ++i) d[i] = ldg_stream(xr + tt + i * T);
  }
  if (kGather || W > 1) __syncthreads();  // the table is staged / s_nfix is zeroed
  if (W > 1 && !live) return;             // CTA-uniform
  uint32_t mx = 0;
  if (live) {
#pragma unroll
    for (int i = 0; i < V; ++i)
      mx = __vmaxu2(mx, __vmaxu2(__vmaxu2(d[i].x & 0x7fff7fffu, d[i].y & 0x7fff7fffu),
                                 __vmaxu2(d[i].z & 0x7fff7fffu, d[i].w & 0x7fff7fffu)));
  }
  uint32_t mag = __reduce_max_sync(0xffffffffu, max(mx & 0xffffu, mx >> 16));
  if (W > 1) {
    if (lane == 0) wmax[warp] = mag;
    __syncthreads();
#pragma unroll
    for (int w = 0; w < W; ++w) mag = max(mag, wmax[w]);
  }
  const bool row_bad = mag >= 0x7f80u;
  const float amax = __uint_as_float(mag << 16);
  ActScale sc;
  sc.fq = static_cast<float>(qmax);
  double s64;
  if (kStatic) {
    const GroupScale g = scale_static(static_scale);
    sc.r = g.r32;
    sc.exact = g.exact;
    s64 = static_scale;
  } else {
    // r = fl(fl(1/amax) * qmax) and s64 = fl64(amax / qmax): see quant_act_rows_kernel
    sc.r = amax > 0.f ? __fmul_rn(__frcp_rn(amax), static_cast<float>(qmax)) : 0.f;
    sc.exact = amax > 0.f && !(sc.r <= FLT_MAX && sc.r >= FLT_MIN);
    if (!(amax > 0.f)) {
      s64 = DBL_MIN;
    } else {
      const double a = static_cast<double>(amax), y = a * rqmax;
      s64 = fma(fma(-y, static_cast<double>(qmax), a), rqmax, y);
    }
  }
  sc.s64 = s64;
  if (live && tt == T - 1) {
    if (s32_out) s32_out[row] = (kStatic || amax > 0.f) ? __double2float_rn(s64) : 0.f;
    if (s64_out) s64_out[row] = s64;
    s_s64[team] = s64;
  }
  int8_t* qr = q + row * ldq;
  // rare rows: non-finite input (reported) or an unusable fp32 reciprocal -- every code by the
  // exact division, out of line (inlined per chunk this path was three quarters of the code)
  const bool slow = live && (row_bad || sc.exact);
  if (slow) {
    if (kGather) act_slow_row_g(x + row * ldx, gidx, k, k_out, qr, tt, T, s64, qmax, err, row * k_out);
    else act_slow_row(x + row * ldx, k, qr, tt, T, V, s64, qmax, err, row * k_out);
  }
  // Fast codes in natural column order from the registers, 8 per lane per step: plan-order rows
  // store them, gathered rows write them to the team's shared slot.  A chunk with a value within
  // the tie guard is queued for the CTA-shared repair below: after the fast pass every thread of
  // the CTA takes queued chunks (the reference's division for their 8 values), so a row with
  // dozens of near-ties no longer serialises them on its own warp (4680 x 1536: 14.2 -> 11.9 us
  // in the microbenchmark).  A full queue repairs inline.
  uint8_t* crow = reinterpret_cast<uint8_t*>(k1r_smem + team * row_stride);
  if (live && !slow) {
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int c0 = (tt + i * T) * 8;
      const uint32_t w[4] = {d[i].x, d[i].y, d[i].z, d[i].w};
      uint32_t c[8];
      float dmax = 0.f;
#pragma unroll
      for (int h = 0; h < 4; ++h)
        act_codes2<kStatic>(__uint_as_float(w[h] << 16), __uint_as_float(w[h] & 0xffff0000u), sc, c[2 * h],
                            c[2 * h + 1], dmax);
      uint2 out = make_uint2(pack4(c[0], c[1], c[2], c[3]), pack4(c[4], c[5], c[6], c[7]));
      if (dmax > tie_guard<kStatic>()) {
        const unsigned int slot = atomicAdd(&s_nfix, 1u);
        if (slot < kK1RepairCap) s_fix[slot] = (static_cast<unsigned int>(team) << 16) | (tt << 4) | i;
        else out = act_fix8_div(d[i], s64, qmax);
      }
      if (kGather) *reinterpret_cast<uint2*>(crow + c0) = out;
      else *reinterpret_cast<uint2*>(qr + c0) = out;
    }
    if (kGather && tt < 8) crow[k + tt] = 0;  // the pad columns' sentinel (the table maps pads to k)
  }
  __syncthreads();  // the fast pass of every team is done, the queue complete
  const unsigned int nfix = min(s_nfix, kK1RepairCap);
  for (unsigned int e = threadIdx.x; e < nfix; e += blockDim.x) {
    const unsigned int en = s_fix[e];
    const int tm = static_cast<int>(en >> 16), lt = static_cast<int>((en >> 4) & 0xfffu), i = static_cast<int>(en & 15u);
    const int64_t rw = static_cast<int64_t>(blockIdx.x) * kTeams + tm;
    const int c0 = (lt + i * T) * 8;
    const uint4 dd = *reinterpret_cast<const uint4*>(x + rw * ldx + c0);
    const uint2 fixed = act_fix8_div(dd, s_s64[tm], qmax);
    if (kGather) *reinterpret_cast<uint2*>(reinterpret_cast<uint8_t*>(k1r_smem + tm * row_stride) + c0) = fixed;
    else *reinterpret_cast<uint2*>(q + rw * ldq + c0) = fixed;
  }
  if (kGather) {
    __syncthreads();  // the slots hold the final codes
    if (live && !slow) {
      // the plan's gather on the codes, 8 per lane per step: a run chunk by two funnel shifts of
      // three aligned words (the slot holds k + 8 bytes), the others byte by byte
      const uint32_t* crow32 = reinterpret_cast<const uint32_t*>(crow);
#pragma unroll 2
      for (int c0 = tt * 8; c0 < k_out; c0 += T * 8) {
        const int r = runs[c0 >> 3];
        uint2 out;
        if (r >= 0) {
          const uint32_t w0 = crow32[r >> 2], w1 = crow32[(r >> 2) + 1], w2 = crow32[(r >> 2) + 2];
          const uint32_t sh = static_cast<uint32_t>(r & 3) * 8u;
          out = make_uint2(__funnelshift_r(w0, w1, sh), __funnelshift_r(w1, w2, sh));
        } else {
          const uint4 gp = *reinterpret_cast<const uint4*>(gidx + c0);
          out = make_uint2(pack4(crow[gp.x & 0xffffu], crow[gp.x >> 16], crow[gp.y & 0xffffu], crow[gp.y >> 16]),
                           pack4(crow[gp.z & 0xffffu], crow[gp.z >> 16], crow[gp.w & 0xffffu], crow[gp.w >> 16]));
        }
        *reinterpret_cast<uint2*>(qr + c0) = out;
      }
    }
  }
}

// exact codes of one flagged 8-value chunk (plan-order rows) / 4 gathered values
template <int V, int W, bool kStatic, bool kGather>
__device__ __noinline__ uint2 act_fix8_reg(uint4 d, ActScale sc, double s64, int qmax) {
  const uint32_t w[4] = {d.x, d.y, d.z, d.w};
  uint16_t hv[8];
  uint32_t c[8];
  float dmax = 0.f;
#pragma unroll
  for (int h = 0; h < 8; ++h) hv[h] = static_cast<uint16_t>(h & 1 ? w[h >> 1] >> 16 : w[h >> 1] & 0xffffu);
#pragma unroll
  for (int h = 0; h < 4; ++h)
    act_codes2<kStatic>(__uint_as_float(w[h] << 16), __uint_as_float(w[h] & 0xffff0000u), sc, c[2 * h], c[2 * h + 1],
                        dmax);
  bool rescan = false;
  act_fix_chunk<kStatic, 8, false>(hv, c, sc, s64, qmax, rescan);
  if (rescan) act_fix_chunk<kStatic, 8, true>(hv, c, sc, s64, qmax, rescan);
  return make_uint2(pack4(c[0], c[1], c[2], c[3]), pack4(c[4], c[5], c[6], c[7]));
}
template <bool kStatic>
__device__ __noinline__ uint32_t act_fix4_reg(uint2 hv2, ActScale sc, double s64, int qmax) {
  const uint16_t hv[4] = {static_cast<uint16_t>(hv2.x & 0xffffu), static_cast<uint16_t>(hv2.x >> 16),
                          static_cast<uint16_t>(hv2.y & 0xffffu), static_cast<uint16_t>(hv2.y >> 16)};
  uint32_t c[4];
  float dmax = 0.f;
  act_codes2<kStatic>(__uint_as_float(static_cast<uint32_t>(hv[0]) << 16),
                      __uint_as_float(static_cast<uint32_t>(hv[1]) << 16), sc, c[0], c[1], dmax);
  act_codes2<kStatic>(__uint_as_float(static_cast<uint32_t>(hv[2]) << 16),
                      __uint_as_float(static_cast<uint32_t>(hv[3]) << 16), sc, c[2], c[3], dmax);
  bool rescan = false;
  act_fix_chunk<kStatic, 4, false>(hv, c, sc, s64, qmax, rescan);
  if (rescan) act_fix_chunk<kStatic, 4, true>(hv, c, sc, s64, qmax, rescan);
  return pack4(c[0], c[1], c[2], c[3]);
}

template <int V, int W, bool kStatic, bool kGather>
int launch_act_reg_t(const uint16_t* x, int64_t m, int k, int64_t ldx, const int32_t* gather, int k_out,
                     double static_scale, int qmax, int8_t* q, int64_t ldq, float* s32, double* s64,
                     unsigned long long* err, cudaStream_t stream) {
  constexpr int kTeams = W == 1 ? 8 : 1;
  constexpr int kThreads = W == 1 ? 256 : 32 * W;
  auto kern = quant_act_reg_kernel<V, W, kStatic, kGather>;
  const size_t smem =
      kGather ? static_cast<size_t>(kTeams) * ((k + 8 + 63) & ~63) * 2 + static_cast<size_t>((k_out + 7) & ~7) * 2 +
                    static_cast<size_t>((k_out + 7) / 8) * 2
              : 0;
  static std::once_flag once;
  static cudaError_t attr = cudaSuccess;
  std::call_once(once, [&] { attr = set_smem_attrs(kern, 64 * 1024); });
  QARVD_CUDA_TRY(attr);
  const int64_t grid = (m + kTeams - 1) / kTeams;
  QARVD_CUDA_TRY(launch_pdl(kern, dim3(static_cast<unsigned>(grid)), dim3(kThreads), smem, stream, 1, x, m, k,
                            ldx, gather, k_out, static_scale, qmax, 1.0 / static_cast<double>(qmax), q, ldq, s32,
                            s64, err));
  return QARVD_OK;
}

// (V chunks per thread, W warps per team) of a row of nvec 16-byte chunks, or {0, 0}
inline void k1_reg_shape(int nvec, int& V, int& W) {
  V = W = 0;
  if (nvec % 32 == 0 && nvec / 32 <= 8) {
    V = nvec / 32;
    W = 1;
    return;
  }
  for (int w = 8; w >= 2; --w)
    if (nvec % (32 * w) == 0 && nvec / (32 * w) <= 8) {
      V = nvec / (32 * w);
      W = w;
      return;
    }
}

template <bool kStatic, bool kGather>
int launch_act_reg(const uint16_t* x, int64_t m, int k, int64_t ldx, const int32_t* gather, int k_out,
                   double static_scale, int qmax, int8_t* q, int64_t ldq, float* s32, double* s64,
                   unsigned long long* err, cudaStream_t stream) {
  int V, W;
  k1_reg_shape(k / 8, V, W);
  switch (W * 16 + V) {
#define QARVD_K1R_CASE(WW, VV) \
  case WW * 16 + VV:           \
    return launch_act_reg_t<VV, WW, kStatic, kGather>(x, m, k, ldx, gather, k_out, static_scale, qmax, q, ldq, s32, s64, err, stream);
    QARVD_K1R_CASE(1, 1) QARVD_K1R_CASE(1, 2) QARVD_K1R_CASE(1, 3) QARVD_K1R_CASE(1, 4)
    QARVD_K1R_CASE(1, 5) QARVD_K1R_CASE(1, 6) QARVD_K1R_CASE(1, 7) QARVD_K1R_CASE(1, 8)
    QARVD_K1R_CASE(4, 3) QARVD_K1R_CASE(4, 4) QARVD_K1R_CASE(4, 5) QARVD_K1R_CASE(4, 6)
    QARVD_K1R_CASE(5, 5) QARVD_K1R_CASE(5, 6) QARVD_K1R_CASE(6, 5) QARVD_K1R_CASE(6, 6)
    QARVD_K1R_CASE(7, 4) QARVD_K1R_CASE(7, 5) QARVD_K1R_CASE(7, 6) QARVD_K1R_CASE(8, 4)
    QARVD_K1R_CASE(8, 5) QARVD_K1R_CASE(8, 6) QARVD_K1R_CASE(8, 7) QARVD_K1R_CASE(8, 8)
#undef QARVD_K1R_CASE
  }
  return -1;  // no register shape: the caller takes the slot-ring kernel
}

// ---------------------------------------------------------------------------
// K1, bulk-staged variant (opt-in, QARVD_K1_BULK=1): persistent CTAs of 256 threads; a
// team (one warp for rows of < 4096 values, eight teams per CTA; else the whole CTA) owns
// every nteams-th row and keeps S of its rows in flight as 1-D bulk copies (cp.async.bulk,
// mbarrier completion) into shared-memory slots.  Registers no longer bound the bytes in
// flight (the register kernel held one row per team: 0.3-0.47 of HBM, long_scoreboard), and
// there is no per-row CTA launch.  Per row: |x| max from the slot (team reduction), the row
// scale, then the codes from the slot (plan order: 8 per lane per step; with a gather: 4
// per lane through the staged int16 table, the slot's 8 trailing zero sentinels serving the
// pad columns) -- same arithmetic, tie repair and error reporting as the register kernel.
template <int TW>
struct K1Bulk {
  static constexpr int kThreads = 256;
  static constexpr int kTeams = kThreads / (32 * TW);
  static __host__ __device__ int slot_stride(int k) { return (k * 2 + 16 + 127) & ~127; }  // bytes
};

template <int TW, int S, bool kStatic, bool kGather>
__global__ void __launch_bounds__(256)
    quant_act_bulk_kernel(const uint16_t* __restrict__ x, int64_t m, int k, int64_t ldx,
                          const int32_t* __restrict__ gather, int k_out, double static_scale, int qmax,
                          double rqmax, int8_t* __restrict__ q, int64_t ldq, float* __restrict__ s32_out,
                          double* __restrict__ s64_out, unsigned long long* __restrict__ err) {
  using B = K1Bulk<TW>;
  constexpr int T = 32 * TW;
  extern __shared__ __align__(128) uint8_t k1b_smem[];
  __shared__ __align__(8) uint64_t full[B::kTeams][S];
  __shared__ uint32_t wmax[TW];
  const int stride = B::slot_stride(k);
  const int team = static_cast<int>(threadIdx.x) / T, tt = static_cast<int>(threadIdx.x) % T;
  const int lane = threadIdx.x & 31, warp = tt >> 5;
  uint8_t* slots = k1b_smem + team * S * stride;
  int16_t* gidx = reinterpret_cast<int16_t*>(k1b_smem + B::kTeams * S * stride);
  if (threadIdx.x < B::kTeams * S) ptx::mbar_init(&full[threadIdx.x / S][threadIdx.x % S], 1);
  // zero sentinels after every slot's row (the bulk copies never write them)
  for (int i = threadIdx.x; i < B::kTeams * S; i += blockDim.x)
    *reinterpret_cast<uint4*>(k1b_smem + i * stride + k * 2) = make_uint4(0u, 0u, 0u, 0u);
  if (kGather) {
    for (int c4 = threadIdx.x; c4 < (k_out >> 2); c4 += blockDim.x) {
      const int4 g = __ldg(reinterpret_cast<const int4*>(gather) + c4);
      reinterpret_cast<uint2*>(gidx)[c4] =
          make_uint2(static_cast<uint16_t>(g.x < 0 ? k : g.x) | (static_cast<uint32_t>(g.y < 0 ? k : g.y) << 16),
                     static_cast<uint16_t>(g.z < 0 ? k : g.z) | (static_cast<uint32_t>(g.w < 0 ? k : g.w) << 16));
    }
  }
  ptx::fence_mbar_init();
  __syncthreads();
  pdl_wait();  // x is written by the previous kernel of the chain
  pdl_launch_dependents();
  const int64_t nteams = static_cast<int64_t>(gridDim.x) * B::kTeams;
  const int64_t team_id = static_cast<int64_t>(blockIdx.x) * B::kTeams + team;
  const uint32_t row_bytes = static_cast<uint32_t>(k) * 2u;
  const bool producer = tt == 0;
  if (producer) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int64_t row = team_id + s * nteams;
      if (row < m) {
        ptx::mbar_expect_tx(&full[team][s], row_bytes);
        ptx::bulk_load_1d(slots + s * stride, x + row * ldx, row_bytes, &full[team][s]);
      }
    }
  }
  const int nvec = k >> 3;
  ActScale sc;
  sc.fq = static_cast<float>(qmax);
  for (int i = 0;; ++i) {
    const int64_t row = team_id + static_cast<int64_t>(i) * nteams;
    if (row >= m) break;
    const int s = i % S;
    ptx::mbar_wait(&full[team][s], static_cast<uint32_t>((i / S) & 1));
    const uint16_t* srow = reinterpret_cast<const uint16_t*>(slots + s * stride);
    const uint4* srow4 = reinterpret_cast<const uint4*>(srow);
    uint32_t mx = 0;
    for (int c = tt; c < nvec; c += T) {
      const uint4 d = srow4[c];
      mx = __vmaxu2(mx, __vmaxu2(__vmaxu2(d.x & 0x7fff7fffu, d.y & 0x7fff7fffu),
                                 __vmaxu2(d.z & 0x7fff7fffu, d.w & 0x7fff7fffu)));
    }
    uint32_t mag = __reduce_max_sync(0xffffffffu, max(mx & 0xffffu, mx >> 16));
    if (TW > 1) {
      if (lane == 0) wmax[warp] = mag;
      __syncthreads();
#pragma unroll
      for (int w = 0; w < TW; ++w) mag = max(mag, wmax[w]);
    }
    const bool row_bad = mag >= 0x7f80u;
    const float amax = __uint_as_float(mag << 16);
    double s64;
    if (kStatic) {
      const GroupScale g = scale_static(static_scale);
      sc.r = g.r32;
      sc.exact = g.exact;
      s64 = static_scale;
    } else {  // r = fl(fl(1/amax) * qmax), s64 = fl64(amax / qmax): see quant_act_rows_kernel
      sc.r = amax > 0.f ? __fmul_rn(__frcp_rn(amax), static_cast<float>(qmax)) : 0.f;
      sc.exact = amax > 0.f && !(sc.r <= FLT_MAX && sc.r >= FLT_MIN);
      if (!(amax > 0.f)) {
        s64 = DBL_MIN;
      } else {
        const double a = static_cast<double>(amax), y = a * rqmax;
        s64 = fma(fma(-y, static_cast<double>(qmax), a), rqmax, y);
      }
    }
    sc.s64 = s64;
    if (tt == T - 1) {
      if (s32_out) s32_out[row] = (kStatic || amax > 0.f) ? __double2float_rn(s64) : 0.f;
      if (s64_out) s64_out[row] = s64;
    }
    int8_t* qr = q + row * ldq;
    const bool slow = row_bad || sc.exact;  // rare rows: non-finite input (reported) or no usable fp32 reciprocal
    if (!kGather) {
      for (int c = tt; c < nvec; c += T) {
        const uint4 d = srow4[c];
        const uint32_t w[4] = {d.x, d.y, d.z, d.w};
        uint32_t cd[8];
        if (slow) {
#pragma unroll
          for (int h = 0; h < 8; ++h)
            cd[h] = act_code_slow(static_cast<uint16_t>(h & 1 ? w[h >> 1] >> 16 : w[h >> 1] & 0xffffu), s64, qmax,
                                  err, row * k_out + c * 8 + h);
        } else {
          float dmax = 0.f;
#pragma unroll
          for (int h = 0; h < 4; ++h)
            act_codes2<kStatic>(__uint_as_float(w[h] << 16), __uint_as_float(w[h] & 0xffff0000u), sc, cd[2 * h],
                                cd[2 * h + 1], dmax);
          if (dmax > tie_guard<kStatic>()) {  // a value within the tie guard: decide exactly
            *reinterpret_cast<uint2*>(qr + c * 8) = act_fix8_reg<1, 1, kStatic, false>(d, sc, s64, qmax);
            continue;
          }
        }
        *reinterpret_cast<uint2*>(qr + c * 8) =
            make_uint2(pack4(cd[0], cd[1], cd[2], cd[3]), pack4(cd[4], cd[5], cd[6], cd[7]));
      }
    } else {
      for (int c0 = tt * 4; c0 < k_out; c0 += T * 4) {
        const uint2 gp = *reinterpret_cast<const uint2*>(gidx + c0);
        const uint16_t hv[4] = {srow[gp.x & 0xffffu], srow[gp.x >> 16], srow[gp.y & 0xffffu], srow[gp.y >> 16]};
        uint32_t cd[4];
        if (slow) {
#pragma unroll
          for (int e = 0; e < 4; ++e) cd[e] = act_code_slow(hv[e], s64, qmax, err, row * k_out + c0 + e);
        } else {
          float dmax = 0.f;
          act_codes2<kStatic>(__uint_as_float(static_cast<uint32_t>(hv[0]) << 16),
                              __uint_as_float(static_cast<uint32_t>(hv[1]) << 16), sc, cd[0], cd[1], dmax);
          act_codes2<kStatic>(__uint_as_float(static_cast<uint32_t>(hv[2]) << 16),
                              __uint_as_float(static_cast<uint32_t>(hv[3]) << 16), sc, cd[2], cd[3], dmax);
          if (dmax > tie_guard<kStatic>()) {
            *reinterpret_cast<uint32_t*>(qr + c0) =
                act_fix4_reg<kStatic>(make_uint2(hv[0] | (static_cast<uint32_t>(hv[1]) << 16),
                                                 hv[2] | (static_cast<uint32_t>(hv[3]) << 16)), sc, s64, qmax);
            continue;
          }
        }
        *reinterpret_cast<uint32_t*>(qr + c0) = pack4(cd[0], cd[1], cd[2], cd[3]);
      }
    }
    // the slot is free once the whole team has read it: refill it with the team's row i + S
    if (TW > 1) __syncthreads();
    else __syncwarp();
    const int64_t next = row + S * nteams;
    if (producer && next < m) {
      ptx::fence_proxy_async_smem();  // generic-proxy reads of the slot before the async write
      ptx::mbar_expect_tx(&full[team][s], row_bytes);
      ptx::bulk_load_1d(slots + s * stride, x + next * ldx, row_bytes, &full[team][s]);
    }
  }
}

template <int TW, int S, bool kStatic, bool kGather>
int launch_act_bulk_t(const uint16_t* x, int64_t m, int k, int64_t ldx, const int32_t* gather, int k_out,
                      double static_scale, int qmax, int8_t* q, int64_t ldq, float* s32, double* s64,
                      unsigned long long* err, cudaStream_t stream) {
  using B = K1Bulk<TW>;
  auto kern = quant_act_bulk_kernel<TW, S, kStatic, kGather>;
  const size_t smem = static_cast<size_t>(B::kTeams) * S * B::slot_stride(k) +
                      (kGather ? static_cast<size_t>((k_out + 7) & ~7) * 2 : 0);
  static std::once_flag once;
  static cudaError_t attr = cudaSuccess;
  static int per_sm = 1, sms = kNumSMs;
  std::call_once(once, [&] {
    attr = set_smem_attrs(kern, 200 * 1024);
    if (attr == cudaSuccess) attr = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, B::kThreads, smem);
    int dev = 0;
    if (attr == cudaSuccess) attr = cudaGetDevice(&dev);
    if (attr == cudaSuccess) attr = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  });
  QARVD_CUDA_TRY(attr);
  const int64_t teams = (m + B::kTeams - 1) / B::kTeams;
  const int64_t grid = std::min<int64_t>(teams, static_cast<int64_t>(sms) * std::max(per_sm, 1));
  QARVD_CUDA_TRY(launch_pdl(kern, dim3(static_cast<unsigned>(grid)), dim3(B::kThreads), smem, stream, 1, x, m,
                            k, ldx, gather, k_out, static_scale, qmax, 1.0 / static_cast<double>(qmax), q, ldq,
                            s32, s64, err));
  return QARVD_OK;
}

// bulk-staged K1: rows of >= 4096 values as whole-CTA teams with 4 slots (3 CTAs per SM at
// K = 8960), shorter rows as warp teams with 3 slots each
template <bool kStatic, bool kGather>
int launch_act_bulk(const uint16_t* x, int64_t m, int k, int64_t ldx, const int32_t* gather, int k_out,
                    double static_scale, int qmax, int8_t* q, int64_t ldq, float* s32, double* s64,
                    unsigned long long* err, cudaStream_t stream) {
  if (k >= 4096)
    return launch_act_bulk_t<8, 4, kStatic, kGather>(x, m, k, ldx, gather, k_out, static_scale, qmax, q, ldq, s32,
                                                     s64, err, stream);
  return launch_act_bulk_t<1, 3, kStatic, kGather>(x, m, k, ldx, gather, k_out, static_scale, qmax, q, ldq, s32,
                                                   s64, err, stream);
}

template <bool kStatic>
int launch_act_rows(bool gathered, const uint16_t* x, int64_t m, int k, int64_t ldx,
                    const int32_t* gather, int k_out, double static_scale, int qmax, int8_t* q,
                    int64_t ldq, float* s32, double* s64, unsigned long long* err,
                    cudaStream_t stream) {
  // register-resident K1 for every row shape it covers (round 2, after the tie repair became the
  // plain division and gathered rows quantize in natural order before the gather: U 34.5 us,
  // gathered 4680 x 1536 16.4 us vs the slot ring's 18.4; scripts/k1_flush_probe.py).
  // QARVD_K1_REG=0 / =1: never / plan-order rows only.
  // QARVD_K1_BULK=1: the bulk-staged kernel (opt-in: measured slower on the Wan shapes, x 23.6 vs
  // 17.4 us and U 37.7 vs 33.8 us under the bench's L2 flush, scripts/k1_flush_probe.py -- it
  // issues ~12 instructions per value and stays issue-bound with the bytes in flight solved)
  const int bulk = getenv("QARVD_K1_BULK") ? atoi(getenv("QARVD_K1_BULK")) : 0;  // per call (tests A/B it)
  const int64_t bulk_smem = static_cast<int64_t>(k >= 4096 ? 4 : 8 * 3) * K1Bulk<1>::slot_stride(k) +
                            (gathered ? ((k_out + 7) & ~7) * 2 : 0);
  if (bulk > 0 && (!gathered || k_out % 4 == 0) && bulk_smem <= 200 * 1024)
    return gathered ? launch_act_bulk<kStatic, true>(x, m, k, ldx, gather, k_out, static_scale, qmax, q, ldq, s32,
                                                     s64, err, stream)
                    : launch_act_bulk<kStatic, false>(x, m, k, ldx, gather, k_out, static_scale, qmax, q, ldq, s32,
                                                      s64, err, stream);
  static const int reg = getenv("QARVD_K1_REG") ? atoi(getenv("QARVD_K1_REG")) : 2;
  if (reg > 0 && (!gathered || (reg == 2 && k_out % 8 == 0 && ldq % 8 == 0))) {
    const int st = gathered ? launch_act_reg<kStatic, true>(x, m, k, ldx, gather, k_out, static_scale, qmax, q,
                                                            ldq, s32, s64, err, stream)
                            : launch_act_reg<kStatic, false>(x, m, k, ldx, gather, k_out, static_scale, qmax, q,
                                                             ldq, s32, s64, err, stream);
    if (st >= 0) return st;
  }
  return gathered ? launch_act_rows_g<kStatic, true>(x, m, k, ldx, gather, k_out, static_scale, qmax, q,
                                                     ldq, s32, s64, err, stream)
                  : launch_act_rows_g<kStatic, false>(x, m, k, ldx, gather, k_out, static_scale, qmax,
                                                      q, ldq, s32, s64, err, stream);
}

template <int MODE>
int launch_rows(const void* x, int dtype, int64_t m, int64_t k, int64_t ldx, const int32_t* gather,
                int64_t k_out, int64_t k_o, double static_scale, int bits, int8_t* q, int64_t ldq,
                float* s32_o, double* s64_o, float* s32_n, double* s64_n, int64_t* err_index,
                cudaStream_t stream) {
  const int qmax = (1 << (bits - 1)) - 1;
  unsigned long long* err = reinterpret_cast<unsigned long long*>(err_index);
  if (err) {
    init_err_kernel<<<1, 1, 0, stream>>>(err);
    count_launch();
  }
  if (m == 0) return QARVD_OK;
  const int grid = grid_for_rows(m);
  const bool fast_ok = MODE != kWeightDual && dtype == QARVD_BF16 && k <= 32 * kK1Vec * 8 * 8 &&
                       (k % 8) == 0 && (ldx % 8) == 0 && (k_out % 16) == 0 && (ldq % 16) == 0 &&
                       (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                       (reinterpret_cast<uintptr_t>(q) & 15) == 0 &&
                       (reinterpret_cast<uintptr_t>(gather) & 15) == 0;
  // shared memory of the team slots (+ int16 permutation table) must fit the 110 KB opt-in
  const int64_t k1_smem = fast_ok ? ((k / 8 <= 256 ? 4 * 1 : 3) * ((k + 8 + 63) & ~int64_t(63)) * 2 +
                                     (gather ? ((k_out + 7) & ~int64_t(7)) * 2 : 0))
                                  : 0;
  if (fast_ok && k1_smem <= 110 * 1024) {
    if (int st = launch_act_rows<MODE == kActStatic>(gather != nullptr, static_cast<const uint16_t*>(x), m,
                                                     static_cast<int>(k), ldx, gather,
                                                     static_cast<int>(k_out), static_scale, qmax, q,
                                                     ldq, s32_n, s64_n, err, stream))
      return st;
  } else if (dtype == QARVD_BF16 && k <= kMaxSmemK) {
    const size_t smem = static_cast<size_t>(kWarpsPerCta) * (((k + 7) & ~int64_t(7)) * 2);
    static std::once_flag once;
    static cudaError_t attr = cudaSuccess;
    std::call_once(once, [] {
      attr = set_smem_attrs(quant_rows_bf16_kernel<MODE>, kWarpsPerCta * kMaxSmemK * 2);
    });
    QARVD_CUDA_TRY(attr);
    quant_rows_bf16_kernel<MODE><<<grid, kWarpsPerCta * 32, smem, stream>>>(
        static_cast<const uint16_t*>(x), m, k, ldx, gather, k_out, k_o, static_scale, qmax, q,
        ldq, s32_o, s64_o, s32_n, s64_n, err);
  } else if (dtype == QARVD_BF16) {
    quant_rows_generic_kernel<MODE, uint16_t><<<grid, kWarpsPerCta * 32, 0, stream>>>(
        static_cast<const uint16_t*>(x), m, k, ldx, gather, k_out, k_o, static_scale, qmax, q,
        ldq, s32_o, s64_o, s32_n, s64_n, err);
  } else if (dtype == QARVD_F32) {
    quant_rows_generic_kernel<MODE, float><<<grid, kWarpsPerCta * 32, 0, stream>>>(
        static_cast<const float*>(x), m, k, ldx, gather, k_out, k_o, static_scale, qmax, q, ldq,
        s32_o, s64_o, s32_n, s64_n, err);
  } else {
    quant_rows_generic_kernel<MODE, double><<<grid, kWarpsPerCta * 32, 0, stream>>>(
        static_cast<const double*>(x), m, k, ldx, gather, k_out, k_o, static_scale, qmax, q, ldq,
        s32_o, s64_o, s32_n, s64_n, err);
  }
  count_launch();
  QARVD_LAUNCH_CHECK();
  return QARVD_OK;
}

int check_common(const void* x, int dtype, int64_t m, int64_t k, int64_t ldx, int64_t k_out,
                 int bits, const int8_t* q, int64_t ldq, const int32_t* gather) {
  if (bits < 2 || bits > 8)
    QARVD_FAIL(QARVD_ERR_UNSUPPORTED,
               "bit width out of the int8 storage range [2,8]: " + std::to_string(bits));
  if (dtype != QARVD_BF16 && dtype != QARVD_F32 && dtype != QARVD_F64)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "unknown input dtype");
  if (m < 0 || k <= 0 || k_out <= 0 || ldx < k || ldq < k_out)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "invalid shape or leading dimension");
  if (!gather && k_out != k)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT,
               "permute_activations: plan does not match activation width");
  if ((m > 0) && (!x || !q)) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "null pointer argument");
  return QARVD_OK;
}

}  // namespace
}  // namespace qarvd_b200

using namespace qarvd_b200;

extern "C" int qarvd_quantize_act(const void* x, int x_dtype, int64_t m, int64_t k, int64_t ldx,
                                  const int32_t* gather, int64_t k_out, int granularity,
                                  double static_scale, int bits, int8_t* xq, int64_t ldq,
                                  float* scale_f32, double* scale_f64, int64_t* err_index,
                                  void* stream) {
  clear_error();
  if (int st = check_common(x, x_dtype, m, k, ldx, k_out, bits, xq, ldq, gather)) return st;
  if (granularity == QARVD_ACT_PER_TENSOR) {
    if (!(static_scale > 0.0) || !(static_scale <= DBL_MAX))
      QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "quant params: scale must be positive and finite");
  } else if (granularity != QARVD_ACT_PER_TOKEN) {
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "unknown activation granularity");
  }
  if (int st = require_device()) return st;
  if (granularity == QARVD_ACT_PER_TOKEN)
    return launch_rows<kActPerToken>(x, x_dtype, m, k, ldx, gather, k_out, 0, 0.0, bits, xq, ldq,
                                     nullptr, nullptr, scale_f32, scale_f64, err_index,
                                     as_stream(stream));
  return launch_rows<kActStatic>(x, x_dtype, m, k, ldx, gather, k_out, 0, static_scale, bits, xq,
                                 ldq, nullptr, nullptr, scale_f32, scale_f64, err_index,
                                 as_stream(stream));
}

extern "C" int qarvd_prepare_weights(const void* w, int w_dtype, int64_t n, int64_t k, int64_t ldw,
                                     const int32_t* gather, int64_t k_pad, int64_t k_outlier,
                                     int bits, int8_t* wq, int64_t ldq, double* scale_outlier_f64,
                                     double* scale_normal_f64, float* scale_outlier_f32,
                                     float* scale_normal_f32, int64_t* err_index, void* stream) {
  clear_error();
  if (int st = check_common(w, w_dtype, n, k, ldw, k_pad, bits, wq, ldq, gather)) return st;
  if (k_outlier < 0 || k_outlier >= k_pad)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT,
               "build_plan: outlier set would leave no normal channels");
  if (int st = require_device()) return st;
  return launch_rows<kWeightDual>(w, w_dtype, n, k, ldw, gather, k_pad, k_outlier, 0.0, bits, wq,
                                  ldq, scale_outlier_f32, scale_outlier_f64, scale_normal_f32,
                                  scale_normal_f64, err_index, as_stream(stream));
}

extern "C" int qarvd_quantize_act_rowmax(const uint16_t* x, int64_t m, int64_t k, int64_t ldx,
                                         uint32_t* row_absmax, int granularity,
                                         double static_scale, int bits, int8_t* xq, int64_t ldq,
                                         float* scale_f32, double* scale_f64, int64_t* err_index,
                                         void* stream) {
  clear_error();
  if (bits < 2 || bits > 8)
    QARVD_FAIL(QARVD_ERR_UNSUPPORTED, "bit width out of the int8 storage range [2,8]: " + std::to_string(bits));
  if (m < 0 || k <= 0 || ldx < k || ldq < k)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "invalid shape or leading dimension");
  if (k % 8 || ldx % 8 || ldq % 8 || (reinterpret_cast<uintptr_t>(x) & 15) ||
      (reinterpret_cast<uintptr_t>(xq) & 7))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT,
               "quantize (rowmax): k, ldx, ldq must be multiples of 8 and x 16-byte aligned");
  if (m > 0 && (!x || !xq)) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "null pointer argument");
  if (granularity == QARVD_ACT_PER_TENSOR) {
    if (!(static_scale > 0.0) || !(static_scale <= DBL_MAX))
      QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "quant params: scale must be positive and finite");
  } else if (granularity == QARVD_ACT_PER_TOKEN) {
    if (!row_absmax) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "quantize (rowmax): null row |x| max buffer");
  } else {
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "unknown activation granularity");
  }
  if (int st = require_device()) return st;
  cudaStream_t s = as_stream(stream);
  const int qmax = (1 << (bits - 1)) - 1;
  unsigned long long* err = reinterpret_cast<unsigned long long*>(err_index);
  if (err) {
    init_err_kernel<<<1, 1, 0, s>>>(err);
    count_launch();
  }
  if (m == 0) return QARVD_OK;
  const int64_t cap = static_cast<int64_t>(kNumSMs) * 4;
  const unsigned grid = static_cast<unsigned>(m < cap ? m : cap);
  const bool ring = granularity == QARVD_ACT_PER_TOKEN && k / 8 > 256 &&
                    4 * ((k + 8 + 63) & ~int64_t(63)) * 2 <= 110 * 1024 &&
                    !getenv("QARVD_K1_STREAM");  // diagnostics: force the streaming kernel
  if (ring) {  // (launches through launch_pdl)
    if (int st = launch_act_rowmax(x, m, static_cast<int>(k), ldx, row_absmax, qmax, xq, ldq,
                                   scale_f32, scale_f64, err, s))
      return st;
  } else if (granularity == QARVD_ACT_PER_TOKEN) {
    QARVD_CUDA_TRY(launch_pdl(quant_act_stream_kernel<false>, dim3(grid), dim3(kStreamThreads), 0, s, 1,
                              x, m, static_cast<int>(k), ldx, row_absmax, 0.0, qmax, 1.0 / qmax, xq,
                              ldq, scale_f32, scale_f64, err));
  } else {
    QARVD_CUDA_TRY(launch_pdl(quant_act_stream_kernel<true>, dim3(grid), dim3(kStreamThreads), 0, s, 1,
                              x, m, static_cast<int>(k), ldx, static_cast<uint32_t*>(nullptr),
                              static_scale, qmax, 1.0 / qmax, xq, ldq, scale_f32, scale_f64, err));
  }
  count_launch();
  QARVD_LAUNCH_CHECK();
  return QARVD_OK;
}

extern "C" int qarvd_quantize_act_pmax(const uint16_t* x, int64_t m, int64_t k, int64_t ldx,
                                       const uint32_t* row_pmax, int64_t pm_count, int granularity,
                                       double static_scale, int bits, int8_t* xq, int64_t ldq,
                                       float* scale_f32, double* scale_f64, int64_t* err_index,
                                       void* stream) {
  clear_error();
  if (bits < 2 || bits > 8)
    QARVD_FAIL(QARVD_ERR_UNSUPPORTED, "bit width out of the int8 storage range [2,8]: " + std::to_string(bits));
  if (m < 0 || k <= 0 || ldx < k || ldq < k)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "invalid shape or leading dimension");
  if (k % 8 || k < 512 || ldx % 8 || ldq % 8 || (reinterpret_cast<uintptr_t>(x) & 15) ||
      (reinterpret_cast<uintptr_t>(xq) & 7))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT,
               "quantize (pmax): k >= 512; k, ldx, ldq multiples of 8; x 16-byte aligned");
  if (m > 0 && (!x || !xq)) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "null pointer argument");
  if (granularity == QARVD_ACT_PER_TENSOR) {
    if (!(static_scale > 0.0) || !(static_scale <= DBL_MAX))
      QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "quant params: scale must be positive and finite");
  } else if (granularity == QARVD_ACT_PER_TOKEN) {
    if (!row_pmax || pm_count <= 0)
      QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "quantize (pmax): missing row partial maxima");
  } else {
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "unknown activation granularity");
  }
  if (int st = require_device()) return st;
  cudaStream_t s = as_stream(stream);
  const int qmax = (1 << (bits - 1)) - 1;
  unsigned long long* err = reinterpret_cast<unsigned long long*>(err_index);
  if (err) {
    init_err_kernel<<<1, 1, 0, s>>>(err);
    count_launch();
  }
  if (m == 0) return QARVD_OK;
  const int64_t chunks = m * (k / 8);
  const unsigned grid = static_cast<unsigned>((chunks + kFlatSpan - 1) / kFlatSpan);
  if (granularity == QARVD_ACT_PER_TOKEN)
    QARVD_CUDA_TRY(launch_pdl(quant_act_flat_kernel<false>, dim3(grid), dim3(kFlatThreads), 0, s, 1, x,
                              m, static_cast<int>(k), ldx, row_pmax, static_cast<int>(pm_count), 0.0,
                              qmax, 1.0 / qmax, xq, ldq, scale_f32, scale_f64, err));
  else
    QARVD_CUDA_TRY(launch_pdl(quant_act_flat_kernel<true>, dim3(grid), dim3(kFlatThreads), 0, s, 1, x, m,
                              static_cast<int>(k), ldx, static_cast<const uint32_t*>(nullptr), 0,
                              static_scale, qmax, 1.0 / qmax, xq, ldq, scale_f32, scale_f64, err));
  count_launch();
  QARVD_LAUNCH_CHECK();
  return QARVD_OK;
}

namespace qarvd_b200 {
namespace {
// Launch the batched K5 kernel over bf16 jobs: two launches, rows of <= 2048 values (small
// shared-memory footprint, many CTAs per SM) and the wide rows, each with its own slot size.
int launch_prep_batched(const std::vector<WeightJobDev>& fast, int qmax, unsigned long long* err,
                        cudaStream_t s) {
  static std::once_flag once;
  static cudaError_t attr = cudaSuccess;
  std::call_once(once, [] {
    attr = set_smem_attrs(prep_weights_batched_kernel<1, kWTeams>, 200 * 1024);
    if (attr == cudaSuccess) attr = set_smem_attrs(prep_weights_batched_kernel<8, 1>, 200 * 1024);
  });
  QARVD_CUDA_TRY(attr);
  for (int group = 0; group < 2; ++group) {
    std::vector<WeightJobDev> sel;
    int64_t g_n = 0, g_k = 0, g_kp = 0;
    for (const WeightJobDev& jd : fast)
      if ((jd.k <= 2048) == (group == 0)) {
        sel.push_back(jd);
        g_n = jd.n > g_n ? jd.n : g_n;
        g_k = jd.k > g_k ? jd.k : g_k;
        g_kp = jd.k_pad > g_kp ? jd.k_pad : g_kp;
      }
    if (sel.empty() || g_n == 0) continue;
    WeightJobDev* d_jobs = nullptr;
    const size_t bytes = sel.size() * sizeof(WeightJobDev);
    QARVD_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&d_jobs), bytes, s));
    QARVD_CUDA_TRY(cudaMemcpyAsync(d_jobs, sel.data(), bytes, cudaMemcpyHostToDevice, s));
    // group 0: warp teams (kWTeams per CTA); group 1 (wide rows): one 8-warp team per CTA
    const int teams = group == 0 ? kWTeams : 1, threads = group == 0 ? 32 * kWTeams : 256;
    // row slots, the int16 gather (k_pad values of the widest job, as the kernel lays it out per
    // job) and the outlier-column bitmask
    size_t smem = static_cast<size_t>(teams) * 2 * ((g_k + 8 + 63) & ~int64_t(63)) * 2 + ((g_kp + 7) & ~int64_t(7)) * 2 +
                  static_cast<size_t>((g_k + 31) / 32) * 4;
    if (smem > 200 * 1024) QARVD_FAIL(QARVD_ERR_LOGIC, "prepare_weights_batched: rows too wide");
    // enough CTAs per layer to fill the GPU a few times over, rows strided across teams
    int64_t gx = (g_n + teams - 1) / teams;
    const int64_t cap = (static_cast<int64_t>(kNumSMs) * 16 + static_cast<int64_t>(sel.size()) - 1) /
                        static_cast<int64_t>(sel.size());
    gx = gx < cap ? gx : (cap < 1 ? 1 : cap);
    static const cudaError_t carve_prep = prefer_max_shared(prep_weights_batched_kernel<1, kWTeams>) == cudaSuccess
                                              ? prefer_max_shared(prep_weights_batched_kernel<8, 1>)
                                              : cudaErrorInvalidValue;
    QARVD_CUDA_TRY(carve_prep);
    if (group == 0)
      prep_weights_batched_kernel<1, kWTeams><<<dim3(static_cast<unsigned>(gx), static_cast<unsigned>(sel.size())),
                                                threads, smem, s>>>(d_jobs, qmax, 1.0 / qmax, err);
    else
      prep_weights_batched_kernel<8, 1><<<dim3(static_cast<unsigned>(gx), static_cast<unsigned>(sel.size())),
                                          threads, smem, s>>>(d_jobs, qmax, 1.0 / qmax, err);
    count_launch();
    QARVD_LAUNCH_CHECK();
    QARVD_CUDA_TRY(cudaFreeAsync(d_jobs, s));
  }
  return QARVD_OK;
}
}  // namespace
}  // namespace qarvd_b200

namespace qarvd_b200 {
namespace {
struct PlanJobDev {
  int64_t k;
  const int32_t* aligned;
  const int32_t* counts;
  int32_t* gather;
  int64_t gather_cap;
  int64_t* plan_info;
};
// build_plan's column split on the device (engine.build_plan / dual_scale.cpp:44-90): gather =
// [aligned outliers ascending | -1 to a multiple of 32 | normal columns ascending | -1 ...],
// plan_info = {k_outlier, k_pad}; an empty outlier set is the single-scale identity plan.
constexpr int kPlanThreads = 256;
__global__ void __launch_bounds__(kPlanThreads) build_plan_kernel(const PlanJobDev* __restrict__ jobs) {
  const PlanJobDev J = jobs[blockIdx.x];
  __shared__ uint32_t mask[10240 / 32 + 1];
  __shared__ uint32_t pre[10240 / 32 + 1];  // outliers below each 32-column word
  const int k = static_cast<int>(J.k), words = (k + 31) / 32;
  const int n_o = J.counts[1];
  for (int w = threadIdx.x; w < words; w += kPlanThreads) mask[w] = 0u;
  __syncthreads();
  for (int i = threadIdx.x; i < n_o; i += kPlanThreads) {
    const int c = J.aligned[i];
    atomicOr(&mask[c >> 5], 1u << (c & 31));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t acc = 0;
    for (int w = 0; w < words; ++w) {
      pre[w] = acc;
      acc += __popc(mask[w]);
    }
  }
  __syncthreads();
  const int k_o = n_o > 0 ? (n_o + 31) / 32 * 32 : 0;
  const int k_pad = k_o + (k - n_o + 31) / 32 * 32;
  for (int i = threadIdx.x; i < J.gather_cap; i += kPlanThreads) {
    int g = -1;
    if (i < n_o) g = J.aligned[i];
    J.gather[i] = g;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += kPlanThreads) {
    const uint32_t m = mask[c >> 5];
    if (!((m >> (c & 31)) & 1u)) {
      const int below = static_cast<int>(pre[c >> 5]) + __popc(m & ((1u << (c & 31)) - 1u));
      J.gather[k_o + c - below] = c;
    }
  }
  if (threadIdx.x == 0) {
    J.plan_info[0] = k_o;
    J.plan_info[1] = k_pad;
  }
  pdl_launch_dependents();
}
}  // namespace
}  // namespace qarvd_b200

extern "C" int qarvd_prepare_weights_planned(const qarvd_planned_weight_job* jobs, int num_jobs, int bits,
                                             int64_t* err_index, void* stream) {
  clear_error();
  if (num_jobs < 0 || (num_jobs > 0 && !jobs))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "prepare_weights_planned: invalid job table");
  if (bits < 2 || bits > 8)
    QARVD_FAIL(QARVD_ERR_UNSUPPORTED, "bit width out of the int8 storage range [2,8]: " + std::to_string(bits));
  if (num_jobs == 0) return QARVD_OK;
  std::vector<PlanJobDev> plans;
  std::vector<WeightJobDev> fast;
  for (int i = 0; i < num_jobs; ++i) {
    const qarvd_planned_weight_job& j = jobs[i];
    const int64_t need = (j.k + 64 + 15) / 16 * 16;
    if (j.n <= 0 || j.k <= 0 || j.k > 10240 || j.k % 8 || j.ldw < j.k || j.ldw % 8 || !j.w || !j.aligned_idx ||
        !j.counts || !j.gather || !j.plan_info || !j.wq || j.gather_cap < need || j.gather_cap % 4 ||
        j.ldq < need || j.ldq % 4 || (reinterpret_cast<uintptr_t>(j.w) & 15) ||
        (reinterpret_cast<uintptr_t>(j.gather) & 15) || (reinterpret_cast<uintptr_t>(j.wq) & 3))
      QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT,
                 "prepare_weights_planned: bf16 rows of <= 10240 values (k, ldw multiples of 8), "
                 "gather_cap and ldq >= k + 64 (multiples of 4), aligned buffers");
    plans.push_back(PlanJobDev{j.k, j.aligned_idx, j.counts, j.gather, j.gather_cap, j.plan_info});
    fast.push_back(WeightJobDev{static_cast<const uint16_t*>(j.w), j.n, j.k, j.ldw, j.gather, j.gather_cap, 0,
                                j.plan_info, j.wq, j.ldq, j.scale_outlier_f64, j.scale_normal_f64,
                                j.scale_outlier_f32, j.scale_normal_f32});
  }
  if (int st = require_device()) return st;
  cudaStream_t s = as_stream(stream);
  const int qmax = (1 << (bits - 1)) - 1;
  unsigned long long* err = reinterpret_cast<unsigned long long*>(err_index);
  if (err) {
    init_err_kernel<<<1, 1, 0, s>>>(err);
    count_launch();
  }
  PlanJobDev* d_plans = nullptr;
  QARVD_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&d_plans), plans.size() * sizeof(PlanJobDev), s));
  QARVD_CUDA_TRY(cudaMemcpyAsync(d_plans, plans.data(), plans.size() * sizeof(PlanJobDev),
                                 cudaMemcpyHostToDevice, s));
  static const cudaError_t carve_plan = prefer_max_shared(build_plan_kernel);
  QARVD_CUDA_TRY(carve_plan);
  build_plan_kernel<<<static_cast<unsigned>(plans.size()), kPlanThreads, 0, s>>>(d_plans);
  count_launch();
  QARVD_LAUNCH_CHECK();
  QARVD_CUDA_TRY(cudaFreeAsync(d_plans, s));
  return launch_prep_batched(fast, qmax, err, s);
}

extern "C" int qarvd_prepare_weights_batched(const qarvd_weight_job* jobs, int num_jobs, int w_dtype,
                                             int bits, int64_t* err_index, void* stream) {
  clear_error();
  if (num_jobs < 0 || (num_jobs > 0 && !jobs))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "prepare_weights_batched: invalid job table");
  if (bits < 2 || bits > 8)
    QARVD_FAIL(QARVD_ERR_UNSUPPORTED, "bit width out of the int8 storage range [2,8]: " + std::to_string(bits));
  if (num_jobs == 0) return QARVD_OK;
  if (int st = require_device()) return st;
  cudaStream_t s = as_stream(stream);
  const int qmax = (1 << (bits - 1)) - 1;
  unsigned long long* err = reinterpret_cast<unsigned long long*>(err_index);
  if (err) {
    init_err_kernel<<<1, 1, 0, s>>>(err);
    count_launch();
  }
  // jobs the batched bf16 kernel serves; the rest take the per-layer path
  std::vector<WeightJobDev> fast;
  for (int i = 0; i < num_jobs; ++i) {
    const qarvd_weight_job& j = jobs[i];
    if (int st = check_common(j.w, w_dtype, j.n, j.k, j.ldw, j.k_pad, bits, j.wq, j.ldq, j.gather)) return st;
    if (j.k_outlier < 0 || j.k_outlier >= j.k_pad)
      QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "build_plan: outlier set would leave no normal channels");
    const bool ok = w_dtype == QARVD_BF16 && j.gather && j.k % 8 == 0 && j.ldw % 8 == 0 &&
                    j.k_pad % 4 == 0 && j.ldq % 4 == 0 && j.k_outlier % 4 == 0 && j.k <= 10240 &&
                    j.k_pad <= 16384 && (reinterpret_cast<uintptr_t>(j.w) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(j.gather) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(j.wq) & 3) == 0;
    if (ok) {
      fast.push_back(WeightJobDev{static_cast<const uint16_t*>(j.w), j.n, j.k, j.ldw, j.gather, j.k_pad,
                                  j.k_outlier, nullptr, j.wq, j.ldq, j.scale_outlier_f64, j.scale_normal_f64,
                                  j.scale_outlier_f32, j.scale_normal_f32});
    } else if (j.n > 0) {
      if (int st = launch_rows<kWeightDual>(j.w, w_dtype, j.n, j.k, j.ldw, j.gather, j.k_pad, j.k_outlier,
                                            0.0, bits, j.wq, j.ldq, j.scale_outlier_f32, j.scale_outlier_f64,
                                            j.scale_normal_f32, j.scale_normal_f64, nullptr, s))
        return st;
    }
  }
  return launch_prep_batched(fast, qmax, err, s);
}
