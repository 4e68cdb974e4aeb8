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

#include "common.cuh"

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
// Activation fast path (bf16, per-token or static): persistent CTAs stream row
// groups through a 4-stage shared-memory ring filled by TMA bulk copies
// (cp.async.bulk, one per row), so HBM reads overlap the rounding of earlier
// rows.  A group is G rows (G*K*2 ~ 16-24 KB); each row is owned by 8/G warps
// which split its columns, combine their |x| maxima through shared memory,
// then emit 16 codes per lane per step through an int16 gather table.
// Rounding: t = v * (qmax/absmax) in fp32, q = rint(t).  |t - v/s| < 3.1e-5
// for |t| <= 254, so q is the f64 round_half_even(v/s) unless t lies within
// 1e-4 of a half-integer; those (~0.04%) are recomputed with __ddiv_rn.
constexpr int kActThreads = 256;
constexpr int kActStages = 4;

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
      "l"(src), "r"(bytes), "r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
      : "memory");
}
__device__ __forceinline__ void mbar_init_(uint64_t* bar, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
               "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx_(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}

constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: an fp32 add rounds to an integer (RNE)

__device__ __noinline__ int act_code_exact(float v, double s64, int qmax) {
  return quant_code_exact(static_cast<double>(v), s64, qmax);
}

__device__ __forceinline__ uint32_t pack4(uint32_t b0, uint32_t b1, uint32_t b2, uint32_t b3) {
  return __byte_perm(__byte_perm(b0, b1, 0x0040), __byte_perm(b2, b3, 0x0040), 0x5410);
}

template <bool kStatic>
__global__ void __launch_bounds__(kActThreads)
    quant_act_tma_kernel(const uint16_t* __restrict__ x, int64_t m, int k, int64_t ldx,
                         const int32_t* __restrict__ gather, int k_out, int G,
                         double static_scale, int qmax, int8_t* __restrict__ q, int64_t ldq,
                         float* __restrict__ s32_out, double* __restrict__ s64_out,
                         unsigned long long* err, int k1_debug) {
  extern __shared__ __align__(128) uint8_t smem_act[];
  __shared__ long long ktrace[3][32];
  const long long k_entry = clock64();
  unsigned long long g_entry;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_entry));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int row_elems = (k + 1 + 7) & ~7;  // +1: zero sentinel read by pad columns
  const int stage_elems = row_elems * G;
  uint16_t* rows = reinterpret_cast<uint16_t*>(smem_act);
  int16_t* gidx = reinterpret_cast<int16_t*>(rows + kActStages * stage_elems);
  uint64_t* full = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(gidx + ((k_out + 7) & ~7)) + 15) & ~uintptr_t(15));
  uint32_t* part = reinterpret_cast<uint32_t*>(full + kActStages);  // per-warp |x| maxima (bits)

  const int64_t num_groups = (m + G - 1) / G;
  const int W = 8 / G;          // warps per row
  const int my_row = warp / W;  // row inside the group
  const int sub = warp % W;     // column share of this warp

  auto issue = [&](int64_t it, int slot) {
    const int64_t g = blockIdx.x + it * gridDim.x;
    if (g >= num_groups) return;
    const int64_t r0 = g * G;
    const int nr = static_cast<int>((m - r0) < G ? (m - r0) : G);
    const uint32_t bytes = static_cast<uint32_t>(k) * 2u;
    mbar_expect_tx_(&full[slot], bytes * nr);
    for (int r = 0; r < nr; ++r)
      bulk_load(rows + slot * stage_elems + r * row_elems, x + (r0 + r) * ldx, bytes, &full[slot]);
  };
  // the first row groups are requested before anything else, so HBM latency overlaps
  // the gather-table setup (the copies write [0, k) of each row, the sentinel column k
  // and the table are disjoint)
  if (tid == 0) {
    for (int s = 0; s < kActStages; ++s) mbar_init_(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < kActStages; ++s) issue(s, s);
  }
  if (gather && (k_out & 3) == 0 && (reinterpret_cast<uintptr_t>(gather) & 15) == 0) {
#pragma unroll 4
    for (int c4 = tid; c4 < (k_out >> 2); c4 += kActThreads) {
      const int4 gi = __ldg(reinterpret_cast<const int4*>(gather) + c4);
      const int src[4] = {gi.x, gi.y, gi.z, gi.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) gidx[4 * c4 + e] = static_cast<int16_t>(src[e] < 0 ? k : src[e]);
    }
  } else {
    for (int c = tid; c < k_out; c += kActThreads) {
      const int src = gather ? __ldg(gather + c) : c;
      gidx[c] = static_cast<int16_t>(src < 0 ? k : src);
    }
  }
  for (int r = tid; r < kActStages * G; r += kActThreads)
    for (int e = k; e < row_elems; ++e) rows[r * row_elems + e] = 0;
  __syncthreads();

  const int csz = (((k + W - 1) / W) + 7) & ~7;     // source columns per warp (absmax)
  const int osz = (((k_out + W - 1) / W) + 15) & ~15;  // output columns per warp
  const float fq = static_cast<float>(qmax);

  for (int64_t it = 0;; ++it) {
    const int64_t g = blockIdx.x + it * gridDim.x;
    if (g >= num_groups) break;
    const int slot = static_cast<int>(it % kActStages);
    const long long tw0 = clock64();
    mbar_wait_(&full[slot], static_cast<uint32_t>((it / kActStages) & 1));
    if (k1_debug == 2 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1) && tid == 0 && it < 32) {
      ktrace[0][it] = tw0;
      ktrace[1][it] = clock64();
    }
    const int64_t row = g * G + my_row;
    const bool active = row < m;
    const uint16_t* rs = rows + slot * stage_elems + my_row * row_elems;

    // ---- |x| max as packed 16-bit integer max of the sign-cleared bf16 bits;
    //      non-finite values (exponent all ones) are exactly the maxima >= 0x7f80
    uint32_t mx = 0;
    if (active) {
      const int c0 = sub * csz, c1 = min(c0 + csz, k);
      int c = c0 + lane * 8;
      for (; c + 8 <= c1; c += 256) {
        const uint4 d = *reinterpret_cast<const uint4*>(rs + c);
        mx = __vmaxu2(mx, __vmaxu2(__vmaxu2(d.x & 0x7fff7fffu, d.y & 0x7fff7fffu),
                                   __vmaxu2(d.z & 0x7fff7fffu, d.w & 0x7fff7fffu)));
      }
      for (; c < c1; ++c) mx = max(mx, static_cast<uint32_t>(rs[c] & 0x7fffu));
    }
    uint32_t mag = max(mx & 0xffffu, mx >> 16);
    mag = __reduce_max_sync(0xffffffffu, mag);
    if (W > 1) {
      if (lane == 0) part[warp] = mag;
      __syncthreads();
      for (int w = 0; w < W; ++w) mag = max(mag, part[my_row * W + w]);
    }
    const bool row_bad = mag >= 0x7f80u;
    // fp32 reciprocal for the fast path; the f64 scale (a division) only where it is
    // written or where the rare exact path needs it
    const float amax = __uint_as_float(mag << 16);
    GroupScale gsc;
    if (kStatic) {
      gsc = scale_static(static_scale);
    } else {
      gsc.r32 = amax > 0.f ? __fdiv_rn(static_cast<float>(qmax), amax) : 0.f;
      gsc.exact = amax > 0.f && !(gsc.r32 <= FLT_MAX && gsc.r32 >= FLT_MIN);
      gsc.s64 = 0.0;
      gsc.s32 = 0.f;
    }
    auto row_s64 = [&]() -> double {
      return kStatic ? static_scale
                     : (amax > 0.f ? __ddiv_rn(static_cast<double>(amax), static_cast<double>(qmax))
                                   : DBL_MIN);
    };
    if (active && sub == 0 && lane == 0) {
      const double s64 = row_s64();
      if (s32_out) s32_out[row] = amax > 0.f || kStatic ? __double2float_rn(s64) : 0.f;
      if (s64_out) s64_out[row] = s64;
    }
    if (!kStatic && (gsc.exact || row_bad)) gsc.s64 = row_s64();

    if (active && k1_debug != 1) {
      int8_t* qr = q + row * ldq;
      const int o0 = sub * osz, o1 = min(o0 + osz, k_out);
      if (!row_bad && !gsc.exact) {
        const float r = gsc.r32;
        for (int c0 = o0 + lane * 16; c0 < o1; c0 += 512) {
          const uint4 ga = *reinterpret_cast<const uint4*>(gidx + c0);
          const uint4 gb = *reinterpret_cast<const uint4*>(gidx + c0 + 8);
          const uint32_t gw[8] = {ga.x, ga.y, ga.z, ga.w, gb.x, gb.y, gb.z, gb.w};
          float v[16];
          uint32_t rr[16];
          bool need = false;
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const uint32_t src = (gw[e >> 1] >> (16 * (e & 1))) & 0xffffu;
            v[e] = __uint_as_float(static_cast<uint32_t>(rs[src]) << 16);
            float t, d;
            if (kStatic) {
              t = fminf(fmaxf(__fmul_rn(v[e], r), -fq), fq);
              const float y = __fadd_rn(t, kMagic);
              d = __fsub_rn(t, __fsub_rn(y, kMagic));
              rr[e] = __float_as_uint(y);
            } else {
              const float y = __fmaf_rn(v[e], r, kMagic);
              d = __fmaf_rn(v[e], r, -__fsub_rn(y, kMagic));
              rr[e] = __float_as_uint(y);
            }
            need |= fabsf(d) > 0.4999f;
          }
          if (need) {  // within 1e-4 of a .5 tie: the exact f64 division decides
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const float t = kStatic ? fminf(fmaxf(__fmul_rn(v[e], r), -fq), fq) : 0.f;
              const float d = kStatic ? __fsub_rn(t, rintf(t))
                                      : __fmaf_rn(v[e], r, -__fsub_rn(__uint_as_float(rr[e]), kMagic));
              if (fabsf(d) > 0.4999f) rr[e] = static_cast<uint32_t>(act_code_exact(v[e], row_s64(), qmax));
            }
          }
          *reinterpret_cast<uint4*>(qr + c0) =
              make_uint4(pack4(rr[0], rr[1], rr[2], rr[3]), pack4(rr[4], rr[5], rr[6], rr[7]),
                         pack4(rr[8], rr[9], rr[10], rr[11]), pack4(rr[12], rr[13], rr[14], rr[15]));
        }
      } else {
        // rare rows: a non-finite input (reported, reference throws) or an unusable fp32 reciprocal
        for (int c = o0 + lane; c < o1; c += 32) {
          const int src = gidx[c];
          const uint16_t h = rs[src];
          int code = 0;
          if ((h & 0x7f80u) == 0x7f80u) {
            if (err) atomicMin(err, static_cast<unsigned long long>(row * k_out + c));
          } else {
            code = gsc.exact ? act_code_exact(bf16_bits_to_float(h), gsc.s64, qmax)
                             : quant_code_fast(bf16_bits_to_float(h), gsc.r32, gsc.s64, qmax);
          }
          qr[c] = static_cast<int8_t>(code);
        }
      }
    }
    if (k1_debug == 2 && blockIdx.x == 0 && tid == 0 && it < 32) ktrace[2][it] = clock64();
    __syncthreads();  // every warp is done with this slot (and with part[])
    if (tid == 0) issue(it + kActStages, slot);
  }
  if (k1_debug == 2 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1) && tid == 0) {
    unsigned long long g_exit;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_exit));
    printf("cta %d: entry %lld clk before first wait; globaltimer entry %llu exit %llu (%llu ns)\n",
           blockIdx.x, ktrace[0][0] - k_entry, g_entry, g_exit, g_exit - g_entry);
  }
  if (k1_debug == 2 && blockIdx.x == 0 && tid == 0) {
    const long long t0 = ktrace[0][0];
    for (int i = 0; i < 32 && blockIdx.x + static_cast<int64_t>(i) * gridDim.x < num_groups; ++i)
      printf("group %2d: wait %7lld..%7lld done %7lld\n", i, ktrace[0][i] - t0, ktrace[1][i] - t0,
             ktrace[2][i] - t0);
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
  const bool tma_ok = MODE != kWeightDual && dtype == QARVD_BF16 && k < 16384 &&
                      (k % 8) == 0 && (ldx % 8) == 0 && (k_out % 16) == 0 && (ldq % 16) == 0 &&
                      (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                      (reinterpret_cast<uintptr_t>(q) & 15) == 0;
  if (tma_ok) {
    const int G = k <= 1536 ? 8 : (k <= 3072 ? 4 : (k <= 6144 ? 2 : 1));
    const size_t row_elems = (k + 1 + 7) & ~int64_t(7);
    const size_t smem = static_cast<size_t>(kActStages) * G * row_elems * 2 + k_out * 2 + 64 +
                        kActStages * 8 + 16 * 4 + 16;
    auto kern = quant_act_tma_kernel<MODE == kActStatic>;
    static std::once_flag once;
    static cudaError_t attr = cudaSuccess;
    std::call_once(once, [&] {
      attr = set_smem_attrs(kern, 200 * 1024);
    });
    QARVD_CUDA_TRY(attr);
    const int64_t groups = (m + G - 1) / G;
    const int ctas_per_sm = smem <= 110 * 1024 ? 2 : 1;
    const int64_t cap = static_cast<int64_t>(kNumSMs) * ctas_per_sm;
    const int g = static_cast<int>(groups < cap ? groups : cap);
    kern<<<g, kActThreads, smem, stream>>>(static_cast<const uint16_t*>(x), m, static_cast<int>(k),
                                           ldx, gather, static_cast<int>(k_out), G, static_scale,
                                           qmax, q, ldq, s32_n, s64_n, err,
                                           getenv("QARVD_K1_DEBUG") ? atoi(getenv("QARVD_K1_DEBUG")) : 0);
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
