// K1 structure microbenchmark (not product code): per-token int8 quantization of M x 1536 bf16
// rows, one warp per row, variants of the rows per warp and of the grid; tie repair omitted (the
// point is the memory / latency structure).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../../include/qarvd_b200.h"

__device__ __forceinline__ uint4 ldg_nc(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t q8(uint32_t w, float r) {
  const float lo = __uint_as_float(w << 16), hi = __uint_as_float(w & 0xffff0000u);
  const int a = __float2int_rn(lo * r), b = __float2int_rn(hi * r);
  return (static_cast<uint32_t>(a) & 0xffu) | ((static_cast<uint32_t>(b) & 0xffu) << 8);
}
// exact repair of a flagged chunk (f64 division per value), out of line like the product's
__device__ __noinline__ uint2 fix8(uint4 d, double s64) {
  const uint32_t w[4] = {d.x, d.y, d.z, d.w};
  uint32_t c[8];
#pragma unroll
  for (int h = 0; h < 8; ++h) {
    const uint32_t bits = h & 1 ? (w[h >> 1] & 0xffff0000u) : (w[h >> 1] << 16);
    c[h] = static_cast<uint32_t>(static_cast<int>(rint(__ddiv_rn(static_cast<double>(__uint_as_float(bits)), s64)))) & 0xffu;
  }
  return make_uint2(c[0] | c[1] << 8 | c[2] << 16 | c[3] << 24, c[4] | c[5] << 8 | c[6] << 16 | c[7] << 24);
}
// inline variant: the value near a tie decided by one f64 fma against the half-integer
// boundary (no division): r = v - hc*s64 exactly in sign
__device__ __forceinline__ uint2 fix8_fma(uint4 d, float rr, double s64) {
  const uint32_t w[4] = {d.x, d.y, d.z, d.w};
  uint32_t c[8];
#pragma unroll
  for (int h = 0; h < 8; ++h) {
    const float v = __uint_as_float(h & 1 ? (w[h >> 1] & 0xffff0000u) : (w[h >> 1] << 16));
    const float t = v * rr;
    const float lower = floorf(t);
    const double hc = static_cast<double>(lower) + 0.5;
    const double r = fma(-hc, s64, static_cast<double>(v));
    const int lo = static_cast<int>(lower);
    const int code = r > 0.0 ? lo + 1 : (r < 0.0 ? lo : ((lo & 1) ? lo + 1 : lo));
    c[h] = static_cast<uint32_t>(code) & 0xffu;
  }
  return make_uint2(c[0] | c[1] << 8 | c[2] << 16 | c[3] << 24, c[4] | c[5] << 8 | c[6] << 16 | c[7] << 24);
}
__device__ __noinline__ uint2 fix8_fma_ool(uint4 d, float rr, double s64) { return fix8_fma(d, rr, s64); }
__device__ __noinline__ uint2 fix8_f32_ool(uint4 d, float rr) {  // fp32-only work of similar size
  const uint32_t w[4] = {d.x, d.y, d.z, d.w};
  uint32_t c[8];
#pragma unroll
  for (int h = 0; h < 8; ++h) {
    const float v = __uint_as_float(h & 1 ? (w[h >> 1] & 0xffff0000u) : (w[h >> 1] << 16));
    const float t = v * rr;
    const float lower = floorf(t);
    const float r = fmaf(-(lower + 0.5f), 1.0f / rr, v);
    const int lo = static_cast<int>(lower);
    c[h] = static_cast<uint32_t>(r > 0.f ? lo + 1 : (r < 0.f ? lo : ((lo & 1) ? lo + 1 : lo))) & 0xffu;
  }
  return make_uint2(c[0] | c[1] << 8 | c[2] << 16 | c[3] << 24, c[4] | c[5] << 8 | c[6] << 16 | c[7] << 24);
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
// FEAT bit 0: exact f64 scale (fma correction) + s64 store; bit 1: tie detection + out-of-line fix
// bit 2: the fix inline with the fma decision instead
__device__ long long g_t[4680][4];
__device__ unsigned int g_smid[4680];
template <int V, int FEAT>
__global__ void __launch_bounds__(256) k1f(const uint16_t* __restrict__ x, int m, int8_t* __restrict__ q,
                                           float* __restrict__ s, double* __restrict__ s64o) {
  const int lane = threadIdx.x & 31;
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= m) return;
  long long t0 = 0;
  unsigned int nfix = 0;
  if (FEAT & 2048) { unsigned long long g; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g)); t0 = (long long)g; }
  uint4 d[V];
#pragma unroll
  for (int i = 0; i < V; ++i) d[i] = ldg_nc(reinterpret_cast<const uint4*>(x + (int64_t)row * (V * 256)) + lane + 32 * i);
  uint32_t mx = 0;
#pragma unroll
  for (int i = 0; i < V; ++i)
    mx = __vmaxu2(mx, __vmaxu2(__vmaxu2(d[i].x & 0x7fff7fffu, d[i].y & 0x7fff7fffu),
                               __vmaxu2(d[i].z & 0x7fff7fffu, d[i].w & 0x7fff7fffu)));
  const uint32_t mag = __reduce_max_sync(0xffffffffu, max(mx & 0xffffu, mx >> 16));
  const float amax = __uint_as_float(mag << 16);
  const float rr = amax > 0.f ? __fmul_rn(__frcp_rn(amax), 127.f) : 0.f;
  double s64 = 1.0;
  if (FEAT & 1) {
    const double a = amax, y = a * (1.0 / 127.0);
    s64 = fma(fma(-y, 127.0, a), 1.0 / 127.0, y);
    if (lane == 31) { s[row] = __double2float_rn(s64); s64o[row] = s64; }
  } else if (lane == 0) s[row] = amax / 127.f;
  int8_t* qr = q + (int64_t)row * (V * 256);
  uint32_t tailmask = 0;
  const bool p2 = (mag & 0x7fu) == 0u && mag >= 0x80u;
  const bool tie_dn = p2 && fma(s64, 127.0, -(double)amax) > 0.0;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const uint32_t w[4] = {d[i].x, d[i].y, d[i].z, d[i].w};
    uint32_t c[8];
    float dmax = 0.f;
    uint32_t vmask = 0;  // FEAT 8192: values within the guard
    if (FEAT & 512) {  // the product's packed FFMA2 rounding (act_codes2)
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const uint64_t v2 = pk2(__uint_as_float(w[h] << 16), __uint_as_float(w[h] & 0xffff0000u));
        const uint64_t r2 = pk2(rr, rr), m2 = pk2(12582912.0f, 12582912.0f);
        const uint64_t y2 = ffma2(v2, r2, m2);
        const uint64_t n2 = ffma2(y2, pk2(-1.f, -1.f), m2);
        const uint64_t d2 = ffma2(v2, r2, n2);
        float d0, d1, y0, y1;
        upk2(d2, d0, d1);
        upk2(y2, y0, y1);
        dmax = fmaxf(dmax, fmaxf(fabsf(d0), fabsf(d1)));
        c[2 * h] = __float_as_uint(y0) & 0xffu;
        c[2 * h + 1] = __float_as_uint(y1) & 0xffu;
      }
    } else {
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      const float v = __uint_as_float(h & 1 ? (w[h >> 1] & 0xffff0000u) : (w[h >> 1] << 16));
      const float t = v * rr;
      const float y = t + 12582912.0f;
      c[h] = __float_as_uint(y) & 0xffu;
      const float dd = fabsf(t - (y - 12582912.0f));
      dmax = fmaxf(dmax, dd);
      if (FEAT & 8192) vmask |= (dd > 0.49997f ? 1u : 0u) << h;
    }
    }
    if (FEAT & 64) {  // per-value inline exact decision of the values within the guard
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        const float v = __uint_as_float(h & 1 ? (w[h >> 1] & 0xffff0000u) : (w[h >> 1] << 16));
        const float t = v * rr;
        const float fr = t - floorf(t);
        if (fabsf(fr - 0.5f) < 3e-5f) {
          const float lower = floorf(t);
          const double r = fma(-(static_cast<double>(lower) + 0.5), s64, static_cast<double>(v));
          const int lo = static_cast<int>(lower);
          c[h] = static_cast<uint32_t>(r > 0.0 ? lo + 1 : (r < 0.0 ? lo : ((lo & 1) ? lo + 1 : lo))) & 0xffu;
        }
      }
    }
    uint2 out = make_uint2(c[0] | c[1] << 8 | c[2] << 16 | c[3] << 24, c[4] | c[5] << 8 | c[6] << 16 | c[7] << 24);
    if ((FEAT & 1024) && dmax > 0.49997f) tailmask |= 1u << i;
    if ((FEAT & 8192) && vmask) {  // divide only the flagged values
      while (vmask) {
        const int h = __ffs(vmask) - 1;
        vmask &= vmask - 1;
        const float v = __uint_as_float(h & 1 ? (w[h >> 1] & 0xffff0000u) : (w[h >> 1] << 16));
        c[h] = static_cast<uint32_t>(static_cast<int>(rint(__ddiv_rn(static_cast<double>(v), s64)))) & 0xffu;
      }
      out = make_uint2(c[0] | c[1] << 8 | c[2] << 16 | c[3] << 24, c[4] | c[5] << 8 | c[6] << 16 | c[7] << 24);
      ++nfix;
    } else if ((FEAT & 2) && dmax > 0.49997f) {
      if ((FEAT & 4096) && p2) {  // power-of-two |x|max: fp32 rule, ties by the sign of s64's rounding
        uint32_t cc[8];
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          const float v = __uint_as_float(h & 1 ? (w[h >> 1] & 0xffff0000u) : (w[h >> 1] << 16));
          const float t = v * rr;
          const float fl_ = floorf(t);
          const float qq = (t - fl_) == 0.5f ? ((tie_dn != (t < 0.f)) ? fl_ : fl_ + 1.f) : rintf(t);
          cc[h] = static_cast<uint32_t>(static_cast<int>(qq)) & 0xffu;
        }
        out = make_uint2(cc[0] | cc[1] << 8 | cc[2] << 16 | cc[3] << 24, cc[4] | cc[5] << 8 | cc[6] << 16 | cc[7] << 24);
      } else {
        out = fix8(d[i], s64);
      }
      ++nfix;
    }
    if ((FEAT & 4) && dmax > 0.49997f) out = fix8_fma(d[i], rr, s64);
    if ((FEAT & 128) && dmax > 0.49997f) out = fix8_fma_ool(d[i], rr, s64);
    if ((FEAT & 256) && dmax > 0.49997f) out = fix8_f32_ool(d[i], rr);
    if (FEAT & 8) out.x ^= dmax > 0.49997f ? 1u : 0u;  // dmax kept, no branch
    if ((FEAT & 16) && dmax > 0.49997f) out.x ^= 1u;   // trivial branch
    if ((FEAT & 32) && dmax > 0.4999999f) out = fix8(d[i], s64);  // tight guard (count test)
    *reinterpret_cast<uint2*>(qr + (lane + 32 * i) * 8) = out;
  }
  if (FEAT & 2048) {
    unsigned long long g; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    const unsigned int nf = __reduce_add_sync(0xffffffffu, nfix);
    if (lane == 0) { g_t[row][0] = t0; g_t[row][1] = (long long)g; g_t[row][2] = nf; unsigned int sm; asm("mov.u32 %0, %%smid;" : "=r"(sm)); g_smid[row] = sm; }
  }
  if (FEAT & 1024) {  // repairs after every fast store of the row
    while (tailmask) {
      const int i = __ffs(tailmask) - 1;
      tailmask &= tailmask - 1;
      const uint4 dd = ldg_nc(reinterpret_cast<const uint4*>(x + (int64_t)row * (V * 256)) + lane + 32 * i);
      *reinterpret_cast<uint2*>(qr + (lane + 32 * i) * 8) = fix8(dd, s64);
    }
  }
}
__device__ unsigned int g_flag_count;
template <int V>
__global__ void countflags(const uint16_t* __restrict__ x, int m, float guard) {
  const int lane = threadIdx.x & 31;
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= m) return;
  uint4 d[V];
#pragma unroll
  for (int i = 0; i < V; ++i) d[i] = ldg_nc(reinterpret_cast<const uint4*>(x + (int64_t)row * (V * 256)) + lane + 32 * i);
  uint32_t mx = 0;
#pragma unroll
  for (int i = 0; i < V; ++i)
    mx = __vmaxu2(mx, __vmaxu2(__vmaxu2(d[i].x & 0x7fff7fffu, d[i].y & 0x7fff7fffu),
                               __vmaxu2(d[i].z & 0x7fff7fffu, d[i].w & 0x7fff7fffu)));
  const uint32_t mag = __reduce_max_sync(0xffffffffu, max(mx & 0xffffu, mx >> 16));
  const float amax = __uint_as_float(mag << 16);
  const float rr = amax > 0.f ? __fmul_rn(__frcp_rn(amax), 127.f) : 0.f;
  unsigned int n = 0;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const uint32_t w[4] = {d[i].x, d[i].y, d[i].z, d[i].w};
    float dmax = 0.f;
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      const float v = __uint_as_float(h & 1 ? (w[h >> 1] & 0xffff0000u) : (w[h >> 1] << 16));
      const float t = v * rr;
      const float y = t + 12582912.0f;
      dmax = fmaxf(dmax, fabsf(t - (y - 12582912.0f)));
    }
    n += dmax > guard;
  }
  atomicAdd(&g_flag_count, n);
}
// CTA-shared repair: each lane records its flagged chunks; after the fast pass the CTA's 256
// threads divide the flagged chunks of all 8 rows together (a heavy row's repairs no longer
// serialize on its own warp)
template <int V>
__global__ void __launch_bounds__(256) k1cta(const uint16_t* __restrict__ x, int m, int8_t* __restrict__ q,
                                             float* __restrict__ s, double* __restrict__ s64o) {
  __shared__ unsigned int s_n;
  __shared__ unsigned int s_list[1024];  // (warp << 13) | (lane << 3) | i
  __shared__ double s_s64[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  if (row < m) {
    uint4 d[V];
#pragma unroll
    for (int i = 0; i < V; ++i) d[i] = ldg_nc(reinterpret_cast<const uint4*>(x + (int64_t)row * (V * 256)) + lane + 32 * i);
    uint32_t mx = 0;
#pragma unroll
    for (int i = 0; i < V; ++i)
      mx = __vmaxu2(mx, __vmaxu2(__vmaxu2(d[i].x & 0x7fff7fffu, d[i].y & 0x7fff7fffu),
                                 __vmaxu2(d[i].z & 0x7fff7fffu, d[i].w & 0x7fff7fffu)));
    const uint32_t mag = __reduce_max_sync(0xffffffffu, max(mx & 0xffffu, mx >> 16));
    const float amax = __uint_as_float(mag << 16);
    const float rr = amax > 0.f ? __fmul_rn(__frcp_rn(amax), 127.f) : 0.f;
    const double a = amax, y = a * (1.0 / 127.0);
    const double s64 = fma(fma(-y, 127.0, a), 1.0 / 127.0, y);
    if (lane == 31) { s[row] = __double2float_rn(s64); s64o[row] = s64; s_s64[warp] = s64; }
    int8_t* qr = q + (int64_t)row * (V * 256);
    uint32_t flagged = 0;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const uint32_t w[4] = {d[i].x, d[i].y, d[i].z, d[i].w};
      uint32_t c[8];
      float dmax = 0.f;
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        const float v = __uint_as_float(h & 1 ? (w[h >> 1] & 0xffff0000u) : (w[h >> 1] << 16));
        const float t = v * rr;
        const float yy = t + 12582912.0f;
        c[h] = __float_as_uint(yy) & 0xffu;
        dmax = fmaxf(dmax, fabsf(t - (yy - 12582912.0f)));
      }
      flagged |= (dmax > 0.49997f ? 1u : 0u) << i;
      *reinterpret_cast<uint2*>(qr + (lane + 32 * i) * 8) =
          make_uint2(c[0] | c[1] << 8 | c[2] << 16 | c[3] << 24, c[4] | c[5] << 8 | c[6] << 16 | c[7] << 24);
    }
    while (flagged) {
      const int i = __ffs(flagged) - 1;
      flagged &= flagged - 1;
      const unsigned int slot = atomicAdd(&s_n, 1u);
      if (slot < 1024) s_list[slot] = (warp << 13) | (lane << 3) | i;
    }
  }
  __syncthreads();
  const unsigned int n = min(s_n, 1024u);
  for (unsigned int e = threadIdx.x; e < n; e += blockDim.x) {
    const unsigned int code = s_list[e];
    const int wp = code >> 13, ln = (code >> 3) & 31, i = code & 7;
    const int rw = blockIdx.x * 8 + wp;
    const int c0 = (ln + 32 * i) * 8;
    const uint4 dd = ldg_nc(reinterpret_cast<const uint4*>(x + (int64_t)rw * (V * 256) + c0));
    *reinterpret_cast<uint2*>(q + (int64_t)rw * (V * 256) + c0) = fix8(dd, s_s64[wp]);
  }
}
template <int V, int R>  // V uint4 per lane per row, R rows per warp
__global__ void __launch_bounds__(256) k1v(const uint16_t* __restrict__ x, int m, int8_t* __restrict__ q,
                                           float* __restrict__ s, int rows_per_grid_step) {
  const int lane = threadIdx.x & 31;
  const int warp_g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int base = warp_g * R; base < m; base += nw * R) {
    uint4 d[R][V];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int i = 0; i < V; ++i)
        if (base + r < m) d[r][i] = ldg_nc(reinterpret_cast<const uint4*>(x + (int64_t)(base + r) * (V * 256)) + lane + 32 * i);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (base + r >= m) break;
      uint32_t mx = 0;
#pragma unroll
      for (int i = 0; i < V; ++i)
        mx = __vmaxu2(mx, __vmaxu2(__vmaxu2(d[r][i].x & 0x7fff7fffu, d[r][i].y & 0x7fff7fffu),
                                   __vmaxu2(d[r][i].z & 0x7fff7fffu, d[r][i].w & 0x7fff7fffu)));
      const uint32_t mag = __reduce_max_sync(0xffffffffu, max(mx & 0xffffu, mx >> 16));
      const float amax = __uint_as_float(mag << 16);
      const float rr = amax > 0.f ? 127.f / amax : 0.f;
      if (lane == 0) s[base + r] = amax / 127.f;
      int8_t* qr = q + (int64_t)(base + r) * (V * 256);
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const uint32_t a = q8(d[r][i].x, rr), b = q8(d[r][i].y, rr), c = q8(d[r][i].z, rr), e = q8(d[r][i].w, rr);
        *reinterpret_cast<uint2*>(qr + (lane + 32 * i) * 8) = make_uint2(a | (b << 16), c | (e << 16));
      }
    }
  }
}
__global__ void copyk(const uint4* __restrict__ a, uint4* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) b[i] = a[i];
}
int main(int argc, char** argv) {
  const int m = 4680, k = 1536;
  uint16_t* x; int8_t* q; float* s; uint8_t* fl; uint4* y;
  cudaMalloc(&x, (size_t)m * k * 2); cudaMalloc(&q, (size_t)m * k); cudaMalloc(&s, m * 4);
  cudaMalloc(&fl, 256 << 20); cudaMalloc(&y, (size_t)m * k * 2);
  std::vector<uint16_t> h((size_t)m * k);
  uint32_t st = 1;
  for (auto& v : h) { st = st * 1664525u + 1013904223u; v = 0x3c00 + (st >> 20) % 0x600; if (st & 1) v |= 0x8000; }
  if (argc > 1) {  // real activations (bf16 bits, m x k) from a file
    FILE* f = fopen(argv[1], "rb");
    if (f) { size_t got = fread(h.data(), 2, h.size(), f); fclose(f); printf("loaded %zu values from %s\n", got, argv[1]); }
  }
  cudaMemcpy(x, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto timeit = [&](const char* name, auto fn) {
    float best = 1e9, sum = 0;
    for (int it = 0; it < 30; ++it) {
      cudaMemset(fl, it, 256 << 20);
      cudaEventRecord(a); fn(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best; if (it >= 5) sum += ms;
    }
    printf("%-40s best %6.1f us  mean %6.1f us\n", name, best * 1e3, sum / 25 * 1e3);
  };
  timeit("copy (2x bytes)", [&] { copyk<<<148 * 8, 256>>>(reinterpret_cast<uint4*>(x), y, (int64_t)m * k / 8); });
  timeit("1 row/warp, 1 wave (585 CTAs)", [&] { k1v<6, 1><<<(m + 7) / 8, 256>>>(x, m, q, s, 0); });
  timeit("2 rows/warp (293 CTAs)", [&] { k1v<6, 2><<<(m + 15) / 16, 256>>>(x, m, q, s, 0); });
  timeit("1 row/warp, persistent 148x4", [&] { k1v<6, 1><<<148 * 4, 256>>>(x, m, q, s, 0); });
  timeit("1 row/warp, persistent 148x2", [&] { k1v<6, 1><<<148 * 2, 256>>>(x, m, q, s, 0); });
  timeit("2 rows/warp, persistent 148x2", [&] { k1v<6, 2><<<148 * 2, 256>>>(x, m, q, s, 0); });
  timeit("1 row/warp, 128-thread CTAs (1170)", [&] { k1v<6, 1><<<(m + 3) / 4, 128>>>(x, m, q, s, 0); });
  timeit("1 row/warp, 64-thread CTAs (2340)", [&] { k1v<6, 1><<<(m + 1) / 2, 64>>>(x, m, q, s, 0); });
  double* s64o; cudaMalloc(&s64o, m * 8);
  timeit("feat 0 (magic rounding)", [&] { k1f<6, 0><<<(m + 7) / 8, 256>>>(x, m, q, s, s64o); });
  timeit("feat 1 (+ exact f64 scale, s64 store)", [&] { k1f<6, 1><<<(m + 7) / 8, 256>>>(x, m, q, s, s64o); });
  timeit("feat 2 (+ tie detect, out-of-line fix)", [&] { k1f<6, 2><<<(m + 7) / 8, 256>>>(x, m, q, s, s64o); });
  timeit("feat 3 (both)", [&] { k1f<6, 3><<<(m + 7) / 8, 256>>>(x, m, q, s, s64o); });
  timeit("feat 5 (scale + inline fma tie fix)", [&] { k1f<6, 5><<<(m + 7) / 8, 256>>>(x, m, q, s, s64o); });
  timeit("feat 9 (dmax, no branch)", [&] { k1f<6, 9><<<(m + 7) / 8, 256>>>(x, m, q, s, s64o); });
  timeit("feat 17 (dmax, trivial branch)", [&] { k1f<6, 17><<<(m + 7) / 8, 256>>>(x, m, q, s, s64o); });
  timeit("feat 33 (out-of-line fix, guard 1e-7)", [&] { k1f<6, 33><<<(m + 7) / 8, 256>>>(x, m, q, s, s64o); });
  timeit("feat 65 (per-value inline fma decision)", [&] { k1f<6, 65><<<(m + 7) / 8, 256>>>(x, m, q, s, s64o); });
  timeit("feat 129 (out-of-line fma fix)", [&] { k1f<6, 129><<<(m + 7) / 8, 256>>>(x, m, q, s, s64o); });
  timeit("feat 257 (out-of-line fp32-only fix)", [&] { k1f<6, 257><<<(m + 7) / 8, 256>>>(x, m, q, s, s64o); });
  timeit("feat 1 again", [&] { k1f<6, 1><<<(m + 7) / 8, 256>>>(x, m, q, s, s64o); });
  timeit("feat 3 again", [&] { k1f<6, 3><<<(m + 7) / 8, 256>>>(x, m, q, s, s64o); });
  {  // the product's K1 through the C-ABI (plan-order rows, per-token), same data and flush
    int8_t* q2; cudaMalloc(&q2, (size_t)m * k);
    float* s32; cudaMalloc(&s32, m * 4);
    timeit("product qarvd_quantize_act (C-ABI)", [&] {
      qarvd_quantize_act(x, QARVD_BF16, m, k, k, nullptr, k, QARVD_ACT_PER_TOKEN, 0.0, 8, q2, k, s32, nullptr, nullptr, nullptr);
    });
    // agreement with the fix-free microkernel on the non-tie values
    k1f<6, 3><<<(m + 7) / 8, 256>>>(x, m, q, s, s64o);
    std::vector<int8_t> a((size_t)m * k), b((size_t)m * k);
    cudaMemcpy(a.data(), q, a.size(), cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), q2, b.size(), cudaMemcpyDeviceToHost);
    size_t diff = 0;
    for (size_t i = 0; i < a.size(); ++i) diff += a[i] != b[i];
    printf("microkernel (feat 3) vs product codes: %zu of %zu differ\n", diff, a.size());
  }
  {  // both kernels captured into CUDA graphs (no host time in the timed region)
    cudaStream_t cs; cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    int8_t* q3; cudaMalloc(&q3, (size_t)m * k);
    float* s33; cudaMalloc(&s33, m * 4);
    auto graph_of = [&](auto fn) {
      cudaGraph_t g; cudaGraphExec_t ge;
      cudaStreamBeginCapture(cs, cudaStreamCaptureModeGlobal);
      fn();
      cudaStreamEndCapture(cs, &g);
      cudaGraphInstantiate(&ge, g, 0);
      return ge;
    };
    cudaGraphExec_t gp = graph_of([&] {
      const int st = qarvd_quantize_act(x, QARVD_BF16, m, k, k, nullptr, k, QARVD_ACT_PER_TOKEN, 0.0, 8, q3, k, s33, nullptr, nullptr, cs);
      if (st) printf("capture: status %d %s\n", st, qarvd_last_error());
    });
    cudaGraphExec_t gm = graph_of([&] { k1f<6, 3><<<(m + 7) / 8, 256, 0, cs>>>(x, m, q, s, s64o); });
    cudaGraphExec_t gm2 = graph_of([&] { k1f<6, 515><<<(m + 7) / 8, 256, 0, cs>>>(x, m, q, s, s64o); });
    cudaGraphExec_t gm3 = graph_of([&] { k1f<6, 513><<<(m + 7) / 8, 256, 0, cs>>>(x, m, q, s, s64o); });
    auto gtime = [&](const char* name, cudaGraphExec_t ge) {
      float best = 1e9;
      for (int it = 0; it < 30; ++it) {
        cudaMemsetAsync(fl, it, 256 << 20, cs);
        cudaEventRecord(a, cs); cudaGraphLaunch(ge, cs); cudaEventRecord(b, cs); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best;
      }
      printf("%-40s graph best %6.1f us\n", name, best * 1e3);
    };
    gtime("product K1 (graph)", gp);
    gtime("microkernel feat 3 (graph)", gm);
    gtime("microkernel feat 515 (FFMA2 + fix)", gm2);
    gtime("microkernel feat 513 (FFMA2, no fix)", gm3);
    cudaGraphExec_t gm4 = graph_of([&] { k1f<6, 1025><<<(m + 7) / 8, 256, 0, cs>>>(x, m, q, s, s64o); });
    gtime("microkernel feat 1025 (tail repair)", gm4);
    cudaGraphExec_t gm5 = graph_of([&] { k1f<6, 3 + 4096><<<(m + 7) / 8, 256, 0, cs>>>(x, m, q, s, s64o); });
    gtime("microkernel feat 4099 (p2 rule + division)", gm5);
    cudaGraphExec_t gm6 = graph_of([&] { k1f<6, 1 + 8192><<<(m + 7) / 8, 256, 0, cs>>>(x, m, q, s, s64o); });
    gtime("microkernel feat 8193 (divide flagged values)", gm6);
    cudaGraphExec_t gm7 = graph_of([&] { k1cta<6><<<(m + 7) / 8, 256, 0, cs>>>(x, m, q, s, s64o); });
    gtime("k1cta (CTA-shared repair)", gm7);
    {
      int8_t* q4; cudaMalloc(&q4, (size_t)m * k);
      k1cta<6><<<(m + 7) / 8, 256>>>(x, m, q4, s, s64o);
      qarvd_quantize_act(x, QARVD_BF16, m, k, k, nullptr, k, QARVD_ACT_PER_TOKEN, 0.0, 8, q, k, nullptr, nullptr, nullptr, nullptr);
      cudaDeviceSynchronize();
      std::vector<int8_t> a1((size_t)m * k), b1((size_t)m * k);
      cudaMemcpy(a1.data(), q4, a1.size(), cudaMemcpyDeviceToHost);
      cudaMemcpy(b1.data(), q, b1.size(), cudaMemcpyDeviceToHost);
      size_t df = 0; for (size_t i = 0; i < a1.size(); ++i) df += a1[i] != b1[i];
      printf("k1cta vs product: %zu differ\n", df);
    }
    for (int feat : {2049 + 2, 2049, 2049 + 8192}) {
      cudaMemset(fl, 1, 256 << 20);
      cudaDeviceSynchronize();
      if (feat == 2051) k1f<6, 2051><<<(m + 7) / 8, 256>>>(x, m, q, s, s64o);
      else if (feat == 2049 + 8192) k1f<6, 2049 + 8192><<<(m + 7) / 8, 256>>>(x, m, q, s, s64o);
      else k1f<6, 2049><<<(m + 7) / 8, 256>>>(x, m, q, s, s64o);
      cudaDeviceSynchronize();
      static long long ht[4680][4]; static unsigned int hs[4680];
      cudaMemcpyFromSymbol(ht, g_t, sizeof(ht)); cudaMemcpyFromSymbol(hs, g_smid, sizeof(hs));
      long long tmin = ht[0][0], tmax = 0;
      for (int r = 0; r < m; ++r) { tmin = ht[r][0] < tmin ? ht[r][0] : tmin; tmax = ht[r][1] > tmax ? ht[r][1] : tmax; }
      double dfix = 0, dnofix = 0; int nf = 0, nn = 0; long long worst = 0; int worst_r = 0;
      for (int r = 0; r < m; ++r) { long long du = ht[r][1] - ht[r][0]; if (ht[r][2]) { dfix += du; ++nf; } else { dnofix += du; ++nn; } if (ht[r][1] > worst) { worst = ht[r][1]; worst_r = r; } }
      printf("feat %d: span %lld ns; warps with repairs %d (mean %.0f ns), without %d (mean %.0f ns); last to finish row %d (%lld fixes, start +%lld ns, dur %lld ns, sm %u)\n",
             feat, tmax - tmin, nf, nf ? dfix / nf : 0, nn, nn ? dnofix / nn : 0, worst_r, ht[worst_r][2], ht[worst_r][0] - tmin, ht[worst_r][1] - ht[worst_r][0], hs[worst_r]);
      // start-time distribution
      long long late = 0; for (int r = 0; r < m; ++r) late = (ht[r][0] - tmin) > late ? (ht[r][0] - tmin) : late;
      printf("   latest warp start +%lld ns\n", late);
    }
  }
  for (float gd : {0.49997f, 0.4999999f}) {
    unsigned int z = 0;
    cudaMemcpyToSymbol(g_flag_count, &z, 4);
    countflags<6><<<(m + 7) / 8, 256>>>(x, m, gd);
    cudaMemcpyFromSymbol(&z, g_flag_count, 4);
    printf("guard %.7f: %u flagged lane-chunks of %d\n", gd, z, m * 32 * 6);
  }
  cudaDeviceSynchronize();
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
