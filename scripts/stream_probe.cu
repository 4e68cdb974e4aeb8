// Probe: achievable HBM throughput for K1's traffic shape (M x K bf16 read, M x K int8 write)
// under different kernel structures, trivial per-element work.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_probe stream_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int M = 4680, K = 8960, NV = K / 8;

__device__ __forceinline__ uint2 xform(uint4 d) {  // 8 bf16 -> 8 bytes (high bytes)
  return make_uint2(__byte_perm(d.x, d.y, 0x7531), __byte_perm(d.z, d.w, 0x7531));
}
__device__ __forceinline__ uint4 ldg_na(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

// (1) flat: one chunk per thread
__global__ void flat1(const uint4* x, uint2* q, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) q[i] = xform(ldg_na(x + i));
}
// (2) flat: U chunks per thread, loads first
template <int U>
__global__ void flatU(const uint4* x, uint2* q, int64_t n) {
  int64_t base = (blockIdx.x * (int64_t)blockDim.x) * U + threadIdx.x;
  uint4 d[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    int64_t i = base + u * (int64_t)blockDim.x;
    if (i < n) d[u] = ldg_na(x + i);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    int64_t i = base + u * (int64_t)blockDim.x;
    if (i < n) q[i] = xform(d[u]);
  }
}
// (3) persistent, CTA per row, threads stride the row
__global__ void rows_persistent(const uint4* x, uint2* q) {
  for (int r = blockIdx.x; r < M; r += gridDim.x) {
    const uint4* xr = x + (int64_t)r * NV;
    uint2* qr = q + (int64_t)r * NV;
#pragma unroll 5
    for (int v = threadIdx.x; v < NV; v += blockDim.x) qr[v] = xform(ldg_na(xr + v));
  }
}
// (4) non-persistent, CTA per row
__global__ void rows_flat(const uint4* x, uint2* q) {
  const int r = blockIdx.x;
  const uint4* xr = x + (int64_t)r * NV;
  uint2* qr = q + (int64_t)r * NV;
#pragma unroll 5
  for (int v = threadIdx.x; v < NV; v += blockDim.x) qr[v] = xform(ldg_na(xr + v));
}
// (5) TMA 1-D bulk ring: warp 0 lane 0 produces S slots, other warps consume
template <int S>
__global__ void rows_bulk(const uint16_t* x, uint2* q) {
  extern __shared__ __align__(128) uint16_t sm[];
  __shared__ __align__(8) uint64_t full[S], empty[S];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nc = blockDim.x - 32;  // consumers
  const int rs = K + 64;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&empty[s])), "r"(nc / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  int nrows = 0;
  for (int r = blockIdx.x; r < M; r += gridDim.x) ++nrows;
  auto wait = [](uint64_t* b, uint32_t ph) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(b), done;
    do {
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                   : "=r"(done) : "r"(a), "r"(ph) : "memory");
    } while (!done);
  };
  if (warp == 0) {
    if (lane == 0)
      for (int j = 0; j < nrows; ++j) {
        const int s = j % S;
        if (j >= S) wait(&empty[s], (j / S - 1) & 1);
        const int r = blockIdx.x + j * gridDim.x;
        uint32_t bar = (uint32_t)__cvta_generic_to_shared(&full[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(K * 2) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"((uint32_t)__cvta_generic_to_shared(sm + s * rs)), "l"(x + (int64_t)r * K), "r"(K * 2), "r"(bar)
                     : "memory");
      }
  } else {
    const int t = threadIdx.x - 32;
    for (int j = 0; j < nrows; ++j) {
      const int s = j % S;
      wait(&full[s], (j / S) & 1);
      const int r = blockIdx.x + j * gridDim.x;
      const uint4* src = reinterpret_cast<const uint4*>(sm + s * rs);
      uint2* qr = q + (int64_t)r * NV;
      for (int v = t; v < NV; v += nc) qr[v] = xform(src[v]);
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(&empty[s])) : "memory");
    }
  }
}

template <typename F>
float timeit(F launch, void* flush, size_t flush_bytes) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9, tot = 0;
  for (int rep = 0; rep < 12; ++rep) {
    cudaMemsetAsync(flush, rep, flush_bytes);
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep >= 2) { tot += ms; if (ms < best) best = ms; }
  }
  return tot / 10 * 1e3f;
}

int main() {
  uint16_t* x;
  uint2* q;
  void* flush;
  const size_t fb = 256ull << 20;
  cudaMalloc(&x, (size_t)M * K * 2);
  cudaMalloc(&q, (size_t)M * K);
  cudaMalloc(&flush, fb);
  cudaMemset(x, 1, (size_t)M * K * 2);
  const int64_t n = (int64_t)M * NV;
  const double bytes = (double)M * K * 3;
  auto rep = [&](const char* name, float us) {
    printf("%-40s %7.1f us  %6.0f GB/s  (%s)\n", name, us, bytes / us / 1e3, cudaGetErrorString(cudaGetLastError()));
  };
  rep("flat1 256thr", timeit([&] { flat1<<<(n + 255) / 256, 256>>>((const uint4*)x, q, n); }, flush, fb));
  rep("flat4 256thr", timeit([&] { flatU<4><<<(n + 1023) / 1024, 256>>>((const uint4*)x, q, n); }, flush, fb));
  rep("flat8 256thr", timeit([&] { flatU<8><<<(n + 2047) / 2048, 256>>>((const uint4*)x, q, n); }, flush, fb));
  for (int ctas : {148 * 4, 148 * 8})
    for (int thr : {256, 512}) {
      char nm[64];
      snprintf(nm, 64, "rows_persistent %d x %d", ctas, thr);
      rep(nm, timeit([&] { rows_persistent<<<ctas, thr>>>((const uint4*)x, q); }, flush, fb));
    }
  for (int thr : {256, 512}) {
    char nm[64];
    snprintf(nm, 64, "rows_flat %d thr", thr);
    rep(nm, timeit([&] { rows_flat<<<M, thr>>>((const uint4*)x, q); }, flush, fb));
  }
  {
    const int smem4 = 4 * (K + 64) * 2;
    cudaFuncSetAttribute(rows_bulk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem4);
    for (int ctas : {148 * 2, 148 * 3})
      for (int thr : {256, 288}) {
        char nm[64];
        snprintf(nm, 64, "rows_bulk<4> %d x %d", ctas, thr);
        rep(nm, timeit([&] { rows_bulk<4><<<ctas, thr, smem4>>>(x, q); }, flush, fb));
      }
    const int smem6 = 6 * (K + 64) * 2;
    cudaFuncSetAttribute(rows_bulk<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem6);
    rep("rows_bulk<6> 148*2 x 288", timeit([&] { rows_bulk<6><<<296, 288, smem6>>>(x, q); }, flush, fb));
  }
  return 0;
}
