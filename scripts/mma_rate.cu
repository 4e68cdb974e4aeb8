// Standalone probe: issue rate of tcgen05.mma on one SM (clock64 around N back-to-back MMAs
// into one TMEM accumulator, operands = a fixed zeroed smem tile).  Not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu && ./mma_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  uint64_t d = 0;
  d |= (uint64_t)((a & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int KIND, int N>  // KIND 0 = i8 (K=32), 1 = f16/bf16 (K=16), 2 = f8f6f4 e4m3 (K=32)
__global__ void __launch_bounds__(128, 1) probe(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 64 * 1024; i += blockDim.x) sm[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = tslot;
  if (threadIdx.x == 0) {
    uint32_t idesc;
    if (KIND == 0) idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    else if (KIND == 1) idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    else idesc = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    const uint64_t a = desc(smem_u32(sm)), b = desc(smem_u32(sm + 16384));
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (KIND == 0)
          asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;}"
                       ::"r"(t), "l"(a + 2 * j), "l"(b + 2 * j), "r"(idesc), "r"(i | j));
        else if (KIND == 1)
          asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                       ::"r"(t), "l"(a + 2 * j), "l"(b + 2 * j), "r"(idesc), "r"(i | j));
        else
          asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;}"
                       ::"r"(t), "l"(a + 2 * j), "l"(b + 2 * j), "r"(idesc), "r"(i | j));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t done = 0;
    while (!done)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p;}"
                   : "=r"(done) : "r"(smem_u32(&bar)));
    const unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
}

template <int KIND, int N>
void run(const char* name, int kdim, int blocks) {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 1024);
  cudaFuncSetAttribute(probe<KIND, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024 + 2048);
  const int iters = 2000;
  probe<KIND, N><<<blocks, 128, 64 * 1024 + 2048>>>(iters, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<KIND, N><<<blocks, 128, 64 * 1024 + 2048>>>(iters, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[1024];
  cudaMemcpy(h, d, 8 * blocks, cudaMemcpyDeviceToHost);
  const double cyc = (double)h[0] / (iters * 4);
  const double ops = 2.0 * 128 * N * kdim * iters * 4 * blocks;
  std::printf("%-28s blocks %3d: %.1f cycles/MMA  -> %.0f T(FL)OPS (events, %.3f ms) err=%s\n", name, blocks, cyc,
              ops / (ms * 1e-3) / 1e12, ms, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<0, 256>("i8   M128 N256 K32", 32, 1);
  run<0, 256>("i8   M128 N256 K32", 32, 148);
  run<0, 128>("i8   M128 N128 K32", 32, 148);
  run<1, 256>("bf16 M128 N256 K16", 16, 1);
  run<1, 256>("bf16 M128 N256 K16", 16, 148);
  run<1, 128>("bf16 M128 N128 K16", 16, 148);
  run<2, 256>("e4m3 M128 N256 K32", 32, 148);
  return 0;
}
