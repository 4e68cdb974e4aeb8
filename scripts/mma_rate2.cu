// Probe: which part of a pipelined MMA issue loop costs throughput?  One CTA per SM,
// one thread issues 4 x tcgen05.mma.kind::i8 (M128 N128 K32, 64 clk each at full rate)
// per "k-block", optionally adding the per-k-block work of a real mainloop.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate2 mma_rate2.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return (uint64_t)((a & 0x3FFFF) >> 4) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void wait_bar(uint64_t* b, uint32_t ph) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p;}"
                 : "=r"(done) : "r"(su(b)), "r"(ph) : "memory");
}

// V bits: 1 = commit per k-block, 2 = try_wait(already complete) per k-block,
//         4 = fence::after_thread_sync per k-block, 8 = rotate 5 stage descriptors,
//         16 = real pipeline: commit -> empty[s], wait full[s] (arrived by a 2nd warp on empty)
template <int V>
__global__ void __launch_bounds__(64, 1) probe(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar, dummy, full[5], empty[5];
  for (int i = threadIdx.x; i < 5 * 32768; i += blockDim.x) sm[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&dummy)));
    for (int s = 0; s < 5; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0 && (V & 2)) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&dummy)));
  const uint32_t t = tslot;
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | (8u << 24);
  if ((V & 16) && threadIdx.x == 32) {
    // producer: wait empty[s], arrive full[s]
    int s = 0; uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) {
      wait_bar(&empty[s], ph ^ 1);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&full[s])) : "memory");
      if (++s == 5) { s = 0; ph ^= 1; }
    }
  }
  if (threadIdx.x == 0) {
    const unsigned long long t0 = clock64();
    int s = 0; uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) {
      if (V & 16) wait_bar(&full[s], ph);
      if (V & 2) wait_bar(&dummy, 0);
      if (V & 4) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t off = (V & 8) ? (uint32_t)(s * 32768) : 0u;
      const uint64_t a = desc(su(sm) + off), b = desc(su(sm) + off + 16384);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;}"
                     ::"r"(t), "l"(a + 2 * j), "l"(b + 2 * j), "r"(idesc), "r"(i | j) : "memory");
      if (V & 16)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&empty[s])) : "memory");
      else if (V & 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar)) : "memory");
      if (++s == 5) { s = 0; ph ^= 1; }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&dummy)) : "memory");
    const unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
}

template <int V>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 256);
  const int smem = 5 * 32768 + 1024;
  cudaFuncSetAttribute(probe<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4000;
  probe<V><<<148, 64, smem>>>(iters, d);
  cudaDeviceSynchronize();
  probe<V><<<148, 64, smem>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
  std::printf("%-44s issue %.1f clk per k-block of 4 MMAs (ideal 256)  %s\n", name, (double)h[0] / iters,
              cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0>("baseline (4 MMAs, same descriptors)");
  run<1>("+ commit per k-block");
  run<2>("+ try_wait (complete) per k-block");
  run<4>("+ fence::after_thread_sync per k-block");
  run<8>("+ rotating stage descriptors");
  run<1 | 2 | 4 | 8>("all of the above");
  run<16 | 4 | 8>("real full/empty pipeline (5 stages)");
  return 0;
}
