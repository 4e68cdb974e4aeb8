// Probe: tensor-memory load / store throughput per SM (tcgen05.ld/st .32x32b.x32).
// W warps (W/4 per lane quadrant) repeatedly load 32 columns x 32 lanes x 4 B each.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_rate tmem_rate.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
}

template <int MODE>  // 0: loads, wait per load; 1: 2 loads then wait; 2: stores; 3: 4 loads per wait
__global__ void probe(int iters, unsigned long long* out, uint32_t* sink) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = tslot + ((uint32_t)((warp & 3) * 32) << 16);
  const int sub = warp >> 2;  // warps sharing a quadrant take different columns
  uint32_t acc = 0, r[32], r2[32], r3[32], r4[32];
  for (int i = 0; i < 32; ++i) r[i] = i;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t col = (uint32_t)(((it * 4 + sub) * 32) & 511);
    if (MODE == 0) {
      ld32(base + col, r);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc ^= r[0] ^ r[31];
    } else if (MODE == 1) {
      ld32(base + col, r);
      ld32(base + ((col + 256) & 511), r2);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc ^= r[0] ^ r2[31];
    } else if (MODE == 2) {
      st32(base + col, r);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    } else {
      ld32(base + col, r);
      ld32(base + ((col + 128) & 511), r2);
      ld32(base + ((col + 256) & 511), r3);
      ld32(base + ((col + 384) & 511), r4);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc ^= r[0] ^ r2[31] ^ r3[5] ^ r4[7];
    }
  }
  const unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tslot));
}

template <int MODE>
void run(int warps, const char* name) {
  unsigned long long* d;
  uint32_t* sink;
  cudaMalloc(&d, 8 * 148);
  cudaMalloc(&sink, 4 * 148 * 1024);
  const int iters = 2000;
  probe<MODE><<<148, warps * 32>>>(iters, d, sink);
  cudaDeviceSynchronize();
  probe<MODE><<<148, warps * 32>>>(iters, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double per_it = (double)h / iters;
  const int loads = MODE == 1 ? 2 : (MODE == 3 ? 4 : 1);
  const double bytes = (double)warps * loads * 32 * 32 * 4;  // per iteration per SM
  printf("%-34s %2d warps: %7.1f clk/iter  %7.1f B/clk/SM  (%s)\n", name, warps, per_it, bytes / per_it,
         cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(sink);
}


template <int N>
__device__ __forceinline__ void ldN(uint32_t taddr, uint32_t* r);
#define REGS16(o) "=r"(r[o+0]),"=r"(r[o+1]),"=r"(r[o+2]),"=r"(r[o+3]),"=r"(r[o+4]),"=r"(r[o+5]),"=r"(r[o+6]),"=r"(r[o+7]),"=r"(r[o+8]),"=r"(r[o+9]),"=r"(r[o+10]),"=r"(r[o+11]),"=r"(r[o+12]),"=r"(r[o+13]),"=r"(r[o+14]),"=r"(r[o+15])
template <>
__device__ __forceinline__ void ldN<16>(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : REGS16(0) : "r"(taddr));
}
template <>
__device__ __forceinline__ void ldN<64>(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
               "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
               "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
               : REGS16(0), REGS16(16), REGS16(32), REGS16(48) : "r"(taddr));
}
// 16x256b.x8: 16 lanes x 256 bits x 8 = 32 regs per thread
__device__ __forceinline__ void ld16x256_x8(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : REGS16(0), REGS16(16) : "r"(taddr));
}

template <int N, int SHAPE>  // SHAPE 0: 32x32b.xN ; 1: 16x256b.x8
__global__ void probe2(int iters, unsigned long long* out, uint32_t* sink) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = tslot + ((uint32_t)((warp & 3) * 32) << 16);
  const int sub = warp >> 2;
  uint32_t acc = 0, r[64];
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t col = (uint32_t)(((it * 4 + sub) * 64) & 511);
    if (SHAPE == 0) ldN<N>(base + col, r);
    else ld16x256_x8(base + col, r);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    acc ^= r[0] ^ r[N - 1];
  }
  const unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tslot));
}

template <int N, int SHAPE>
void run2(int warps, const char* name) {
  unsigned long long* d;
  uint32_t* sink;
  cudaMalloc(&d, 8 * 148);
  cudaMalloc(&sink, 4 * 148 * 1024);
  const int iters = 2000;
  probe2<N, SHAPE><<<148, warps * 32>>>(iters, d, sink);
  cudaDeviceSynchronize();
  probe2<N, SHAPE><<<148, warps * 32>>>(iters, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double per_it = (double)h / iters;
  const double bytes = (double)warps * N * 32 * 4;
  printf("%-34s %2d warps: %7.1f clk/iter  %7.1f B/clk/SM  (%s)\n", name, warps, per_it, bytes / per_it,
         cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  for (int w : {4, 8, 16}) run<0>(w, "ld x32, wait each");
  for (int w : {4, 8, 16}) run<1>(w, "2x ld x32, wait");
  for (int w : {4, 8}) run<3>(w, "4x ld x32, wait");
  for (int w : {4, 8, 16}) run<2>(w, "st x32, wait each");
  for (int w : {4, 8, 16}) run2<16, 0>(w, "ld 32x32b.x16");
  for (int w : {4, 8, 16}) run2<64, 0>(w, "ld 32x32b.x64");
  for (int w : {4, 8, 16}) run2<32, 1>(w, "ld 16x256b.x8 (32 regs)");
  return 0;
}
