// Probe: per-SM throughput (ops/clk/SM) of the epilogue's instruction classes, measured
// with 8 independent chains per thread and 2048 threads per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_rate pipe_rate.cu
#include <cstdio>
#include <cstdint>

template <int MODE>
__global__ void __launch_bounds__(1024, 2) k(float* out, int iters) {
  float f[8];
  int v[8];
  for (int j = 0; j < 8; ++j) {
    f[j] = 1.0f + threadIdx.x * 1e-6f + j;
    v[j] = threadIdx.x + j;
  }
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE == 0) f[j] += __int2float_rn(v[j] + i);                     // I2FP (+FADD)
      if (MODE == 1) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[j]));  // MUFU.EX2
      if (MODE == 2) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(f[j]));  // MUFU.RCP
      if (MODE == 3) f[j] = __fmaf_rn(f[j], 1.0001f, 0.5f);                   // FFMA
      if (MODE == 4) {                                                          // FFMA2
        uint64_t a;
        asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(f[j]), "f"(f[(j + 1) & 7]));
        asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(a));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(f[j]), "=f"(f[(j + 1) & 7]) : "l"(a));
      }
      if (MODE == 5) v[j] = __shfl_xor_sync(0xffffffffu, v[j], 1) + 1;        // SHFL (MIO)
    }
  }
  const long long t1 = clock64();
  float s = 0;
  for (int j = 0; j < 8; ++j) s += f[j] + v[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const double per_iter = (double)(t1 - t0) / iters;  // cycles per iteration (8 ops/thread)
    printf("mode %d: %.1f ops/clk/SM\n", MODE, 8.0 * 2048 / per_iter);
  }
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 2 * 1024 * 4);
  const int it = 4000;
  k<0><<<296, 1024>>>(out, it); cudaDeviceSynchronize();
  k<1><<<296, 1024>>>(out, it); cudaDeviceSynchronize();
  k<2><<<296, 1024>>>(out, it); cudaDeviceSynchronize();
  k<3><<<296, 1024>>>(out, it); cudaDeviceSynchronize();
  k<4><<<296, 1024>>>(out, it); cudaDeviceSynchronize();
  k<5><<<296, 1024>>>(out, it); cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
