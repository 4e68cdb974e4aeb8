// Probe: per-SM throughput of int32->fp32 conversion (I2FP) vs alternatives, and packed FMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o alu_rate alu_rate.cu
#include <cstdio>
#include <cstdint>

template <int MODE>
__global__ void k(const int* in, float* out, int iters) {
  int x[8];
  for (int j = 0; j < 8; ++j) x[j] = in[threadIdx.x * 8 + j];
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float f;
      if (MODE == 0) f = __int2float_rn(x[j] + i);                      // I2FP
      else if (MODE == 1) f = __int_as_float((x[j] + i) + 0x4B400000) - 12582912.0f;  // magic
      else f = __fmaf_rn(__int_as_float(x[j] + i), 1.0001f, acc[j]);     // FFMA baseline
      acc[j] += f;
    }
  }
  const long long t1 = clock64();
  float s = 0;
  for (int j = 0; j < 8; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0)
    printf("mode %d: %.2f clk per warp-instruction-group of 8 (1024 threads/SM) -> %.1f conversions/clk/SM\n", MODE,
           (double)(t1 - t0) / iters, 8.0 * 1024 / ((double)(t1 - t0) / iters));
}

int main() {
  int* in;
  float* out;
  cudaMalloc(&in, 1024 * 8 * 4);
  cudaMemset(in, 0, 1024 * 8 * 4);
  cudaMalloc(&out, 148 * 1024 * 4);
  k<0><<<148, 1024>>>(in, out, 20000);
  cudaDeviceSynchronize();
  k<1><<<148, 1024>>>(in, out, 20000);
  cudaDeviceSynchronize();
  k<2><<<148, 1024>>>(in, out, 20000);
  cudaDeviceSynchronize();
  return 0;
}
