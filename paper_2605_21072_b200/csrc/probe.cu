// Live INT8 tensor-pipe peak of this GPU (the roofline denominator bench.py reports K2 against).
//
// MEASURED_PEAKS.json holds the copy bandwidth and a cuBLAS bf16 GEMM rate, but no INT8 figure;
// the datasheet's 4.5 POPS assumes the 1965 MHz boost clock that a power-capped B200 does not hold
// under a dense tensor load.  This kernel issues back-to-back tcgen05.mma.cta_group::1.kind::i8
// (M128 x N256 x K32, the K2 tile's instruction) from one elected thread per SM into one TMEM
// accumulator, operands a zeroed shared-memory tile: no memory traffic, the issue rate only.
// One CTA per SM; the achieved int-ops / s over the launch (CUDA events) is the dense INT8 peak
// at the clocks this board sustains under tensor load.
#include "common.cuh"
#include "ptx.cuh"

namespace qarvd_b200 {
namespace {

constexpr int kProbeN = 256;
constexpr int kProbeSmem = 64 * 1024 + 1024;

__global__ void __launch_bounds__(128, 1) int8_peak_kernel(int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  if (threadIdx.x < 32) ptx::tmem_alloc(&tslot, 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t t = tslot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = ptx::idesc_i8(128, kProbeN);
    const uint64_t a = ptx::sw128_kmajor_desc(ptx::smem_u32(sm));
    const uint64_t b = ptx::sw128_kmajor_desc(ptx::smem_u32(sm + 16384));
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < 4; ++j) ptx::mma_i8(t, a + 2 * j, b + 2 * j, idesc, (i | j) ? 1u : 0u);
    }
    ptx::mma_commit(&bar);
    ptx::mbar_wait(&bar, 0);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (threadIdx.x < 32) ptx::tmem_dealloc(t, 512);
}

}  // namespace
}  // namespace qarvd_b200

using namespace qarvd_b200;

extern "C" int qarvd_probe_int8_peak(int iters, double* tops_out, double* ms_out, void* stream) {
  clear_error();
  if (!tops_out || iters <= 0) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "qarvd_probe_int8_peak: invalid argument");
  if (int st = require_device()) return st;
  cudaStream_t s = as_stream(stream);
  QARVD_CUDA_TRY(set_smem_attrs(int8_peak_kernel, kProbeSmem));
  int sms = 0, dev = 0;
  QARVD_CUDA_TRY(cudaGetDevice(&dev));
  QARVD_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int8_peak_kernel<<<sms, 128, kProbeSmem, s>>>(iters / 8 > 0 ? iters / 8 : 1);  // warm the clocks
  cudaEvent_t e0, e1;
  QARVD_CUDA_TRY(cudaEventCreate(&e0));
  QARVD_CUDA_TRY(cudaEventCreate(&e1));
  QARVD_CUDA_TRY(cudaEventRecord(e0, s));
  int8_peak_kernel<<<sms, 128, kProbeSmem, s>>>(iters);
  QARVD_CUDA_TRY(cudaEventRecord(e1, s));
  count_launch(2);
  QARVD_LAUNCH_CHECK();
  QARVD_CUDA_TRY(cudaEventSynchronize(e1));
  float ms = 0.f;
  QARVD_CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double ops = 2.0 * 128 * kProbeN * 32 * 4.0 * static_cast<double>(iters) * sms;
  *tops_out = ops / (static_cast<double>(ms) * 1e-3) / 1e12;
  if (ms_out) *ms_out = ms;
  return QARVD_OK;
}
