// Shared host/device helpers for libqarvd_b200.so (sm_100a only).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <utility>
#include <string>

#include "../../include/qarvd_b200.h"

namespace qarvd_b200 {

// ---- error plumbing (C-ABI: int status + thread-local message) ----------
void set_error(const std::string& msg);
const char* last_error_cstr();
void clear_error();
std::atomic<uint64_t>& launch_counter();
inline void count_launch(uint64_t n = 1) { launch_counter().fetch_add(n, std::memory_order_relaxed); }

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Returns QARVD_ERR_CUDA with a message when no device is usable.
int require_device();

#define QARVD_FAIL(code, msg)              \
  do {                                     \
    ::qarvd_b200::set_error(msg);          \
    return (code);                         \
  } while (0)

#define QARVD_CUDA_TRY(expr)                                                             \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess) {                                                             \
      ::qarvd_b200::set_error(std::string("CUDA error: ") + cudaGetErrorString(_e) +     \
                              " at " + __FILE__ + ":" + std::to_string(__LINE__));       \
      return QARVD_ERR_CUDA;                                                             \
    }                                                                                    \
  } while (0)

#define QARVD_LAUNCH_CHECK() QARVD_CUDA_TRY(cudaGetLastError())

constexpr int kNumSMs = 148;

// Large-smem kernels all request the maximum shared-memory carveout, so consecutive
// kernels of a pipeline never force an SM carveout reconfiguration between launches.
// Programmatic dependent launch (PDL): a kernel launched with the programmatic stream
// serialisation attribute may start while its predecessor drains; it runs its prologue
// (barrier init, TMEM allocation, tensor-map prefetch, table staging) and then waits in
// pdl_wait() until the predecessor grid has completed and its writes are visible.
// QARVD_PDL=0 launches without the attribute (A/B).
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("QARVD_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// cudaLaunchKernelEx with the PDL attribute (and an optional cluster dimension)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, int cluster, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (cluster > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = cluster;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

template <typename Kernel>
inline cudaError_t set_smem_attrs(Kernel kern, int dynamic_bytes) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       dynamic_bytes);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                              static_cast<int>(cudaSharedmemCarveoutMaxShared));
}

// Kernels that may run beside a large-shared-memory kernel (e.g. K3 / K5 next to the K4
// histogram pass) ask for the max-shared carveout too: an SM only hosts CTAs of one carveout.
template <typename Kernel>
inline cudaError_t prefer_max_shared(Kernel kern) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                              static_cast<int>(cudaSharedmemCarveoutMaxShared));
}

// ---- bf16 helpers (bit patterns; RNE as bytes.hpp:40-45) -----------------
__device__ __forceinline__ float bf16_bits_to_float(uint16_t h) {
  return __uint_as_float(static_cast<uint32_t>(h) << 16);
}

// ---- the bit-exact quantizer ---------------------------------------------
// Reference contract (quant.cpp:132-135): code = clamp(round_half_even(v / s)).
// round_half_even (quant.hpp:14-20) equals IEEE rint in the default rounding
// mode, and v / s is an IEEE f64 division.  Fast path: t = v * r32 in fp32
// with r32 ~= qmax/absmax (or 1/s).  |t - v/s| <= |t| * 2^-22 < 3.1e-5 for
// |t| <= 254, so whenever frac(t) is >= 1e-4 away from 0.5 the f64 result
// rounds to the same integer; otherwise recompute exactly with __ddiv_rn.
__device__ __forceinline__ int quant_code_fast(float v, float r32, double s64, int qmax) {
  const float t = __fmul_rn(v, r32);
  const float at = fabsf(t);
  if (at > 2.0f * qmax + 2.0f) return t > 0.f ? qmax : -qmax;  // far outside: clamps either way
  const float fl = floorf(t);
  const float fr = __fsub_rn(t, fl);  // exact for |t| < 2^23
  int q;
  if (fabsf(__fsub_rn(fr, 0.5f)) < 1e-4f) {
    q = static_cast<int>(rint(__ddiv_rn(static_cast<double>(v), s64)));
  } else {
    q = static_cast<int>(rintf(t));
  }
  return q > qmax ? qmax : (q < -qmax ? -qmax : q);
}

// Exact path for any input precision (used when r32 is not a normal float,
// and for f64 inputs): rint(v / s) in f64, then clamp.
__device__ __forceinline__ int quant_code_exact(double v, double s64, int qmax) {
  const double q = rint(__ddiv_rn(v, s64));
  if (q > static_cast<double>(qmax)) return qmax;
  if (q < -static_cast<double>(qmax)) return -qmax;
  return static_cast<int>(q);
}

template <typename T>
struct InType;
template <>
struct InType<uint16_t> {
  static constexpr int code = QARVD_BF16;
  __device__ static __forceinline__ double to_double(uint16_t v) {
    return static_cast<double>(bf16_bits_to_float(v));
  }
  __device__ static __forceinline__ bool finite(uint16_t v) { return (v & 0x7f80u) != 0x7f80u; }
};
template <>
struct InType<float> {
  static constexpr int code = QARVD_F32;
  __device__ static __forceinline__ double to_double(float v) { return static_cast<double>(v); }
  __device__ static __forceinline__ bool finite(float v) { return isfinite(v); }
};
template <>
struct InType<double> {
  static constexpr int code = QARVD_F64;
  __device__ static __forceinline__ double to_double(double v) { return v; }
  __device__ static __forceinline__ bool finite(double v) { return isfinite(v); }
};

}  // namespace qarvd_b200
