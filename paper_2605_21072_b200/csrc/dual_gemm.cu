// K2 — dual-scale W8A8 linear on the sm_100a tensor cores.
//
// Replaces the reference's scalar triple loop kernel_b_gemm_dequant
// (/root/reference/proj/core/src/engine.cpp:46-105).  The reference keeps one
// int64 accumulator per (row, column, group) and combines the groups in f64,
// outlier group first (engine.cpp:86-94).  Here both operands are int8 codes
// already permuted [outlier | normal] along K (calibrate.cpp:474-480 for the
// weights, K1 for the activations); TMA streams 128-byte K-slices of both into
// a 128B-swizzled shared-memory ring, a single elected thread issues
// tcgen05.mma.kind::i8 (M=128, N=BN, K=32) and routes every K=32 step to one of
// two int32 tensor-memory accumulators: acc_o for k < k_outlier, acc_n after.
// int32 is exact because |code| <= 127 and k <= 132104 (D4 in SURVEY.md).
// Four epilogue warps read both accumulators with tcgen05.ld and apply
//   y = s_x[i] * (s_wo[j]*acc_o + s_wn[j]*acc_n) (+ bias[j]) -> bf16.
// Persistent, warp-specialised: warp 0 = TMA producer, warp 1 = MMA issuer,
// warp 2 = TMEM allocator, warps 4..7 = epilogue.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "ptx.cuh"

namespace qarvd_b200 {
namespace {

constexpr int BM = 128;  // rows of the activation tile (one TMEM lane per row)
constexpr int BK = 128;  // bytes (= int8 elements) of K per pipeline stage: one swizzle row
constexpr int kThreads = 384;  // 4 control warps + 8 epilogue warps
constexpr int kEpiWarps = 8;

template <int BN>
struct GemmCfg {
  static constexpr int kStages = (BN == 256) ? 4 : 6;
  static constexpr int kABytes = BM * BK;
  static constexpr int kBBytes = BN * BK;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kAccStages = 512 / (2 * BN);  // two accumulators per stage
  static constexpr uint32_t kTmemCols = 512;
  static constexpr size_t kSmemBytes =
      static_cast<size_t>(kStages) * kStageBytes + 1024 /*align slack*/ + 512 /*barriers*/ +
      kEpiWarps * 96 * sizeof(float) /*epilogue scale staging*/;
};

struct GemmParams {
  int64_t m, n, k, k_o;
  const float* scale_x;
  const float* scale_wo;
  const float* scale_wn;
  const float* bias;
  void* y;
  int64_t ldy;
  int32_t* acc_o_dbg;
  int32_t* acc_n_dbg;
  int epilogue;
  int out_dtype;
  int num_m_blks, num_n_blks, num_tiles;
};

__device__ __forceinline__ float gelu_erf(float v) {
  return 0.5f * v * (1.0f + erff(v * 0.70710678118654752f));
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    dual_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                     const __grid_constant__ CUtensorMap tmB, const GemmParams p) {
  using C = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kStages * C::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::kStages * C::kBBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + C::kAccStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + C::kAccStages);
  float* epi_scratch = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + 512);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < C::kAccStages; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], kEpiWarps);  // one arrive per epilogue warp
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, C::kTmemCols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int num_kb = static_cast<int>((p.k + BK - 1) / BK);

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        const int m_blk = t % p.num_m_blks;
        const int n_blk = t / p.num_m_blks;
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          ptx::mbar_expect_tx(&full[stage], C::kStageBytes);
          ptx::tma_load_2d(sA + stage * C::kABytes, &tmA, &full[stage], kb * BK, m_blk * BM);
          ptx::tma_load_2d(sB + stage * C::kBBytes, &tmB, &full[stage], kb * BK, n_blk * BN);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (one thread) =====================
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_i8(BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_o = tmem_base + static_cast<uint32_t>(acc * 2 * BN);
        const uint32_t d_n = d_o + BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint64_t a_desc = ptx::sw128_kmajor_desc(ptx::smem_u32(sA + stage * C::kABytes));
          const uint64_t b_desc = ptx::sw128_kmajor_desc(ptx::smem_u32(sB + stage * C::kBBytes));
#pragma unroll
          for (int j = 0; j < BK / 32; ++j) {
            const int64_t kk = static_cast<int64_t>(kb) * BK + j * 32;
            if (kk >= p.k) break;
            const bool outl = kk < p.k_o;
            const uint32_t accumulate = (kk == 0 || kk == p.k_o) ? 0u : 1u;
            // +32 bytes along K inside the 128B swizzle row = +2 in the >>4 address field
            ptx::mma_i8(outl ? d_o : d_n, a_desc + 2 * j, b_desc + 2 * j, idesc, accumulate);
          }
          ptx::mma_commit(&empty[stage]);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        ptx::mma_commit(&tfull[acc]);
        if (++acc == C::kAccStages) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue: 8 warps, 2 per TMEM lane quadrant =====================
    // warp w may only touch TMEM lanes 32*(w%4)..+31; the two warps of a quadrant
    // split the tile's 32-column chunks (even / odd).
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;
    const int row_in_tile = q * 32 + lane;
    const bool has_outlier = p.k_o > 0;
    float* scr = epi_scratch + (warp - 4) * 96;  // per-warp staging of the chunk's column scales
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      const int m_blk = t % p.num_m_blks;
      const int n_blk = t / p.num_m_blks;
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const int64_t row = static_cast<int64_t>(m_blk) * BM + row_in_tile;
      const bool row_ok = row < p.m;
      const float sx = row_ok ? __ldg(p.scale_x + row) : 0.f;
      const uint32_t t_lane = static_cast<uint32_t>(q * 32) << 16;
      const uint32_t t_o = tmem_base + t_lane + static_cast<uint32_t>(acc * 2 * BN);
      const uint32_t t_n = t_o + BN;
#pragma unroll 1
      for (int c = half; c < BN / 32; c += 2) {
        const int64_t col0 = static_cast<int64_t>(n_blk) * BN + c * 32;
        if (col0 >= p.n) break;  // warp-uniform
        const int ncols = (p.n - col0) < 32 ? static_cast<int>(p.n - col0) : 32;
        {
          const int64_t jc = col0 + (lane < ncols ? lane : 0);
          scr[lane] = __ldg(p.scale_wn + jc);
          scr[32 + lane] = has_outlier ? __ldg(p.scale_wo + jc) : 0.f;
          scr[64 + lane] = p.bias ? __ldg(p.bias + jc) : 0.f;
        }
        uint32_t rn[32], ro[32];
        ptx::tmem_ld32(t_n + c * 32, rn);
        if (has_outlier) ptx::tmem_ld32(t_o + c * 32, ro);
        ptx::tmem_wait_ld();
        __syncwarp();
        if (row_ok) {
          if (p.acc_n_dbg) {
#pragma unroll
            for (int e = 0; e < 32; ++e) {
              if (e >= ncols) continue;
              p.acc_n_dbg[row * p.n + col0 + e] = static_cast<int32_t>(rn[e]);
              if (p.acc_o_dbg)
                p.acc_o_dbg[row * p.n + col0 + e] = has_outlier ? static_cast<int32_t>(ro[e]) : 0;
            }
          }
          // y overwrites rn (as float bits): t = s_wo*acc_o; t = fmaf(s_wn, acc_n, t); y = s_x*t (+bias)
#pragma unroll
          for (int e4 = 0; e4 < 8; ++e4) {
            const float4 sn4 = reinterpret_cast<const float4*>(scr)[e4];
            const float4 so4 = reinterpret_cast<const float4*>(scr + 32)[e4];
            const float4 sb4 = reinterpret_cast<const float4*>(scr + 64)[e4];
            const float sn[4] = {sn4.x, sn4.y, sn4.z, sn4.w};
            const float so[4] = {so4.x, so4.y, so4.z, so4.w};
            const float sb[4] = {sb4.x, sb4.y, sb4.z, sb4.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int e = 4 * e4 + u;
              const float an = __int2float_rn(static_cast<int>(rn[e]));
              float tacc;
              if (has_outlier)
                tacc = __fmaf_rn(sn[u], an, __fmul_rn(so[u], __int2float_rn(static_cast<int>(ro[e]))));
              else
                tacc = __fmul_rn(sn[u], an);
              float v = p.bias ? __fmaf_rn(sx, tacc, sb[u]) : __fmul_rn(sx, tacc);
              if (p.epilogue & QARVD_EPI_GELU) v = gelu_erf(v);
              rn[e] = __float_as_uint(v);
            }
          }
          if (p.out_dtype == QARVD_BF16) {
            __nv_bfloat16* yr = reinterpret_cast<__nv_bfloat16*>(p.y) + row * p.ldy + col0;
            if (ncols == 32 && ((reinterpret_cast<uintptr_t>(yr) & 15) == 0)) {
              uint32_t pk[16];
#pragma unroll
              for (int e = 0; e < 16; ++e) {
                const __nv_bfloat162 h2 =
                    __floats2bfloat162_rn(__uint_as_float(rn[2 * e]), __uint_as_float(rn[2 * e + 1]));
                pk[e] = *reinterpret_cast<const uint32_t*>(&h2);
              }
              uint4* dst = reinterpret_cast<uint4*>(yr);
#pragma unroll
              for (int v4 = 0; v4 < 4; ++v4)
                dst[v4] = make_uint4(pk[4 * v4], pk[4 * v4 + 1], pk[4 * v4 + 2], pk[4 * v4 + 3]);
            } else {
#pragma unroll
              for (int e = 0; e < 32; ++e)
                if (e < ncols) yr[e] = __float2bfloat16_rn(__uint_as_float(rn[e]));
            }
          } else {
            float* yr = reinterpret_cast<float*>(p.y) + row * p.ldy + col0;
            if (ncols == 32 && ((reinterpret_cast<uintptr_t>(yr) & 15) == 0)) {
              float4* dst = reinterpret_cast<float4*>(yr);
#pragma unroll
              for (int v4 = 0; v4 < 8; ++v4)
                dst[v4] = make_float4(__uint_as_float(rn[4 * v4]), __uint_as_float(rn[4 * v4 + 1]),
                                      __uint_as_float(rn[4 * v4 + 2]), __uint_as_float(rn[4 * v4 + 3]));
            } else {
#pragma unroll
              for (int e = 0; e < 32; ++e)
                if (e < ncols) yr[e] = __uint_as_float(rn[e]);
            }
          }
        }
        __syncwarp();  // scr is rewritten by the next chunk
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
      if (++acc == C::kAccStages) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, C::kTmemCols);
  }
}

// ---- host side -------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult qres;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qres) ==
            cudaSuccess &&
        qres == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

// 2-D int8 K-major operand [rows x k] (ld bytes), box = box_rows x 128 B, 128B swizzle.
int make_operand_tmap(CUtensorMap* map, const int8_t* base, int64_t rows, int64_t k, int64_t ld,
                      int box_rows) {
  auto encode = get_encode_fn();
  if (!encode) QARVD_FAIL(QARVD_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(base), dims,
                      strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    QARVD_FAIL(QARVD_ERR_CUDA, "cuTensorMapEncodeTiled failed with CUresult " + std::to_string(r));
  return QARVD_OK;
}

int sm_count() {
  static int count = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&count, cudaDevAttrMultiProcessorCount, dev);
    if (count <= 0) count = kNumSMs;
  });
  return count;
}

template <int BN>
int launch_gemm(const int8_t* xq, int64_t ldq, const int8_t* wq, int64_t ldw, GemmParams p,
                cudaStream_t stream) {
  using C = GemmCfg<BN>;
  static std::once_flag attr_once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(attr_once, [] {
    attr_err = cudaFuncSetAttribute(dual_gemm_kernel<BN>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(C::kSmemBytes));
  });
  QARVD_CUDA_TRY(attr_err);
  CUtensorMap ta, tb;
  int st = make_operand_tmap(&ta, xq, p.m, p.k, ldq, BM);
  if (st) return st;
  st = make_operand_tmap(&tb, wq, p.n, p.k, ldw, BN);
  if (st) return st;
  p.num_m_blks = static_cast<int>((p.m + BM - 1) / BM);
  p.num_n_blks = static_cast<int>((p.n + BN - 1) / BN);
  p.num_tiles = p.num_m_blks * p.num_n_blks;
  const int grid = p.num_tiles < sm_count() ? p.num_tiles : sm_count();
  dual_gemm_kernel<BN><<<grid, kThreads, C::kSmemBytes, stream>>>(ta, tb, p);
  count_launch();
  QARVD_LAUNCH_CHECK();
  return QARVD_OK;
}

// Tile-width choice: minimise waves x BN (per-SM work on the critical path).
int choose_bn(int64_t m, int64_t n) {
  if (const char* env = getenv("QARVD_GEMM_BN")) {
    const int v = atoi(env);
    if (v == 128 || v == 256) return v;
  }
  const int64_t mb = (m + BM - 1) / BM;
  const int64_t sms = sm_count();
  int best = 256;
  int64_t best_cost = -1;
  for (int bn : {256, 128}) {
    const int64_t tiles = mb * ((n + bn - 1) / bn);
    const int64_t cost = ((tiles + sms - 1) / sms) * bn;
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = bn;
    }
  }
  return best;
}

}  // namespace

int dual_gemm_launch(const int8_t* xq, int64_t ldq, const int8_t* wq, int64_t ldw, int64_t m,
                     int64_t n, int64_t k, int64_t k_outlier, const float* scale_x,
                     const float* scale_wo, const float* scale_wn, const float* bias,
                     int epilogue, int out_dtype, void* y, int64_t ldy, int32_t* acc_o,
                     int32_t* acc_n, cudaStream_t stream) {
  GemmParams p{};
  p.m = m;
  p.n = n;
  p.k = k;
  p.k_o = k_outlier;
  p.scale_x = scale_x;
  p.scale_wo = scale_wo;
  p.scale_wn = scale_wn;
  p.bias = bias;
  p.y = y;
  p.ldy = ldy;
  p.acc_o_dbg = acc_o;
  p.acc_n_dbg = acc_n;
  p.epilogue = epilogue;
  p.out_dtype = out_dtype;
  return choose_bn(m, n) == 256 ? launch_gemm<256>(xq, ldq, wq, ldw, p, stream)
                                : launch_gemm<128>(xq, ldq, wq, ldw, p, stream);
}

}  // namespace qarvd_b200

using namespace qarvd_b200;

extern "C" int qarvd_dual_gemm(const int8_t* xq, int64_t ldq, const int8_t* wq, int64_t ldw,
                               int64_t m, int64_t n, int64_t k, int64_t k_outlier,
                               const float* scale_x, const float* scale_w_outlier,
                               const float* scale_w_normal, const float* bias, int epilogue,
                               int out_dtype, void* y, int64_t ldy, int32_t* acc_outlier,
                               int32_t* acc_normal, void* stream) {
  clear_error();
  if (m <= 0 || n <= 0 || k <= 0)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: empty shape");
  if (k % 32 != 0 || k_outlier % 32 != 0 || k_outlier < 0 || k_outlier >= k)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT,
               "kernel_b: k and k_outlier must be multiples of 32 with 0 <= k_outlier < k");
  if (k > 132104)
    QARVD_FAIL(QARVD_ERR_LOGIC,
               "kernel_b: reduction dimension too large for exact int32 accumulation");
  if (ldq < k || ldw < k || ldq % 16 || ldw % 16 || ldy < n)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: leading dimensions must be >= k (n for y) and multiples of 16");
  if ((reinterpret_cast<uintptr_t>(xq) & 15) || (reinterpret_cast<uintptr_t>(wq) & 15))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: operand pointers must be 16-byte aligned");
  if (!xq || !wq || !scale_x || !scale_w_normal || !y || (k_outlier > 0 && !scale_w_outlier))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: null pointer argument");
  if (out_dtype != QARVD_BF16 && out_dtype != QARVD_F32)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "kernel_b: output dtype must be bf16 or f32");
  if (int st = require_device()) return st;
  return dual_gemm_launch(xq, ldq, wq, ldw, m, n, k, k_outlier, scale_x, scale_w_outlier,
                          scale_w_normal, bias, epilogue, out_dtype, y, ldy, acc_outlier,
                          acc_normal, as_stream(stream));
}
