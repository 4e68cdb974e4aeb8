// Eq. 5 — the frame-weighted output-space reconstruction objective on the tensor cores.
//
// Replaces weighted_recon_loss / weighted_loss (/root/reference/proj/core/src/
// calibrate.cpp:201-224): for every calibration sample X_s (rows of one captured chunk)
//     err_s = || X_s W^T - FQ(X_s) What^T ||_F^2,   loss = (1/B) sum_s w[chunk_s] err_s.
// The reference runs two f64 GEMMs per sample and materialises both [rows x N] outputs.
// Here ONE persistent kernel computes, per 256 x 128 output tile (an SM pair,
// cta_group::2, 256-byte K stages), three tensor-memory
// accumulators from one shared-memory pipeline:
//   acc_t = X W^T            tcgen05.mma.kind::f16 (bf16 x bf16 -> f32), K = 16 per MMA
//   acc_o = xq_o . wq_o^T    tcgen05.mma.kind::i8 over the outlier K-slab (k < K_o)
//   acc_n = xq_n . wq_n^T    tcgen05.mma.kind::i8 over the normal K-slab
// and the epilogue reduces d = acc_t - s_x (s_wo acc_o + s_wn acc_n) to per-row partial
// sums of d^2 (f64) without writing either GEMM output.  X / W are bf16 in the original
// column order (the target's order is irrelevant to the product); xq / wq are the K1 / K5
// int8 codes in plan order ([outlier | normal], K_o a multiple of 32).  A second kernel sums
// the partials per sample in a fixed order and a third forms the weighted mean, so the
// result is deterministic (no floating-point atomics).
//
// TMEM: four 128-column slots; tile i of a CTA uses slots 3i, 3i+1, 3i+2 (mod 4) for
// (acc_t, acc_o, acc_n).  The next tile's bf16 phase accumulates into the spare slot while
// the epilogue drains the previous tile; its int8 phase waits only for the slots it reuses.
// Warp roles: 0 = TMA producer, 1 = MMA issuer (leader CTA), 2 = TMEM allocator,
// 4..11 = epilogue (two warps per TMEM lane quadrant, 64 columns each, in both CTAs).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "ptx.cuh"

namespace qarvd_b200 {
namespace {

constexpr int LBM = 128;          // rows per CTA (TMEM lanes); an SM pair computes 256-row tiles
constexpr int LTM = 2 * LBM;      // rows of a pair tile
constexpr int LBN = 256;          // columns per tile (each CTA of the pair holds half of B)
constexpr int LKS = 2;            // 128-byte K sub-tiles per stage (8 MMAs per mbarrier wait)
constexpr int kLossSubA = LBM * 128;
constexpr int kLossSubB = (LBN / 2) * 128;
constexpr int kLossStageA = LKS * kLossSubA;
constexpr int kLossStageB = LKS * kLossSubB;
constexpr int kLossStageBytes = kLossStageA + kLossStageB;
constexpr int kLossStages = 3;
constexpr int kLossEpiWarps = 16;  // 4 per TMEM lane quadrant, 64 columns each
constexpr int kLossThreads = 128 + 32 * kLossEpiWarps;
constexpr int kLossCtrlRegs = 32;  // setmaxnreg split of 640 x 96 registers
constexpr int kLossEpiRegs = 112;
constexpr size_t kLossSmem = static_cast<size_t>(kLossStages) * kLossStageBytes + 1024;
constexpr int kLossParts = 4;      // column partials per row and tile (one per epilogue warp)

struct LossParams {
  int64_t m, n, k, k_pad, k_o;
  const float* scale_x;   // [m]
  const float* scale_wo;  // [n]
  const float* scale_wn;  // [n]
  double* part;           // [kLossParts * num_n_blks][m] per-row partial sums of d^2
  int num_m_blks, num_n_blks, num_tiles;
};

// kind::f16 instruction descriptor: D = F32 (c_format 1), A = B = BF16 (format 1), K-major.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Stage sequence of one tile: F1 (first half of the bf16 target stages), O (int8 stages holding
// outlier steps; only those issue), F2 (the other bf16 stages), N (int8 stages holding normal
// steps).  Every TMEM hand-off then overlaps MMA work: acc_o is folded during F2, acc_t read
// during N, acc_n read during the next tile's F1.  A stage straddling K_o loads in O and N.
struct LossPhases {
  int no, nf, nf1, nn, n0;  // stage counts; n0 = first int8 stage of N
  __device__ LossPhases(const LossParams& p) {
    const int ko32 = static_cast<int>(p.k_o / 32), k32 = static_cast<int>(p.k_pad / 32);
    no = (ko32 + 4 * LKS - 1) / (4 * LKS);
    nf = static_cast<int>((p.k + 64 * LKS - 1) / (64 * LKS));
    nf1 = no > 0 ? nf / 2 : nf;
    n0 = ko32 / (4 * LKS);
    nn = (k32 + 4 * LKS - 1) / (4 * LKS) - n0;
  }
  __device__ int total() const { return no + nf + nn; }
  // stage i of a tile -> kind (0 bf16, 1 int8 outlier, 2 int8 normal) and K block
  __device__ void at(int i, int& kind, int& blk) const {
    if (i < nf1) { kind = 0; blk = i; }
    else if (i < nf1 + no) { kind = 1; blk = i - nf1; }
    else if (i < nf + no) { kind = 0; blk = i - no; }
    else { kind = 2; blk = n0 + i - nf - no; }
  }
};

// SM-pair kernel (cluster of 2, cta_group::2).  TMEM: R1 = columns [0, 256) hold acc_t; R2 =
// [256, 512) holds acc_o, then (after the epilogue folded s_wo*acc_o into registers) acc_n.
// Epilogue per row and column: e = acc_t - s_x*(s_wo*acc_o) once acc_t lands (R1 released),
// then d = e - s_x*(s_wn*acc_n) once acc_n lands (R2 released).
__global__ void __launch_bounds__(kLossThreads, 1)
    recon_loss_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                      const __grid_constant__ CUtensorMap tmXq, const __grid_constant__ CUtensorMap tmWq,
                      const LossParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + kLossStages * kLossStageA;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kLossStages * kLossStageBytes);
  uint64_t* empty = full + kLossStages;
  uint64_t* ofull = empty + kLossStages;  // acc_o complete (both CTAs)
  uint64_t* ffull = ofull + 1;            // acc_t complete (both CTAs)
  uint64_t* tfull = ffull + 1;            // acc_n complete: tile done (both CTAs)
  uint64_t* r1free = tfull + 1;           // R1 read by every epilogue warp (leader's copy)
  uint64_t* r2free = r1free + 1;          // R2 read (once per use)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(r2free + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = static_cast<int>(blockIdx.x) / 2;
  const int num_pairs = static_cast<int>(gridDim.x) / 2;
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmX);
    ptx::prefetch_tmap(&tmW);
    ptx::prefetch_tmap(&tmXq);
    ptx::prefetch_tmap(&tmWq);
    for (int s = 0; s < kLossStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(ofull, 1);
    ptx::mbar_init(ffull, 1);
    ptx::mbar_init(tfull, 1);
    ptx::mbar_init(r1free, 2 * kLossEpiWarps);
    ptx::mbar_init(r2free, 2 * kLossEpiWarps);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc_2sm(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();  // peer barriers initialised before any remote arrive
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();

  const LossPhases ph(p);
  const int k16 = static_cast<int>((p.k + 15) / 16);
  const int k32 = static_cast<int>(p.k_pad / 32), ko32 = static_cast<int>(p.k_o / 32);
  const bool has_o = ko32 > 0;

  if (warp == 0) {
    // ===================== TMA producer (both CTAs; bytes land on the leader's barrier) =====
    ptx::setmaxnreg_dec<kLossCtrlRegs>();
    int stage = 0;
    uint32_t phase = 0;
    for (int t = pair; t < p.num_tiles; t += num_pairs) {
      // n-fastest tile order: the pairs in flight share a few A row blocks (L2-resident), so X
      // and xq stream from HBM about once instead of once per column block
      const int a_row = (t / p.num_n_blks) * LTM + static_cast<int>(rank) * LBM;
      const int b_row = (t % p.num_n_blks) * LBN + static_cast<int>(rank) * (LBN / 2);
      for (int i = 0; i < ph.total(); ++i) {
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        if (lane == 0) {
          if (leader) ptx::mbar_expect_tx(&full[stage], 2 * kLossStageBytes);
          int kind, blk;
          ph.at(i, kind, blk);
          const bool bf = kind == 0;
#pragma unroll
          for (int ks = 0; ks < LKS; ++ks) {
            uint8_t* a = sA + stage * kLossStageA + ks * kLossSubA;
            uint8_t* b = sB + stage * kLossStageB + ks * kLossSubB;
            if (bf) {
              const int kc = (blk * LKS + ks) * 64;
              ptx::tma_load_2d_2sm(a, &tmX, &full[stage], kc, a_row);
              ptx::tma_load_2d_2sm(b, &tmW, &full[stage], kc, b_row);
            } else {
              const int kc = (blk * LKS + ks) * 128;
              ptx::tma_load_2d_2sm(a, &tmXq, &full[stage], kc, a_row);
              ptx::tma_load_2d_2sm(b, &tmWq, &full[stage], kc, b_row);
            }
          }
        }
        __syncwarp();
        if (++stage == kLossStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA) =====================
    ptx::setmaxnreg_dec<kLossCtrlRegs>();
    if (leader) {
      constexpr uint32_t id_f = idesc_bf16(LTM, LBN);
      constexpr uint32_t id_i = ptx::idesc_i8(LTM, LBN);
      const uint64_t a0 = ptx::sw128_kmajor_desc(ptx::smem_u32(sA));
      const uint64_t b0 = ptx::sw128_kmajor_desc(ptx::smem_u32(sB));
      const uint32_t r1 = tmem_base, r2 = tmem_base + LBN;
      int stage = 0;
      uint32_t phase = 0, u1 = 0, u2 = 0;  // uses of R1 / R2 so far
      auto take = [&](uint64_t* bar, uint32_t& u) {
        ptx::mbar_wait(bar, (u & 1u) ^ 1u);
        ++u;
        ptx::tc_fence_after();
      };
      for (int t = pair; t < p.num_tiles; t += num_pairs) {
        for (int i = 0; i < ph.total(); ++i) {
          int kind, blk;
          ph.at(i, kind, blk);
          if (kind == 0 && blk == 0) take(r1free, u1);        // acc_t(prev) read
          if (kind == 1 && blk == 0) take(r2free, u2);        // acc_n(prev) read
          if (kind == 2 && blk == ph.n0) take(r2free, u2);    // acc_o folded (or acc_n(prev) read)
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint64_t ad = a0 + static_cast<uint64_t>(stage * (kLossStageA >> 4));
          const uint64_t bd = b0 + static_cast<uint64_t>(stage * (kLossStageB >> 4));
          if (lane == 0) {
#pragma unroll
            for (int j = 0; j < 4 * LKS; ++j) {
              const uint64_t ao = static_cast<uint64_t>((j >> 2) * (kLossSubA >> 4) + 2 * (j & 3));
              const uint64_t bo = static_cast<uint64_t>((j >> 2) * (kLossSubB >> 4) + 2 * (j & 3));
              if (kind == 0) {
                const int s16 = blk * 4 * LKS + j;
                if (s16 < k16) mma_bf16_2sm(r1, ad + ao, bd + bo, id_f, s16 > 0 ? 1u : 0u);
              } else {
                const int s32 = blk * 4 * LKS + j;
                const bool outl = kind == 1;
                if (s32 < k32 && (s32 < ko32) == outl) {
                  const uint32_t acc = (outl ? s32 == 0 : s32 == ko32) ? 0u : 1u;
                  ptx::mma_i8_2sm(r2, ad + ao, bd + bo, id_i, acc);
                }
              }
            }
            ptx::mma_commit_2sm_mc(&empty[stage], 0x3);
            if (kind == 1 && blk == ph.no - 1) ptx::mma_commit_2sm_mc(ofull, 0x3);
            if (kind == 0 && blk == ph.nf - 1) ptx::mma_commit_2sm_mc(ffull, 0x3);
          }
          __syncwarp();
          if (++stage == kLossStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (lane == 0) ptx::mma_commit_2sm_mc(tfull, 0x3);
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue (both CTAs, own 128 rows) =====================
    ptx::setmaxnreg_inc<kLossEpiRegs>();
    const int ew = warp - 4;
    const int q = warp & 3;          // TMEM lane quadrant
    const int h = ew >> 2;           // 64-column quarter of the tile
    const uint32_t t_lane = static_cast<uint32_t>(q * 32) << 16;
    const uint32_t r1 = tmem_base + t_lane + static_cast<uint32_t>(h * 64);
    const uint32_t r2 = r1 + LBN;
    int ti = 0;
    for (int t = pair; t < p.num_tiles; t += num_pairs, ++ti) {
      const int m_blk = t / p.num_n_blks, n_blk = t % p.num_n_blks;
      const int64_t row = static_cast<int64_t>(m_blk) * LTM + rank * LBM + q * 32 + lane;
      const int64_t col0 = static_cast<int64_t>(n_blk) * LBN + h * 64;
      const float sx = row < p.m ? p.scale_x[row] : 0.f;
      float ev[64];  // s_wo*acc_o, then e = acc_t - s_x*(s_wo*acc_o), of this row's 64 columns
      if (has_o) {
        ptx::mbar_wait(ofull, ti & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int c = 0; c < 64; c += 16) {
          uint32_t ro[16];
          ptx::tmem_ld16(r2 + c, ro);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int64_t j = col0 + c + e;
            const float swo = j < p.n ? __ldg(p.scale_wo + j) : 0.f;
            ev[c + e] = __fmul_rn(swo, __int2float_rn(static_cast<int>(ro[e])));
          }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_leader(r2free);
      } else {
#pragma unroll
        for (int c = 0; c < 64; ++c) ev[c] = 0.f;
      }
      ptx::mbar_wait(ffull, ti & 1);
      ptx::tc_fence_after();
#pragma unroll
      for (int c = 0; c < 64; c += 16) {
        uint32_t rt[16];
        ptx::tmem_ld16(r1 + c, rt);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 16; ++e)
          ev[c + e] = __fmaf_rn(-sx, ev[c + e], __uint_as_float(rt[e]));
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_leader(r1free);
      ptx::mbar_wait(tfull, ti & 1);
      ptx::tc_fence_after();
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < 64; c += 16) {
        uint32_t rn[16];
        ptx::tmem_ld16(r2 + c, rn);
        ptx::tmem_wait_ld();
        float part = 0.f;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int64_t j = col0 + c + e;
          const float swn = j < p.n ? __ldg(p.scale_wn + j) : 0.f;
          const float d = __fmaf_rn(-sx, __fmul_rn(swn, __int2float_rn(static_cast<int>(rn[e]))), ev[c + e]);
          part = __fmaf_rn(d, d, part);
        }
        acc += static_cast<double>(part);
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_leader(r2free);
      if (row < p.m) p.part[static_cast<int64_t>(kLossParts * n_blk + h) * p.m + row] = acc;
    }
  } else {
    ptx::setmaxnreg_dec<kLossCtrlRegs>();  // warps 2-3
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();  // the leader's MMAs wrote this CTA's TMEM / read its smem
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_2sm(tmem_base, 512);
  }
}

// err[s] = sum over the sample's rows and all column partials, in a fixed order:
// thread i sums rows r0+i, r0+i+256, ... (partials in column-block order), then a
// fixed-shape tree over the 256 thread sums.
constexpr int kReduceThreads = 256;
__global__ void __launch_bounds__(kReduceThreads)
    sample_err_kernel(const double* part, int64_t m, int pcount, const int64_t* row_off,
                      double* err) {
  const int s = blockIdx.x;
  const int64_t r0 = row_off[s], r1 = row_off[s + 1];
  double acc = 0.0;
  for (int64_t r = r0 + threadIdx.x; r < r1; r += kReduceThreads) {
    double rs = 0.0;
    for (int c = 0; c < pcount; ++c) rs += part[static_cast<int64_t>(c) * m + r];
    acc += rs;
  }
  __shared__ double red[kReduceThreads];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = kReduceThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) err[s] = red[0];
}

// loss = (sum_s wsamp[s] * err[s]) / B, summed in sample order (calibrate.cpp:212-215)
__global__ void weighted_mean_kernel(const double* err, const double* wsamp, int64_t b,
                                     double* loss) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double total = 0.0;
  for (int64_t s = 0; s < b; ++s) total += wsamp[s] * err[s];
  *loss = total / static_cast<double>(b);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

// K-major [rows x cols] operand, box = 128 bytes of K x 128 rows, 128B swizzle
int make_kmajor_tmap(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int esize,
                     int64_t rows, int64_t cols, int64_t ld_elems, int box_rows) {
  auto encode = encode_fn();
  if (!encode) QARVD_FAIL(QARVD_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld_elems * esize)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / esize), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    QARVD_FAIL(QARVD_ERR_CUDA, "cuTensorMapEncodeTiled failed with CUresult " + std::to_string(r));
  return QARVD_OK;
}

int loss_sm_count() {
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

int64_t part_count(int64_t n) { return kLossParts * ((n + LBN - 1) / LBN); }

}  // namespace
}  // namespace qarvd_b200

using namespace qarvd_b200;

extern "C" int64_t qarvd_weighted_loss_workspace(int64_t m, int64_t n, int64_t n_samples) {
  if (m <= 0 || n <= 0 || n_samples <= 0) return 0;
  // partials [2*n_blks][m] f64, then row offsets (B+1) i64, per-sample weights B f64
  return (part_count(n) * m + (n_samples + 1) + n_samples) * 8;
}

extern "C" int qarvd_weighted_loss(const uint16_t* x, int64_t ldx, const uint16_t* w, int64_t ldw,
                                   const int8_t* xq, int64_t ldq, const int8_t* wq, int64_t ldwq,
                                   int64_t m, int64_t n, int64_t k, int64_t k_pad, int64_t k_outlier,
                                   const float* scale_x, const float* scale_w_outlier,
                                   const float* scale_w_normal, const int64_t* sample_rows,
                                   const int64_t* sample_chunk, int64_t n_samples,
                                   const double* chunk_weights, int64_t n_chunks, double* sample_err,
                                   double* loss, void* workspace, int64_t workspace_bytes,
                                   void* stream) {
  clear_error();
  if (n_samples <= 0) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "weighted loss: empty batch");
  if (!sample_rows || !sample_chunk || !chunk_weights)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "weighted loss: null sample metadata");
  // calibrate.cpp:207-208: every sample's 1-based chunk must index the weight vector
  for (int64_t s = 0; s < n_samples; ++s)
    if (sample_chunk[s] < 1 || sample_chunk[s] > n_chunks)
      QARVD_FAIL(QARVD_ERR_OUT_OF_RANGE, "weighted loss: sample chunk outside the weight vector");
  if (sample_rows[0] != 0 || sample_rows[n_samples] != m)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "weighted loss: sample rows must partition [0, m)");
  for (int64_t s = 0; s < n_samples; ++s)
    if (sample_rows[s + 1] < sample_rows[s])
      QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "weighted loss: sample rows must be non-decreasing");
  if (m <= 0 || n <= 0 || k <= 0) QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "weighted loss: empty shape");
  if (k_pad % 32 || k_outlier % 32 || k_outlier < 0 || k_outlier >= k_pad)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT,
               "weighted loss: k_pad and k_outlier must be multiples of 32 with 0 <= k_outlier < k_pad");
  if (k_pad > 132104)
    QARVD_FAIL(QARVD_ERR_LOGIC, "weighted loss: reduction dimension too large for exact int32 accumulation");
  if (ldx < k || ldw < k || ldq < k_pad || ldwq < k_pad || ldx % 8 || ldw % 8 || ldq % 16 || ldwq % 16)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "weighted loss: invalid leading dimension");
  if (!x || !w || !xq || !wq || !scale_x || !scale_w_normal || !loss || !sample_err ||
      (k_outlier > 0 && !scale_w_outlier))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "weighted loss: null pointer argument");
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w) |
       reinterpret_cast<uintptr_t>(xq) | reinterpret_cast<uintptr_t>(wq)) & 15)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "weighted loss: operand pointers must be 16-byte aligned");
  const int64_t need = qarvd_weighted_loss_workspace(m, n, n_samples);
  if (!workspace || workspace_bytes < need || (reinterpret_cast<uintptr_t>(workspace) & 7))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "weighted loss: workspace too small (see qarvd_weighted_loss_workspace)");
  if (int st = require_device()) return st;
  cudaStream_t s = as_stream(stream);

  static std::once_flag attr_once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(attr_once, [] { attr_err = set_smem_attrs(recon_loss_kernel, static_cast<int>(kLossSmem)); });
  QARVD_CUDA_TRY(attr_err);
  CUtensorMap tx, tw, txq, twq;
  int st;
  if ((st = make_kmajor_tmap(&tx, x, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, m, k, ldx, LBM))) return st;
  if ((st = make_kmajor_tmap(&tw, w, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, n, k, ldw, LBN / 2))) return st;
  if ((st = make_kmajor_tmap(&txq, xq, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, m, k_pad, ldq, LBM))) return st;
  if ((st = make_kmajor_tmap(&twq, wq, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, n, k_pad, ldwq, LBN / 2))) return st;

  LossParams p{};
  p.m = m;
  p.n = n;
  p.k = k;
  p.k_pad = k_pad;
  p.k_o = k_outlier;
  p.scale_x = scale_x;
  p.scale_wo = scale_w_outlier;
  p.scale_wn = scale_w_normal;
  p.num_m_blks = static_cast<int>((m + LTM - 1) / LTM);
  p.num_n_blks = static_cast<int>((n + LBN - 1) / LBN);
  p.num_tiles = p.num_m_blks * p.num_n_blks;
  double* ws = static_cast<double*>(workspace);
  p.part = ws;
  const int64_t pc = part_count(n);
  int64_t* d_rows = reinterpret_cast<int64_t*>(ws + pc * m);
  double* d_wsamp = ws + pc * m + (n_samples + 1);
  // sample metadata: host -> workspace (weights resolved per sample on the host)
  std::vector<double> wsamp(static_cast<size_t>(n_samples));
  for (int64_t i = 0; i < n_samples; ++i) wsamp[i] = chunk_weights[sample_chunk[i] - 1];
  QARVD_CUDA_TRY(cudaMemcpyAsync(d_rows, sample_rows, sizeof(int64_t) * (n_samples + 1),
                                 cudaMemcpyHostToDevice, s));
  QARVD_CUDA_TRY(cudaMemcpyAsync(d_wsamp, wsamp.data(), sizeof(double) * n_samples,
                                 cudaMemcpyHostToDevice, s));
  const int pairs = loss_sm_count() / 2;
  const int grid = 2 * (p.num_tiles < pairs ? p.num_tiles : pairs);
  QARVD_CUDA_TRY(launch_pdl(recon_loss_kernel, dim3(grid), dim3(kLossThreads), kLossSmem, s, 2, tx,
                            tw, txq, twq, p));
  count_launch();
  QARVD_LAUNCH_CHECK();
  double* err = sample_err;
  sample_err_kernel<<<static_cast<unsigned>(n_samples), kReduceThreads, 0, s>>>(
      p.part, m, static_cast<int>(pc), d_rows, err);
  count_launch();
  QARVD_LAUNCH_CHECK();
  weighted_mean_kernel<<<1, 32, 0, s>>>(err, d_wsamp, n_samples, loss);
  count_launch();
  QARVD_LAUNCH_CHECK();
  // the host metadata vector dies with this call: pageable copies are staged at enqueue
  return QARVD_OK;
}
