// C-ABI plumbing: error state, device checks, launch accounting, the
// device-resident quantized linear handle (K1 + K2 behind one call, with a
// host-buffer entry for end-to-end use) and the synthetic data generator.
#include <cuda_bf16.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <mutex>
#include <vector>
#include <new>

#include "common.cuh"

namespace qarvd_b200 {

namespace {
thread_local std::string g_last_error;
}

void set_error(const std::string& msg) { g_last_error = msg; }
void clear_error() { g_last_error.clear(); }
const char* last_error_cstr() { return g_last_error.c_str(); }

std::atomic<uint64_t>& launch_counter() {
  static std::atomic<uint64_t> counter{0};
  return counter;
}

int require_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    QARVD_FAIL(QARVD_ERR_CUDA, "no CUDA device available (this library has no CPU fallback)");
  }
  // Stream-ordered workspaces (K3 job tables, K4 histograms -- ~0.8 GB per calibration step)
  // come from the device's default memory pool; keep what it has instead of returning it to
  // the driver at every synchronisation (re-mapping the histograms each step cost up to
  // 10x the step itself when the caching allocators hold most of the device).
  static thread_local int pool_device = -1;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess && dev != pool_device) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
    pool_device = dev;
  }
  return QARVD_OK;
}


// ---- synthetic data ---------------------------------------------------------
namespace {

__device__ __forceinline__ uint64_t splitmix64_dev(uint64_t z) {
  // one splitmix64 output for counter state z (rng.hpp:11-16 constants)
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__global__ void synth_bf16_kernel(uint16_t* out, int64_t rows, int64_t cols, int64_t ld,
                                  uint64_t seed, float stddev) {
  const int64_t total = rows * cols;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    const uint64_t h = splitmix64_dev(seed ^ (static_cast<uint64_t>(i) * 0xd1b54a32d192ed03ULL));
    // Box-Muller on two 24-bit uniforms in (0, 1]
    const float u1 = (static_cast<float>(h >> 40) + 1.0f) * (1.0f / 16777216.0f);
    const float u2 = static_cast<float>((h >> 16) & 0xffffffu) * (1.0f / 16777216.0f);
    const float g = sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2);
    const __nv_bfloat16 b = __float2bfloat16_rn(g * stddev);
    out[r * ld + c] = *reinterpret_cast<const uint16_t*>(&b);
  }
}

__global__ void scale_cols_bf16_kernel(uint16_t* out, int64_t rows, int64_t ld,
                                       const int32_t* cols, int64_t ncols, float gamma) {
  const int64_t total = rows * ncols;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / ncols, j = i - r * ncols;
    uint16_t* p = out + r * ld + cols[j];
    const __nv_bfloat16 b = __float2bfloat16_rn(bf16_bits_to_float(*p) * gamma);
    *p = *reinterpret_cast<const uint16_t*>(&b);
  }
}

}  // namespace
}  // namespace qarvd_b200

using namespace qarvd_b200;

// ---- the quantized linear handle ---------------------------------------------
struct qarvd_linear {
  const int8_t* wq;
  int64_t n, k_pad, k_o, k_in;
  const int32_t* gather;
  const float* s_wo;
  const float* s_wn;
  const float* bias;
  int granularity;
  double static_scale;
  int epilogue;
  // workspace (grown on demand)
  int64_t cap_m = 0;
  int8_t* xq = nullptr;
  float* sx = nullptr;
  uint16_t* x_dev = nullptr;
  uint16_t* y_dev = nullptr;
  uint32_t* rowmax = nullptr;  // per-row |y| max for a chained consumer (zero between steps)
  uint64_t ws_gen = 0;         // process-unique id of the current workspace allocation
  // host-chain pipelining (owned by the chain's first layer): copy-in / copy-out streams and
  // per-chunk events, created on first use
  cudaStream_t s_in = nullptr, s_out = nullptr, s_cmp = nullptr;
  cudaEvent_t ev_start = nullptr, ev_in[8] = {}, ev_comp[8] = {}, ev_out = nullptr;
  // graph of the whole pipelined chain call, keyed by (host buffers, rows, layers)
  struct ChainGraph {
    const void* x_host = nullptr;
    void* y_host = nullptr;
    int64_t m = 0;
    std::vector<const qarvd_linear*> layers;
    std::vector<uint64_t> gens;
    int calls = 0;
    cudaGraphExec_t exec = nullptr;
  } chain_graph;
  std::mutex mu;  // forward() is re-entrant per handle (reference providers are shared const)
};

namespace {
// Workspace ids come from one process-wide counter, so a cached chain graph can never match a
// handle that was destroyed and re-created at the same address (its buffers are new).
std::atomic<uint64_t> g_ws_gen{0};

// Capturing cudaMemcpyAsync on pageable host memory is not permitted; only page-locked
// (cudaMallocHost / cudaHostRegister) buffers take the cached-graph path.
bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

int ensure_workspace(qarvd_linear* L, int64_t m, bool host_io) {
  if (m <= L->cap_m && (!host_io || L->x_dev)) return QARVD_OK;
  const int64_t cap = m > L->cap_m ? m : L->cap_m;
  cudaFree(L->xq);
  cudaFree(L->sx);
  cudaFree(L->x_dev);
  cudaFree(L->y_dev);
  cudaFree(L->rowmax);
  L->xq = nullptr;
  L->sx = nullptr;
  L->x_dev = nullptr;
  L->y_dev = nullptr;
  L->rowmax = nullptr;
  QARVD_CUDA_TRY(cudaMalloc(&L->xq, static_cast<size_t>(cap) * L->k_pad));
  QARVD_CUDA_TRY(cudaMalloc(&L->sx, static_cast<size_t>(cap) * sizeof(float)));
  QARVD_CUDA_TRY(cudaMalloc(&L->rowmax, static_cast<size_t>(cap) * sizeof(uint32_t)));
  QARVD_CUDA_TRY(cudaMemset(L->rowmax, 0, static_cast<size_t>(cap) * sizeof(uint32_t)));
  if (host_io) {
    QARVD_CUDA_TRY(cudaMalloc(&L->x_dev, static_cast<size_t>(cap) * L->k_in * 2));
    QARVD_CUDA_TRY(cudaMalloc(&L->y_dev, static_cast<size_t>(cap) * L->n * 2));
  }
  L->cap_m = cap;
  L->ws_gen = ++g_ws_gen;  // cached chain graphs referencing the old buffers are stale
  return QARVD_OK;
}

int linear_forward_dev(qarvd_linear* L, const uint16_t* x, int64_t m, uint16_t* y,
                       cudaStream_t s) {
  int st = qarvd_quantize_act(x, QARVD_BF16, m, L->k_in, L->k_in, L->gather, L->k_pad,
                              L->granularity, L->static_scale, 8, L->xq, L->k_pad, L->sx, nullptr,
                              nullptr, s);
  if (st) return st;
  return qarvd_dual_gemm(L->xq, L->k_pad, L->wq, L->k_pad, m, L->n, L->k_pad, L->k_o, L->sx,
                         L->s_wo, L->s_wn, L->bias, L->epilogue, QARVD_BF16, y, L->n, nullptr,
                         nullptr, s);
}
}  // namespace

extern "C" {

int qarvd_abi_version(void) { return QARVD_B200_ABI_VERSION; }
const char* qarvd_last_error(void) { return qarvd_b200::last_error_cstr(); }

int qarvd_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

uint64_t qarvd_launch_count(void) { return launch_counter().load(); }

int qarvd_linear_create(const int8_t* wq_dev, int64_t n, int64_t k_pad, int64_t k_outlier,
                        const int32_t* gather_dev, int64_t k_in, const float* scale_w_outlier_dev,
                        const float* scale_w_normal_dev, const float* bias_dev, int granularity,
                        double static_scale, int epilogue, qarvd_linear_t* out) {
  clear_error();
  if (!out || !wq_dev || !scale_w_normal_dev || n <= 0 || k_pad <= 0 || k_in <= 0)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "qarvd_linear_create: invalid argument");
  if (!gather_dev && k_in != k_pad)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "qarvd_linear_create: identity layout needs k_in == k_pad");
  if (k_pad % 32 || k_outlier % 32 || k_outlier < 0 || k_outlier >= k_pad)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "qarvd_linear_create: k_pad / k_outlier must be multiples of 32");
  if (granularity == QARVD_ACT_PER_TENSOR && !(static_scale > 0.0 && static_scale <= DBL_MAX))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "quant params: scale must be positive and finite");
  auto* L = new (std::nothrow) qarvd_linear();
  if (!L) QARVD_FAIL(QARVD_ERR_RUNTIME, "out of host memory");
  L->wq = wq_dev;
  L->n = n;
  L->k_pad = k_pad;
  L->k_o = k_outlier;
  L->k_in = k_in;
  L->gather = gather_dev;
  L->s_wo = k_outlier > 0 ? scale_w_outlier_dev : scale_w_normal_dev;
  L->s_wn = scale_w_normal_dev;
  L->bias = bias_dev;
  L->granularity = granularity;
  L->static_scale = static_scale;
  L->epilogue = epilogue;
  *out = L;
  return QARVD_OK;
}

int qarvd_linear_destroy(qarvd_linear_t L) {
  clear_error();
  if (!L) return QARVD_OK;
  cudaFree(L->xq);
  cudaFree(L->sx);
  cudaFree(L->x_dev);
  cudaFree(L->y_dev);
  cudaFree(L->rowmax);
  if (L->s_in) cudaStreamDestroy(L->s_in);
  if (L->s_out) cudaStreamDestroy(L->s_out);
  if (L->s_cmp) cudaStreamDestroy(L->s_cmp);
  for (cudaEvent_t ev : L->ev_in) if (ev) cudaEventDestroy(ev);
  for (cudaEvent_t ev : L->ev_comp) if (ev) cudaEventDestroy(ev);
  if (L->ev_start) cudaEventDestroy(L->ev_start);
  if (L->ev_out) cudaEventDestroy(L->ev_out);
  if (L->chain_graph.exec) cudaGraphExecDestroy(L->chain_graph.exec);
  delete L;
  return QARVD_OK;
}

int qarvd_linear_forward(qarvd_linear_t L, const uint16_t* x_dev, int64_t m, uint16_t* y_dev,
                         void* stream) {
  clear_error();
  if (!L || !x_dev || !y_dev || m <= 0)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "qarvd_linear_forward: invalid argument");
  if (int st = require_device()) return st;
  std::lock_guard<std::mutex> lock(L->mu);
  if (int st = ensure_workspace(L, m, false)) return st;
  return linear_forward_dev(L, x_dev, m, y_dev, as_stream(stream));
}

int qarvd_linear_forward_host(qarvd_linear_t L, const uint16_t* x_host, int64_t m,
                              uint16_t* y_host, void* stream) {
  clear_error();
  if (!L || !x_host || !y_host || m <= 0)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "qarvd_linear_forward_host: invalid argument");
  if (int st = require_device()) return st;
  std::lock_guard<std::mutex> lock(L->mu);
  if (int st = ensure_workspace(L, m, true)) return st;
  cudaStream_t s = as_stream(stream);
  QARVD_CUDA_TRY(cudaMemcpyAsync(L->x_dev, x_host, static_cast<size_t>(m) * L->k_in * 2,
                                 cudaMemcpyHostToDevice, s));
  if (int st = linear_forward_dev(L, L->x_dev, m, L->y_dev, s)) return st;
  QARVD_CUDA_TRY(cudaMemcpyAsync(y_host, L->y_dev, static_cast<size_t>(m) * L->n * 2,
                                 cudaMemcpyDeviceToHost, s));
  QARVD_CUDA_TRY(cudaStreamSynchronize(s));
  return QARVD_OK;
}

int qarvd_linear_chain_forward_host(const qarvd_linear_t* layers, int num_layers,
                                    const uint16_t* x_host, int64_t m, uint16_t* y_host,
                                    void* stream) {
  clear_error();
  if (!layers || num_layers <= 0 || !x_host || !y_host || m <= 0)
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "qarvd_linear_chain_forward_host: invalid argument");
  for (int i = 0; i + 1 < num_layers; ++i)
    if (!layers[i] || !layers[i + 1] || layers[i]->n != layers[i + 1]->k_in)
      QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "qarvd_linear_chain_forward_host: layer widths do not chain");
  if (int st = require_device()) return st;
  cudaStream_t s = as_stream(stream);
  // Lock each distinct handle once, in address order: a chain may repeat a handle (a square
  // layer applied twice), and concurrent chains sharing handles must not deadlock.
  std::vector<qarvd_linear*> locked(layers, layers + num_layers);
  std::sort(locked.begin(), locked.end());
  locked.erase(std::unique(locked.begin(), locked.end()), locked.end());
  for (qarvd_linear* L : locked) L->mu.lock();
  auto unlock_all = [&]() {
    for (auto it = locked.rbegin(); it != locked.rend(); ++it) (*it)->mu.unlock();
  };
  for (int i = 0; i < num_layers; ++i) {
    const int st = ensure_workspace(layers[i], m, true);
    if (st) {
      unlock_all();
      return st;
    }
  }
  // Row-chunk pipeline: chunk c's H2D (copy-in stream), K1+K2 per layer (the caller's
  // stream) and D2H (copy-out stream) are ordered by events, so the copies of neighbouring
  // chunks overlap the compute and each other (PCIe is full duplex).  QARVD_HOST_CHUNKS
  // overrides the chunk count (1 = the sequential H2D -> chain -> D2H).
  qarvd_linear* L0 = layers[0];
  // Equal row chunks, 128-row aligned (so the last one is the smallest).  Measured per Wan
  // FFN step (M = 4680, 3 x 300 steps each): 3 chunks 488 µs, 4: 469-477, 5: 447-455,
  // 6: 467-471; sequential 0.73 ms; the PCIe floor with both directions busy is 0.33 ms.
  // More chunks lose more GEMM efficiency -- N = 1536 has only 6 tile columns -- than they
  // gain in pipeline fill.
  int nchunks = m >= 2048 ? 5 : 1;
  if (const char* env = getenv("QARVD_HOST_CHUNKS")) nchunks = atoi(env);
  nchunks = nchunks < 1 ? 1 : (nchunks > 8 ? 8 : nchunks);
  int64_t bounds[9] = {0};
  {
    int64_t crow = (m + nchunks - 1) / nchunks;
    crow = (crow + 127) / 128 * 128;
    for (int c = 0; c < nchunks; ++c) bounds[c + 1] = (c + 1) * crow < m ? (c + 1) * crow : m;
  }
  // QARVD_HOST_CHUNK_ROWS="r0,r1,...": explicit leading chunk sizes (the rest is the last chunk),
  // for A/B.  Measured (round 2): small first / last chunks do not beat the equal split --
  // 384,1024x3 620 us, 256,768,1024x3 568, 256,512,1024x3,512 484, 6 equal 473, default 452.
  if (const char* env = getenv("QARVD_HOST_CHUNK_ROWS")) {
    int c = 0;
    int64_t acc = 0;
    const char* p = env;
    while (*p && c < 7) {
      const int64_t r = atoll(p);
      if (r <= 0 || acc + r >= m) break;
      acc += r;
      bounds[++c] = acc;
      while (*p && *p != ',') ++p;
      if (*p == ',') ++p;
    }
    bounds[++c] = m;
    nchunks = c;
  }
  cudaError_t e = cudaSuccess;
  if (!L0->s_in) {
    e = cudaStreamCreateWithFlags(&L0->s_in, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&L0->s_out, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&L0->s_cmp, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&L0->ev_start, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&L0->ev_out, cudaEventDisableTiming);
    for (int c = 0; c < 8 && e == cudaSuccess; ++c) {
      e = cudaEventCreateWithFlags(&L0->ev_in[c], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&L0->ev_comp[c], cudaEventDisableTiming);
    }
  }
  int st = QARVD_OK;
  cudaStream_t cs = L0->s_cmp;
  auto enqueue = [&]() {
    // A layer whose input already arrives in plan order (no gather: the producer's output
    // channels were folded, pipeline.fold_output_permutation) may take the streaming K1 with
    // the producer reducing the row |y| max in its epilogue
    // (off by default, like pipeline.QuantizedChain(fuse_rowmax=False); QARVD_FUSE_ROWMAX=1)
    static const bool fuse = getenv("QARVD_FUSE_ROWMAX") && getenv("QARVD_FUSE_ROWMAX")[0] == '1';
    auto streams_from = [&](int i) {
      return fuse && i + 1 < num_layers && !layers[i + 1]->gather && layers[i + 1]->k_in % 8 == 0;
    };
    const int64_t n_last = layers[num_layers - 1]->n;
    if (e == cudaSuccess) e = cudaEventRecord(L0->ev_start, cs);  // (cs waited for the caller's prior work)
    if (e == cudaSuccess) e = cudaStreamWaitEvent(L0->s_in, L0->ev_start, 0);
    for (int c = 0; c < nchunks && e == cudaSuccess && st == QARVD_OK; ++c) {
      const int64_t r0 = bounds[c];
      const int64_t rows = bounds[c + 1] - r0;
      if (rows <= 0) continue;
      e = cudaMemcpyAsync(L0->x_dev + r0 * L0->k_in, x_host + r0 * L0->k_in,
                          static_cast<size_t>(rows) * L0->k_in * 2, cudaMemcpyHostToDevice, L0->s_in);
      if (e == cudaSuccess) e = cudaEventRecord(L0->ev_in[c], L0->s_in);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, L0->ev_in[c], 0);
      const uint16_t* in = L0->x_dev + r0 * L0->k_in;
      for (int i = 0; i < num_layers && e == cudaSuccess && st == QARVD_OK; ++i) {
        qarvd_linear* L = layers[i];
        int8_t* xq = L->xq + r0 * L->k_pad;
        float* sx = L->sx + r0;
        uint16_t* yo = L->y_dev + r0 * L->n;
        if (i > 0 && streams_from(i - 1)) {
          qarvd_linear* P = layers[i - 1];
          st = qarvd_quantize_act_rowmax(in, rows, L->k_in, L->k_in,
                                         L->granularity == QARVD_ACT_PER_TOKEN ? P->rowmax + r0 : nullptr,
                                         L->granularity, L->static_scale, 8, xq, L->k_pad, sx, nullptr,
                                         nullptr, cs);
        } else {
          st = qarvd_quantize_act(in, QARVD_BF16, rows, L->k_in, L->k_in, L->gather, L->k_pad,
                                  L->granularity, L->static_scale, 8, xq, L->k_pad, sx, nullptr,
                                  nullptr, cs);
        }
        if (st) break;
        if (streams_from(i) && layers[i + 1]->granularity == QARVD_ACT_PER_TOKEN)
          st = qarvd_dual_gemm_rowmax(xq, L->k_pad, L->wq, L->k_pad, rows, L->n, L->k_pad, L->k_o, sx,
                                      L->s_wo, L->s_wn, L->bias, L->epilogue, yo, L->n, L->rowmax + r0, cs);
        else
          st = qarvd_dual_gemm(xq, L->k_pad, L->wq, L->k_pad, rows, L->n, L->k_pad, L->k_o, sx, L->s_wo,
                               L->s_wn, L->bias, L->epilogue, QARVD_BF16, yo, L->n, nullptr, nullptr, cs);
        in = yo;
      }
      if (st) break;
      e = cudaEventRecord(L0->ev_comp[c], cs);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(L0->s_out, L0->ev_comp[c], 0);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(y_host + r0 * n_last, in, static_cast<size_t>(rows) * n_last * 2,
                            cudaMemcpyDeviceToHost, L0->s_out);
    }
    if (e == cudaSuccess) e = cudaEventRecord(L0->ev_out, L0->s_out);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, L0->ev_out, 0);
  };
  // The first call for a (host buffers, rows, layers) key runs eagerly (it also performs
  // first-use setup: kernel attributes, occupancy queries), the second captures the whole
  // pipelined sequence -- copies, events, both streams -- into a graph, later calls replay it
  // (one launch instead of ~16 kernel launches and 8 copies; QARVD_HOST_GRAPH=0 disables).
  static const bool graph_enabled =
      !(getenv("QARVD_HOST_GRAPH") && getenv("QARVD_HOST_GRAPH")[0] == '0');
  const bool use_graph = graph_enabled && is_pinned(x_host) && is_pinned(y_host);
  auto& cg = L0->chain_graph;
  std::vector<const qarvd_linear*> key(layers, layers + num_layers);
  std::vector<uint64_t> gens;
  for (int i = 0; i < num_layers; ++i) gens.push_back(layers[i]->ws_gen);
  if (cg.x_host != x_host || cg.y_host != y_host || cg.m != m || cg.layers != key || cg.gens != gens) {
    if (cg.exec) cudaGraphExecDestroy(cg.exec);
    cg = qarvd_linear::ChainGraph{};
    cg.x_host = x_host;
    cg.y_host = y_host;
    cg.m = m;
    cg.layers = key;
    cg.gens = gens;
  }
  // all pipelined work runs on the chain's own compute stream (capturable even when the
  // caller passes the legacy default stream), forked from and joined back to `s`
  if (e == cudaSuccess) e = cudaEventRecord(L0->ev_start, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, L0->ev_start, 0);
  if (e == cudaSuccess && use_graph && cg.exec) {
    e = cudaGraphLaunch(cg.exec, cs);
  } else if (e == cudaSuccess && use_graph && cg.calls == 1) {
    cudaGraph_t g = nullptr;
    e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      enqueue();
      cudaGraph_t tmp = nullptr;
      const cudaError_t ec = cudaStreamEndCapture(cs, &tmp);
      if (e == cudaSuccess) e = ec;
      g = tmp;
    }
    if (e == cudaSuccess && st == QARVD_OK) e = cudaGraphInstantiate(&cg.exec, g, 0);
    if (g) cudaGraphDestroy(g);
    if (e == cudaSuccess && st == QARVD_OK) e = cudaGraphLaunch(cg.exec, cs);
  } else if (e == cudaSuccess) {
    enqueue();
  }
  ++cg.calls;
  if (e == cudaSuccess) e = cudaEventRecord(L0->ev_out, cs);  // join back to the caller
  if (e == cudaSuccess) e = cudaStreamWaitEvent(s, L0->ev_out, 0);
  if (e == cudaSuccess && st == QARVD_OK) {
    e = cudaStreamSynchronize(s);
  } else {  // drain whatever was enqueued before releasing the workspaces
    if (L0->s_in) cudaStreamSynchronize(L0->s_in);
    if (L0->s_out) cudaStreamSynchronize(L0->s_out);
    cudaStreamSynchronize(s);
  }
  unlock_all();
  if (st) return st;
  QARVD_CUDA_TRY(e);
  return QARVD_OK;
}

int qarvd_synth_bf16(uint16_t* out, int64_t rows, int64_t cols, int64_t ld, uint64_t seed,
                     double stddev, const int32_t* outlier_cols, int64_t num_outliers,
                     double gamma, void* stream) {
  clear_error();
  if (!out || rows < 0 || cols <= 0 || ld < cols || num_outliers < 0 ||
      (num_outliers > 0 && !outlier_cols))
    QARVD_FAIL(QARVD_ERR_INVALID_ARGUMENT, "qarvd_synth_bf16: invalid argument");
  if (int st = require_device()) return st;
  if (rows == 0) return QARVD_OK;
  cudaStream_t s = as_stream(stream);
  synth_bf16_kernel<<<kNumSMs * 8, 256, 0, s>>>(out, rows, cols, ld, seed,
                                                static_cast<float>(stddev));
  count_launch();
  QARVD_LAUNCH_CHECK();
  if (num_outliers > 0) {
    scale_cols_bf16_kernel<<<kNumSMs * 4, 256, 0, s>>>(out, rows, ld, outlier_cols, num_outliers,
                                                       static_cast<float>(gamma));
    count_launch();
    QARVD_LAUNCH_CHECK();
  }
  return QARVD_OK;
}

}  // extern "C"
