// tlora_capi.cu — implementation of the C-ABI in include/tlora.h.
//
// Host side: layer registry (frozen base + packed adapters), plan upload, launch
// sequencing of the six tcgen05 GEMM launches per fused fwd+bwd, and the reference
// cost model / nano-batch plan / AIMD restated bit-exactly.  No CPU compute path:
// every numeric entry point enqueues sm_100a kernels and fails if there is no device.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <tuple>
#include <memory>
#include <atomic>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tlora.h"
#include "lora_gemm.cuh"
#include "lora_gemm2.cuh"
#include "lora_grad.cuh"
#include "tlora_plan.hpp"

using tlora::GemmArgs;
using tlora::TileDesc;

namespace {

thread_local std::string g_last_error;

struct Status : std::runtime_error {
  int code;
  Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define TL_CUDA(x)                                                                         \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      throw Status(TLORA_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));       \
  } while (0)

template <class F>
int guarded(F&& f) {
  try {
    (void)cudaGetLastError();  // drop stale non-sticky errors of unrelated earlier calls
    f();
    return TLORA_OK;
  } catch (const Status& s) {
    g_last_error = s.what();
    return s.code;
  } catch (const std::out_of_range& e) {
    g_last_error = e.what();
    return TLORA_ERR_REGISTRY;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return TLORA_ERR_PLAN;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return TLORA_ERR_ARG;
  }
}

void require(bool ok, int code, const std::string& msg) {
  if (!ok) throw Status(code, msg);
}

// ------------------------------------------------------------------ TMA descriptors
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  require(fn != nullptr, TLORA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// 2-D bf16 row-major [outer x inner] with leading dimension ld (elements), 128B swizzle.
CUtensorMap make_tmap(const void* ptr, int64_t inner, int64_t outer, int64_t ld, int box_inner,
                      int box_outer) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  require(r == CUDA_SUCCESS, TLORA_ERR_CUDA,
          "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}
// K-major operand tile: [rows x 64] boxes.
CUtensorMap tmap_k(const void* p, int64_t K, int64_t rows, int box_rows) {
  return make_tmap(p, K, rows, K, tlora::kBK, box_rows);
}
// MN-major operand tile: [64 K-rows x 64 MN] boxes over a [K x MN] row-major matrix.
CUtensorMap tmap_mn(const void* p, int64_t MN, int64_t K) {
  return make_tmap(p, MN, K, MN, 64, tlora::kBK);
}

// ------------------------------------------------------------------ SM budgets
// Persistent grids are sized to min(tiles, budget). Splitting the SMs between the
// tensor-bound fused GEMMs and the HBM-bound low-rank launches lets a driver run the two
// concurrently on two streams (tlora_set_sm_budget). 0 = all SMs.
std::mutex g_budget_mu;
std::map<int, std::pair<int, int>> g_budget;  // device -> (gemm SMs, low-rank SMs)

int sm_budget(int device, int all, bool gemm) {
  std::lock_guard<std::mutex> lk(g_budget_mu);
  auto it = g_budget.find(device);
  if (it == g_budget.end()) return all;
  const int b = gemm ? it->second.first : it->second.second;
  return b > 0 ? std::min(b, all) : all;
}

// ------------------------------------------------------------------ launch profiling
// Optional CUDA-event brackets around every GEMM launch, recorded on the launch stream
// (tlora_profile_begin/_end). Used by bench.py for the live roofline of each launch kind.
struct ProfRec {
  int launch;
  double flops;
  cudaEvent_t e0, e1;
};
std::mutex g_prof_mu;
std::atomic<long long> g_launches{0};  // every kernel this library enqueues
bool g_prof_on = false;
std::vector<ProfRec> g_prof;

struct ProfScope {
  ProfRec rec{};
  cudaStream_t s;
  bool on = false;
  unsigned flags = 0;
  ProfScope(int launch, double flops, cudaStream_t st) : s(st) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (!g_prof_on) return;
    on = true;
    rec.launch = launch;
    rec.flops = flops;
    TL_CUDA(cudaEventCreate(&rec.e0));
    TL_CUDA(cudaEventCreate(&rec.e1));
    // under CUDA-graph capture a plain record only expresses a dependency; External makes
    // it an event-record node that every replay re-records
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    TL_CUDA(cudaStreamIsCapturing(s, &cs));
    flags = cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0u;
    TL_CUDA(cudaEventRecordWithFlags(rec.e0, s, flags));
  }
  ~ProfScope() {
    if (!on) return;
    cudaEventRecordWithFlags(rec.e1, s, flags);
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof.push_back(rec);
  }
};

// ------------------------------------------------------------------ launch helpers
// Launch a persistent kernel with programmatic stream serialisation (PDL): it may begin
// while the previous kernel on the stream drains; the kernel itself waits
// (griddepcontrol.wait) before touching data the previous launch produced.
template <typename Kern, typename... Args>
void launch_pdl(Kern kern, int grid, int smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(tlora::kGemmThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = TLORA_PDL ? 1 : 0;
  TL_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}

template <int BN, bool AMN, bool BMN, int EPI, int ST>
void launch_gemm(const CUtensorMap& a0, const CUtensorMap& b0, const CUtensorMap& a1,
                 const CUtensorMap& b1, const GemmArgs& args, int sm_count, cudaStream_t s,
                 int launch_kind = -1, double flops = 0.0) {
  if (args.num_tiles == 0) return;
  auto kern = tlora::lora_gemm_kernel<BN, AMN, BMN, EPI, ST>;
  constexpr int smem = tlora::GemmSmem<BN, ST>::kDynamic;
  TL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int dev = 0;
  TL_CUDA(cudaGetDevice(&dev));
  const int grid = std::min(args.num_tiles, sm_budget(dev, sm_count, false));
  ProfScope ps(launch_kind, flops, s);
  launch_pdl(kern, grid, smem, s, a0, b0, a1, b1, args);
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

#ifndef TLORA_GEMM2_STAGES
#define TLORA_GEMM2_STAGES 6
#endif
// Secondary tile job of a 2-CTA launch (lora_gemm2.cuh): another layer's shrink / dH.
struct Gemm2Secondary {
  CUtensorMap a, b;
  GemmArgs args;
  double flops;
  const std::vector<tlora::PlanTile>* host = nullptr;  // the same tiles, host copy
};

// Dynamic tile scheduler tickets for the fused GEMM (lora_gemm2_kernel): a per-device pool
// of self-resetting int32 counters, one per stream that launches fused GEMMs (launches on
// one stream are serialised by PDL's griddepcontrol.wait, so they can share a ticket).
// Opt-in (TLORA_DYN_SCHED=1): measured 1.1% slower than the static round-robin schedule
// on C2 (4 interleaved A/B pairs, profiles/r1c_summary.md), so static stays the default.
// Per-device override (tlora_set_tile_scheduler): the data-parallel step executor switches
// its device to the dynamic scheduler, because NCCL kernels on the comm stream take SMs
// while a persistent GEMM's static tile list assumes all of them (C3 DP2: 426 -> 389 ms).
std::mutex g_sched_mu;
std::map<int, int> g_sched_mode;  // device -> 0 static, 1 dynamic

bool dyn_sched(int dev) {
  static const bool env_on = [] {
    const char* e = std::getenv("TLORA_DYN_SCHED");
    return e && e[0] == '1';
  }();
  std::lock_guard<std::mutex> lk(g_sched_mu);
  auto it = g_sched_mode.find(dev);
  return it == g_sched_mode.end() ? env_on : it->second == 1;
}
int32_t* tile_ticket(int dev, cudaStream_t s) {
  constexpr int kPool = 64;
  static std::mutex mu;
  static std::map<int, std::pair<int32_t*, std::map<cudaStream_t, int>>> pools;
  std::lock_guard<std::mutex> lk(mu);
  auto& pool = pools[dev];
  if (!pool.first) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    TL_CUDA(cudaStreamIsCapturing(s, &cs));
    if (cs != cudaStreamCaptureStatusNone) return nullptr;  // static schedule in this capture
    TL_CUDA(cudaMalloc(&pool.first, kPool * sizeof(int32_t)));
    TL_CUDA(cudaMemset(pool.first, 0, kPool * sizeof(int32_t)));
    TL_CUDA(cudaDeviceSynchronize());
  }
  auto it = pool.second.find(s);
  if (it == pool.second.end()) {
    const int slot = (int)(pool.second.size() % kPool);
    it = pool.second.emplace(s, slot).first;
  }
  return pool.first + it->second;
}

template <int EPI, int ST>
void launch_gemm2(const CUtensorMap& a0, const CUtensorMap& b0, const CUtensorMap& a1,
                  const CUtensorMap& b1, const GemmArgs& args_in, int sm_count, cudaStream_t s,
                  int launch_kind, double flops, const Gemm2Secondary* sec = nullptr) {
  GemmArgs args = args_in;
  GemmArgs args2{};
  const int total = args.num_tiles + (sec ? sec->args.num_tiles : 0);
  if (total == 0) return;
  if (sec) args2 = sec->args;
  auto kern = tlora::lora_gemm2_kernel<EPI, ST>;
  constexpr int smem = EPI == tlora::EPI_PEER ? tlora::Gemm2Smem<ST>::kDynamicPeer
                                              : tlora::Gemm2Smem<ST>::kDynamic;
  TL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int dev = 0;
  TL_CUDA(cudaGetDevice(&dev));
  const int grid = std::min(2 * total, sm_budget(dev, sm_count, true) / 2 * 2);
  if (dyn_sched(dev) && args.num_tiles > 0) args.tile_counter = tile_ticket(dev, s);
  ProfScope ps(launch_kind, flops + (sec ? sec->flops : 0.0), s);
  launch_pdl(kern, grid, smem, s, a0, b0, a1, b1, sec ? sec->a : a0, sec ? sec->b : b0, args,
             args2);
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

// ------------------------------------------------------------------ small kernels
template <typename T>
__device__ __forceinline__ float load_as_float(const void* p, int64_t i, int dtype) {
  if (dtype == TLORA_F64) return (float)reinterpret_cast<const double*>(p)[i];
  if (dtype == TLORA_F32) return reinterpret_cast<const float*>(p)[i];
  return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
}

// W (d x k, any dtype) -> W16 (d x k) and Wt16 (k x d), bf16, tiled transpose.
__global__ void pack_base_kernel(const void* W, int dtype, int64_t d, int64_t k,
                                 __nv_bfloat16* W16, __nv_bfloat16* Wt16) {
  __shared__ float tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < d && c < k) {
      const float v = load_as_float<float>(W, r * k + c, dtype);
      tile[i][threadIdx.x] = v;
      W16[r * k + c] = __float2bfloat16_rn(v);
    }
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < d && c < k) Wt16[c * d + r] = __float2bfloat16_rn(tile[threadIdx.x][i]);
  }
}

// Adapter of one slot (A: d x r, B: r x k) -> the four packed bf16 layouts.
__global__ void pack_adapter_kernel(const void* A, const void* B, int dtype, int64_t d, int64_t k,
                                    int r, int off, int R, __nv_bfloat16* AT, __nv_bfloat16* Acat,
                                    __nv_bfloat16* BcatT, __nv_bfloat16* Bcat, float* ATm,
                                    float* Bm) {
  const int64_t nA = d * r, nB = (int64_t)r * k;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nA + nB;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < nA) {
      const int64_t row = i / r, j = i % r;  // A[row, j]
      const float f = load_as_float<float>(A, i, dtype);
      const __nv_bfloat16 v = __float2bfloat16_rn(f);
      AT[(off + j) * d + row] = v;
      Acat[row * R + off + j] = v;
      ATm[(off + j) * d + row] = f;
    } else {
      const int64_t q = i - nA, j = q / k, col = q % k;  // B[j, col]
      const float f = load_as_float<float>(B, q, dtype);
      const __nv_bfloat16 v = __float2bfloat16_rn(f);
      Bcat[(off + j) * k + col] = v;
      BcatT[col * R + off + j] = v;
      Bm[(off + j) * k + col] = f;
    }
  }
}

// out (N x R) = in (R x N)ᵀ for bf16, 32 x 32 tiles through shared memory: the transposed
// operand copies (Acat, BcatT) rebuilt from the row-major ones (AT, Bcat) after a
// data-parallel all-gather of the refreshed row shards.
__global__ void transpose_bf16_kernel(const __nv_bfloat16* __restrict__ in, int64_t R, int64_t N,
                                      __nv_bfloat16* __restrict__ out) {
  __shared__ __nv_bfloat16 tile[32][34];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < R && c < N) tile[i][threadIdx.x] = in[r * N + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < R && c < N) out[c * R + r] = tile[threadIdx.x][i];
  }
}

// Fused multi-job AdamW over a layer's packed adapters P (R x N, fp32 master) with
// gradient G and moments; per-row job hyperparameters via row_slot -> hp[slot]. Writes the
// bf16 operand copies in both layouts the kernels read: P16 (R x N) and P16t (N x R).
// Padding-gap rows stay exactly zero. HBM-bound: 16 B read + 12 B written (fp32) + 4 B
// (bf16 x2) per parameter.
// One launch updates both packed matrices of a layer (job[0] = Aᵀcat R x d, job[1] = Bcat
// R x k). Block = 32 packed rows x 64 columns; each thread moves float4s (4 consecutive
// columns) of G, P, M, V and writes P16 as 4 x bf16; the tile goes through shared memory
// for the transposed bf16 copy (64 B runs of P16t per column). Job hyperparameters and bias
// corrections are per ROW (slot), computed once per row, not per element. The last block to
// finish (atomic ticket) bumps the per-slot step counters and resets the ticket, so the
// launch is self-contained and graph-replayable.
struct AdamJob {
  const float* G;
  float* P;
  float* M;
  float* V;
  __nv_bfloat16* P16;
  __nv_bfloat16* P16t;
  int64_t N;
  int32_t blocks_x;
  int32_t nblocks;
};

__global__ void __launch_bounds__(256, 4) adamw_layer_kernel(
    const AdamJob j0, const AdamJob j1, const int32_t* __restrict__ row_slot,
    const float2* __restrict__ hp, int32_t* __restrict__ steps, int32_t num_slots, float b1,
    float b2, float eps, float grad_scale, int64_t R, const int32_t* __restrict__ present,
    int64_t row_lo, int64_t row_hi) {
  // rows [row_lo, row_hi) of both packed matrices (the whole [0, R) unless a data-parallel
  // rank updates only its shard); R stays the row pitch of the transposed copies
  __shared__ float tile[32][65];
  __shared__ bool last;
  __shared__ int s_sl[32];
  __shared__ float s_c1[32], s_c2[32], s_lr[32], s_wd[32];
  const int tid = threadIdx.x;
  // persistent: a grid of a few blocks per SM walks the (32-row x 64-column) tiles of both
  // problems, so small layers do not pay a partial second wave
  for (int tix = blockIdx.x; tix < j0.nblocks + j1.nblocks; tix += gridDim.x) {
    __syncthreads();  // the previous tile's shared rows / transpose tile are consumed
    const bool second = tix >= j0.nblocks;
    const AdamJob& J = second ? j1 : j0;
    const int b = second ? tix - j0.nblocks : tix;
    const int64_t r0 = row_lo + (int64_t)(b / J.blocks_x) * 32, c0 = (int64_t)(b % J.blocks_x) * 64;
    const int N = (int)J.N;
    // Per-row constants once per block (32 rows): the row's slot (-1 padding gap, -2 slot
    // absent from the step: no optimizer step, masters / moments / counter unchanged, bf16
    // copies rewritten unchanged), its lr / weight decay and bias corrections.
    if (tid < 32) {
      const int64_t r = r0 + tid;
      int sl = r < row_hi ? row_slot[r] : -1;
      if (sl >= 0 && present != nullptr && !present[sl]) sl = -2;
      s_sl[tid] = sl;
      if (sl >= 0) {
        const float2 h = hp[sl];
        const float t = (float)(steps[sl] + 1);
        s_c1[tid] = 1.f / (1.f - powf(b1, t));
        s_c2[tid] = 1.f / (1.f - powf(b2, t));
        s_lr[tid] = h.x;
        s_wd[tid] = h.y;
      }
    }
    __syncthreads();
    // Both row groups' G / P / M / V float4s are loaded before any arithmetic (8 x 16 B in
    // flight per thread). Everything but the bf16 operand copies is touched once per step and
    // re-read only by the next step's optimizer: streaming loads / stores (evict-first), so
    // the concurrently running fused GEMMs keep their operand panels in L2.
    bool on[2];
    int64_t idx[2];
    float4 g4[2], p4[2], m4[2], v4[2];
#pragma unroll
    for (int it = 0; it < 2; ++it) {
      const int i = it * 16 + tid / 16, cq = (tid % 16) * 4;
      const int64_t r = r0 + i, c = c0 + cq;
      on[it] = r < row_hi && c < N;
      idx[it] = r * N + c;
      if (on[it]) p4[it] = __ldcs(reinterpret_cast<const float4*>(J.P + idx[it]));
      if (on[it] && s_sl[i] >= 0) {
        g4[it] = __ldcs(reinterpret_cast<const float4*>(J.G + idx[it]));
        m4[it] = __ldcs(reinterpret_cast<const float4*>(J.M + idx[it]));
        v4[it] = __ldcs(reinterpret_cast<const float4*>(J.V + idx[it]));
      }
    }
#pragma unroll
    for (int it = 0; it < 2; ++it) {
      const int i = it * 16 + tid / 16, cq = (tid % 16) * 4;
      float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
      if (on[it]) {
        const int sl = s_sl[i];
        if (sl == -2) {
          val = p4[it];
        } else if (sl >= 0) {
          const float c1 = s_c1[i], c2 = s_c2[i], lr = s_lr[i], wd = s_wd[i];
          const float* gp = &g4[it].x;
          float* pp = &p4[it].x;
          float* mp = &m4[it].x;
          float* vp = &v4[it].x;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float g = gp[q] * grad_scale;
            float p = pp[q];
            const float m = b1 * mp[q] + (1.f - b1) * g;
            const float v = b2 * vp[q] + (1.f - b2) * g * g;
            // fast reciprocal division (relative error ~2^-21, far inside the optimizer's
            // tolerance): the IEEE division was most of the kernel's issued instructions
            p -= lr * (__fdividef(m * c1, sqrtf(v * c2) + eps) + wd * p);
            pp[q] = p;
            mp[q] = m;
            vp[q] = v;
          }
          __stcs(reinterpret_cast<float4*>(J.P + idx[it]), p4[it]);
          __stcs(reinterpret_cast<float4*>(J.M + idx[it]), m4[it]);
          __stcs(reinterpret_cast<float4*>(J.V + idx[it]), v4[it]);
          val = p4[it];
        }
        uint2 w;
        w.x = tlora::ptx::pack_bf16x2(val.x, val.y);
        w.y = tlora::ptx::pack_bf16x2(val.z, val.w);
        *reinterpret_cast<uint2*>(J.P16 + idx[it]) = w;
      }
      tile[i][cq + 0] = val.x;
      tile[i][cq + 1] = val.y;
      tile[i][cq + 2] = val.z;
      tile[i][cq + 3] = val.w;
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int cc = it * 16 + tid / 16, rr = (tid % 16) * 2;
      const int64_t c = c0 + cc, r = r0 + rr;
      if (c < N && r < row_hi)  // row_lo, row_hi even: r + 1 < row_hi too
        *reinterpret_cast<uint32_t*>(J.P16t + c * R + r) =
            tlora::ptx::pack_bf16x2(tile[rr][cc], tile[rr + 1][cc]);
    }
  }

  // ticket: every block has read steps[] before it arrives; the last one bumps them
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const int t = atomicAdd(steps + num_slots, 1);
    last = t == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    for (int sl = tid; sl < num_slots; sl += blockDim.x)
      if (present == nullptr || present[sl]) steps[sl] += 1;
    if (tid == 0) steps[num_slots] = 0;
  }
}

// out[r][c] = sum_{p < world} recv[p][row0 + r][c]: fixed-order (deterministic) sum of the
// slots a fused GEMM + reduce-scatter wrote into this rank's receive buffer.
__global__ void reduce_slots_kernel(const __nv_bfloat16* __restrict__ recv, int world,
                                    int64_t slot_rows, int64_t row0, int64_t rows, int64_t k,
                                    __nv_bfloat16* __restrict__ out) {
  const int64_t n8 = rows * k / 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i * 8, r = e / k, c = e % k;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int p = 0; p < world; ++p) {
      const uint4 v = *reinterpret_cast<const uint4*>(recv + ((int64_t)p * slot_rows + row0 + r) * k + c);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(h[j]);
        acc[2 * j] += f.x;
        acc[2 * j + 1] += f.y;
      }
    }
    uint4 w;
    w.x = tlora::ptx::pack_bf16x2(acc[0], acc[1]);
    w.y = tlora::ptx::pack_bf16x2(acc[2], acc[3]);
    w.z = tlora::ptx::pack_bf16x2(acc[4], acc[5]);
    w.w = tlora::ptx::pack_bf16x2(acc[6], acc[7]);
    *reinterpret_cast<uint4*>(out + r * k + c) = w;
  }
}

// Elementwise dtype conversion (device), used by the host-buffer copy entry points.
__global__ void convert_kernel(const void* src, int sdt, void* dst, int ddt, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v;
    if (sdt == TLORA_F64) v = reinterpret_cast<const double*>(src)[i];
    else if (sdt == TLORA_F32) v = reinterpret_cast<const float*>(src)[i];
    else v = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(src)[i]);
    if (ddt == TLORA_F64) reinterpret_cast<double*>(dst)[i] = v;
    else if (ddt == TLORA_F32) reinterpret_cast<float*>(dst)[i] = (float)v;
    else reinterpret_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn((float)v);
  }
}

// Counter-based normal samples: element i of stream `seed` is Box-Muller of two uniforms
// from splitmix64(seed, 2i) / (seed, 2i+1). Deterministic across devices and launch shapes.
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__global__ void fill_normal_kernel(void* dst, int dtype, int64_t n, uint64_t seed, float scale) {
  const uint64_t key = splitmix64(seed ^ 0x5851F42D4C957F2Dull);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t a = splitmix64(key + 2 * (uint64_t)i), b = splitmix64(key + 2 * (uint64_t)i + 1);
    const double u1 = ((a >> 11) + 1) * (1.0 / 9007199254740993.0);  // (0, 1]
    const double u2 = (b >> 11) * (1.0 / 9007199254740992.0);        // [0, 1)
    const float v = scale * (float)(sqrt(-2.0 * log(u1)) * cospi(2.0 * u2));
    if (dtype == TLORA_F32) reinterpret_cast<float*>(dst)[i] = v;
    else reinterpret_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn(v);
  }
}

// dAT rows [off, off+r) (r x d) -> dA (d x r); dB rows -> dB (r x k).
__global__ void read_grad_kernel(const float* dAT, const float* dBc, int64_t d, int64_t k, int r,
                                 int off, float* dA, float* dB) {
  const int64_t nA = d * r, nB = (int64_t)r * k;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nA + nB;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < nA) {
      const int64_t row = i / r, j = i % r;
      dA[i] = dAT[(off + j) * d + row];
    } else {
      const int64_t q = i - nA;
      dB[q] = dBc[(int64_t)off * k + q];
    }
  }
}

// Two reductions in one launch: problem j covers R x N_j; index space concatenated.
// out[i, :] = in[perm[i], :] for up to four bf16 row-major tensors (row widths in 16-byte
// units): the job-sorted operand copies of an interleaved batch's gradient launches.
struct GatherJob {
  const uint4* src;
  uint4* dst;
  int64_t w16;
};
__global__ void gather_rows_kernel(GatherJob j0, GatherJob j1, GatherJob j2, GatherJob j3,
                                   const int32_t* __restrict__ perm, int64_t rows) {
  const GatherJob js[4] = {j0, j1, j2, j3};
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int q = 0; q < 4; ++q) {
    const GatherJob& J = js[q];
    if (!J.src) continue;
    const int64_t n = rows * J.w16;
    for (int64_t i = tid; i < n; i += stride) {
      const int64_t r = i / J.w16, c = i % J.w16;
      J.dst[i] = J.src[(int64_t)perm[r] * J.w16 + c];
    }
  }
}

struct ReduceJob {
  const float* partial;
  const int32_t* cnt;
  float* grads;
  int64_t N;
};
__global__ void reduce_splits2_kernel(ReduceJob j0, ReduceJob j1, int64_t R, float beta) {
  const int64_t n0 = j0.partial ? R * j0.N / 4 : 0, n1 = j1.partial ? R * j1.N / 4 : 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n0 + n1;
       i += (int64_t)gridDim.x * blockDim.x) {
    const ReduceJob& J = i < n0 ? j0 : j1;
    const int64_t q = i < n0 ? i : i - n0;
    const int64_t n4 = J.N / 4, row = q / n4, plane = R * J.N;
    const int c = J.cnt[row];
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < c; ++s) {
      const float4 p = reinterpret_cast<const float4*>(J.partial + s * plane)[q];
      acc.x += p.x; acc.y += p.y; acc.z += p.z; acc.w += p.w;
    }
    float4* g = reinterpret_cast<float4*>(J.grads) + q;
    if (beta != 0.f) {
      const float4 o = *g;
      acc.x += beta * o.x; acc.y += beta * o.y; acc.z += beta * o.z; acc.w += beta * o.w;
    }
    *g = acc;
  }
}


template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  void alloc(size_t count) {
    release();
    if (count) {
      TL_CUDA(cudaMalloc(&p, count * sizeof(T)));
      n = count;
    }
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { release(); }
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) TL_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

int device_sm_count(int dev) {
  int n = 0;
  cudaDeviceProp prop;
  TL_CUDA(cudaGetDeviceProperties(&prop, dev));
  require(prop.major == 10 && prop.minor == 0, TLORA_ERR_NO_DEVICE,
          "device " + std::to_string(dev) + " is sm_" + std::to_string(prop.major) +
              std::to_string(prop.minor) + "; the fused LoRA kernels are built for sm_100a only");
  n = prop.multiProcessorCount;
  // TLORA_SM_RESERVE=r leaves r SMs free of the persistent grids (for concurrent NCCL
  // kernels on a comm stream); even so CTA pairs stay whole.
  if (const char* e = std::getenv("TLORA_SM_RESERVE")) n = std::max(2, n - std::atoi(e)) / 2 * 2;
  return n;
}

void check_align(const void* p, const char* what) {
  require(p != nullptr, TLORA_ERR_ARG, std::string(what) + " is null");
  require((reinterpret_cast<uintptr_t>(p) & 15) == 0, TLORA_ERR_ARG,
          std::string(what) + " must be 16-byte aligned");
}

}  // namespace

// ==================================================================== objects
std::atomic<uint64_t> g_next_layer_id{1};

struct tlora_layer {
  uint64_t id = g_next_layer_id.fetch_add(1);
  int device = 0;
  int sm_count = 148;
  tlora::RegistryLayout L;
  std::vector<char> loaded;
  DevBuf<__nv_bfloat16> W16, Wt16, AT, Acat, BcatT, Bcat;
  DevBuf<float> dAT, dB;
  DevBuf<int32_t> col_lo, col_hi;
  bool base_set = false;
  // fused multi-job AdamW state (fp32 masters of the packed adapters + moments)
  DevBuf<float> ATm, Bm, mA, vA, mB, vB;
  DevBuf<int32_t> row_slot;  // packed rank row -> slot, -1 in padding gaps
  DevBuf<float2> hparams;    // per slot {lr, weight_decay}
  DevBuf<int32_t> steps_dev; // per slot AdamW step count (device-side: graph-capturable)
  std::vector<float> lr, wd;
  float beta1 = 0.9f, beta2 = 0.999f, eps = 1e-8f;
  bool opt_set = false;
};

namespace {
// TLORA_GRAD_LPT=0: round-robin gradient tiles instead of the LPT schedule (A/B knob).
bool grad_lpt() {
  static const bool on = [] {
    const char* e = std::getenv("TLORA_GRAD_LPT");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace

struct tlora_plan {
  tlora_layer* layer = nullptr;  // only dereferenced after checking layer_id (see bound())
  uint64_t layer_id = 0;
  int device = 0;
  tlora::PlanTables P;
  DevBuf<TileDesc> tiles[TLORA_L_COUNT];
  DevBuf<int32_t> token_slot, cnt_db, cnt_da;
  // Interleaved batches (some job's token range also holds other jobs' tokens): the
  // per-job gradient launches would stream every interleaved row once per job. They run
  // instead on job-sorted gathered copies (stable order: rows keep their order within a
  // job) with the gradient tables of the sorted order's plan.
  bool interleaved = false;
  tlora::PlanTables Ps;             // plan of the job-sorted token order (grad tables used)
  DevBuf<TileDesc> stiles[2];       // Ps.tiles[TLORA_L_DB], Ps.tiles[TLORA_L_DA]
  DevBuf<int32_t> scnt_db, scnt_da, perm;  // sorted row i <- token perm[i]
  // Gathered plan (tlora_plan_create_gathered): P is the plan of the job-sorted order;
  // X / dY operands come in that order (tlora_gather_rows), H / dH stay in it, and the
  // fused GEMM epilogues store Y / dX row i to the caller's token row_map[i].
  bool gathered = false;
  DevBuf<int32_t> row_map;
  // LPT schedule of the combined dB+dA gradient launch for gsched_ctas CTAs (CSR)
  int gsched_ctas = 0;
  DevBuf<int32_t> gsched_off, gsched_idx;
  // per-slot presence in this batch (1 = the slot owns >= 1 token), device copy: the
  // optimizer mask of a step built from this plan (tlora_plan_present_mask)
  DevBuf<int32_t> present;
  // Scratch owned by the plan (split-K partial planes, tlora_backward's dH, the gather
  // copies of an interleaved plain plan). Each kind is allocated once, at its maximum
  // size for this plan, on first use (never during CUDA-graph capture) and never regrown,
  // so distinct plans never share scratch and a returned pointer stays valid for the
  // plan's lifetime. Calls on ONE plan are serialised on one stream (tlora.h).
  mutable std::mutex scratch_mu;
  mutable DevBuf<char> scratch[3];  // 0 partial planes, 1 dH, 2 gather
  // tail split-K tile tables of the fused fwd / dX launches (tail_split), per (launch,
  // CTA pairs, secondary-tile signature); built on first eager use
  struct SplitTable {
    DevBuf<TileDesc> tiles;
    int n = 0, q = 0;
  };
  mutable std::map<std::tuple<int, int, int64_t>, std::unique_ptr<SplitTable>> split_tables;
};

namespace {
enum { kScratchPartial = 0, kScratchDh = 1, kScratchGather = 2 };

// Bytes of each scratch kind a plan can ever need (the maximum over the launches).
size_t scratch_bytes(const tlora_plan* plan, int kind) {
  const auto& L = plan->P.layout;
  const int64_t T = plan->P.T, R = L.R;
  if (kind == kScratchDh) return (size_t)T * R * 2;
  if (kind == kScratchGather) return (size_t)T * (L.k + R + L.d + R) * 2;
  const tlora::PlanTables& PT = plan->interleaved ? plan->Ps : plan->P;
  size_t n = 0;
  if (PT.splits_db > 1) n += (size_t)PT.splits_db * R * L.k;
  if (PT.splits_da > 1) n += (size_t)PT.splits_da * R * L.d;
  return n * 4;
}

template <class T>
T* plan_scratch(const tlora_plan* plan, cudaStream_t s, int kind, size_t count) {
  std::lock_guard<std::mutex> lk(plan->scratch_mu);
  DevBuf<char>& b = plan->scratch[kind];
  const size_t bytes = count * sizeof(T);
  if (b.n < bytes) {
    const size_t full = std::max(bytes, scratch_bytes(plan, kind));
    require(b.n == 0, TLORA_ERR_ARG, "plan scratch request exceeds its planned size");
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    TL_CUDA(cudaStreamIsCapturing(s, &cs));
    require(cs == cudaStreamCaptureStatusNone, TLORA_ERR_ARG,
            "plan scratch is allocated on first use: run the step once before capturing");
    b.alloc(full);
    if (kind == kScratchDh) TL_CUDA(cudaMemset(b.p, 0, full));
  }
  return reinterpret_cast<T*>(b.p);
}
}  // namespace

namespace {

size_t dtype_size(int dtype) {
  require(dtype == TLORA_F64 || dtype == TLORA_F32 || dtype == TLORA_BF16, TLORA_ERR_ARG,
          "unknown dtype");
  return dtype == TLORA_F64 ? 8 : dtype == TLORA_F32 ? 4 : 2;
}

// Returns a device pointer to `count` elements of `src`, staging host data if needed.
const void* stage_input(const void* src, size_t count, int dtype, int where, DevBuf<char>& tmp,
                        cudaStream_t s) {
  require(src != nullptr, TLORA_ERR_ARG, "input pointer is null");
  if (where == TLORA_DEVICE) return src;
  require(where == TLORA_HOST, TLORA_ERR_ARG, "unknown memory location");
  const size_t bytes = count * dtype_size(dtype);
  tmp.alloc(bytes);
  TL_CUDA(cudaMemcpyAsync(tmp.p, src, bytes, cudaMemcpyHostToDevice, s));
  return tmp.p;
}

}  // namespace

// Error hook for the library's other translation units (tlora_step.cu): same
// thread-local slot tlora_last_error() reads.
namespace tlora {
void set_last_error(const std::string& msg) { g_last_error = msg; }
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace tlora

// ==================================================================== C-ABI
extern "C" {

const char* tlora_last_error(void) { return g_last_error.c_str(); }
int tlora_abi_version(void) { return TLORA_ABI_VERSION; }

int tlora_device_check(int device, int* sm_count) {
  return guarded([&] {
    int n = 0;
    TL_CUDA(cudaGetDeviceCount(&n));
    require(device >= 0 && device < n, TLORA_ERR_NO_DEVICE,
            "no CUDA device " + std::to_string(device));
    const int sms = device_sm_count(device);
    if (sm_count) *sm_count = sms;
  });
}

int tlora_buffer_alloc(int device, size_t bytes, void** out) {
  return guarded([&] {
    require(out != nullptr, TLORA_ERR_ARG, "out is null");
    *out = nullptr;
    int n = 0;
    TL_CUDA(cudaGetDeviceCount(&n));
    require(device >= 0 && device < n, TLORA_ERR_NO_DEVICE, "no CUDA device " + std::to_string(device));
    DeviceGuard g(device);
    if (bytes) TL_CUDA(cudaMalloc(out, bytes));
  });
}

int tlora_buffer_free(int device, void* ptr) {
  return guarded([&] {
    if (!ptr) return;
    DeviceGuard g(device);
    TL_CUDA(cudaFree(ptr));
  });
}

int tlora_copy_to_device(void* dst, int dst_dtype, const void* src_host, int src_dtype,
                         int64_t count, void* stream) {
  return guarded([&] {
    require(count >= 0, TLORA_ERR_ARG, "negative count");
    if (count == 0) return;
    require(dst && src_host, TLORA_ERR_ARG, "null pointer");
    require(dst_dtype == TLORA_F32 || dst_dtype == TLORA_BF16, TLORA_ERR_ARG,
            "device dtype must be f32 or bf16");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const size_t sb = dtype_size(src_dtype);
    if (src_dtype == dst_dtype) {
      TL_CUDA(cudaMemcpyAsync(dst, src_host, count * sb, cudaMemcpyHostToDevice, s));
      TL_CUDA(cudaStreamSynchronize(s));
      return;
    }
    DevBuf<char> tmp;
    tmp.alloc(count * sb);
    TL_CUDA(cudaMemcpyAsync(tmp.p, src_host, count * sb, cudaMemcpyHostToDevice, s));
    convert_kernel<<<(unsigned)std::min<int64_t>(tlora::ceil_div(count, 256), 4096), 256, 0, s>>>(
        tmp.p, src_dtype, dst, dst_dtype, count);
    TL_CUDA(cudaGetLastError());
    TL_CUDA(cudaStreamSynchronize(s));
  });
}

int tlora_copy_to_host(void* dst_host, int dst_dtype, const void* src, int src_dtype,
                       int64_t count, void* stream) {
  return guarded([&] {
    require(count >= 0, TLORA_ERR_ARG, "negative count");
    if (count == 0) return;
    require(dst_host && src, TLORA_ERR_ARG, "null pointer");
    require(src_dtype == TLORA_F32 || src_dtype == TLORA_BF16, TLORA_ERR_ARG,
            "device dtype must be f32 or bf16");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const size_t db = dtype_size(dst_dtype);
    if (src_dtype == dst_dtype) {
      TL_CUDA(cudaMemcpyAsync(dst_host, src, count * db, cudaMemcpyDeviceToHost, s));
      TL_CUDA(cudaStreamSynchronize(s));
      return;
    }
    DevBuf<char> tmp;
    tmp.alloc(count * db);
    convert_kernel<<<(unsigned)std::min<int64_t>(tlora::ceil_div(count, 256), 4096), 256, 0, s>>>(
        src, src_dtype, tmp.p, dst_dtype, count);
    TL_CUDA(cudaGetLastError());
    TL_CUDA(cudaMemcpyAsync(dst_host, tmp.p, count * db, cudaMemcpyDeviceToHost, s));
    TL_CUDA(cudaStreamSynchronize(s));
  });
}

int tlora_fill_normal(void* dst, int dtype, int64_t count, uint64_t seed, float scale,
                      void* stream) {
  return guarded([&] {
    require(count >= 0, TLORA_ERR_ARG, "negative count");
    if (count == 0) return;
    require(dst != nullptr, TLORA_ERR_ARG, "dst is null");
    require(dtype == TLORA_F32 || dtype == TLORA_BF16, TLORA_ERR_ARG, "dtype must be f32 or bf16");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int blocks = (int)std::min<int64_t>(tlora::ceil_div(count, 256), 8192);
    fill_normal_kernel<<<blocks, 256, 0, s>>>(dst, dtype, count, seed, scale);
    TL_CUDA(cudaGetLastError());
    g_launches.fetch_add(1, std::memory_order_relaxed);
  });
}

int tlora_stream_sync(void* stream) {
  return guarded([&] { TL_CUDA(cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream))); });
}

// Stream memory operations (executed by the GPU front end, no SM): the copy-engine
// all-gather's completion flags in peer-mapped memory.
namespace {
using StreamValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
StreamValueFn stream_value_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  require(cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess &&
              q == cudaDriverEntryPointSuccess && p != nullptr,
          TLORA_ERR_CUDA, std::string(name) + " unavailable");
  return reinterpret_cast<StreamValueFn>(p);
}
}  // namespace

int tlora_copy_async(void* dst, const void* src, size_t bytes, void* stream) {
  return guarded([&] {
    if (bytes == 0) return;
    require(dst != nullptr && src != nullptr, TLORA_ERR_ARG, "null pointer");
    TL_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault,
                            reinterpret_cast<cudaStream_t>(stream)));
  });
}

int tlora_stream_write_u32(void* stream, void* addr, uint32_t value) {
  return guarded([&] {
    static StreamValueFn fn = stream_value_fn("cuStreamWriteValue32");
    require(addr != nullptr, TLORA_ERR_ARG, "null address");
    const CUresult r = fn(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(addr),
                          value, 0 /* CU_STREAM_WRITE_VALUE_DEFAULT: fenced after prior work */);
    require(r == CUDA_SUCCESS, TLORA_ERR_CUDA, "cuStreamWriteValue32 failed (" + std::to_string((int)r) + ")");
  });
}

int tlora_stream_wait_u32(void* stream, void* addr, uint32_t value) {
  return guarded([&] {
    static StreamValueFn fn = stream_value_fn("cuStreamWaitValue32");
    require(addr != nullptr, TLORA_ERR_ARG, "null address");
    const CUresult r = fn(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(addr),
                          value, 0 /* CU_STREAM_WAIT_VALUE_GEQ */);
    require(r == CUDA_SUCCESS, TLORA_ERR_CUDA, "cuStreamWaitValue32 failed (" + std::to_string((int)r) + ")");
  });
}

int tlora_layer_create(int device, int64_t d, int64_t k, int32_t num_slots, const int32_t* ranks,
                       tlora_layer** out) {
  return guarded([&] {
    require(out != nullptr, TLORA_ERR_ARG, "out is null");
    *out = nullptr;
    require(d >= 1 && k >= 1, TLORA_ERR_SHAPE, "d and k must be >= 1");
    require(d % 8 == 0 && k % 8 == 0, TLORA_ERR_SHAPE,
            "d and k must be multiples of 8 (16-byte TMA row pitch); pad on the host");
    require(num_slots >= 1 && ranks != nullptr, TLORA_ERR_ARG, "need at least one adapter slot");
    std::vector<int32_t> rv(ranks, ranks + num_slots);
    for (int s = 0; s < num_slots; ++s)
      // fused_forward accepts any r >= 1 (fused_lora.hpp:75 checks only consistency);
      // r <= min(d, k) is a JobSpec invariant (workload.hpp:54-56), not a layer one.
      require(rv[s] >= 1 && rv[s] <= 65536, TLORA_ERR_SHAPE,
              "slot " + std::to_string(s) + ": rank must be in [1, 65536]");
    int n = 0;
    TL_CUDA(cudaGetDeviceCount(&n));
    require(device >= 0 && device < n, TLORA_ERR_NO_DEVICE,
            "no CUDA device " + std::to_string(device) + " (there is no CPU fallback)");
    auto layer = std::make_unique<tlora_layer>();
    layer->device = device;
    DeviceGuard g(device);
    layer->sm_count = device_sm_count(device);
    layer->L = tlora::RegistryLayout::make(d, k, rv);
    layer->loaded.assign(num_slots, 0);
    const int64_t R = layer->L.R;
    layer->W16.alloc(d * k);
    layer->Wt16.alloc(d * k);
    layer->AT.alloc(R * d);
    layer->Acat.alloc(d * R);
    layer->BcatT.alloc(k * R);
    layer->Bcat.alloc(R * k);
    layer->dAT.alloc(R * d);
    layer->dB.alloc(R * k);
    layer->ATm.alloc(R * d);
    layer->Bm.alloc(R * k);
    TL_CUDA(cudaMemset(layer->ATm.p, 0, R * d * 4));
    TL_CUDA(cudaMemset(layer->Bm.p, 0, R * k * 4));
    {
      std::vector<int32_t> rs(R, -1);
      for (int s2 = 0; s2 < num_slots; ++s2)
        for (int i = 0; i < rv[s2]; ++i) rs[layer->L.offset[s2] + i] = s2;
      layer->row_slot.alloc(R);
      TL_CUDA(cudaMemcpy(layer->row_slot.p, rs.data(), R * 4, cudaMemcpyHostToDevice));
    }
    TL_CUDA(cudaMemset(layer->AT.p, 0, R * d * 2));
    TL_CUDA(cudaMemset(layer->Acat.p, 0, R * d * 2));
    TL_CUDA(cudaMemset(layer->BcatT.p, 0, R * k * 2));
    TL_CUDA(cudaMemset(layer->Bcat.p, 0, R * k * 2));
    TL_CUDA(cudaMemset(layer->dAT.p, 0, R * d * 4));
    TL_CUDA(cudaMemset(layer->dB.p, 0, R * k * 4));
    std::vector<int32_t> lo(num_slots), hi(num_slots);
    for (int s = 0; s < num_slots; ++s) {
      lo[s] = layer->L.offset[s];
      hi[s] = layer->L.offset[s] + rv[s];
    }
    layer->col_lo.alloc(num_slots);
    layer->col_hi.alloc(num_slots);
    TL_CUDA(cudaMemcpy(layer->col_lo.p, lo.data(), num_slots * 4, cudaMemcpyHostToDevice));
    TL_CUDA(cudaMemcpy(layer->col_hi.p, hi.data(), num_slots * 4, cudaMemcpyHostToDevice));
    *out = layer.release();
  });
}

int tlora_layer_destroy(tlora_layer* layer) {
  return guarded([&] {
    if (!layer) return;
    DeviceGuard g(layer->device);
    delete layer;
  });
}

int tlora_layer_set_base(tlora_layer* layer, const void* W, int dtype, int where, void* stream) {
  return guarded([&] {
    require(layer != nullptr, TLORA_ERR_ARG, "layer is null");
    DeviceGuard g(layer->device);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int64_t d = layer->L.d, k = layer->L.k;
    DevBuf<char> tmp;
    const void* src = stage_input(W, d * k, dtype, where, tmp, s);
    dim3 grid((unsigned)tlora::ceil_div(k, 32), (unsigned)tlora::ceil_div(d, 32));
    pack_base_kernel<<<grid, dim3(32, 8), 0, s>>>(src, dtype, d, k, layer->W16.p, layer->Wt16.p);
    TL_CUDA(cudaGetLastError());
    if (tmp.p) TL_CUDA(cudaStreamSynchronize(s));
    layer->base_set = true;
  });
}

int tlora_layer_set_adapter(tlora_layer* layer, int32_t slot, const void* A, const void* B,
                            int dtype, int where, void* stream) {
  return guarded([&] {
    require(layer != nullptr, TLORA_ERR_ARG, "layer is null");
    require(slot >= 0 && slot < (int)layer->L.rank.size(), TLORA_ERR_REGISTRY,
            "slot " + std::to_string(slot) + " is not in the registry");
    DeviceGuard g(layer->device);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int64_t d = layer->L.d, k = layer->L.k;
    const int r = layer->L.rank[slot];
    DevBuf<char> ta, tb;
    const void* a = stage_input(A, d * r, dtype, where, ta, s);
    const void* b = stage_input(B, (size_t)r * k, dtype, where, tb, s);
    pack_adapter_kernel<<<256, 256, 0, s>>>(a, b, dtype, d, k, r, layer->L.offset[slot],
                                            layer->L.R, layer->AT.p, layer->Acat.p,
                                            layer->BcatT.p, layer->Bcat.p, layer->ATm.p,
                                            layer->Bm.p);
    TL_CUDA(cudaGetLastError());
    if (ta.p || tb.p) TL_CUDA(cudaStreamSynchronize(s));
    layer->loaded[slot] = 1;
  });
}

int tlora_layer_layout(const tlora_layer* layer, int32_t* offsets, int32_t* rank_pad_total) {
  return guarded([&] {
    require(layer != nullptr, TLORA_ERR_ARG, "layer is null");
    if (offsets)
      std::memcpy(offsets, layer->L.offset.data(), layer->L.offset.size() * sizeof(int32_t));
    if (rank_pad_total) *rank_pad_total = layer->L.R;
  });
}

int tlora_layer_zero_grad(tlora_layer* layer, void* stream) {
  return guarded([&] {
    require(layer != nullptr, TLORA_ERR_ARG, "layer is null");
    DeviceGuard g(layer->device);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    TL_CUDA(cudaMemsetAsync(layer->dAT.p, 0, layer->dAT.n * 4, s));
    TL_CUDA(cudaMemsetAsync(layer->dB.p, 0, layer->dB.n * 4, s));
  });
}

int tlora_layer_grad_ptrs(tlora_layer* layer, float** dAT, float** dB) {
  return guarded([&] {
    require(layer != nullptr, TLORA_ERR_ARG, "layer is null");
    if (dAT) *dAT = layer->dAT.p;
    if (dB) *dB = layer->dB.p;
  });
}

int tlora_layer_read_grad(tlora_layer* layer, int32_t slot, float* dA, float* dB, int where,
                          void* stream) {
  return guarded([&] {
    require(layer != nullptr, TLORA_ERR_ARG, "layer is null");
    require(slot >= 0 && slot < (int)layer->L.rank.size(), TLORA_ERR_REGISTRY,
            "slot " + std::to_string(slot) + " is not in the registry");
    require(dA != nullptr && dB != nullptr, TLORA_ERR_ARG, "output pointer is null");
    DeviceGuard g(layer->device);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int64_t d = layer->L.d, k = layer->L.k;
    const int r = layer->L.rank[slot];
    DevBuf<float> tmp;
    float* oa = dA;
    float* ob = dB;
    if (where == TLORA_HOST) {
      tmp.alloc(d * r + (int64_t)r * k);
      oa = tmp.p;
      ob = tmp.p + d * r;
    }
    read_grad_kernel<<<256, 256, 0, s>>>(layer->dAT.p, layer->dB.p, d, k, r,
                                         layer->L.offset[slot], oa, ob);
    TL_CUDA(cudaGetLastError());
    if (where == TLORA_HOST) {
      TL_CUDA(cudaMemcpyAsync(dA, oa, d * r * 4, cudaMemcpyDeviceToHost, s));
      TL_CUDA(cudaMemcpyAsync(dB, ob, (size_t)r * k * 4, cudaMemcpyDeviceToHost, s));
      TL_CUDA(cudaStreamSynchronize(s));
    }
  });
}

int tlora_layer_set_optimizer(tlora_layer* layer, const float* lr, const float* weight_decay,
                              float beta1, float beta2, float eps) {
  return guarded([&] {
    require(layer != nullptr && lr != nullptr, TLORA_ERR_ARG, "null argument");
    require(beta1 >= 0.f && beta1 < 1.f && beta2 >= 0.f && beta2 < 1.f && eps > 0.f,
            TLORA_ERR_ARG, "invalid AdamW hyperparameters");
    DeviceGuard g(layer->device);
    const int S = (int)layer->L.rank.size();
    const int64_t R = layer->L.R, d = layer->L.d, k = layer->L.k;
    layer->lr.assign(lr, lr + S);
    layer->wd.assign(S, 0.f);
    if (weight_decay) layer->wd.assign(weight_decay, weight_decay + S);
    layer->beta1 = beta1;
    layer->beta2 = beta2;
    layer->eps = eps;
    if (!layer->opt_set) {
      layer->mA.alloc(R * d);
      layer->vA.alloc(R * d);
      layer->mB.alloc(R * k);
      layer->vB.alloc(R * k);
      layer->hparams.alloc(S);
      layer->steps_dev.alloc(S + 1);  // + the optimizer launch's completion ticket
    }
    TL_CUDA(cudaMemset(layer->mA.p, 0, R * d * 4));
    TL_CUDA(cudaMemset(layer->vA.p, 0, R * d * 4));
    TL_CUDA(cudaMemset(layer->mB.p, 0, R * k * 4));
    TL_CUDA(cudaMemset(layer->vB.p, 0, R * k * 4));
    TL_CUDA(cudaMemset(layer->steps_dev.p, 0, (S + 1) * 4));
    std::vector<float2> hp(S);
    for (int i = 0; i < S; ++i) hp[i] = make_float2(layer->lr[i], layer->wd[i]);
    TL_CUDA(cudaMemcpy(layer->hparams.p, hp.data(), S * sizeof(float2), cudaMemcpyHostToDevice));
    layer->opt_set = true;
  });
}

int tlora_layer_optimizer_step(tlora_layer* layer, float grad_scale, void* stream) {
  return tlora_layer_optimizer_step_masked(layer, nullptr, grad_scale, stream);
}

namespace {
void adamw_rows(tlora_layer* layer, const int32_t* present, float grad_scale, int64_t row_lo,
                int64_t row_hi, cudaStream_t s) {
  require(layer->opt_set, TLORA_ERR_ARG, "optimizer not configured (tlora_layer_set_optimizer)");
  const int S = (int)layer->L.rank.size();
  const int64_t R = layer->L.R, d = layer->L.d, k = layer->L.k;
  require(row_lo >= 0 && row_lo <= row_hi && row_hi <= R && row_lo % 2 == 0 && row_hi % 2 == 0,
          TLORA_ERR_ARG, "optimizer row range must be even bounds inside [0, R]");
  // enqueue-only, no host data: capturable in a CUDA graph
  AdamJob job[2];
  const int64_t Ns[2] = {d, k};
  float* G[2] = {layer->dAT.p, layer->dB.p};
  float* P[2] = {layer->ATm.p, layer->Bm.p};
  float* M[2] = {layer->mA.p, layer->mB.p};
  float* V[2] = {layer->vA.p, layer->vB.p};
  __nv_bfloat16* P16[2] = {layer->AT.p, layer->Bcat.p};
  __nv_bfloat16* P16t[2] = {layer->Acat.p, layer->BcatT.p};
  const int64_t rows = std::max<int64_t>(row_hi - row_lo, 1);
  for (int j = 0; j < 2; ++j) {
    const int bx = (int)tlora::ceil_div(Ns[j], 64);
    job[j] = {G[j], P[j], M[j], V[j], P16[j], P16t[j], Ns[j], bx,
              bx * (int)tlora::ceil_div(rows, 32)};
  }
  const int grid = std::min(job[0].nblocks + job[1].nblocks, 4 * layer->sm_count);
  adamw_layer_kernel<<<grid, 256, 0, s>>>(
      job[0], job[1], layer->row_slot.p, layer->hparams.p, layer->steps_dev.p, S, layer->beta1,
      layer->beta2, layer->eps, grad_scale, R, present, row_lo, row_hi);
  TL_CUDA(cudaGetLastError());
  g_launches.fetch_add(1, std::memory_order_relaxed);
}
}  // namespace

int tlora_layer_optimizer_step_masked(tlora_layer* layer, const int32_t* present, float grad_scale,
                                      void* stream) {
  return guarded([&] {
    require(layer != nullptr, TLORA_ERR_ARG, "layer is null");
    DeviceGuard g(layer->device);
    adamw_rows(layer, present, grad_scale, 0, layer->L.R, reinterpret_cast<cudaStream_t>(stream));
  });
}

int tlora_layer_optimizer_step_rows(tlora_layer* layer, const int32_t* present, float grad_scale,
                                    int64_t row_lo, int64_t row_hi, void* stream) {
  return guarded([&] {
    require(layer != nullptr, TLORA_ERR_ARG, "layer is null");
    DeviceGuard g(layer->device);
    adamw_rows(layer, present, grad_scale, row_lo, row_hi, reinterpret_cast<cudaStream_t>(stream));
  });
}

int tlora_layer_read_adapter(tlora_layer* layer, int32_t slot, float* A, float* B, int where,
                             void* stream) {
  return guarded([&] {
    require(layer != nullptr, TLORA_ERR_ARG, "layer is null");
    require(slot >= 0 && slot < (int)layer->L.rank.size(), TLORA_ERR_REGISTRY,
            "slot " + std::to_string(slot) + " is not in the registry");
    require(A != nullptr && B != nullptr, TLORA_ERR_ARG, "output pointer is null");
    DeviceGuard g(layer->device);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int64_t d = layer->L.d, k = layer->L.k;
    const int r = layer->L.rank[slot];
    DevBuf<float> tmp;
    float* oa = A;
    float* ob = B;
    if (where == TLORA_HOST) {
      tmp.alloc(d * r + (int64_t)r * k);
      oa = tmp.p;
      ob = tmp.p + d * r;
    }
    read_grad_kernel<<<256, 256, 0, s>>>(layer->ATm.p, layer->Bm.p, d, k, r, layer->L.offset[slot],
                                         oa, ob);
    TL_CUDA(cudaGetLastError());
    if (where == TLORA_HOST) {
      TL_CUDA(cudaMemcpyAsync(A, oa, d * r * 4, cudaMemcpyDeviceToHost, s));
      TL_CUDA(cudaMemcpyAsync(B, ob, (size_t)r * k * 4, cudaMemcpyDeviceToHost, s));
      TL_CUDA(cudaStreamSynchronize(s));
    }
  });
}

int tlora_plan_create(tlora_layer* layer, int64_t tokens, const int32_t* token_slot,
                      tlora_plan** out) {
  return guarded([&] {
    require(out != nullptr && layer != nullptr, TLORA_ERR_ARG, "null argument");
    *out = nullptr;
    require(tokens >= 1, TLORA_ERR_SHAPE, "plan needs at least one token");
    require(tokens < (int64_t(1) << 31) - 256, TLORA_ERR_SHAPE, "too many tokens for one plan");
    require(token_slot != nullptr, TLORA_ERR_ARG, "token_slot is null");
    DeviceGuard g(layer->device);
    auto plan = std::make_unique<tlora_plan>();
    plan->layer = layer;
    plan->layer_id = layer->id;
    plan->device = layer->device;
    plan->P = tlora::build_plan(layer->L, tokens, token_slot);
    for (int64_t t = 0; t < tokens; ++t)
      require(layer->loaded[token_slot[t]], TLORA_ERR_REGISTRY,
              "slot " + std::to_string(token_slot[t]) + " has no adapter loaded");
    for (int l = 0; l < TLORA_L_COUNT; ++l) {
      auto& v = plan->P.tiles[l];
      plan->tiles[l].alloc(v.size());
      if (!v.empty())
        TL_CUDA(cudaMemcpy(plan->tiles[l].p, v.data(), v.size() * sizeof(TileDesc),
                           cudaMemcpyHostToDevice));
    }
    plan->token_slot.alloc(tokens);
    TL_CUDA(cudaMemcpy(plan->token_slot.p, token_slot, tokens * 4, cudaMemcpyHostToDevice));
    {
      const auto& P = plan->P;
      const int S = (int)layer->L.rank.size();
      std::vector<int64_t> cnt(S + 1, 0);
      for (int64_t t = 0; t < tokens; ++t) ++cnt[token_slot[t] + 1];
      for (int s_ = 0; s_ < S; ++s_)
        if (P.slot_first[s_] >= 0 && P.slot_last[s_] + 1 - P.slot_first[s_] > cnt[s_ + 1])
          plan->interleaved = true;
      if (plan->interleaved) {
        for (int s_ = 0; s_ < S; ++s_) cnt[s_ + 1] += cnt[s_];
        std::vector<int32_t> perm(tokens), sorted(tokens);
        for (int64_t t = 0; t < tokens; ++t) perm[cnt[token_slot[t]]++] = (int32_t)t;
        for (int64_t i = 0; i < tokens; ++i) sorted[i] = token_slot[perm[i]];
        plan->Ps = tlora::build_plan(layer->L, tokens, sorted.data());
        for (int w = 0; w < 2; ++w) {
          const auto& v = plan->Ps.tiles[w == 0 ? TLORA_L_DB : TLORA_L_DA];
          plan->stiles[w].alloc(v.size());
          if (!v.empty())
            TL_CUDA(cudaMemcpy(plan->stiles[w].p, v.data(), v.size() * sizeof(TileDesc),
                               cudaMemcpyHostToDevice));
        }
        plan->scnt_db.alloc(plan->Ps.split_count_db.size());
        TL_CUDA(cudaMemcpy(plan->scnt_db.p, plan->Ps.split_count_db.data(),
                           plan->Ps.split_count_db.size() * 4, cudaMemcpyHostToDevice));
        plan->scnt_da.alloc(plan->Ps.split_count_da.size());
        TL_CUDA(cudaMemcpy(plan->scnt_da.p, plan->Ps.split_count_da.data(),
                           plan->Ps.split_count_da.size() * 4, cudaMemcpyHostToDevice));
        plan->perm.alloc(tokens);
        TL_CUDA(cudaMemcpy(plan->perm.p, perm.data(), tokens * 4, cudaMemcpyHostToDevice));
      }
    }
    if (!plan->interleaved && grad_lpt()) {
      std::vector<int32_t> off, idx;
      const int G = layer->sm_count;
      tlora::grad_schedule(plan->P.tiles[TLORA_L_DB], plan->P.tiles[TLORA_L_DA], G, off, idx);
      if (!idx.empty()) {
        plan->gsched_ctas = G;
        plan->gsched_off.alloc(off.size());
        TL_CUDA(cudaMemcpy(plan->gsched_off.p, off.data(), off.size() * 4, cudaMemcpyHostToDevice));
        plan->gsched_idx.alloc(idx.size());
        TL_CUDA(cudaMemcpy(plan->gsched_idx.p, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice));
      }
    }
    {
      const int S = (int)layer->L.rank.size();
      std::vector<int32_t> pres(S);
      for (int s_ = 0; s_ < S; ++s_) pres[s_] = plan->P.slot_first[s_] >= 0 ? 1 : 0;
      plan->present.alloc(S);
      TL_CUDA(cudaMemcpy(plan->present.p, pres.data(), S * 4, cudaMemcpyHostToDevice));
    }
    plan->cnt_db.alloc(plan->P.split_count_db.size());
    TL_CUDA(cudaMemcpy(plan->cnt_db.p, plan->P.split_count_db.data(),
                       plan->P.split_count_db.size() * 4, cudaMemcpyHostToDevice));
    plan->cnt_da.alloc(plan->P.split_count_da.size());
    TL_CUDA(cudaMemcpy(plan->cnt_da.p, plan->P.split_count_da.data(),
                       plan->P.split_count_da.size() * 4, cudaMemcpyHostToDevice));
    *out = plan.release();
  });
}

int tlora_plan_create_gathered(tlora_layer* layer, int64_t tokens, const int32_t* token_slot,
                               tlora_plan** out) {
  return guarded([&] {
    require(out != nullptr && layer != nullptr, TLORA_ERR_ARG, "null argument");
    *out = nullptr;
    require(tokens >= 1, TLORA_ERR_SHAPE, "plan needs at least one token");
    require(tokens < (int64_t(1) << 31) - 256, TLORA_ERR_SHAPE, "too many tokens for one plan");
    require(token_slot != nullptr, TLORA_ERR_ARG, "token_slot is null");
    const int32_t S = (int32_t)layer->L.rank.size();
    std::vector<int64_t> perm64(tokens), offsets(S + 1);
    // stable job-sorted order: the segment permutation (fused_lora.hpp:56-61 for all jobs)
    const int rc = tlora_segments(tokens, token_slot, S, perm64.data(), offsets.data());
    if (rc != TLORA_OK) throw Status(rc, g_last_error);
    std::vector<int32_t> perm(tokens), sorted(tokens);
    for (int64_t i = 0; i < tokens; ++i) {
      perm[i] = (int32_t)perm64[i];
      sorted[i] = token_slot[perm[i]];
    }
    tlora_plan* p = nullptr;
    const int rc2 = tlora_plan_create(layer, tokens, sorted.data(), &p);
    if (rc2 != TLORA_OK) throw Status(rc2, g_last_error);
    std::unique_ptr<tlora_plan> plan(p);
    DeviceGuard g(layer->device);
    plan->gathered = true;
    plan->row_map.alloc(tokens);
    TL_CUDA(cudaMemcpy(plan->row_map.p, perm.data(), tokens * 4, cudaMemcpyHostToDevice));
    *out = plan.release();
  });
}

int tlora_plan_row_map(const tlora_plan* plan, int32_t* row_map) {
  return guarded([&] {
    require(plan != nullptr && row_map != nullptr, TLORA_ERR_ARG, "null argument");
    const int64_t T = plan->P.T;
    if (!plan->gathered) {
      for (int64_t i = 0; i < T; ++i) row_map[i] = (int32_t)i;
      return;
    }
    DeviceGuard g(plan->device);
    TL_CUDA(cudaMemcpy(row_map, plan->row_map.p, (size_t)T * 4, cudaMemcpyDeviceToHost));
  });
}

int tlora_gather_rows(const tlora_plan* plan, int32_t n, const void* const* src, void* const* dst,
                      const int64_t* width, void* stream) {
  return guarded([&] {
    require(plan != nullptr, TLORA_ERR_ARG, "plan is null");
    require(plan->gathered, TLORA_ERR_PLAN, "tlora_gather_rows needs a gathered plan");
    require(n >= 0 && (n == 0 || (src && dst && width)), TLORA_ERR_ARG, "null argument");
    DeviceGuard g(plan->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t T = plan->P.T;
    for (int32_t i0 = 0; i0 < n; i0 += 4) {  // four tensors per launch
      GatherJob jobs[4] = {};
      int64_t work = 0;
      for (int q = 0; q < 4 && i0 + q < n; ++q) {
        const int32_t i = i0 + q;
        require(src[i] && dst[i] && src[i] != dst[i], TLORA_ERR_ARG,
                "gather needs distinct non-null source and destination");
        require(width[i] > 0 && width[i] % 8 == 0, TLORA_ERR_SHAPE,
                "gather row width must be a positive multiple of 8 bf16 elements");
        require(((uintptr_t)src[i] | (uintptr_t)dst[i]) % 16 == 0, TLORA_ERR_ARG,
                "gather operands must be 16-byte aligned");
        jobs[q] = {reinterpret_cast<const uint4*>(src[i]), reinterpret_cast<uint4*>(dst[i]),
                   width[i] / 8};
        work += T * (width[i] / 8);
      }
      const int blocks = (int)std::min<int64_t>(tlora::ceil_div(work, 256),
                                                8 * (int64_t)device_sm_count(plan->device));
      gather_rows_kernel<<<blocks, 256, 0, s>>>(jobs[0], jobs[1], jobs[2], jobs[3],
                                                plan->row_map.p, T);
      g_launches.fetch_add(1, std::memory_order_relaxed);
      TL_CUDA(cudaGetLastError());
    }
  });
}

int tlora_plan_present_mask(const tlora_plan* plan, const int32_t** present) {
  return guarded([&] {
    require(plan != nullptr && present != nullptr, TLORA_ERR_ARG, "null argument");
    *present = plan->present.p;
  });
}

int tlora_plan_destroy(tlora_plan* plan) {
  return guarded([&] {
    if (!plan) return;
    DeviceGuard g(plan->device);
    delete plan;
  });
}

int tlora_plan_get_info(const tlora_plan* plan, tlora_plan_info* info) {
  return guarded([&] {
    require(plan != nullptr && info != nullptr, TLORA_ERR_ARG, "null argument");
    const auto& L = plan->P.layout;
    info->tokens = plan->P.T;
    info->d = L.d;
    info->k = L.k;
    info->num_slots = (int32_t)L.rank.size();
    info->rank_pad_total = L.R;
    for (int l = 0; l < TLORA_L_COUNT; ++l) info->num_tiles[l] = (int32_t)plan->P.tiles[l].size();
    info->splits_db = plan->P.splits_db;
    info->splits_da = plan->P.splits_da;
    info->useful_ext_cols = plan->P.useful_ext_cols;
    info->packed_ext_cols = plan->P.packed_ext_cols;
  });
}

int tlora_plan_get_tiles(const tlora_plan* plan, int launch, tlora_tile* out, int32_t cap,
                         int32_t* count) {
  return guarded([&] {
    require(plan != nullptr, TLORA_ERR_ARG, "plan is null");
    require(launch >= 0 && launch < TLORA_L_COUNT, TLORA_ERR_ARG, "unknown launch id");
    const auto& v = plan->P.tiles[launch];
    if (count) *count = (int32_t)v.size();
    if (out) std::memcpy(out, v.data(), std::min<size_t>(cap, v.size()) * sizeof(tlora_tile));
  });
}

int tlora_plan_read_device(const tlora_plan* plan, int launch, tlora_tile* out, int32_t cap,
                           int32_t* count, int32_t* token_slot) {
  return guarded([&] {
    require(plan != nullptr, TLORA_ERR_ARG, "plan is null");
    require(launch >= 0 && launch < TLORA_L_COUNT, TLORA_ERR_ARG, "unknown launch id");
    DeviceGuard g(plan->device);
    const int32_t n = (int32_t)plan->P.tiles[launch].size();
    if (count) *count = n;
    const int32_t m = std::min(cap, n);
    if (out && m > 0)
      TL_CUDA(cudaMemcpy(out, plan->tiles[launch].p, (size_t)m * sizeof(tlora_tile),
                         cudaMemcpyDeviceToHost));
    if (token_slot)
      TL_CUDA(cudaMemcpy(token_slot, plan->token_slot.p, (size_t)plan->P.T * sizeof(int32_t),
                         cudaMemcpyDeviceToHost));
  });
}

int tlora_plan_tiles_host(int64_t d, int64_t k, int32_t num_slots, const int32_t* ranks,
                          int64_t tokens, const int32_t* token_slot, int launch, tlora_tile* out,
                          int32_t cap, int32_t* count) {
  return guarded([&] {
    require(num_slots >= 1 && ranks != nullptr && token_slot != nullptr, TLORA_ERR_ARG,
            "null argument");
    require(tokens >= 1, TLORA_ERR_SHAPE, "plan needs at least one token");
    require(launch >= 0 && launch < TLORA_L_COUNT, TLORA_ERR_ARG, "unknown launch id");
    const auto L = tlora::RegistryLayout::make(d, k, std::vector<int32_t>(ranks, ranks + num_slots));
    const auto P = tlora::build_plan(L, tokens, token_slot);
    const auto& v = P.tiles[launch];
    if (count) *count = (int32_t)v.size();
    if (out) std::memcpy(out, v.data(), std::min<size_t>(cap, v.size()) * sizeof(tlora_tile));
  });
}

int tlora_plan_grad_schedule_host(int64_t d, int64_t k, int32_t num_slots, const int32_t* ranks,
                                  int64_t tokens, const int32_t* token_slot, int32_t ctas,
                                  int32_t* off, int32_t* idx, int32_t cap, int32_t* count) {
  return guarded([&] {
    require(num_slots >= 1 && ranks != nullptr && token_slot != nullptr, TLORA_ERR_ARG,
            "null argument");
    require(tokens >= 1, TLORA_ERR_SHAPE, "plan needs at least one token");
    require(ctas >= 1, TLORA_ERR_ARG, "ctas must be >= 1");
    const auto L = tlora::RegistryLayout::make(d, k, std::vector<int32_t>(ranks, ranks + num_slots));
    const auto P = tlora::build_plan(L, tokens, token_slot);
    std::vector<int32_t> o, x;
    tlora::grad_schedule(P.tiles[TLORA_L_DB], P.tiles[TLORA_L_DA], ctas, o, x);
    if (count) *count = (int32_t)x.size();
    if (off) std::memcpy(off, o.data(), o.size() * sizeof(int32_t));
    if (idx) std::memcpy(idx, x.data(), std::min<size_t>(cap, x.size()) * sizeof(int32_t));
  });
}

}  // extern "C"

// ==================================================================== launch bodies
namespace {

void check_bound(const tlora_layer* layer, const tlora_plan* plan) {
  require(layer != nullptr && plan != nullptr, TLORA_ERR_ARG, "null layer/plan");
  // a plan serves every layer with the same registry layout (d, k, ranks) on its device,
  // e.g. one plan per projection shape for a whole layer stack
  const auto& a = plan->P.layout;
  const auto& b = layer->L;
  require(plan->layer_id == layer->id ||
              (plan->device == layer->device && a.d == b.d && a.k == b.k && a.rank == b.rank),
          TLORA_ERR_PLAN, "plan was built for a layer with a different registry layout");
  require(layer->base_set, TLORA_ERR_ARG, "base weight not set");
}

// H = X·Aᵀcatᵀ masked to each token's own packed columns. Shrink tiles write only their
// token tile's rank window; the gradient launches read H over whole job token ranges, so
// every other column must be an exact zero (memset first).
Gemm2Secondary make_lowrank2(tlora_layer* layer, const tlora_plan* plan, int which, const void* A,
                             void* out);
void launch_lowrank_pairs(tlora_layer* layer, const Gemm2Secondary& sec, int kind, cudaStream_t s);

// Standalone shrink / dH on CTA pairs (the SHRINK2 / DH2 tables, lora_gemm2_kernel with no
// main tiles) instead of the 1-CTA kernel; identical results (same K order per element).
// TLORA_LOWRANK_PAIR=0 selects the 1-CTA kernel.
bool lowrank_pairs() {
  static const bool on = [] {
    const char* e = std::getenv("TLORA_LOWRANK_PAIR");
    return e ? std::atoi(e) != 0 : true;
  }();
  return on;
}

void run_shrink(tlora_layer* layer, const tlora_plan* plan, const void* X, void* H, cudaStream_t s) {
  const auto& L = layer->L;
  const int64_t T = plan->P.T, d = L.d, R = L.R;
  TL_CUDA(cudaMemsetAsync(H, 0, (size_t)T * R * 2, s));
  if (lowrank_pairs()) {
    launch_lowrank_pairs(layer, make_lowrank2(layer, plan, 0, X, H), TLORA_L_SHRINK, s);
    return;
  }
  GemmArgs a{};
  a.tiles = plan->tiles[TLORA_L_SHRINK].p;
  a.num_tiles = (int)plan->P.tiles[TLORA_L_SHRINK].size();
  a.M = (int)T;
  a.N = (int)R;
  a.out = H;
  a.ldo = R;
  a.row_slot = plan->token_slot.p;
  a.slot_col_lo = layer->col_lo.p;
  a.slot_col_hi = layer->col_hi.p;
  const CUtensorMap ma = tmap_k(X, d, T, tlora::kBM);
  const CUtensorMap mb = tmap_k(layer->AT.p, d, R, tlora::kPlanBNLow);
  launch_gemm<128, false, false, tlora::EPI_BF16_MASK, 6>(ma, mb, ma, mb, a, layer->sm_count, s,
                                                          TLORA_L_SHRINK,
                                                          2.0 * (double)plan->P.tok_rank * d);
}

// The shrink (which = 0: H = X·Aᵀcatᵀ, K = d) or dH (which = 1: dH = dY·Bᵀ, K = k) of a
// layer as secondary pair tiles of another layer's fused GEMM launch (plan tables SHRINK2 /
// DH2: 256-token tiles, N 128 or 256 over the token tile's rank window). Masked like
// run_shrink / run_dh; the caller guarantees the output is zero outside the windows.
Gemm2Secondary make_lowrank2(tlora_layer* layer, const tlora_plan* plan, int which, const void* A,
                             void* out) {
  const auto& L = layer->L;
  const int64_t T = plan->P.T, R = L.R, K = which == 0 ? L.d : L.k;
  const int launch = which == 0 ? TLORA_L_SHRINK2 : TLORA_L_DH2;
  Gemm2Secondary g{};
  g.args.tiles = plan->tiles[launch].p;
  g.args.num_tiles = (int)plan->P.tiles[launch].size();
  g.args.M = (int)T;
  g.args.N = (int)R;
  g.args.out = out;
  g.args.ldo = R;
  g.args.row_slot = plan->token_slot.p;
  g.args.slot_col_lo = layer->col_lo.p;
  g.args.slot_col_hi = layer->col_hi.p;
  g.a = tmap_k(A, K, T, 128);
  g.b = tmap_k(which == 0 ? layer->AT.p : layer->Bcat.p, K, R, 64);
  g.flops = 2.0 * (double)plan->P.tok_rank * K;
  g.host = &plan->P.tiles[launch];
  return g;
}

void launch_lowrank_pairs(tlora_layer* layer, const Gemm2Secondary& sec, int kind,
                          cudaStream_t s) {
  GemmArgs none{};  // no main tiles: every tile of the launch is a secondary (low-rank) tile
  Gemm2Secondary g = sec;
  const double flops = g.flops;
  g.flops = 0.0;
  launch_gemm2<tlora::EPI_BF16, TLORA_GEMM2_STAGES>(g.a, g.b, g.a, g.b, none, layer->sm_count, s,
                                                    kind, flops, &g);
}

// ------------------------------------------------------------------ tail split-K
// A persistent fused GEMM launch walks its tiles round-robin over the CTA pairs, so its
// last wave is partial (C2 fwd up: 3072 tiles = 41.5 waves of 74 pairs) and the pairs
// without a tile idle at the end. With TLORA_TAIL_SPLIT=1 the last q main tiles of a
// launch are split in two along K: the first half writes an fp32 partial, the second half
// (with the LoRA K-extension) adds it in its epilogue (GemmArgs::split_ws; deterministic,
// one bf16 rounding). q minimises the round-robin makespan of the launch's tile costs
// (k-blocks; the secondary tiles of the chained schedule included), and is 0 unless the
// model gains >= 1%. All first halves precede all second halves in the tile order, so
// a waiting second half never blocks a first half of its own pair.
bool tail_split_on() {
  static const bool on = [] {
    const char* e = std::getenv("TLORA_TAIL_SPLIT");
    return e && e[0] == '1';
  }();
  return on;
}

constexpr int kSplitSlots = 128;  // >= CTA pairs of any launch (q <= pairs)

struct SplitWs {
  float* ws = nullptr;
  int32_t* flags = nullptr;
};

// One workspace per (device, stream): fused GEMM launches on one stream are serialised.
const SplitWs* split_ws(int dev, cudaStream_t s) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, SplitWs> pool;
  std::lock_guard<std::mutex> lk(mu);
  auto& w = pool[{dev, s}];
  if (!w.ws) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    TL_CUDA(cudaStreamIsCapturing(s, &cs));
    if (cs != cudaStreamCaptureStatusNone) return nullptr;
    TL_CUDA(cudaMalloc(&w.ws, (size_t)kSplitSlots * tlora::kBM2 * tlora::kBN2 * sizeof(float)));
    TL_CUDA(cudaMalloc(&w.flags, (size_t)kSplitSlots * 8 * sizeof(int32_t)));
    TL_CUDA(cudaMemset(w.flags, 0, (size_t)kSplitSlots * 8 * sizeof(int32_t)));
    TL_CUDA(cudaDeviceSynchronize());
  }
  return &w;
}

double main_tile_cost(const tlora::PlanTile& t) {
  return (double)(t.ke0 - t.kb0 + std::max(0, t.ke1 - t.kb1)) / tlora::kBK;
}
double sec_tile_cost(const tlora::PlanTile& t) {
  // A-operand streaming bounds a narrow secondary tile (~0.45 of a full-N k-block)
  return (double)(t.ke0 - t.kb0) / tlora::kBK * std::max(t.pad / 256.0, 0.45);
}

const tlora_plan::SplitTable* plan_split(const tlora_plan* plan, int launch, int pairs,
                                         const Gemm2Secondary* sec, cudaStream_t s) {
  const auto& M = plan->P.tiles[launch];
  int64_t sig = 0;
  std::vector<double> sc;
  if (sec && sec->host)
    for (const auto& t : *sec->host) {
      sc.push_back(sec_tile_cost(t));
      sig = sig * 1000003 + (int64_t)(t.ke0 - t.kb0) * 517 + t.pad;
    }
  const auto key = std::make_tuple(launch, pairs, sig);
  std::lock_guard<std::mutex> lk(plan->scratch_mu);
  auto it = plan->split_tables.find(key);
  if (it != plan->split_tables.end()) return it->second.get();
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  TL_CUDA(cudaStreamIsCapturing(s, &cs));
  if (cs != cudaStreamCaptureStatusNone) return nullptr;
  const int n = (int)M.size();
  constexpr double kFix = 4.0;  // partial write / read per half, in k-block units
  std::vector<double> load(pairs);
  auto makespan = [&](int q) {
    std::fill(load.begin(), load.end(), 0.0);
    int idx = 0;
    for (int i = 0; i < n - q; ++i) load[idx++ % pairs] += main_tile_cost(M[i]);
    for (int h = 0; h < 2; ++h)
      for (int i = n - q; i < n; ++i) {
        const auto& t = M[i];
        const int nk = (t.ke0 - t.kb0) / tlora::kBK;
        const double c0 = (double)(nk / 2);
        load[idx++ % pairs] += (h == 0 ? c0 : main_tile_cost(t) - c0) + kFix;
      }
    for (double c : sc) load[idx++ % pairs] += c;
    return *std::max_element(load.begin(), load.end());
  };
  const double base = makespan(0);
  int best_q = 0;
  double best = base;
  const int qmax = std::min({n, pairs, kSplitSlots});
  for (int q = 1; q <= qmax; ++q) {
    bool ok = true;  // both halves need >= 1 k-block
    for (int i = n - q; i < n && ok; ++i) ok = (M[i].ke0 - M[i].kb0) / tlora::kBK >= 2;
    if (!ok) break;
    const double m = makespan(q);
    if (m < best) {
      best = m;
      best_q = q;
    }
  }
  if (best > 0.99 * base) best_q = 0;
  if (std::getenv("TLORA_TAIL_SPLIT_DEBUG"))
    std::fprintf(stderr, "[tail_split] launch %d tiles %d + %zu secondary, %d pairs: q = %d, "
                 "modelled makespan %.1f -> %.1f k-blocks\n", launch, n, sc.size(), pairs, best_q,
                 base, best_q ? best : base);
  auto tab = std::make_unique<tlora_plan::SplitTable>();
  tab->q = best_q;
  if (best_q > 0) {
    std::vector<TileDesc> out;
    out.reserve(n + best_q);
    auto desc = [](const tlora::PlanTile& t) {
      return TileDesc{t.m0, t.n0, t.kb0, t.ke0, t.kb1, t.ke1, t.split, t.pad};
    };
    for (int i = 0; i < n - best_q; ++i) out.push_back(desc(M[i]));
    for (int h = 0; h < 2; ++h)
      for (int j = 0; j < best_q; ++j) {
        TileDesc d = desc(M[n - best_q + j]);
        const int mid = d.kb0 + ((d.ke0 - d.kb0) / tlora::kBK / 2) * tlora::kBK;
        if (h == 0) {  // first K half, no K-extension: the partial writer
          d.ke0 = mid;
          d.kb1 = d.ke1 = 0;
          d.pad = 1 + 2 * j;
        } else {  // the rest + the LoRA K-extension: the finisher
          d.kb0 = mid;
          d.pad = 2 + 2 * j;
        }
        out.push_back(d);
      }
    tab->n = (int)out.size();
    tab->tiles.alloc(out.size());
    TL_CUDA(cudaMemcpy(tab->tiles.p, out.data(), out.size() * sizeof(TileDesc),
                       cudaMemcpyHostToDevice));
  }
  auto* ret = tab.get();
  plan->split_tables.emplace(key, std::move(tab));
  return ret;
}

// Swap a fused fwd / dX launch's main tiles for its split table (no-op unless enabled and
// the model gains).
void apply_tail_split(tlora_layer* layer, const tlora_plan* plan, int launch, GemmArgs& a,
                      const Gemm2Secondary* sec, cudaStream_t s) {
  if (!tail_split_on() || a.num_tiles == 0 || dyn_sched(layer->device)) return;
  const int total = a.num_tiles + (sec ? sec->args.num_tiles : 0);
  const int pairs = std::min(2 * total, sm_budget(layer->device, layer->sm_count, true) / 2 * 2) / 2;
  if (pairs < 2) return;
  const tlora_plan::SplitTable* t = plan_split(plan, launch, pairs, sec, s);
  if (!t || t->q == 0) return;
  const SplitWs* w = split_ws(layer->device, s);
  if (!w) return;
  a.tiles = t->tiles.p;
  a.num_tiles = t->n;
  a.split_ws = w->ws;
  a.split_flags = w->flags;
}

// Y = X·W + H·Bᵀcatᵀ: 2-CTA fused GEMM, K-extension over each tile's packed-rank window.
void run_fwd_gemm(tlora_layer* layer, const tlora_plan* plan, const void* X, const void* H, void* Y,
                  int y_dtype, cudaStream_t s, const Gemm2Secondary* sec = nullptr) {
  const auto& L = layer->L;
  const int64_t T = plan->P.T, d = L.d, k = L.k, R = L.R;
  const double flops = 2.0 * T * d * k + 2.0 * (double)plan->P.tok_rank * k;
  GemmArgs a{};
  a.tiles = plan->tiles[TLORA_L_FWD].p;
  a.num_tiles = (int)plan->P.tiles[TLORA_L_FWD].size();
  a.M = (int)T;
  a.N = (int)k;
  a.out = Y;
  a.ldo = k;
  a.beta = 0.f;
  a.row_map = plan->row_map.p;  // null unless gathered
  const CUtensorMap ma0 = tmap_k(X, d, T, 128);
  const CUtensorMap mb0 = tmap_k(layer->Wt16.p, d, k, 128);
  const CUtensorMap ma1 = tmap_k(H, R, T, 128);
  const CUtensorMap mb1 = tmap_k(layer->BcatT.p, R, k, 128);
  if (y_dtype == TLORA_BF16) {
    apply_tail_split(layer, plan, TLORA_L_FWD, a, sec, s);
    launch_gemm2<tlora::EPI_BF16, TLORA_GEMM2_STAGES>(ma0, mb0, ma1, mb1, a, layer->sm_count, s,
                                                      TLORA_L_FWD, flops, sec);
  }
  else
    launch_gemm2<tlora::EPI_F32, TLORA_GEMM2_STAGES>(ma0, mb0, ma1, mb1, a, layer->sm_count, s,
                                                     TLORA_L_FWD, flops, sec);
}

// dH = dY·Bᵀ (masked; zero outside the windows, as H)
void run_dh(tlora_layer* layer, const tlora_plan* plan, const void* dY, void* dH, cudaStream_t s) {
  const auto& L = layer->L;
  const int64_t T = plan->P.T, k = L.k, R = L.R;
  TL_CUDA(cudaMemsetAsync(dH, 0, (size_t)T * R * 2, s));
  if (lowrank_pairs()) {
    launch_lowrank_pairs(layer, make_lowrank2(layer, plan, 1, dY, dH), TLORA_L_DH, s);
    return;
  }
  GemmArgs a{};
  a.tiles = plan->tiles[TLORA_L_DH].p;
  a.num_tiles = (int)plan->P.tiles[TLORA_L_DH].size();
  a.M = (int)T;
  a.N = (int)R;
  a.out = dH;
  a.ldo = R;
  a.row_slot = plan->token_slot.p;
  a.slot_col_lo = layer->col_lo.p;
  a.slot_col_hi = layer->col_hi.p;
  const CUtensorMap ma = tmap_k(dY, k, T, tlora::kBM);
  const CUtensorMap mb = tmap_k(layer->Bcat.p, k, R, tlora::kPlanBNLow);
  launch_gemm<128, false, false, tlora::EPI_BF16_MASK, 6>(ma, mb, ma, mb, a, layer->sm_count, s,
                                                          TLORA_L_DH,
                                                          2.0 * (double)plan->P.tok_rank * k);
}

// dX = dY·Wᵀ + dH·Aᵀ (2-CTA fused GEMM)
void run_dx(tlora_layer* layer, const tlora_plan* plan, const void* dY, const void* dH, void* dX,
            float beta, cudaStream_t s, const Gemm2Secondary* sec = nullptr) {
  const auto& L = layer->L;
  const int64_t T = plan->P.T, d = L.d, k = L.k, R = L.R;
  GemmArgs a{};
  a.tiles = plan->tiles[TLORA_L_DX].p;
  a.num_tiles = (int)plan->P.tiles[TLORA_L_DX].size();
  a.M = (int)T;
  a.N = (int)d;
  a.out = dX;
  a.ldo = d;
  a.beta = beta;
  a.row_map = plan->row_map.p;  // null unless gathered
  const CUtensorMap ma0 = tmap_k(dY, k, T, 128);
  const CUtensorMap mb0 = tmap_k(layer->W16.p, k, d, 128);
  const CUtensorMap ma1 = tmap_k(dH, R, T, 128);
  const CUtensorMap mb1 = tmap_k(layer->Acat.p, R, d, 128);
  apply_tail_split(layer, plan, TLORA_L_DX, a, sec, s);
  launch_gemm2<tlora::EPI_BF16, TLORA_GEMM2_STAGES>(ma0, mb0, ma1, mb1, a, layer->sm_count, s,
                                                    TLORA_L_DX,
                                                    2.0 * T * d * k + 2.0 * (double)plan->P.tok_rank * d,
                                                    sec);
}

// Adapter gradients, per job in transposed form (lora_grad.cuh), dB and/or dA in ONE
// persistent launch:  dBcat = Hᵀ·dY (N = k)  and  dAᵀcat = dHᵀ·X (N = d), over each job's
// token range; grads = beta·grads + result, split-K partials reduced in fixed order (one
// combined reduce launch).
void run_grads(tlora_layer* layer, const tlora_plan* plan, const void* H, const void* dY,
               const void* dH, const void* X, bool do_b, bool do_a, float beta, cudaStream_t s) {
  const auto& L = layer->L;
  const int64_t T = plan->P.T, R = L.R;
  tlora::GradArgs g{};
  CUtensorMap ma[2], mb[2];
  ReduceJob rj[2] = {};
  const bool on[2] = {do_b, do_a};
  const int64_t Ns[2] = {L.k, L.d};
  // interleaved batch: gather job-sorted copies of the operands, use the sorted plan
  const bool srt = plan->interleaved;
  const tlora::PlanTables& PT = srt ? plan->Ps : plan->P;
  const int nsp[2] = {PT.splits_db, PT.splits_da};
  float* grads[2] = {layer->dB.p, layer->dAT.p};
  const int32_t* cnts[2] = {srt ? plan->scnt_db.p : plan->cnt_db.p,
                            srt ? plan->scnt_da.p : plan->cnt_da.p};
  const void* full[2] = {dY, X};
  const void* low[2] = {H, dH};
  if (srt) {
    const int64_t widths[4] = {L.k, R, L.d, R};  // dY, H, X, dH (bf16 row widths)
    const void* src[4] = {dY, H, X, dH};
    size_t total = 0;
    for (int q = 0; q < 4; ++q)
      if (on[q / 2]) total += (size_t)T * widths[q];
    __nv_bfloat16* gbuf = plan_scratch<__nv_bfloat16>(plan, s, kScratchGather, total);
    GatherJob jobs[4] = {};
    size_t o = 0;
    for (int q = 0; q < 4; ++q) {
      if (!on[q / 2]) continue;
      jobs[q] = {reinterpret_cast<const uint4*>(src[q]), reinterpret_cast<uint4*>(gbuf + o),
                 widths[q] / 8};
      (q % 2 == 0 ? full : low)[q / 2] = gbuf + o;
      o += (size_t)T * widths[q];
    }
    const int64_t work = T * ((on[0] ? L.k + R : 0) + (on[1] ? L.d + R : 0)) / 8;
    const int blocks = (int)std::min<int64_t>(tlora::ceil_div(work, 256), 8 * layer->sm_count);
    gather_rows_kernel<<<blocks, 256, 0, s>>>(jobs[0], jobs[1], jobs[2], jobs[3], plan->perm.p, T);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    TL_CUDA(cudaGetLastError());
  }
  // workspace: [problem 0 planes][problem 1 planes]
  size_t need = 0;
  for (int j = 0; j < 2; ++j)
    if (on[j] && nsp[j] > 1) need += (size_t)nsp[j] * R * Ns[j];
  float* ws = need ? plan_scratch<float>(plan, s, kScratchPartial, need) : nullptr;
  size_t off = 0;
  double flops = 0.0;
  for (int j = 0; j < 2; ++j) {
    const int launch = j == 0 ? TLORA_L_DB : TLORA_L_DA;
    GemmArgs& a = g.job[j];
    if (!on[j]) {
      a.num_tiles = 0;
      ma[j] = ma[0];
      mb[j] = mb[0];
      continue;
    }
    const int64_t N = Ns[j];
    a.tiles = srt ? plan->stiles[j].p : plan->tiles[launch].p;
    a.num_tiles = (int)PT.tiles[launch].size();
    a.M = (int)N;  // transposed form: M = layer dimension, output rows = packed rank columns
    a.N = (int)N;
    a.ldo = N;
    if (nsp[j] > 1) {
      a.out = ws + off;
      a.split_stride = R * N;
      a.beta = 0.f;
      rj[j] = {ws + off, cnts[j], grads[j], N};
      off += (size_t)nsp[j] * R * N;
    } else {
      a.out = grads[j];
      a.beta = beta;
    }
    ma[j] = tmap_mn(full[j], N, T);
    mb[j] = tmap_mn(low[j], R, T);
    flops += 2.0 * (double)plan->P.tok_rank * N;
  }
  if (!on[0]) {  // problem 1 alone: keep its maps in slot 1, slot 0 unused
    ma[0] = ma[1];
    mb[0] = mb[1];
  }
  const int tiles = g.job[0].num_tiles + g.job[1].num_tiles;
#ifndef TLORA_GRAD_STAGES
#define TLORA_GRAD_STAGES 6
#endif
  auto kern = tlora::lora_grad_kernel<TLORA_GRAD_STAGES>;
  constexpr int smem = tlora::GradSmem<TLORA_GRAD_STAGES>::kDynamic;
  TL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int grid = std::min(tiles, sm_budget(layer->device, layer->sm_count, false));
  if (on[0] && on[1] && !srt && plan->gsched_ctas == grid) {  // LPT-balanced CTA tile lists
    g.sched_off = plan->gsched_off.p;
    g.sched_idx = plan->gsched_idx.p;
  }
  {
    ProfScope ps(do_b ? TLORA_L_DB : TLORA_L_DA, flops, s);  // dB+dA together: booked on dB
    if (tiles > 0) {
      launch_pdl(kern, grid, smem, s, ma[0], mb[0], ma[1], mb[1], g);
      g_launches.fetch_add(1, std::memory_order_relaxed);
    }
  }
  if (rj[0].partial || rj[1].partial) {
    const int64_t work = (rj[0].partial ? R * rj[0].N / 4 : 0) + (rj[1].partial ? R * rj[1].N / 4 : 0);
    const int blocks = (int)std::min<int64_t>(tlora::ceil_div(work, 256), 4 * layer->sm_count);
    reduce_splits2_kernel<<<blocks, 256, 0, s>>>(rj[0], rj[1], R, beta);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    TL_CUDA(cudaGetLastError());
  }
}

}  // namespace

extern "C" {

int tlora_forward(tlora_layer* layer, const tlora_plan* plan, const void* X, void* Y, int y_dtype,
                  void* H_stash, void* stream) {
  return guarded([&] {
    check_bound(layer, plan);
    check_align(X, "X");
    check_align(Y, "Y");
    check_align(H_stash, "H_stash");
    require(y_dtype == TLORA_BF16 || y_dtype == TLORA_F32, TLORA_ERR_ARG,
            "Y dtype must be bf16 or f32");
    DeviceGuard g(layer->device);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    run_shrink(layer, plan, X, H_stash, s);
    run_fwd_gemm(layer, plan, X, H_stash, Y, y_dtype, s);
  });
}

int tlora_forward_shrink(tlora_layer* layer, const tlora_plan* plan, const void* X, void* H,
                         void* stream) {
  return guarded([&] {
    check_bound(layer, plan);
    check_align(X, "X");
    check_align(H, "H");
    DeviceGuard g(layer->device);
    run_shrink(layer, plan, X, H, reinterpret_cast<cudaStream_t>(stream));
  });
}

int tlora_forward_gemm(tlora_layer* layer, const tlora_plan* plan, const void* X, const void* H,
                       void* Y, int y_dtype, void* stream) {
  return guarded([&] {
    check_bound(layer, plan);
    check_align(X, "X");
    check_align(H, "H");
    check_align(Y, "Y");
    require(y_dtype == TLORA_BF16 || y_dtype == TLORA_F32, TLORA_ERR_ARG,
            "Y dtype must be bf16 or f32");
    DeviceGuard g(layer->device);
    run_fwd_gemm(layer, plan, X, H, Y, y_dtype, reinterpret_cast<cudaStream_t>(stream));
  });
}

int tlora_forward_gemm_shrink(tlora_layer* layer, const tlora_plan* plan, const void* X,
                              const void* H, void* Y, int y_dtype, tlora_layer* next,
                              const tlora_plan* next_plan, const void* X_next, void* H_next,
                              int zero_next, void* stream) {
  return guarded([&] {
    check_bound(layer, plan);
    check_bound(next, next_plan);
    check_align(X, "X");
    check_align(H, "H");
    check_align(Y, "Y");
    check_align(X_next, "X_next");
    check_align(H_next, "H_next");
    require(y_dtype == TLORA_BF16 || y_dtype == TLORA_F32, TLORA_ERR_ARG,
            "Y dtype must be bf16 or f32");
    require(next->device == layer->device, TLORA_ERR_ARG, "layers on different devices");
    require(H_next != H && H_next != Y && H_next != X, TLORA_ERR_ARG,
            "H_next must not alias this layer's operands");
    DeviceGuard g(layer->device);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (zero_next)
      TL_CUDA(cudaMemsetAsync(H_next, 0, (size_t)next_plan->P.T * next->L.R * 2, s));
    const Gemm2Secondary sec = make_lowrank2(next, next_plan, 0, X_next, H_next);
    run_fwd_gemm(layer, plan, X, H, Y, y_dtype, s, &sec);
  });
}

int tlora_forward_gemm_dh(tlora_layer* layer, const tlora_plan* plan, const void* X,
                          const void* H, void* Y, int y_dtype, tlora_layer* next,
                          const tlora_plan* next_plan, const void* dY_next, void* dH_next,
                          int zero_next, void* stream) {
  return guarded([&] {
    check_bound(layer, plan);
    check_bound(next, next_plan);
    check_align(X, "X");
    check_align(H, "H");
    check_align(Y, "Y");
    check_align(dY_next, "dY_next");
    check_align(dH_next, "dH_next");
    require(y_dtype == TLORA_BF16 || y_dtype == TLORA_F32, TLORA_ERR_ARG,
            "Y dtype must be bf16 or f32");
    require(next->device == layer->device, TLORA_ERR_ARG, "layers on different devices");
    require(dH_next != H && dH_next != Y && dH_next != X, TLORA_ERR_ARG,
            "dH_next must not alias this layer's operands");
    DeviceGuard g(layer->device);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (zero_next)
      TL_CUDA(cudaMemsetAsync(dH_next, 0, (size_t)next_plan->P.T * next->L.R * 2, s));
    const Gemm2Secondary sec = make_lowrank2(next, next_plan, 1, dY_next, dH_next);
    run_fwd_gemm(layer, plan, X, H, Y, y_dtype, s, &sec);
  });
}

int tlora_forward_gemm_rs(tlora_layer* layer, const tlora_plan* plan, const void* X, const void* H,
                          void* const* recv_ptrs, int32_t world, int32_t rank, int64_t slot_rows,
                          int64_t dst_row0, void* stream) {
  return guarded([&] {
    check_bound(layer, plan);
    check_align(X, "X");
    check_align(H, "H");
    require(!plan->gathered, TLORA_ERR_PLAN,
            "the fused reduce-scatter epilogue does not take a gathered plan");
    require(recv_ptrs != nullptr && world >= 1 && world <= 8 && rank >= 0 && rank < world,
            TLORA_ERR_ARG, "need 1..8 receive buffers and a rank in [0, world)");
    const auto& L = layer->L;
    const int64_t T = plan->P.T, d = L.d, k = L.k, R = L.R;
    require(T % world == 0, TLORA_ERR_SHAPE, "tokens must divide evenly over the ranks");
    require(k % 64 == 0, TLORA_ERR_SHAPE, "fused reduce-scatter needs k % 64 == 0");
    require(dst_row0 >= 0 && dst_row0 + T / world <= slot_rows, TLORA_ERR_ARG,
            "receive slot too small for this plan");
    for (int p = 0; p < world; ++p) check_align(recv_ptrs[p], "receive buffer");
    DeviceGuard g(layer->device);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    GemmArgs a{};
    a.tiles = plan->tiles[TLORA_L_FWD].p;
    a.num_tiles = (int)plan->P.tiles[TLORA_L_FWD].size();
    a.M = (int)T;
    a.N = (int)k;
    a.ldo = k;
    for (int p = 0; p < world; ++p) a.peer[p] = recv_ptrs[p];
    a.peer_rank = rank;
    a.peer_world = world;
    a.rows_per_rank = T / world;
    a.slot_rows = slot_rows;
    a.dst_row0 = dst_row0;
    const CUtensorMap ma0 = tmap_k(X, d, T, 128);
    const CUtensorMap mb0 = tmap_k(layer->Wt16.p, d, k, 128);
    const CUtensorMap ma1 = tmap_k(H, R, T, 128);
    const CUtensorMap mb1 = tmap_k(layer->BcatT.p, R, k, 128);
    launch_gemm2<tlora::EPI_PEER, 5>(ma0, mb0, ma1, mb1, a, layer->sm_count, s, TLORA_L_FWD,
                                     2.0 * T * d * k + 2.0 * (double)plan->P.tok_rank * k);
  });
}

int tlora_reduce_slots(const void* recv, int32_t world, int64_t slot_rows, int64_t row0,
                       int64_t rows, int64_t k, void* out, void* stream) {
  return guarded([&] {
    check_align(recv, "recv");
    check_align(out, "out");
    require(world >= 1 && rows >= 0 && k % 8 == 0 && row0 + rows <= slot_rows, TLORA_ERR_ARG,
            "bad slot geometry");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int64_t n8 = rows * k / 8;
    if (n8 == 0) return;
    const int blocks = (int)std::min<int64_t>(tlora::ceil_div(n8, 256), 4 * 148);
    reduce_slots_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<const __nv_bfloat16*>(recv), world,
                                               slot_rows, row0, rows, k,
                                               reinterpret_cast<__nv_bfloat16*>(out));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    TL_CUDA(cudaGetLastError());
  });
}

int tlora_backward(tlora_layer* layer, const tlora_plan* plan, const void* dY, const void* X,
                   const void* H_stash, void* dX, float beta, void* stream) {
  return guarded([&] {
    check_bound(layer, plan);
    check_align(dY, "dY");
    check_align(X, "X");
    check_align(H_stash, "H_stash");
    if (dX) check_align(dX, "dX");
    DeviceGuard g(layer->device);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    __nv_bfloat16* dH =
        plan_scratch<__nv_bfloat16>(plan, s, kScratchDh, (size_t)plan->P.T * layer->L.R);
    run_dh(layer, plan, dY, dH, s);
    if (dX) run_dx(layer, plan, dY, dH, dX, 0.f, s);
    run_grads(layer, plan, H_stash, dY, dH, X, true, true, beta, s);
  });
}

int tlora_backward_dh(tlora_layer* layer, const tlora_plan* plan, const void* dY, void* dH,
                      void* stream) {
  return guarded([&] {
    check_bound(layer, plan);
    check_align(dY, "dY");
    check_align(dH, "dH");
    DeviceGuard g(layer->device);
    run_dh(layer, plan, dY, dH, reinterpret_cast<cudaStream_t>(stream));
  });
}

int tlora_backward_dx(tlora_layer* layer, const tlora_plan* plan, const void* dY, const void* dH,
                      void* dX, float beta, void* stream) {
  return guarded([&] {
    check_bound(layer, plan);
    check_align(dY, "dY");
    check_align(dH, "dH");
    check_align(dX, "dX");
    DeviceGuard g(layer->device);
    run_dx(layer, plan, dY, dH, dX, beta, reinterpret_cast<cudaStream_t>(stream));
  });
}

int tlora_backward_dx_dh(tlora_layer* layer, const tlora_plan* plan, const void* dY,
                         const void* dH, void* dX, float beta, tlora_layer* next,
                         const tlora_plan* next_plan, const void* dY_next, void* dH_next,
                         int zero_next, void* stream) {
  return guarded([&] {
    check_bound(layer, plan);
    check_bound(next, next_plan);
    check_align(dY, "dY");
    check_align(dH, "dH");
    check_align(dX, "dX");
    check_align(dY_next, "dY_next");
    check_align(dH_next, "dH_next");
    require(next->device == layer->device, TLORA_ERR_ARG, "layers on different devices");
    require(dH_next != dH && dH_next != dX && dH_next != dY, TLORA_ERR_ARG,
            "dH_next must not alias this layer's operands");
    DeviceGuard g(layer->device);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (zero_next)
      TL_CUDA(cudaMemsetAsync(dH_next, 0, (size_t)next_plan->P.T * next->L.R * 2, s));
    const Gemm2Secondary sec = make_lowrank2(next, next_plan, 1, dY_next, dH_next);
    run_dx(layer, plan, dY, dH, dX, beta, s, &sec);
  });
}

int tlora_backward_dx_shrink(tlora_layer* layer, const tlora_plan* plan, const void* dY,
                             const void* dH, void* dX, float beta, tlora_layer* next,
                             const tlora_plan* next_plan, const void* X_next, void* H_next,
                             int zero_next, void* stream) {
  return guarded([&] {
    check_bound(layer, plan);
    check_bound(next, next_plan);
    check_align(dY, "dY");
    check_align(dH, "dH");
    check_align(dX, "dX");
    check_align(X_next, "X_next");
    check_align(H_next, "H_next");
    require(next->device == layer->device, TLORA_ERR_ARG, "layers on different devices");
    require(H_next != dH && H_next != dX && H_next != dY, TLORA_ERR_ARG,
            "H_next must not alias this layer's operands");
    DeviceGuard g(layer->device);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (zero_next)
      TL_CUDA(cudaMemsetAsync(H_next, 0, (size_t)next_plan->P.T * next->L.R * 2, s));
    const Gemm2Secondary sec = make_lowrank2(next, next_plan, 0, X_next, H_next);
    run_dx(layer, plan, dY, dH, dX, beta, s, &sec);
  });
}

int tlora_backward_grads(tlora_layer* layer, const tlora_plan* plan, const void* H,
                         const void* dY, const void* X, const void* dH, float beta, void* stream) {
  return guarded([&] {
    check_bound(layer, plan);
    check_align(H, "H");
    check_align(dY, "dY");
    check_align(X, "X");
    check_align(dH, "dH");
    DeviceGuard g(layer->device);
    run_grads(layer, plan, H, dY, dH, X, true, true, beta, reinterpret_cast<cudaStream_t>(stream));
  });
}

int tlora_backward_grad_b(tlora_layer* layer, const tlora_plan* plan, const void* H,
                          const void* dY, float beta, void* stream) {
  return guarded([&] {
    check_bound(layer, plan);
    check_align(H, "H");
    check_align(dY, "dY");
    DeviceGuard g(layer->device);
    run_grads(layer, plan, H, dY, nullptr, nullptr, true, false, beta,
              reinterpret_cast<cudaStream_t>(stream));
  });
}

int tlora_backward_grad_a(tlora_layer* layer, const tlora_plan* plan, const void* X,
                          const void* dH, float beta, void* stream) {
  return guarded([&] {
    check_bound(layer, plan);
    check_align(X, "X");
    check_align(dH, "dH");
    DeviceGuard g(layer->device);
    run_grads(layer, plan, nullptr, nullptr, dH, X, false, true, beta,
              reinterpret_cast<cudaStream_t>(stream));
  });
}

long long tlora_launch_count(void) { return g_launches.load(); }

int tlora_set_tile_scheduler(int device, int mode) {
  return guarded([&] {
    require(mode >= -1 && mode <= 1, TLORA_ERR_ARG, "mode must be -1 (environment), 0 or 1");
    std::lock_guard<std::mutex> lk(g_sched_mu);
    if (mode < 0) g_sched_mode.erase(device);
    else g_sched_mode[device] = mode;
  });
}

int tlora_set_sm_budget(int device, int32_t gemm_sms, int32_t lowrank_sms) {
  return guarded([&] {
    require(gemm_sms >= 0 && lowrank_sms >= 0, TLORA_ERR_ARG, "negative SM budget");
    std::lock_guard<std::mutex> lk(g_budget_mu);
    if (gemm_sms == 0 && lowrank_sms == 0) g_budget.erase(device);
    else g_budget[device] = {gemm_sms, lowrank_sms};
  });
}

int tlora_profile_begin(void) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (auto& r : g_prof) {
      cudaEventDestroy(r.e0);
      cudaEventDestroy(r.e1);
    }
    g_prof.clear();
    g_prof_on = true;
  });
}

int tlora_profile_end(int32_t* counts, double* total_ms, double* total_flops) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_on = false;
    for (int l = 0; l < TLORA_PROF_KINDS; ++l) {
      if (counts) counts[l] = 0;
      if (total_ms) total_ms[l] = 0.0;
      if (total_flops) total_flops[l] = 0.0;
    }
    for (auto& r : g_prof) {
      TL_CUDA(cudaEventSynchronize(r.e1));
      float ms = 0.f;
      TL_CUDA(cudaEventElapsedTime(&ms, r.e0, r.e1));
      if (r.launch >= 0 && r.launch < TLORA_PROF_KINDS) {
        if (counts) counts[r.launch] += 1;
        if (total_ms) total_ms[r.launch] += ms;
        if (total_flops) total_flops[r.launch] += r.flops;
      }
      cudaEventDestroy(r.e0);
      cudaEventDestroy(r.e1);
    }
    g_prof.clear();
  });
}

int tlora_op_cost(int64_t tokens, int64_t d, int64_t k, int32_t num_slots,
                  const int64_t* tokens_per_slot, const int32_t* ranks, int fused, double* flops,
                  double* bytes_moved, long long* kernel_launches) {
  return guarded([&] {
    require(num_slots >= 0 && (num_slots == 0 || (tokens_per_slot && ranks)), TLORA_ERR_ARG,
            "bad slot arrays");
    // fused_lora.hpp:95-100 / :148-151 — identical operation order, so bit-identical doubles
    const double T = static_cast<double>(tokens);
    const double dd = static_cast<double>(d), kk = static_cast<double>(k);
    double f = 2.0 * T * dd * kk;
    double b = 8.0 * (T * dd + dd * kk + T * kk);
    long long l = 1;
    for (int s = 0; s < num_slots; ++s) {
      if (tokens_per_slot[s] == 0) continue;  // fused_lora.hpp:104 / :154
      const double n = static_cast<double>(tokens_per_slot[s]);
      const double r = static_cast<double>(ranks[s]);
      f += 2.0 * n * dd * r + 2.0 * n * r * kk;
      if (fused) {
        b += 8.0 * (dd * r + r * kk + 2.0 * n * r);  // :116
      } else {
        b += 8.0 * (2.0 * n * dd + dd * r + r * kk + 4.0 * n * r + 2.0 * n * kk);  // :159
        l += 4;                                                                  // :160
      }
    }
    if (flops) *flops = f;
    if (bytes_moved) *bytes_moved = b;
    if (kernel_launches) *kernel_launches = l;
  });
}

int tlora_segments(int64_t tokens, const int32_t* token_slot, int32_t num_slots, int64_t* perm,
                   int64_t* offsets) {
  return guarded([&] {
    require(tokens >= 0 && num_slots >= 1, TLORA_ERR_ARG, "bad sizes");
    require(tokens == 0 || (token_slot && perm), TLORA_ERR_ARG, "null argument");
    require(offsets != nullptr, TLORA_ERR_ARG, "offsets is null");
    std::vector<int64_t> cnt(num_slots + 1, 0);  // counting sort: stable, rows ascending
    for (int64_t t = 0; t < tokens; ++t) {
      const int32_t s = token_slot[t];
      require(s >= 0 && s < num_slots, TLORA_ERR_REGISTRY,
              "token " + std::to_string(t) + " names slot " + std::to_string(s) +
                  " outside the registry");
      ++cnt[s + 1];
    }
    for (int32_t s = 0; s < num_slots; ++s) cnt[s + 1] += cnt[s];
    std::memcpy(offsets, cnt.data(), (num_slots + 1) * sizeof(int64_t));
    for (int64_t t = 0; t < tokens; ++t) perm[cnt[token_slot[t]]++] = t;
  });
}

int tlora_partition(int32_t group_batch, int32_t n, int32_t* n_out, int32_t* per_nano) {
  return guarded([&] {
    // nano_pipeline.hpp:51-60
    if (group_batch < 1) throw std::invalid_argument("partition: group_batch must be >= 1");
    if (n < 1) throw std::invalid_argument("partition: N must be >= 1");
    const int32_t nn = std::min(n, group_batch);
    const int32_t base = group_batch / nn, extra = group_batch % nn;
    if (n_out) *n_out = nn;
    if (per_nano)
      for (int32_t i = 0; i < nn; ++i) per_nano[i] = base + (i < extra ? 1 : 0);
  });
}

int tlora_aimd_step(int32_t* n, int32_t* has_prev, double* t_prev, int32_t alpha, double beta,
                    double tau_rel, double t_t) {
  return guarded([&] {
    require(n && has_prev && t_prev, TLORA_ERR_ARG, "null AIMD state");
    // nano_pipeline.hpp:43-46 (validate) and :99-112
    if (*n < 1 || alpha < 1 || beta <= 0.0 || beta >= 1.0 || tau_rel < 0.0)
      throw std::invalid_argument("AimdState: invalid controller parameters");
    if (t_t < 0.0) throw std::invalid_argument("aimd_step: negative iteration time");
    int32_t next = *n;
    if (*has_prev) {
      const double margin = tau_rel * (*t_prev);
      if (t_t <= *t_prev - margin)
        next = *n + alpha;
      else
        next = std::max(1, static_cast<int>(std::floor(beta * *n)));
    }
    *n = next;
    *has_prev = 1;
    *t_prev = t_t;
  });
}

}  // extern "C"

#include "tlora_comm.cuh"
