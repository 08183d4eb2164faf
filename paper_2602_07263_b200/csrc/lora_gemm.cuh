// lora_gemm.cuh — the one tcgen05 GEMM engine behind every fused multi-LoRA launch.
//
//   D[m0:m0+128, n0:n0+BN] = sum over K-segments s of  A_s[m, k] * B_s[n, k]
//
// Every launch walks a host-built tile table (the rank-aware tile plan, see
// tlora_plan.cpp): each entry names an output tile and up to two K-segments.
//   * fused forward  Y  = X·W  (+ segment 1: H·Bᵀcat over the tile's packed rank range)
//   * shrink         H  = X·Acat, masked to each token's own job columns
//   * backward       dX = dY·Wᵀ (+ segment 1: dH·Aᵀcat), dH = dY·Bᵀcat (masked)
//   (the 2-CTA variant for the base GEMMs is lora_gemm2.cuh; the per-job adapter-gradient
//    GEMM with MN-major operands is lora_grad.cuh)
// Reference semantics: proj/include/lora_fleet/fused_lora.hpp:84-119 (forward); the
// backward is new (the reference has none).
//
// Structure (persistent, warp-specialised, 1 CTA per SM):
//   warp 0      TMA producer (one elected lane), STAGES-deep smem ring
//   warp 1      MMA issuer (one lane) — tcgen05.mma 128xBNx16, accumulator in TMEM
//   warp 2      TMEM allocator (2 x BN fp32 columns: double-buffered accumulator)
//   warps 4..7  epilogue: tcgen05.ld -> convert / mask / accumulate -> st.global
#pragma once
#include "sm100_ptx.cuh"

namespace tlora {

constexpr int kBM = 128;
constexpr int kBK = 64;  // one 128-byte swizzle atom of bf16 along K per stage
constexpr int kGemmThreads = 256;

// One output tile and its (up to two) K-segments, in elements. Built on the host.
struct TileDesc {
  int32_t m0, n0;
  int32_t kb0, ke0;  // segment 0 (operands A0/B0)
  int32_t kb1, ke1;  // segment 1 (operands A1/B1); empty when kb1 >= ke1
  int32_t split;     // split-K partial index (EPI_F32 only)
  int32_t pad;
};
static_assert(sizeof(TileDesc) == 32, "TileDesc layout is part of the plan ABI");

enum EpiMode : int {
  EPI_BF16 = 0,       // out bf16 [M x N], ldo
  EPI_BF16_MASK = 1,  // as EPI_BF16, zero where column is outside the row's job range
  EPI_F32 = 2,        // out fp32, optional beta-accumulate, split partial buffers
  EPI_PEER = 3,       // bf16 rows stored into the owning rank's receive slot (NVLink peer
                      // memory): fused reduce-scatter of a row-parallel TP GEMM
};

struct GemmArgs {
  const TileDesc* tiles;
  int num_tiles;
  int M, N;          // output bounds (rows, cols)
  void* out;
  int64_t ldo;       // elements
  int64_t split_stride;  // elements between split-K partial planes (EPI_F32)
  float beta;        // EPI_F32 / EPI_BF16: out = acc + beta * out
  // EPI_BF16_MASK: column window per row = [col_lo[slot], col_hi[slot])
  const int32_t* row_slot;
  const int32_t* slot_col_lo;
  const int32_t* slot_col_hi;
  // EPI_PEER: output row r goes to rank r / rows_per_rank, into its receive buffer
  // peer[dest] laid out [world][slot_rows][ldo], slot = this rank, row dst_row0 + r % rpr
  void* peer[8];
  int32_t peer_rank, peer_world;
  int64_t rows_per_rank, slot_rows, dst_row0;
  // EPI_BF16 / EPI_F32 (non-split): accumulator row r is stored to output row row_map[r]
  // (gathered plans: operands in job-sorted order, Y / dX in the caller's token order)
  const int32_t* row_map;
  // 2-CTA fused GEMM: dynamic tile scheduler (self-resetting global ticket; null = static
  // round-robin). Only read from args (the main tiles' GemmArgs) of a launch.
  int32_t* tile_counter;
  // 2-CTA fused GEMM, EPI_BF16 main tiles: tail split-K (tlora_capi.cu tail_split). A tile
  // with pad = 1 + 2*slot accumulates the first K half and writes its fp32 partial to
  // split_ws[slot] (256 x 256), then raises split_flags[slot*8 + cta*4 + warp]; the tile
  // with pad = 2 + 2*slot accumulates the rest (+ the LoRA K-extension), waits for those
  // flags, adds the partial and stores as usual (one bf16 rounding), and clears them.
  float* split_ws;
  int32_t* split_flags;
};

template <int BN, int STAGES>
struct GemmSmem {
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kBarOffset = STAGES * kStageBytes;
  // full[STAGES], empty[STAGES], tmem_full[2], tmem_empty[2], tmem base (u32)
  static constexpr int kTotal = kBarOffset + (2 * STAGES + 4) * 8 + 16;
  static constexpr int kDynamic = kTotal + 1024;  // slack for 1024-B alignment
};

// Store one 32-column chunk of an accumulator row (fp32 bits in v) per the epilogue mode.
template <int EPI>
__device__ __forceinline__ void epi_store32(const GemmArgs& args, int split, int row, int col0,
                                            const uint32_t (&v)[32], int lo, int hi) {
  using namespace ptx;
  if (row >= args.M || col0 >= args.N) return;
  if constexpr (EPI == EPI_PEER) {
    const int64_t dest = row / args.rows_per_rank, lrow = row % args.rows_per_rank;
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(args.peer[dest]) +
                       ((int64_t)args.peer_rank * args.slot_rows + args.dst_row0 + lrow) * args.ldo +
                       col0;
    uint4* o4 = reinterpret_cast<uint4*>(o);  // N % 32 == 0 is required for this mode
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 w;
      w.x = pack_bf16x2(__uint_as_float(v[8 * q + 0]), __uint_as_float(v[8 * q + 1]));
      w.y = pack_bf16x2(__uint_as_float(v[8 * q + 2]), __uint_as_float(v[8 * q + 3]));
      w.z = pack_bf16x2(__uint_as_float(v[8 * q + 4]), __uint_as_float(v[8 * q + 5]));
      w.w = pack_bf16x2(__uint_as_float(v[8 * q + 6]), __uint_as_float(v[8 * q + 7]));
      o4[q] = w;
    }
    return;
  } else if constexpr (EPI == EPI_BF16 || EPI == EPI_BF16_MASK) {
    float f[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      f[i] = __uint_as_float(v[i]);
      if constexpr (EPI == EPI_BF16_MASK) {
        const int col = col0 + i;
        if (col < lo || col >= hi) f[i] = 0.f;
      }
    }
    const int64_t orow = (EPI == EPI_BF16 && args.row_map) ? (int64_t)args.row_map[row] : row;
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(args.out) + orow * args.ldo + col0;
    if (col0 + 32 <= args.N) {
      uint4* o4 = reinterpret_cast<uint4*>(o);
      if (args.beta != 0.f) {  // out = acc + beta * out (in fp32, one bf16 rounding)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint4 p = o4[q];
          const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&p);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 pf = __bfloat1622float2(h[e]);
            f[8 * q + 2 * e] += args.beta * pf.x;
            f[8 * q + 2 * e + 1] += args.beta * pf.y;
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 w;
        w.x = pack_bf16x2(f[8 * q + 0], f[8 * q + 1]);
        w.y = pack_bf16x2(f[8 * q + 2], f[8 * q + 3]);
        w.z = pack_bf16x2(f[8 * q + 4], f[8 * q + 5]);
        w.w = pack_bf16x2(f[8 * q + 6], f[8 * q + 7]);
        // Y / dX: nothing in the step re-reads them soon, so they go out evict-first and
        // their DRAM write-back happens under this tensor-bound GEMM instead of being left
        // dirty in L2 for the next (HBM-bound) launch to pay. H / dH (MASK) stay normal:
        // the next fused GEMM reads them.
        if constexpr (EPI == EPI_BF16 && TLORA_EPI_EVICT_FIRST)
          st_global_v4_evict_first(o4 + q, w);
        else
          o4[q] = w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col0 + i < args.N)
          o[i] = __float2bfloat16_rn(args.beta != 0.f ? f[i] + args.beta * __bfloat162float(o[i])
                                                      : f[i]);
    }
  } else {
    const int64_t orow = args.row_map ? (int64_t)args.row_map[row] : row;
    float* o = reinterpret_cast<float*>(args.out) + (int64_t)split * args.split_stride +
               orow * args.ldo + col0;
    if (col0 + 32 <= args.N) {
      float4* o4 = reinterpret_cast<float4*>(o);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 w = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                               __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
        if (args.beta != 0.f) {
          const float4 p = o4[q];
          w.x += args.beta * p.x; w.y += args.beta * p.y;
          w.z += args.beta * p.z; w.w += args.beta * p.w;
        }
        o4[q] = w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        if (col0 + i >= args.N) continue;
        float w = __uint_as_float(v[i]);
        if (args.beta != 0.f) w += args.beta * o[i];
        o[i] = w;
      }
    }
  }
}

template <int BN, bool A_MN, bool B_MN, int EPI, int STAGES>
__global__ void __launch_bounds__(kGemmThreads, 1)
    lora_gemm_kernel(const __grid_constant__ CUtensorMap tmA0,
                     const __grid_constant__ CUtensorMap tmB0,
                     const __grid_constant__ CUtensorMap tmA1,
                     const __grid_constant__ CUtensorMap tmB1, const GemmArgs args) {
  using namespace ptx;
  using L = GemmSmem<BN, STAGES>;
  static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "BN");
  constexpr uint32_t kTmemCols = 2 * BN;  // 64..512, power of two for BN in {32,64,128,256}
  static_assert((kTmemCols & (kTmemCols - 1)) == 0, "TMEM columns must be a power of two");
  constexpr uint32_t kIdesc = make_idesc_bf16(kBM, BN, A_MN, B_MN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x / 32;
  const uint32_t lane = threadIdx.x % 32;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA0);
    tma_prefetch_desc(&tmB0);
    tma_prefetch_desc(&tmA1);
    tma_prefetch_desc(&tmB1);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 4);  // one arrive per epilogue warp
    }
    fence_mbar_init();
    fence_proxy_async_smem();
  }
  if (warp == 2) tmem_alloc(tmem_base_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;
  pdl_launch_dependents();   // persistent grid: all CTAs are resident, dependents may queue
  pdl_wait_prerequisites();  // inputs written by the previous launch are visible after this

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < args.num_tiles; t += gridDim.x) {
        const TileDesc td = args.tiles[t];
#pragma unroll 1
        for (int seg = 0; seg < 2; ++seg) {
          const int kb = seg == 0 ? td.kb0 : td.kb1;
          const int ke = seg == 0 ? td.ke0 : td.ke1;
          const CUtensorMap* ma = seg == 0 ? &tmA0 : &tmA1;
          const CUtensorMap* mb = seg == 0 ? &tmB0 : &tmB1;
#pragma unroll 1
          for (int k = kb; k < ke; k += kBK) {
            mbar_wait(&empty_bar[stage], phase ^ 1);
            uint8_t* sa = smem + stage * L::kStageBytes;
            uint8_t* sb = sa + L::kABytes;
            mbar_arrive_expect_tx(&full_bar[stage], L::kStageBytes);
            if constexpr (!A_MN) {
              tma_load_2d(sa, ma, &full_bar[stage], k, td.m0);
            } else {
#pragma unroll
              for (int c = 0; c < kBM / 64; ++c)
                tma_load_2d(sa + c * (64 * kBK * 2), ma, &full_bar[stage], td.m0 + 64 * c, k);
            }
            if constexpr (!B_MN) {
              tma_load_2d(sb, mb, &full_bar[stage], k, td.n0);
            } else {
#pragma unroll
              for (int c = 0; c < BN / 64; ++c)
                tma_load_2d(sb + c * (64 * kBK * 2), mb, &full_bar[stage], td.n0 + 64 * c, k);
            }
#ifndef TLORA_PREFETCH_LOWRANK
#define TLORA_PREFETCH_LOWRANK 0
#endif
            if constexpr (TLORA_PREFETCH_LOWRANK && !A_MN && !B_MN) {  // L2 prefetch ahead
              const int kp = k + STAGES * kBK;
              if (kp < ke) {
                tma_prefetch_2d(ma, kp, td.m0);
                tma_prefetch_2d(mb, kp, td.n0);
              }
            }
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc_iter = 0;
      for (int t = blockIdx.x; t < args.num_tiles; t += gridDim.x) {
        const TileDesc td = args.tiles[t];
        const int nkb = (td.ke0 > td.kb0 ? (td.ke0 - td.kb0 + kBK - 1) / kBK : 0) +
                        (td.ke1 > td.kb1 ? (td.ke1 - td.kb1 + kBK - 1) / kBK : 0);
        if (nkb == 0) continue;
        const int acc = acc_iter & 1;
        const uint32_t acc_phase = (acc_iter >> 1) & 1;
        ++acc_iter;
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
#pragma unroll 1
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * L::kStageBytes);
          const uint32_t sb = sa + L::kABytes;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            uint64_t ad, bd;
            if constexpr (!A_MN) ad = make_smem_desc_kmajor(sa + kk * 32);
            else ad = make_smem_desc_mnmajor(sa + kk * 16 * 128, 64 * kBK * 2);
            if constexpr (!B_MN) bd = make_smem_desc_kmajor(sb + kk * 32);
            else bd = make_smem_desc_mnmajor(sb + kk * 16 * 128, 64 * kBK * 2);
            mma_bf16_ss(d_tmem, ad, bd, kIdesc, (kb | kk) != 0 ? 1u : 0u);
          }
          mma_commit(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull_bar[acc]);
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    const int ew = warp & 3;  // TMEM lane quadrant this warp may access
    int acc_iter = 0;
    for (int t = blockIdx.x; t < args.num_tiles; t += gridDim.x) {
      const TileDesc td = args.tiles[t];
      const bool empty_k = !(td.ke0 > td.kb0) && !(td.ke1 > td.kb1);
      const int row = td.m0 + ew * 32 + (int)lane;
      int acc = 0;
      if (!empty_k) {
        acc = acc_iter & 1;
        const uint32_t acc_phase = (acc_iter >> 1) & 1;
        ++acc_iter;
        mbar_wait(&tfull_bar[acc], acc_phase);
        tc_fence_after();
      }
      int lo = 0, hi = 0x7fffffff;
      if constexpr (EPI == EPI_BF16_MASK) {
        if (row < args.M) {
          const int s = args.row_slot[row];
          lo = args.slot_col_lo[s];
          hi = args.slot_col_hi[s];
        }
      }
      const uint32_t t_row = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t v[32];
        if (!empty_k) {
          tmem_ld_32x32b_x32(t_row + c, v);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0u;
        }
        epi_store32<EPI>(args, td.split, row, td.n0 + c, v, lo, hi);
      }
      if (!empty_k) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty_bar[acc]);
      }
    }
  }

  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
}

}  // namespace tlora
