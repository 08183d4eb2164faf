// lora_grad.cuh — per-job adapter-gradient GEMM in transposed form.
//
//   dB_jᵀ [k x r_j] = dY_jᵀ [k x T_j] · H_j  [T_j x r_j]
//   dA_j  [d x r_j] = X_jᵀ  [d x T_j] · dH_j [T_j x r_j]      (dA_jᵀ is what is stored)
//
// M = the layer dimension (k or d, 128-row tiles), N = the job's own rank columns
// (64-column MMA granules, runtime N <= 128), K = the job's token range only. A packed
// formulation (M = packed rank space, K = tokens of every job in the tile) multiplies the
// masked zeros of H/dH; here no MMA work is spent on other jobs' rows, and dY / X are read
// once per M-tile row band: the launch is HBM-bound at ~the minimal bytes.
//
// Operands are both MN-major (read straight from the row-major T x N activations and the
// T x R masked H / dH stash): A box 64(M) x 64(K) x 2 chunks, B box 64(N) x 64(K) x N/64
// chunks, SWIZZLE_128B. The epilogue stores the fp32 accumulator transposed into the packed
// gradient layout (row = packed rank column, col = M index): for a fixed rank column the 32
// lanes of a warp write 32 consecutive floats (coalesced). Columns >= r_j belong to the next
// job and are never stored. Split-K partials go to per-split planes reduced in fixed order.
#pragma once
#include "lora_gemm.cuh"

namespace tlora {

template <int STAGES>
struct GradSmem {
  static constexpr int kABytes = 128 * kBK * 2;  // 2 MN chunks
  static constexpr int kBBytes = 128 * kBK * 2;  // up to 2 MN chunks (N <= 128)
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kBarOffset = STAGES * kStageBytes;
  static constexpr int kTotal = kBarOffset + (2 * STAGES + 4) * 8 + 16;
  static constexpr int kDynamic = kTotal + 1024;
};

// Up to two independent gradient problems in one persistent launch (dB and dA of a
// projection): tiles [0, n0) come from problem 0 (operand maps tmA0 / tmB0), tiles
// [n0, n0 + n1) from problem 1 (tmA1 / tmB1); each CTA continues across the boundary, so the
// tail of one fills with the other.
struct GradArgs {
  GemmArgs job[2];
  // optional static schedule (tlora::grad_schedule, built for gridDim.x CTAs): CTA b runs
  // tiles sched_idx[sched_off[b] .. sched_off[b+1]); null -> round-robin t += gridDim.x
  const int32_t* sched_off;
  const int32_t* sched_idx;
};

// Tile fields: m0 = M offset, n0 = first packed rank column of the job (chunk), kb0/ke0 =
// token range, split = partial plane, pad = number of valid rank columns (<= 128).
template <int STAGES>
__global__ void __launch_bounds__(kGemmThreads, 1)
    lora_grad_kernel(const __grid_constant__ CUtensorMap tmA0,
                     const __grid_constant__ CUtensorMap tmB0,
                     const __grid_constant__ CUtensorMap tmA1,
                     const __grid_constant__ CUtensorMap tmB1, const GradArgs gargs) {
  using namespace ptx;
  using L = GradSmem<STAGES>;
  constexpr uint32_t kTmemCols = 256;
  constexpr uint32_t kChunk = 64 * kBK * 2;

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

  const int n_first = gargs.job[0].num_tiles;
  const int n_total = n_first + gargs.job[1].num_tiles;
  // tile t -> (problem, its tile descriptor)
  auto tile_of = [&](int t, int& j) -> TileDesc {
    j = t < n_first ? 0 : 1;
    return gargs.job[j].tiles[j == 0 ? t : t - n_first];
  };
  // this CTA's tile sequence: positions [i0, i1) step di, tile = at(i)
  const bool sched = gargs.sched_off != nullptr;
  const int i0 = sched ? gargs.sched_off[blockIdx.x] : (int)blockIdx.x;
  const int i1 = sched ? gargs.sched_off[blockIdx.x + 1] : n_total;
  const int di = sched ? 1 : (int)gridDim.x;
  auto at = [&](int i) { return sched ? gargs.sched_idx[i] : i; };

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
      mbar_init(&tempty_bar[a], 4);
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
    if (lane == 0) {  // TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int i = i0; i < i1; i += di) {
        const int t = at(i);
        int j;
        const TileDesc td = tile_of(t, j);
        const CUtensorMap* tmA = j == 0 ? &tmA0 : &tmA1;
        const CUtensorMap* tmB = j == 0 ? &tmB0 : &tmB1;
        const int nch = (td.pad + 63) / 64;
#pragma unroll 1
        for (int k = td.kb0; k < td.ke0; k += kBK) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * L::kStageBytes;
          uint8_t* sb = sa + L::kABytes;
          mbar_arrive_expect_tx(&full_bar[stage], L::kABytes + nch * kChunk);
          tma_load_2d(sa, tmA, &full_bar[stage], td.m0, k);
          tma_load_2d(sa + kChunk, tmA, &full_bar[stage], td.m0 + 64, k);
          for (int c = 0; c < nch; ++c)
            tma_load_2d(sb + c * kChunk, tmB, &full_bar[stage], td.n0 + 64 * c, k);
          // L2 prefetch one smem ring ahead (HBM latency > what the ring covers)
#ifndef TLORA_PREFETCH_GRAD
#define TLORA_PREFETCH_GRAD 0
#endif
          const int kp = k + STAGES * kBK;
          if (TLORA_PREFETCH_GRAD && kp < td.ke0) {
            tma_prefetch_2d(tmA, td.m0, kp);
            tma_prefetch_2d(tmA, td.m0 + 64, kp);
            for (int c = 0; c < nch; ++c) tma_prefetch_2d(tmB, td.n0 + 64 * c, kp);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      int stage = 0;
      uint32_t phase = 0;
      int acc_iter = 0;
      for (int i = i0; i < i1; i += di) {
        const int t = at(i);
        int j;
        const TileDesc td = tile_of(t, j);
        const int nkb = td.ke0 > td.kb0 ? (td.ke0 - td.kb0 + kBK - 1) / kBK : 0;
        if (nkb == 0) continue;
        const uint32_t idesc = make_idesc_bf16(kBM, 64 * ((td.pad + 63) / 64), true, true);
        const int acc = acc_iter & 1;
        const uint32_t acc_phase = (acc_iter >> 1) & 1;
        ++acc_iter;
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 128;
#pragma unroll 1
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * L::kStageBytes);
          const uint32_t sb = sa + L::kABytes;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk)
            mma_bf16_ss(d_tmem, make_smem_desc_mnmajor(sa + kk * 16 * 128, kChunk),
                        make_smem_desc_mnmajor(sb + kk * 16 * 128, kChunk), idesc,
                        (kb | kk) != 0 ? 1u : 0u);
          mma_commit(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull_bar[acc]);
      }
    }
  } else if (warp >= 4) {  // epilogue: transposed, column-masked fp32 store
    const int ew = warp & 3;
    int acc_iter = 0;
    for (int i = i0; i < i1; i += di) {
      const int t = at(i);
      int j;
      const TileDesc td = tile_of(t, j);
      const GemmArgs& args = gargs.job[j];
      const bool empty_k = !(td.ke0 > td.kb0);
      const int mi = td.m0 + ew * 32 + (int)lane;  // M index (k or d)
      int acc = 0;
      if (!empty_k) {
        acc = acc_iter & 1;
        const uint32_t acc_phase = (acc_iter >> 1) & 1;
        ++acc_iter;
        mbar_wait(&tfull_bar[acc], acc_phase);
        tc_fence_after();
      }
      const uint32_t t_row = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * 128;
      float* out = reinterpret_cast<float*>(args.out) + (int64_t)td.split * args.split_stride;
#pragma unroll 1
      for (int c0 = 0; c0 < td.pad; c0 += 32) {
        uint32_t v[32];
        if (!empty_k) {
          tmem_ld_32x32b_x32(t_row + c0, v);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0u;
        }
        if (mi < args.M) {
#pragma unroll 4
          for (int i = 0; i < 32; ++i) {
            if (c0 + i >= td.pad) break;
            float* o = out + (int64_t)(td.n0 + c0 + i) * args.ldo + mi;
            float w = __uint_as_float(v[i]);
            if (args.beta != 0.f) w += args.beta * *o;
            *o = w;
          }
        }
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
