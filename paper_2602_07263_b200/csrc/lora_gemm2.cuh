// lora_gemm2.cuh — 2-CTA (cta_group::2) variant of the fused base+LoRA GEMM.
//
// The fused forward  Y = X·W (+ H·Bᵀcat over the tile's packed rank window) and the fused
// backward dX = dY·Wᵀ (+ dH·Aᵀcat) are >95% of the layer's FLOPs. They run here on CTA
// pairs: a cluster of 2 CTAs (one TPC) owns a 256 x 256 output tile; each CTA stages half
// of A (its 128 rows) and half of B (128 of the 256 N rows) per K block, and the leader
// CTA issues tcgen05.mma.cta_group::2 (M = 256, N = 256, K = 16) which reads both CTAs'
// shared memory. Per SM this halves operand shared-memory traffic versus a 1-CTA 128x256
// tile (64 B/clk of MMA reads + 64 B/clk of TMA writes), which is what lets the tensor
// pipe run at rate. Each CTA's TMEM holds its 128 rows x 256 fp32 columns, double
// buffered (512 columns), so the epilogue of tile i overlaps the MMAs of tile i+1.
//
// Synchronisation (barrier ownership):
//   full[s]   leader only; expect_tx(2 x stage bytes) by the leader's producer, the TMA
//             loads of BOTH CTAs complete on it (cp.async.bulk.tensor .cta_group::2).
//   empty[s]  both CTAs; the leader's tcgen05.commit multicasts one arrive to each.
//   tfull[a]  both CTAs; multicast commit after the last K block of a tile.
//   tempty[a] leader only; 8 arrives = 4 epilogue warps x 2 CTAs (remote arrive).
#pragma once
#include "lora_gemm.cuh"

namespace tlora {

#ifndef TLORA_TAIL_SPLIT_KERNEL
#define TLORA_TAIL_SPLIT_KERNEL 1  // 0: compile the fused GEMM without the split-K epilogue
#endif

constexpr int kBM2 = 256;  // rows per CTA pair
constexpr int kBN2 = 256;

template <int STAGES>
struct Gemm2Smem {
  static constexpr int kABytes = 128 * kBK * 2;  // this CTA's half of A
  static constexpr int kBBytes = 128 * kBK * 2;  // this CTA's half of B
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kBarOffset = STAGES * kStageBytes;
  static constexpr int kQ = 8;  // dynamic-scheduler tile queue depth
  // barriers: full[S], empty[S], tfull[2], tempty[2], qfull[kQ], qempty[kQ]; then the TMEM
  // base slot (16 B) and the tile queue (kQ x int32)
  static constexpr int kTotal = kBarOffset + (2 * STAGES + 4 + 2 * kQ) * 8 + 16 + kQ * 4;
  static constexpr int kDynamic = kTotal + 1024;
  // EPI_PEER staging: per epilogue warp two buffers of 32 rows x 64 bf16 columns, rows
  // padded to 144 B (conflict-free 16-B shared stores; each row stays one contiguous
  // 128-B bulk copy source)
  static constexpr int kStgRow = 144;
  static constexpr int kStgBuf = 32 * kStgRow;
  static constexpr int kStagingOffset = (kTotal + 127) / 128 * 128;
  static constexpr int kDynamicPeer = kStagingOffset + 4 * 2 * kStgBuf + 1024;
};

// Secondary tiles (args2, maps tmA2 / tmB2): another layer's shrink or dH on 256-token
// pair tiles, appended after the main tiles of the launch. They do not depend on the main
// tiles; they fill the tail of the persistent schedule. Tile: one K-segment [kb0, ke0),
// runtime N = td.pad (128 or 256, split N/2 per CTA; tmB2 boxes are 64 rows), masked bf16
// epilogue (EPI_BF16_MASK semantics with args2's row -> slot -> column window).
template <int EPI, int STAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1)
    lora_gemm2_kernel(const __grid_constant__ CUtensorMap tmA0,
                      const __grid_constant__ CUtensorMap tmB0,
                      const __grid_constant__ CUtensorMap tmA1,
                      const __grid_constant__ CUtensorMap tmB1,
                      const __grid_constant__ CUtensorMap tmA2,
                      const __grid_constant__ CUtensorMap tmB2, const GemmArgs args,
                      const GemmArgs args2) {
  using namespace ptx;
  using L = Gemm2Smem<STAGES>;
  constexpr uint32_t kTmemCols = 2 * kBN2;
  constexpr uint32_t kIdesc = make_idesc_bf16(kBM2, kBN2, false, false);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* qfull_bar = tempty_bar + 2;
  uint64_t* qempty_bar = qfull_bar + L::kQ;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(qempty_bar + L::kQ);
  int32_t* tile_q = reinterpret_cast<int32_t*>(tmem_base_slot + 4);

  const int warp = threadIdx.x / 32;
  const uint32_t lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster_id = blockIdx.x / 2;
  const int num_clusters = gridDim.x / 2;
  const int n_main = args.num_tiles;
  const int n_total = n_main + args2.num_tiles;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA0);
    tma_prefetch_desc(&tmB0);
    tma_prefetch_desc(&tmA1);
    tma_prefetch_desc(&tmB1);
    if (args2.num_tiles > 0) {
      tma_prefetch_desc(&tmA2);
      tma_prefetch_desc(&tmB2);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 8);
    }
    for (int q = 0; q < L::kQ; ++q) {
      mbar_init(&qfull_bar[q], 1);
      // leader: MMA issuer + 4 epilogue warps; peer: producer + 4 epilogue warps
      mbar_init(&qempty_bar[q], 10);
    }
    fence_mbar_init();
    fence_proxy_async_smem();
  }
  if (warp == 2) tmem_alloc_cg2(tmem_base_slot, kTmemCols);
  tc_fence_before();
  cluster_sync();  // peer barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;
  pdl_launch_dependents();   // persistent grid: all CTAs are resident, dependents may queue
  pdl_wait_prerequisites();  // inputs written by the previous launch are visible after this

  // Tile sequence of this CTA pair. Static: cluster_id, + num_clusters, ... Dynamic
  // (args.tile_counter): the leader's producer claims tiles from a global ticket (one tile
  // ahead) and publishes each index into a kQ-deep queue in BOTH CTAs' shared memory
  // (qfull: local arrive + remote arrive on the peer); every other role of both CTAs pops
  // the same sequence and releases the slot on the leader's qempty. Index n_total ends the
  // sequence. The ticket's last claim (value n_total + num_clusters - 1: every pair makes
  // exactly one failing claim) resets it to 0 for the next launch, which reads it only
  // after griddepcontrol.wait, i.e. after this grid has completed.
  const bool dyn = args.tile_counter != nullptr;
  uint32_t qseq = 0;
  auto q_pop = [&](bool remote_wait) -> int {  // one thread per consumer role
    const uint32_t slot = qseq % L::kQ, ph = (qseq / L::kQ) & 1;
    ++qseq;
    if (remote_wait) mbar_wait_cluster(&qfull_bar[slot], ph);
    else mbar_wait(&qfull_bar[slot], ph);
    const int t = *reinterpret_cast<volatile int32_t*>(&tile_q[slot]);
    if (leader) mbar_arrive(&qempty_bar[slot]);
    else mbar_arrive_cluster(mapa_shared(smem_u32(&qempty_bar[slot]), 0));
    return t;
  };
  auto q_push = [&](int t) {  // leader producer only
    const uint32_t slot = qseq % L::kQ, ph = (qseq / L::kQ) & 1;
    ++qseq;
    mbar_wait_cluster(&qempty_bar[slot], ph ^ 1);
    tile_q[slot] = t;
    st_shared_cluster_u32(mapa_shared(smem_u32(&tile_q[slot]), 1), (uint32_t)t);
    mbar_arrive(&qfull_bar[slot]);
    mbar_arrive_cluster(mapa_shared(smem_u32(&qfull_bar[slot]), 1));
  };
  // claim(): issue the ticket atomic only; its value is first used at the NEXT tile switch,
  // so the producer never stalls on the atomic's round trip before issuing a tile's loads.
  auto claim = [&]() -> int { return atomicAdd(args.tile_counter, 1); };
  auto resolve = [&](int v) -> int {
    if (v == n_total + num_clusters - 1) atomicExch(args.tile_counter, 0);
    return v < n_total ? v : n_total;
  };

  if (warp == 0) {
    // ===================== TMA producer (both CTAs) =====================
    if (lane == 0) {
      const uint32_t full0 = mapa_shared(smem_u32(full_bar), 0);
      int stage = 0;
      uint32_t phase = 0;
      int t_ahead = dyn && leader ? claim() : 0;
      auto next_tile = [&](int cur) -> int {
        if (!dyn) return cur < 0 ? cluster_id : cur + num_clusters;
        if (!leader) return q_pop(true);
        const int t = resolve(t_ahead);
        q_push(t);
        if (t < n_total) t_ahead = claim();  // claim the next tile while this one loads
        return t;
      };
      for (int t = next_tile(-1); t < n_total; t = next_tile(t)) {
        const bool sec = t >= n_main;
        const TileDesc td = sec ? args2.tiles[t - n_main] : args.tiles[t];
        const int am = td.m0 + 128 * (int)rank;
        if (sec) {  // another layer's shrink / dH: B half = N/2 rows in 64-row boxes
          const int half = td.pad / 2;
          const int bn = td.n0 + half * (int)rank;
#pragma unroll 1
          for (int k = td.kb0; k < td.ke0; k += kBK) {
            mbar_wait(&empty_bar[stage], phase ^ 1);
            uint8_t* sa = smem + stage * L::kStageBytes;
            uint8_t* sb = sa + L::kABytes;
            if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * (L::kABytes + half * kBK * 2));
            const uint32_t fb = full0 + stage * 8;
            tma_load_2d_cg2(sa, &tmA2, fb, k, am);
            for (int c = 0; c < half / 64; ++c)
              tma_load_2d_cg2(sb + c * 64 * kBK * 2, &tmB2, fb, k, bn + 64 * c);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          continue;
        }
        const int bn = td.n0 + 128 * (int)rank;
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
            if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * L::kStageBytes);
            const uint32_t fb = full0 + stage * 8;
            tma_load_2d_cg2(sa, ma, fb, k, am);
            tma_load_2d_cg2(sb, mb, fb, k, bn);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA only) =====================
    if (leader && lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc_iter = 0;
      auto next_tile = [&](int cur) -> int {
        if (!dyn) return cur < 0 ? cluster_id : cur + num_clusters;
        return q_pop(false);
      };
      for (int t = next_tile(-1); t < n_total; t = next_tile(t)) {
        const bool sec = t >= n_main;
        const TileDesc td = sec ? args2.tiles[t - n_main] : args.tiles[t];
        const int nkb = (td.ke0 > td.kb0 ? (td.ke0 - td.kb0 + kBK - 1) / kBK : 0) +
                        (!sec && td.ke1 > td.kb1 ? (td.ke1 - td.kb1 + kBK - 1) / kBK : 0);
        if (nkb == 0) continue;
        const uint32_t idesc = sec ? make_idesc_bf16(kBM2, td.pad, false, false) : kIdesc;
        const int acc = acc_iter & 1;
        const uint32_t acc_phase = (acc_iter >> 1) & 1;
        ++acc_iter;
        mbar_wait_cluster(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kBN2;
#pragma unroll 1
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * L::kStageBytes);
          const uint32_t sb = sa + L::kABytes;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk)
            mma_bf16_ss_cg2(d_tmem, make_smem_desc_kmajor(sa + kk * 32),
                            make_smem_desc_kmajor(sb + kk * 32), idesc, (kb | kk) != 0 ? 1u : 0u);
          mma_commit_cg2_mc(&empty_bar[stage], 0x3);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit_cg2_mc(&tfull_bar[acc], 0x3);
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue (both CTAs: own 128 rows x 256 cols) =====================
    const int ew = warp & 3;
    const uint32_t tempty0 = mapa_shared(smem_u32(tempty_bar), 0);
    int acc_iter = 0;
    auto next_tile = [&](int cur) -> int {
      if (!dyn) return cur < 0 ? cluster_id : cur + num_clusters;
      int t = 0;
      if (lane == 0) t = q_pop(!leader);
      return __shfl_sync(0xffffffffu, t, 0);
    };
    for (int t = next_tile(-1); t < n_total; t = next_tile(t)) {
      const bool sec = t >= n_main;
      const TileDesc td = sec ? args2.tiles[t - n_main] : args.tiles[t];
      const bool empty_k = !(td.ke0 > td.kb0) && (sec || !(td.ke1 > td.kb1));
      const int row = td.m0 + 128 * (int)rank + ew * 32 + (int)lane;
      int acc = 0;
      if (!empty_k) {
        acc = acc_iter & 1;
        const uint32_t acc_phase = (acc_iter >> 1) & 1;
        ++acc_iter;
        mbar_wait(&tfull_bar[acc], acc_phase);
        tc_fence_after();
      }
      int lo = 0, hi = 0x7fffffff;
      if (sec && row < args2.M) {
        const int sl = args2.row_slot[row];
        lo = args2.slot_col_lo[sl];
        hi = args2.slot_col_hi[sl];
      }
      const int ncols = sec ? td.pad : kBN2;
      const uint32_t t_row = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * kBN2;
      if constexpr (EPI == EPI_PEER) {
        if (!sec) {
          // Reduce-scatter epilogue: 64-column row chunks are converted to bf16 into a
          // shared-memory staging row, and each lane bulk-copies its row's 128 B straight
          // into the owner rank's receive slot (cp.async.bulk over NVLink): one 128-B
          // transfer per row and chunk instead of eight 16-B stores.
          uint8_t* stg = smem + L::kStagingOffset + ew * 2 * L::kStgBuf;
          const bool live = row < args.M;
          __nv_bfloat16* dst = nullptr;
          if (live) {
            const int64_t dest = row / args.rows_per_rank, lrow = row % args.rows_per_rank;
            dst = reinterpret_cast<__nv_bfloat16*>(args.peer[dest]) +
                  ((int64_t)args.peer_rank * args.slot_rows + args.dst_row0 + lrow) * args.ldo +
                  td.n0;
          }
#pragma unroll 1
          for (int c = 0; c < kBN2; c += 64) {
            uint32_t v0[32], v1[32];
            if (!empty_k) {
              tmem_ld_32x32b_x32(t_row + c, v0);
              tmem_ld_32x32b_x32(t_row + c + 32, v1);
              tmem_wait_ld();
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i) v0[i] = v1[i] = 0u;
            }
            uint8_t* rowp = stg + ((c >> 6) & 1) * L::kStgBuf + lane * L::kStgRow;
            bulk_wait_read<1>();  // the copy that last read this buffer has finished reading
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const uint32_t* src = q < 4 ? v0 + 8 * q : v1 + 8 * (q - 4);
              uint4 w;
              w.x = pack_bf16x2(__uint_as_float(src[0]), __uint_as_float(src[1]));
              w.y = pack_bf16x2(__uint_as_float(src[2]), __uint_as_float(src[3]));
              w.z = pack_bf16x2(__uint_as_float(src[4]), __uint_as_float(src[5]));
              w.w = pack_bf16x2(__uint_as_float(src[6]), __uint_as_float(src[7]));
              *reinterpret_cast<uint4*>(rowp + 16 * q) = w;
            }
            fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the bulk copy
            if (live && td.n0 + c < args.N) bulk_store_s2g(dst + c, rowp, 128);
            bulk_commit();
          }
          if (!empty_k) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty0 + acc * 8);
          }
          continue;
        }
      }
      // tail split-K roles (GemmArgs::split_ws): 1 = partial writer, 2 = finisher
#if TLORA_TAIL_SPLIT_KERNEL
      const int role = (EPI == EPI_BF16 && !sec && td.pad > 0) ? 2 - (td.pad & 1) : 0;
#else
      constexpr int role = 0;
#endif
      float* part = nullptr;
      int32_t* flag = nullptr;
      if (role) {
        const int slot = (td.pad - 1) >> 1;
        part = args.split_ws + ((size_t)slot * kBM2 + 128 * rank + ew * 32 + lane) * kBN2;
        flag = args.split_flags + slot * 8 + (int)rank * 4 + ew;
        if (role == 2) {  // the writer warp of the same rows has published its partial
          int f;
          do {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(f) : "l"(flag) : "memory");
            if (f != 0) break;
            __nanosleep(32);
          } while (true);
        }
      }
#pragma unroll 1
      for (int c = 0; c < ncols; c += 32) {
        uint32_t v[32];
        if (!empty_k) {
          tmem_ld_32x32b_x32(t_row + c, v);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0u;
        }
        if (role == 1) {
          float4* w = reinterpret_cast<float4*>(part + c);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            __stcg(w + q, make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                      __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3])));
          continue;
        }
        if (role == 2) {
          const float4* r4 = reinterpret_cast<const float4*>(part + c);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 pv = __ldcg(r4 + q);
            v[4 * q] = __float_as_uint(pv.x + __uint_as_float(v[4 * q]));
            v[4 * q + 1] = __float_as_uint(pv.y + __uint_as_float(v[4 * q + 1]));
            v[4 * q + 2] = __float_as_uint(pv.z + __uint_as_float(v[4 * q + 2]));
            v[4 * q + 3] = __float_as_uint(pv.w + __uint_as_float(v[4 * q + 3]));
          }
        }
        if (sec)
          epi_store32<EPI_BF16_MASK>(args2, 0, row, td.n0 + c, v, lo, hi);
        else
          epi_store32<EPI>(args, td.split, row, td.n0 + c, v, 0, 0x7fffffff);
      }
      if (role == 1) {  // every lane's partial row is written before the flag
        __threadfence();
        __syncwarp();
        if (lane == 0) asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flag), "r"(1) : "memory");
      } else if (role == 2) {
        __syncwarp();
        if (lane == 0) *reinterpret_cast<volatile int32_t*>(flag) = 0;  // for the next launch
      }
      if (!empty_k) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty0 + acc * 8);
      }
    }
    if constexpr (EPI == EPI_PEER) {
      bulk_wait_all();        // every bulk copy to a peer has been performed
      __threadfence_system();  // peer stores before completion
    }
  }

  tc_fence_before();
  cluster_sync();  // no CTA frees TMEM / exits while its peer may still address it
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_cg2(tmem_base, kTmemCols);
  }
}

}  // namespace tlora
