// tlora_plan.hpp — host-side rank-aware tile packer (pure C++, no CUDA).
//
// Given the registry layout (rank r_s and packed column offset off_s of every slot,
// slots in reference adapter order = std::map by job_id, fused_lora.hpp:48-53) and the
// owning slot of every token (TokenBatch::segment_map, fused_lora.hpp:28-31), build the
// tile tables of the six launches of one fused fwd+bwd:
//
//   packed rank space: slot s owns columns [off_s, off_s + r_s), off_{s+1} = off_s +
//   round_up(r_s, 8). Jobs of rank 8..128 therefore share 64-wide K blocks instead of
//   each padding to a full MMA tile.  For an M-tile of 128 tokens the K-extension of the
//   fused GEMM covers only [floor64(off_min), ceil64(off_max + r_max)) of the slots
//   present in that tile — for job-contiguous batches one or two jobs' ranks.
//
// Because H (and dH) are masked to each token's own columns, any K-range that is a
// superset of a tile's own columns gives the exact result; the plan only decides how
// much zero work is issued.  The plan is deterministic and bit-exactly checkable
// (tests/test_plan.py re-derives it from oracle/tlora_oracle.c).
#pragma once
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstdint>
#include <functional>
#include <queue>
#include <stdexcept>
#include <string>
#include <vector>

namespace tlora {

struct PlanTile {
  int32_t m0, n0, kb0, ke0, kb1, ke1, split, pad;
};

struct RegistryLayout {
  int64_t d = 0, k = 0;
  std::vector<int32_t> rank;    // per slot
  std::vector<int32_t> offset;  // per slot, packed rank column offset
  int32_t R = 0;                // packed rank columns (multiple of 8)

  static RegistryLayout make(int64_t d, int64_t k, const std::vector<int32_t>& ranks) {
    RegistryLayout L;
    L.d = d;
    L.k = k;
    L.rank = ranks;
    int32_t off = 0;
    for (int32_t r : ranks) {
      L.offset.push_back(off);
      off += (r + 7) / 8 * 8;
    }
    L.R = std::max<int32_t>(off, 8);
    return L;
  }
};

constexpr int kPlanBM = 128;      // MMA M tile (tokens or packed-rank rows), 1-CTA launches
constexpr int kPlanBMBase = 256;  // M tile of the fused base GEMMs (2-CTA pair)
constexpr int kPlanBK = 64;       // K block
constexpr int kPlanBNBase = 256;  // N tile of the fused base GEMMs (fwd, dX)
constexpr int kPlanBNLow = 128;   // N tile of the low-rank launches (shrink, dH, dA, dB)
constexpr int kPlanGradMaxN = 128;            // rank columns per gradient tile
#ifndef TLORA_GRAD_TARGET_TILES
#define TLORA_GRAD_TARGET_TILES 74  // dB + dA share a launch: ~one wave of tiles in total
#endif
constexpr int kPlanGradTargetTiles = TLORA_GRAD_TARGET_TILES;  // split-K target per problem
constexpr int kPlanMinSplitTokens = 512;

struct PlanTables {
  RegistryLayout layout;
  int64_t T = 0;
  std::vector<PlanTile> tiles[8];  // indexed by tlora_launch
  std::vector<int32_t> split_count_db, split_count_da;  // per packed rank row (R entries)
  int32_t splits_db = 1, splits_da = 1;
  int64_t useful_ext_cols = 0, packed_ext_cols = 0;
  int64_t tok_rank = 0;  // sum over tokens of the owning slot's rank (algorithmic work)
  std::vector<int32_t> slot_col_lo, slot_col_hi;  // per slot: [off, off + r)
  std::vector<int64_t> slot_first, slot_last;     // per slot token range, -1 if absent
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

constexpr int64_t kPlanL2Budget = 48ll << 20;  // bytes of operand panel kept hot in L2

// Experiment hook: TLORA_L2_BUDGET_MB overrides the panel budget (the plan oracle and the
// tests use the default; only set it to measure raster variants).
inline int64_t l2_budget() {
  static const int64_t b = [] {
    const char* e = std::getenv("TLORA_L2_BUDGET_MB");
    return e ? std::max<int64_t>(1, std::atoll(e)) << 20 : kPlanL2Budget;
  }();
  return b;
}

// L2-aware raster of an (n_mt x n_nt) output-tile grid for a GEMM with reduction depth K
// (bf16 operands). A persistent grid runs ~148 consecutive tiles at once; ordering tiles
// in panels (a group of M-tiles swept across all N-tiles, or a group of N-tiles swept
// across all M-tiles) keeps one operand panel (<= kPlanL2Budget) resident in L2 while the
// other streams. The orientation that streams fewer total bytes wins (ties: M panels).
// Returns (m, n) tile coordinates in launch order.
inline std::vector<std::pair<int32_t, int32_t>> raster_order(int64_t n_mt, int64_t n_nt,
                                                             int64_t K, int64_t bm, int64_t bn) {
  const int64_t a_panel = bm * K * 2, b_panel = bn * K * 2;  // bytes per M / N tile panel
  const int64_t gm = std::max<int64_t>(1, std::min(n_mt, l2_budget() / a_panel));
  const int64_t gn = std::max<int64_t>(1, std::min(n_nt, l2_budget() / b_panel));
  const int64_t bytes_m = n_mt * a_panel + ceil_div(n_mt, gm) * n_nt * b_panel;
  const int64_t bytes_n = n_nt * b_panel + ceil_div(n_nt, gn) * n_mt * a_panel;
  std::vector<std::pair<int32_t, int32_t>> order;
  order.reserve(n_mt * n_nt);
  if (bytes_m <= bytes_n) {
    for (int64_t g0 = 0; g0 < n_mt; g0 += gm)
      for (int64_t n = 0; n < n_nt; ++n)
        for (int64_t m = g0; m < std::min(n_mt, g0 + gm); ++m) order.push_back({(int32_t)m, (int32_t)n});
  } else {
    for (int64_t g0 = 0; g0 < n_nt; g0 += gn)
      for (int64_t m = 0; m < n_mt; ++m)
        for (int64_t n = g0; n < std::min(n_nt, g0 + gn); ++n) order.push_back({(int32_t)m, (int32_t)n});
  }
  return order;
}

// Gradient launches, per job in transposed form (lora_grad.cuh):
//   dB: M-dim = k, dA: M-dim = d; N = the job's own rank columns (<= 256 per tile);
//   K = the job's token range [first, last] (only its own tokens when job-contiguous).
// Long token ranges are split so that the largest tile is about total/kPlanGradTargetTiles
// of the work; each split except a range's last ends on a 64-token boundary (TMA boxes of
// split s never overlap split s+1). split_cnt has one entry per packed rank row. Tiles are
// ordered largest-work first (stable), so the static round-robin over CTAs is balanced.
inline void build_grad_tiles(const RegistryLayout& L, const PlanTables& P, int64_t Mdim,
                             std::vector<PlanTile>& out, std::vector<int32_t>& split_cnt,
                             int32_t& max_split) {
  const int64_t n_mt = ceil_div(Mdim, kPlanBM);
  auto round64 = [](int64_t x) { return ceil_div(x, 64) * 64; };
  split_cnt.assign(L.R, 0);
  max_split = 1;
  int64_t total = 0;
  for (size_t s = 0; s < L.rank.size(); ++s) {
    if (P.slot_first[s] < 0) continue;
    const int64_t len = P.slot_last[s] + 1 - P.slot_first[s];
    for (int64_t q = 0; q < L.rank[s]; q += kPlanGradMaxN)
      total += len * (kPlanBM + round64(std::min<int64_t>(kPlanGradMaxN, L.rank[s] - q))) * n_mt;
  }
  const int64_t w_star = std::max<int64_t>(1, total / kPlanGradTargetTiles);
  std::vector<std::pair<int64_t, PlanTile>> tiles;
  for (size_t s = 0; s < L.rank.size(); ++s) {
    for (int64_t q = 0; q < L.rank[s]; q += kPlanGradMaxN) {
      const int32_t c0 = L.offset[s] + (int32_t)q;
      const int32_t nc = (int32_t)std::min<int64_t>(kPlanGradMaxN, L.rank[s] - q);
      if (P.slot_first[s] < 0) {  // job absent from this batch: zero (beta-scaled) grads
        for (int64_t mt = 0; mt < n_mt; ++mt)
          tiles.push_back({0, {(int32_t)(mt * kPlanBM), c0, 0, 0, 0, 0, 0, nc}});
        for (int32_t r = c0; r < c0 + nc; ++r) split_cnt[r] = 1;
        continue;
      }
      const int64_t tlo = P.slot_first[s], thi = P.slot_last[s] + 1, len = thi - tlo;
      const int64_t per_tile = len * (kPlanBM + round64(nc));
      const int64_t c = std::max<int64_t>(
          1, std::min(ceil_div(per_tile, w_star), std::max<int64_t>(1, len / 256)));
      const int64_t chunk = ceil_div(ceil_div(len, c), kPlanBK) * kPlanBK;
      int32_t used = 0;
      for (int64_t sp = 0; sp < c; ++sp) {
        const int64_t kb = tlo + sp * chunk, ke = std::min(thi, kb + chunk);
        if (kb >= ke) break;
        for (int64_t mt = 0; mt < n_mt; ++mt)
          tiles.push_back({(ke - kb) * (kPlanBM + round64(nc)),
                           {(int32_t)(mt * kPlanBM), c0, (int32_t)kb, (int32_t)ke, 0, 0,
                            (int32_t)sp, nc}});
        ++used;
      }
      for (int32_t r = c0; r < c0 + nc; ++r) split_cnt[r] = used;
      max_split = std::max(max_split, used);
    }
  }
  std::stable_sort(tiles.begin(), tiles.end(),
                   [](const auto& x, const auto& y) { return x.first > y.first; });
  for (auto& t : tiles) out.push_back(t.second);
}

// Static longest-processing-time assignment of one combined gradient launch's tiles (the
// dB tiles, then the dA tiles: indices into that concatenation) to `ctas` persistent CTAs.
// Round-robin over the largest-first list leaves the busiest CTA ~1.2-1.45x the mean on
// the C2 projections (1024-4096-token tiles, 3-7 per CTA); greedy LPT (each tile, largest
// first, to the least-loaded CTA, ties to the lower index) brings it to ~1.0x. Cost model
// = bytes the tile moves: its operand rows (tokens x (128 + pad64) bf16) plus the fp32
// epilogue store (128 x pad). CSR out: CTA c runs idx[off[c] .. off[c+1]) in that order.
inline int64_t grad_tile_cost(const PlanTile& t) {
  const int64_t pad64 = ceil_div(t.pad, 64) * 64;
  return (int64_t)(t.ke0 - t.kb0) * 2 * (kPlanBM + pad64) + 4ll * kPlanBM * t.pad;
}

inline void grad_schedule(const std::vector<PlanTile>& first, const std::vector<PlanTile>& second,
                          int ctas, std::vector<int32_t>& off, std::vector<int32_t>& idx) {
  const int32_t n = (int32_t)(first.size() + second.size());
  std::vector<std::pair<int64_t, int32_t>> order(n);
  for (int32_t i = 0; i < n; ++i)
    order[i] = {grad_tile_cost(i < (int32_t)first.size() ? first[i] : second[i - first.size()]), i};
  std::stable_sort(order.begin(), order.end(),
                   [](const auto& x, const auto& y) { return x.first > y.first; });
  using Slot = std::pair<int64_t, int32_t>;  // (load, cta)
  std::priority_queue<Slot, std::vector<Slot>, std::greater<Slot>> heap;
  for (int32_t c = 0; c < ctas; ++c) heap.push({0, c});
  std::vector<std::vector<int32_t>> per(ctas);
  for (const auto& [cost, i] : order) {
    Slot s = heap.top();
    heap.pop();
    per[s.second].push_back(i);
    heap.push({s.first + cost, s.second});
  }
  off.assign(ctas + 1, 0);
  idx.clear();
  idx.reserve(n);
  for (int32_t c = 0; c < ctas; ++c) {
    idx.insert(idx.end(), per[c].begin(), per[c].end());
    off[c + 1] = (int32_t)idx.size();
  }
}

inline PlanTables build_plan(const RegistryLayout& L, int64_t T, const int32_t* token_slot) {
  PlanTables P;
  P.layout = L;
  P.T = T;
  const int S = (int)L.rank.size();
  for (int64_t t = 0; t < T; ++t)
    if (token_slot[t] < 0 || token_slot[t] >= S)
      throw std::out_of_range("token " + std::to_string(t) + " has slot " +
                              std::to_string(token_slot[t]) + " with no adapter");
  P.slot_col_lo.resize(S);
  P.slot_col_hi.resize(S);
  for (int s = 0; s < S; ++s) {
    P.slot_col_lo[s] = L.offset[s];
    P.slot_col_hi[s] = L.offset[s] + L.rank[s];
  }
  P.slot_first.assign(S, -1);
  P.slot_last.assign(S, -1);
  for (int64_t t = 0; t < T; ++t) {
    const int s = token_slot[t];
    P.tok_rank += L.rank[s];
    if (P.slot_first[s] < 0) P.slot_first[s] = t;
    P.slot_last[s] = t;
  }

  const int64_t n_mt = ceil_div(T, kPlanBM);
  std::vector<int32_t> c_lo(n_mt), c_hi(n_mt);
  for (int64_t m = 0; m < n_mt; ++m) {
    const int64_t t0 = m * kPlanBM, t1 = std::min(T, t0 + kPlanBM);
    int smin = S, smax = -1;
    std::vector<char> present(S, 0);
    for (int64_t t = t0; t < t1; ++t) {
      const int s = token_slot[t];
      smin = std::min(smin, s);
      smax = std::max(smax, s);
      present[s] = 1;
    }
    c_lo[m] = L.offset[smin] / kPlanBK * kPlanBK;
    c_hi[m] = (int32_t)(ceil_div(L.offset[smax] + L.rank[smax], kPlanBK) * kPlanBK);
  }
  // packing efficiency of the fused GEMM's K-extension, per 256-token tile
  for (int64_t m2 = 0; m2 < ceil_div(T, kPlanBMBase); ++m2) {
    std::vector<char> present(S, 0);
    int32_t lo = INT32_MAX, hi = 0;
    for (int64_t t = m2 * kPlanBMBase; t < std::min(T, (m2 + 1) * kPlanBMBase); ++t) {
      const int s = token_slot[t];
      present[s] = 1;
      lo = std::min(lo, L.offset[s] / kPlanBK * kPlanBK);
      hi = std::max(hi, (int32_t)(ceil_div(L.offset[s] + L.rank[s], kPlanBK) * kPlanBK));
    }
    for (int s = 0; s < S; ++s)
      if (present[s]) P.useful_ext_cols += L.rank[s];
    P.packed_ext_cols += hi - lo;
  }

  // shrink / dH: per M-tile, N-tiles over that tile's packed rank window
  for (int which = 0; which < 2; ++which) {
    const int64_t K = which == 0 ? L.d : L.k;
    auto& v = P.tiles[which == 0 ? 0 : 2];
    for (int64_t m = 0; m < n_mt; ++m)
      for (int32_t n0 = c_lo[m]; n0 < c_hi[m]; n0 += kPlanBNLow)
        v.push_back({(int32_t)(m * kPlanBM), n0, 0, (int32_t)K, 0, 0, 0, 0});
  }
  // fused base GEMMs on 256-token tiles (CTA pairs): fwd (N = k, K = d) and dX (N = d,
  // K = k); the K-extension window of a 256-tile is the union of its two 128-halves'.
  const int64_t n_mt2 = ceil_div(T, kPlanBMBase);
  std::vector<int32_t> w_lo(n_mt2), w_hi(n_mt2);
  for (int64_t m = 0; m < n_mt2; ++m) {
    w_lo[m] = c_lo[2 * m];
    w_hi[m] = c_hi[2 * m];
    if (2 * m + 1 < n_mt) {
      w_lo[m] = std::min(w_lo[m], c_lo[2 * m + 1]);
      w_hi[m] = std::max(w_hi[m], c_hi[2 * m + 1]);
    }
  }
  // shrink / dH on 256-token CTA-pair tiles (secondary tiles of a fused GEMM launch):
  // N-chunks of <= 256 over the pair's window, each rounded up to 128 columns (the extra
  // columns belong to other jobs and are written as masked zeros)
  for (int which = 0; which < 2; ++which) {
    const int64_t K = which == 0 ? L.d : L.k;
    auto& v = P.tiles[which == 0 ? 6 : 7];
    for (int64_t m = 0; m < n_mt2; ++m)
      for (int32_t n0 = w_lo[m]; n0 < w_hi[m]; n0 += 256) {
        const int32_t n = std::min<int32_t>(256, (int32_t)(ceil_div(w_hi[m] - n0, 128) * 128));
        v.push_back({(int32_t)(m * kPlanBMBase), n0, 0, (int32_t)K, 0, 0, 0, n});
      }
  }
  for (int which = 0; which < 2; ++which) {
    const int64_t N = which == 0 ? L.k : L.d;
    const int64_t K = which == 0 ? L.d : L.k;
    auto& v = P.tiles[which == 0 ? 1 : 3];
    for (auto [m, n] : raster_order(n_mt2, ceil_div(N, kPlanBNBase), K, kPlanBMBase, kPlanBNBase))
      v.push_back({m * kPlanBMBase, n * kPlanBNBase, 0, (int32_t)K, w_lo[m], w_hi[m], 0, 0});
  }
  build_grad_tiles(L, P, L.k, P.tiles[4], P.split_count_db, P.splits_db);
  build_grad_tiles(L, P, L.d, P.tiles[5], P.split_count_da, P.splits_da);
  return P;
}

}  // namespace tlora
