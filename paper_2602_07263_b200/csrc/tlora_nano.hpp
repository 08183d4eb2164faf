// tlora_nano.hpp — rank-aware nano-batch map (host side, pure C++).
//
// The reference plans a group iteration as partition(combined_batch, N): N balanced sample
// COUNTS (nano_pipeline.hpp:51-60) and nothing about which job's samples land in which
// nano-batch. The executor needs the map. Job-order slicing (round 1) leaves the LoRA work
// of the nano-batches unbalanced (a rank-128 job costs 16x a rank-8 job per token), so the
// map here balances work: every sample carries its job's weight (the caller's per-sample
// cost: seq_len x (base + rank-dependent LoRA work), integers so the map is bit-exact), the
// counts stay exactly partition()'s, and samples are placed heaviest first, each on the
// least-loaded nano-batch with room left (ties: lower nano), then pairwise swaps between
// the heaviest nano-batch and the others while they lower its load. That fixes how many samples
// of each job every nano-batch gets; a job's samples then go to the nano-batches in nano
// order, so each (nano, job) pair is one contiguous range of the job's samples.
// Restated independently in oracle/tlora_oracle.c (orc_nano_assign).
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <set>
#include <stdexcept>
#include <utility>
#include <vector>

namespace tlora {

struct NanoMap {
  int32_t n = 0;                      // nano-batches actually used (= min(N, total))
  std::vector<int32_t> per_nano;      // samples per nano-batch (partition's counts)
  std::vector<int32_t> sample_nano;   // nano of each sample, samples enumerated job-major
  std::vector<int32_t> nano_slot;     // [n x S] samples of slot s in nano i
};

inline NanoMap nano_assign(const std::vector<int32_t>& batch, const std::vector<int64_t>& weight,
                           int32_t n_req) {
  const int32_t S = (int32_t)batch.size();
  if (S < 1 || (int32_t)weight.size() != S)
    throw std::invalid_argument("nano_assign: need one batch size and weight per slot");
  int64_t total = 0;
  for (int32_t s = 0; s < S; ++s) {
    if (batch[s] < 0 || weight[s] < 0)
      throw std::invalid_argument("nano_assign: negative batch size or weight");
    total += batch[s];
  }
  // nano_pipeline.hpp:51-60 (same errors)
  if (total < 1) throw std::invalid_argument("partition: group_batch must be >= 1");
  if (total > INT32_MAX) throw std::invalid_argument("nano_assign: too many samples");
  if (n_req < 1) throw std::invalid_argument("partition: N must be >= 1");
  NanoMap m;
  m.n = (int32_t)std::min<int64_t>(n_req, total);
  const int32_t base = (int32_t)(total / m.n), extra = (int32_t)(total % m.n);
  for (int32_t i = 0; i < m.n; ++i) m.per_nano.push_back(base + (i < extra ? 1 : 0));
  m.sample_nano.assign((size_t)total, 0);
  m.nano_slot.assign((size_t)m.n * S, 0);

  std::vector<int64_t> first(S, 0);
  for (int32_t s = 1; s < S; ++s) first[s] = first[s - 1] + batch[s - 1];
  std::vector<int32_t> order(S);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int32_t a, int32_t b) { return weight[a] > weight[b]; });
  std::vector<int32_t> room = m.per_nano;
  std::set<std::pair<int64_t, int32_t>> open;  // (load, nano) of nanos with room left
  for (int32_t i = 0; i < m.n; ++i) open.insert({0, i});
  for (int32_t s : order) {
    for (int32_t q = 0; q < batch[s]; ++q) {
      auto it = open.begin();  // least load, then lowest index
      const auto [load, i] = *it;
      open.erase(it);
      ++m.nano_slot[(size_t)i * S + s];
      if (--room[i] > 0) open.insert({load + weight[s], i});
    }
  }
  // Refinement (LPT under fixed counts can overshoot): while some swap of one sample of job
  // a in the heaviest nano-batch h (lowest index on ties) with one sample of a lighter job b
  // in another nano-batch o lowers h's load without making o the new maximum, apply the
  // first such swap in (o, a, b) ascending order. h's load strictly drops each time, so the
  // sorted load vector decreases and the loop ends.
  std::vector<int64_t> load(m.n, 0);
  for (int32_t i = 0; i < m.n; ++i)
    for (int32_t s = 0; s < S; ++s) load[i] += (int64_t)m.nano_slot[(size_t)i * S + s] * weight[s];
  for (bool swapped = true; swapped;) {
    swapped = false;
    const int32_t h = (int32_t)(std::max_element(load.begin(), load.end()) - load.begin());
    for (int32_t o = 0; o < m.n && !swapped; ++o) {
      if (o == h) continue;
      for (int32_t a = 0; a < S && !swapped; ++a) {
        if (m.nano_slot[(size_t)h * S + a] == 0) continue;
        for (int32_t b = 0; b < S; ++b) {
          if (m.nano_slot[(size_t)o * S + b] == 0 || weight[a] <= weight[b]) continue;
          const int64_t delta = weight[a] - weight[b];
          if (load[o] + delta >= load[h]) continue;
          --m.nano_slot[(size_t)h * S + a];
          ++m.nano_slot[(size_t)h * S + b];
          --m.nano_slot[(size_t)o * S + b];
          ++m.nano_slot[(size_t)o * S + a];
          load[h] -= delta;
          load[o] += delta;
          swapped = true;
          break;
        }
      }
    }
  }
  // which samples: job s's first nano_slot[0][s] samples go to nano 0, the next ones to
  // nano 1, ... — every (nano, job) pair is one contiguous range of the job's samples
  for (int32_t s = 0; s < S; ++s) {
    size_t q = (size_t)first[s];
    for (int32_t i = 0; i < m.n; ++i)
      for (int32_t c = 0; c < m.nano_slot[(size_t)i * S + s]; ++c) m.sample_nano[q++] = i;
  }
  return m;
}

// Ramped variant for a pipeline whose boundary traffic is exposed only at its ends (the
// tensor-parallel step: nano 0's all-gather before any compute, the last nano's reduce-
// scatter after it): nano-batch i gets a share of the samples proportional to
// min(g^i, g^(n-1-i)), so the first and last nano-batches are small and each one's traffic
// still hides behind its neighbour's compute while g <= compute / traffic. Samples are
// placed heaviest first on the nano-batch with the least load per unit of its share (ties:
// lower nano); (nano, job) ranges stay contiguous as in nano_assign. g <= 1 or n < 3 is
// nano_assign itself.
inline NanoMap nano_assign_ramp(const std::vector<int32_t>& batch,
                                const std::vector<int64_t>& weight, int32_t n_req, double g) {
  NanoMap m = nano_assign(batch, weight, n_req);  // validation, n, uniform fallback
  if (g <= 1.0 || m.n < 3) return m;
  const int32_t S = (int32_t)batch.size();
  int64_t total = 0;
  for (int32_t b : batch) total += b;
  // shares -> integer counts (largest remainder), every nano-batch >= 1 sample
  std::vector<double> share(m.n);
  double ssum = 0.0;
  for (int32_t i = 0; i < m.n; ++i) {
    share[i] = std::pow(g, (double)std::min(i, m.n - 1 - i));
    ssum += share[i];
  }
  std::vector<int32_t> cnt(m.n, 1);
  int64_t left = total - m.n;
  std::vector<std::pair<double, int32_t>> rem;
  for (int32_t i = 0; i < m.n; ++i) {
    const double want = share[i] / ssum * (double)total - 1.0;
    const int32_t f = want > 0.0 ? (int32_t)std::floor(want) : 0;
    cnt[i] += f;
    left -= f;
    rem.push_back({-(want - f), i});
  }
  std::sort(rem.begin(), rem.end());
  for (size_t r = 0; left > 0 && r < rem.size(); ++r, --left) ++cnt[rem[r].second];
  for (int32_t i = 0; left > 0; i = (i + 1) % m.n, --left) ++cnt[i];
  m.per_nano = cnt;
  std::fill(m.nano_slot.begin(), m.nano_slot.end(), 0);
  std::vector<int32_t> order(S);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int32_t a, int32_t b) { return weight[a] > weight[b]; });
  std::vector<int32_t> room = cnt;
  std::vector<int64_t> load(m.n, 0);
  for (int32_t s : order)
    for (int32_t q = 0; q < batch[s]; ++q) {
      int32_t best = -1;
      for (int32_t i = 0; i < m.n; ++i) {
        if (room[i] == 0) continue;
        // least load per share: load_i / cnt_i < load_b / cnt_b, in integers
        if (best < 0 || (__int128)load[i] * cnt[best] < (__int128)load[best] * cnt[i]) best = i;
      }
      ++m.nano_slot[(size_t)best * S + s];
      --room[best];
      load[best] += weight[s];
    }
  std::vector<int64_t> first(S, 0);
  for (int32_t s = 1; s < S; ++s) first[s] = first[s - 1] + batch[s - 1];
  for (int32_t s = 0; s < S; ++s) {
    size_t q = (size_t)first[s];
    for (int32_t i = 0; i < m.n; ++i)
      for (int32_t c = 0; c < m.nano_slot[(size_t)i * S + s]; ++c) m.sample_nano[q++] = i;
  }
  return m;
}

}  // namespace tlora
