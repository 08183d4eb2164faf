// tlora_step.cu — the SSM layer-set training step executor (C++ host; C-ABI tlora_step_*).
//
// This is the caller of the hot path, executed for real: the reference's iteration loop
// (proj/include/lora_fleet/sim_engine.hpp:306-315)
//
//     n_use = fixed_n ? *fixed_n : aimd.n
//     sched = partition(combined_batch, n_use)          nano_pipeline.hpp:51-60
//     trace = simulate_iteration(plan, sched, hw)        (modelled)
//     aimd  = aimd_step(aimd, trace.t_iter_event)        nano_pipeline.hpp:99-112
//     aimd.n = min(aimd.n, combined_batch)
//
// with the model replaced by the device: every step builds (or reuses) the rank-aware
// nano-batch map of n_use (tlora_nano.hpp: partition's counts, LoRA work balanced across
// nano-batches), runs forward + backward of every (layer, projection) for each nano-batch
// (gradients accumulate across nano-batches), applies the fused multi-job AdamW once, times
// the step with CUDA events on the caller's stream and feeds that time to aimd_step.
//
// One step is a fixed op schedule (build_schedule below, readable from the host with
// tlora_step_schedule_host):
//   main stream   the fused base+LoRA GEMMs, chained: every forward launch carries the
//                 next forward's shrink as extra tiles, the last forward launch of a
//                 nano-batch carries its backward's first dH, every dX launch carries the
//                 next dH, and the last dX of a nano-batch carries the next nano-batch's
//                 first shrink — 2 x keys x nano-batches launches, no standalone low-rank
//                 launch after the first shrink of the step;
//   side stream   per (key, nano) the combined dB+dA launch (accumulating over nano-
//                 batches), then, after the last nano-batch, the key's AdamW;
//   comm stream   (data-parallel replicas) the key's gradient all-reduce as soon as its
//                 last nano-batch's gradients exist, then its AdamW (grads / replicas); or,
//                 with the sharded optimizer, reduce-scatter -> AdamW of this rank's row
//                 shard -> all-gather of the refreshed bf16 operands.
// The backward's dH values live in a ring of buffers; a dX launch that overwrites a ring
// slot waits for the side-stream reader of that slot.
// Buffers are row-major bf16, one step-sized buffer per tensor; nano-batch i is the row
// range [t0_i, t0_i + T_i) of each (nano-major token layout, job-contiguous inside a
// nano-batch: tlora_step_layout). The step is enqueue-only; at a single replica it is
// captured into one CUDA graph per (nano count, input set) after its first eager run.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tlora.h"
#include "tlora_nano.hpp"

namespace tlora {
void set_last_error(const std::string& msg);  // tlora_capi.cu
}

namespace {

struct StepError : std::runtime_error {
  int code;
  StepError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void chk(int rc) {
  if (rc != TLORA_OK) throw StepError(rc, tlora_last_error());
}

#define ST_CUDA(x)                                                                          \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess)                                                                  \
      throw StepError(TLORA_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));     \
  } while (0)

void need(bool ok, int code, const std::string& msg) {
  if (!ok) throw StepError(code, msg);
}

template <class F>
int step_guard(F&& f) {
  try {
    f();
    return TLORA_OK;
  } catch (const StepError& e) {
    tlora::set_last_error(e.what());
    return e.code;
  } catch (const std::invalid_argument& e) {
    tlora::set_last_error(e.what());
    return TLORA_ERR_PLAN;
  } catch (const std::exception& e) {
    tlora::set_last_error(e.what());
    return TLORA_ERR_ARG;
  }
}

// ------------------------------------------------------------------ op schedule
struct Op {
  int32_t kind, stream, key, nano;
  int32_t slot;                            // dH ring slot read (DX, GRADS)
  int32_t sec_kind, sec_key, sec_nano;     // secondary tiles of a FWD / DX launch
  int32_t sec_slot;                        // ring slot a secondary dH writes
  int32_t beta;                            // GRADS: 1 = accumulate (nano > 0)
  int32_t wait0, wait1;                    // op indices waited on (other streams), -1
};

// early: a GRADS op waits only for the launch that produced its dH (it may then overlap the
// key's own dX launch) instead of for the key's dX launch.
// dp: 0 one replica, 1 all-reduce + full AdamW, 2 sharded optimizer (reduce-scatter,
// AdamW on this rank's rows, all-gather of the refreshed bf16 operands)
std::vector<Op> build_schedule(int32_t keys, int32_t n, int32_t ring, bool side, int dp,
                               bool early = false) {
  need(keys >= 1 && n >= 1 && ring >= 2, TLORA_ERR_ARG, "schedule: bad sizes");
  std::vector<Op> ops;
  std::vector<int32_t> grads_op;  // global backward index -> GRADS op index
  auto push = [&](Op o) {
    ops.push_back(o);
    return (int32_t)ops.size() - 1;
  };
  const int32_t gstream = side ? TLORA_STREAM_SIDE : TLORA_STREAM_MAIN;
  auto ring_wait = [&](int32_t g) {  // the GRADS op that last read ring slot g % ring
    const int32_t prev = g - ring;
    return prev >= 0 ? grads_op[prev] : -1;
  };
  int32_t g = 0, dh_producer = -1;
  for (int32_t i = 0; i < n; ++i) {
    if (i == 0)
      push({TLORA_OP_SHRINK, TLORA_STREAM_MAIN, 0, 0, -1, -1, -1, -1, -1, 0, -1, -1});
    for (int32_t key = 0; key < keys; ++key) {
      Op o{TLORA_OP_FWD, TLORA_STREAM_MAIN, key, i, -1, -1, -1, -1, -1, 0, -1, -1};
      if (key + 1 < keys) {
        o.sec_kind = TLORA_OP_SHRINK;
        o.sec_key = key + 1;
        o.sec_nano = i;
      } else {  // prefetch the backward's first dH (the last key, this nano-batch)
        o.sec_kind = TLORA_OP_DH;
        o.sec_key = keys - 1;
        o.sec_nano = i;
        o.sec_slot = g % ring;
        o.wait0 = ring_wait(g);
      }
      dh_producer = push(o);
    }
    for (int32_t j = 0; j < keys; ++j) {
      const int32_t key = keys - 1 - j, gi = g + j;
      Op o{TLORA_OP_DX, TLORA_STREAM_MAIN, key, i, gi % ring, -1, -1, -1, -1, 0, -1, -1};
      if (j + 1 < keys) {
        o.sec_kind = TLORA_OP_DH;
        o.sec_key = key - 1;
        o.sec_nano = i;
        o.sec_slot = (gi + 1) % ring;
        o.wait0 = ring_wait(gi + 1);
      } else if (i + 1 < n) {
        o.sec_kind = TLORA_OP_SHRINK;
        o.sec_key = 0;
        o.sec_nano = i + 1;
      }
      const int32_t dx = push(o);
      const int32_t after = early ? dh_producer : dx;
      dh_producer = dx;
      const int32_t gr = push({TLORA_OP_GRADS, gstream, key, i, gi % ring, -1, -1, -1, -1,
                               i > 0 ? 1 : 0, gstream == TLORA_STREAM_MAIN ? -1 : after, -1});
      grads_op.push_back(gr);
      if (i + 1 == n) {
        if (dp == 2) {
          push({TLORA_OP_REDUCE_SCATTER, TLORA_STREAM_COMM, key, i, -1, -1, -1, -1, -1, 0, gr, -1});
          push({TLORA_OP_ADAMW, TLORA_STREAM_COMM, key, i, -1, -1, -1, -1, -1, 0, -1, -1});
          push({TLORA_OP_ALLGATHER, TLORA_STREAM_COMM, key, i, -1, -1, -1, -1, -1, 0, -1, -1});
        } else if (dp) {
          push({TLORA_OP_ALLREDUCE, TLORA_STREAM_COMM, key, i, -1, -1, -1, -1, -1, 0, gr, -1});
          push({TLORA_OP_ADAMW, TLORA_STREAM_COMM, key, i, -1, -1, -1, -1, -1, 0, -1, -1});
        } else {
          push({TLORA_OP_ADAMW, gstream, key, i, -1, -1, -1, -1, -1, 0, -1, -1});
        }
      }
    }
    g += keys;
  }
  return ops;
}

// ------------------------------------------------------------------ layout of one N
struct Layout {
  tlora::NanoMap map;
  std::vector<int64_t> t0;                  // n + 1 row offsets
  std::vector<int64_t> sample_row;          // first row of each sample (job-major)
  std::vector<std::vector<tlora_plan*>> plans;  // [nano][projection]
  std::vector<Op> ops;
  std::vector<char> needs_event;
  cudaGraphExec_t graph[2] = {nullptr, nullptr};
  long long launches = 0;  // kernels of one step of this layout (counted on its eager run)
};

}  // namespace

struct tlora_step {
  int device = 0;
  tlora_step_desc desc{};
  std::vector<int64_t> d, k;
  std::vector<int32_t> input, ranks, batch, seq;
  std::vector<int64_t> weight;  // per-sample work of each slot (nano map balance)
  int32_t L = 1, P = 1, S = 1, groups = 1, ring = 8, sets = 1;
  int64_t T = 0;
  int32_t R = 0, total_samples = 0;
  tlora_comm* comm = nullptr;
  int32_t dp = 1;
  std::vector<tlora_layer*> layers;  // [L * P], key = layer * P + proj
  // device buffers (owned)
  std::vector<void*> owned;
  std::vector<void*> X[2], dY[2];  // per input group / per projection, per input set
  std::vector<void*> Y, dX;        // per projection
  void* H = nullptr;               // [keys][T][R]
  void* dH = nullptr;              // [ring][T][R]
  int32_t* present = nullptr;      // per slot: batch > 0
  // exec: the step's own main stream (a captured graph needs a capturable stream; the
  // caller's may be the legacy default stream); it joins the caller's stream both ways
  cudaStream_t exec = nullptr, side = nullptr, comm_s = nullptr;
  cudaEvent_t ev_side = nullptr, ev_comm = nullptr, ev_in = nullptr;
  // step timing events, a ring of 4 (begin, end) pairs: with a fixed N nothing needs the
  // host to wait for a step, so run() returns right after enqueueing and reports the time
  // of the latest step that has completed
  static constexpr int kTimeRing = 4;
  cudaEvent_t t_begin_r[kTimeRing] = {}, t_end_r[kTimeRing] = {};
  long long t_step_r[kTimeRing] = {-1, -1, -1, -1};
  std::vector<cudaEvent_t> events;  // per op of the largest schedule
  std::map<int32_t, std::unique_ptr<Layout>> layouts;
  int32_t zeroed_for = -1;          // nano count the H / dH arenas were last zeroed for
  // AIMD controller (nano_pipeline.hpp:36-47; sim_engine.hpp config.aimd_*)
  int32_t aimd_n = 4, has_prev = 0;
  double t_prev = 0.0;
  std::vector<std::pair<int32_t, double>> trajectory;
  long long steps_run = 0;

  ~tlora_step();
  void* alloc(size_t bytes) {
    void* p = nullptr;
    if (bytes) {
      ST_CUDA(cudaMalloc(&p, bytes));
      owned.push_back(p);
    }
    return p;
  }
  int32_t key(int32_t layer, int32_t proj) const { return layer * P + proj; }
  tlora_layer* lay(int32_t key) const { return layers[(size_t)key]; }
  int32_t proj_of(int32_t key) const { return key % P; }
  char* x_ptr(int set, int32_t proj, int64_t row) const {
    return (char*)X[set][(size_t)input[(size_t)proj]] + row * d[(size_t)proj] * 2;
  }
  char* dy_ptr(int set, int32_t proj, int64_t row) const {
    return (char*)dY[set][(size_t)proj] + row * k[(size_t)proj] * 2;
  }
  char* h_ptr(int32_t key, int64_t row) const {
    return (char*)H + ((size_t)key * T + row) * R * 2;
  }
  char* dh_ptr(int32_t slot, int64_t row) const {
    return (char*)dH + ((size_t)slot * T + row) * R * 2;
  }
  Layout& layout(int32_t n);
  void enqueue(Layout& lo, int set, cudaStream_t main, bool trace = false);
  // trace of the last TLORA_RUN_TRACE step: per op its stream and end time (ms after the
  // step's start event)
  std::vector<cudaEvent_t> trace_ev;
  std::vector<Op> trace_ops;
  std::vector<double> trace_ms;
};

tlora_step::~tlora_step() {
  for (auto& [n, lo] : layouts) {
    for (auto& g : lo->graph)
      if (g) cudaGraphExecDestroy(g);
    for (auto& pl : lo->plans)
      for (auto* p : pl) tlora_plan_destroy(p);
  }
  for (auto* l : layers) tlora_layer_destroy(l);
  for (auto e : events) cudaEventDestroy(e);
  for (auto e : trace_ev) cudaEventDestroy(e);
  for (auto e : {ev_side, ev_comm, ev_in})
    if (e) cudaEventDestroy(e);
  for (int i = 0; i < kTimeRing; ++i)
    for (auto e : {t_begin_r[i], t_end_r[i]})
      if (e) cudaEventDestroy(e);
  if (exec) cudaStreamDestroy(exec);
  if (side) cudaStreamDestroy(side);
  if (comm_s) cudaStreamDestroy(comm_s);
  for (void* p : owned) cudaFree(p);
}

namespace {

// Token layout of a nano count: nano-major; inside nano-batch i the jobs in slot order,
// each job's samples assigned to i contiguous (tlora_nano.hpp).
void fill_layout(const tlora_step& st, Layout& lo) {
  const auto& m = lo.map;
  const int32_t S = st.S;
  lo.t0.assign((size_t)m.n + 1, 0);
  for (int32_t i = 0; i < m.n; ++i) {
    int64_t rows = 0;
    for (int32_t s = 0; s < S; ++s) rows += (int64_t)m.nano_slot[(size_t)i * S + s] * st.seq[(size_t)s];
    lo.t0[(size_t)i + 1] = lo.t0[(size_t)i] + rows;
  }
  lo.sample_row.assign((size_t)st.total_samples, 0);
  std::vector<int64_t> first(S, 0);
  for (int32_t s = 1; s < S; ++s) first[(size_t)s] = first[(size_t)s - 1] + st.batch[(size_t)s - 1];
  for (int32_t i = 0; i < m.n; ++i) {
    int64_t row = lo.t0[(size_t)i];
    for (int32_t s = 0; s < S; ++s) {
      // the (nano, job) sample range: samples of s before nano i go to earlier nanos
      int64_t q = first[(size_t)s];
      for (int32_t j = 0; j < i; ++j) q += m.nano_slot[(size_t)j * S + s];
      for (int32_t c = 0; c < m.nano_slot[(size_t)i * S + s]; ++c) {
        lo.sample_row[(size_t)(q + c)] = row;
        row += st.seq[(size_t)s];
      }
    }
  }
}

}  // namespace

Layout& tlora_step::layout(int32_t n) {
  auto it = layouts.find(n);
  if (it != layouts.end()) return *it->second;
  auto lo = std::make_unique<Layout>();
  lo->map = tlora::nano_assign(batch, weight, n);
  fill_layout(*this, *lo);
  const auto& m = lo->map;
  lo->plans.assign((size_t)m.n, std::vector<tlora_plan*>((size_t)P, nullptr));
  for (int32_t i = 0; i < m.n; ++i) {
    std::vector<int32_t> slots;
    for (int32_t s = 0; s < S; ++s)
      slots.insert(slots.end(), (size_t)m.nano_slot[(size_t)i * S + s] * seq[(size_t)s], s);
    for (int32_t p = 0; p < P; ++p)
      chk(tlora_plan_create(lay(key(0, p)), (int64_t)slots.size(), slots.data(),
                            &lo->plans[(size_t)i][(size_t)p]));
  }
  lo->ops = build_schedule(L * P, m.n, ring, (desc.flags & TLORA_STEP_SIDE_GRADS) != 0,
                           comm == nullptr ? 0 : (desc.flags & TLORA_STEP_SHARDED_OPT) ? 2 : 1,
                           (desc.flags & TLORA_STEP_EARLY_GRADS) != 0);
  lo->needs_event.assign(lo->ops.size(), 0);
  for (const auto& o : lo->ops)
    for (int32_t w : {o.wait0, o.wait1})
      if (w >= 0) lo->needs_event[(size_t)w] = 1;
  while (events.size() < lo->ops.size()) {
    cudaEvent_t e;
    ST_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    events.push_back(e);
  }
  auto& ref = *lo;
  layouts.emplace(n, std::move(lo));
  return ref;
}

void tlora_step::enqueue(Layout& lo, int set, cudaStream_t main, bool trace) {
  if (trace)
    while (trace_ev.size() < lo.ops.size()) {
      cudaEvent_t e;
      ST_CUDA(cudaEventCreate(&e));
      trace_ev.push_back(e);
    }
  const cudaStream_t streams[3] = {main, side ? side : main, comm_s ? comm_s : main};
  const int y_dt = desc.y_dtype;
  const float gscale = 1.0f / (float)dp;
  for (size_t idx = 0; idx < lo.ops.size(); ++idx) {
    const Op& o = lo.ops[idx];
    cudaStream_t s = streams[o.stream];
    for (int32_t w : {o.wait0, o.wait1})
      if (w >= 0 && lo.ops[(size_t)w].stream != o.stream)
        ST_CUDA(cudaStreamWaitEvent(s, events[(size_t)w], 0));
    const int32_t p = proj_of(o.key);
    tlora_layer* l = lay(o.key);
    const int64_t r0 = o.nano >= 0 ? lo.t0[(size_t)o.nano] : 0;
    tlora_plan* pl = o.nano >= 0 ? lo.plans[(size_t)o.nano][(size_t)p] : nullptr;
    void* sv = reinterpret_cast<void*>(s);
    switch (o.kind) {
      case TLORA_OP_SHRINK:
        chk(tlora_forward_shrink(l, pl, x_ptr(set, p, r0), h_ptr(o.key, r0), sv));
        break;
      case TLORA_OP_FWD:
      case TLORA_OP_DX: {
        const bool fwd = o.kind == TLORA_OP_FWD;
        char* out = fwd ? (char*)Y[(size_t)p] + r0 * k[(size_t)p] * 2
                        : (char*)dX[(size_t)p] + r0 * d[(size_t)p] * 2;
        if (o.sec_kind < 0) {
          if (fwd)
            chk(tlora_forward_gemm(l, pl, x_ptr(set, p, r0), h_ptr(o.key, r0), out, y_dt, sv));
          else
            chk(tlora_backward_dx(l, pl, dy_ptr(set, p, r0), dh_ptr(o.slot, r0), out, 0.f, sv));
          break;
        }
        const int32_t q = proj_of(o.sec_key);
        const int64_t s0 = lo.t0[(size_t)o.sec_nano];
        tlora_plan* npl = lo.plans[(size_t)o.sec_nano][(size_t)q];
        tlora_layer* nl = lay(o.sec_key);
        if (o.sec_kind == TLORA_OP_SHRINK) {
          if (fwd)
            chk(tlora_forward_gemm_shrink(l, pl, x_ptr(set, p, r0), h_ptr(o.key, r0), out, y_dt,
                                          nl, npl, x_ptr(set, q, s0), h_ptr(o.sec_key, s0), 0, sv));
          else
            chk(tlora_backward_dx_shrink(l, pl, dy_ptr(set, p, r0), dh_ptr(o.slot, r0), out, 0.f,
                                         nl, npl, x_ptr(set, q, s0), h_ptr(o.sec_key, s0), 0, sv));
        } else {
          if (fwd)
            chk(tlora_forward_gemm_dh(l, pl, x_ptr(set, p, r0), h_ptr(o.key, r0), out, y_dt, nl,
                                      npl, dy_ptr(set, q, s0), dh_ptr(o.sec_slot, s0), 0, sv));
          else
            chk(tlora_backward_dx_dh(l, pl, dy_ptr(set, p, r0), dh_ptr(o.slot, r0), out, 0.f, nl,
                                     npl, dy_ptr(set, q, s0), dh_ptr(o.sec_slot, s0), 0, sv));
        }
        break;
      }
      case TLORA_OP_DH:
        chk(tlora_backward_dh(l, pl, dy_ptr(set, p, r0), dh_ptr(o.slot, r0), sv));
        break;
      case TLORA_OP_GRADS:
        chk(tlora_backward_grads(l, pl, h_ptr(o.key, r0), dy_ptr(set, p, r0), x_ptr(set, p, r0),
                                 dh_ptr(o.slot, r0), o.beta ? 1.f : 0.f, sv));
        break;
      case TLORA_OP_ALLREDUCE:
        chk(tlora_layer_allreduce_grads(l, comm, TLORA_GROUP_DP, 0, sv));
        break;
      case TLORA_OP_REDUCE_SCATTER:
        chk(tlora_layer_reduce_scatter_grads(l, comm, TLORA_GROUP_DP, sv));
        break;
      case TLORA_OP_ALLGATHER:
        chk(tlora_layer_allgather_operands(l, comm, TLORA_GROUP_DP, sv));
        break;
      case TLORA_OP_ADAMW:
        if (comm && (desc.flags & TLORA_STEP_SHARDED_OPT)) {
          int64_t lo = 0, hi = 0;
          chk(tlora_layer_dp_shard(l, comm, TLORA_GROUP_DP, &lo, &hi));
          chk(tlora_layer_optimizer_step_rows(l, present, gscale, lo, hi, sv));
        } else {
          chk(tlora_layer_optimizer_step_masked(l, present, gscale, sv));
        }
        break;
      default:
        throw StepError(TLORA_ERR_ARG, "unknown op kind");
    }
    if (lo.needs_event[idx]) ST_CUDA(cudaEventRecord(events[idx], s));
    if (trace) ST_CUDA(cudaEventRecord(trace_ev[idx], s));
  }
  // join: the step ends on the main stream after the side / comm work
  if (side) {
    ST_CUDA(cudaEventRecord(ev_side, side));
    ST_CUDA(cudaStreamWaitEvent(main, ev_side, 0));
  }
  if (comm_s) {
    ST_CUDA(cudaEventRecord(ev_comm, comm_s));
    ST_CUDA(cudaStreamWaitEvent(main, ev_comm, 0));
  }
}

extern "C" {

int tlora_step_schedule_host(int32_t keys, int32_t nano, int32_t ring, int32_t side_grads,
                             int32_t data_parallel, tlora_step_op* out, int32_t cap,
                             int32_t* count) {
  return step_guard([&] {
    const auto ops = build_schedule(keys, nano, ring, side_grads != 0, data_parallel,
                                    side_grads == 2);
    if (count) *count = (int32_t)ops.size();
    if (out)
      for (size_t i = 0; i < ops.size() && (int32_t)i < cap; ++i) {
        const Op& o = ops[i];
        out[i] = {o.kind, o.stream, o.key, o.nano, o.slot, o.sec_kind, o.sec_key, o.sec_nano,
                  o.sec_slot, o.beta, o.wait0, o.wait1};
      }
  });
}

int tlora_nano_assign(int32_t num_slots, const int32_t* batch, const int64_t* weight, int32_t n,
                      int32_t* n_out, int32_t* per_nano, int32_t* sample_nano,
                      int32_t* nano_slot) {
  return step_guard([&] {
    need(num_slots >= 1 && batch && weight, TLORA_ERR_ARG, "null argument");
    const auto m = tlora::nano_assign(std::vector<int32_t>(batch, batch + num_slots),
                                      std::vector<int64_t>(weight, weight + num_slots), n);
    if (n_out) *n_out = m.n;
    if (per_nano) std::memcpy(per_nano, m.per_nano.data(), m.per_nano.size() * 4);
    if (sample_nano) std::memcpy(sample_nano, m.sample_nano.data(), m.sample_nano.size() * 4);
    if (nano_slot) std::memcpy(nano_slot, m.nano_slot.data(), m.nano_slot.size() * 4);
  });
}

int tlora_step_create(const tlora_step_desc* desc, tlora_comm* comm, tlora_step** out) {
  return step_guard([&] {
    need(desc != nullptr && out != nullptr, TLORA_ERR_ARG, "null argument");
    *out = nullptr;
    const tlora_step_desc& D = *desc;
    need(D.num_layers >= 1 && D.num_projections >= 1 && D.num_slots >= 1, TLORA_ERR_ARG,
         "need >= 1 layer, projection and slot");
    need(D.proj_d && D.proj_k && D.proj_input && D.ranks && D.batch && D.seq_len, TLORA_ERR_ARG,
         "null descriptor array");
    need(D.y_dtype == TLORA_BF16 || D.y_dtype == TLORA_F32, TLORA_ERR_ARG, "Y dtype must be bf16 or f32");
    need(D.input_sets == 0 || D.input_sets == 1 || D.input_sets == 2, TLORA_ERR_ARG,
         "input_sets must be 1 or 2");
    auto st = std::make_unique<tlora_step>();
    st->desc = D;
    st->device = D.device;
    st->L = D.num_layers;
    st->P = D.num_projections;
    st->S = D.num_slots;
    st->sets = D.input_sets ? D.input_sets : 1;
    st->ring = D.dh_ring > 0 ? std::max(2, D.dh_ring) : 8;
    st->d.assign(D.proj_d, D.proj_d + st->P);
    st->k.assign(D.proj_k, D.proj_k + st->P);
    st->input.assign(D.proj_input, D.proj_input + st->P);
    st->ranks.assign(D.ranks, D.ranks + st->S);
    st->batch.assign(D.batch, D.batch + st->S);
    st->seq.assign(D.seq_len, D.seq_len + st->S);
    st->groups = 0;
    for (int32_t p = 0; p < st->P; ++p) {
      need(st->input[(size_t)p] >= 0 && st->input[(size_t)p] < st->P, TLORA_ERR_ARG,
           "input group ids must be in [0, num_projections)");
      st->groups = std::max(st->groups, st->input[(size_t)p] + 1);
      for (int32_t q = 0; q < p; ++q)
        if (st->input[(size_t)q] == st->input[(size_t)p])
          need(st->d[(size_t)q] == st->d[(size_t)p], TLORA_ERR_SHAPE,
               "projections sharing an input group must have the same d");
    }
    // per-sample work (integers: the nano map is bit-exact): seq x (base GEMMs + LoRA)
    int64_t base = 0, ext = 0;
    for (int32_t p = 0; p < st->P; ++p) {
      base += 2 * st->d[(size_t)p] * st->k[(size_t)p];
      ext += 3 * (st->d[(size_t)p] + st->k[(size_t)p]);
    }
    for (int32_t s = 0; s < st->S; ++s) {
      need(st->batch[(size_t)s] >= 0 && st->seq[(size_t)s] >= 1, TLORA_ERR_ARG,
           "batch must be >= 0 and seq_len >= 1 per slot");
      st->weight.push_back((int64_t)st->seq[(size_t)s] * (base + ext * st->ranks[(size_t)s]));
      st->T += (int64_t)st->batch[(size_t)s] * st->seq[(size_t)s];
      st->total_samples += st->batch[(size_t)s];
    }
    need(st->total_samples >= 1, TLORA_ERR_ARG, "the step needs at least one sample");
    need(D.nano_fixed >= 0 && D.nano_init >= 0, TLORA_ERR_ARG, "negative nano count");
    st->aimd_n = std::min(std::max(1, D.nano_init > 0 ? D.nano_init : 4), st->total_samples);
    if (D.aimd_alpha || D.aimd_beta != 0.0 || D.aimd_tau_rel != 0.0) {
      need(D.aimd_alpha >= 1 && D.aimd_beta > 0.0 && D.aimd_beta < 1.0 && D.aimd_tau_rel >= 0.0,
           TLORA_ERR_PLAN, "AimdState: invalid controller parameters");
    }
    st->comm = comm;
    if (comm) {
      int32_t w = 1, r = 0, tp = 1, dpn = 1;
      chk(tlora_comm_info(comm, &w, &r, &tp, &dpn));
      need(tp == 1, TLORA_ERR_ARG, "the step executor runs data-parallel replicas (tp_size 1)");
      st->dp = dpn;
      // NCCL kernels on the comm stream take SMs from the persistent fused GEMMs: for layer
      // stacks (hundreds of per-key all-reduces per step) dynamic tile scheduling keeps the
      // GEMMs balanced (C3 8 layers DP2: 426 -> 389 ms); a single layer set measured 3%
      // better with the static lists (C2 DP2, 2 interleaved pairs). TLORA_DYN_SCHED overrides.
      if (!std::getenv("TLORA_DYN_SCHED") && D.num_layers > 1)
        chk(tlora_set_tile_scheduler(D.device, 1));
    }
    int prev = -1;
    ST_CUDA(cudaGetDevice(&prev));
    ST_CUDA(cudaSetDevice(D.device));
    struct Restore {
      int p;
      ~Restore() { if (p >= 0) cudaSetDevice(p); }
    } restore{prev};
    for (int32_t l = 0; l < st->L; ++l)
      for (int32_t p = 0; p < st->P; ++p) {
        tlora_layer* lay = nullptr;
        chk(tlora_layer_create(D.device, st->d[(size_t)p], st->k[(size_t)p], st->S, st->ranks.data(), &lay));
        st->layers.push_back(lay);
      }
    chk(tlora_layer_layout(st->layers[0], nullptr, &st->R));
    const int64_t T = st->T, R = st->R;
    std::vector<int64_t> gdim((size_t)st->groups, 0);
    for (int32_t p = 0; p < st->P; ++p) gdim[(size_t)st->input[(size_t)p]] = st->d[(size_t)p];
    for (int set = 0; set < st->sets; ++set) {
      for (int32_t g = 0; g < st->groups; ++g) st->X[set].push_back(st->alloc((size_t)T * gdim[(size_t)g] * 2));
      for (int32_t p = 0; p < st->P; ++p) st->dY[set].push_back(st->alloc((size_t)T * st->k[(size_t)p] * 2));
    }
    const int ysz = D.y_dtype == TLORA_BF16 ? 2 : 4;
    for (int32_t p = 0; p < st->P; ++p) {
      st->Y.push_back(st->alloc((size_t)T * st->k[(size_t)p] * ysz));
      st->dX.push_back(st->alloc((size_t)T * st->d[(size_t)p] * 2));
    }
    st->H = st->alloc((size_t)st->L * st->P * T * R * 2);
    st->dH = st->alloc((size_t)st->ring * T * R * 2);
    st->present = (int32_t*)st->alloc((size_t)st->S * 4);
    {
      std::vector<int32_t> pres((size_t)st->S);
      for (int32_t s = 0; s < st->S; ++s) pres[(size_t)s] = st->batch[(size_t)s] > 0;
      ST_CUDA(cudaMemcpy(st->present, pres.data(), (size_t)st->S * 4, cudaMemcpyHostToDevice));
    }
    ST_CUDA(cudaStreamCreateWithFlags(&st->exec, cudaStreamNonBlocking));
    if (D.flags & TLORA_STEP_SIDE_GRADS) {
      // TLORA_SIDE_PRIORITY=1 (A/B knob): the side stream's CTAs are scheduled ahead of the
      // main stream's when SMs free up (the fused GEMM's tail)
      const char* e = std::getenv("TLORA_SIDE_PRIORITY");
      if (e && e[0] == '1') {
        int lo = 0, hi = 0;
        ST_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        ST_CUDA(cudaStreamCreateWithPriority(&st->side, cudaStreamNonBlocking, hi));
      } else {
        ST_CUDA(cudaStreamCreateWithFlags(&st->side, cudaStreamNonBlocking));
      }
    }
    if (comm) ST_CUDA(cudaStreamCreateWithFlags(&st->comm_s, cudaStreamNonBlocking));
    for (int i = 0; i < tlora_step::kTimeRing; ++i) {
      ST_CUDA(cudaEventCreate(&st->t_begin_r[i]));
      ST_CUDA(cudaEventCreate(&st->t_end_r[i]));
    }
    ST_CUDA(cudaEventCreateWithFlags(&st->ev_side, cudaEventDisableTiming));
    ST_CUDA(cudaEventCreateWithFlags(&st->ev_comm, cudaEventDisableTiming));
    ST_CUDA(cudaEventCreateWithFlags(&st->ev_in, cudaEventDisableTiming));
    *out = st.release();
  });
}

int tlora_step_destroy(tlora_step* step) {
  return step_guard([&] {
    if (!step) return;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(step->device);
    cudaDeviceSynchronize();
    delete step;
    if (prev >= 0) cudaSetDevice(prev);
  });
}

int tlora_step_layer(tlora_step* step, int32_t layer, int32_t proj, tlora_layer** out) {
  return step_guard([&] {
    need(step && out, TLORA_ERR_ARG, "null argument");
    need(layer >= 0 && layer < step->L && proj >= 0 && proj < step->P, TLORA_ERR_ARG,
         "(layer, projection) out of range");
    *out = step->lay(step->key(layer, proj));
  });
}

int tlora_step_buffer(tlora_step* step, int32_t kind, int32_t index, int32_t set, void** ptr,
                      int64_t* rows, int64_t* cols) {
  return step_guard([&] {
    need(step && ptr, TLORA_ERR_ARG, "null argument");
    need(set >= 0 && set < step->sets, TLORA_ERR_ARG, "input set out of range");
    const int32_t P = step->P;
    int64_t r = step->T, c = 0;
    switch (kind) {
      case TLORA_BUF_X: {
        need(index >= 0 && index < step->groups, TLORA_ERR_ARG, "input group out of range");
        *ptr = step->X[set][(size_t)index];
        for (int32_t p = 0; p < P; ++p)
          if (step->input[(size_t)p] == index) c = step->d[(size_t)p];
        break;
      }
      case TLORA_BUF_DY:
        need(index >= 0 && index < P, TLORA_ERR_ARG, "projection out of range");
        *ptr = step->dY[set][(size_t)index];
        c = step->k[(size_t)index];
        break;
      case TLORA_BUF_Y:
        need(index >= 0 && index < P, TLORA_ERR_ARG, "projection out of range");
        *ptr = step->Y[(size_t)index];
        c = step->k[(size_t)index];
        break;
      case TLORA_BUF_DX:
        need(index >= 0 && index < P, TLORA_ERR_ARG, "projection out of range");
        *ptr = step->dX[(size_t)index];
        c = step->d[(size_t)index];
        break;
      case TLORA_BUF_H:
        need(index >= 0 && index < step->L * P, TLORA_ERR_ARG, "key out of range");
        *ptr = step->h_ptr(index, 0);
        c = step->R;
        break;
      default:
        throw StepError(TLORA_ERR_ARG, "unknown buffer kind");
    }
    if (rows) *rows = r;
    if (cols) *cols = c;
  });
}

int tlora_step_layout(tlora_step* step, int32_t n, int32_t* n_out, int64_t* nano_t0,
                      int32_t* nano_slot, int64_t* sample_row) {
  return step_guard([&] {
    need(step != nullptr, TLORA_ERR_ARG, "step is null");
    need(n >= 1, TLORA_ERR_PLAN, "partition: N must be >= 1");
    int prev = -1;
    ST_CUDA(cudaGetDevice(&prev));
    ST_CUDA(cudaSetDevice(step->device));
    Layout& lo = step->layout(std::min(n, step->total_samples));
    if (prev >= 0) cudaSetDevice(prev);
    if (n_out) *n_out = lo.map.n;
    if (nano_t0) std::memcpy(nano_t0, lo.t0.data(), lo.t0.size() * 8);
    if (nano_slot) std::memcpy(nano_slot, lo.map.nano_slot.data(), lo.map.nano_slot.size() * 4);
    if (sample_row) std::memcpy(sample_row, lo.sample_row.data(), lo.sample_row.size() * 8);
  });
}

int tlora_step_trace(const tlora_step* step, tlora_step_op* ops, double* end_ms, int32_t cap,
                     int32_t* count) {
  return step_guard([&] {
    need(step != nullptr, TLORA_ERR_ARG, "step is null");
    const auto& o = step->trace_ops;
    if (count) *count = (int32_t)o.size();
    for (size_t i = 0; i < o.size() && (int32_t)i < cap; ++i) {
      if (ops)
        ops[i] = {o[i].kind, o[i].stream, o[i].key, o[i].nano, o[i].slot, o[i].sec_kind,
                  o[i].sec_key, o[i].sec_nano, o[i].sec_slot, o[i].beta, o[i].wait0, o[i].wait1};
      if (end_ms) end_ms[i] = step->trace_ms[i];
    }
  });
}

int tlora_step_set_controller(tlora_step* step, int32_t nano_fixed, int32_t nano_init,
                              int32_t aimd_alpha, double aimd_beta, double aimd_tau_rel) {
  return step_guard([&] {
    need(step != nullptr, TLORA_ERR_ARG, "step is null");
    need(nano_fixed >= 0 && nano_init >= 0, TLORA_ERR_ARG, "negative nano count");
    const int32_t alpha = aimd_alpha ? aimd_alpha : 4;
    const double beta = aimd_beta != 0.0 ? aimd_beta : 0.5;
    if (alpha < 1 || beta <= 0.0 || beta >= 1.0 || aimd_tau_rel < 0.0)
      throw std::invalid_argument("AimdState: invalid controller parameters");
    step->desc.nano_fixed = nano_fixed;
    step->desc.nano_init = nano_init;
    step->desc.aimd_alpha = alpha;
    step->desc.aimd_beta = beta;
    step->desc.aimd_tau_rel = aimd_tau_rel;
    step->aimd_n = std::min(std::max(1, nano_init > 0 ? nano_init : 4), step->total_samples);
    step->has_prev = 0;  // the first observation seeds t_prev again (nano_pipeline.hpp:99-112)
    step->t_prev = 0.0;
  });
}

int tlora_step_next_n(const tlora_step* step, int32_t* n) {
  return step_guard([&] {
    need(step && n, TLORA_ERR_ARG, "null argument");
    *n = step->desc.nano_fixed > 0 ? std::min(step->desc.nano_fixed, step->total_samples)
                                   : step->aimd_n;
  });
}

int tlora_step_run(tlora_step* step, int32_t set, int32_t flags, void* stream,
                   tlora_step_stats* stats) {
  return step_guard([&] {
    need(step != nullptr, TLORA_ERR_ARG, "step is null");
    need(set >= 0 && set < step->sets, TLORA_ERR_ARG, "input set out of range");
    tlora_step& st = *step;
    int prev = -1;
    ST_CUDA(cudaGetDevice(&prev));
    ST_CUDA(cudaSetDevice(st.device));
    struct Restore {
      int p;
      ~Restore() { if (p >= 0) cudaSetDevice(p); }
    } restore{prev};
    cudaStream_t caller = reinterpret_cast<cudaStream_t>(stream);
    cudaStream_t main = st.exec;
    // sim_engine.hpp:307-308: n_use = fixed_n ? *fixed_n : aimd.n; partition(batch, n_use)
    const int32_t n_use = st.desc.nano_fixed > 0 ? std::min(st.desc.nano_fixed, st.total_samples)
                                                 : st.aimd_n;
    Layout& lo = st.layout(n_use);
    const int32_t n = lo.map.n;
    const bool trace = (flags & TLORA_RUN_TRACE) != 0;
    // AIMD needs this step's time before the next step; a fixed N (and no trace) does not
    const bool lazy = st.desc.nano_fixed > 0 && !trace;
    const int tslot = (int)(st.steps_run % tlora_step::kTimeRing);
    cudaEvent_t t_begin = st.t_begin_r[tslot], t_end = st.t_end_r[tslot];
    // the step starts after everything already enqueued on the caller's stream
    ST_CUDA(cudaEventRecord(st.ev_in, caller));
    ST_CUDA(cudaStreamWaitEvent(main, st.ev_in, 0));
    ST_CUDA(cudaEventRecord(t_begin, main));
    if (st.zeroed_for != n) {
      // the H stashes / dH ring must be zero outside each row's own packed-rank columns;
      // a new token layout moves jobs between rows
      ST_CUDA(cudaMemsetAsync(st.H, 0, (size_t)st.L * st.P * st.T * st.R * 2, main));
      ST_CUDA(cudaMemsetAsync(st.dH, 0, (size_t)st.ring * st.T * st.R * 2, main));
      st.zeroed_for = n;
    }
    const bool graphs = (st.desc.flags & TLORA_STEP_GRAPH) && st.comm == nullptr &&
                        !(flags & (TLORA_RUN_EAGER | TLORA_RUN_TRACE));
    const long long l0 = tlora_launch_count();
    bool replayed = false;
    if (graphs && lo.graph[set] != nullptr) {
      ST_CUDA(cudaGraphLaunch(lo.graph[set], main));
      replayed = true;
    } else {
      st.enqueue(lo, set, main, trace);
    }
    ST_CUDA(cudaEventRecord(t_end, main));
    ST_CUDA(cudaStreamWaitEvent(caller, t_end, 0));  // and the caller's stream after it
    st.t_step_r[tslot] = st.steps_run;
    float ms = -1.f;
    if (!lazy) {
      ST_CUDA(cudaEventSynchronize(t_end));
      ST_CUDA(cudaEventElapsedTime(&ms, t_begin, t_end));
    } else {  // the latest step whose end event has completed (-1: none yet)
      long long best = -1;
      for (int i = 0; i < tlora_step::kTimeRing; ++i) {
        if (st.t_step_r[i] <= best || cudaEventQuery(st.t_end_r[i]) != cudaSuccess) continue;
        float t = 0.f;
        if (cudaEventElapsedTime(&t, st.t_begin_r[i], st.t_end_r[i]) == cudaSuccess) {
          best = st.t_step_r[i];
          ms = t;
        }
      }
      (void)cudaGetLastError();  // cudaErrorNotReady of the queries is not an error here
    }
    if (trace) {
      st.trace_ops = lo.ops;
      st.trace_ms.assign(lo.ops.size(), 0.0);
      for (size_t i = 0; i < lo.ops.size(); ++i) {
        float t = 0.f;
        ST_CUDA(cudaEventElapsedTime(&t, t_begin, st.trace_ev[i]));
        st.trace_ms[i] = t;
      }
    }
    if (!replayed) lo.launches = tlora_launch_count() - l0;
    const long long launches = lo.launches;
    if (graphs && !replayed) {
      // capture this layout's step for the next visits (every scratch buffer now exists;
      // the eager run may still be executing: capture only records)
      cudaGraph_t g = nullptr;
      ST_CUDA(cudaStreamBeginCapture(main, cudaStreamCaptureModeThreadLocal));
      try {
        st.enqueue(lo, set, main);
      } catch (...) {
        cudaStreamEndCapture(main, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      ST_CUDA(cudaStreamEndCapture(main, &g));
      ST_CUDA(cudaGraphInstantiate(&lo.graph[set], g, 0));
      ST_CUDA(cudaGraphDestroy(g));
    }
    // nano_pipeline.hpp:99-112 + sim_engine.hpp:314 (clamp to the combined batch)
    if (st.desc.nano_fixed <= 0) {
      const int32_t alpha = st.desc.aimd_alpha ? st.desc.aimd_alpha : 4;
      const double beta = st.desc.aimd_beta != 0.0 ? st.desc.aimd_beta : 0.5;
      chk(tlora_aimd_step(&st.aimd_n, &st.has_prev, &st.t_prev, alpha, beta,
                          st.desc.aimd_tau_rel, (double)ms / 1e3));
      st.aimd_n = std::min(st.aimd_n, st.total_samples);
    }
    st.trajectory.push_back({n, (double)ms});
    ++st.steps_run;
    if (stats) {
      stats->nano_used = n;
      stats->next_nano = st.desc.nano_fixed > 0 ? n_use : st.aimd_n;
      stats->ms = ms;
      stats->replayed_graph = replayed ? 1 : 0;
      stats->launches = launches;
      stats->tokens = st.T;
    }
  });
}

}  // extern "C"
