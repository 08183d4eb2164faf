// tlora_tp.cu — the tensor-parallel layer-set training step (C++ host; C-ABI tlora_tp_*).
//
// SURVEY §8(e) "tensor-parallel over W" executed for real (the reference only simulates the
// timeline: nano_pipeline.hpp:65-97, sim_engine.hpp:306-315). Megatron-SP split of every
// projection over the communicator's ranks (the TP group):
//
//   column-parallel (q, k, v, gate, up)   W[:, k/P], B_j[:, k/P] local, A_j replicated
//     fwd  H_j = X_j·A_j on this rank's SP token shard -> all-gather [X | H] -> fused GEMM
//     bwd  dH = dY·Bᵀ and dX = dY·Wᵀ + dH·Aᵀ are partial over ranks -> reduce-scatter
//          [dX | dH] (dX of the projections of one input group summed in place by the
//          fused GEMM's beta); dB local from the gathered H; dA from the SP shard (X_shard,
//          dH_shard) -> all-reduced once per step (A replicated)
//   row-parallel (o, down)                 W[d/P, :], A_j[d/P, :] local, B_j replicated
//     fwd  H_p = X_p·A_p partial -> fused GEMM -> reduce-scatter Y (sums the partial H·B too)
//     bwd  all-gather dY -> dH exact, dX local, dA local; dB partial -> all-reduced
//
// Per nano-batch (rank-aware map of tlora_nano.hpp, N from AIMD on the group-mean step time,
// as tlora_step_run), the boundary traffic of nano n+1 (all-gathers) and n-1
// (reduce-scatters) runs on a comm stream while nano n's GEMMs run on the main stream; the
// adapter-gradient launches run on a side stream. Boundary traffic is either NCCL (through
// the C-ABI communicator) or, with TLORA_TP_COPY_ENGINE, copy-engine pushes into every
// peer's buffer (CUDA IPC peer mappings, exchanged once over NCCL) followed by a fenced
// stream write of this rank's epoch into every peer's flag array; consumers wait with a
// stream wait-value (no SM is used). With TLORA_TP_FUSED_RS the row-parallel GEMM epilogue
// bulk-copies its output rows into the owner rank's receive slot over NVLink and the owner
// sums its P slots in fixed order (tlora_reduce_slots).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
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
void note_launch();                           // tlora_capi.cu: library launch counter
}

namespace {

// Wait until every peer's epoch flag reached `ep` (lane q polls flags[q]; q = self skipped).
// The kernel form of the flag wait: a spinning 32-thread CTA occupies no front-end channel,
// where a blocked stream wait-value op can hold back unrelated streams sharing its
// hardware queue while later work is already enqueued.
__global__ void flag_wait_kernel(const uint32_t* flags, int P, int self, uint32_t ep) {
  const int q = threadIdx.x;
  if (q < P && q != self) {
    uint32_t v;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + q) : "memory");
      if ((int32_t)(v - ep) >= 0) break;
      __nanosleep(64);
    } while (true);
  }
  __syncwarp();
}

struct TpError : std::runtime_error {
  int code;
  TpError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void chk(int rc) {
  if (rc != TLORA_OK) throw TpError(rc, tlora_last_error());
}

#define TP_CUDA(x)                                                                         \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      throw TpError(TLORA_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));      \
  } while (0)

void need(bool ok, int code, const std::string& msg) {
  if (!ok) throw TpError(code, msg);
}

template <class F>
int tp_guard(F&& f) {
  try {
    f();
    return TLORA_OK;
  } catch (const TpError& e) {
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

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) TP_CUDA(cudaSetDevice(d));
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// A device buffer mapped into every rank's address space (CUDA IPC): ptr[q] is rank q's
// copy as seen from this process (ptr[rank] = the local allocation).
struct PeerBuf {
  std::vector<char*> ptr;
  size_t bytes = 0;
};

struct Nano {
  int64_t t0 = 0, tokens = 0;
  std::vector<int32_t> slots;
  std::vector<tlora_plan*> plan_full;   // per projection: the nano-batch's plan
  std::vector<tlora_plan*> plan_shard;  // per column projection: this rank's SP shard plan
};

struct Layout {
  tlora::NanoMap map;
  std::vector<Nano> nanos;
};

}  // namespace

struct tlora_tp_step {
  int device = 0;
  tlora_tp_desc desc{};
  tlora_comm* comm = nullptr;
  int32_t P = 1, rank = 0, S = 0, NP = 0, groups = 0;
  int64_t T = 0;
  std::vector<int64_t> d, k;      // full dims
  std::vector<int32_t> input, row;
  std::vector<int32_t> ranks, batch, seq;
  std::vector<int64_t> weight;
  int32_t total_samples = 0;
  std::vector<tlora_layer*> layers;
  std::vector<int32_t> R;  // packed rank width per projection
  std::vector<void*> owned;
  std::vector<int64_t> gdim;  // per input group: full d
  // buffers (see tlora.h tlora_tp_buffer_kind)
  std::vector<char*> X_shard, X_full, dX_part, dX_shard;                    // per group
  std::vector<char*> H_shard, H_full, Y, dY, dH_part, dH_shard;              // per column proj
  std::vector<char*> X_loc, H_row, Y_part, Y_shard, dY_shard, dY_full, dH_row, dX_loc;  // row
  // copy-engine / fused reduce-scatter peer buffers
  bool ce = false, fused = false;
  std::map<std::string, PeerBuf> peer;  // X_full[g], H_full[p], dY_full[p], rsX[g], rsH[p], recv[p]
  PeerBuf flags;                        // int32 [P] per rank: epoch raised by each source
  uint32_t epoch = 0;
  std::vector<void*> ipc_opened;
  int32_t* present = nullptr;
  cudaStream_t main = nullptr, comm_s = nullptr, side = nullptr;
  // step timing: a ring of (begin, end) pairs; with a fixed N run() does not wait for the
  // step and reports the latest completed one
  static constexpr int kTimeRing = 4;
  cudaEvent_t t_begin_r[kTimeRing] = {}, t_end_r[kTimeRing] = {};
  long long t_step_r[kTimeRing] = {-1, -1, -1, -1};
  long long steps_run = 0;
  // TLORA_RUN_TRACE: CUDA events around every nano-batch's compute (main stream) and
  // boundary traffic (comm stream): the measured PipelineTrace (nano_pipeline.hpp:28-34)
  bool tracing = false;
  struct Mark {
    int kind, nano, edge;  // kind: 0 compute, 1 communication
    cudaEvent_t ev;
  };
  std::vector<Mark> marks;
  std::vector<cudaEvent_t> mark_pool;
  std::vector<double> trace_comp, trace_comm;  // per nano-batch, ms (last traced step)
  void mark(cudaStream_t s, int kind, int nano, int edge) {
    if (!tracing) return;
    if (marks.size() == mark_pool.size()) {
      cudaEvent_t e;
      TP_CUDA(cudaEventCreate(&e));
      mark_pool.push_back(e);
    }
    cudaEvent_t e = mark_pool[marks.size()];
    TP_CUDA(cudaEventRecord(e, s));
    marks.push_back({kind, nano, edge, e});
  }
  std::vector<cudaEvent_t> evpool;
  size_t ev_next = 0;
  std::map<int32_t, std::unique_ptr<Layout>> layouts;
  int32_t aimd_n = 4, has_prev = 0;
  double t_prev = 0.0;
  double* ms_dev = nullptr;  // the group's mean step time (AIMD input)

  ~tlora_tp_step();
  char* alloc(size_t bytes) {
    void* p = nullptr;
    if (bytes) {
      TP_CUDA(cudaMalloc(&p, bytes));
      owned.push_back(p);
    }
    return (char*)p;
  }
  cudaEvent_t ev() {  // a fresh (reusable per step) sync event
    if (ev_next == evpool.size()) {
      cudaEvent_t e;
      TP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      evpool.push_back(e);
    }
    return evpool[ev_next++];
  }
  void wait(cudaStream_t waiter, cudaStream_t on) {
    cudaEvent_t e = ev();
    TP_CUDA(cudaEventRecord(e, on));
    TP_CUDA(cudaStreamWaitEvent(waiter, e, 0));
  }
  PeerBuf make_peer(size_t bytes);
  Layout& layout(int32_t n);
  void forward(Layout& lo);
  void backward(Layout& lo);
  // boundary traffic
  void all_gather(const std::string& key, char* full, const char* shard, size_t row_bytes,
                  const Nano& b);
  void reduce_scatter(const std::string& key, const char* part, char* out, int64_t width,
                      const Nano& b);
  uint32_t ce_raise();
  void ce_wait(cudaStream_t s, uint32_t ep);
};

tlora_tp_step::~tlora_tp_step() {
  for (auto& [n, lo] : layouts)
    for (auto& nb : lo->nanos) {
      for (auto* p : nb.plan_full) tlora_plan_destroy(p);
      for (auto* p : nb.plan_shard)
        if (p) tlora_plan_destroy(p);
    }
  for (auto* l : layers) tlora_layer_destroy(l);
  for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
  for (auto e : evpool) cudaEventDestroy(e);
  for (auto e : mark_pool) cudaEventDestroy(e);
  for (int i = 0; i < kTimeRing; ++i)
    for (auto e : {t_begin_r[i], t_end_r[i]})
      if (e) cudaEventDestroy(e);
  for (auto s : {main, comm_s, side})
    if (s) cudaStreamDestroy(s);
  for (void* p : owned) cudaFree(p);
}

// Peer-mapped buffer: a local cudaMalloc whose IPC handle is all-gathered over NCCL and
// opened by every other rank (same size everywhere).
PeerBuf tlora_tp_step::make_peer(size_t bytes) {
  PeerBuf b;
  b.bytes = bytes;
  char* mine = alloc(bytes);
  TP_CUDA(cudaMemset(mine, 0, bytes));
  cudaIpcMemHandle_t h;
  TP_CUDA(cudaIpcGetMemHandle(&h, mine));
  static_assert(sizeof(cudaIpcMemHandle_t) % 4 == 0, "handle is whole f32 words");
  const size_t words = sizeof(cudaIpcMemHandle_t) / 4;
  float* dsend = (float*)alloc(sizeof h);
  float* drecv = (float*)alloc(sizeof h * P);
  TP_CUDA(cudaMemcpy(dsend, &h, sizeof h, cudaMemcpyHostToDevice));
  chk(tlora_comm_all_gather(comm, TLORA_GROUP_WORLD, dsend, drecv, words, TLORA_F32, main));
  TP_CUDA(cudaStreamSynchronize(main));
  std::vector<cudaIpcMemHandle_t> all(P);
  TP_CUDA(cudaMemcpy(all.data(), drecv, sizeof h * P, cudaMemcpyDeviceToHost));
  b.ptr.assign(P, nullptr);
  for (int q = 0; q < P; ++q) {
    if (q == rank) {
      b.ptr[q] = mine;
      continue;
    }
    void* p = nullptr;
    TP_CUDA(cudaIpcOpenMemHandle(&p, all[q], cudaIpcMemLazyEnablePeerAccess));
    ipc_opened.push_back(p);
    b.ptr[q] = (char*)p;
  }
  return b;
}

Layout& tlora_tp_step::layout(int32_t n) {
  auto it = layouts.find(n);
  if (it != layouts.end()) return *it->second;
  auto lo = std::make_unique<Layout>();
  // TLORA_TP_RAMP=g (> 1): ramped nano-batch sizes (tlora_nano.hpp nano_assign_ramp)
  static const double ramp = [] {
    const char* e = std::getenv("TLORA_TP_RAMP");
    return e ? std::atof(e) : 0.0;
  }();
  lo->map = tlora::nano_assign_ramp(batch, weight, n, ramp);
  int64_t t0 = 0;
  for (int32_t i = 0; i < lo->map.n; ++i) {
    Nano nb;
    nb.t0 = t0;
    for (int32_t s = 0; s < S; ++s)
      nb.slots.insert(nb.slots.end(), (size_t)lo->map.nano_slot[(size_t)i * S + s] * seq[(size_t)s], s);
    nb.tokens = (int64_t)nb.slots.size();
    need(nb.tokens % P == 0, TLORA_ERR_SHAPE,
         "every nano-batch's token count must split evenly over the TP ranks");
    const int64_t nr = nb.tokens / P;
    for (int32_t p = 0; p < NP; ++p) {
      tlora_plan* pl = nullptr;
      chk(tlora_plan_create(layers[(size_t)p], nb.tokens, nb.slots.data(), &pl));
      nb.plan_full.push_back(pl);
      tlora_plan* ps = nullptr;
      if (!row[(size_t)p])
        chk(tlora_plan_create(layers[(size_t)p], nr, nb.slots.data() + rank * nr, &ps));
      nb.plan_shard.push_back(ps);
    }
    t0 += nb.tokens;
    lo->nanos.push_back(std::move(nb));
  }
  auto& ref = *lo;
  layouts.emplace(n, std::move(lo));
  return ref;
}

// ---- copy-engine epochs: every boundary operation raises this rank's epoch in every peer's
// flag array (fenced after the pushes) and waits until every peer reached it.
uint32_t tlora_tp_step::ce_raise() {
  ++epoch;
  for (int q = 0; q < P; ++q)
    if (q != rank) chk(tlora_stream_write_u32(comm_s, flags.ptr[q] + 4 * rank, epoch));
  return epoch;
}

void tlora_tp_step::ce_wait(cudaStream_t s, uint32_t ep) {
  // TLORA_TP_MEMOP_MAIN=0 (A/B knob): keep the stream wait-value ops off the GEMM stream —
  // the comm stream waits for the flags and the main stream waits for the comm stream
  static const bool off_main = [] {
    const char* e = std::getenv("TLORA_TP_MEMOP_MAIN");
    return e && e[0] == '0';
  }();
  // TLORA_TP_WAIT=memop|kernel (A/B knob): stream wait-value ops or a polling kernel
  static const bool kernel_wait = [] {
    const char* e = std::getenv("TLORA_TP_WAIT");
    return e && std::strcmp(e, "kernel") == 0;
  }();
  cudaStream_t w = (off_main && s == main) ? comm_s : s;
  if (kernel_wait) {
    flag_wait_kernel<<<1, 32, 0, w>>>(reinterpret_cast<const uint32_t*>(flags.ptr[rank]), P, rank,
                                      ep);
    TP_CUDA(cudaGetLastError());
    tlora::note_launch();
  } else {
    for (int q = 0; q < P; ++q)
      if (q != rank) chk(tlora_stream_wait_u32(w, flags.ptr[rank] + 4 * q, ep));
  }
  if (w != s) wait(s, w);
}

// Rows [t0, t0 + tokens) of the gathered buffer: rank q's shard lands at t0 + q * tokens / P
// (all_gather_into_tensor layout).
void tlora_tp_step::all_gather(const std::string& key, char* full, const char* shard,
                               size_t row_bytes, const Nano& b) {
  const int64_t nr = b.tokens / P;
  char* dst = full + b.t0 * row_bytes;
  const char* src = shard + (b.t0 / P) * row_bytes;
  if (!ce) {
    chk(tlora_comm_all_gather(comm, TLORA_GROUP_WORLD, src, dst, nr * row_bytes / 2, TLORA_BF16,
                              comm_s));
    return;
  }
  const PeerBuf& pb = peer.at(key);
  const size_t off = (b.t0 + rank * nr) * row_bytes;
  for (int j = 0; j < P; ++j) {  // peers from the next rank on, self last
    const int q = (rank + 1 + j) % P;
    chk(tlora_copy_async(pb.ptr[q] + off, src, nr * row_bytes, comm_s));
  }
}

// out[rows of this rank's shard of nano b] = sum over ranks of part[the same rows]
void tlora_tp_step::reduce_scatter(const std::string& key, const char* part, char* out,
                                   int64_t width, const Nano& b) {
  const int64_t nr = b.tokens / P;
  const size_t row_bytes = (size_t)width * 2;
  const char* src = part + b.t0 * row_bytes;
  char* dst = out + (b.t0 / P) * row_bytes;
  if (!ce) {
    chk(tlora_comm_reduce_scatter(comm, TLORA_GROUP_WORLD, src, dst, nr * width, TLORA_BF16,
                                  comm_s));
    return;
  }
  // push the rows owned by rank q into q's receive slot `rank` (slot rows = T / P)
  const PeerBuf& pb = peer.at(key);
  const int64_t slot_rows = T / P, row0 = b.t0 / P;
  for (int j = 0; j < P; ++j) {
    const int q = (rank + 1 + j) % P;
    chk(tlora_copy_async(pb.ptr[q] + (rank * slot_rows + row0) * row_bytes,
                         src + q * nr * row_bytes, nr * row_bytes, comm_s));
  }
}

namespace {
char* rows_of(char* base, int64_t row0, int64_t width, int bytes = 2) {
  return base + row0 * width * bytes;
}
}  // namespace

void tlora_tp_step::forward(Layout& lo) {
  const size_t n = lo.nanos.size();
  std::vector<cudaEvent_t> ev_g(n);
  std::vector<uint32_t> ep_g(n, 0);
  // the fused reduce-scatter writes into every owner's receive slots: every rank has
  // consumed the previous step's slots (barrier on the flags)
  if (fused) {
    wait(comm_s, main);
    ce_wait(main, ce_raise());
  }
  auto shrink_gather = [&](size_t i) {
    const Nano& b = lo.nanos[i];
    const int64_t nr = b.tokens / P;
    for (int32_t p = 0; p < NP; ++p) {
      if (row[(size_t)p]) continue;
      const int g = input[(size_t)p];
      chk(tlora_forward_shrink(layers[(size_t)p], b.plan_shard[(size_t)p],
                               rows_of(X_shard[(size_t)g], b.t0 / P, gdim[(size_t)g]),
                               rows_of(H_shard[(size_t)p], b.t0 / P, R[(size_t)p]), main));
    }
    wait(comm_s, main);
    mark(comm_s, 1, (int)i, 0);
    for (int g = 0; g < groups; ++g)
      all_gather("X" + std::to_string(g), X_full[(size_t)g], X_shard[(size_t)g],
                 (size_t)gdim[(size_t)g] * 2, b);
    for (int32_t p = 0; p < NP; ++p)
      if (!row[(size_t)p])
        all_gather("H" + std::to_string(p), H_full[(size_t)p], H_shard[(size_t)p],
                   (size_t)R[(size_t)p] * 2, b);
    if (ce) ep_g[i] = ce_raise();
    mark(comm_s, 1, (int)i, 1);
    ev_g[i] = ev();
    TP_CUDA(cudaEventRecord(ev_g[i], comm_s));
    (void)nr;
  };
  shrink_gather(0);
  for (size_t i = 0; i < n; ++i) {
    if (i + 1 < n) shrink_gather(i + 1);
    const Nano& b = lo.nanos[i];
    TP_CUDA(cudaStreamWaitEvent(main, ev_g[i], 0));
    if (ce) ce_wait(main, ep_g[i]);
    mark(main, 0, (int)i, 0);
    for (int32_t p = 0; p < NP; ++p) {
      if (row[(size_t)p]) continue;
      const int g = input[(size_t)p];
      chk(tlora_forward_gemm(layers[(size_t)p], b.plan_full[(size_t)p],
                             rows_of(X_full[(size_t)g], b.t0, gdim[(size_t)g]),
                             rows_of(H_full[(size_t)p], b.t0, R[(size_t)p]),
                             rows_of(Y[(size_t)p], b.t0, k[(size_t)p] / P), TLORA_BF16, main));
    }
    for (int32_t p = 0; p < NP; ++p) {
      if (!row[(size_t)p]) continue;
      tlora_layer* l = layers[(size_t)p];
      tlora_plan* pl = b.plan_full[(size_t)p];
      const int64_t dl = d[(size_t)p] / P;
      char* Xp = rows_of(X_loc[(size_t)p], b.t0, dl);
      char* Hp = rows_of(H_row[(size_t)p], b.t0, R[(size_t)p]);
      chk(tlora_forward_shrink(l, pl, Xp, Hp, main));
      if (fused) {
        const PeerBuf& rb = peer.at("recv" + std::to_string(p));
        std::vector<void*> ptrs(rb.ptr.begin(), rb.ptr.end());
        chk(tlora_forward_gemm_rs(l, pl, Xp, Hp, ptrs.data(), P, rank, T / P, b.t0 / P, main));
      } else {
        chk(tlora_forward_gemm(l, pl, Xp, Hp, rows_of(Y_part[(size_t)p], b.t0, k[(size_t)p]),
                               TLORA_BF16, main));
      }
    }
    mark(main, 0, (int)i, 1);
    // reduce-scatter of the row-parallel outputs, off the main stream
    wait(comm_s, main);
    mark(comm_s, 1, (int)i, 0);
    for (int32_t p = 0; p < NP; ++p) {
      if (!row[(size_t)p]) continue;
      const int64_t kk = k[(size_t)p];
      if (fused) {
        ce_wait(comm_s, ce_raise());  // every rank's epilogue has written into our slots
        chk(tlora_reduce_slots(peer.at("recv" + std::to_string(p)).ptr[rank], P, T / P, b.t0 / P,
                               b.tokens / P, kk, rows_of(Y_shard[(size_t)p], b.t0 / P, kk), comm_s));
      } else {
        chk(tlora_comm_reduce_scatter(comm, TLORA_GROUP_WORLD, rows_of(Y_part[(size_t)p], b.t0, kk),
                                      rows_of(Y_shard[(size_t)p], b.t0 / P, kk),
                                      (b.tokens / P) * kk, TLORA_BF16, comm_s));
      }
    }
    mark(comm_s, 1, (int)i, 1);
  }
  wait(main, comm_s);
}

void tlora_tp_step::backward(Layout& lo) {
  const size_t n = lo.nanos.size();
  cudaStream_t G = side ? side : main;
  wait(comm_s, main);
  if (G != main) wait(G, main);
  std::vector<cudaEvent_t> ev_dy(n);
  std::vector<uint32_t> ep_dy(n, 0);
  auto gather_dy = [&](size_t i) {
    const Nano& b = lo.nanos[i];
    mark(comm_s, 1, (int)i, 0);
    for (int32_t p = 0; p < NP; ++p)
      if (row[(size_t)p])
        all_gather("dY" + std::to_string(p), dY_full[(size_t)p], dY_shard[(size_t)p],
                   (size_t)k[(size_t)p] * 2, b);
    if (ce) ep_dy[i] = ce_raise();
    mark(comm_s, 1, (int)i, 1);
    ev_dy[i] = ev();
    TP_CUDA(cudaEventRecord(ev_dy[i], comm_s));
  };
  // order: row-parallel projections, then the column-parallel ones in reverse
  std::vector<int32_t> seq;
  for (int32_t p = 0; p < NP; ++p)
    if (row[(size_t)p]) seq.push_back(p);
  for (int32_t p = NP - 1; p >= 0; --p)
    if (!row[(size_t)p]) seq.push_back(p);
  cudaEvent_t ev_prev_rs = nullptr;
  size_t prev_i = 0;
  auto grad_a_cols = [&](size_t i, cudaEvent_t after) {
    const Nano& b = lo.nanos[i];
    TP_CUDA(cudaStreamWaitEvent(G, after, 0));
    for (int32_t p = 0; p < NP; ++p) {
      if (row[(size_t)p]) continue;
      const int g = input[(size_t)p];
      chk(tlora_backward_grad_a(layers[(size_t)p], b.plan_shard[(size_t)p],
                                rows_of(X_shard[(size_t)g], b.t0 / P, gdim[(size_t)g]),
                                rows_of(dH_shard[(size_t)p], b.t0 / P, R[(size_t)p]),
                                i ? 1.f : 0.f, G));
    }
  };
  gather_dy(0);
  for (size_t i = 0; i < n; ++i) {
    if (i + 1 < n) gather_dy(i + 1);
    const Nano& b = lo.nanos[i];
    const float beta = i ? 1.f : 0.f;
    TP_CUDA(cudaStreamWaitEvent(main, ev_dy[i], 0));
    if (ce) ce_wait(main, ep_dy[i]);
    mark(main, 0, (int)i, 0);
    auto dy_dh = [&](int32_t p, char*& dYp, char*& dHp) {
      if (row[(size_t)p]) {
        dYp = rows_of(dY_full[(size_t)p], b.t0, k[(size_t)p]);
        dHp = rows_of(dH_row[(size_t)p], b.t0, R[(size_t)p]);
      } else {
        dYp = rows_of(dY[(size_t)p], b.t0, k[(size_t)p] / P);
        dHp = rows_of(dH_part[(size_t)p], b.t0, R[(size_t)p]);
      }
    };
    char *dY0, *dH0;
    dy_dh(seq[0], dY0, dH0);
    chk(tlora_backward_dh(layers[(size_t)seq[0]], b.plan_full[(size_t)seq[0]], dY0, dH0, main));
    std::vector<char> first(groups, 0);
    for (size_t j = 0; j < seq.size(); ++j) {
      const int32_t p = seq[j];
      tlora_layer* l = layers[(size_t)p];
      tlora_plan* pl = b.plan_full[(size_t)p];
      char *dYp, *dHp;
      dy_dh(p, dYp, dHp);
      char* dXp;
      float bx = 0.f;
      if (row[(size_t)p]) {
        dXp = rows_of(dX_loc[(size_t)p], b.t0, d[(size_t)p] / P);
      } else {
        const int g = input[(size_t)p];
        dXp = rows_of(dX_part[(size_t)g], b.t0, gdim[(size_t)g]);
        bx = first[(size_t)g] ? 1.f : 0.f;
        first[(size_t)g] = 1;
      }
      if (j + 1 < seq.size()) {
        const int32_t pn = seq[j + 1];
        char *dYn, *dHn;
        dy_dh(pn, dYn, dHn);
        chk(tlora_backward_dx_dh(l, pl, dYp, dHp, dXp, bx, layers[(size_t)pn], b.plan_full[(size_t)pn],
                                 dYn, dHn, 1, main));
      } else {
        chk(tlora_backward_dx(l, pl, dYp, dHp, dXp, bx, main));
      }
      if (G != main) wait(G, main);  // dH of p (written by the previous launch) and dY ready
      if (row[(size_t)p])
        chk(tlora_backward_grads(l, pl, rows_of(H_row[(size_t)p], b.t0, R[(size_t)p]), dYp,
                                 rows_of(X_loc[(size_t)p], b.t0, d[(size_t)p] / P), dHp, beta, G));
      else
        chk(tlora_backward_grad_b(l, pl, rows_of(H_full[(size_t)p], b.t0, R[(size_t)p]), dYp, beta, G));
    }
    mark(main, 0, (int)i, 1);
    // reduce-scatter [dX | dH] of the column-parallel projections
    wait(comm_s, main);
    mark(comm_s, 1, (int)i, 0);
    for (int g = 0; g < groups; ++g)
      reduce_scatter("rsX" + std::to_string(g), dX_part[(size_t)g], dX_shard[(size_t)g],
                     gdim[(size_t)g], b);
    for (int32_t p = 0; p < NP; ++p)
      if (!row[(size_t)p])
        reduce_scatter("rsH" + std::to_string(p), dH_part[(size_t)p], dH_shard[(size_t)p],
                       R[(size_t)p], b);
    if (ce) {  // every peer's pushes landed: sum our P slots in fixed order
      ce_wait(comm_s, ce_raise());
      const int64_t slot_rows = T / P, row0 = b.t0 / P, nr = b.tokens / P;
      for (int g = 0; g < groups; ++g)
        chk(tlora_reduce_slots(peer.at("rsX" + std::to_string(g)).ptr[rank], P, slot_rows, row0, nr,
                               gdim[(size_t)g], rows_of(dX_shard[(size_t)g], row0, gdim[(size_t)g]),
                               comm_s));
      for (int32_t p = 0; p < NP; ++p)
        if (!row[(size_t)p])
          chk(tlora_reduce_slots(peer.at("rsH" + std::to_string(p)).ptr[rank], P, slot_rows, row0,
                                 nr, R[(size_t)p], rows_of(dH_shard[(size_t)p], row0, R[(size_t)p]),
                                 comm_s));
    }
    mark(comm_s, 1, (int)i, 1);
    cudaEvent_t ev_r = ev();
    TP_CUDA(cudaEventRecord(ev_r, comm_s));
    if (ev_prev_rs) grad_a_cols(prev_i, ev_prev_rs);
    ev_prev_rs = ev_r;
    prev_i = i;
  }
  grad_a_cols(prev_i, ev_prev_rs);
  // replicated adapter halves: sum the TP partials once per step (dAᵀ of the column-
  // parallel projections, dB of the row-parallel ones)
  if (G != main) wait(main, G);
  wait(comm_s, main);
  for (int32_t p = 0; p < NP; ++p) {
    float *dAT = nullptr, *dB = nullptr;
    chk(tlora_layer_grad_ptrs(layers[(size_t)p], &dAT, &dB));
    const size_t Rp = (size_t)R[(size_t)p];
    if (row[(size_t)p])
      chk(tlora_comm_all_reduce(comm, TLORA_GROUP_WORLD, dB, dB, Rp * k[(size_t)p], TLORA_F32, 0, comm_s));
    else
      chk(tlora_comm_all_reduce(comm, TLORA_GROUP_WORLD, dAT, dAT, Rp * d[(size_t)p], TLORA_F32, 0, comm_s));
  }
  wait(main, comm_s);
}

extern "C" {

int tlora_tp_create(const tlora_tp_desc* desc, tlora_comm* comm, tlora_tp_step** out) {
  return tp_guard([&] {
    need(desc != nullptr && out != nullptr && comm != nullptr, TLORA_ERR_ARG, "null argument");
    *out = nullptr;
    const tlora_tp_desc& D = *desc;
    need(D.num_projections >= 1 && D.num_slots >= 1, TLORA_ERR_ARG, "need projections and slots");
    need(D.proj_d && D.proj_k && D.proj_input && D.proj_row_parallel && D.ranks && D.batch &&
             D.seq_len, TLORA_ERR_ARG, "null descriptor array");
    auto st = std::make_unique<tlora_tp_step>();
    st->desc = D;
    st->device = D.device;
    st->comm = comm;
    int32_t w = 1, r = 0, tp = 1, dp = 1;
    chk(tlora_comm_info(comm, &w, &r, &tp, &dp));
    need(tp == w, TLORA_ERR_ARG, "the TP step runs over the whole communicator (tp_size == world)");
    st->P = w;
    st->rank = r;
    st->NP = D.num_projections;
    st->S = D.num_slots;
    st->d.assign(D.proj_d, D.proj_d + st->NP);
    st->k.assign(D.proj_k, D.proj_k + st->NP);
    st->input.assign(D.proj_input, D.proj_input + st->NP);
    st->row.assign(D.proj_row_parallel, D.proj_row_parallel + st->NP);
    st->ranks.assign(D.ranks, D.ranks + st->S);
    st->batch.assign(D.batch, D.batch + st->S);
    st->seq.assign(D.seq_len, D.seq_len + st->S);
    // TLORA_TP_CE_SELF=1: keep the copy-engine and fused reduce-scatter data paths at P = 1
    // (pushes to this rank's own buffers; single-GPU test coverage of those paths)
    const char* ce_self_env = std::getenv("TLORA_TP_CE_SELF");
    const bool multi = st->P > 1 || (ce_self_env && ce_self_env[0] == '1');
    st->ce = (D.flags & TLORA_TP_COPY_ENGINE) && multi;
    st->fused = (D.flags & TLORA_TP_FUSED_RS) && multi;
    const int32_t P = st->P;
    int64_t base = 0, ext = 0;
    for (int32_t p = 0; p < st->NP; ++p) {
      need(st->row[(size_t)p] ? st->d[(size_t)p] % P == 0 : st->k[(size_t)p] % P == 0,
           TLORA_ERR_SHAPE, "the split dimension must divide evenly over the TP ranks");
      base += 2 * st->d[(size_t)p] * st->k[(size_t)p];
      ext += 3 * (st->d[(size_t)p] + st->k[(size_t)p]);
      if (!st->row[(size_t)p]) st->groups = std::max(st->groups, st->input[(size_t)p] + 1);
    }
    for (int32_t s = 0; s < st->S; ++s) {
      st->weight.push_back((int64_t)st->seq[(size_t)s] * (base + ext * st->ranks[(size_t)s]));
      st->T += (int64_t)st->batch[(size_t)s] * st->seq[(size_t)s];
      st->total_samples += st->batch[(size_t)s];
    }
    need(st->T % P == 0, TLORA_ERR_SHAPE, "tokens must split evenly over the TP ranks");
    st->aimd_n = std::min(std::max(1, D.nano_init > 0 ? D.nano_init : 4), st->total_samples);
    DevGuard g(D.device);
    TP_CUDA(cudaStreamCreateWithFlags(&st->main, cudaStreamNonBlocking));
    TP_CUDA(cudaStreamCreateWithFlags(&st->comm_s, cudaStreamNonBlocking));
    if (D.flags & TLORA_TP_SIDE_GRADS) TP_CUDA(cudaStreamCreateWithFlags(&st->side, cudaStreamNonBlocking));
    for (int i = 0; i < tlora_tp_step::kTimeRing; ++i) {
      TP_CUDA(cudaEventCreate(&st->t_begin_r[i]));
      TP_CUDA(cudaEventCreate(&st->t_end_r[i]));
    }
    st->ms_dev = (double*)st->alloc(sizeof(double));
    for (int32_t p = 0; p < st->NP; ++p) {
      tlora_layer* l = nullptr;
      const bool rp = st->row[(size_t)p];
      chk(tlora_layer_create(D.device, rp ? st->d[(size_t)p] / P : st->d[(size_t)p],
                             rp ? st->k[(size_t)p] : st->k[(size_t)p] / P, st->S, st->ranks.data(), &l));
      st->layers.push_back(l);
      int32_t Rp = 0;
      chk(tlora_layer_layout(l, nullptr, &Rp));
      st->R.push_back(Rp);
    }
    const int64_t T = st->T;
    st->gdim.assign((size_t)st->groups, 0);
    for (int32_t p = 0; p < st->NP; ++p)
      if (!st->row[(size_t)p]) st->gdim[(size_t)st->input[(size_t)p]] = st->d[(size_t)p];
    auto peer_or_local = [&](const std::string& key, size_t bytes) -> char* {
      if (st->ce) {
        st->peer[key] = st->make_peer(bytes);
        return st->peer[key].ptr[st->rank];
      }
      return st->alloc(bytes);
    };
    for (int g2 = 0; g2 < st->groups; ++g2) {
      const size_t gd = (size_t)st->gdim[(size_t)g2];
      st->X_shard.push_back(st->alloc((T / P) * gd * 2));
      st->X_full.push_back(peer_or_local("X" + std::to_string(g2), T * gd * 2));
      st->dX_part.push_back(st->alloc(T * gd * 2));
      st->dX_shard.push_back(st->alloc((T / P) * gd * 2));
      if (st->ce) st->peer["rsX" + std::to_string(g2)] = st->make_peer((size_t)P * (T / P) * gd * 2);
    }
    const size_t NPs = (size_t)st->NP;
    for (auto* v : {&st->H_shard, &st->H_full, &st->Y, &st->dY, &st->dH_part, &st->dH_shard, &st->X_loc,
                    &st->H_row, &st->Y_part, &st->Y_shard, &st->dY_shard, &st->dY_full, &st->dH_row,
                    &st->dX_loc})
      v->assign(NPs, nullptr);
    for (int32_t p = 0; p < st->NP; ++p) {
      const size_t Rp = (size_t)st->R[(size_t)p], dd = (size_t)st->d[(size_t)p], kk = (size_t)st->k[(size_t)p];
      const std::string id = std::to_string(p);
      if (!st->row[(size_t)p]) {
        st->H_shard[(size_t)p] = st->alloc((T / P) * Rp * 2);
        st->H_full[(size_t)p] = peer_or_local("H" + id, T * Rp * 2);
        st->Y[(size_t)p] = st->alloc(T * (kk / P) * 2);
        st->dY[(size_t)p] = st->alloc(T * (kk / P) * 2);
        st->dH_part[(size_t)p] = st->alloc(T * Rp * 2);
        st->dH_shard[(size_t)p] = st->alloc((T / P) * Rp * 2);
        if (st->ce) st->peer["rsH" + id] = st->make_peer((size_t)P * (T / P) * Rp * 2);
      } else {
        st->X_loc[(size_t)p] = st->alloc(T * (dd / P) * 2);
        st->H_row[(size_t)p] = st->alloc(T * Rp * 2);
        st->Y_shard[(size_t)p] = st->alloc((T / P) * kk * 2);
        st->dY_shard[(size_t)p] = st->alloc((T / P) * kk * 2);
        st->dY_full[(size_t)p] = peer_or_local("dY" + id, T * kk * 2);
        st->dH_row[(size_t)p] = st->alloc(T * Rp * 2);
        st->dX_loc[(size_t)p] = st->alloc(T * (dd / P) * 2);
        if (st->fused) {
          st->peer["recv" + id] = st->make_peer((size_t)P * (T / P) * kk * 2);
        } else {
          st->Y_part[(size_t)p] = st->alloc(T * kk * 2);
        }
      }
    }
    // epoch flags: the copy-engine collectives' completion and the fused reduce-scatter's
    // barriers
    if (st->ce || st->fused) st->flags = st->make_peer((size_t)P * 4);
    st->present = (int32_t*)st->alloc((size_t)st->S * 4);
    {
      std::vector<int32_t> pres((size_t)st->S);
      for (int32_t s = 0; s < st->S; ++s) pres[(size_t)s] = st->batch[(size_t)s] > 0;
      TP_CUDA(cudaMemcpy(st->present, pres.data(), (size_t)st->S * 4, cudaMemcpyHostToDevice));
    }
    TP_CUDA(cudaDeviceSynchronize());
    // every rank's flags are zero before any push
    chk(tlora_comm_all_reduce(comm, TLORA_GROUP_WORLD, st->ms_dev, st->ms_dev, 1, TLORA_F64, 0, st->main));
    TP_CUDA(cudaStreamSynchronize(st->main));
    *out = st.release();
  });
}

int tlora_tp_destroy(tlora_tp_step* step) {
  return tp_guard([&] {
    if (!step) return;
    DevGuard g(step->device);
    cudaDeviceSynchronize();
    delete step;
  });
}

int tlora_tp_layer(tlora_tp_step* step, int32_t proj, tlora_layer** out) {
  return tp_guard([&] {
    need(step && out, TLORA_ERR_ARG, "null argument");
    need(proj >= 0 && proj < step->NP, TLORA_ERR_ARG, "projection out of range");
    *out = step->layers[(size_t)proj];
  });
}

int tlora_tp_buffer(tlora_tp_step* step, int32_t kind, int32_t index, void** ptr, int64_t* rows,
                    int64_t* cols) {
  return tp_guard([&] {
    need(step && ptr, TLORA_ERR_ARG, "null argument");
    auto& s = *step;
    const int64_t T = s.T, P = s.P;
    const bool grp = kind == TLORA_TP_X_SHARD || kind == TLORA_TP_DX_SHARD;
    need(grp ? (index >= 0 && index < s.groups) : (index >= 0 && index < s.NP), TLORA_ERR_ARG,
         "index out of range");
    const bool want_row = kind == TLORA_TP_X_LOC || kind == TLORA_TP_DY_SHARD ||
                          kind == TLORA_TP_Y_SHARD || kind == TLORA_TP_DX_LOC;
    if (!grp) need((bool)s.row[(size_t)index] == want_row, TLORA_ERR_ARG,
                   "buffer kind does not match the projection's parallel mode");
    int64_t r = 0, c = 0;
    char* p = nullptr;
    switch (kind) {
      case TLORA_TP_X_SHARD: p = s.X_shard[(size_t)index]; r = T / P; c = s.gdim[(size_t)index]; break;
      case TLORA_TP_DX_SHARD: p = s.dX_shard[(size_t)index]; r = T / P; c = s.gdim[(size_t)index]; break;
      case TLORA_TP_X_LOC: p = s.X_loc[(size_t)index]; r = T; c = s.d[(size_t)index] / P; break;
      case TLORA_TP_DY: p = s.dY[(size_t)index]; r = T; c = s.k[(size_t)index] / P; break;
      case TLORA_TP_DY_SHARD: p = s.dY_shard[(size_t)index]; r = T / P; c = s.k[(size_t)index]; break;
      case TLORA_TP_Y: p = s.Y[(size_t)index]; r = T; c = s.k[(size_t)index] / P; break;
      case TLORA_TP_Y_SHARD: p = s.Y_shard[(size_t)index]; r = T / P; c = s.k[(size_t)index]; break;
      case TLORA_TP_DX_LOC: p = s.dX_loc[(size_t)index]; r = T; c = s.d[(size_t)index] / P; break;
      default: throw TpError(TLORA_ERR_ARG, "unknown buffer kind");
    }
    *ptr = p;
    if (rows) *rows = r;
    if (cols) *cols = c;
  });
}

int tlora_tp_trace(const tlora_tp_step* step, double* t_comp_ms, double* t_comm_ms, int32_t cap,
                   int32_t* count) {
  return tp_guard([&] {
    need(step != nullptr, TLORA_ERR_ARG, "step is null");
    const size_t n = step->trace_comp.size();
    if (count) *count = (int32_t)n;
    for (size_t i = 0; i < n && (int32_t)i < cap; ++i) {
      if (t_comp_ms) t_comp_ms[i] = step->trace_comp[i];
      if (t_comm_ms) t_comm_ms[i] = step->trace_comm[i];
    }
  });
}

int tlora_tp_layout(tlora_tp_step* step, int32_t n, int32_t* n_out, int64_t* nano_t0,
                    int32_t* nano_slot) {
  return tp_guard([&] {
    need(step != nullptr, TLORA_ERR_ARG, "step is null");
    need(n >= 1, TLORA_ERR_PLAN, "partition: N must be >= 1");
    DevGuard g(step->device);
    Layout& lo = step->layout(std::min(n, step->total_samples));
    if (n_out) *n_out = lo.map.n;
    if (nano_t0)
      for (size_t i = 0; i <= lo.nanos.size(); ++i)
        nano_t0[i] = i < lo.nanos.size() ? lo.nanos[i].t0 : step->T;
    if (nano_slot) std::memcpy(nano_slot, lo.map.nano_slot.data(), lo.map.nano_slot.size() * 4);
  });
}

int tlora_tp_run(tlora_tp_step* step, int32_t flags, void* stream, tlora_step_stats* stats) {
  return tp_guard([&] {
    need(step != nullptr, TLORA_ERR_ARG, "step is null");
    auto& st = *step;
    DevGuard g(st.device);
    cudaStream_t caller = reinterpret_cast<cudaStream_t>(stream);
    const int32_t n_use = st.desc.nano_fixed > 0 ? std::min(st.desc.nano_fixed, st.total_samples)
                                                 : st.aimd_n;
    using clk = std::chrono::steady_clock;
    const auto h0 = clk::now();
    Layout& lo = st.layout(n_use);
    st.tracing = (flags & TLORA_RUN_TRACE) != 0;
    st.marks.clear();
    // nothing needs this step's time now (a traced step waits for its events)
    static const bool force_sync = std::getenv("TLORA_TP_SYNC") != nullptr;  // A/B knob
    const bool lazy = st.desc.nano_fixed > 0 && !st.tracing && !force_sync;
    const int tslot = (int)(st.steps_run % tlora_tp_step::kTimeRing);
    cudaEvent_t t_begin = st.t_begin_r[tslot], t_end = st.t_end_r[tslot];
    st.ev_next = 0;
    st.wait(st.main, caller);
    const long long l0 = tlora_launch_count();
    TP_CUDA(cudaEventRecord(t_begin, st.main));
    const auto h1 = clk::now();
    st.forward(lo);
    const auto h2 = clk::now();
    st.backward(lo);
    for (auto* l : st.layers) chk(tlora_layer_optimizer_step_masked(l, st.present, 1.f, st.main));
    TP_CUDA(cudaEventRecord(t_end, st.main));
    st.wait(caller, st.main);
    st.t_step_r[tslot] = st.steps_run++;
    const auto h3 = clk::now();
    float ms = -1.f;
    if (!lazy) {
      TP_CUDA(cudaEventSynchronize(t_end));
      TP_CUDA(cudaEventElapsedTime(&ms, t_begin, t_end));
    } else {
      long long best = -1;
      for (int i = 0; i < tlora_tp_step::kTimeRing; ++i) {
        if (st.t_step_r[i] <= best || cudaEventQuery(st.t_end_r[i]) != cudaSuccess) continue;
        float t = 0.f;
        if (cudaEventElapsedTime(&t, st.t_begin_r[i], st.t_end_r[i]) == cudaSuccess) {
          best = st.t_step_r[i];
          ms = t;
        }
      }
      (void)cudaGetLastError();  // cudaErrorNotReady of the queries is not an error here
    }
    const auto h4 = clk::now();
    if (st.tracing) {  // spans per nano-batch: compute on main, boundary traffic on comm
      st.trace_comp.assign(lo.nanos.size(), 0.0);
      st.trace_comm.assign(lo.nanos.size(), 0.0);
      std::map<std::pair<int, int>, cudaEvent_t> open;
      for (const auto& m : st.marks) {
        const auto key = std::make_pair(m.kind, m.nano);
        if (m.edge == 0) {
          open[key] = m.ev;
          continue;
        }
        float t = 0.f;
        TP_CUDA(cudaEventElapsedTime(&t, open.at(key), m.ev));
        (m.kind == 0 ? st.trace_comp : st.trace_comm)[(size_t)m.nano] += t;
      }
      st.tracing = false;
    }
    if (!lazy) {
      // the group's mean step time: every rank feeds the same value to AIMD, so all ranks
      // take the same N next step
      double msd = ms;
      TP_CUDA(cudaMemcpyAsync(st.ms_dev, &msd, sizeof msd, cudaMemcpyHostToDevice, st.main));
      chk(tlora_comm_all_reduce(st.comm, TLORA_GROUP_WORLD, st.ms_dev, st.ms_dev, 1, TLORA_F64, 1,
                                st.main));
      TP_CUDA(cudaMemcpyAsync(&msd, st.ms_dev, sizeof msd, cudaMemcpyDeviceToHost, st.main));
      TP_CUDA(cudaStreamSynchronize(st.main));
      const int32_t alpha = st.desc.aimd_alpha ? st.desc.aimd_alpha : 4;
      const double beta = st.desc.aimd_beta != 0.0 ? st.desc.aimd_beta : 0.5;
      chk(tlora_aimd_step(&st.aimd_n, &st.has_prev, &st.t_prev, alpha, beta, st.desc.aimd_tau_rel,
                          msd / 1e3));
      st.aimd_n = std::min(st.aimd_n, st.total_samples);
    }
    if (std::getenv("TLORA_TP_DEBUG")) {
      auto ms_ = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
      // device idle time between the previous step's end and this step's begin (only
      // meaningful when the step synchronised: TLORA_TP_SYNC / AIMD)
      float gap = -1.f;
      if (!lazy && st.steps_run >= 2) {
        const int prev = (int)((st.steps_run - 2) % tlora_tp_step::kTimeRing);
        if (cudaEventElapsedTime(&gap, st.t_end_r[prev], t_begin) != cudaSuccess) gap = -1.f;
        (void)cudaGetLastError();
      }
      std::fprintf(stderr, "[tlora_tp rank %d] layout+wait %.3f fwd-enqueue %.3f bwd-enqueue %.3f "
                   "sync %.3f aimd %.3f device %.3f gap-before %.3f ms\n", st.rank, ms_(h0, h1),
                   ms_(h1, h2), ms_(h2, h3), ms_(h3, h4), ms_(h4, clk::now()), (double)ms,
                   (double)gap);
    }
    if (stats) {
      stats->nano_used = lo.map.n;
      stats->next_nano = st.desc.nano_fixed > 0 ? n_use : st.aimd_n;
      stats->ms = ms;
      stats->replayed_graph = 0;
      stats->launches = tlora_launch_count() - l0;
      stats->tokens = st.T;
    }
  });
}

}  // extern "C"
