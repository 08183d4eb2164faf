// trainer.hpp — persistent C++ objects over the C-ABI (include/tlora.h), next to the
// per-call reference drop-in of fused_lora.hpp.
//
// fused_forward(batch, W, adapters) (fused_lora.hpp:84-85) is pure: every call converts
// and uploads its operands. A training host keeps them resident instead:
//
//   FusedLayer        one adapted projection: W uploaded once (bf16, both K-major layouts),
//                     adapters / optimizer state resident; plans per batch; forward /
//                     backward / AdamW on device buffers the host owns.
//   LayerSetTrainer   the whole SSM layer set (ssm_plan.hpp fuse_projections: every
//                     (layer, projection) of a job group) as ONE training step executor
//                     (tlora_step_*): rank-aware nano-batches, AIMD on measured step times
//                     (the loop of sim_engine.hpp:306-315), chained fused GEMMs, side-
//                     stream gradients, fused masked AdamW, optional data-parallel
//                     all-reduce through a Communicator, CUDA-graph replay.
//
// Errors throw std::runtime_error (std::invalid_argument for plan / controller arguments,
// as nano_pipeline.hpp) with tlora_last_error()'s message.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../tlora.h"
#include "lora_fleet/comm.hpp"
#include "lora_fleet/ssm_plan.hpp"

namespace lora_fleet {

namespace detail {
inline void tl_throw(int code) {
  if (code == TLORA_OK) return;
  if (code == TLORA_ERR_PLAN) throw std::invalid_argument(tlora_last_error());
  throw std::runtime_error(std::string("tlora: ") + tlora_last_error());
}
}  // namespace detail

// ---------------------------------------------------------------- one resident layer
class FusedLayer {
 public:
  // ranks: registry layout in job_id order (registry_ranks(fuse(group))).
  FusedLayer(int device, long long d, long long k, const std::vector<int>& ranks) {
    std::vector<int32_t> r(ranks.begin(), ranks.end());
    detail::tl_throw(tlora_layer_create(device, d, k, (int32_t)r.size(), r.data(), &l_));
  }
  ~FusedLayer() {
    for (auto* p : plans_) tlora_plan_destroy(p);
    if (l_) tlora_layer_destroy(l_);
  }
  FusedLayer(const FusedLayer&) = delete;
  FusedLayer& operator=(const FusedLayer&) = delete;

  // W: d x k row-major, dtype TLORA_F64 / F32 / BF16, host or device (TLORA_HOST / DEVICE)
  void set_base(const void* W, int dtype, int where, void* stream = nullptr) {
    detail::tl_throw(tlora_layer_set_base(l_, W, dtype, where, stream));
  }
  void set_adapter(int slot, const void* A, const void* B, int dtype, int where,
                   void* stream = nullptr) {
    detail::tl_throw(tlora_layer_set_adapter(l_, slot, A, B, dtype, where, stream));
  }
  void set_optimizer(const std::vector<float>& lr, const std::vector<float>& weight_decay,
                     float beta1 = 0.9f, float beta2 = 0.999f, float eps = 1e-8f) {
    detail::tl_throw(tlora_layer_set_optimizer(l_, lr.data(), weight_decay.data(), beta1, beta2, eps));
  }
  // Plan of one batch (token -> slot, any interleaving); owned by the layer.
  tlora_plan* plan(const std::vector<int32_t>& token_slot) {
    tlora_plan* p = nullptr;
    detail::tl_throw(tlora_plan_create(l_, (int64_t)token_slot.size(), token_slot.data(), &p));
    plans_.push_back(p);
    return p;
  }
  // Device pointers, bf16 row-major: X T x d, Y T x k (y_dtype), H_stash T x R.
  void forward(const tlora_plan* p, const void* X, void* Y, int y_dtype, void* H_stash,
               void* stream = nullptr) {
    detail::tl_throw(tlora_forward(l_, p, X, Y, y_dtype, H_stash, stream));
  }
  void backward(const tlora_plan* p, const void* dY, const void* X, const void* H_stash,
                void* dX, float beta = 0.f, void* stream = nullptr) {
    detail::tl_throw(tlora_backward(l_, p, dY, X, H_stash, dX, beta, stream));
  }
  void optimizer_step(const tlora_plan* present_from = nullptr, float grad_scale = 1.f,
                      void* stream = nullptr) {
    const int32_t* mask = nullptr;
    if (present_from) detail::tl_throw(tlora_plan_present_mask(present_from, &mask));
    detail::tl_throw(tlora_layer_optimizer_step_masked(l_, mask, grad_scale, stream));
  }
  int rank_pad_total() const {
    int32_t R = 0;
    detail::tl_throw(tlora_layer_layout(l_, nullptr, &R));
    return R;
  }
  tlora_layer* handle() const { return l_; }

 private:
  tlora_layer* l_ = nullptr;
  std::vector<tlora_plan*> plans_;
};

// ---------------------------------------------------------------- the layer-set executor
struct TrainerOptions {
  int device = 0;
  int nano_init = 4;        // AimdState::n default (nano_pipeline.hpp:37)
  int nano_fixed = 0;       // > 0: fixed N (config.fixed_n), no AIMD
  int aimd_alpha = 4;
  double aimd_beta = 0.5;
  double aimd_tau_rel = 0.0;
  bool side_grads = true;
  bool graphs = true;
  int dh_ring = 8;
  int input_sets = 1;
  int y_dtype = TLORA_BF16;
};

class LayerSetTrainer {
 public:
  // layer_set: fuse_projections(group, projections); every job of the group runs
  // batch_size samples of seq_len tokens per step. input_group[p]: projections with the same
  // id read the same activation (e.g. q/k/v); empty = one input per projection.
  LayerSetTrainer(const SsmLayerSet& layer_set, const TrainerOptions& opt,
                  std::vector<int32_t> input_group = {}, Communicator* comm = nullptr)
      : P_((int)layer_set.projections.size()), L_(layer_set.graph.model.num_layers) {
    std::vector<int64_t> d, k;
    for (const auto& p : layer_set.projections) {
      d.push_back(p.d);
      k.push_back(p.k);
    }
    if (input_group.empty())
      for (int p = 0; p < P_; ++p) input_group.push_back(p);
    std::vector<int32_t> ranks, batch, seq;
    for (const auto& j : layer_set.graph.jobs) {
      ranks.push_back(j.rank);
      batch.push_back(j.batch_size);
      seq.push_back(j.seq_len);
    }
    tlora_step_desc desc{};
    desc.device = opt.device;
    desc.num_layers = L_;
    desc.num_projections = P_;
    desc.proj_d = d.data();
    desc.proj_k = k.data();
    desc.proj_input = input_group.data();
    desc.num_slots = (int32_t)ranks.size();
    desc.ranks = ranks.data();
    desc.batch = batch.data();
    desc.seq_len = seq.data();
    desc.y_dtype = opt.y_dtype;
    desc.flags = (opt.side_grads ? TLORA_STEP_SIDE_GRADS : 0) | (opt.graphs ? TLORA_STEP_GRAPH : 0);
    desc.dh_ring = opt.dh_ring;
    desc.input_sets = opt.input_sets;
    desc.nano_init = opt.nano_init;
    desc.nano_fixed = opt.nano_fixed;
    desc.aimd_alpha = opt.aimd_alpha;
    desc.aimd_beta = opt.aimd_beta;
    desc.aimd_tau_rel = opt.aimd_tau_rel;
    detail::tl_throw(tlora_step_create(&desc, comm ? comm->handle() : nullptr, &s_));
  }
  ~LayerSetTrainer() {
    if (s_) tlora_step_destroy(s_);
  }
  LayerSetTrainer(const LayerSetTrainer&) = delete;
  LayerSetTrainer& operator=(const LayerSetTrainer&) = delete;

  int layers() const { return L_; }
  int projections() const { return P_; }
  tlora_layer* layer(int layer, int proj) const {
    tlora_layer* l = nullptr;
    detail::tl_throw(tlora_step_layer(s_, layer, proj, &l));
    return l;
  }
  struct Buffer {
    void* ptr = nullptr;
    int64_t rows = 0, cols = 0;
  };
  Buffer buffer(int kind, int index, int set = 0) const {
    Buffer b;
    detail::tl_throw(tlora_step_buffer(s_, kind, index, set, &b.ptr, &b.rows, &b.cols));
    return b;
  }
  int next_n() const {
    int32_t n = 0;
    detail::tl_throw(tlora_step_next_n(s_, &n));
    return n;
  }
  // One training step (blocks until its CUDA-event time is known; the controller then
  // picks the next N).
  tlora_step_stats step(int set = 0, void* stream = nullptr, bool eager = false) {
    tlora_step_stats st{};
    detail::tl_throw(tlora_step_run(s_, set, eager ? TLORA_RUN_EAGER : 0, stream, &st));
    return st;
  }
  tlora_step* handle() const { return s_; }

 private:
  int P_, L_;
  tlora_step* s_ = nullptr;
};

}  // namespace lora_fleet
