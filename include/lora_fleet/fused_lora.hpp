// fused_lora.hpp — drop-in for the reference's fused multi-LoRA operator API.
//
// Same types, function names, argument meaning, ordering and error behaviour as
// proj/include/lora_fleet/fused_lora.hpp (reference), but the arithmetic runs in the
// sm_100a kernels of libtlora.so through the C-ABI in include/tlora.h:
//   fused_forward            fused_lora.hpp:84-119  -> tlora_forward   (+ new fused_backward)
//   unfused_cost             fused_lora.hpp:139-163 -> tlora_op_cost
//   trainable_param_count    fused_lora.hpp:166-170
//   adapter_flops_per_token  fused_lora.hpp:173-176
//   materialized_oracle      fused_lora.hpp:124-135 — the reference's TEST oracle; only
//                            compiled with -DLORA_FLEET_WITH_TEST_ORACLE (tests), never
//                            on the product path.
// Shape and registry errors are thrown as std::runtime_error with the reference's
// messages (fused_lora.hpp:66-76) before anything touches the device. There is no CPU
// fallback: without an sm_100 GPU the compute calls throw.
//
// Numerics: operands are rounded to bf16, accumulation is fp32, Y is returned from an
// fp32 epilogue (see DESIGN.md §Numerics for the tolerances the tests state).
#pragma once
#include <cstdint>
#include <cstdlib>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../tlora.h"
#include "lora_fleet/matrix.hpp"
#include "lora_fleet/workload.hpp"

namespace lora_fleet {

struct AdapterMatrices {
  std::string job_id;
  Matrix A;  // d x r, down-projection
  Matrix B;  // r x k, up-projection
};

struct TokenBatch {
  Matrix rows;                           // total_tokens x d
  std::vector<std::string> segment_map;  // owning job_id per row, any interleaving
};

struct OpCost {
  double flops = 0.0;
  double bytes_moved = 0.0;
  long long kernel_launches = 0;

  OpCost& operator+=(const OpCost& o) {
    flops += o.flops;
    bytes_moved += o.bytes_moved;
    kernel_launches += o.kernel_launches;
    return *this;
  }
};

// Gradients of L = <dY, Y> (new; the reference has no backward).
struct FusedGradients {
  Matrix dX;                            // total_tokens x d
  std::map<std::string, Matrix> dA;     // job_id -> d x r
  std::map<std::string, Matrix> dB;     // job_id -> r x k
};

namespace detail {

// std::map by job_id; a duplicate id keeps the LAST entry (fused_lora.hpp:48-53).
inline std::map<std::string, const AdapterMatrices*> index_adapters(
    const std::vector<AdapterMatrices>& adapters) {
  std::map<std::string, const AdapterMatrices*> by_id;
  for (const auto& a : adapters) by_id[a.job_id] = &a;
  return by_id;
}

// Ascending rows of `batch` owned by job_id (fused_lora.hpp:56-61).
inline std::vector<Index> segment_rows(const TokenBatch& batch, const std::string& job_id) {
  std::vector<Index> idx;
  for (Index t = 0; t < batch.rows.rows(); ++t)
    if (batch.segment_map[static_cast<size_t>(t)] == job_id) idx.push_back(t);
  return idx;
}

// Validation with the reference's messages (fused_lora.hpp:63-78). Only adapters that
// some token references are shape-checked, as in the reference.
inline void check_shapes(const TokenBatch& batch, const Matrix& base_weight,
                         const std::map<std::string, const AdapterMatrices*>& by_id) {
  const auto d = batch.rows.cols();
  if (base_weight.rows() != d)
    throw std::runtime_error("fused_lora: base weight rows != token dim d");
  if (static_cast<Index>(batch.segment_map.size()) != batch.rows.rows())
    throw std::runtime_error("fused_lora: segment_map length != token count");
  for (const auto& id : batch.segment_map) {
    auto it = by_id.find(id);
    if (it == by_id.end())
      throw std::runtime_error("fused_lora: segment '" + id + "' has no adapter");
    const auto& a = *it->second;
    if (a.A.rows() != d || a.A.cols() != a.B.rows() || a.B.cols() != base_weight.cols())
      throw std::runtime_error("fused_lora: shape mismatch in segment '" + id + "'");
  }
}

inline void tl_check(int code) {
  if (code != TLORA_OK) throw std::runtime_error(std::string("tlora: ") + tlora_last_error());
}

inline int device_index() {
  const char* e = std::getenv("TLORA_DEVICE");
  return e ? std::atoi(e) : 0;
}

inline Index round8(Index n) { return (n + 7) / 8 * 8; }

// Row-major, zero-padded copy of an m x n Matrix into rows x cols (f64).
inline std::vector<double> padded(const Matrix& m, Index rows, Index cols) {
  std::vector<double> v(static_cast<size_t>(rows * cols), 0.0);
  for (Index i = 0; i < m.rows(); ++i)
    for (Index j = 0; j < m.cols(); ++j) v[static_cast<size_t>(i * cols + j)] = m(i, j);
  return v;
}

// Row-major, zero-padded copy with rows gathered through perm: out row i = m.row(perm[i]).
inline std::vector<double> padded_rows(const Matrix& m, const std::vector<int64_t>& perm,
                                       Index cols) {
  std::vector<double> v(perm.size() * static_cast<size_t>(cols), 0.0);
  for (size_t i = 0; i < perm.size(); ++i)
    for (Index j = 0; j < m.cols(); ++j)
      v[i * static_cast<size_t>(cols) + static_cast<size_t>(j)] = m(static_cast<Index>(perm[i]), j);
  return v;
}

// RAII device buffer through the C-ABI.
struct DeviceBuffer {
  int dev = 0;
  void* p = nullptr;
  DeviceBuffer(int d, size_t bytes) : dev(d) { tl_check(tlora_buffer_alloc(d, bytes, &p)); }
  ~DeviceBuffer() { tlora_buffer_free(dev, p); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
};

// One fused layer built from the reference-style inputs: registry (slots in std::map
// order), padded bf16 device copies, and the plan of this batch. Only adapters that some
// token references are registered — the same set check_shapes validates (fused_lora.hpp:
// 70-77) and fused_forward reads (:104 skips jobs without rows) — so an unreferenced
// adapter of any shape is never touched. A referenced rank-0 adapter (A d x 0, B 0 x k:
// its delta is exactly zero) is registered as a zero rank-1 adapter. The batch is laid
// out on the device job-sorted (tlora_segments: the CSR form of segment_rows for every
// job, rows ascending within a job), gathered during the host-side conversion at no extra
// cost, so arbitrarily interleaved segment maps (test_fused_lora.cpp:45-46) run as
// job-contiguous tiles; results are scattered back to the caller's row order.
class DeviceLayer {
 public:
  DeviceLayer(const TokenBatch& batch, const Matrix& W,
              const std::map<std::string, const AdapterMatrices*>& by_id)
      : dev_(device_index()),
        T_(batch.rows.rows()),
        d_(batch.rows.cols()),
        k_(W.cols()),
        dp_(round8(d_)),
        kp_(round8(k_)) {
    std::map<std::string, int32_t> slot_of;
    for (const auto& id : batch.segment_map) slot_of.emplace(id, 0);
    std::vector<int32_t> ranks;
    for (auto& [id, slot] : slot_of) {  // std::map order of the referenced ids
      slot = static_cast<int32_t>(ranks.size());
      const Index r = by_id.at(id)->A.cols();
      ids_.push_back(id);
      true_rank_.push_back(r);
      ranks.push_back(static_cast<int32_t>(r > 0 ? r : 1));
    }
    tl_check(tlora_layer_create(dev_, dp_, kp_, static_cast<int32_t>(ranks.size()), ranks.data(),
                                &layer_));
    const auto wp = padded(W, dp_, kp_);
    tl_check(tlora_layer_set_base(layer_, wp.data(), TLORA_F64, TLORA_HOST, nullptr));
    for (size_t s = 0; s < ids_.size(); ++s) {
      const AdapterMatrices& a = *by_id.at(ids_[s]);
      const Index r = ranks[s];
      // rank 0: zero d x 1 / 1 x k (padded() of an empty matrix is all zeros)
      const auto ap = padded(a.A, dp_, r);
      const auto bp = padded(a.B, r, kp_);
      tl_check(tlora_layer_set_adapter(layer_, static_cast<int32_t>(s), ap.data(), bp.data(),
                                       TLORA_F64, TLORA_HOST, nullptr));
    }
    tl_check(tlora_layer_layout(layer_, nullptr, &R_));
    std::vector<int32_t> slots(static_cast<size_t>(T_));
    for (Index t = 0; t < T_; ++t) slots[static_cast<size_t>(t)] = slot_of.at(batch.segment_map[t]);
    perm_.resize(static_cast<size_t>(T_));
    std::vector<int64_t> offsets(ranks.size() + 1);
    tl_check(tlora_segments(T_, slots.data(), static_cast<int32_t>(ranks.size()), perm_.data(),
                            offsets.data()));
    std::vector<int32_t> sorted(static_cast<size_t>(T_));
    for (size_t i = 0; i < perm_.size(); ++i) sorted[i] = slots[static_cast<size_t>(perm_[i])];
    tl_check(tlora_plan_create(layer_, T_, sorted.data(), &plan_));
    X_ = std::make_unique<DeviceBuffer>(dev_, static_cast<size_t>(T_ * dp_ * 2));
    H_ = std::make_unique<DeviceBuffer>(dev_, static_cast<size_t>(T_ * R_ * 2));
    const auto xp = padded_rows(batch.rows, perm_, dp_);
    tl_check(tlora_copy_to_device(X_->p, TLORA_BF16, xp.data(), TLORA_F64, T_ * dp_, nullptr));
  }
  ~DeviceLayer() {
    tlora_plan_destroy(plan_);
    tlora_layer_destroy(layer_);
  }

  Matrix forward() {
    DeviceBuffer Y(dev_, static_cast<size_t>(T_ * kp_ * 4));
    tl_check(tlora_forward(layer_, plan_, X_->p, Y.p, TLORA_F32, H_->p, nullptr));
    std::vector<double> y(static_cast<size_t>(T_ * kp_));
    tl_check(tlora_copy_to_host(y.data(), TLORA_F64, Y.p, TLORA_F32, T_ * kp_, nullptr));
    Matrix out(T_, k_);
    for (Index i = 0; i < T_; ++i)
      for (Index j = 0; j < k_; ++j)
        out(static_cast<Index>(perm_[static_cast<size_t>(i)]), j) = y[static_cast<size_t>(i * kp_ + j)];
    return out;
  }

  // Gradients of the referenced adapters (the others get zeros from fused_backward).
  FusedGradients backward(const Matrix& dY) {
    DeviceBuffer g(dev_, static_cast<size_t>(T_ * kp_ * 2));
    DeviceBuffer dX(dev_, static_cast<size_t>(T_ * dp_ * 2));
    const auto gp = padded_rows(dY, perm_, kp_);
    tl_check(tlora_copy_to_device(g.p, TLORA_BF16, gp.data(), TLORA_F64, T_ * kp_, nullptr));
    tl_check(tlora_backward(layer_, plan_, g.p, X_->p, H_->p, dX.p, 0.0f, nullptr));
    FusedGradients out;
    std::vector<double> dx(static_cast<size_t>(T_ * dp_));
    tl_check(tlora_copy_to_host(dx.data(), TLORA_F64, dX.p, TLORA_BF16, T_ * dp_, nullptr));
    out.dX = Matrix(T_, d_);
    for (Index i = 0; i < T_; ++i)
      for (Index j = 0; j < d_; ++j)
        out.dX(static_cast<Index>(perm_[static_cast<size_t>(i)]), j) = dx[static_cast<size_t>(i * dp_ + j)];
    for (size_t s = 0; s < ids_.size(); ++s) {
      const auto& id = ids_[s];
      const Index r = true_rank_[s];
      const Index rr = r > 0 ? r : 1;
      std::vector<float> da(static_cast<size_t>(dp_ * rr)), db(static_cast<size_t>(rr * kp_));
      tl_check(tlora_layer_read_grad(layer_, static_cast<int32_t>(s), da.data(), db.data(),
                                     TLORA_HOST, nullptr));
      Matrix A(d_, r), B(r, k_);
      for (Index i = 0; i < d_; ++i)
        for (Index j = 0; j < r; ++j) A(i, j) = da[static_cast<size_t>(i * rr + j)];
      for (Index i = 0; i < r; ++i)
        for (Index j = 0; j < k_; ++j) B(i, j) = db[static_cast<size_t>(i * kp_ + j)];
      out.dA[id] = std::move(A);
      out.dB[id] = std::move(B);
    }
    return out;
  }

 private:
  int dev_;
  Index T_, d_, k_, dp_, kp_;
  int32_t R_ = 0;
  tlora_layer* layer_ = nullptr;
  tlora_plan* plan_ = nullptr;
  std::vector<std::string> ids_;   // referenced job ids, std::map order (= slot order)
  std::vector<Index> true_rank_;   // their ranks (0 allowed)
  std::vector<int64_t> perm_;      // device row i holds the caller's token perm_[i]
  std::unique_ptr<DeviceBuffer> X_, H_;
};

inline std::unique_ptr<DeviceLayer> make_device_layer(
    const TokenBatch& batch, const Matrix& W,
    const std::map<std::string, const AdapterMatrices*>& by_id) {
  return std::make_unique<DeviceLayer>(batch, W, by_id);
}

}  // namespace detail

// Y[t] = X[t]·W + X[t]·A_i·B_i for t's owning job i (fused_lora.hpp:82-119): one shared
// base GEMM with the low-rank expand fused as a K-extension, on the GPU. The returned
// OpCost is the reference's analytic model, bit-identical (tlora_op_cost).
inline std::pair<Matrix, OpCost> fused_forward(const TokenBatch& batch, const Matrix& base_weight,
                                               const std::vector<AdapterMatrices>& adapters) {
  auto by_id = detail::index_adapters(adapters);
  detail::check_shapes(batch, base_weight, by_id);
  std::vector<int64_t> tokens;
  std::vector<int32_t> ranks;
  for (const auto& [id, a] : by_id) {
    tokens.push_back(static_cast<int64_t>(detail::segment_rows(batch, id).size()));
    ranks.push_back(static_cast<int32_t>(a->A.cols()));
  }
  OpCost cost;
  detail::tl_check(tlora_op_cost(batch.rows.rows(), batch.rows.cols(), base_weight.cols(),
                                 static_cast<int32_t>(ranks.size()), tokens.data(), ranks.data(),
                                 1, &cost.flops, &cost.bytes_moved, &cost.kernel_launches));
  if (batch.rows.rows() == 0) return {Matrix(0, base_weight.cols()), cost};
  auto L = detail::make_device_layer(batch, base_weight, by_id);
  return {L->forward(), cost};
}

// Backward of fused_forward for upstream gradient dY (new; SPEC.md:146 has none).
inline FusedGradients fused_backward(const TokenBatch& batch, const Matrix& base_weight,
                                     const std::vector<AdapterMatrices>& adapters,
                                     const Matrix& dY) {
  auto by_id = detail::index_adapters(adapters);
  detail::check_shapes(batch, base_weight, by_id);
  if (dY.rows() != batch.rows.rows() || dY.cols() != base_weight.cols())
    throw std::runtime_error("fused_lora: upstream gradient shape != token count x k");
  if (batch.rows.rows() == 0) {
    FusedGradients out;
    out.dX = Matrix(0, batch.rows.cols());
    for (const auto& [id, a] : by_id) {
      out.dA[id] = Matrix::Zero(a->A.rows(), a->A.cols());
      out.dB[id] = Matrix::Zero(a->B.rows(), a->B.cols());
    }
    return out;
  }
  auto L = detail::make_device_layer(batch, base_weight, by_id);
  L->forward();
  FusedGradients out = L->backward(dY);
  // adapters no token references have zero gradients (shaped like the adapter itself)
  for (const auto& [id, a] : by_id)
    if (!out.dA.count(id)) {
      out.dA[id] = Matrix::Zero(a->A.rows(), a->A.cols());
      out.dB[id] = Matrix::Zero(a->B.rows(), a->B.cols());
    }
  return out;
}

// Unfused accounting (fused_lora.hpp:137-163), via the bit-identical C-ABI restatement.
inline OpCost unfused_cost(const TokenBatch& batch, const Matrix& base_weight,
                           const std::vector<AdapterMatrices>& adapters) {
  auto by_id = detail::index_adapters(adapters);
  detail::check_shapes(batch, base_weight, by_id);
  std::vector<int64_t> tokens;
  std::vector<int32_t> ranks;
  for (const auto& [id, a] : by_id) {
    tokens.push_back(static_cast<int64_t>(detail::segment_rows(batch, id).size()));
    ranks.push_back(static_cast<int32_t>(a->A.cols()));
  }
  OpCost cost;
  detail::tl_check(tlora_op_cost(batch.rows.rows(), batch.rows.cols(), base_weight.cols(),
                                 static_cast<int32_t>(ranks.size()), tokens.data(), ranks.data(),
                                 0, &cost.flops, &cost.bytes_moved, &cost.kernel_launches));
  return cost;
}

// r·(d + k) trainable parameters per adapted layer (fused_lora.hpp:165-170).
inline long long trainable_param_count(const JobSpec& job) {
  job.validate();
  return static_cast<long long>(job.rank) * (job.model.hidden_dim + job.model.proj_dim) *
         job.model.num_layers;
}

// Forward adapter FLOPs per token per adapted layer (fused_lora.hpp:172-176).
inline double adapter_flops_per_token(const JobSpec& job) {
  return 2.0 * static_cast<double>(job.rank) *
         static_cast<double>(job.model.hidden_dim + job.model.proj_dim);
}

#ifdef LORA_FLEET_WITH_TEST_ORACLE
// TEST ORACLE ONLY (fused_lora.hpp:121-135): materialises W_i = W + A_i·B_i on the host.
inline Matrix materialized_oracle(const TokenBatch& batch, const Matrix& base_weight,
                                  const std::vector<AdapterMatrices>& adapters) {
  auto by_id = detail::index_adapters(adapters);
  detail::check_shapes(batch, base_weight, by_id);
  Matrix out(batch.rows.rows(), base_weight.cols());
  for (const auto& [id, adapter] : by_id) {
    Matrix w_i = base_weight + adapter->A * adapter->B;
    for (auto t : detail::segment_rows(batch, id)) out.row(t) = batch.rows.row(t) * w_i;
  }
  return out;
}
#endif

}  // namespace lora_fleet
