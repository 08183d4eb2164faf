// hardware.hpp — the reference's HardwareSpec (proj/include/lora_fleet/hardware.hpp:7-25),
// same fields, defaults and validate(), plus the MEASURED B200 cost profile that replaces
// its analytic constants for the fused multi-LoRA layer.
//
// The reference planner prices a layer as flops / gpu_flops plus kernel_launch_overhead per
// nano-batch (ssm_plan.hpp:115-125, cost_model.hpp:45-49, nano_pipeline.hpp:79). On B200
// those constants come from timing the real kernels: tools/cost_profile.py runs fwd + bwd
// + AdamW of one fused layer over a grid of shapes and fits (model v2)
//
//   step_s = fixed_overhead                      (the layer's launches, fixed part)
//          + gemm_flops / F                       (fwd + dX fused GEMMs, tensor-bound)
//          + lowrank_bytes / BW                   (shrink, dH, dB+dA, HBM-bound)
//          + optimizer_bytes / optimizer_BW       (fused AdamW, HBM-bound)
//
// into profiles/b200_cost_profile.json. CostProfile::load reads it; b200_hardware_spec()
// is the HardwareSpec a reference planner should run with; predict_step_seconds() is the
// per-projection prediction (tests/test_gpu_cost_model.py checks it against measured C5
// cells, tests/test_cost_model.py against the fit's own grid).
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace lora_fleet {

struct HardwareSpec {
  double gpu_flops = 1e13;              // flops/s per GPU
  double gpu_memory = 4e10;             // bytes per GPU
  double intra_node_bw = 1e11;          // bytes/s across GPUs in a node
  double inter_node_bw = 5e8;           // bytes/s across nodes
  double weight_stream_bw = 3e10;       // bytes/s, per-GPU weight streaming
  int gpus_per_node = 8;
  double kernel_launch_overhead = 0.2;  // seconds per nano-batch
  double activation_bytes = 2.0;        // bytes per activation value
  double backward_multiplier = 3.0;     // total flops = fwd * this

  void validate() const {
    if (gpu_flops <= 0 || gpu_memory <= 0 || intra_node_bw <= 0 || inter_node_bw <= 0 ||
        weight_stream_bw <= 0 || gpus_per_node < 1 || kernel_launch_overhead < 0)
      throw std::invalid_argument("HardwareSpec: all rates must be positive");
    if (intra_node_bw < inter_node_bw)
      throw std::invalid_argument("HardwareSpec: intra_node_bw must be >= inter_node_bw");
  }
};

// Fitted coefficients of profiles/b200_cost_profile.json (model_version 2).
struct CostProfile {
  double F = 0.0;               // F_flops_per_s
  double BW = 0.0;              // BW_bytes_per_s
  double optimizer_BW = 0.0;    // optimizer_BW_bytes_per_s
  double fixed_overhead = 0.0;  // fixed_overhead_s
  double fit_rel_err_median = 0.0;

  // Minimal reader: the file is the flat JSON tools/cost_profile.py writes; only these
  // top-level numbers are needed (the first occurrence of each key is the top-level one).
  static CostProfile load(const std::string& path) {
    std::ifstream f(path);
    if (!f) throw std::runtime_error("cost profile not found: " + path);
    std::stringstream ss;
    ss << f.rdbuf();
    const std::string text = ss.str();
    auto num = [&](const char* key) {
      const std::string k = std::string("\"") + key + "\"";
      const size_t at = text.find(k);
      if (at == std::string::npos) throw std::runtime_error(std::string("cost profile lacks ") + key);
      const size_t colon = text.find(':', at + k.size());
      return std::stod(text.substr(colon + 1));
    };
    if (num("model_version") != 2.0) throw std::runtime_error("cost profile: need model_version 2");
    CostProfile p;
    p.F = num("F_flops_per_s");
    p.BW = num("BW_bytes_per_s");
    p.optimizer_BW = num("optimizer_BW_bytes_per_s");
    p.fixed_overhead = num("fixed_overhead_s");
    p.fit_rel_err_median = num("fit_rel_err_median");
    if (!(p.F > 0 && p.BW > 0 && p.optimizer_BW > 0))
      throw std::runtime_error("cost profile: non-positive rates");
    return p;
  }
};

// The workload terms of one fused projection (d -> k) over a job-contiguous batch; ranks and
// tokens in registry (job_id) order. Packed rank width R = sum round_up(r, 8) (the device
// layout).
struct ProjectionWork {
  double gemm_flops = 0.0;       // fwd (X·W + H·B) + dX (dY·Wᵀ + dH·Aᵀ)
  double lowrank_bytes = 0.0;    // X, dY read by shrink / dH / dA / dB; H, dH written + read
  double optimizer_bytes = 0.0;  // 32 B per packed trainable parameter
};

inline ProjectionWork projection_work(long long d, long long k, const std::vector<int>& ranks,
                                      const std::vector<long long>& tokens) {
  if (ranks.size() != tokens.size()) throw std::invalid_argument("ranks / tokens size mismatch");
  double T = 0.0, tok_rank = 0.0, R = 0.0;
  for (size_t s = 0; s < ranks.size(); ++s) {
    T += (double)tokens[s];
    tok_rank += (double)tokens[s] * ranks[s];
    R += (double)((ranks[s] + 7) / 8 * 8);
  }
  ProjectionWork w;
  w.gemm_flops = 4.0 * T * d * k + 2.0 * tok_rank * (double)(d + k);
  w.lowrank_bytes = 2.0 * (2.0 * T * d + 2.0 * T * k + 4.0 * T * R) + 4.0 * R * (double)(d + k);
  w.optimizer_bytes = 32.0 * R * (double)(d + k);
  return w;
}

// Predicted device seconds of one training step (fwd + bwd + fused AdamW) of one projection.
inline double predict_step_seconds(const CostProfile& p, const ProjectionWork& w) {
  return p.fixed_overhead + w.gemm_flops / p.F + w.lowrank_bytes / p.BW +
         w.optimizer_bytes / p.optimizer_BW;
}

// The HardwareSpec a reference planner runs with on one 8x B200 node: gpu_flops = the
// sustained fused-GEMM rate, kernel_launch_overhead = the measured fixed cost of one fused
// layer's training step (charged per nano-batch, nano_pipeline.hpp:79), weight_stream_bw =
// the low-rank launches' effective HBM rate,
// intra-node = NVLink 5 (900 GB/s per direction), 180 GB of HBM3e, bf16 activations, and
// backward = 2x forward (the base is frozen: dX but no dW; the LoRA terms are < 3% here).
inline HardwareSpec b200_hardware_spec(const CostProfile& p) {
  HardwareSpec h;
  h.gpu_flops = p.F;
  h.gpu_memory = 180e9;
  h.intra_node_bw = 900e9;
  h.weight_stream_bw = p.BW;
  h.gpus_per_node = 8;
  h.kernel_launch_overhead = std::max(0.0, p.fixed_overhead);
  h.activation_bytes = 2.0;
  h.backward_multiplier = 2.0;
  h.validate();
  return h;
}

}  // namespace lora_fleet
