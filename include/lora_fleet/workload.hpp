// workload.hpp — job / model registry types of the drop-in API.
//
// Same fields, defaults and invariants as the reference's registry entries
// (proj/include/lora_fleet/workload.hpp:23-63): the fused layer reads job_id, rank,
// batch_size, seq_len and the model's hidden_dim (d) / proj_dim (k). Trace I/O and the
// synthetic trace generator (workload.hpp:65-258) are out of scope (simulator plumbing).
#pragma once
#include <algorithm>
#include <optional>
#include <stdexcept>
#include <string>

namespace lora_fleet {

struct ModelSpec {
  std::string name;
  int num_layers = 1;
  long long hidden_dim = 1;  // d
  long long proj_dim = 1;    // k
  double per_layer_flops_per_token = 0.0;
  double base_memory_bytes = 0.0;

  void validate() const {
    if (num_layers < 1) throw std::invalid_argument("ModelSpec: num_layers must be >= 1");
    if (hidden_dim < 1 || proj_dim < 1)
      throw std::invalid_argument("ModelSpec: hidden_dim and proj_dim must be >= 1");
    if (!(base_memory_bytes > 0.0))
      throw std::invalid_argument("ModelSpec: base_memory_bytes must be > 0");
  }
};

struct JobSpec {
  std::string job_id;
  ModelSpec model;
  int rank = 1;
  int batch_size = 1;
  int seq_len = 512;
  long long step_budget = 1;
  int gpu_demand = 1;
  double submit_time = 0.0;
  double max_slowdown = 1.25;
  std::optional<double> deadline;

  void validate() const {
    model.validate();
    auto bad = [this](const char* what) {
      return std::invalid_argument("JobSpec " + job_id + ": " + what);
    };
    if (rank < 1) throw bad("rank must be >= 1");
    if (rank > std::min(model.hidden_dim, model.proj_dim)) throw bad("rank exceeds min(d, k)");
    if (batch_size < 1) throw bad("batch_size must be >= 1");
    if (gpu_demand < 1) throw bad("gpu_demand must be >= 1");
    if (step_budget < 1) throw bad("step_budget must be >= 1");
    if (max_slowdown < 1.0) throw bad("max_slowdown must be >= 1");
  }
};

}  // namespace lora_fleet
