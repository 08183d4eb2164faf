// nano_pipeline.hpp — nano-batch plan + AIMD controller of the drop-in API.
//
// partition / aimd_step go through the C-ABI (tlora_partition / tlora_aimd_step), which
// restates proj/include/lora_fleet/nano_pipeline.hpp:51-60 and :99-112 bit-exactly; the
// exceptions (std::invalid_argument) and messages are the reference's. monitor() is the
// reference formula (:119-126) applied to MEASURED per-nano times (CUDA events) instead
// of the simulator's modelled ones. The analytic simulate_iteration (:65-95) is replaced
// by real streams and is not part of this API (see DESIGN.md §Out of scope).
#pragma once
#include <numeric>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../tlora.h"

namespace lora_fleet {

struct NanoSchedule {
  int n = 1;
  std::vector<int> per_nano_samples;
};

struct PipelineTrace {
  std::vector<double> t_comp;  // per nano
  std::vector<double> t_comm;  // per nano
  double t_iter_event = 0.0;
  double t_iter_analytic = 0.0;
  int num_stages = 1;
};

struct AimdState {
  int n = 4;
  std::optional<double> t_prev;
  int alpha = 4;
  double beta = 0.5;
  double tau_rel = 0.0;

  void validate() const {
    if (n < 1 || alpha < 1 || beta <= 0.0 || beta >= 1.0 || tau_rel < 0.0)
      throw std::invalid_argument("AimdState: invalid controller parameters");
  }
};

inline NanoSchedule partition(int group_batch, int n) {
  if (group_batch < 1) throw std::invalid_argument("partition: group_batch must be >= 1");
  if (n < 1) throw std::invalid_argument("partition: N must be >= 1");
  NanoSchedule s;
  int32_t out_n = 0;
  std::vector<int32_t> per(static_cast<size_t>(std::min(n, group_batch)));
  if (tlora_partition(group_batch, n, &out_n, per.data()) != TLORA_OK)
    throw std::invalid_argument(tlora_last_error());
  s.n = out_n;
  s.per_nano_samples.assign(per.begin(), per.begin() + out_n);
  return s;
}

inline AimdState aimd_step(const AimdState& state, double t_t) {
  state.validate();
  if (t_t < 0.0) throw std::invalid_argument("aimd_step: negative iteration time");
  AimdState next = state;
  int32_t n = state.n, has_prev = state.t_prev.has_value() ? 1 : 0;
  double t_prev = state.t_prev.value_or(0.0);
  if (tlora_aimd_step(&n, &has_prev, &t_prev, state.alpha, state.beta, state.tau_rel, t_t) !=
      TLORA_OK)
    throw std::invalid_argument(tlora_last_error());
  next.n = n;
  next.t_prev = t_prev;
  return next;
}

struct MonitorReading {
  double eta_util = 0.0;
  double delta_stall = 0.0;
};

inline MonitorReading monitor(const PipelineTrace& trace) {
  MonitorReading r;
  const double sum_c = std::accumulate(trace.t_comp.begin(), trace.t_comp.end(), 0.0);
  if (trace.t_iter_event > 0.0 && trace.num_stages > 0)
    r.eta_util = sum_c / (trace.num_stages * trace.t_iter_event);
  r.delta_stall = trace.t_iter_event - trace.t_iter_analytic;
  return r;
}

}  // namespace lora_fleet
