// ssm_plan.hpp — Shared Super-Model layer descriptor of the drop-in API.
//
// SsmGraph / fuse() as in proj/include/lora_fleet/ssm_plan.hpp:25-30, 58-74: one backbone
// node per layer and one adapter branch per (layer, job), jobs sorted by job_id — the
// same order the fused layer's adapter registry uses for its slots. The pipeline-stage
// planner (bottleneck_partition / plan, ssm_plan.hpp:79-246) is out of scope.
#pragma once
#include <algorithm>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "lora_fleet/workload.hpp"

namespace lora_fleet {

struct SsmGraph {
  ModelSpec model;
  std::vector<JobSpec> jobs;                                  // sorted by job_id
  std::vector<int> backbone_nodes;                            // layer indices
  std::vector<std::pair<int, std::string>> adapter_branches;  // (layer, job_id)
};

inline SsmGraph fuse(const std::vector<JobSpec>& group) {
  if (group.empty()) throw std::invalid_argument("fuse: empty group");
  SsmGraph g;
  g.model = group.front().model;
  g.jobs = group;
  std::sort(g.jobs.begin(), g.jobs.end(),
            [](const JobSpec& a, const JobSpec& b) { return a.job_id < b.job_id; });
  for (const auto& j : g.jobs)
    if (j.model.name != g.model.name)
      throw std::runtime_error("fuse: mixed base models (" + g.model.name + " vs " +
                               j.model.name + ") cannot be grouped");
  g.backbone_nodes.reserve(g.model.num_layers);
  for (int layer = 0; layer < g.model.num_layers; ++layer) {
    g.backbone_nodes.push_back(layer);
    for (const auto& j : g.jobs) g.adapter_branches.emplace_back(layer, j.job_id);
  }
  return g;
}

// Registry slot order of a fused layer for this graph: position of each job in g.jobs.
inline std::vector<int> registry_ranks(const SsmGraph& g) {
  std::vector<int> r;
  for (const auto& j : g.jobs) r.push_back(j.rank);
  return r;
}

}  // namespace lora_fleet
