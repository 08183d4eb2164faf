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

// ---- projection-level extension (new): the reference adapts ONE projection per layer
// (fused_lora.hpp:166-176 counts r·(d+k) per layer). A transformer layer of the configs C2-C4
// adapts seven (q, k, v, o, gate, up, down), each a fused multi-LoRA layer with its own
// registry; every (layer, projection, job) branch maps to registry slot = the job's
// position in the job_id-sorted group, identical for all projections.
struct Projection {
  std::string name;
  long long d = 0, k = 0;  // in-features, out-features
};

// q/k/v/o + gated MLP of a decoder layer (hidden, key/value width, intermediate size).
inline std::vector<Projection> decoder_projections(long long hidden, long long q_out,
                                                   long long kv_out, long long intermediate) {
  return {{"q", hidden, q_out},          {"k", hidden, kv_out},         {"v", hidden, kv_out},
          {"o", q_out, hidden},          {"gate", hidden, intermediate}, {"up", hidden, intermediate},
          {"down", intermediate, hidden}};
}

struct SsmLayerSet {
  SsmGraph graph;
  std::vector<Projection> projections;
  struct Branch {
    int layer;
    int projection;  // index into projections
    std::string job_id;
    int slot;        // registry slot of the projection's fused layer
  };
  std::vector<Branch> branches;  // layer-major, then projection, then job_id order
};

inline SsmLayerSet fuse_projections(const std::vector<JobSpec>& group,
                                    std::vector<Projection> projections) {
  if (projections.empty()) throw std::invalid_argument("fuse_projections: no projections");
  SsmLayerSet s;
  s.graph = fuse(group);
  s.projections = std::move(projections);
  for (int layer : s.graph.backbone_nodes)
    for (int p = 0; p < (int)s.projections.size(); ++p)
      for (int slot = 0; slot < (int)s.graph.jobs.size(); ++slot)
        s.branches.push_back({layer, p, s.graph.jobs[slot].job_id, slot});
  return s;
}

// r·Σ_p(d_p + k_p) per layer × layers: the trainable parameters of one job when every
// listed projection of every layer is adapted (reduces to trainable_param_count(job) for
// the single projection {hidden_dim -> proj_dim}).
inline long long trainable_param_count(const JobSpec& job, const std::vector<Projection>& projections) {
  job.validate();
  long long per_layer = 0;
  for (const auto& p : projections) per_layer += p.d + p.k;
  return static_cast<long long>(job.rank) * per_layer * job.model.num_layers;
}

// Registry slot order of a fused layer for this graph: position of each job in g.jobs.
inline std::vector<int> registry_ranks(const SsmGraph& g) {
  std::vector<int> r;
  for (const auto& j : g.jobs) r.push_back(j.rank);
  return r;
}

}  // namespace lora_fleet
