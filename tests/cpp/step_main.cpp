// step_main.cpp — a pure C++ host for the layer-set training step (no Python, no torch):
// lora_fleet::fuse_projections -> LayerSetTrainer (tlora_step_* C-ABI) -> steps.
//
//   step_main dump <file>                       two steps of a small 2-layer set at N = 2,
//                                               then Y / dX / gradients / adapters -> file
//                                               (tests/test_gpu_executor.py compares it with
//                                               the Python-driven executor, bytewise)
//   step_main bench [C2|C3] [steps] [warmup] [nano] [layers]
//                                               one BENCH-format JSON line (bench.py
//                                               --host cpp); nano 0 = AIMD every step
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "lora_fleet/trainer.hpp"

using namespace lora_fleet;

namespace {

void check(int code) { detail::tl_throw(code); }

struct Config {
  std::string name;
  std::vector<Projection> projections;
  std::vector<int32_t> input_group;
  std::vector<JobSpec> jobs;
  int layers = 1;
};

JobSpec job(const std::string& id, const ModelSpec& m, int rank, int batch, int seq) {
  JobSpec j;
  j.job_id = id;
  j.model = m;
  j.rank = rank;
  j.batch_size = batch;
  j.seq_len = seq;
  return j;
}

Config make_config(const std::string& name, int layers_override) {
  Config c;
  c.name = name;
  ModelSpec m;
  m.base_memory_bytes = 1.0;
  if (name == "mini") {  // tests/test_gpu_executor.py::test_cpp_host_step_matches_...
    m.name = "mini";
    m.num_layers = 2;
    m.hidden_dim = 512;
    m.proj_dim = 768;
    c.projections = {{"q", 512, 768}, {"k", 512, 256}, {"o", 768, 512}};
    c.input_group = {0, 0, 1};
    c.jobs = {job("a", m, 8, 2, 256), job("b", m, 200, 3, 320), job("c", m, 16, 1, 192)};
  } else if (name == "C2" || name == "C3") {
    const bool c2 = name == "C2";
    m.name = c2 ? "qwen3-8b" : "llama3-8b";
    m.num_layers = c2 ? 1 : 32;
    m.hidden_dim = 4096;
    m.proj_dim = 4096;
    c.projections = decoder_projections(4096, 4096, 1024, c2 ? 12288 : 14336);
    c.input_group = {0, 0, 0, 1, 2, 2, 3};
    if (c2) {
      const int ranks[] = {8, 16, 24, 32, 48, 64, 96, 128}, batch[] = {1, 2, 1, 4, 2, 1, 4, 1};
      for (int i = 0; i < 8; ++i) c.jobs.push_back(job("job" + std::to_string(i), m, ranks[i], batch[i], 1024));
    } else {
      const int ranks[] = {8, 16, 32, 64, 128, 24, 48, 96}, batch[] = {1, 2, 4, 8};
      for (int i = 0; i < 16; ++i) {
        char id[16];
        std::snprintf(id, sizeof id, "job%02d", i);
        c.jobs.push_back(job(id, m, ranks[i % 8], batch[i % 4], 1024));
      }
    }
  } else {
    throw std::invalid_argument("unknown config " + name);
  }
  if (layers_override > 0) {
    for (auto& j : c.jobs) j.model.num_layers = layers_override;
  }
  c.layers = c.jobs.front().model.num_layers;
  return c;
}

// Weights and inputs from the library's seeded generator, in a fixed order (the Python side
// of the dump test repeats it): per key W, then per slot A, B; then X per group, dY per
// projection.
void fill(LayerSetTrainer& tr, const Config& c, uint64_t seed, double lr) {
  const int P = (int)c.projections.size();
  const int S = (int)c.jobs.size();
  std::vector<float> lrs, wd;
  for (int s = 0; s < S; ++s) {
    lrs.push_back((float)(lr * (1.0 + 0.25 * (s % 4))));  // as the Python drivers compute it
    wd.push_back(0.01f);
  }
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  auto scratch = [&](size_t bytes) {
    if (bytes > tmp_bytes) {
      if (tmp) cudaFree(tmp);
      if (cudaMalloc(&tmp, bytes) != cudaSuccess) throw std::runtime_error("cudaMalloc");
      tmp_bytes = bytes;
    }
    return tmp;
  };
  for (int L = 0; L < c.layers; ++L)
    for (int p = 0; p < P; ++p) {
      tlora_layer* lay = tr.layer(L, p);
      const long long d = c.projections[p].d, k = c.projections[p].k;
      void* W = scratch((size_t)d * k * 2);
      check(tlora_fill_normal(W, TLORA_BF16, d * k, seed++, (float)(1.0 / std::sqrt((double)d)), nullptr));
      check(tlora_layer_set_base(lay, W, TLORA_BF16, TLORA_DEVICE, nullptr));
      for (int s = 0; s < S; ++s) {
        const int r = c.jobs[s].rank;
        float* A = (float*)scratch((size_t)(d * r + (long long)r * k) * 4);
        float* B = A + d * r;
        check(tlora_fill_normal(A, TLORA_F32, d * r, seed, (float)(1.0 / std::sqrt((double)d)), nullptr));
        check(tlora_fill_normal(B, TLORA_F32, (long long)r * k, seed + 1, (float)(1.0 / std::sqrt((double)r)), nullptr));
        seed += 2;
        check(tlora_layer_set_adapter(lay, s, A, B, TLORA_F32, TLORA_DEVICE, nullptr));
      }
      check(tlora_layer_set_optimizer(lay, lrs.data(), wd.data(), 0.9f, 0.999f, 1e-8f));
    }
  int groups = 0;
  for (int32_t g : c.input_group) groups = std::max(groups, g + 1);
  for (int g = 0; g < groups; ++g) {
    auto b = tr.buffer(TLORA_BUF_X, g);
    check(tlora_fill_normal(b.ptr, TLORA_BF16, b.rows * b.cols, seed++, 1.0f, nullptr));
  }
  for (int p = 0; p < P; ++p) {
    auto b = tr.buffer(TLORA_BUF_DY, p);
    check(tlora_fill_normal(b.ptr, TLORA_BF16, b.rows * b.cols, seed++, 1.0f, nullptr));
  }
  if (cudaDeviceSynchronize() != cudaSuccess) throw std::runtime_error("fill failed");
  if (tmp) cudaFree(tmp);
}

void append(std::vector<uint8_t>& out, const void* dev, size_t bytes) {
  const size_t o = out.size();
  out.resize(o + bytes);
  if (cudaMemcpy(out.data() + o, dev, bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
    throw std::runtime_error("cudaMemcpy D2H");
}

int dump(const char* path) {
  Config c = make_config("mini", 0);
  SsmLayerSet set = fuse_projections(c.jobs, c.projections);
  TrainerOptions opt;
  opt.nano_fixed = 2;
  LayerSetTrainer tr(set, opt, c.input_group);
  fill(tr, c, 1000, 1e-3);
  tr.step();
  tr.step();
  std::vector<uint8_t> out;
  const int P = (int)c.projections.size();
  for (int p = 0; p < P; ++p) {
    auto b = tr.buffer(TLORA_BUF_Y, p);
    append(out, b.ptr, (size_t)b.rows * b.cols * 2);
  }
  for (int p = 0; p < P; ++p) {
    auto b = tr.buffer(TLORA_BUF_DX, p);
    append(out, b.ptr, (size_t)b.rows * b.cols * 2);
  }
  for (int L = 0; L < c.layers; ++L)
    for (int p = 0; p < P; ++p) {
      tlora_layer* lay = tr.layer(L, p);
      const long long d = c.projections[p].d, k = c.projections[p].k;
      std::vector<std::vector<uint8_t>> grads, adapters;
      for (int s = 0; s < (int)c.jobs.size(); ++s) {
        const int r = c.jobs[s].rank;
        std::vector<float> A((size_t)(d * r)), B((size_t)(r * k));
        check(tlora_layer_read_grad(lay, s, A.data(), B.data(), TLORA_HOST, nullptr));
        out.insert(out.end(), (uint8_t*)A.data(), (uint8_t*)(A.data() + A.size()));
        out.insert(out.end(), (uint8_t*)B.data(), (uint8_t*)(B.data() + B.size()));
      }
      for (int s = 0; s < (int)c.jobs.size(); ++s) {
        const int r = c.jobs[s].rank;
        std::vector<float> A((size_t)(d * r)), B((size_t)(r * k));
        check(tlora_layer_read_adapter(lay, s, A.data(), B.data(), TLORA_HOST, nullptr));
        out.insert(out.end(), (uint8_t*)A.data(), (uint8_t*)(A.data() + A.size()));
        out.insert(out.end(), (uint8_t*)B.data(), (uint8_t*)(B.data() + B.size()));
      }
    }
  std::ofstream f(path, std::ios::binary);
  f.write((const char*)out.data(), (std::streamsize)out.size());
  std::printf("dumped %zu bytes\n", out.size());
  return f.good() ? 0 : 1;
}

int bench(int argc, char** argv) {
  const std::string name = argc > 2 ? argv[2] : "C2";
  const int steps = argc > 3 ? std::atoi(argv[3]) : 10;
  const int warmup = argc > 4 ? std::atoi(argv[4]) : 3;
  const int nano = argc > 5 ? std::atoi(argv[5]) : 1;
  const int layers = argc > 6 ? std::atoi(argv[6]) : 0;
  Config c = make_config(name, layers);
  SsmLayerSet set = fuse_projections(c.jobs, c.projections);
  TrainerOptions opt;
  opt.nano_fixed = nano;
  LayerSetTrainer tr(set, opt, c.input_group);
  fill(tr, c, 2602, 1e-4);
  cudaStream_t s;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return 1;
  for (int i = 0; i < warmup; ++i) tr.step(0, s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaStreamSynchronize(s);
  std::string traj;
  cudaEventRecord(e0, s);
  int64_t tokens = 0;
  for (int i = 0; i < steps; ++i) {
    const auto st = tr.step(0, s);
    tokens += st.tokens;
    traj += (i ? "," : "") + std::string("[") + std::to_string(st.nano_used) + "," +
            (st.ms >= 0.f ? std::to_string(st.ms) : std::string("null")) + "]";
  }
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  double flops = 0.0;  // 4 T d k + 6 sum_j T_j r_j (d + k) per projection and layer
  long long T = 0, tr_sum = 0;
  for (const auto& j : c.jobs) {
    T += (long long)j.batch_size * j.seq_len;
    tr_sum += (long long)j.batch_size * j.seq_len * j.rank;
  }
  for (const auto& p : c.projections)
    flops += 4.0 * T * p.d * p.k + 6.0 * (double)tr_sum * (p.d + p.k);
  flops *= c.layers;
  const double ms_step = ms / steps;
  std::printf(
      "{\"metric\": \"aggregate LoRA training tokens/sec (all jobs) at 1/2/4/8 B200; tensor-pipe %%\", "
      "\"value\": %.1f, \"unit\": \"tokens/s\", \"n_gpus\": 1, \"steps\": %d, \"warmup\": %d, "
      "\"ms_per_step\": %.4f, \"higher_is_better\": true, \"scaling\": \"weak\", "
      "\"vs_baseline\": null, \"dtype\": \"bf16\", \"data\": \"synthetic (tlora_fill_normal)\", "
      "\"host\": \"cpp\", \"config\": {\"workload\": \"%s\", \"layers_per_step\": %d, "
      "\"tokens_per_gpu\": %lld, \"nano\": \"%s\", \"aimd_trajectory_n_ms\": [%s], "
      "\"achieved_tflops_step\": %.1f}}\n",
      tokens / (ms / 1e3), steps, warmup, ms_step, c.name.c_str(), c.layers, T,
      nano > 0 ? std::to_string(nano).c_str() : "aimd", traj.c_str(), flops / (ms_step / 1e3) / 1e12);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc >= 3 && std::strcmp(argv[1], "dump") == 0) return dump(argv[2]);
    if (argc >= 2 && std::strcmp(argv[1], "bench") == 0) return bench(argc, argv);
    std::fprintf(stderr, "usage: step_main dump <file> | bench [C2|C3] [steps] [warmup] [nano] [layers]\n");
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "step_main: %s\n", e.what());
    return 1;
  }
}
