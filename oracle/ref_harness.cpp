// ref_harness.cpp — drives the UNMODIFIED reference hot path (test infrastructure only).
//
// Compiled by oracle/Makefile against /root/reference/proj/include (read in place, never
// copied) plus the self-written Eigen-subset shim in oracle/eigen_shim/. Output goes to
// oracle/_ref/ (git-ignored). Two modes:
//
//   ref_harness golden <dir>   regenerate the reference's own seeded test instances and
//                              dump inputs + reference outputs as golden vectors:
//        fused_2024.bin   test_fused_lora.cpp:18-62 generator, mt19937_64(2024), 50 inst.
//        fused_101.bin    acceptance.cpp:56-100 generator, mt19937_64(101), 200 inst.
//        fused_99.bin     test_fused_lora.cpp:115-125, mt19937_64(99), 20 inst.
//        kat.json         fused KAT (:75-91), SPEC.md:113-122 examples, partition /
//                         aimd_step / fuse / trainable_param_count known answers.
//   ref_harness bench ...      time the reference path on the host cores (bench.py's
//                              reference arm / cpu_baseline, see usage below).
//
// The generators restate the reference tests' RNG call order exactly (libstdc++
// distributions, same declaration scopes), so the instances are the reference's own.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "lora_fleet/fused_lora.hpp"
#include "lora_fleet/nano_pipeline.hpp"
#include "lora_fleet/ssm_plan.hpp"

using namespace lora_fleet;

namespace {

struct Instance {
  TokenBatch batch;
  Matrix W;
  std::vector<AdapterMatrices> adapters;
};

Matrix randm(std::mt19937_64& rng, std::normal_distribution<double>& val, int rows, int cols) {
  Matrix m(rows, cols);
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) m(i, j) = val(rng);
  return m;
}

// test_fused_lora.cpp:18-48 (normal_distribution is local to each call there)
Instance unit_test_instance(std::mt19937_64& rng, int max_adapters = 4) {
  std::uniform_int_distribution<int> dim_dist(2, 64), tok_dist(1, 32);
  const int ranks[] = {2, 4, 8, 16};
  const int d = dim_dist(rng), k = dim_dist(rng);
  const int n_adapters = 1 + static_cast<int>(rng() % max_adapters);
  std::normal_distribution<double> val;
  Instance inst;
  inst.W = randm(rng, val, d, k);
  int total = 0;
  std::vector<int> counts;
  for (int a = 0; a < n_adapters; ++a) {
    int r = ranks[rng() % 4];
    Matrix A = randm(rng, val, d, r);
    Matrix B = randm(rng, val, r, k);
    inst.adapters.push_back({"job" + std::to_string(a), A, B});
    counts.push_back(tok_dist(rng));
    total += counts.back();
  }
  inst.batch.rows = randm(rng, val, total, d);
  for (int a = 0; a < n_adapters; ++a)
    for (int t = 0; t < counts[a]; ++t) inst.batch.segment_map.push_back("job" + std::to_string(a));
  std::shuffle(inst.batch.segment_map.begin(), inst.batch.segment_map.end(), rng);
  return inst;
}

// acceptance.cpp:58-86 (distributions shared across all 200 trials)
std::vector<Instance> acceptance_instances() {
  std::mt19937_64 rng(101);
  std::uniform_int_distribution<int> dim_dist(2, 64), tok_dist(1, 32);
  std::normal_distribution<double> val;
  const int ranks[] = {2, 4, 8, 16};
  std::vector<Instance> out;
  for (int trial = 0; trial < 200; ++trial) {
    const int d = dim_dist(rng), k = dim_dist(rng);
    const int n_adapters = 1 + static_cast<int>(rng() % 4);
    Instance inst;
    inst.W = randm(rng, val, d, k);
    std::vector<std::string> owners;
    for (int a = 0; a < n_adapters; ++a) {
      int r = ranks[rng() % 4];
      Matrix A = randm(rng, val, d, r);
      Matrix B = randm(rng, val, r, k);
      inst.adapters.push_back({"j" + std::to_string(a), A, B});
      int tokens = tok_dist(rng);
      for (int t = 0; t < tokens; ++t) owners.push_back("j" + std::to_string(a));
    }
    while (owners.size() > 128) owners.pop_back();
    std::shuffle(owners.begin(), owners.end(), rng);
    inst.batch.rows = randm(rng, val, static_cast<int>(owners.size()), d);
    inst.batch.segment_map = owners;
    out.push_back(std::move(inst));
  }
  return out;
}

void put_i32(std::ofstream& f, int32_t v) { f.write(reinterpret_cast<const char*>(&v), 4); }
void put_f64(std::ofstream& f, double v) { f.write(reinterpret_cast<const char*>(&v), 8); }
void put_mat(std::ofstream& f, const Matrix& m) {  // row-major
  for (Eigen::Index i = 0; i < m.rows(); ++i)
    for (Eigen::Index j = 0; j < m.cols(); ++j) put_f64(f, m(i, j));
}

// Record layout (little endian):
//   i32 d, k, S, T ; per adapter: i32 rank, i32 len, bytes id ; T x i32 adapter index
//   f64 W[d*k], X[T*d], per adapter A[d*r], B[r*k] ; f64 Y_fused[T*k], Y_mat[T*k]
//   f64 flops, bytes ; i64 launches ; f64 u_flops, u_bytes ; i64 u_launches
void dump(std::ofstream& f, const Instance& in) {
  const auto& b = in.batch;
  put_i32(f, (int32_t)b.rows.cols());
  put_i32(f, (int32_t)in.W.cols());
  put_i32(f, (int32_t)in.adapters.size());
  put_i32(f, (int32_t)b.rows.rows());
  for (const auto& a : in.adapters) {
    put_i32(f, (int32_t)a.A.cols());
    put_i32(f, (int32_t)a.job_id.size());
    f.write(a.job_id.data(), (std::streamsize)a.job_id.size());
  }
  for (const auto& id : b.segment_map) {
    int32_t idx = -1;
    for (size_t a = 0; a < in.adapters.size(); ++a)
      if (in.adapters[a].job_id == id) idx = (int32_t)a;
    put_i32(f, idx);
  }
  put_mat(f, in.W);
  put_mat(f, b.rows);
  for (const auto& a : in.adapters) {
    put_mat(f, a.A);
    put_mat(f, a.B);
  }
  auto [y, cost] = fused_forward(b, in.W, in.adapters);
  Matrix ym = materialized_oracle(b, in.W, in.adapters);
  OpCost u = unfused_cost(b, in.W, in.adapters);
  put_mat(f, y);
  put_mat(f, ym);
  put_f64(f, cost.flops);
  put_f64(f, cost.bytes_moved);
  int64_t l = cost.kernel_launches;
  f.write(reinterpret_cast<const char*>(&l), 8);
  put_f64(f, u.flops);
  put_f64(f, u.bytes_moved);
  l = u.kernel_launches;
  f.write(reinterpret_cast<const char*>(&l), 8);
}

std::string jnum(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

int golden(const std::string& dir) {
  {
    std::ofstream f(dir + "/fused_2024.bin", std::ios::binary);
    std::mt19937_64 rng(2024);
    for (int t = 0; t < 50; ++t) dump(f, unit_test_instance(rng));
  }
  {
    std::ofstream f(dir + "/fused_101.bin", std::ios::binary);
    for (const auto& in : acceptance_instances()) dump(f, in);
  }
  {
    std::ofstream f(dir + "/fused_99.bin", std::ios::binary);
    std::mt19937_64 rng(99);
    for (int t = 0; t < 20; ++t) dump(f, unit_test_instance(rng));
  }
  std::ostringstream j;
  j << "{\n";
  {  // test_fused_lora.cpp:75-91
    Matrix W(3, 2);
    W << 1, 0, 0, 1, 1, 1;
    Matrix A(3, 1), B(1, 2);
    A << 1, 0, 0;
    B << 2, 3;
    TokenBatch batch;
    batch.rows = Matrix(2, 3);
    batch.rows << 1, 2, 3, 0, 1, 0;
    batch.segment_map = {"j", "j"};
    auto [y, cost] = fused_forward(batch, W, {{"j", A, B}});
    j << " \"kat_single_segment\": {\"Y\": [[" << jnum(y(0, 0)) << "," << jnum(y(0, 1)) << "],["
      << jnum(y(1, 0)) << "," << jnum(y(1, 1)) << "]], \"flops\": " << jnum(cost.flops)
      << ", \"bytes\": " << jnum(cost.bytes_moved) << ", \"launches\": " << cost.kernel_launches
      << "},\n";
  }
  {  // rank-1 outer product and scalar example
    Matrix W = Matrix::Zero(4, 4), A = Matrix::Zero(4, 1), B = Matrix::Zero(1, 4);
    A(0, 0) = 1;
    B(0, 0) = 1;
    TokenBatch batch;
    batch.rows = Matrix::Zero(4, 4);
    for (int i = 0; i < 4; ++i) batch.rows(i, i) = 1;
    batch.segment_map = {"a", "a", "a", "a"};
    auto [y, cost] = fused_forward(batch, W, {{"a", A, B}});
    j << " \"kat_rank1\": [";
    for (int i = 0; i < 4; ++i) {
      j << "[";
      for (int c = 0; c < 4; ++c) j << jnum(y(i, c)) << (c < 3 ? "," : "");
      j << "]" << (i < 3 ? "," : "");
    }
    j << "],\n";
    Matrix w1(1, 1), a1(1, 1), b1(1, 1);
    w1 << 1;
    a1 << 2;
    b1 << 3;
    TokenBatch bs;
    bs.rows = Matrix(1, 1);
    bs.rows << 1;
    bs.segment_map = {"s"};
    auto [ys, cs] = fused_forward(bs, w1, {{"s", a1, b1}});
    j << " \"kat_scalar\": " << jnum(ys(0, 0)) << ",\n";
  }
  {  // nano_pipeline.hpp partition / aimd_step (test_nano_pipeline.cpp:28-38, 90-123)
    j << " \"partition\": [";
    const int cases[][2] = {{10, 4}, {3, 8}, {60, 4}, {60, 7}, {1, 1}, {17, 17}, {16, 5}};
    for (size_t c = 0; c < sizeof(cases) / sizeof(cases[0]); ++c) {
      auto s = partition(cases[c][0], cases[c][1]);
      j << "{\"batch\":" << cases[c][0] << ",\"n\":" << cases[c][1] << ",\"out_n\":" << s.n
        << ",\"per_nano\":[";
      for (size_t i = 0; i < s.per_nano_samples.size(); ++i)
        j << s.per_nano_samples[i] << (i + 1 < s.per_nano_samples.size() ? "," : "");
      j << "]}" << (c + 1 < sizeof(cases) / sizeof(cases[0]) ? "," : "");
    }
    j << "],\n";
    // a deterministic AIMD trajectory: n=8, alpha=4, beta=0.5, tau_rel in {0, 0.1}
    for (double tau : {0.0, 0.1}) {
      AimdState s;
      s.n = 8;
      s.tau_rel = tau;
      const double ts[] = {10.0, 9.0, 9.5, 9.5, 9.4, 8.0, 8.0, 12.0, 3.0, 2.9, 2.95, 2.0};
      j << " \"aimd_tau" << (tau == 0.0 ? "0" : "01") << "\": [";
      for (size_t i = 0; i < sizeof(ts) / sizeof(ts[0]); ++i) {
        s = aimd_step(s, ts[i]);
        j << "[" << jnum(ts[i]) << "," << s.n << "]" << (i + 1 < sizeof(ts) / sizeof(ts[0]) ? "," : "");
      }
      j << "],\n";
    }
  }
  {  // ssm_plan.hpp fuse (test_ssm_plan.cpp:62-78) and fused_lora.hpp:166-176
    ModelSpec m;
    m.name = "tiny";
    m.num_layers = 6;
    m.hidden_dim = 64;
    m.proj_dim = 64;
    m.base_memory_bytes = 1e9;
    auto mk = [&](const std::string& id, int rank) {
      JobSpec jb;
      jb.job_id = id;
      jb.model = m;
      jb.rank = rank;
      return jb;
    };
    auto g = fuse({mk("b", 4), mk("a", 8), mk("c", 16)});
    j << " \"fuse_jobs\": [";
    for (size_t i = 0; i < g.jobs.size(); ++i)
      j << "\"" << g.jobs[i].job_id << "\"" << (i + 1 < g.jobs.size() ? "," : "");
    j << "], \"fuse_branches\": " << g.adapter_branches.size() << ", \"fuse_first\": [" << g.adapter_branches[0].first
      << ",\"" << g.adapter_branches[0].second << "\"],\n";
    j << " \"trainable_params_r4_L6\": " << trainable_param_count(mk("x", 4))
      << ", \"adapter_flops_per_token_r4\": " << jnum(adapter_flops_per_token(mk("x", 4))) << "\n";
  }
  j << "}\n";
  std::ofstream(dir + "/kat.json") << j.str();
  return 0;
}

// ------------------------------------------------------------------------- bench mode
// ref_harness bench <threads> <tokens_per_job> <repeats> <ranks csv> <d:k;d:k;...> [min_s]
// Setup (weights, inputs) is untimed; one warm-up repetition, then `repeats` timed
// repetitions (or more, until min_s seconds have elapsed); per-repetition times printed.
// One "step" = for every projection: reference fused_forward (fwd), reference
// fused_forward on the transposed problem (dX = dY·(W + A_j B_j)ᵀ, exact), and the
// adapter gradients dB_j = (X_j A_j)ᵀ dY_j, dA_j = X_jᵀ (dY_j B_jᵀ) with the shim GEMM
// (the reference has no backward). Tokens are sharded across threads;
// each thread calls the pure, reentrant reference functions on its own shard.
std::vector<int> parse_csv(const std::string& s) {
  std::vector<int> v;
  std::stringstream ss(s);
  std::string x;
  while (std::getline(ss, x, ',')) v.push_back(std::stoi(x));
  return v;
}

Matrix transpose(const Matrix& m) {
  Matrix t(m.cols(), m.rows());
  for (Eigen::Index i = 0; i < m.rows(); ++i)
    for (Eigen::Index c = 0; c < m.cols(); ++c) t(c, i) = m(i, c);
  return t;
}

int bench(int argc, char** argv) {
  if (argc < 7) {
    std::fprintf(stderr, "usage: ref_harness bench threads tokens_per_job repeats ranks d:k;...\n");
    return 2;
  }
  const int threads = std::max(1, std::atoi(argv[2]));
  const int tpj = std::max(1, std::atoi(argv[3]));
  const int repeats = std::max(1, std::atoi(argv[4]));
  const auto ranks = parse_csv(argv[5]);
  std::vector<std::pair<int, int>> projs;
  {
    std::stringstream ss(argv[6]);
    std::string p;
    while (std::getline(ss, p, ';')) {
      auto c = p.find(':');
      projs.push_back({std::stoi(p.substr(0, c)), std::stoi(p.substr(c + 1))});
    }
  }
  // Values do not affect the timing; a cheap counter-hash fill keeps setup of the
  // multi-GB weight set to a few seconds (normal_distribution would dominate the run).
  uint64_t state = 2602;
  auto val = [&state](std::mt19937_64&) {
    state = state * 6364136223846793005ULL + 1442695040888963407ULL;
    return ((double)(state >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
  };
  std::mt19937_64 rng(2602);
  struct Proj {
    Matrix W, Wt;
    std::vector<AdapterMatrices> ad, adT;
  };
  std::vector<Proj> P;
  for (auto [d, k] : projs) {
    Proj p;
    p.W = Matrix(d, k);
    for (Eigen::Index i = 0; i < d; ++i)
      for (Eigen::Index c = 0; c < k; ++c) p.W(i, c) = val(rng) / std::sqrt((double)d);
    p.Wt = transpose(p.W);
    for (size_t s = 0; s < ranks.size(); ++s) {
      const int r = ranks[s];
      Matrix A(d, r), B(r, k);
      for (Eigen::Index i = 0; i < d; ++i)
        for (int c = 0; c < r; ++c) A(i, c) = val(rng) / std::sqrt((double)d);
      for (int i = 0; i < r; ++i)
        for (Eigen::Index c = 0; c < k; ++c) B(i, c) = val(rng) / std::sqrt((double)r);
      std::string id = "job" + std::to_string(s);
      p.ad.push_back({id, A, B});
      p.adT.push_back({id, transpose(B), transpose(A)});
    }
    P.push_back(std::move(p));
  }
  // per-thread token shard: round-robin the jobs' tokens over threads
  const int S = (int)ranks.size();
  std::vector<std::vector<std::string>> shard(threads);
  int tcount = 0;
  for (int s = 0; s < S; ++s)
    for (int t = 0; t < tpj; ++t) shard[(tcount++) % threads].push_back("job" + std::to_string(s));
  std::vector<std::vector<Matrix>> Xs(threads), dYs(threads);
  for (int th = 0; th < threads; ++th)
    for (size_t p = 0; p < P.size(); ++p) {
      const int T = (int)shard[th].size();
      Matrix X(T, P[p].W.rows()), dY(T, P[p].W.cols());
      for (Eigen::Index i = 0; i < X.rows(); ++i)
        for (Eigen::Index c = 0; c < X.cols(); ++c) X(i, c) = val(rng);
      for (Eigen::Index i = 0; i < dY.rows(); ++i)
        for (Eigen::Index c = 0; c < dY.cols(); ++c) dY(i, c) = val(rng);
      Xs[th].push_back(X);
      dYs[th].push_back(dY);
    }
  double checksum = 0.0;
  auto work = [&](int th, double* sink) {
    double acc = 0.0;
    for (size_t p = 0; p < P.size(); ++p) {
      if (shard[th].empty()) continue;
      TokenBatch b{Xs[th][p], shard[th]};
      auto [y, cost] = fused_forward(b, P[p].W, P[p].ad);  // forward (reference)
      TokenBatch g{dYs[th][p], shard[th]};
      auto [dx, c2] = fused_forward(g, P[p].Wt, P[p].adT);  // dX (reference, transposed)
      for (int s = 0; s < S; ++s) {                          // dA, dB (shim GEMMs)
        auto rows = detail::segment_rows(b, P[p].ad[s].job_id);
        if (rows.empty()) continue;
        Matrix xs(rows.size(), b.rows.cols()), gs(rows.size(), g.rows.cols());
        for (size_t i = 0; i < rows.size(); ++i) {
          xs.row((Eigen::Index)i) = b.rows.row(rows[i]);
          gs.row((Eigen::Index)i) = g.rows.row(rows[i]);
        }
        Matrix h = xs * P[p].ad[s].A;
        Matrix dB = transpose(h) * gs;
        Matrix dh = gs * P[p].adT[s].A;  // dY_j B_jᵀ
        Matrix dA = transpose(xs) * dh;
        acc += dA(0, 0) + dB(0, 0);
      }
      acc += y(0, 0) + dx(0, 0);
    }
    *sink = acc;
  };
  std::vector<double> sinks(threads);
  auto run_once = [&] {
    std::vector<std::thread> ts;
    for (int th = 0; th < threads; ++th) ts.emplace_back(work, th, &sinks[th]);
    for (auto& t : ts) t.join();
    for (double v : sinks) checksum += v;
  };
  const double min_s = argc > 7 ? std::atof(argv[7]) : 0.0;
  run_once();  // warm-up
  std::vector<double> per;
  double secs = 0.0;
  while ((int)per.size() < repeats || secs < min_s) {
    const auto t0 = std::chrono::steady_clock::now();
    run_once();
    per.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    secs += per.back();
    if (per.size() >= 100000) break;
  }
  std::printf("{\"seconds\": %.6f, \"tokens\": %d, \"repeats\": %d, \"threads\": %d, "
              "\"checksum\": %.6e, \"per_repeat\": [",
              secs, tcount * (int)per.size(), (int)per.size(), threads, checksum);
  for (size_t i = 0; i < per.size(); ++i) std::printf("%s%.6f", i ? ", " : "", per[i]);
  std::printf("]}\n");
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc >= 3 && std::strcmp(argv[1], "golden") == 0) return golden(argv[2]);
  if (argc >= 2 && std::strcmp(argv[1], "bench") == 0) return bench(argc, argv);
  std::fprintf(stderr, "usage: ref_harness golden <dir> | bench ...\n");
  return 2;
}
