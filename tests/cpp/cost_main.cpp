// cost_main.cpp — the measured B200 cost model of include/lora_fleet/hardware.hpp from C++.
//
//   cost_main <profile.json>   reads lines "d k r1,r2,... t1,t2,..." (ranks and tokens per
//                              job) from stdin; prints the b200_hardware_spec() as one JSON
//                              line, then one predicted step time (seconds) per input line.
// Used by tests/test_cost_model.py (the fit's own grid, CPU) and tests/test_gpu_cost_model.py
// (measured C5 cells on a B200).
#include <cstdio>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "lora_fleet/hardware.hpp"

using namespace lora_fleet;

template <class T>
std::vector<T> csv(const std::string& s) {
  std::vector<T> v;
  std::stringstream ss(s);
  std::string x;
  while (std::getline(ss, x, ',')) v.push_back((T)std::stoll(x));
  return v;
}

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: cost_main <profile.json> < cells\n");
    return 2;
  }
  try {
    const CostProfile p = CostProfile::load(argv[1]);
    const HardwareSpec h = b200_hardware_spec(p);
    std::printf("{\"gpu_flops\": %.6e, \"gpu_memory\": %.6e, \"intra_node_bw\": %.6e, "
                "\"weight_stream_bw\": %.6e, \"kernel_launch_overhead\": %.6e, "
                "\"backward_multiplier\": %.1f}\n",
                h.gpu_flops, h.gpu_memory, h.intra_node_bw, h.weight_stream_bw,
                h.kernel_launch_overhead, h.backward_multiplier);
    std::string line;
    while (std::getline(std::cin, line)) {
      if (line.empty()) continue;
      std::stringstream ss(line);
      long long d, k;
      std::string rs, ts;
      ss >> d >> k >> rs >> ts;
      const auto w = projection_work(d, k, csv<int>(rs), csv<long long>(ts));
      std::printf("%.9e\n", predict_step_seconds(p, w));
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "cost_main: %s\n", e.what());
    return 1;
  }
  return 0;
}
