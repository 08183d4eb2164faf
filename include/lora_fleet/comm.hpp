// comm.hpp — C++ handle for the C-ABI communicator (include/tlora.h, tlora_comm_*).
//
// The reference has no communicator: its TP / DP behaviour is simulated
// (proj/include/lora_fleet/sim_engine.hpp:306-315, nano_pipeline.hpp:65-97). This RAII
// wrapper is what a C++ host uses to run the fused layer data- / tensor-parallel:
//
//   auto id = lora_fleet::Communicator::unique_id();        // rank 0; share out of band
//   lora_fleet::Communicator comm(device, id, world, rank, tp_size);
//   comm.allreduce_grads(layer, TLORA_GROUP_DP, /*average=*/true, stream);
//
// Errors throw std::runtime_error with tlora_last_error()'s message (as fused_lora.hpp).
#pragma once
#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "../tlora.h"

namespace lora_fleet {

class Communicator {
 public:
  using Id = std::array<uint8_t, TLORA_UNIQUE_ID_BYTES>;

  static Id unique_id() {
    Id id{};
    check(tlora_comm_get_unique_id(id.data()));
    return id;
  }

  Communicator(int device, const Id& id, int world, int rank, int tp_size = 1) {
    check(tlora_comm_create(device, id.data(), world, rank, tp_size, &c_));
  }
  ~Communicator() {
    if (c_) tlora_comm_destroy(c_);
  }
  Communicator(const Communicator&) = delete;
  Communicator& operator=(const Communicator&) = delete;

  int world() const { return info()[0]; }
  int rank() const { return info()[1]; }
  int tp_size() const { return info()[2]; }
  int dp_size() const { return info()[3]; }

  void allreduce_grads(tlora_layer* layer, int group = TLORA_GROUP_DP, bool average = true,
                       void* stream = nullptr) {
    check(tlora_layer_allreduce_grads(layer, c_, group, average ? 1 : 0, stream));
  }
  void all_gather(int group, const void* send, void* recv, size_t send_count, int dtype,
                  void* stream = nullptr) {
    check(tlora_comm_all_gather(c_, group, send, recv, send_count, dtype, stream));
  }
  void reduce_scatter(int group, const void* send, void* recv, size_t recv_count, int dtype,
                      void* stream = nullptr) {
    check(tlora_comm_reduce_scatter(c_, group, send, recv, recv_count, dtype, stream));
  }
  void all_reduce(int group, const void* send, void* recv, size_t count, int dtype,
                  bool average = false, void* stream = nullptr) {
    check(tlora_comm_all_reduce(c_, group, send, recv, count, dtype, average ? 1 : 0, stream));
  }
  tlora_comm* handle() const { return c_; }

 private:
  static void check(int code) {
    if (code != TLORA_OK) throw std::runtime_error(std::string("tlora: ") + tlora_last_error());
  }
  std::array<int32_t, 4> info() const {
    std::array<int32_t, 4> v{};
    check(tlora_comm_info(c_, &v[0], &v[1], &v[2], &v[3]));
    return v;
  }
  tlora_comm* c_ = nullptr;
};

}  // namespace lora_fleet
