// tlora_comm.cuh — NCCL communicator behind the C-ABI (include/tlora.h "communicator").
//
// SURVEY §8(b) "comm": init from an ncclUniqueId plus TP / DP group sizes. The reference
// has no communicator (its multi-GPU behaviour is simulated, sim_engine.hpp:306-315); this
// is what a C++ host needs to run the layer tensor-parallel / data-parallel without Python.
// Rank layout: world = tp * dp, rank = dp_index * tp + tp_index; the TP group is the tp
// consecutive ranks of one replica (NVLink neighbours), the DP group the ranks with the
// same tp_index. NCCL is loaded at run time (dlopen "libnccl.so.2"): a process that already
// loaded one (e.g. PyTorch's) reuses it, a pure C++ host gets the system library, and the
// library itself has no link-time NCCL dependency. Included once, at the end of
// tlora_capi.cu (it uses that file's status / guard helpers).
#pragma once
#include <dlfcn.h>
#include <nccl.h>

namespace {

struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommSplit) split = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclReduceScatter) reduce_scatter = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  decltype(&ncclGetVersion) version = nullptr;
  std::string load_error;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      api.load_error = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
#define TL_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(sym(name))
    TL_SYM(get_unique_id, "ncclGetUniqueId");
    TL_SYM(init_rank, "ncclCommInitRank");
    TL_SYM(split, "ncclCommSplit");
    TL_SYM(destroy, "ncclCommDestroy");
    TL_SYM(all_reduce, "ncclAllReduce");
    TL_SYM(all_gather, "ncclAllGather");
    TL_SYM(reduce_scatter, "ncclReduceScatter");
    TL_SYM(group_start, "ncclGroupStart");
    TL_SYM(group_end, "ncclGroupEnd");
    TL_SYM(error_string, "ncclGetErrorString");
    TL_SYM(version, "ncclGetVersion");
#undef TL_SYM
    if (!api.get_unique_id || !api.init_rank || !api.split || !api.destroy || !api.all_reduce ||
        !api.all_gather || !api.reduce_scatter || !api.group_start || !api.group_end ||
        !api.error_string)
      api.load_error = "libnccl.so.2 lacks a required symbol (need NCCL >= 2.18)";
  });
  require(api.load_error.empty(), TLORA_ERR_NCCL, api.load_error);
  return api;
}

#define TL_NCCL(x)                                                                          \
  do {                                                                                      \
    ncclResult_t r_ = (x);                                                                  \
    if (r_ != ncclSuccess)                                                                  \
      throw Status(TLORA_ERR_NCCL, std::string(#x) + ": " + nccl().error_string(r_));       \
  } while (0)

ncclDataType_t nccl_dtype(int dtype) {
  require(dtype == TLORA_F32 || dtype == TLORA_BF16 || dtype == TLORA_F64, TLORA_ERR_ARG,
          "unknown dtype");
  return dtype == TLORA_F32 ? ncclFloat32 : dtype == TLORA_BF16 ? ncclBfloat16 : ncclFloat64;
}

}  // namespace

struct tlora_comm {
  int device = 0;
  int32_t world = 1, rank = 0, tp = 1, dp = 1;
  ncclComm_t comm[3] = {nullptr, nullptr, nullptr};  // TLORA_GROUP_WORLD / _TP / _DP
  // Destroys every communicator that exists (a failed split in create must not leak the
  // world comm). Returns the first NCCL error; keeps destroying after one fails.
  ncclResult_t release() {
    ncclResult_t first = ncclSuccess;
    for (int i = 2; i >= 0; --i) {
      if (!comm[i]) continue;
      const ncclResult_t r = nccl().destroy(comm[i]);
      comm[i] = nullptr;
      if (r != ncclSuccess && first == ncclSuccess) first = r;
    }
    return first;
  }
  ~tlora_comm() {
    if (comm[0] || comm[1] || comm[2]) {
      int prev = -1;
      cudaGetDevice(&prev);
      if (prev != device) cudaSetDevice(device);
      release();
      if (prev >= 0 && prev != device) cudaSetDevice(prev);
    }
  }
};

extern "C" {

int tlora_comm_get_unique_id(uint8_t* id) {
  return guarded([&] {
    require(id != nullptr, TLORA_ERR_ARG, "id is null");
    ncclUniqueId u;
    TL_NCCL(nccl().get_unique_id(&u));
    std::memcpy(id, u.internal, TLORA_UNIQUE_ID_BYTES);
  });
}

int tlora_comm_create(int device, const uint8_t* id, int32_t world, int32_t rank,
                      int32_t tp_size, tlora_comm** out) {
  return guarded([&] {
    require(out != nullptr && id != nullptr, TLORA_ERR_ARG, "null argument");
    *out = nullptr;
    require(world >= 1 && rank >= 0 && rank < world, TLORA_ERR_ARG, "rank must be in [0, world)");
    require(tp_size >= 1 && world % tp_size == 0, TLORA_ERR_ARG,
            "tp_size must divide the world size");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0 || device < 0 || device >= n)
      throw Status(TLORA_ERR_NO_DEVICE, "no CUDA device " + std::to_string(device));
    const NcclApi& api = nccl();
    DeviceGuard g(device);
    auto c = std::make_unique<tlora_comm>();
    c->device = device;
    c->world = world;
    c->rank = rank;
    c->tp = tp_size;
    c->dp = world / tp_size;
    ncclUniqueId u;
    std::memcpy(u.internal, id, TLORA_UNIQUE_ID_BYTES);
    TL_NCCL(api.init_rank(&c->comm[TLORA_GROUP_WORLD], world, u, rank));
    // collective over the world comm: every rank makes both splits in the same order
    TL_NCCL(api.split(c->comm[TLORA_GROUP_WORLD], rank / tp_size, rank % tp_size,
                      &c->comm[TLORA_GROUP_TP], nullptr));
    TL_NCCL(api.split(c->comm[TLORA_GROUP_WORLD], rank % tp_size, rank / tp_size,
                      &c->comm[TLORA_GROUP_DP], nullptr));
    *out = c.release();
  });
}

int tlora_comm_destroy(tlora_comm* comm) {
  return guarded([&] {
    if (!comm) return;
    std::unique_ptr<tlora_comm> c(comm);
    DeviceGuard g(c->device);
    TL_NCCL(c->release());  // all three are destroyed even if one fails; first error wins
  });
}

int tlora_comm_info(const tlora_comm* comm, int32_t* world, int32_t* rank, int32_t* tp_size,
                    int32_t* dp_size) {
  return guarded([&] {
    require(comm != nullptr, TLORA_ERR_ARG, "comm is null");
    if (world) *world = comm->world;
    if (rank) *rank = comm->rank;
    if (tp_size) *tp_size = comm->tp;
    if (dp_size) *dp_size = comm->dp;
  });
}

namespace {
ncclComm_t group_comm(const tlora_comm* c, int group) {
  require(c != nullptr, TLORA_ERR_ARG, "comm is null");
  require(group >= TLORA_GROUP_WORLD && group <= TLORA_GROUP_DP, TLORA_ERR_ARG, "unknown group");
  return c->comm[group];
}
}  // namespace

int tlora_comm_all_gather(tlora_comm* comm, int group, const void* send, void* recv,
                          size_t send_count, int dtype, void* stream) {
  return guarded([&] {
    ncclComm_t c = group_comm(comm, group);
    DeviceGuard g(comm->device);
    TL_NCCL(nccl().all_gather(send, recv, send_count, nccl_dtype(dtype), c,
                              reinterpret_cast<cudaStream_t>(stream)));
  });
}

int tlora_comm_reduce_scatter(tlora_comm* comm, int group, const void* send, void* recv,
                              size_t recv_count, int dtype, void* stream) {
  return guarded([&] {
    ncclComm_t c = group_comm(comm, group);
    DeviceGuard g(comm->device);
    TL_NCCL(nccl().reduce_scatter(send, recv, recv_count, nccl_dtype(dtype), ncclSum, c,
                                  reinterpret_cast<cudaStream_t>(stream)));
  });
}

int tlora_comm_all_reduce(tlora_comm* comm, int group, const void* send, void* recv,
                          size_t count, int dtype, int average, void* stream) {
  return guarded([&] {
    ncclComm_t c = group_comm(comm, group);
    DeviceGuard g(comm->device);
    TL_NCCL(nccl().all_reduce(send, recv, count, nccl_dtype(dtype), average ? ncclAvg : ncclSum,
                              c, reinterpret_cast<cudaStream_t>(stream)));
  });
}

int tlora_layer_allreduce_grads(tlora_layer* layer, tlora_comm* comm, int group, int average,
                                void* stream) {
  return guarded([&] {
    require(layer != nullptr, TLORA_ERR_ARG, "layer is null");
    ncclComm_t c = group_comm(comm, group);
    require(comm->device == layer->device, TLORA_ERR_ARG, "comm and layer on different devices");
    DeviceGuard g(layer->device);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const size_t R = (size_t)layer->L.R;
    const NcclApi& api = nccl();
    const ncclRedOp_t op = average ? ncclAvg : ncclSum;
    TL_NCCL(api.group_start());
    TL_NCCL(api.all_reduce(layer->dAT.p, layer->dAT.p, R * layer->L.d, ncclFloat32, op, c, s));
    TL_NCCL(api.all_reduce(layer->dB.p, layer->dB.p, R * layer->L.k, ncclFloat32, op, c, s));
    TL_NCCL(api.group_end());
  });
}

// Sharded data-parallel optimizer (ZeRO-1 style over the packed adapters): reduce-scatter
// the fp32 gradients by packed-row shards, AdamW on this rank's shard, all-gather the
// refreshed bf16 operands and rebuild their transposed copies.
int tlora_layer_dp_shard(const tlora_layer* layer, const tlora_comm* comm, int group,
                         int64_t* row_lo, int64_t* row_hi) {
  return guarded([&] {
    require(layer != nullptr && comm != nullptr, TLORA_ERR_ARG, "null argument");
    require(group == TLORA_GROUP_DP || group == TLORA_GROUP_WORLD, TLORA_ERR_ARG,
            "shard over the DP (or world) group");
    const int32_t P = group == TLORA_GROUP_DP ? comm->dp : comm->world;
    const int32_t me = group == TLORA_GROUP_DP ? comm->rank / comm->tp : comm->rank;
    const int64_t R = layer->L.R;
    require(R % P == 0 && (R / P) % 2 == 0, TLORA_ERR_SHAPE,
            "packed rank width R must split into even row shards over the group");
    if (row_lo) *row_lo = me * (R / P);
    if (row_hi) *row_hi = (me + 1) * (R / P);
  });
}

int tlora_layer_reduce_scatter_grads(tlora_layer* layer, tlora_comm* comm, int group,
                                     void* stream) {
  return guarded([&] {
    int64_t lo = 0, hi = 0;
    if (tlora_layer_dp_shard(layer, comm, group, &lo, &hi) != TLORA_OK)
      throw Status(TLORA_ERR_SHAPE, g_last_error);
    ncclComm_t c = group_comm(comm, group);
    DeviceGuard g(layer->device);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const NcclApi& api = nccl();
    const size_t nA = (size_t)(hi - lo) * layer->L.d, nB = (size_t)(hi - lo) * layer->L.k;
    // in place: this rank's shard of rows [lo, hi) receives the sum (recv = send + rank * n)
    TL_NCCL(api.group_start());
    TL_NCCL(api.reduce_scatter(layer->dAT.p, layer->dAT.p + (size_t)lo * layer->L.d, nA,
                               ncclFloat32, ncclSum, c, s));
    TL_NCCL(api.reduce_scatter(layer->dB.p, layer->dB.p + (size_t)lo * layer->L.k, nB,
                               ncclFloat32, ncclSum, c, s));
    TL_NCCL(api.group_end());
  });
}

int tlora_layer_allgather_operands(tlora_layer* layer, tlora_comm* comm, int group, void* stream) {
  return guarded([&] {
    int64_t lo = 0, hi = 0;
    if (tlora_layer_dp_shard(layer, comm, group, &lo, &hi) != TLORA_OK)
      throw Status(TLORA_ERR_SHAPE, g_last_error);
    ncclComm_t c = group_comm(comm, group);
    DeviceGuard g(layer->device);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const NcclApi& api = nccl();
    const int64_t R = layer->L.R, d = layer->L.d, k = layer->L.k;
    TL_NCCL(api.group_start());
    TL_NCCL(api.all_gather(layer->AT.p + (size_t)lo * d, layer->AT.p, (size_t)(hi - lo) * d,
                           ncclBfloat16, c, s));
    TL_NCCL(api.all_gather(layer->Bcat.p + (size_t)lo * k, layer->Bcat.p, (size_t)(hi - lo) * k,
                           ncclBfloat16, c, s));
    TL_NCCL(api.group_end());
    const dim3 blk(32, 8);
    transpose_bf16_kernel<<<dim3((unsigned)tlora::ceil_div(d, 32), (unsigned)tlora::ceil_div(R, 32)),
                            blk, 0, s>>>(layer->AT.p, R, d, layer->Acat.p);
    transpose_bf16_kernel<<<dim3((unsigned)tlora::ceil_div(k, 32), (unsigned)tlora::ceil_div(R, 32)),
                            blk, 0, s>>>(layer->Bcat.p, R, k, layer->BcatT.p);
    TL_CUDA(cudaGetLastError());
    g_launches.fetch_add(2, std::memory_order_relaxed);
  });
}

}  // extern "C"
