/*
 * tlora.h — C-ABI of the B200-native fused multi-LoRA linear layer (tLoRA hot path).
 *
 * This is the drop-in boundary for the reference's header-only C++ operator API
 * (proj/include/lora_fleet/fused_lora.hpp, nano_pipeline.hpp, ssm_plan.hpp). The
 * C++ mirror of that API (include/lora_fleet/*.hpp) and the Python binding
 * (paper_2602_07263_b200/capi.py) are both written on top of these entry points.
 *
 * Conventions
 *   - Plain pointers and sizes only; no C++ or torch types cross this boundary.
 *   - Every function returns an int status (TLORA_OK = 0). On failure a message is
 *     available from tlora_last_error() (thread-local). Nothing throws across the ABI.
 *   - Device-side compute entry points are enqueue-only on the given CUDA stream
 *     (passed as void* = cudaStream_t; NULL = legacy default stream).
 *   - Matrices are dense row-major. Activations/weights on device are bf16; adapter
 *     gradients are fp32. Host-side loaders accept f64 / f32 / bf16.
 *   - Distinct layers/plans are independent: every plan owns its scratch (split-K
 *     partial planes, dH of tlora_backward, gather copies), so gradient launches of
 *     different plans may run concurrently on different streams. Calls that use ONE plan
 *     are serialised on one stream by the caller, and so are calls that write one layer's
 *     gradients (reference contract: pure and reentrant).
 */
#ifndef TLORA_H_
#define TLORA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TLORA_ABI_VERSION 5

enum tlora_status {
  TLORA_OK = 0,
  TLORA_ERR_ARG = 1,       /* bad argument (null pointer, negative size, bad enum)     */
  TLORA_ERR_SHAPE = 2,     /* shape mismatch (fused_lora.hpp:66-76 messages)           */
  TLORA_ERR_REGISTRY = 3,  /* unknown / unregistered adapter slot (":73 has no adapter") */
  TLORA_ERR_PLAN = 4,      /* invalid plan / partition / AIMD arguments                  */
  TLORA_ERR_CUDA = 5,      /* CUDA runtime / driver failure                              */
  TLORA_ERR_NO_DEVICE = 6, /* no sm_100 device available: there is no CPU fallback      */
  TLORA_ERR_NCCL = 7       /* NCCL missing or a collective failed                        */
};

enum tlora_dtype { TLORA_F64 = 0, TLORA_F32 = 1, TLORA_BF16 = 2 };
enum tlora_where { TLORA_HOST = 0, TLORA_DEVICE = 1 };

typedef struct tlora_layer tlora_layer;
typedef struct tlora_plan tlora_plan;
typedef struct tlora_comm tlora_comm;

/* One output tile of a plan launch and its (up to two) K-segments, in elements.
 * Mirrors tlora::TileDesc in paper_2602_07263_b200/csrc/lora_gemm.cuh. */
typedef struct tlora_tile {
  int32_t m0, n0;
  int32_t kb0, ke0;
  int32_t kb1, ke1;
  int32_t split;
  int32_t pad;
} tlora_tile;

/* Which launch of a plan a tile table belongs to. */
enum tlora_launch {
  TLORA_L_SHRINK = 0,  /* H   = X·A_j (masked to job columns)             */
  TLORA_L_FWD = 1,     /* Y   = X·W + H·B_j (K-extension over rank range)  */
  TLORA_L_DH = 2,      /* dH  = dY·B_jᵀ (masked)                           */
  TLORA_L_DX = 3,      /* dX  = dY·Wᵀ + dH·A_jᵀ                            */
  TLORA_L_DB = 4,      /* dB_j = H_jᵀ·dY_j     (fp32, token-range K)       */
  TLORA_L_DA = 5,      /* dA_jᵀ = dH_jᵀ·X_j    (fp32, token-range K)       */
  /* the same shrink / dH work on 256-token CTA-pair tiles (N = 128 or 256 packed rank
   * columns), run as secondary tiles inside another layer's fused GEMM launch */
  TLORA_L_SHRINK2 = 6,
  TLORA_L_DH2 = 7,
  TLORA_L_COUNT = 8
};
/* launch kinds reported by the live profiler (tlora_profile_end arrays) */
#define TLORA_PROF_KINDS 6

typedef struct tlora_plan_info {
  int64_t tokens;          /* T                                                    */
  int64_t d, k;            /* layer dims                                           */
  int32_t num_slots;       /* registry size                                        */
  int32_t rank_pad_total;  /* R: packed rank columns (sum of round_up(r_j, 8))     */
  int32_t num_tiles[TLORA_L_COUNT];
  int32_t splits_db, splits_da; /* max split-K planes of the gradient launches    */
  int64_t useful_ext_cols;  /* sum over fwd M-tiles of ranks actually owned         */
  int64_t packed_ext_cols;  /* sum over fwd M-tiles of K-extension columns issued   */
} tlora_plan_info;

/* ---- library / errors -------------------------------------------------------- */
const char* tlora_last_error(void);
int tlora_abi_version(void);
/* Fails with TLORA_ERR_NO_DEVICE unless device `device` is an sm_100 GPU. */
int tlora_device_check(int device, int* sm_count);

/* ---- device buffers (so non-CUDA hosts — C++, cgo, JNI, ctypes — need no cudart) --- */
int tlora_buffer_alloc(int device, size_t bytes, void** out);
int tlora_buffer_free(int device, void* ptr);
/* count elements host -> device, converting src_dtype -> dst_dtype (f64/f32/bf16 in,
 * f32/bf16 out; bf16 rounding is round-to-nearest-even). Synchronous w.r.t. the host
 * buffer: it may be reused when the call returns. */
int tlora_copy_to_device(void* dst, int dst_dtype, const void* src_host, int src_dtype,
                         int64_t count, void* stream);
/* count elements device -> host with conversion (f32/bf16 in, f64/f32/bf16 out).
 * Returns after the data has landed in dst_host. */
int tlora_copy_to_host(void* dst_host, int dst_dtype, const void* src, int src_dtype,
                       int64_t count, void* stream);
int tlora_stream_sync(void* stream);
/* Enqueue-only helpers for copy-engine collectives over peer-mapped (NVLink) memory:
 * cudaMemcpyAsync(cudaMemcpyDefault); a 32-bit flag write ordered after all prior work
 * of the stream (cuStreamWriteValue32, fenced); a wait until *addr >= value
 * (cuStreamWaitValue32 GEQ). No SM is used by any of the three. */
int tlora_copy_async(void* dst, const void* src, size_t bytes, void* stream);
int tlora_stream_write_u32(void* stream, void* addr, uint32_t value);
int tlora_stream_wait_u32(void* stream, void* addr, uint32_t value);

/* ---- layer: one adapted projection (frozen base W + adapter registry) --------- */
/* ranks[num_slots]: registry layout in reference adapter order (std::map by job_id,
 * fused_lora.hpp:48-53). Slot s owns packed rank columns [off_s, off_s + ranks[s]). */
int tlora_layer_create(int device, int64_t d, int64_t k, int32_t num_slots,
                       const int32_t* ranks, tlora_layer** out);
int tlora_layer_destroy(tlora_layer* layer);
/* Base weight W: d x k row-major. Stored frozen as bf16 in both K-major layouts. */
int tlora_layer_set_base(tlora_layer* layer, const void* W, int dtype, int where, void* stream);
/* Adapter of `slot`: A is d x r, B is r x k (row-major), r = ranks[slot]. */
int tlora_layer_set_adapter(tlora_layer* layer, int32_t slot, const void* A, const void* B,
                            int dtype, int where, void* stream);
/* Packed-rank column offset of each slot (num_slots entries) and R. */
int tlora_layer_layout(const tlora_layer* layer, int32_t* offsets, int32_t* rank_pad_total);
/* Zero the fp32 adapter-gradient accumulators. */
int tlora_layer_zero_grad(tlora_layer* layer, void* stream);
/* Device pointers of the packed fp32 gradients: dAᵀcat (R x d) and dBcat (R x k). */
int tlora_layer_grad_ptrs(tlora_layer* layer, float** dAT, float** dB);
/* Copy one slot's gradients out: dA is d x r, dB is r x k (row-major fp32). */
int tlora_layer_read_grad(tlora_layer* layer, int32_t slot, float* dA, float* dB, int where,
                          void* stream);

/* ---- fused multi-job AdamW over the packed adapters (optimizer step) -- */
/* Per-slot learning rate and (decoupled) weight decay (num_slots entries; weight_decay
 * may be NULL = 0); shared beta1/beta2/eps. Resets the moments and step counters. The
 * fp32 masters are the values given to tlora_layer_set_adapter. */
int tlora_layer_set_optimizer(tlora_layer* layer, const float* lr, const float* weight_decay,
                              float beta1, float beta2, float eps);
/* One AdamW step of every slot on grads * grad_scale (e.g. 1/world for a DP mean); writes
 * the fp32 masters/moments and refreshes the bf16 operand layouts the kernels read. */
int tlora_layer_optimizer_step(tlora_layer* layer, float grad_scale, void* stream);
/* The same step restricted to the slots with present[slot] != 0 (device int32 array of
 * num_slots entries, e.g. tlora_plan_present_mask of the step's batch): a job with no
 * tokens in the step takes no optimizer step (masters, moments and step counter stay as
 * they are). present == NULL updates every slot (= tlora_layer_optimizer_step). */
int tlora_layer_optimizer_step_masked(tlora_layer* layer, const int32_t* present, float grad_scale,
                                      void* stream);
/* AdamW on the packed rows [row_lo, row_hi) only (even bounds): a data-parallel rank's
 * shard of the sharded optimizer (tlora_layer_dp_shard). Step counters advance for every
 * present slot, so all ranks stay in step. */
int tlora_layer_optimizer_step_rows(tlora_layer* layer, const int32_t* present, float grad_scale,
                                    int64_t row_lo, int64_t row_hi, void* stream);
/* Copy one slot's fp32 master adapter out: A is d x r, B is r x k. */
int tlora_layer_read_adapter(tlora_layer* layer, int32_t slot, float* A, float* B, int where,
                             void* stream);

/* ---- plan: the rank-aware tile-packing / indexing plan of one (nano-)batch ------ */
/* token_slot[T] (host): owning slot of each token row, any interleaving allowed
 * (fused_lora.hpp:28-31). Errors: slot out of range -> TLORA_ERR_REGISTRY. A plan may be
 * used with any layer of the same registry layout (d, k, ranks) on the same device. */
int tlora_plan_create(tlora_layer* layer, int64_t tokens, const int32_t* token_slot,
                      tlora_plan** out);
/* Gathered plan for interleaved batches: the plan of the stable job-sorted order of
 * token_slot (rows of one job keep their order, fused_lora.hpp:56-61), so every tile sees
 * one job's rank window, as for a job-contiguous batch. Operands X / dY passed with it must
 * be in that gathered order (tlora_gather_rows); the H / dH stashes stay in it; the fused
 * forward / dX epilogues store Y / dX row i straight to the caller's token row_map[i], so
 * outputs come back in the original order. Not accepted by the reduce-scatter epilogue. */
int tlora_plan_create_gathered(tlora_layer* layer, int64_t tokens, const int32_t* token_slot,
                               tlora_plan** out);
/* row_map[i] = original token of gathered row i (identity for a plain plan). Synchronous. */
int tlora_plan_row_map(const tlora_plan* plan, int32_t* row_map);
/* dst[i][r, :] = src[i][row_map[r], :] for n bf16 row-major T x width[i] tensors (width a
 * multiple of 8, 16-byte aligned, dst != src); four tensors per launch. Enqueue-only. */
int tlora_gather_rows(const tlora_plan* plan, int32_t n, const void* const* src, void* const* dst,
                      const int64_t* width, void* stream);
int tlora_plan_destroy(tlora_plan* plan);
/* Device pointer (valid for the plan's lifetime) to num_slots int32 flags: 1 if the slot
 * owns at least one token of this plan's batch. */
int tlora_plan_present_mask(const tlora_plan* plan, const int32_t** present);
int tlora_plan_get_info(const tlora_plan* plan, tlora_plan_info* info);
/* Copy the tile table of `launch` into out[cap]; *count gets the table length. */
int tlora_plan_get_tiles(const tlora_plan* plan, int launch, tlora_tile* out, int32_t cap,
                         int32_t* count);

/* Debug readback of what the device actually holds for a plan: the tile table of `launch`
 * as uploaded (copied back from device memory; cap entries max) and, if token_slot is
 * non-NULL, the uploaded owner slot of every token (tokens entries). Synchronous. Lets a
 * test memcmp the device plan against the plan oracle. */
int tlora_plan_read_device(const tlora_plan* plan, int launch, tlora_tile* out, int32_t cap,
                           int32_t* count, int32_t* token_slot);
/* Host-only plan builder (no device needed): the same tile table tlora_plan_create
 * uploads, for the registry layout `ranks` and the token->slot map. For bit-exact checks
 * against the plan oracle and for planning on a host without a GPU. */
int tlora_plan_tiles_host(int64_t d, int64_t k, int32_t num_slots, const int32_t* ranks,
                          int64_t tokens, const int32_t* token_slot, int launch, tlora_tile* out,
                          int32_t cap, int32_t* count);

/* Host-only: the LPT schedule a plan uploads for its combined dB+dA gradient launch on
 * `ctas` persistent CTAs: CTA c runs tiles idx[off[c] .. off[c+1]) of the
 * concatenated (dB table, dA table). off has ctas + 1 entries; *count gets the tile count. */
int tlora_plan_grad_schedule_host(int64_t d, int64_t k, int32_t num_slots, const int32_t* ranks,
                                  int64_t tokens, const int32_t* token_slot, int32_t ctas,
                                  int32_t* off, int32_t* idx, int32_t cap, int32_t* count);

/* ---- compute (enqueue-only) ----------------------------------------------------- */
/* Forward: Y = X·W + scatter_j((X_j·A_j)·B_j). X: T x d bf16, Y: T x k (bf16 or f32),
 * H_stash: T x R bf16 (the per-token low-rank intermediate, kept for backward). */
int tlora_forward(tlora_layer* layer, const tlora_plan* plan, const void* X, void* Y,
                  int y_dtype, void* H_stash, void* stream);
/* Backward: dX = dY·Wᵀ + scatter_j(dH_j·A_jᵀ) (skipped when dX == NULL);
 * grads  (fp32, packed)  = beta·grads + [dA_j = X_jᵀ·dH_j, dB_j = H_jᵀ·dY_j].
 * dY: T x k bf16, X: T x d bf16, H_stash from tlora_forward. */
int tlora_backward(tlora_layer* layer, const tlora_plan* plan, const void* dY, const void* X,
                   const void* H_stash, void* dX, float beta, void* stream);

/* Per-launch entry points of the same computation, for drivers that interleave
 * collectives between the launches (tensor-parallel nano-batch pipeline). tlora_forward
 * = shrink + gemm; tlora_backward = dh + dx + grad_b(H, dY) + grad_a(X, dH). H / dH are
 * T x R bf16, masked to each token's own packed-rank columns (zero elsewhere), so partial
 * H / dH summed across ranks stay valid operands. Calls on one plan are serialised on
 * one stream (the split-K partial planes belong to the plan). */
int tlora_forward_shrink(tlora_layer* layer, const tlora_plan* plan, const void* X, void* H,
                         void* stream);
int tlora_forward_gemm(tlora_layer* layer, const tlora_plan* plan, const void* X, const void* H,
                       void* Y, int y_dtype, void* stream);
/* Row-parallel tensor-parallel forward with the reduce-scatter fused into the GEMM: each
 * output row r (token of this plan) is stored, as its tile finishes, into the receive
 * buffer of the rank that owns it (dest = r / (T / world)) through NVLink peer memory.
 * recv_ptrs[world]: every rank's receive buffer [world][slot_rows][k] bf16 (peer-mapped,
 * e.g. symmetric memory); this rank writes slot `rank`, rows dst_row0 + r % (T / world).
 * After a cross-rank barrier, tlora_reduce_slots sums the slots in fixed order. */
/* tlora_forward_gemm with the dH of `next` (dH_next = dY_next·Bᵀcat masked, as
 * tlora_backward_dh) as extra tiles: a training step's LAST forward launch can carry the
 * FIRST dH of its backward (dY is an input of the step). zero_next as above. */
int tlora_forward_gemm_dh(tlora_layer* layer, const tlora_plan* plan, const void* X,
                          const void* H, void* Y, int y_dtype, tlora_layer* next,
                          const tlora_plan* next_plan, const void* dY_next, void* dH_next,
                          int zero_next, void* stream);
/* tlora_forward_gemm of `layer` with the shrink of `next` (H_next = X_next·Aᵀcat masked, as
 * tlora_forward_shrink) carried as extra CTA-pair tiles of the SAME launch (plan table
 * TLORA_L_SHRINK2 of next_plan), so the next projection's shrink fills this GEMM's tail
 * instead of paying its own launch ramp. H_next must be zero outside next_plan's windows:
 * zero_next = 1 memsets it first; 0 when the caller keeps it zeroed (same-slot plans only
 * ever write the same windows). H_next must not alias H, Y or X. Bit-identical to the
 * two separate calls. */
int tlora_forward_gemm_shrink(tlora_layer* layer, const tlora_plan* plan, const void* X,
                              const void* H, void* Y, int y_dtype, tlora_layer* next,
                              const tlora_plan* next_plan, const void* X_next, void* H_next,
                              int zero_next, void* stream);
int tlora_forward_gemm_rs(tlora_layer* layer, const tlora_plan* plan, const void* X, const void* H,
                          void* const* recv_ptrs, int32_t world, int32_t rank, int64_t slot_rows,
                          int64_t dst_row0, void* stream);
/* out[rows x k] = sum_{p < world} recv[p][row0 .. row0 + rows)[k] (fp32 sum, bf16 out). */
int tlora_reduce_slots(const void* recv, int32_t world, int64_t slot_rows, int64_t row0,
                       int64_t rows, int64_t k, void* out, void* stream);
int tlora_backward_dh(tlora_layer* layer, const tlora_plan* plan, const void* dY, void* dH,
                      void* stream);
/* dX = dY·Wᵀ + dH·Aᵀ + beta·dX (beta = 1 sums the dX of projections sharing an input) */
int tlora_backward_dx(tlora_layer* layer, const tlora_plan* plan, const void* dY, const void* dH,
                      void* dX, float beta, void* stream);
/* tlora_backward_dx of `layer` with the dH of `next` (dH_next = dY_next·Bᵀcat masked, as
 * tlora_backward_dh) as extra tiles of the same launch (plan table TLORA_L_DH2); zero_next
 * as in tlora_forward_gemm_shrink. Bit-identical to the two separate calls. */
int tlora_backward_dx_dh(tlora_layer* layer, const tlora_plan* plan, const void* dY,
                         const void* dH, void* dX, float beta, tlora_layer* next,
                         const tlora_plan* next_plan, const void* dY_next, void* dH_next,
                         int zero_next, void* stream);
/* tlora_backward_dx of `layer` with the SHRINK of `next` (H_next = X_next·Aᵀcat masked, as
 * tlora_forward_shrink) as extra tiles of the same launch: the last dX launch of one
 * nano-batch carries the first shrink of the next nano-batch's forward. */
int tlora_backward_dx_shrink(tlora_layer* layer, const tlora_plan* plan, const void* dY,
                             const void* dH, void* dX, float beta, tlora_layer* next,
                             const tlora_plan* next_plan, const void* X_next, void* H_next,
                             int zero_next, void* stream);
/* Both adapter gradients in ONE persistent launch (+ one split-K reduce): dB from (H, dY)
 * and dA from (X, dH); = tlora_backward_grad_b then tlora_backward_grad_a. */
int tlora_backward_grads(tlora_layer* layer, const tlora_plan* plan, const void* H,
                         const void* dY, const void* X, const void* dH, float beta, void* stream);
int tlora_backward_grad_b(tlora_layer* layer, const tlora_plan* plan, const void* H,
                          const void* dY, float beta, void* stream);
int tlora_backward_grad_a(tlora_layer* layer, const tlora_plan* plan, const void* X,
                          const void* dH, float beta, void* stream);

/* Cap the persistent grid sizes on `device`: fused GEMM launches (fwd / dX) use at most
 * gemm_sms SMs (rounded down to CTA pairs), low-rank launches (shrink, dH, dA, dB) at
 * most lowrank_sms. With gemm_sms + lowrank_sms <= SM count a driver can run the two
 * classes concurrently on two streams. 0 = no cap (default). */
int tlora_set_sm_budget(int device, int32_t gemm_sms, int32_t lowrank_sms);

/* Tile scheduler of the fused GEMM launches on `device`: 0 = static per-CTA tile lists,
 * 1 = dynamic (a per-stream ticket counter; CTAs that start late because other kernels hold
 * SMs take fewer tiles), -1 = the TLORA_DYN_SCHED environment default (static). Results are
 * bitwise identical either way. The data-parallel step executor selects 1 for its device. */
int tlora_set_tile_scheduler(int device, int mode);

/* ---- live launch profiling (CUDA events on each launch's own stream) ------------- */
/* Between begin and end every GEMM launch is bracketed by CUDA events. end() waits for
 * them and returns, per tlora_launch kind, the launch count, summed device ms and the
 * summed algorithmic FLOPs (padding and packing waste excluded). Arrays have
 * TLORA_PROF_KINDS entries; any may be NULL. A fused GEMM launch that also carries another
 * layer's shrink / dH tiles is booked under its main kind (FWD / DX). */
int tlora_profile_begin(void);
/* Total number of kernels this library has enqueued since load (monotonic). */
long long tlora_launch_count(void);
int tlora_profile_end(int32_t* counts, double* total_ms, double* total_flops);

/* ---- reference cost model (bit-identical to fused_lora.hpp:95-116, :139-163) ----- */
/* tokens_per_slot[num_slots], ranks[num_slots], in reference adapter order. */
int tlora_op_cost(int64_t tokens, int64_t d, int64_t k, int32_t num_slots,
                  const int64_t* tokens_per_slot, const int32_t* ranks, int fused,
                  double* flops, double* bytes_moved, long long* kernel_launches);

/* ---- job segments (fused_lora.hpp:56-61 detail::segment_rows, for every job at once) -- */
/* CSR form of the ragged batch: offsets[s] .. offsets[s+1] index into perm the rows owned
 * by slot s, ascending within a slot (= segment_rows of that job); perm is therefore the
 * stable job-sorted permutation (device row i <- token perm[i]). Host-only, O(T + S).
 * perm: tokens entries; offsets: num_slots + 1 entries. Slots outside [0, num_slots)
 * -> TLORA_ERR_REGISTRY. */
int tlora_segments(int64_t tokens, const int32_t* token_slot, int32_t num_slots, int64_t* perm,
                   int64_t* offsets);

/* ---- nano-batch plan + AIMD (nano_pipeline.hpp:51-60, 99-112) --------------------- */
/* per_nano must hold min(n, group_batch) entries; *n_out receives the clamped N. */
int tlora_partition(int32_t group_batch, int32_t n, int32_t* n_out, int32_t* per_nano);
/* has_prev/t_prev carry std::optional<double>; updates n / has_prev / t_prev in place. */
int tlora_aimd_step(int32_t* n, int32_t* has_prev, double* t_prev, int32_t alpha, double beta,
                    double tau_rel, double t_t);

/* ---- communicator (SURVEY §8(b) "comm"; no reference counterpart: the reference
 * simulates its multi-GPU timeline, sim_engine.hpp:306-315) ------------------------------
 * One communicator per rank over NCCL (loaded at run time; TLORA_ERR_NCCL if absent).
 * world = tp_size * dp; rank = dp_index * tp_size + tp_index. Groups: WORLD, TP (the
 * tp_size consecutive ranks of one replica) and DP (ranks with the same tp_index).
 * Rank 0 makes the id, the host shares it out of band, every rank calls create
 * (collective). Collectives are enqueued on `stream`. */
#define TLORA_UNIQUE_ID_BYTES 128
enum tlora_group { TLORA_GROUP_WORLD = 0, TLORA_GROUP_TP = 1, TLORA_GROUP_DP = 2 };
int tlora_comm_get_unique_id(uint8_t* id /* [TLORA_UNIQUE_ID_BYTES] */);
int tlora_comm_create(int device, const uint8_t* id, int32_t world, int32_t rank,
                      int32_t tp_size, tlora_comm** out);
int tlora_comm_destroy(tlora_comm* comm);
int tlora_comm_info(const tlora_comm* comm, int32_t* world, int32_t* rank, int32_t* tp_size,
                    int32_t* dp_size);
/* recv = concat over the group's ranks of send (send_count elements each) */
int tlora_comm_all_gather(tlora_comm* comm, int group, const void* send, void* recv,
                          size_t send_count, int dtype, void* stream);
/* recv (recv_count elements) = this rank's slice of the sum over the group of send */
int tlora_comm_reduce_scatter(tlora_comm* comm, int group, const void* send, void* recv,
                              size_t recv_count, int dtype, void* stream);
int tlora_comm_all_reduce(tlora_comm* comm, int group, const void* send, void* recv,
                          size_t count, int dtype, int average, void* stream);
/* Data-parallel exchange: all-reduce (sum, or mean if average) of the layer's fp32
 * adapter gradients dA / dB over `group` (normally TLORA_GROUP_DP), in place. */
int tlora_layer_allreduce_grads(tlora_layer* layer, tlora_comm* comm, int group, int average,
                                void* stream);

/* ---- synthetic data (seeded, deterministic on any device) --------------------------- */
/* dst[i] = scale * N(0,1) sample i of the counter-based generator keyed by seed (bf16 or
 * f32 device buffer, count elements). Lets C++ hosts and tests build identical inputs. */
int tlora_fill_normal(void* dst, int dtype, int64_t count, uint64_t seed, float scale,
                      void* stream);

/* ---- rank-aware nano-batch map (nano_pipeline.hpp:51-60 gives only counts) -------------
 * Samples enumerated job-major (slot 0's batch[0] samples, then slot 1's, ...). per_nano =
 * partition(sum batch, n) (bit-exact); samples are placed by weight[slot] descending (ties:
 * lower slot), each on the least-loaded nano-batch with room left (ties: lower nano), which
 * fixes nano_slot[n_out x num_slots] (samples of slot s in nano i); job s's samples then go
 * to the nano-batches in nano order (its first nano_slot[0][s] to nano 0, ...): sample_nano
 * [sum batch]. Errors as partition (TLORA_ERR_PLAN). Host-only. */
int tlora_nano_assign(int32_t num_slots, const int32_t* batch, const int64_t* weight, int32_t n,
                      int32_t* n_out, int32_t* per_nano, int32_t* sample_nano, int32_t* nano_slot);

/* ---- the layer-set training step executor (the caller of the path: the iteration body of
 * sim_engine.hpp:306-315 executed for real) ---------------------------------------------
 * A step = for each nano-batch of the rank-aware map of N: forward of every (layer,
 * projection) key in order, then backward in reverse order (gradients accumulate over the
 * nano-batches), then the fused masked AdamW of every key (after the key's gradient
 * all-reduce over the DP group when a communicator is given). N = nano_fixed if > 0, else
 * the AIMD controller's n (nano_pipeline.hpp:99-112, driven by the CUDA-event time of every
 * step, clamped to the combined batch as sim_engine.hpp:314). The step owns its layers
 * (tlora_step_layer: set base / adapters / optimizer through the layer API) and its
 * step-sized buffers (tlora_step_buffer); nano-batch i is the row range
 * [nano_t0[i], nano_t0[i+1]) of every buffer (tlora_step_layout). */
typedef struct tlora_step tlora_step;
enum tlora_step_flags {
  TLORA_STEP_SIDE_GRADS = 1, /* dB+dA (and AdamW) of each key on a side stream             */
  TLORA_STEP_GRAPH = 2,      /* capture each (N, input set) step into a CUDA graph after its
                                first eager run and replay it (single replica only)        */
  TLORA_STEP_EARLY_GRADS = 4, /* a key's dB+dA waits only for the launch that produced its
                                 dH, so it may overlap the key's own dX launch              */
  TLORA_STEP_SHARDED_OPT = 8  /* with a communicator: reduce-scatter the gradients, AdamW on
                                 this rank's row shard, all-gather the bf16 operands         */
};
enum tlora_run_flags {
  TLORA_RUN_EAGER = 1, /* launch eagerly even if a graph exists                          */
  TLORA_RUN_TRACE = 2  /* eager, with a timing event after every op (tlora_step_trace)   */
};
typedef struct tlora_step_desc {
  int32_t device;
  int32_t num_layers;
  int32_t num_projections;
  const int64_t* proj_d;      /* [P] in-features                                          */
  const int64_t* proj_k;      /* [P] out-features                                         */
  const int32_t* proj_input;  /* [P] input group: projections with one id read one X       */
  int32_t num_slots;
  const int32_t* ranks;       /* [S] registry layout, reference adapter order             */
  const int32_t* batch;       /* [S] samples of each job in the step (JobSpec.batch_size) */
  const int32_t* seq_len;     /* [S] tokens per sample (JobSpec.seq_len)                  */
  int32_t y_dtype;            /* TLORA_BF16 or TLORA_F32                                  */
  int32_t flags;              /* tlora_step_flags                                         */
  int32_t dh_ring;            /* dH ring depth, 0 = 8                                     */
  int32_t input_sets;         /* 1 or 2 input buffer sets (double-buffered host inputs)   */
  int32_t nano_init;          /* AIMD initial n, 0 = 4 (sim_engine.hpp:63)                */
  int32_t nano_fixed;         /* > 0: fixed N, no AIMD (the reference's config.fixed_n)   */
  int32_t aimd_alpha;         /* 0 = 4                                                    */
  double aimd_beta;           /* 0 = 0.5                                                  */
  double aimd_tau_rel;        /* >= 0                                                     */
} tlora_step_desc;
typedef struct tlora_step_stats {
  int32_t nano_used;      /* N of the step just run                                        */
  int32_t next_nano;      /* N the controller chose for the next step                      */
  double ms;              /* CUDA-event time of the step (see tlora_step_run; -1 unknown)  */
  int32_t replayed_graph; /* 1 if the step was a CUDA-graph replay                         */
  long long launches;     /* kernels in the step (a replay re-launches the eager run's)     */
  int64_t tokens;
} tlora_step_stats;
enum tlora_buffer_kind {
  TLORA_BUF_X = 0,  /* index = input group, per input set: T x d  bf16                     */
  TLORA_BUF_DY = 1, /* index = projection, per input set: T x k  bf16 (upstream gradient) */
  TLORA_BUF_Y = 2,  /* index = projection: T x k (y_dtype)                                 */
  TLORA_BUF_DX = 3, /* index = projection: T x d bf16                                      */
  TLORA_BUF_H = 4   /* index = key (layer * P + projection): T x R bf16 stash             */
};
int tlora_step_create(const tlora_step_desc* desc, tlora_comm* comm /* NULL: one replica */,
                      tlora_step** out);
int tlora_step_destroy(tlora_step* step);
int tlora_step_layer(tlora_step* step, int32_t layer, int32_t proj, tlora_layer** out);
int tlora_step_buffer(tlora_step* step, int32_t kind, int32_t index, int32_t set, void** ptr,
                      int64_t* rows, int64_t* cols);
/* Token layout for nano count n (plans are built on first use): *n_out = min(n, samples),
 * nano_t0[n_out + 1] row offsets, nano_slot[n_out x S], sample_row[samples] first row of
 * each sample (samples job-major). Any output may be NULL. */
int tlora_step_layout(tlora_step* step, int32_t n, int32_t* n_out, int64_t* nano_t0,
                      int32_t* nano_slot, int64_t* sample_row);
/* Switch the nano-batch controller: nano_fixed > 0 pins N; 0 = AIMD from nano_init (0 = 4)
 * with a fresh AimdState (alpha 0 = 4, beta 0 = 0.5). Layouts, plans and graphs of N values
 * seen before are kept. */
int tlora_step_set_controller(tlora_step* step, int32_t nano_fixed, int32_t nano_init,
                              int32_t aimd_alpha, double aimd_beta, double aimd_tau_rel);
/* N the next tlora_step_run will use (fill the inputs in that layout). */
int tlora_step_next_n(const tlora_step* step, int32_t* n);
/* One training step on input set `set`, enqueued on `stream`. Under AIMD (nano_fixed 0) or
 * TLORA_RUN_TRACE the call waits for the step (its time feeds the controller) and stats->ms
 * is this step's time; with a fixed N it returns right after enqueueing and stats->ms is
 * the time of the latest completed step (-1 if none). stats may be NULL. */
int tlora_step_run(tlora_step* step, int32_t set, int32_t flags, void* stream,
                   tlora_step_stats* stats);

/* After a TLORA_RUN_TRACE step: its ops (schedule order) and each op's completion time on
 * its own stream in ms after the step's start event (ops, end_ms: cap entries; NULL ok). */
typedef struct tlora_step_op tlora_step_op;
int tlora_step_trace(const tlora_step* step, tlora_step_op* ops, double* end_ms, int32_t cap,
                     int32_t* count);

/* One op of the step schedule (host-only view for tests and drivers). */
enum tlora_op_kind { TLORA_OP_SHRINK = 0, TLORA_OP_FWD = 1, TLORA_OP_DH = 2, TLORA_OP_DX = 3,
                     TLORA_OP_GRADS = 4, TLORA_OP_ALLREDUCE = 5, TLORA_OP_ADAMW = 6,
                     TLORA_OP_REDUCE_SCATTER = 7, TLORA_OP_ALLGATHER = 8 };
enum tlora_stream_id { TLORA_STREAM_MAIN = 0, TLORA_STREAM_SIDE = 1, TLORA_STREAM_COMM = 2 };
typedef struct tlora_step_op {
  int32_t kind, stream, key, nano;
  int32_t slot;                         /* dH ring slot read (DX, GRADS), -1            */
  int32_t sec_kind, sec_key, sec_nano;  /* secondary tiles of a FWD / DX launch, -1     */
  int32_t sec_slot;                     /* ring slot the secondary dH writes, -1         */
  int32_t beta;                         /* GRADS: 1 = accumulate onto earlier nano-batches */
  int32_t wait0, wait1;                 /* ops (on other streams) waited for, -1         */
} tlora_step_op;
/* side_grads: 0 = gradients on the main stream, 1 = side stream, 2 = side stream with
 * TLORA_STEP_EARLY_GRADS. data_parallel: 0 = one replica, 1 = all-reduce, 2 = sharded
 * optimizer (TLORA_STEP_SHARDED_OPT). */
int tlora_step_schedule_host(int32_t keys, int32_t nano, int32_t ring, int32_t side_grads,
                             int32_t data_parallel, tlora_step_op* out, int32_t cap,
                             int32_t* count);

/* ---- tensor-parallel layer-set step (C++ host; the TP path of SURVEY §8(e)) ------------
 * One process per GPU, the communicator's world = the TP group. Column-parallel projections
 * (q, k, v, gate, up: proj_row_parallel 0) hold W[:, k/P], B_j[:, k/P] and the replicated
 * A_j; row-parallel ones (o, down: 1) hold W[d/P, :], A_j[d/P, :] and the replicated B_j.
 * Sequence-parallel activations between groups. Per nano-batch (rank-aware map, AIMD as
 * tlora_step_run): shrink on the SP shard -> all-gather [X | H] -> column GEMMs; row GEMMs
 * -> reduce-scatter Y (fused into the GEMM epilogue over NVLink peer memory with
 * TLORA_TP_FUSED_RS); backward all-gather dY (row), reduce-scatter [dX | dH] (column);
 * the replicated adapter halves' gradients are all-reduced once per step; masked AdamW.
 * Collectives of nano n+1 / n-1 run on a comm stream while nano n's GEMMs run; with
 * TLORA_TP_COPY_ENGINE the all-gathers / reduce-scatters are copy-engine pushes into
 * peer-mapped (CUDA IPC) buffers with stream-memory-op flags instead of NCCL kernels. */
typedef struct tlora_tp_step tlora_tp_step;
enum tlora_tp_flags {
  TLORA_TP_FUSED_RS = 1,     /* row-parallel reduce-scatter fused into the GEMM epilogue  */
  TLORA_TP_COPY_ENGINE = 2,  /* all-gather / reduce-scatter by copy-engine push            */
  TLORA_TP_SIDE_GRADS = 4    /* adapter-gradient launches on a side stream                 */
};
typedef struct tlora_tp_desc {
  int32_t device;
  int32_t num_projections;
  const int64_t* proj_d;             /* [P] full in-features                             */
  const int64_t* proj_k;             /* [P] full out-features                            */
  const int32_t* proj_input;         /* [P] input group of the column-parallel projections */
  const int32_t* proj_row_parallel;  /* [P] 1 = row-parallel, 0 = column-parallel        */
  int32_t num_slots;
  const int32_t* ranks;
  const int32_t* batch;
  const int32_t* seq_len;
  int32_t flags;                     /* tlora_tp_flags                                    */
  int32_t nano_init, nano_fixed, aimd_alpha;
  double aimd_beta, aimd_tau_rel;
} tlora_tp_desc;
enum tlora_tp_buffer_kind {
  TLORA_TP_X_SHARD = 0,   /* index = input group: T/P x d   (column inputs, SP shard)   */
  TLORA_TP_X_LOC = 1,     /* index = projection (row): T x d/P                           */
  TLORA_TP_DY = 2,        /* index = projection (column): T x k/P                        */
  TLORA_TP_DY_SHARD = 3,  /* index = projection (row): T/P x k                           */
  TLORA_TP_Y = 4,         /* index = projection (column): T x k/P                        */
  TLORA_TP_Y_SHARD = 5,   /* index = projection (row): T/P x k                           */
  TLORA_TP_DX_SHARD = 6,  /* index = input group: T/P x d (summed over the group)        */
  TLORA_TP_DX_LOC = 7     /* index = projection (row): T x d/P                           */
};
int tlora_tp_create(const tlora_tp_desc* desc, tlora_comm* comm, tlora_tp_step** out);
int tlora_tp_destroy(tlora_tp_step* step);
/* This rank's shard layer of projection p (set base / adapters / optimizer through it). */
int tlora_tp_layer(tlora_tp_step* step, int32_t proj, tlora_layer** out);
int tlora_tp_buffer(tlora_tp_step* step, int32_t kind, int32_t index, void** ptr, int64_t* rows,
                    int64_t* cols);
/* nano_t0[n_out + 1] (global token rows) and nano_slot[n_out x S] of nano count n. */
int tlora_tp_layout(tlora_tp_step* step, int32_t n, int32_t* n_out, int64_t* nano_t0,
                    int32_t* nano_slot);
/* One training step (collective: every rank calls it). Under AIMD (nano_fixed 0) it waits
 * for the step's CUDA-event time, averaged over the group before the AIMD update (so all
 * ranks agree on the next N); with a fixed N it returns after enqueueing and stats->ms is
 * the latest completed step's time (-1 if none). */
int tlora_tp_run(tlora_tp_step* step, int32_t flags, void* stream, tlora_step_stats* stats);
/* After a tlora_tp_run with TLORA_RUN_TRACE: per nano-batch the summed compute spans (main
 * stream, forward + backward) and boundary-traffic spans (comm stream), ms — the measured
 * PipelineTrace t_comp / t_comm (nano_pipeline.hpp:28-34). */
int tlora_tp_trace(const tlora_tp_step* step, double* t_comp_ms, double* t_comm_ms, int32_t cap,
                   int32_t* count);

/* Sharded data-parallel optimizer (the alternative to tlora_layer_allreduce_grads + a full
 * AdamW on every rank): the packed rank rows are split evenly over `group`; this rank owns
 * [row_lo, row_hi). reduce_scatter_grads sums the fp32 gradients of the owned rows over the
 * group (in place); tlora_layer_optimizer_step_rows updates them; allgather_operands
 * gathers every rank's refreshed bf16 rows (Aᵀcat, Bcat) and rebuilds the transposed copies
 * the kernels read. fp32 masters / moments of rows a rank does not own are not kept
 * current on that rank. Needs R % group size == 0 with even shards. */
int tlora_layer_dp_shard(const tlora_layer* layer, const tlora_comm* comm, int group,
                         int64_t* row_lo, int64_t* row_hi);
int tlora_layer_reduce_scatter_grads(tlora_layer* layer, tlora_comm* comm, int group,
                                     void* stream);
int tlora_layer_allgather_operands(tlora_layer* layer, tlora_comm* comm, int group, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TLORA_H_ */
