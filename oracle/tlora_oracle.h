/*
 * tlora_oracle.h — CPU oracle for the fused multi-LoRA layer. TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this.
 * It is the checker, never the thing measured or shipped; the product path
 * (paper_2602_07263_b200/libtlora.so) has no CPU fallback.
 *
 * Parity pinning: the forward restatement is checked against golden vectors produced by
 * the UNMODIFIED reference (oracle/ref_harness.cpp -> tests/golden/), at the reference's
 * own tolerance (1e-9 relative, acceptance.cpp:91-94). The backward has no reference
 * (SPEC.md:146); it is pinned to the reference forward by bilinearity identities
 * (tests/test_oracle.py).
 *
 * Conventions: row-major doubles; slots are in reference adapter order (std::map by
 * job_id, fused_lora.hpp:48-53); A[s] is d x r_s, B[s] is r_s x k.
 * round_bf16 != 0 emulates the device numerics: operands are taken as given (callers
 * pass bf16-representable values) and the low-rank intermediates H = X_j·A_j and
 * dH = dY_j·B_jᵀ are rounded to bf16 (round-to-nearest-even) before use, as the
 * kernels stash them in bf16.
 */
#ifndef TLORA_ORACLE_H_
#define TLORA_ORACLE_H_
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* fused_lora.hpp:84-119 — Y = X·W, then for each slot with >= 1 token (in slot order):
 * gather rows, mid = X_j·A_j, delta = mid·B_j, scatter-add. Returns 0, or -1 when a
 * token names a slot outside [0, S) ("has no adapter", :72-73). */
int orc_fused_forward(int64_t T, int64_t d, int64_t k, int32_t S, const int32_t* ranks,
                      const double* const* A, const double* const* B, const double* X,
                      const double* W, const int32_t* token_slot, int32_t round_bf16,
                      double* Y, double* H /* optional T x sum(r) packed, may be NULL */);

/* fused_lora.hpp:124-135 — Y[t] = X[t]·(W + A_j·B_j), materialising W_j. */
int orc_materialized(int64_t T, int64_t d, int64_t k, int32_t S, const int32_t* ranks,
                     const double* const* A, const double* const* B, const double* X,
                     const double* W, const int32_t* token_slot, double* Y);

/* Backward of the forward above for L = <dY, Y> (new; the reference has none):
 *   dH_j = dY_j·B_jᵀ,  dX = dY·Wᵀ + scatter_j(dH_j·A_jᵀ),
 *   dB_j = H_jᵀ·dY_j,  dA_j = X_jᵀ·dH_j   (H_j = X_j·A_j).
 * dX may be NULL; dA[s] (d x r_s) and dB[s] (r_s x k) are overwritten. */
int orc_fused_backward(int64_t T, int64_t d, int64_t k, int32_t S, const int32_t* ranks,
                       const double* const* A, const double* const* B, const double* X,
                       const double* W, const int32_t* token_slot, const double* dY,
                       int32_t round_bf16, double* dX, double* const* dA, double* const* dB);

/* fused_lora.hpp:95-116 (fused != 0) and :139-163 (unfused): OpCost, bit-identical. */
void orc_op_cost(int64_t T, int64_t d, int64_t k, int32_t S, const int64_t* tokens_per_slot,
                 const int32_t* ranks, int32_t fused, double* flops, double* bytes,
                 long long* launches);

/* nano_pipeline.hpp:51-60. Returns 0, or -1 for group_batch < 1 / n < 1. */
int orc_partition(int32_t group_batch, int32_t n, int32_t* n_out, int32_t* per_nano);

/* nano_pipeline.hpp:99-112 (+ validate :43-46). Returns 0 or -1 (invalid_argument). */
int orc_aimd_step(int32_t* n, int32_t* has_prev, double* t_prev, int32_t alpha, double beta,
                  double tau_rel, double t_t);

/* Plan oracle: brute-force restatement of the rank-aware tile tables of one plan, in the
 * documented enumeration order. `which` is a tlora_launch id. Writes up
 * to cap tiles of 8 int32 each into out; returns the table length (or -1 on bad input). */
int64_t orc_plan_tiles(int64_t T, int64_t d, int64_t k, int32_t S, const int32_t* ranks,
                       const int32_t* token_slot, int32_t which, int32_t* out, int64_t cap);

/* Schedule oracle: static LPT assignment of one dB+dA gradient launch's tiles (the dB table
 * then the dA table, 8 int32 per tile as orc_plan_tiles returns them) to `ctas` CTAs.
 * Tile cost = (ke0 - kb0) * 2 * (128 + ceil64(pad)) + 4 * 128 * pad; tiles taken by cost
 * descending (ties: lower index first), each to the least-loaded CTA (ties: lower CTA).
 * Writes off[ctas + 1] and idx[n_db + n_da] (CSR, CTA c runs idx[off[c] .. off[c+1])).
 * Restates the plan's documented schedule; returns 0 or -1. */
int orc_grad_schedule(const int32_t* tiles_db, int64_t n_db, const int32_t* tiles_da,
                      int64_t n_da, int32_t ctas, int32_t* off, int32_t* idx);

/* Rank-aware nano-batch map (restates tlora_nano_assign, include/tlora.h; the reference
 * only gives counts: nano_pipeline.hpp:51-60). Samples are enumerated job-major (slot 0's
 * batch[0] samples, then slot 1's, ...). counts = partition(sum batch, n). Samples are
 * taken by weight[slot] descending (ties: lower slot, then lower sample index) and each
 * goes to the nano with the least accumulated weight among those with room left (ties:
 * lower nano), then single-sample swaps between the heaviest nano and the others while
 * they lower its load (first improving (o, a, b) in ascending order); this fixes nano_slot[n_out * S] (samples of slot s in nano i). Which
 * samples: job s's samples go to the nano-batches in nano order (its first nano_slot[0][s]
 * samples to nano 0, and so on), so every (nano, job) pair is one contiguous sample range.
 * Writes *n_out, per_nano[n] (= partition's counts), sample_nano[sum batch] and nano_slot.
 * Returns 0 or -1. */
int orc_nano_assign(int32_t S, const int32_t* batch, const int64_t* weight, int32_t n,
                    int32_t* n_out, int32_t* per_nano, int32_t* sample_nano, int32_t* nano_slot);

/* fp32 training step of one fused layer (CPU baseline of bench.py, BASELINE.md §4 item 2:
 * the repo's oracle, fp32 fwd+bwd, OpenMP over all host cores). Job-contiguous batch:
 * slot s owns token rows [off[s], off[s+1]). Y = X·W + H·B, H_s = X_s·A_s; dH_s = dY_s·B_sᵀ,
 * dX = dY·Wᵀ + dH·Aᵀ, dA_s = X_sᵀ·dH_s, dB_s = H_sᵀ·dY_s. Row-major fp32, cache-blocked. */
void orc_train_step_f32(int64_t T, int64_t d, int64_t k, int32_t S, const int32_t* ranks,
                        const int64_t* off, const float* X, const float* W,
                        const float* const* A, const float* const* B, const float* dY, float* Y,
                        float* dX, float* const* dA, float* const* dB);

/* bf16 round-to-nearest-even of a double (via fp32), returned as a double. */
double orc_round_bf16(double x);

#ifdef __cplusplus
}
#endif
#endif
