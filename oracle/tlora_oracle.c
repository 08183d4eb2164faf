/*
 * tlora_oracle.c — CPU oracle for the fused multi-LoRA layer. TEST INFRASTRUCTURE ONLY.
 * See tlora_oracle.h for the contract and the parity pinning. Each function cites the
 * reference lines it restates (paths relative to /root/reference/proj/include/lora_fleet).
 */
#include "tlora_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

double orc_round_bf16(double x) {
  float f = (float)x;
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return (double)f; /* inf / nan */
  const uint32_t lsb = (u >> 16) & 1u;
  u += 0x7fffu + lsb;
  u &= 0xffff0000u;
  memcpy(&f, &u, 4);
  return (double)f;
}

/* rows of slot s, ascending (fused_lora.hpp:56-61) */
static int64_t segment_rows(int64_t T, const int32_t* slot, int32_t s, int64_t* rows) {
  int64_t n = 0;
  for (int64_t t = 0; t < T; ++t)
    if (slot[t] == s) rows[n++] = t;
  return n;
}

static int check_slots(int64_t T, int32_t S, const int32_t* slot) {
  for (int64_t t = 0; t < T; ++t)
    if (slot[t] < 0 || slot[t] >= S) return -1; /* fused_lora.hpp:72-73 */
  return 0;
}

/* C[m x n] = A[m x p] · B[p x n], row-major, OpenMP over rows */
static void gemm_nn(int64_t m, int64_t p, int64_t n, const double* A, const double* B, double* C) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    double* c = C + i * n;
    for (int64_t j = 0; j < n; ++j) c[j] = 0.0;
    for (int64_t q = 0; q < p; ++q) {
      const double a = A[i * p + q];
      const double* b = B + q * n;
      for (int64_t j = 0; j < n; ++j) c[j] += a * b[j];
    }
  }
}

/* C[m x n] = A[m x p] · B[n x p]ᵀ */
static void gemm_nt(int64_t m, int64_t p, int64_t n, const double* A, const double* B, double* C) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double acc = 0.0;
      const double* a = A + i * p;
      const double* b = B + j * p;
      for (int64_t q = 0; q < p; ++q) acc += a[q] * b[q];
      C[i * n + j] = acc;
    }
}

/* C[p x n] = A[m x p]ᵀ · B[m x n] */
static void gemm_tn(int64_t m, int64_t p, int64_t n, const double* A, const double* B, double* C) {
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < p; ++q) {
    double* c = C + q * n;
    for (int64_t j = 0; j < n; ++j) c[j] = 0.0;
    for (int64_t i = 0; i < m; ++i) {
      const double a = A[i * p + q];
      const double* b = B + i * n;
      for (int64_t j = 0; j < n; ++j) c[j] += a * b[j];
    }
  }
}

int orc_fused_forward(int64_t T, int64_t d, int64_t k, int32_t S, const int32_t* ranks,
                      const double* const* A, const double* const* B, const double* X,
                      const double* W, const int32_t* slot, int32_t round_bf16, double* Y,
                      double* H) {
  if (check_slots(T, S, slot)) return -1;
  int64_t R = 0;
  for (int32_t s = 0; s < S; ++s) R += ranks[s];
  gemm_nn(T, d, k, X, W, Y); /* :93 shared base term, computed once */
  if (H) memset(H, 0, sizeof(double) * (size_t)(T * R));
  int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)(T > 0 ? T : 1));
  int64_t hoff = 0;
  for (int32_t s = 0; s < S; ++s) { /* :102 map order */
    const int64_t n = segment_rows(T, slot, s, rows);
    const int64_t r = ranks[s];
    if (n > 0) { /* :104 empty segments skipped */
      double* g = (double*)malloc(sizeof(double) * (size_t)(n * d));
      double* mid = (double*)malloc(sizeof(double) * (size_t)(n * r));
      double* delta = (double*)malloc(sizeof(double) * (size_t)(n * k));
      for (int64_t i = 0; i < n; ++i) memcpy(g + i * d, X + rows[i] * d, sizeof(double) * d); /* :108-109 */
      gemm_nn(n, d, r, g, A[s], mid); /* :111 */
      if (round_bf16)
        for (int64_t i = 0; i < n * r; ++i) mid[i] = orc_round_bf16(mid[i]);
      gemm_nn(n, r, k, mid, B[s], delta); /* :112 */
      for (int64_t i = 0; i < n; ++i) /* :113 scatter-add */
        for (int64_t j = 0; j < k; ++j) Y[rows[i] * k + j] += delta[i * k + j];
      if (H)
        for (int64_t i = 0; i < n; ++i)
          memcpy(H + rows[i] * R + hoff, mid + i * r, sizeof(double) * r);
      free(g);
      free(mid);
      free(delta);
    }
    hoff += r;
  }
  free(rows);
  return 0;
}

int orc_materialized(int64_t T, int64_t d, int64_t k, int32_t S, const int32_t* ranks,
                     const double* const* A, const double* const* B, const double* X,
                     const double* W, const int32_t* slot, double* Y) {
  if (check_slots(T, S, slot)) return -1;
  double* Wi = (double*)malloc(sizeof(double) * (size_t)(d * k));
  for (int32_t s = 0; s < S; ++s) { /* :130-133 */
    gemm_nn(d, ranks[s], k, A[s], B[s], Wi);
    for (int64_t i = 0; i < d * k; ++i) Wi[i] += W[i];
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < T; ++t) {
      if (slot[t] != s) continue;
      for (int64_t j = 0; j < k; ++j) {
        double acc = 0.0;
        for (int64_t q = 0; q < d; ++q) acc += X[t * d + q] * Wi[q * k + j];
        Y[t * k + j] = acc;
      }
    }
  }
  free(Wi);
  return 0;
}

int orc_fused_backward(int64_t T, int64_t d, int64_t k, int32_t S, const int32_t* ranks,
                       const double* const* A, const double* const* B, const double* X,
                       const double* W, const int32_t* slot, const double* dY,
                       int32_t round_bf16, double* dX, double* const* dA, double* const* dB) {
  if (check_slots(T, S, slot)) return -1;
  if (dX) gemm_nt(T, k, d, dY, W, dX); /* dX = dY·Wᵀ */
  int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)(T > 0 ? T : 1));
  for (int32_t s = 0; s < S; ++s) {
    const int64_t r = ranks[s];
    const int64_t n = segment_rows(T, slot, s, rows);
    if (n == 0) {
      memset(dA[s], 0, sizeof(double) * (size_t)(d * r));
      memset(dB[s], 0, sizeof(double) * (size_t)(r * k));
      continue;
    }
    double* xs = (double*)malloc(sizeof(double) * (size_t)(n * d));
    double* gs = (double*)malloc(sizeof(double) * (size_t)(n * k));
    double* h = (double*)malloc(sizeof(double) * (size_t)(n * r));
    double* dh = (double*)malloc(sizeof(double) * (size_t)(n * r));
    for (int64_t i = 0; i < n; ++i) {
      memcpy(xs + i * d, X + rows[i] * d, sizeof(double) * d);
      memcpy(gs + i * k, dY + rows[i] * k, sizeof(double) * k);
    }
    gemm_nn(n, d, r, xs, A[s], h);    /* H_j = X_j·A_j (forward intermediate) */
    gemm_nt(n, k, r, gs, B[s], dh);   /* dH_j = dY_j·B_jᵀ */
    if (round_bf16)
      for (int64_t i = 0; i < n * r; ++i) {
        h[i] = orc_round_bf16(h[i]);
        dh[i] = orc_round_bf16(dh[i]);
      }
    gemm_tn(n, r, k, h, gs, dB[s]);   /* dB_j = H_jᵀ·dY_j */
    gemm_tn(n, d, r, xs, dh, dA[s]);  /* dA_j = X_jᵀ·dH_j */
    if (dX) {                         /* dX_j += dH_j·A_jᵀ */
      double* t = (double*)malloc(sizeof(double) * (size_t)(n * d));
      gemm_nt(n, r, d, dh, A[s], t);
      for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < d; ++j) dX[rows[i] * d + j] += t[i * d + j];
      free(t);
    }
    free(xs);
    free(gs);
    free(h);
    free(dh);
  }
  free(rows);
  return 0;
}

void orc_op_cost(int64_t T, int64_t d, int64_t k, int32_t S, const int64_t* tokens_per_slot,
                 const int32_t* ranks, int32_t fused, double* flops, double* bytes,
                 long long* launches) {
  const double tt = (double)T, dd = (double)d, kk = (double)k;
  double f = 2.0 * tt * dd * kk;                     /* :96 / :149 */
  double b = 8.0 * (tt * dd + dd * kk + tt * kk);    /* :97-99 / :150 */
  long long l = 1;                                   /* :100 / :151 */
  for (int32_t s = 0; s < S; ++s) {
    if (tokens_per_slot[s] == 0) continue;           /* :104 / :154 */
    const double n = (double)tokens_per_slot[s], r = (double)ranks[s];
    f += 2.0 * n * dd * r + 2.0 * n * r * kk;        /* :115 / :157 */
    if (fused) {
      b += 8.0 * (dd * r + r * kk + 2.0 * n * r);    /* :116 */
    } else {
      b += 8.0 * (2.0 * n * dd + dd * r + r * kk + 4.0 * n * r + 2.0 * n * kk); /* :159 */
      l += 4;                                        /* :160 */
    }
  }
  *flops = f;
  *bytes = b;
  *launches = l;
}

int orc_partition(int32_t group_batch, int32_t n, int32_t* n_out, int32_t* per_nano) {
  if (group_batch < 1 || n < 1) return -1; /* :52-53 */
  const int32_t nn = n < group_batch ? n : group_batch;
  *n_out = nn;
  for (int32_t i = 0; i < nn; ++i) per_nano[i] = group_batch / nn + (i < group_batch % nn ? 1 : 0);
  return 0;
}

int orc_aimd_step(int32_t* n, int32_t* has_prev, double* t_prev, int32_t alpha, double beta,
                  double tau_rel, double t_t) {
  if (*n < 1 || alpha < 1 || beta <= 0.0 || beta >= 1.0 || tau_rel < 0.0) return -1; /* :43-46 */
  if (t_t < 0.0) return -1;                                                            /* :101 */
  if (*has_prev) {
    if (t_t <= *t_prev - tau_rel * *t_prev)
      *n = *n + alpha;
    else {
      const int32_t m = (int32_t)floor(beta * *n);
      *n = m > 1 ? m : 1;
    }
  }
  *has_prev = 1;
  *t_prev = t_t;
  return 0;
}

/* ---------------------------------------------------------------- plan oracle */
enum { BM = 128, BM2 = 256, BK = 64, BN_BASE = 256, BN_LOW = 128, GRAD_MAX_N = 128,
       GRAD_TARGET = 74 };
#define L2_BUDGET (48ll << 20)

static int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

typedef struct {
  int32_t* out;
  int64_t cap, n;
} TileSink;

static void emit(TileSink* s, int32_t m0, int32_t n0, int32_t kb0, int32_t ke0, int32_t kb1,
                 int32_t ke1, int32_t split) {
  if (s->n < s->cap) {
    int32_t* t = s->out + 8 * s->n;
    t[0] = m0; t[1] = n0; t[2] = kb0; t[3] = ke0; t[4] = kb1; t[5] = ke1; t[6] = split; t[7] = 0;
  }
  s->n++;
}

int64_t orc_plan_tiles(int64_t T, int64_t d, int64_t k, int32_t S, const int32_t* ranks,
                       const int32_t* slot, int32_t which, int32_t* out, int64_t cap) {
  if (T < 1 || S < 1 || which < 0 || which > 7 || check_slots(T, S, slot)) return -1;
  int32_t* off = (int32_t*)malloc(sizeof(int32_t) * S);
  int32_t R = 0;
  for (int32_t s = 0; s < S; ++s) {
    off[s] = R;
    R += (ranks[s] + 7) / 8 * 8;
  }
  if (R < 8) R = 8;
  TileSink sink = {out, cap, 0};
  const int64_t n_mt = cdiv(T, BM);
  if (which <= 3 || which >= 6) {
    int32_t* win_lo = (int32_t*)malloc(sizeof(int32_t) * (size_t)n_mt);
    int32_t* win_hi = (int32_t*)malloc(sizeof(int32_t) * (size_t)n_mt);
    for (int64_t m = 0; m < n_mt; ++m) {
      /* brute force: smallest / largest packed column owned by any token of the tile */
      int64_t lo = -1, hi = -1;
      for (int64_t c = 0; c < R; ++c) {
        int owned = 0;
        for (int64_t t = m * BM; t < T && t < (m + 1) * BM && !owned; ++t)
          owned = c >= off[slot[t]] && c < off[slot[t]] + ranks[slot[t]];
        if (owned) {
          if (lo < 0) lo = c;
          hi = c + 1;
        }
      }
      const int32_t c_lo = (int32_t)(lo / BK * BK), c_hi = (int32_t)(cdiv(hi, BK) * BK);
      win_lo[m] = c_lo;
      win_hi[m] = c_hi;
      if (which == 0 || which == 2)
        for (int32_t n0 = c_lo; n0 < c_hi; n0 += BN_LOW)
          emit(&sink, (int32_t)(m * BM), n0, 0, (int32_t)(which == 0 ? d : k), 0, 0, 0);
    }
    if (which >= 6) {
      /* shrink / dH on 256-token pair tiles: window = union of the halves, N-chunks of <= 256
       * each rounded up to a multiple of 128 columns */
      const int64_t n_m2 = cdiv(T, BM2), K = which == 6 ? d : k;
      for (int64_t m = 0; m < n_m2; ++m) {
        int32_t lo = win_lo[2 * m], hi = win_hi[2 * m];
        if (2 * m + 1 < n_mt) {
          if (win_lo[2 * m + 1] < lo) lo = win_lo[2 * m + 1];
          if (win_hi[2 * m + 1] > hi) hi = win_hi[2 * m + 1];
        }
        for (int32_t n0 = lo; n0 < hi; n0 += 256) {
          int32_t n = (int32_t)(cdiv(hi - n0, 128) * 128);
          if (n > 256) n = 256;
          emit(&sink, (int32_t)(m * BM2), n0, 0, (int32_t)K, 0, 0, 0);
          if (sink.n <= sink.cap) sink.out[8 * (sink.n - 1) + 7] = n;
        }
      }
    }
    if (which == 1 || which == 3) {
      /* fused base GEMMs: 256-token tiles (CTA pairs); window = union of the two halves.
       * L2 panel raster: keep a <= L2_BUDGET operand panel hot, stream the other one;
       * choose the orientation streaming fewer bytes (ties: M panels). */
      const int64_t N = which == 1 ? k : d, K = which == 1 ? d : k;
      const int64_t n_m2 = cdiv(T, BM2), n_nt = cdiv(N, BN_BASE);
      const int64_t a_panel = (int64_t)BM2 * K * 2, b_panel = (int64_t)BN_BASE * K * 2;
      int64_t gm = L2_BUDGET / a_panel, gn = L2_BUDGET / b_panel;
      gm = gm < 1 ? 1 : (gm > n_m2 ? n_m2 : gm);
      gn = gn < 1 ? 1 : (gn > n_nt ? n_nt : gn);
      const int64_t bytes_m = n_m2 * a_panel + cdiv(n_m2, gm) * n_nt * b_panel;
      const int64_t bytes_n = n_nt * b_panel + cdiv(n_nt, gn) * n_m2 * a_panel;
#define WLO(m) (2 * (m) + 1 < n_mt && win_lo[2 * (m) + 1] < win_lo[2 * (m)] ? win_lo[2 * (m) + 1] : win_lo[2 * (m)])
#define WHI(m) (2 * (m) + 1 < n_mt && win_hi[2 * (m) + 1] > win_hi[2 * (m)] ? win_hi[2 * (m) + 1] : win_hi[2 * (m)])
      for (int64_t g0 = 0; bytes_m <= bytes_n && g0 < n_m2; g0 += gm)
        for (int64_t n = 0; n < n_nt; ++n)
          for (int64_t m = g0; m < n_m2 && m < g0 + gm; ++m)
            emit(&sink, (int32_t)(m * BM2), (int32_t)(n * BN_BASE), 0, (int32_t)K, WLO(m), WHI(m), 0);
      for (int64_t g0 = 0; bytes_m > bytes_n && g0 < n_nt; g0 += gn)
        for (int64_t m = 0; m < n_m2; ++m)
          for (int64_t n = g0; n < n_nt && n < g0 + gn; ++n)
            emit(&sink, (int32_t)(m * BM2), (int32_t)(n * BN_BASE), 0, (int32_t)K, WLO(m), WHI(m), 0);
#undef WLO
#undef WHI
    }
    free(win_lo);
    free(win_hi);
  } else {
    /* per-job transposed gradient tiles (dB: M-dim = k, dA: M-dim = d), brute force:
     * token range of a job = [first token, last token] found by scanning. */
    const int64_t Md = which == 4 ? k : d;
    const int64_t n_mt = cdiv(Md, BM);
    int64_t total = 0;
    int64_t* first = (int64_t*)malloc(sizeof(int64_t) * S);
    int64_t* last = (int64_t*)malloc(sizeof(int64_t) * S);
    for (int32_t s = 0; s < S; ++s) {
      first[s] = -1;
      last[s] = -1;
      for (int64_t t = 0; t < T; ++t)
        if (slot[t] == s) {
          if (first[s] < 0) first[s] = t;
          last[s] = t;
        }
      if (first[s] < 0) continue;
      for (int64_t q = 0; q < ranks[s]; q += GRAD_MAX_N) {
        const int64_t nc = ranks[s] - q < GRAD_MAX_N ? ranks[s] - q : GRAD_MAX_N;
        total += (last[s] + 1 - first[s]) * (BM + cdiv(nc, 64) * 64) * n_mt;
      }
    }
    int64_t w_star = total / GRAD_TARGET;
    if (w_star < 1) w_star = 1;
    /* collect (work, order, tile) then sort by work desc, order asc (== stable sort) */
    int64_t cap_t = 16, nt = 0;
    int64_t* keyw = (int64_t*)malloc(sizeof(int64_t) * cap_t);
    int32_t* tl = (int32_t*)malloc(sizeof(int32_t) * 8 * cap_t);
#define PUSH(W_, m0_, n0_, kb_, ke_, sp_, nc_)                                   \
  do {                                                                           \
    if (nt == cap_t) {                                                           \
      cap_t *= 2;                                                                \
      keyw = (int64_t*)realloc(keyw, sizeof(int64_t) * cap_t);                   \
      tl = (int32_t*)realloc(tl, sizeof(int32_t) * 8 * cap_t);                   \
    }                                                                            \
    keyw[nt] = (W_);                                                             \
    int32_t* t_ = tl + 8 * nt;                                                   \
    t_[0] = (m0_); t_[1] = (n0_); t_[2] = (kb_); t_[3] = (ke_);                  \
    t_[4] = 0; t_[5] = 0; t_[6] = (sp_); t_[7] = (nc_);                          \
    ++nt;                                                                        \
  } while (0)
    for (int32_t s = 0; s < S; ++s) {
      for (int64_t q = 0; q < ranks[s]; q += GRAD_MAX_N) {
        const int32_t c0 = off[s] + (int32_t)q;
        const int32_t nc = (int32_t)(ranks[s] - q < GRAD_MAX_N ? ranks[s] - q : GRAD_MAX_N);
        if (first[s] < 0) {
          for (int64_t mt = 0; mt < n_mt; ++mt) PUSH(0, (int32_t)(mt * BM), c0, 0, 0, 0, nc);
          continue;
        }
        const int64_t tlo = first[s], thi = last[s] + 1, len = thi - tlo;
        const int64_t per_tile = len * (BM + cdiv(nc, 64) * 64);
        int64_t c = cdiv(per_tile, w_star);
        const int64_t cmax = len / 256 < 1 ? 1 : len / 256;
        if (c > cmax) c = cmax;
        if (c < 1) c = 1;
        const int64_t chunk = cdiv(cdiv(len, c), BK) * BK;
        for (int64_t sp = 0; sp < c; ++sp) {
          const int64_t kb = tlo + sp * chunk;
          const int64_t ke = thi < kb + chunk ? thi : kb + chunk;
          if (kb >= ke) break;
          for (int64_t mt = 0; mt < n_mt; ++mt)
            PUSH((ke - kb) * (BM + cdiv(nc, 64) * 64), (int32_t)(mt * BM), c0, (int32_t)kb,
                 (int32_t)ke, (int32_t)sp, nc);
        }
      }
    }
#undef PUSH
    /* insertion-free stable order: repeatedly emit in (work desc, index asc) order */
    int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (nt > 0 ? nt : 1));
    for (int64_t i = 0; i < nt; ++i) idx[i] = i;
    /* merge sort by (keyw desc, idx asc) */
    int64_t* tmp = (int64_t*)malloc(sizeof(int64_t) * (nt > 0 ? nt : 1));
    for (int64_t width = 1; width < nt; width *= 2) {
      for (int64_t lo = 0; lo < nt; lo += 2 * width) {
        int64_t mid = lo + width < nt ? lo + width : nt, hi = lo + 2 * width < nt ? lo + 2 * width : nt;
        int64_t i = lo, j = mid, o = lo;
        while (i < mid && j < hi) tmp[o++] = keyw[idx[j]] > keyw[idx[i]] ? idx[j++] : idx[i++];
        while (i < mid) tmp[o++] = idx[i++];
        while (j < hi) tmp[o++] = idx[j++];
      }
      memcpy(idx, tmp, sizeof(int64_t) * nt);
    }
    for (int64_t i = 0; i < nt; ++i) {
      const int32_t* t_ = tl + 8 * idx[i];
      if (sink.n < sink.cap) memcpy(sink.out + 8 * sink.n, t_, 8 * sizeof(int32_t));
      sink.n++;
    }
    free(idx);
    free(tmp);
    free(keyw);
    free(tl);
    free(first);
    free(last);
  }
  free(off);
  return sink.n;
}

/* ---- gradient-launch schedule (LPT), restated from the documented rule ------------------ */
typedef struct {
  int64_t cost;
  int32_t i;
} orc_costed;

static int orc_costed_cmp(const void* a, const void* b) {
  const orc_costed* x = (const orc_costed*)a;
  const orc_costed* y = (const orc_costed*)b;
  if (x->cost != y->cost) return x->cost > y->cost ? -1 : 1; /* cost descending */
  return x->i < y->i ? -1 : (x->i > y->i); /* then index ascending (a stable sort) */
}

int orc_grad_schedule(const int32_t* tiles_db, int64_t n_db, const int32_t* tiles_da,
                      int64_t n_da, int32_t ctas, int32_t* off, int32_t* idx) {
  if (ctas < 1 || n_db < 0 || n_da < 0) return -1;
  const int64_t n = n_db + n_da;
  orc_costed* order = (orc_costed*)malloc(sizeof(orc_costed) * (n > 0 ? n : 1));
  int64_t* load = (int64_t*)calloc(ctas, sizeof(int64_t));
  int32_t* owner = (int32_t*)malloc(sizeof(int32_t) * (n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) {
    const int32_t* t = i < n_db ? tiles_db + 8 * i : tiles_da + 8 * (i - n_db);
    const int64_t pad = t[7], pad64 = (pad + 63) / 64 * 64;
    order[i].cost = (int64_t)(t[3] - t[2]) * 2 * (128 + pad64) + 4 * 128 * pad;
    order[i].i = (int32_t)i;
  }
  qsort(order, (size_t)n, sizeof(orc_costed), orc_costed_cmp);
  for (int64_t q = 0; q < n; ++q) { /* least-loaded CTA, lowest index on ties */
    int32_t best = 0;
    for (int32_t c = 1; c < ctas; ++c)
      if (load[c] < load[best]) best = c;
    owner[q] = best;
    load[best] += order[q].cost;
  }
  off[0] = 0;
  int32_t w = 0;
  for (int32_t c = 0; c < ctas; ++c) { /* per CTA, in assignment order */
    for (int64_t q = 0; q < n; ++q)
      if (owner[q] == c) idx[w++] = order[q].i;
    off[c + 1] = w;
  }
  free(order);
  free(load);
  free(owner);
  return 0;
}


/* ---------------------------------------------------------------- nano-batch map */
int orc_nano_assign(int32_t S, const int32_t* batch, const int64_t* weight, int32_t n,
                    int32_t* n_out, int32_t* per_nano, int32_t* sample_nano, int32_t* nano_slot) {
  if (S < 1) return -1;
  int64_t total = 0;
  for (int32_t s = 0; s < S; ++s) {
    if (batch[s] < 0 || weight[s] < 0) return -1;
    total += batch[s];
  }
  if (total < 1 || total > 2147483647) return -1;
  int32_t nn = 0;
  if (orc_partition((int32_t)total, n, &nn, per_nano) != 0) return -1;
  *n_out = nn;
  int64_t* load = (int64_t*)calloc((size_t)nn, sizeof(int64_t));
  int32_t* room = (int32_t*)malloc((size_t)nn * sizeof(int32_t));
  char* done = (char*)calloc((size_t)S, 1);
  int64_t* first = (int64_t*)malloc((size_t)S * sizeof(int64_t));
  if (!load || !room || !done || !first) return -1;
  for (int32_t i = 0; i < nn; ++i) room[i] = per_nano[i];
  for (int64_t i = 0; i < (int64_t)nn * S; ++i) nano_slot[i] = 0;
  int64_t acc = 0;
  for (int32_t s = 0; s < S; ++s) {
    first[s] = acc;
    acc += batch[s];
  }
  /* slots by weight descending, ties by slot: brute-force selection (S is small) */
  for (int32_t round = 0; round < S; ++round) {
    int32_t best = -1;
    for (int32_t s = 0; s < S; ++s)
      if (!done[s] && (best < 0 || weight[s] > weight[best])) best = s;
    done[best] = 1;
    for (int32_t q = 0; q < batch[best]; ++q) {
      int32_t pick = -1;
      for (int32_t i = 0; i < nn; ++i)
        if (room[i] > 0 && (pick < 0 || load[i] < load[pick])) pick = i;
      --room[pick];
      load[pick] += weight[best];
      ++nano_slot[(int64_t)pick * S + best];
    }
  }
  /* swap refinement: heaviest nano h (first on ties); first (o, a, b) in ascending order
   * with nano_slot[h][a] > 0, nano_slot[o][b] > 0, weight[a] > weight[b] and
   * load[o] + (weight[a] - weight[b]) < load[h]; swap one sample; repeat until none */
  for (int32_t i = 0; i < nn; ++i) {
    load[i] = 0;
    for (int32_t s = 0; s < S; ++s) load[i] += (int64_t)nano_slot[(int64_t)i * S + s] * weight[s];
  }
  for (;;) {
    int32_t h = 0, found = 0;
    for (int32_t i = 1; i < nn; ++i)
      if (load[i] > load[h]) h = i;
    for (int32_t o = 0; o < nn && !found; ++o) {
      if (o == h) continue;
      for (int32_t a = 0; a < S && !found; ++a) {
        if (!nano_slot[(int64_t)h * S + a]) continue;
        for (int32_t b = 0; b < S && !found; ++b) {
          if (!nano_slot[(int64_t)o * S + b] || weight[a] <= weight[b]) continue;
          const int64_t delta = weight[a] - weight[b];
          if (load[o] + delta >= load[h]) continue;
          nano_slot[(int64_t)h * S + a]--;
          nano_slot[(int64_t)h * S + b]++;
          nano_slot[(int64_t)o * S + b]--;
          nano_slot[(int64_t)o * S + a]++;
          load[h] -= delta;
          load[o] += delta;
          found = 1;
        }
      }
    }
    if (!found) break;
  }
  /* which samples: a job's samples go to the nano-batches in nano order (the first
   * nano_slot[0][s] samples to nano 0, ...), so each (nano, job) is a contiguous range */
  for (int32_t s = 0; s < S; ++s) {
    int64_t q = first[s];
    for (int32_t i = 0; i < nn; ++i)
      for (int32_t c = 0; c < nano_slot[(int64_t)i * S + s]; ++c) sample_nano[q++] = i;
  }
  free(load);
  free(room);
  free(done);
  free(first);
  return 0;
}

/* ---------------------------------------------------------------- fp32 CPU train step */
#define ORC_RB 32 /* token rows per block: one W row is reused RB times from cache */

/* C[rows x n] (+)= A[rows x p] · B[p x n] for a block of rows (all row-major, lda/ldc) */
static void blk_nn_f32(int64_t rows, int64_t p, int64_t n, const float* A, int64_t lda,
                       const float* B, float* C, int64_t ldc, int accumulate) {
  if (!accumulate)
    for (int64_t i = 0; i < rows; ++i)
      for (int64_t j = 0; j < n; ++j) C[i * ldc + j] = 0.f;
  for (int64_t q = 0; q < p; ++q) {
    const float* b = B + q * n;
    for (int64_t i = 0; i < rows; ++i) {
      const float a = A[i * lda + q];
      float* c = C + i * ldc;
#pragma omp simd
      for (int64_t j = 0; j < n; ++j) c[j] += a * b[j];
    }
  }
}

/* C[rows x n] (+)= A[rows x p] · B[n x p]ᵀ */
static void blk_nt_f32(int64_t rows, int64_t p, int64_t n, const float* A, int64_t lda,
                       const float* B, float* C, int64_t ldc, int accumulate) {
  for (int64_t j = 0; j < n; ++j) {
    const float* b = B + j * p;
    for (int64_t i = 0; i < rows; ++i) {
      const float* a = A + i * lda;
      float acc = 0.f;
#pragma omp simd reduction(+ : acc)
      for (int64_t q = 0; q < p; ++q) acc += a[q] * b[q];
      C[i * ldc + j] = accumulate ? C[i * ldc + j] + acc : acc;
    }
  }
}

void orc_train_step_f32(int64_t T, int64_t d, int64_t k, int32_t S, const int32_t* ranks,
                        const int64_t* off, const float* X, const float* W,
                        const float* const* A, const float* const* B, const float* dY, float* Y,
                        float* dX, float* const* dA, float* const* dB) {
  int32_t rmax = 1;
  for (int32_t s = 0; s < S; ++s) rmax = ranks[s] > rmax ? ranks[s] : rmax;
  float* H = (float*)malloc((size_t)T * rmax * sizeof(float));
  float* dH = (float*)malloc((size_t)T * rmax * sizeof(float));
  const int64_t nblk = (T + ORC_RB - 1) / ORC_RB;
  /* forward + dH + dX, token-row blocks in parallel (each block inside one job) */
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t b = 0; b < nblk; ++b) {
    const int64_t t0 = b * ORC_RB, t1 = t0 + ORC_RB < T ? t0 + ORC_RB : T;
    for (int32_t s = 0; s < S; ++s) {
      const int64_t lo = off[s] > t0 ? off[s] : t0, hi = off[s + 1] < t1 ? off[s + 1] : t1;
      if (lo >= hi) continue;
      const int64_t r = ranks[s];
      blk_nn_f32(hi - lo, d, r, X + lo * d, d, A[s], H + lo * rmax, rmax, 0);
      blk_nt_f32(hi - lo, k, r, dY + lo * k, k, B[s], dH + lo * rmax, rmax, 0);
    }
    blk_nn_f32(t1 - t0, d, k, X + t0 * d, d, W, Y + t0 * k, k, 0);
    blk_nt_f32(t1 - t0, k, d, dY + t0 * k, k, W, dX + t0 * d, d, 0);
    for (int32_t s = 0; s < S; ++s) {
      const int64_t lo = off[s] > t0 ? off[s] : t0, hi = off[s + 1] < t1 ? off[s + 1] : t1;
      if (lo >= hi) continue;
      const int64_t r = ranks[s];
      blk_nn_f32(hi - lo, r, k, H + lo * rmax, rmax, B[s], Y + lo * k, k, 1);
      blk_nt_f32(hi - lo, r, d, dH + lo * rmax, rmax, A[s], dX + lo * d, d, 1);
    }
  }
  /* dA_s = X_sᵀ·dH_s (d x r), dB_s = H_sᵀ·dY_s (r x k): parallel over output rows */
  for (int32_t s = 0; s < S; ++s) {
    const int64_t r = ranks[s], lo = off[s], hi = off[s + 1];
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < d; ++i) {
      float* out = dA[s] + i * r;
      for (int64_t j = 0; j < r; ++j) out[j] = 0.f;
      for (int64_t t = lo; t < hi; ++t) {
        const float x = X[t * d + i];
        const float* g = dH + t * rmax;
        for (int64_t j = 0; j < r; ++j) out[j] += x * g[j];
      }
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < r; ++i) {
      float* out = dB[s] + i * k;
      for (int64_t j = 0; j < k; ++j) out[j] = 0.f;
      for (int64_t t = lo; t < hi; ++t) {
        const float h = H[t * rmax + i];
        const float* g = dY + t * k;
#pragma omp simd
        for (int64_t j = 0; j < k; ++j) out[j] += h * g[j];
      }
    }
  }
  free(H);
  free(dH);
}
