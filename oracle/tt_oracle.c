/*
 * tt_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, fp64 restatement of the reference ttgnn hot path
 * (/root/reference/proj/core/src/{tt_config,tt_embedding,autodiff}.cpp),
 * used as the parity checker for the CUDA engine and as the CPU baseline
 * ("port") in bench.py.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2206_10581_b200) never links or calls it.
 *
 * Every function cites the reference lines it follows.  Eigen's GEMM
 * summation order is unspecified (Eigen >= 3.3, core/CMakeLists.txt:1, no
 * lockfile), so the chains are restated as fixed-order loops; reductions
 * run over the contraction index in ascending order.
 *
 * Pinning: tests/test_oracle_kats.py checks this library against every
 * hot-path known-answer / property test the reference holds
 * and against the reference's own tt_config.cpp compiled into oracle/_ref.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_MAXD 16

typedef struct {
  int64_t num_nodes;        /* M  */
  int64_t emb_dim;          /* N  */
  int32_t d;                /* number of cores */
  int32_t pad_;
  int64_t m[OR_MAXD];       /* row factors m_1..m_d */
  int64_t n[OR_MAXD];       /* col factors n_1..n_d */
  int64_t R[OR_MAXD + 1];   /* ranks R_0..R_d */
} or_cfg;

/* ---- tt_config.cpp:78-113 ---------------------------------------------- */
int64_t or_padded_rows(const or_cfg* c) {
  int64_t p = 1;
  for (int k = 0; k < c->d; ++k) p *= c->m[k];
  return p;
}
int64_t or_padded_cols(const or_cfg* c) {
  int64_t p = 1;
  for (int k = 0; k < c->d; ++k) p *= c->n[k];
  return p;
}
int64_t or_core_size(const or_cfg* c, int k) { /* tt_config.cpp:87-90 */
  return c->R[k] * c->m[k] * c->n[k] * c->R[k + 1];
}

/* TTConfig::validate (tt_config.cpp:92-113).  Returns 0 if valid, else the
 * 1-based number of the first violated invariant in source order. */
int or_validate(const or_cfg* c) {
  if (c->num_nodes <= 0) return 1;
  if (c->emb_dim <= 0) return 2;
  if (c->d < 2) return 3;
  if (c->d > OR_MAXD) return 4;
  if (c->R[0] != 1 || c->R[c->d] != 1) return 6;
  for (int k = 0; k <= c->d; ++k)
    if (c->R[k] <= 0) return 7;
  for (int k = 0; k < c->d; ++k)
    if (c->m[k] <= 0 || c->n[k] <= 0) return 8;
  if (or_padded_rows(c) < c->num_nodes) return 9;
  if (or_padded_cols(c) < c->emb_dim) return 10;
  return 0;
}

/* count_params (tt_config.cpp:204-208). */
int64_t or_count_params(const or_cfg* c) {
  int64_t t = 0;
  for (int k = 0; k < c->d; ++k) t += or_core_size(c, k);
  return t;
}

/* index_to_coordinate (tt_config.cpp:176-189): mixed radix, i_1 most
 * significant.  Returns 0, or -1 for row outside [0, prod(m)). */
int or_index_to_coordinate(const or_cfg* c, int64_t row, int64_t* parts) {
  if (row < 0 || row >= or_padded_rows(c)) return -1;
  int64_t rem = row;
  for (int k = c->d - 1; k >= 0; --k) {
    parts[k] = rem % c->m[k];
    rem /= c->m[k];
  }
  return 0;
}

/* coordinate_to_index (tt_config.cpp:191-202). */
int64_t or_coordinate_to_index(const or_cfg* c, const int64_t* parts) {
  int64_t row = 0;
  for (int k = 0; k < c->d; ++k) {
    if (parts[k] < 0 || parts[k] >= c->m[k]) return -1;
    row = row * c->m[k] + parts[k];
  }
  return row;
}

enum { OR_SGD = 0, OR_ADAM = 1, OR_ADAGRAD = 2 };

/* fp64: the reference's arithmetic (parity checker, reference arm) */
#define REAL double
#define SQRT sqrt
#define FN(x) x
#include "tt_oracle_path.inc"
#undef REAL
#undef SQRT
#undef FN
/* fp32: the multithreaded fp32 CPU baseline (bench.py cpu_baseline) */
#define REAL float
#define SQRT sqrtf
#define FN(x) x##_f32
#include "tt_oracle_path.inc"
#undef REAL
#undef SQRT
#undef FN

/* ---- scalar elementwise oracle: tests/test_oracles.hpp:48-75 -------------- */
double or_ttm_entry(const or_cfg* c, const double* const* cores, int64_t row, int64_t col) {
  const int d = c->d;
  int64_t i[OR_MAXD], j[OR_MAXD];
  int64_t ri = row, rj = col;
  for (int k = d - 1; k >= 0; --k) {
    i[k] = ri % c->m[k]; ri /= c->m[k];
    j[k] = rj % c->n[k]; rj /= c->n[k];
  }
  double cur[1024], nxt[1024];
#define ENTRY(k, r, s) cores[k][(((r) * c->m[k] + i[k]) * c->n[k] + j[k]) * c->R[(k) + 1] + (s)]
  for (int64_t s = 0; s < c->R[1]; ++s) cur[s] = ENTRY(0, 0, s);
  for (int k = 1; k < d; ++k) {
    for (int64_t s = 0; s < c->R[k + 1]; ++s) {
      nxt[s] = 0.0;
      for (int64_t r = 0; r < c->R[k]; ++r) nxt[s] += cur[r] * ENTRY(k, r, s);
    }
    for (int64_t s = 0; s < c->R[k + 1]; ++s) cur[s] = nxt[s];
  }
#undef ENTRY
  return cur[0];
}

/* ---- sort / unique / prefix counts (new; SPEC.md:71,220 permit dedupe) ---- */
/* Stable sort of (key, position) by key (ties keep position order), via a
 * bottom-up merge sort -- the semantics of std::stable_sort.  perm[s] is the
 * batch position of the s-th sorted entry; uniq receives the distinct keys
 * in ascending order; returns their count. */
int64_t or_sort_unique(const int64_t* keys, int64_t B, int64_t* perm, int64_t* uniq) {
  int64_t* tmp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(B > 0 ? B : 1));
  for (int64_t b = 0; b < B; ++b) perm[b] = b;
  for (int64_t w = 1; w < B; w *= 2) {
    for (int64_t lo = 0; lo < B; lo += 2 * w) {
      int64_t mid = lo + w < B ? lo + w : B, hi = lo + 2 * w < B ? lo + 2 * w : B;
      int64_t a = lo, b = mid, o = lo;
      while (a < mid && b < hi) tmp[o++] = keys[perm[b]] < keys[perm[a]] ? perm[b++] : perm[a++];
      while (a < mid) tmp[o++] = perm[a++];
      while (b < hi) tmp[o++] = perm[b++];
    }
    memcpy(perm, tmp, sizeof(int64_t) * (size_t)B);
  }
  free(tmp);
  int64_t U = 0;
  for (int64_t s = 0; s < B; ++s)
    if (s == 0 || keys[perm[s]] != keys[perm[s - 1]]) uniq[U++] = keys[perm[s]];
  return U;
}

/* U_l for l = 1..d: the number of distinct prefixes (i_1..i_l) among the
 * batch's IDs (counts[d-1] = distinct IDs).  Requires valid indices. */
void or_prefix_counts(const or_cfg* c, const int64_t* idx, int64_t B, int64_t* counts) {
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)(B > 0 ? B : 1));
  int64_t* uniq = (int64_t*)malloc(sizeof(int64_t) * (size_t)(B > 0 ? B : 1));
  int64_t U = or_sort_unique(idx, B, perm, uniq);
  int64_t suffix = 1;
  for (int l = c->d; l >= 1; --l) {
    int64_t cnt = 0;
    for (int64_t u = 0; u < U; ++u)
      if (u == 0 || uniq[u] / suffix != uniq[u - 1] / suffix) ++cnt;
    counts[l - 1] = cnt;
    suffix *= c->m[l - 1];
  }
  free(perm); free(uniq);
}

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
