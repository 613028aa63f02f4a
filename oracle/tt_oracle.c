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

/* ---- forward: tt_embedding.cpp:31-71 ------------------------------------ */
static int64_t chain_cap(const or_cfg* c) { /* tt_embedding.cpp:48-56 */
  int64_t cap = 0, cols = 1;
  for (int k = 0; k < c->d; ++k) {
    cols *= c->n[k];
    int64_t v = cols * c->R[k + 1];
    if (v > cap) cap = v;
  }
  return cap;
}

/* reconstruct_padded_into: buf = G_1[i_1] (1 x n_1R_1); for k = 2..d the
 * running (N_{k-1} x R_{k-1}) product times the slice unfolding
 * G_k(:, i_k, :, :) (R_{k-1} x n_kR_k, outer stride m_k n_k R_k,
 * tt_embedding.cpp:31-37), reinterpreted row-major as N_k x R_k. */
static void reconstruct_padded_into(const or_cfg* c, const double* const* cores,
                                    int64_t row, double* out, double* buf, double* next) {
  int64_t parts[OR_MAXD];
  or_index_to_coordinate(c, row, parts);
  const int64_t inner0 = c->n[0] * c->R[1];
  const double* s0 = cores[0] + parts[0] * inner0;  /* R_0 = 1 */
  for (int64_t q = 0; q < inner0; ++q) buf[q] = s0[q];
  int64_t cols_done = c->n[0];
  for (int k = 1; k < c->d; ++k) {
    const int64_t rk = c->R[k];
    const int64_t inner = c->n[k] * c->R[k + 1];
    const int64_t outer = c->m[k] * inner;
    const double* base = cores[k] + parts[k] * inner;
    for (int64_t a = 0; a < cols_done; ++a)
      for (int64_t q = 0; q < inner; ++q) {
        double acc = 0.0;
        for (int64_t r = 0; r < rk; ++r) acc += buf[a * rk + r] * base[r * outer + q];
        next[a * inner + q] = acc;
      }
    cols_done *= c->n[k];
    double* t = buf; buf = next; next = t;
  }
  const int64_t pc = or_padded_cols(c);
  for (int64_t j = 0; j < pc; ++j) out[j] = buf[j];
}

/* lookup_batch (tt_embedding.cpp:110-125): validate every index against
 * num_nodes first (returns the first offending position, else -1), then
 * rows in input order, truncated to emb_dim. */
int64_t or_lookup_batch(const or_cfg* c, const double* const* cores, const int64_t* idx,
                        int64_t B, double* out, int nthreads) {
  for (int64_t b = 0; b < B; ++b)
    if (idx[b] < 0 || idx[b] >= c->num_nodes) return b;
  const int64_t cap = chain_cap(c), pc = or_padded_cols(c), N = c->emb_dim;
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads)
#endif
  {
    double* buf = (double*)malloc(sizeof(double) * (size_t)cap);
    double* next = (double*)malloc(sizeof(double) * (size_t)cap);
    double* padded = (double*)malloc(sizeof(double) * (size_t)pc);
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
    for (int64_t b = 0; b < B; ++b) {
      reconstruct_padded_into(c, cores, idx[b], padded, buf, next);
      for (int64_t j = 0; j < N; ++j) out[b * N + j] = padded[j];
    }
    free(buf); free(next); free(padded);
  }
  (void)nthreads;
  return -1;
}

/* ---- backward: autodiff.cpp:27-118 --------------------------------------- */
typedef struct {
  double* unf[OR_MAXD];
  double* left[OR_MAXD];
  double* right[OR_MAXD];
  double* prod;
  double* tmp;
  double* padded;
} bwd_scratch;

static void bwd_row(const or_cfg* c, const double* const* cores, int64_t row,
                    const double* up, double* const* grads, bwd_scratch* s,
                    const int64_t* left_cols, const int64_t* right_cols) {
  const int d = c->d;
  int64_t parts[OR_MAXD];
  or_index_to_coordinate(c, row, parts);
  /* slice_unfolding_copy (autodiff.cpp:27-36) */
  for (int k = 0; k < d; ++k) {
    const int64_t rp = c->R[k], inner = c->n[k] * c->R[k + 1], outer = c->m[k] * inner;
    const double* base = cores[k] + parts[k] * inner;
    for (int64_t r = 0; r < rp; ++r)
      for (int64_t q = 0; q < inner; ++q) s->unf[k][r * inner + q] = base[r * outer + q];
  }
  /* left chain (autodiff.cpp:81-85): left[k] is left_cols[k] x R_k */
  s->left[0][0] = 1.0;
  for (int k = 0; k + 1 < d; ++k) {
    const int64_t lc = left_cols[k], rk = c->R[k], inner = c->n[k] * c->R[k + 1];
    for (int64_t a = 0; a < lc; ++a)
      for (int64_t q = 0; q < inner; ++q) {
        double acc = 0.0;
        for (int64_t r = 0; r < rk; ++r) acc += s->left[k][a * rk + r] * s->unf[k][r * inner + q];
        s->left[k + 1][a * inner + q] = acc;  /* reshape to left_cols[k+1] x R_{k+1} */
      }
  }
  /* right chain (autodiff.cpp:87-94): right[k] is R_{k+1} x right_cols[k] */
  s->right[d - 1][0] = 1.0;
  for (int k = d - 1; k > 0; --k) {
    const int64_t rows = c->R[k] * c->n[k], rn = c->R[k + 1], rc = right_cols[k];
    for (int64_t a = 0; a < rows; ++a)
      for (int64_t q = 0; q < rc; ++q) {
        double acc = 0.0;
        for (int64_t t = 0; t < rn; ++t) acc += s->unf[k][a * rn + t] * s->right[k][t * rc + q];
        s->right[k - 1][a * rc + q] = acc;  /* reshape to R_k x n_k*right_cols[k] */
      }
  }
  /* zero-padded upstream (autodiff.cpp:96-97) */
  const int64_t pc = or_padded_cols(c);
  for (int64_t j = 0; j < pc; ++j) s->padded[j] = j < c->emb_dim ? up[j] : 0.0;
  /* contributions (autodiff.cpp:99-115): contrib = left^T * u_slice * right^T */
  for (int k = 0; k < d; ++k) {
    const int64_t n = c->n[k], rp = c->R[k], rn = c->R[k + 1], ik = parts[k];
    const int64_t lc = left_cols[k], rc = right_cols[k];
    double* g = grads[k];
    for (int64_t j = 0; j < n; ++j) {
      const double* u = s->padded + j * rc;  /* rows stride n*rc */
      /* tmp = left^T (rp x lc) * u_slice (lc x rc) */
      for (int64_t r = 0; r < rp; ++r)
        for (int64_t q = 0; q < rc; ++q) {
          double acc = 0.0;
          for (int64_t a = 0; a < lc; ++a) acc += s->left[k][a * rp + r] * u[a * n * rc + q];
          s->tmp[r * rc + q] = acc;
        }
      /* contrib = tmp (rp x rc) * right^T (rc x rn) */
      for (int64_t r = 0; r < rp; ++r)
        for (int64_t t = 0; t < rn; ++t) {
          double acc = 0.0;
          for (int64_t q = 0; q < rc; ++q) acc += s->tmp[r * rc + q] * s->right[k][t * rc + q];
          g[((r * c->m[k] + ik) * n + j) * rn + t] += acc;
        }
    }
  }
}

/* backward_lookup (autodiff.cpp:48-118).  Returns -1, or the first
 * out-of-range batch position.  grads[k] must hold core_size(k) doubles;
 * they are zero-filled here (CoreGradients::zeros, autodiff.cpp:40-46).
 * Rows accumulate in input order; with nthreads > 1 each thread owns a
 * contiguous row range and partial gradients are summed in thread order
 * (fixed-order reduction, SPEC.md "backward_lookup may parallelize ...
 * provided the final accumulation is deterministic"). */
int64_t or_backward_lookup(const or_cfg* c, const double* const* cores, const int64_t* idx,
                           int64_t B, const double* upstream, double* const* grads,
                           int nthreads) {
  const int d = c->d;
  for (int64_t b = 0; b < B; ++b)
    if (idx[b] < 0 || idx[b] >= c->num_nodes) return b;
  for (int k = 0; k < d; ++k) memset(grads[k], 0, sizeof(double) * (size_t)or_core_size(c, k));
  int64_t left_cols[OR_MAXD], right_cols[OR_MAXD];
  {
    int64_t acc = 1;
    for (int k = 0; k < d; ++k) { left_cols[k] = acc; acc *= c->n[k]; }
    acc = 1;
    for (int k = d - 1; k >= 0; --k) { right_cols[k] = acc; acc *= c->n[k]; }
  }
  int64_t maxsz = 1;
  for (int k = 0; k < d; ++k) {
    int64_t v = c->R[k] * c->n[k] * c->R[k + 1];
    if (left_cols[k] * c->R[k] > maxsz) maxsz = left_cols[k] * c->R[k];
    if (v > maxsz) maxsz = v;
    if (c->R[k + 1] * right_cols[k] > maxsz) maxsz = c->R[k + 1] * right_cols[k];
    if (c->R[k] * right_cols[k] > maxsz) maxsz = c->R[k] * right_cols[k];
    if (left_cols[k] * c->n[k] * c->R[k + 1] > maxsz) maxsz = left_cols[k] * c->n[k] * c->R[k + 1];
    if (c->R[k] * c->n[k] * right_cols[k] > maxsz) maxsz = c->R[k] * c->n[k] * right_cols[k];
  }
  maxsz += or_padded_cols(c);
  int nt = 1;
#ifdef _OPENMP
  nt = nthreads <= 0 ? omp_get_max_threads() : nthreads;
#endif
  if (nt > B) nt = B > 0 ? (int)B : 1;
  double** part = (double**)calloc((size_t)nt * d, sizeof(double*));
  for (int t = 1; t < nt; ++t)
    for (int k = 0; k < d; ++k)
      part[t * d + k] = (double*)calloc((size_t)or_core_size(c, k), sizeof(double));
  for (int k = 0; k < d; ++k) part[k] = grads[k];
#ifdef _OPENMP
#pragma omp parallel num_threads(nt)
#endif
  {
    int t = 0;
#ifdef _OPENMP
    t = omp_get_thread_num();
#endif
    bwd_scratch s;
    for (int k = 0; k < d; ++k) {
      s.unf[k] = (double*)malloc(sizeof(double) * (size_t)maxsz);
      s.left[k] = (double*)malloc(sizeof(double) * (size_t)maxsz);
      s.right[k] = (double*)malloc(sizeof(double) * (size_t)maxsz);
    }
    s.prod = (double*)malloc(sizeof(double) * (size_t)maxsz);
    s.tmp = (double*)malloc(sizeof(double) * (size_t)maxsz);
    s.padded = (double*)malloc(sizeof(double) * (size_t)maxsz);
    const int64_t lo = B * t / nt, hi = B * (t + 1) / nt;
    for (int64_t b = lo; b < hi; ++b)
      bwd_row(c, cores, idx[b], upstream + b * c->emb_dim, part + t * d, &s, left_cols, right_cols);
    for (int k = 0; k < d; ++k) { free(s.unf[k]); free(s.left[k]); free(s.right[k]); }
    free(s.prod); free(s.tmp); free(s.padded);
  }
  for (int t = 1; t < nt; ++t)
    for (int k = 0; k < d; ++k) {
      const int64_t sz = or_core_size(c, k);
      for (int64_t e = 0; e < sz; ++e) grads[k][e] += part[t * d + k][e];
      free(part[t * d + k]);
    }
  free(part);
  return -1;
}

/* ---- optimizer: autodiff.cpp:120-173 + Adagrad (new) --------------------- */
enum { OR_SGD = 0, OR_ADAM = 1, OR_ADAGRAD = 2 };

/* apply_update (autodiff.cpp:147-173): reject before any mutation if any
 * gradient entry is non-finite (returns that core's index); else step++
 * (also for SGD) and update every entry densely.
 *   SGD      G -= lr g                                   (:165-167)
 *   Adam     bias-corrected, adam_step (:135-145)          state1=m state2=v
 *   Adagrad  h += g^2; G -= lr g / (sqrt(h) + eps), h_0=0  state1=h  (new;
 *            pinned formula, BASELINE.md "CPU-baseline plan")             */
int or_apply_update(const or_cfg* c, double* const* cores, const double* const* grads,
                    int kind, double lr, double beta1, double beta2, double eps,
                    int64_t* step, double* const* state1, double* const* state2) {
  for (int k = 0; k < c->d; ++k) {
    const int64_t sz = or_core_size(c, k);
    for (int64_t e = 0; e < sz; ++e)
      if (!isfinite(grads[k][e])) return k;
  }
  *step += 1;
  for (int k = 0; k < c->d; ++k) {
    const int64_t sz = or_core_size(c, k);
    double* p = cores[k];
    const double* g = grads[k];
    if (kind == OR_SGD) {
      for (int64_t e = 0; e < sz; ++e) p[e] -= lr * g[e];
    } else if (kind == OR_ADAM) {
      const double bc1 = 1.0 - pow(beta1, (double)*step);
      const double bc2 = 1.0 - pow(beta2, (double)*step);
      double* m = state1[k];
      double* v = state2[k];
      for (int64_t e = 0; e < sz; ++e) {
        m[e] = beta1 * m[e] + (1.0 - beta1) * g[e];
        v[e] = beta2 * v[e] + (1.0 - beta2) * g[e] * g[e];
        p[e] -= lr * (m[e] / bc1) / (sqrt(v[e] / bc2) + eps);
      }
    } else {
      double* h = state1[k];
      for (int64_t e = 0; e < sz; ++e) {
        h[e] += g[e] * g[e];
        p[e] -= lr * g[e] / (sqrt(h[e]) + eps);
      }
    }
  }
  return -1;
}

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
