/*
 * longctx_oracle.c -- CPU restatement of the reference's sparse + DCA prefill
 * attention path, in plain C11 / fp64.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py may load this library, and only as the checker.
 * The product (paper_2501_15383_b200/) never links or calls it.
 *
 * Every function restates one reference function (paths relative to
 * /root/reference/proj); it is compiled with -ffp-contract=off like the
 * reference (core/CMakeLists.txt:21-22) so summation order and rounding match.
 * Pinned against the reference itself (oracle/_ref, built from the reference
 * sources by oracle/Makefile) and against the committed goldens in
 * proj/out/sparsity/*  (tests/test_oracle_pin.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define LCO_OK 0
#define LCO_E_DIMENSION 1
#define LCO_E_CONFIG 2
#define LCO_E_DOMAIN 3
#define LCO_E_CAUSALITY 4
#define LCO_E_EMPTY_ROW 5
#define LCO_E_EMPTY_CALIBRATION 6
#define LCO_E_ALLOC 99

/* ------------------------------------------------------------------------ */
/* RNG restatement: std::mt19937_64 + libstdc++ generate_canonical<double,53>,
 * uniform_real_distribution and normal_distribution (Marsaglia polar).
 * Used by the planted / random_input fixture generators
 * (tests/testutil.hpp:18-41, core/src/planted.cpp:33-150). */

typedef struct {
  uint64_t mt[312];
  int idx;
} lco_mt64;

void lco_mt64_seed(lco_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i) {
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  }
  g->idx = 312;
}

uint64_t lco_mt64_next(lco_mt64* g) {
  if (g->idx >= 312) {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    for (int k = 0; k < 312; ++k) {
      uint64_t y = (g->mt[k] & upper) | (g->mt[(k + 1) % 312] & lower);
      uint64_t v = g->mt[(k + 156) % 312] ^ (y >> 1);
      if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
      g->mt[k] = v;
    }
    g->idx = 0;
  }
  uint64_t z = g->mt[g->idx++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= (z >> 43);
  return z;
}

/* generate_canonical<double, 53>(mt19937_64): one draw, x / 2^64, clamped < 1 */
double lco_canonical(lco_mt64* g) {
  double x = (double)lco_mt64_next(g);
  double r = x / 18446744073709551616.0;
  if (r >= 1.0) r = nextafter(1.0, 0.0);
  return r;
}

double lco_uniform(lco_mt64* g, double a, double b) { return lco_canonical(g) * (b - a) + a; }

typedef struct {
  double saved;
  int has_saved;
} lco_normal;

double lco_normal_draw(lco_normal* nd, lco_mt64* g) {
  if (nd->has_saved) {
    nd->has_saved = 0;
    return nd->saved;
  }
  double x, y, r2;
  do {
    x = 2.0 * lco_canonical(g) - 1.0;
    y = 2.0 * lco_canonical(g) - 1.0;
    r2 = x * x + y * y;
  } while (r2 > 1.0 || r2 == 0.0);
  const double mult = sqrt(-2 * log(r2) / r2);
  nd->saved = x * mult;
  nd->has_saved = 1;
  return y * mult;
}

/* testutil.hpp:18-41 / harness.cpp:123-140: q, k, v uniform(-1, 1) in that
 * order, row-major n x dim each. */
void lco_random_input(uint64_t seed, int64_t n, int64_t dim, double* q, double* k, double* v) {
  lco_mt64 g;
  lco_mt64_seed(&g, seed);
  for (int64_t i = 0; i < n * dim; ++i) q[i] = lco_uniform(&g, -1.0, 1.0);
  for (int64_t i = 0; i < n * dim; ++i) k[i] = lco_uniform(&g, -1.0, 1.0);
  for (int64_t i = 0; i < n * dim; ++i) v[i] = lco_uniform(&g, -1.0, 1.0);
}

/* Continue an existing generator (for tests that draw several inputs from one rng). */
void lco_random_input_from(lco_mt64* g, int64_t n, int64_t dim, double* q, double* k, double* v) {
  for (int64_t i = 0; i < n * dim; ++i) q[i] = lco_uniform(g, -1.0, 1.0);
  for (int64_t i = 0; i < n * dim; ++i) k[i] = lco_uniform(g, -1.0, 1.0);
  for (int64_t i = 0; i < n * dim; ++i) v[i] = lco_uniform(g, -1.0, 1.0);
}

size_t lco_mt64_size(void) { return sizeof(lco_mt64); }

/* ------------------------------------------------------------------------ */
/* RoPE: attention.cpp:14-33 (interleaved pairs (2p, 2p+1), fp64 angle). */

void lco_rope_thetas(int64_t dim, double base, double* thetas) {
  for (int64_t p = 0; p < dim / 2; ++p) thetas[p] = pow(base, -(double)(2 * p) / (double)dim);
}

void lco_rope_rotate_row(const double* row, int64_t dim, int64_t position, const double* thetas,
                         double* out) {
  for (int64_t p = 0; p < dim / 2; ++p) {
    const double angle = (double)position * thetas[p];
    const double c = cos(angle);
    const double s = sin(angle);
    const double x = row[2 * p];
    const double y = row[2 * p + 1];
    out[2 * p] = x * c - y * s;
    out[2 * p + 1] = x * s + y * c;
  }
}

/* ------------------------------------------------------------------------ */
/* DCA: dca.cpp:11-113. */

int lco_chunk_validate(int64_t s, int64_t c, int64_t w) {
  if (s <= 0) return LCO_E_CONFIG;
  if (c <= 0) return LCO_E_CONFIG;
  if (s > c) return LCO_E_CONFIG;
  int64_t bound = s < (c - s) ? s : (c - s);
  if (w > bound) return LCO_E_CONFIG;
  return LCO_OK;
}

double lco_yarn_temperature(double scale) {
  if (scale <= 1.0) return 1.0;
  const double root = 0.1 * log(scale) + 1.0;
  return 1.0 / (root * root);
}

/* 0 intra, 1 successive, 2 inter (dca.cpp:53-60) */
int lco_classify_pair(int64_t i, int64_t j, int64_t s) {
  const int64_t qc = i / s, kc = j / s;
  if (qc == kc) return 0;
  if (qc == kc + 1) return 1;
  return 2;
}

int64_t lco_dca_relative(int64_t i, int64_t j, int64_t s, int64_t c) {
  const int kind = lco_classify_pair(i, j, s);
  const int64_t key_pos = j % s;
  int64_t query_pos;
  if (kind == 0) {
    query_pos = i % s;
  } else if (kind == 1) {
    query_pos = (i % s + s) < (c - 1) ? (i % s + s) : (c - 1);
  } else {
    query_pos = c - 1;
  }
  return query_pos - key_pos;
}

/* ------------------------------------------------------------------------ */
/* Softmax + accumulate over an admitted list: attention.cpp:35-51. */

static double attend_admitted(const double* logits, const int64_t* admitted, int64_t cnt,
                              const double* v, int64_t dim, double* out_row) {
  double row_max = -INFINITY;
  for (int64_t a = 0; a < cnt; ++a) {
    const double l = logits[admitted[a]];
    if (l > row_max) row_max = l;
  }
  double sum = 0.0;
  for (int64_t a = 0; a < cnt; ++a) sum += exp(logits[admitted[a]] - row_max);
  for (int64_t d = 0; d < dim; ++d) out_row[d] = 0.0;
  for (int64_t a = 0; a < cnt; ++a) {
    const int64_t j = admitted[a];
    const double w = exp(logits[j] - row_max) / sum;
    for (int64_t d = 0; d < dim; ++d) out_row[d] += w * v[j * dim + d];
  }
  return row_max + log(sum);
}

/* ------------------------------------------------------------------------ */
/* Estimator: sparse.cpp:142-188.  q is nq x dim (the chunk rows), k is nk x dim
 * (the key timeline, queries trail it).  pos_mode 0 = Standard, 1 = DcaContinuous
 * (rel clamped to c-1).  est_out is block x nk, block = min(last_q, nq). */
int lco_estimate_block(const double* q, int64_t nq, const double* k, int64_t nk, int64_t dim,
                       int64_t last_q, int pos_mode, int64_t c, double rope_base,
                       double* est_out) {
  if (last_q <= 0) return LCO_E_CONFIG;
  if (dim <= 0 || dim % 2 != 0) return LCO_E_CONFIG;
  if (nq == 0 || nk == 0) return LCO_E_DIMENSION;
  if (nq > nk) return LCO_E_DIMENSION;
  if (pos_mode == 1 && c <= 0) return LCO_E_CONFIG;
  const int64_t block = last_q < nq ? last_q : nq;
  const int64_t offset = nk - nq;
  const double inv_scale = 1.0 / sqrt((double)dim);
  double* thetas = (double*)malloc(sizeof(double) * (size_t)(dim / 2));
  double* logits = (double*)malloc(sizeof(double) * (size_t)nk);
  double* q_rot = (double*)malloc(sizeof(double) * (size_t)dim);
  if (!thetas || !logits || !q_rot) return LCO_E_ALLOC;
  lco_rope_thetas(dim, rope_base, thetas);
  memset(est_out, 0, sizeof(double) * (size_t)(block * nk));
  for (int64_t r = 0; r < block; ++r) {
    const int64_t qrow = nq - block + r;
    const int64_t gi = offset + qrow;
    for (int64_t j = 0; j <= gi; ++j) {
      int64_t rel = gi - j;
      if (pos_mode == 1 && rel > c - 1) rel = c - 1;
      lco_rope_rotate_row(q + qrow * dim, dim, rel, thetas, q_rot);
      double acc = 0.0;
      for (int64_t d = 0; d < dim; ++d) acc += q_rot[d] * k[j * dim + d];
      logits[j] = acc * inv_scale;
    }
    double row_max = -INFINITY;
    for (int64_t j = 0; j <= gi; ++j)
      if (logits[j] > row_max) row_max = logits[j];
    double sum = 0.0;
    for (int64_t j = 0; j <= gi; ++j) sum += exp(logits[j] - row_max);
    for (int64_t j = 0; j <= gi; ++j) est_out[r * nk + j] = exp(logits[j] - row_max) / sum;
  }
  free(thetas);
  free(logits);
  free(q_rot);
  return LCO_OK;
}

/* ------------------------------------------------------------------------ */
/* Selection: sparse.cpp:15-24 (top_lines), 190-230 (select_critical). */

static const double* g_sort_scores;
static int cmp_line(const void* a, const void* b) {
  const int64_t ia = *(const int64_t*)a, ib = *(const int64_t*)b;
  const double sa = g_sort_scores[ia], sb = g_sort_scores[ib];
  if (sa != sb) return sa > sb ? -1 : 1;
  return ia < ib ? -1 : (ia > ib ? 1 : 0);
}
static int cmp_i64(const void* a, const void* b) {
  const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* total order (score desc, index asc) => equivalent to the reference's
 * stable_sort with that comparator; take the first count. */
static int64_t top_lines(const double* scores, int64_t n, int64_t count, int64_t* out) {
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  g_sort_scores = scores;
  qsort(order, (size_t)n, sizeof(int64_t), cmp_line);
  const int64_t m = count < n ? count : n;
  for (int64_t i = 0; i < m; ++i) out[i] = order[i];
  free(order);
  return m;
}

static int64_t sort_unique(int64_t* v, int64_t cnt) {
  if (cnt == 0) return 0;
  qsort(v, (size_t)cnt, sizeof(int64_t), cmp_i64);
  int64_t w = 1;
  for (int64_t i = 1; i < cnt; ++i)
    if (v[i] != v[w - 1]) v[w++] = v[i];
  return w;
}

/* Selection from already-reduced line scores (the stage after the row sums of
 * select_critical, sparse.cpp:219-229).  out_v needs V+1, out_s needs S+block. */
int lco_select_from_scores(const double* col_score, const double* slash_score, int64_t n,
                           int64_t block, int64_t budget_v, int64_t budget_s, int force_sink,
                           int force_band, int64_t* out_v, int64_t* nv, int64_t* out_s,
                           int64_t* ns) {
  int64_t cv = top_lines(col_score, n, budget_v, out_v);
  int64_t cs = top_lines(slash_score, n, budget_s, out_s);
  if (force_sink) out_v[cv++] = 0;
  if (force_band)
    for (int64_t d = 0; d < block; ++d) out_s[cs++] = d;
  *nv = sort_unique(out_v, cv);
  *ns = sort_unique(out_s, cs);
  return LCO_OK;
}

int lco_select_critical(const double* est, int64_t block, int64_t n, int64_t budget_v,
                        int64_t budget_s, int force_sink, int force_band, int slash_mean,
                        int64_t* out_v, int64_t* nv, int64_t* out_s, int64_t* ns,
                        double* col_out, double* slash_out) {
  if (block == 0 || block > n) return LCO_E_DIMENSION;
  double* col = (double*)calloc((size_t)n, sizeof(double));
  double* ssum = (double*)calloc((size_t)n, sizeof(double));
  int64_t* scnt = (int64_t*)calloc((size_t)n, sizeof(int64_t));
  double* sscore = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t r = 0; r < block; ++r) {
    const int64_t gi = n - block + r;
    for (int64_t j = 0; j <= gi; ++j) {
      const double w = est[r * n + j];
      col[j] += w;
      ssum[gi - j] += w;
      scnt[gi - j] += 1;
    }
  }
  for (int64_t d = 0; d < n; ++d) {
    if (scnt[d] == 0)
      sscore[d] = -INFINITY;
    else
      sscore[d] = slash_mean ? ssum[d] / (double)scnt[d] : ssum[d];
  }
  if (col_out) memcpy(col_out, col, sizeof(double) * (size_t)n);
  if (slash_out) memcpy(slash_out, sscore, sizeof(double) * (size_t)n);
  int st = lco_select_from_scores(col, sscore, n, block, budget_v, budget_s, force_sink,
                                  force_band, out_v, nv, out_s, ns);
  free(col);
  free(ssum);
  free(scnt);
  free(sscore);
  return st;
}

/* ------------------------------------------------------------------------ */
/* CriticalSet row semantics: sparse.cpp:85-113 (admitted_row), 115-119, 286-291. */

int64_t lco_admitted_row(const int64_t* verts, int64_t nv, const int64_t* slashes, int64_t ns,
                         int64_t i, int64_t* out) {
  int64_t cnt = 0;
  int64_t a = 0;         /* verticals ascending */
  int64_t b = ns - 1;    /* slashes descending -> keys ascending */
  while (b >= 0 && slashes[b] > i) --b;
  while (a < nv && verts[a] <= i && b >= 0) {
    const int64_t v = verts[a], s = i - slashes[b];
    if (v == s) {
      out[cnt++] = v;
      ++a;
      --b;
    } else if (v < s) {
      out[cnt++] = v;
      ++a;
    } else {
      out[cnt++] = s;
      --b;
    }
  }
  for (; a < nv && verts[a] <= i; ++a) out[cnt++] = verts[a];
  for (; b >= 0; --b) out[cnt++] = i - slashes[b];
  if (cnt == 0) out[cnt++] = i;
  return cnt;
}

int64_t lco_admitted_count(const int64_t* verts, int64_t nv, const int64_t* slashes, int64_t ns,
                           int64_t n) {
  int64_t* buf = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nv + ns + 1));
  int64_t total = 0;
  for (int64_t i = 0; i < n; ++i) total += lco_admitted_row(verts, nv, slashes, ns, i, buf);
  free(buf);
  return total;
}

/* ------------------------------------------------------------------------ */
/* Attention over admitted rows.  One routine covers
 *   sparse_attention (sparse.cpp:232-284),
 *   full_attention (attention.cpp:142-185; verts == NULL && slashes == NULL and
 *                   dense != 0),
 *   chunked_prefill's per-chunk row loop (sparse.cpp:368-396).
 * rel_mode 0: q, k pre-rotated by positions_q / positions_k (standard path).
 * rel_mode 1: per entry rope(q_i, dca_relative(i, j)) . k_j (override path).
 * rows [row_begin, row_end) are computed. */
static int attention_rows(const double* q, const double* k, const double* v, int64_t n,
                          int64_t dim, const int64_t* pos_q, const int64_t* pos_k,
                          double rope_base, double temperature, const int64_t* verts,
                          int64_t nv, const int64_t* slashes, int64_t ns, int dense,
                          int rel_mode, int64_t s, int64_t c, int64_t row_begin,
                          int64_t row_end, double* out, double* lse) {
  const double inv_scale = 1.0 / (temperature * sqrt((double)dim));
  double* thetas = (double*)malloc(sizeof(double) * (size_t)(dim / 2));
  lco_rope_thetas(dim, rope_base, thetas);
  double* qr = NULL;
  double* kr = NULL;
  if (rel_mode == 0) {
    qr = (double*)malloc(sizeof(double) * (size_t)(n * dim));
    kr = (double*)malloc(sizeof(double) * (size_t)(n * dim));
    for (int64_t i = 0; i < n; ++i) {
      lco_rope_rotate_row(q + i * dim, dim, pos_q[i], thetas, qr + i * dim);
      lco_rope_rotate_row(k + i * dim, dim, pos_k[i], thetas, kr + i * dim);
    }
  }
  double* logits = (double*)malloc(sizeof(double) * (size_t)n);
  int64_t* adm = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + nv + ns + 1));
  double* q_rot = (double*)malloc(sizeof(double) * (size_t)dim);
  for (int64_t i = row_begin; i < row_end; ++i) {
    int64_t cnt;
    if (dense) {
      for (int64_t j = 0; j <= i; ++j) adm[j] = j;
      cnt = i + 1;
    } else {
      cnt = lco_admitted_row(verts, nv, slashes, ns, i, adm);
    }
    for (int64_t a = 0; a < cnt; ++a) {
      const int64_t j = adm[a];
      double acc = 0.0;
      if (rel_mode == 0) {
        for (int64_t d = 0; d < dim; ++d) acc += qr[i * dim + d] * kr[j * dim + d];
      } else {
        lco_rope_rotate_row(q + i * dim, dim, lco_dca_relative(i, j, s, c), thetas, q_rot);
        for (int64_t d = 0; d < dim; ++d) acc += q_rot[d] * k[j * dim + d];
      }
      logits[j] = acc * inv_scale;
    }
    lse[i] = attend_admitted(logits, adm, cnt, v, dim, out + i * dim);
  }
  free(thetas);
  free(qr);
  free(kr);
  free(logits);
  free(adm);
  free(q_rot);
  return LCO_OK;
}

static int validate_input(const double* q, const double* k, const double* v, int64_t n,
                          int64_t dim, const int64_t* pos_q, const int64_t* pos_k,
                          double rope_base, double temperature) {
  if (n == 0) return LCO_E_DIMENSION;
  if (dim == 0 || dim % 2 != 0) return LCO_E_CONFIG;
  for (int64_t i = 0; i < n; ++i)
    if (pos_q[i] < 0 || pos_k[i] < 0) return LCO_E_DOMAIN;
  if (!(rope_base > 0.0)) return LCO_E_DOMAIN;
  if (!(temperature > 0.0)) return LCO_E_DOMAIN;
  for (int64_t i = 0; i < n * dim; ++i)
    if (!isfinite(q[i]) || !isfinite(k[i]) || !isfinite(v[i])) return LCO_E_DOMAIN;
  return LCO_OK;
}

int lco_sparse_attention(const double* q, const double* k, const double* v, int64_t n,
                         int64_t dim, const int64_t* pos_q, const int64_t* pos_k,
                         double rope_base, double temperature, const int64_t* verts,
                         int64_t nv, const int64_t* slashes, int64_t ns, int rel_mode,
                         int64_t s, int64_t c, double* out, double* lse) {
  int st = validate_input(q, k, v, n, dim, pos_q, pos_k, rope_base, temperature);
  if (st) return st;
  return attention_rows(q, k, v, n, dim, pos_q, pos_k, rope_base, temperature, verts, nv,
                        slashes, ns, 0, rel_mode, s, c, 0, n, out, lse);
}

/* Listed rows only (row-sampled parity at 128K-1M, where whole-sequence oracle runs are
 * infeasible): the same per-row computation as attention_rows / sparse_attention
 * (sparse.cpp:232-284; DCA override sparse.cpp:385-393), out [nrows][dim], lse [nrows].
 * dense != 0: every key j <= i (full_attention). */
int lco_attention_row_list(const double* q, const double* k, const double* v, int64_t n,
                           int64_t dim, const int64_t* pos_q, const int64_t* pos_k,
                           double rope_base, double temperature, const int64_t* verts,
                           int64_t nv, const int64_t* slashes, int64_t ns, int dense,
                           int rel_mode, int64_t s, int64_t c, const int64_t* rows,
                           int64_t nrows, double* out, double* lse) {
  const double inv_scale = 1.0 / (temperature * sqrt((double)dim));
  double* thetas = (double*)malloc(sizeof(double) * (size_t)(dim / 2));
  lco_rope_thetas(dim, rope_base, thetas);
  double* logits = (double*)malloc(sizeof(double) * (size_t)n);
  int64_t* adm = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + nv + ns + 1));
  double* q_rot = (double*)malloc(sizeof(double) * (size_t)dim);
  double* k_rot = (double*)malloc(sizeof(double) * (size_t)dim);
  for (int64_t x = 0; x < nrows; ++x) {
    const int64_t i = rows[x];
    if (i < 0 || i >= n) {
      free(thetas); free(logits); free(adm); free(q_rot); free(k_rot);
      return LCO_E_DIMENSION;
    }
    int64_t cnt;
    if (dense) {
      for (int64_t j = 0; j <= i; ++j) adm[j] = j;
      cnt = i + 1;
    } else {
      cnt = lco_admitted_row(verts, nv, slashes, ns, i, adm);
    }
    if (rel_mode == 0) lco_rope_rotate_row(q + i * dim, dim, pos_q[i], thetas, q_rot);
    for (int64_t a = 0; a < cnt; ++a) {
      const int64_t j = adm[a];
      double acc = 0.0;
      if (rel_mode == 0) {
        lco_rope_rotate_row(k + j * dim, dim, pos_k[j], thetas, k_rot);
        for (int64_t d = 0; d < dim; ++d) acc += q_rot[d] * k_rot[d];
      } else {
        lco_rope_rotate_row(q + i * dim, dim, lco_dca_relative(i, j, s, c), thetas, q_rot);
        for (int64_t d = 0; d < dim; ++d) acc += q_rot[d] * k[j * dim + d];
      }
      logits[j] = acc * inv_scale;
    }
    lse[x] = attend_admitted(logits, adm, cnt, v, dim, out + x * dim);
  }
  free(thetas);
  free(logits);
  free(adm);
  free(q_rot);
  free(k_rot);
  return LCO_OK;
}

int lco_full_attention(const double* q, const double* k, const double* v, int64_t n,
                       int64_t dim, const int64_t* pos_q, const int64_t* pos_k,
                       double rope_base, double temperature, int rel_mode, int64_t s,
                       int64_t c, double* out, double* lse) {
  int st = validate_input(q, k, v, n, dim, pos_q, pos_k, rope_base, temperature);
  if (st) return st;
  return attention_rows(q, k, v, n, dim, pos_q, pos_k, rope_base, temperature, NULL, 0, NULL,
                        0, 1, rel_mode, s, c, 0, n, out, lse);
}

/* dca.cpp:93-113: iota positions, yarn temperature, identity shortcut. */
int lco_dca_attention(const double* q, const double* k, const double* v, int64_t n, int64_t dim,
                      double rope_base, int64_t s, int64_t c, int64_t w, double scale_factor,
                      double* out, double* lse) {
  int st = lco_chunk_validate(s, c, w);
  if (st) return st;
  if (!(scale_factor > 0.0)) return LCO_E_DOMAIN;
  const double temp = lco_yarn_temperature(scale_factor);
  int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) pos[i] = i;
  if (n <= s && scale_factor <= 1.0)
    st = lco_full_attention(q, k, v, n, dim, pos, pos, rope_base, temp, 0, s, c, out, lse);
  else
    st = lco_full_attention(q, k, v, n, dim, pos, pos, rope_base, temp, 1, s, c, out, lse);
  free(pos);
  return st;
}

/* ------------------------------------------------------------------------ */
/* chunked_prefill: sparse.cpp:293-399.
 * mode 0 = Full, 1 = Sparse; pos_mode 0 = Standard, 1 = DcaContinuous.
 * Selections are written per chunk: sel_v[chunk * cap_v ...], sel_nv[chunk],
 * same for slashes (cap_v >= V+1, cap_s >= S+last_q). */
int lco_chunked_prefill(const double* q, const double* k, const double* v, int64_t n,
                        int64_t dim, const int64_t* pos_q, const int64_t* pos_k,
                        double rope_base, double temperature, int64_t chunk_len,
                        int64_t last_q, int64_t budget_v, int64_t budget_s, int mode,
                        int pos_mode, int64_t s, int64_t c, int64_t w, int force_sink,
                        int force_band, int slash_mean, double* out, double* lse,
                        int64_t* sel_v, int64_t* sel_nv, int64_t cap_v, int64_t* sel_s,
                        int64_t* sel_ns, int64_t cap_s) {
  int st = validate_input(q, k, v, n, dim, pos_q, pos_k, rope_base, temperature);
  if (st) return st;
  if (chunk_len <= 0) return LCO_E_CONFIG;
  if (last_q <= 0) return LCO_E_CONFIG;
  if (mode == 1 && chunk_len < last_q) return LCO_E_CONFIG;
  const int dca = pos_mode == 1;
  if (dca) {
    st = lco_chunk_validate(s, c, w);
    if (st) return st;
  }
  int64_t chunk = 0;
  double* est = NULL;
  int64_t* vbuf = (int64_t*)malloc(sizeof(int64_t) * (size_t)(budget_v + 2));
  int64_t* sbuf = (int64_t*)malloc(sizeof(int64_t) * (size_t)(budget_s + last_q + 1));
  for (int64_t t0 = 0; t0 < n; t0 += chunk_len, ++chunk) {
    const int64_t t1 = (t0 + chunk_len) < n ? (t0 + chunk_len) : n;
    int64_t nv = 0, ns = 0;
    if (mode == 1) {
      const int64_t block = last_q < (t1 - t0) ? last_q : (t1 - t0);
      est = (double*)realloc(est, sizeof(double) * (size_t)(block * t1));
      st = lco_estimate_block(q + t0 * dim, t1 - t0, k, t1, dim, last_q, pos_mode, c, rope_base,
                              est);
      if (st) break;
      st = lco_select_critical(est, block, t1, budget_v, budget_s, force_sink, force_band,
                               slash_mean, vbuf, &nv, sbuf, &ns, NULL, NULL);
      if (st) break;
      if (sel_nv) {
        sel_nv[chunk] = nv;
        sel_ns[chunk] = ns;
        for (int64_t a = 0; a < nv && a < cap_v; ++a) sel_v[chunk * cap_v + a] = vbuf[a];
        for (int64_t a = 0; a < ns && a < cap_s; ++a) sel_s[chunk * cap_s + a] = sbuf[a];
      }
    }
    /* rows [t0, t1) see keys [0, t1): the prefix of the full input */
    st = attention_rows(q, k, v, t1, dim, pos_q, pos_k, rope_base, temperature, vbuf, nv, sbuf,
                        ns, mode == 0, dca ? 1 : 0, s, c, t0, t1, out, lse);
    if (st) break;
  }
  free(est);
  free(vbuf);
  free(sbuf);
  return st;
}

/* ------------------------------------------------------------------------ */
/* Recall: refine.cpp:51-72 (attention_recall), 16-27 (reduce). */
int lco_attention_recall(const double* lse_sparse, const double* lse_full, int64_t n,
                         double slack, double* per_query, double* aggregate) {
  if (n == 0) return LCO_E_DIMENSION;
  double sum = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double r = exp(lse_sparse[i] - lse_full[i]);
    if (r > 1.0 + slack) return LCO_E_DOMAIN;
    if (r > 1.0) r = 1.0;
    if (per_query) per_query[i] = r;
    sum += r;
  }
  *aggregate = sum / (double)n;
  return LCO_OK;
}

double lco_reduce_fraction_above(const double* per_query, int64_t n, double tau) {
  int64_t above = 0;
  for (int64_t i = 0; i < n; ++i)
    if (per_query[i] >= tau) ++above;
  return (double)above / (double)n;
}

/* ------------------------------------------------------------------------ */
/* Planted generator: planted.cpp:33-150 (+ the random_unit helper 15-29). */

static void random_unit(lco_mt64* g, int64_t dim, double* v) {
  lco_normal nd = {0.0, 0};
  double norm2;
  do {
    norm2 = 0.0;
    for (int64_t d = 0; d < dim; ++d) {
      v[d] = lco_normal_draw(&nd, g);
      norm2 += v[d] * v[d];
    }
  } while (norm2 == 0.0);
  const double inv = 1.0 / sqrt(norm2);
  for (int64_t d = 0; d < dim; ++d) v[d] *= inv;
}

int lco_make_planted(int64_t n, int64_t dim, double rope_base, const int64_t* vcols, int64_t nvc,
                     const int64_t* soffs, int64_t nso, double strength, double vstrength,
                     double sstrength, double query_noise, double shared_scale, uint64_t seed,
                     int use_dca, int64_t s, int64_t c, int64_t w, const int64_t* carrier_pairs,
                     int64_t ncp, double* q, double* k, double* v) {
  if (n == 0 || dim == 0 || dim % 2 != 0) return LCO_E_CONFIG;
  const int64_t P = dim / 2;
  for (int64_t a = 0; a < ncp; ++a)
    if (carrier_pairs[a] >= P) return LCO_E_CONFIG;
  for (int64_t a = 0; a < nvc; ++a)
    if (vcols[a] >= n) return LCO_E_CONFIG;
  for (int64_t a = 0; a < nso; ++a)
    if (soffs[a] >= n) return LCO_E_CONFIG;
  if (use_dca) {
    int st = lco_chunk_validate(s, c, w);
    if (st) return st;
  }
  lco_mt64 g;
  lco_mt64_seed(&g, seed);
  double* thetas = (double*)malloc(sizeof(double) * (size_t)P);
  lco_rope_thetas(dim, rope_base, thetas);

  /* shared pairs: p >= 1 with theta_p * n <= 0.5, else the last pair */
  int* is_shared = (int*)calloc((size_t)P, sizeof(int));
  int64_t nshared = 0;
  for (int64_t p = 1; p < P; ++p)
    if (thetas[p] * (double)n <= 0.5) {
      is_shared[p] = 1;
      ++nshared;
    }
  if (nshared == 0) {
    is_shared[P - 1] = 1;
    nshared = 1;
  }
  int* is_carrier = (int*)calloc((size_t)P, sizeof(int));
  int64_t ncarrier = 0;
  if (ncp > 0) {
    for (int64_t a = 0; a < ncp; ++a) is_carrier[carrier_pairs[a]] = 1;
    for (int64_t p = 0; p < P; ++p) ncarrier += is_carrier[p];
  } else {
    for (int64_t p = 0; p < P; ++p)
      if (!is_shared[p]) {
        is_carrier[p] = 1;
        ++ncarrier;
      }
  }
  if (ncarrier == 0) {
    free(thetas);
    free(is_shared);
    free(is_carrier);
    return LCO_E_CONFIG;
  }
  /* carrier pair order: the reference iterates its carrier_pairs vector in
   * order (user-given order, or ascending complement) */
  int64_t* corder = (int64_t*)malloc(sizeof(int64_t) * (size_t)P);
  int64_t nco = 0;
  if (ncp > 0) {
    for (int64_t a = 0; a < ncp; ++a) corder[nco++] = carrier_pairs[a];
  } else {
    for (int64_t p = 0; p < P; ++p)
      if (is_carrier[p]) corder[nco++] = p;
  }

  double* shared = (double*)calloc((size_t)dim, sizeof(double));
  {
    lco_normal nd = {0.0, 0};
    double norm2 = 0.0;
    for (int64_t p = 1; p < P; ++p) {
      if (!is_shared[p]) continue;
      shared[2 * p] = lco_normal_draw(&nd, &g);
      shared[2 * p + 1] = lco_normal_draw(&nd, &g);
      norm2 += shared[2 * p] * shared[2 * p] + shared[2 * p + 1] * shared[2 * p + 1];
    }
    if (is_shared[0]) { /* only reachable when P == 1 */
      shared[0] = lco_normal_draw(&nd, &g);
      shared[1] = lco_normal_draw(&nd, &g);
      norm2 += shared[0] * shared[0] + shared[1] * shared[1];
    }
    const double inv = 1.0 / sqrt(norm2);
    for (int64_t d = 0; d < dim; ++d) shared[d] *= inv;
  }
  double* carrier = (double*)calloc((size_t)(n * dim), sizeof(double));
  {
    lco_normal nd = {0.0, 0};
    for (int64_t i = 0; i < n; ++i) {
      double* u = carrier + i * dim;
      double norm2 = 0.0;
      for (int64_t a = 0; a < nco; ++a) {
        const int64_t p = corder[a];
        u[2 * p] = lco_normal_draw(&nd, &g);
        u[2 * p + 1] = lco_normal_draw(&nd, &g);
        norm2 += u[2 * p] * u[2 * p] + u[2 * p + 1] * u[2 * p + 1];
      }
      const double inv = 1.0 / sqrt(norm2);
      for (int64_t d = 0; d < dim; ++d) u[d] *= inv;
    }
  }
  double* tmp = (double*)malloc(sizeof(double) * (size_t)dim);
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t d = 0; d < dim; ++d)
      q[i * dim + d] = shared_scale * shared[d] + query_noise * carrier[i * dim + d];
    random_unit(&g, dim, tmp);
    for (int64_t d = 0; d < dim; ++d) k[i * dim + d] = tmp[d];
    random_unit(&g, dim, tmp);
    for (int64_t d = 0; d < dim; ++d) v[i * dim + d] = tmp[d];
  }
  const double ss = sstrength > 0.0 ? sstrength : strength;
  const double vs = vstrength > 0.0 ? vstrength : strength;
  for (int64_t a = 0; a < nso; ++a) {
    const int64_t off = soffs[a];
    for (int64_t j = 0; j + off < n; ++j) {
      const int64_t i = j + off;
      const int64_t rel = use_dca ? lco_dca_relative(i, j, s, c) : off;
      lco_rope_rotate_row(carrier + i * dim, dim, rel, thetas, tmp);
      for (int64_t d = 0; d < dim; ++d) k[j * dim + d] += ss * tmp[d];
    }
  }
  for (int64_t a = 0; a < nvc; ++a)
    for (int64_t d = 0; d < dim; ++d) k[vcols[a] * dim + d] = vs * shared[d];
  free(thetas);
  free(is_shared);
  free(is_carrier);
  free(corder);
  free(shared);
  free(carrier);
  free(tmp);
  return LCO_OK;
}
