/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Linked only by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference
 * legs, always as the checker or the CPU baseline, never as the product.
 *
 * Plain-C restatement of the reference bulk sampler (`gnnbulk`, Python):
 *   - sample_epoch_bulk           pkg/src/gnnbulk/sampler.py:325-387
 *   - its_sample_row              pkg/src/gnnbulk/sampler.py:157-189
 *   - sample_rows_ordered         pkg/src/gnnbulk/sampler.py:192-207
 *   - frontier_from_rows          pkg/src/gnnbulk/sampler.py:210-222
 *   - global_row_keys             pkg/src/gnnbulk/sampler.py:309-322
 *   - SAGE extraction             pkg/src/gnnbulk/sampler.py:390-417,465-472
 *                                 (compact_columns sparse.py:345-357,
 *                                  block_diag sparse.py:321-342)
 *   - LADIES extraction           pkg/src/gnnbulk/sampler.py:420-462,475-483
 *                                 (build_column_extraction sparse.py:430-446)
 *   - norm_rows_sage/_ladies      pkg/src/gnnbulk/sparse.py:254-286
 *     (numpy add.reduceat = a[0] + pairwise(a[1:]); exact here because the
 *      sampler's row values are integers)
 * with RowRng.stream (sampler.py:112-116) replaced by the injected
 * counter-based uniform u(seed, epoch, depth, row, t) of oracle/philox.py
 * (Philox4x64-10).
 *
 * The ITS is the literal remove-and-renormalise loop: a fresh sequential
 * fp64 cumsum per draw, searchsorted(side="right"), clamp, walk back over
 * removed (zero) weights.  Pinned against the reference's own outputs in
 * tests/golden (tests/test_oracle.py).
 *
 * Parallelism (CPU baseline only): OpenMP over rows / batches; each row's
 * draws are independent because the streams are keyed per row
 * (the same property the reference relies on, sampler.py:9-11).
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- RNG -- */

static inline void mulhilo64(uint64_t a, uint64_t b, uint64_t *hi, uint64_t *lo) {
  __uint128_t p = (__uint128_t)a * b;
  *hi = (uint64_t)(p >> 64);
  *lo = (uint64_t)p;
}

void orc_philox4x64_10(const uint64_t in_ctr[4], const uint64_t in_key[2], uint64_t out[4]) {
  uint64_t c0 = in_ctr[0], c1 = in_ctr[1], c2 = in_ctr[2], c3 = in_ctr[3];
  uint64_t k0 = in_key[0], k1 = in_key[1];
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B97F4A7C15ULL;
      k1 += 0xBB67AE8584CAA73BULL;
    }
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(0xD2E7470EE14C6C93ULL, c0, &hi0, &lo0);
    mulhilo64(0xCA5A826395121157ULL, c2, &hi1, &lo1);
    uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

double orc_uniform(uint64_t seed, uint64_t epoch, uint64_t depth, uint64_t row, uint64_t t) {
  uint64_t ctr[4] = {row, depth, t >> 2, 0};
  uint64_t key[2] = {seed, epoch};
  uint64_t out[4];
  orc_philox4x64_10(ctr, key, out);
  return (double)(out[t & 3] >> 11) * 0x1.0p-53;
}

/* ----------------------------------------------------------------- ITS -- */

/* its_sample_row (sampler.py:157-189).  w is modified (drawn weights are
 * zeroed), cdf is scratch of length m.  Uniforms come from `us` when non-NULL
 * else from the keyed stream.  Returns take = min(s, m); picks in draw order. */
static int64_t its_row(double *w, double *cdf, int64_t m, int64_t s, const double *us,
                       uint64_t seed, uint64_t epoch, uint64_t depth, uint64_t key,
                       int64_t *out) {
  if (m == 0) return 0;
  int64_t take = s < m ? s : m;
  if (take == m) {
    for (int64_t i = 0; i < m; ++i) out[i] = i;
    return m;
  }
  for (int64_t t = 0; t < take; ++t) {
    double acc = 0.0;
    for (int64_t i = 0; i < m; ++i) { acc = acc + w[i]; cdf[i] = acc; }
    double total = cdf[m - 1];
    double u = us ? us[t] : orc_uniform(seed, epoch, depth, key, (uint64_t)t);
    double target = u * total;
    /* searchsorted(cdf, target, side="right"): first i with cdf[i] > target */
    int64_t lo = 0, hi = m;
    while (lo < hi) {
      int64_t mid = lo + (hi - lo) / 2;
      if (cdf[mid] > target) hi = mid; else lo = mid + 1;
    }
    int64_t idx = lo;
    if (idx >= m) idx = m - 1;
    while (w[idx] == 0.0) idx -= 1;
    out[t] = idx;
    w[idx] = 0.0;
  }
  return take;
}

/* Exposed for the its_rows golden fixture. */
int64_t orc_its_sample_row(const double *probs, int64_t m, int64_t s, const double *us,
                           int64_t *out) {
  double *w = (double *)malloc(sizeof(double) * (m ? m : 1));
  double *cdf = (double *)malloc(sizeof(double) * (m ? m : 1));
  memcpy(w, probs, sizeof(double) * m);
  int64_t r = its_row(w, cdf, m, s, us, 0, 0, 0, 0, out);
  free(w);
  free(cdf);
  return r;
}

/* numpy add.reduce order for one segment: a[0] + pairwise(a[1:]). */
static double pairwise(const double *a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res += a[i];
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise(a, n2) + pairwise(a + n2, n - n2);
}

double orc_segment_sum(const double *a, int64_t n) {
  if (n == 0) return 0.0;
  return a[0] + pairwise(a + 1, n - 1);
}

/* ------------------------------------------------------------- output -- */

typedef struct {
  int64_t n_rows, n_cols, nnz;
  int64_t *ptr;  /* n_rows + 1 */
  int32_t *col;  /* nnz */
} orc_csr;

typedef struct {
  orc_csr frontier;
  orc_csr adj;
  int64_t *rowv_off; int32_t *rowv;   /* k+1, total */
  int64_t *colv_off; int32_t *colv;
  int64_t *sampv_off; int32_t *sampv;
} orc_layer;

typedef struct {
  int64_t n_layers;
  int64_t k;
  int64_t status;     /* 0 ok; <0 contract violation */
  orc_layer *layers;
} orc_epoch;

static void csr_free(orc_csr *c) { free(c->ptr); free(c->col); }

void orc_epoch_free(orc_epoch *e) {
  if (!e) return;
  for (int64_t l = 0; l < e->n_layers; ++l) {
    orc_layer *L = &e->layers[l];
    csr_free(&L->frontier); csr_free(&L->adj);
    free(L->rowv_off); free(L->rowv); free(L->colv_off); free(L->colv);
    free(L->sampv_off); free(L->sampv);
  }
  free(e->layers);
  free(e);
}

static int cmp_i64(const void *a, const void *b) {
  int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  return (x > y) - (x < y);
}
static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

static int64_t lower_bound_i32(const int32_t *a, int64_t n, int32_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) { int64_t mid = (lo + hi) / 2; if (a[mid] < v) lo = mid + 1; else hi = mid; }
  return lo;
}

/* ---------------------------------------------------------- SAGE bulk -- */

/* sample_epoch_bulk with cfg.kind == SAGE (sampler.py:325-387). */
orc_epoch *orc_sage_bulk(int64_t n, const int64_t *rowptr, const int32_t *col,
                         int64_t k, const int64_t *bptr, const int64_t *bverts,
                         int64_t batch_size, int64_t L, const int64_t *fanouts,
                         uint64_t seed, uint64_t epoch, int64_t batch_offset,
                         int nthreads) {
  if (nthreads > 0) omp_set_num_threads(nthreads);
  orc_epoch *E = (orc_epoch *)calloc(1, sizeof(orc_epoch));
  E->k = k;
  E->layers = (orc_layer *)calloc((size_t)(L > 0 ? L : 1), sizeof(orc_layer));
  /* current rows */
  int64_t R = bptr[k];
  int32_t *v = (int32_t *)malloc(sizeof(int32_t) * (R ? R : 1));
  int64_t *brow = (int64_t *)malloc(sizeof(int64_t) * (k + 1));
  for (int64_t i = 0; i < R; ++i) {
    if (bverts[i] < 0 || bverts[i] >= n) { E->status = -1; free(v); free(brow); return E; }
    v[i] = (int32_t)bverts[i];
  }
  memcpy(brow, bptr, sizeof(int64_t) * (k + 1));
  int64_t stride = batch_size;
  for (int64_t d = 1; d <= L; ++d) {
    int64_t s = fanouts[d - 1];
    if (d > 1) stride *= fanouts[d - 2];
    orc_layer *Ly = &E->layers[d - 1];
    E->n_layers = d;
    /* global_row_keys: actual rows per batch may not exceed the stride */
    for (int64_t b = 0; b < k; ++b)
      if (brow[b + 1] - brow[b] > stride) E->status = -2;
    int64_t *cnt = (int64_t *)malloc(sizeof(int64_t) * (R + 1));
    for (int64_t r = 0; r < R; ++r) {
      int64_t deg = rowptr[v[r] + 1] - rowptr[v[r]];
      cnt[r] = deg < s ? deg : s;
    }
    int64_t *fptr = (int64_t *)malloc(sizeof(int64_t) * (R + 1));
    fptr[0] = 0;
    for (int64_t r = 0; r < R; ++r) fptr[r + 1] = fptr[r] + cnt[r];
    int64_t F = fptr[R];
    int32_t *fcol = (int32_t *)malloc(sizeof(int32_t) * (F ? F : 1));
    /* batch of each row */
    int64_t *rb = (int64_t *)malloc(sizeof(int64_t) * (R ? R : 1));
    for (int64_t b = 0; b < k; ++b)
      for (int64_t r = brow[b]; r < brow[b + 1]; ++r) rb[r] = b;
#pragma omp parallel
    {
      int64_t cap = 0;
      double *w = NULL, *cdf = NULL;
      int64_t *picks = (int64_t *)malloc(sizeof(int64_t) * (s + 1));
#pragma omp for schedule(dynamic, 64)
      for (int64_t r = 0; r < R; ++r) {
        int64_t lo = rowptr[v[r]], m = rowptr[v[r] + 1] - lo;
        if (m == 0) continue;
        if (m > cap) {
          cap = m;
          w = (double *)realloc(w, sizeof(double) * cap);
          cdf = (double *)realloc(cdf, sizeof(double) * cap);
        }
        /* norm_rows_sage: every value 1.0 divided by the row sum deg */
        double wv = 1.0 / (double)m;
        for (int64_t i = 0; i < m; ++i) w[i] = wv;
        uint64_t key = (uint64_t)((batch_offset + rb[r]) * stride + (r - brow[rb[r]]));
        int64_t take = its_row(w, cdf, m, s, NULL, seed, epoch, (uint64_t)d, key, picks);
        qsort(picks, (size_t)take, sizeof(int64_t), cmp_i64);
        for (int64_t t = 0; t < take; ++t) fcol[fptr[r] + t] = col[lo + picks[t]];
      }
      free(w); free(cdf); free(picks);
    }
    /* frontier */
    Ly->frontier.n_rows = R; Ly->frontier.n_cols = n; Ly->frontier.nnz = F;
    Ly->frontier.ptr = fptr; Ly->frontier.col = fcol;
    /* extraction: per batch sorted-unique picks, renumber, block diagonal */
    int64_t *eoff = (int64_t *)malloc(sizeof(int64_t) * (k + 1));
    for (int64_t b = 0; b <= k; ++b) eoff[b] = fptr[brow[b]];
    int32_t *uniq = (int32_t *)malloc(sizeof(int32_t) * (F ? F : 1));
    int64_t *ucnt = (int64_t *)calloc((size_t)(k + 1), sizeof(int64_t));
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < k; ++b) {
      int64_t a0 = eoff[b], a1 = eoff[b + 1];
      memcpy(uniq + a0, fcol + a0, sizeof(int32_t) * (a1 - a0));
      qsort(uniq + a0, (size_t)(a1 - a0), sizeof(int32_t), cmp_i32);
      int64_t u = 0;
      for (int64_t i = a0; i < a1; ++i)
        if (i == a0 || uniq[i] != uniq[i - 1]) uniq[a0 + u++] = uniq[i];
      ucnt[b] = u;
    }
    int64_t *coff = (int64_t *)malloc(sizeof(int64_t) * (k + 1));
    coff[0] = 0;
    for (int64_t b = 0; b < k; ++b) coff[b + 1] = coff[b] + ucnt[b];
    int32_t *colv = (int32_t *)malloc(sizeof(int32_t) * (coff[k] ? coff[k] : 1));
    int32_t *acol = (int32_t *)malloc(sizeof(int32_t) * (F ? F : 1));
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < k; ++b) {
      int64_t a0 = eoff[b], a1 = eoff[b + 1];
      memcpy(colv + coff[b], uniq + a0, sizeof(int32_t) * ucnt[b]);
      for (int64_t i = a0; i < a1; ++i)
        acol[i] = (int32_t)(coff[b] + lower_bound_i32(uniq + a0, ucnt[b], fcol[i]));
    }
    Ly->adj.n_rows = R; Ly->adj.n_cols = coff[k]; Ly->adj.nnz = F;
    Ly->adj.ptr = (int64_t *)malloc(sizeof(int64_t) * (R + 1));
    memcpy(Ly->adj.ptr, fptr, sizeof(int64_t) * (R + 1));
    Ly->adj.col = acol;
    Ly->rowv_off = brow; Ly->rowv = v;
    Ly->colv_off = coff; Ly->colv = colv;
    Ly->sampv_off = eoff;
    Ly->sampv = (int32_t *)malloc(sizeof(int32_t) * (F ? F : 1));
    memcpy(Ly->sampv, fcol, sizeof(int32_t) * F);
    /* next seed: one one-hot row per pick (expand_row_extraction) */
    int32_t *nv = (int32_t *)malloc(sizeof(int32_t) * (F ? F : 1));
    memcpy(nv, fcol, sizeof(int32_t) * F);
    int64_t *nbrow = (int64_t *)malloc(sizeof(int64_t) * (k + 1));
    memcpy(nbrow, eoff, sizeof(int64_t) * (k + 1));
    v = nv; brow = nbrow; R = F;
    free(cnt); free(rb); free(uniq); free(ucnt);
  }
  free(v); free(brow);
  return E;
}

/* -------------------------------------------------------- LADIES bulk -- */

/* sample_epoch_bulk with cfg.kind == LADIES (sampler.py:325-387,475-483). */
orc_epoch *orc_ladies_bulk(int64_t n, const int64_t *rowptr, const int32_t *col,
                           int64_t k, const int64_t *bptr, const int64_t *bverts,
                           int64_t L, const int64_t *fanouts, uint64_t seed,
                           uint64_t epoch, int64_t batch_offset, int nthreads) {
  if (nthreads > 0) omp_set_num_threads(nthreads);
  orc_epoch *E = (orc_epoch *)calloc(1, sizeof(orc_epoch));
  E->k = k;
  E->layers = (orc_layer *)calloc((size_t)(L > 0 ? L : 1), sizeof(orc_layer));
  /* Q: per batch sorted distinct vertex lists (ladies_seed_matrix) */
  int64_t *qoff = (int64_t *)malloc(sizeof(int64_t) * (k + 1));
  memcpy(qoff, bptr, sizeof(int64_t) * (k + 1));
  int64_t QN = bptr[k];
  int32_t *q = (int32_t *)malloc(sizeof(int32_t) * (QN ? QN : 1));
  for (int64_t i = 0; i < QN; ++i) {
    if (bverts[i] < 0 || bverts[i] >= n) { E->status = -1; free(q); free(qoff); return E; }
    q[i] = (int32_t)bverts[i];
  }
  for (int64_t b = 0; b < k; ++b) {
    qsort(q + qoff[b], (size_t)(qoff[b + 1] - qoff[b]), sizeof(int32_t), cmp_i32);
    for (int64_t i = qoff[b] + 1; i < qoff[b + 1]; ++i)
      if (q[i] == q[i - 1]) { E->status = -3; free(q); free(qoff); return E; }
  }
  for (int64_t d = 1; d <= L; ++d) {
    int64_t s = fanouts[d - 1];
    orc_layer *Ly = &E->layers[d - 1];
    E->n_layers = d;
    int32_t **S = (int32_t **)calloc((size_t)(k ? k : 1), sizeof(int32_t *));
    int64_t *take = (int64_t *)calloc((size_t)(k ? k : 1), sizeof(int64_t));
#pragma omp parallel
    {
      int32_t *cnt = (int32_t *)calloc((size_t)n, sizeof(int32_t));
#pragma omp for schedule(dynamic, 1)
      for (int64_t b = 0; b < k; ++b) {
        /* P row b = sum of A rows of Q_b: neighbour counts e_v (spgemm) */
        int64_t cap = 1024, N = 0;
        int32_t *touched = (int32_t *)malloc(sizeof(int32_t) * cap);
        for (int64_t i = qoff[b]; i < qoff[b + 1]; ++i) {
          int32_t u = q[i];
          for (int64_t e = rowptr[u]; e < rowptr[u + 1]; ++e) {
            int32_t x = col[e];
            if (cnt[x]++ == 0) {
              if (N == cap) { cap *= 2; touched = (int32_t *)realloc(touched, sizeof(int32_t) * cap); }
              touched[N++] = x;
            }
          }
        }
        qsort(touched, (size_t)N, sizeof(int32_t), cmp_i32);
        double *vals = (double *)malloc(sizeof(double) * (N ? N : 1));
        for (int64_t i = 0; i < N; ++i) {
          double e = (double)cnt[touched[i]];
          vals[i] = e * e;
          cnt[touched[i]] = 0;
        }
        /* norm_rows_ladies: e^2 / (a[0] + pairwise(a[1:])) */
        double sum = orc_segment_sum(vals, N);
        for (int64_t i = 0; i < N; ++i) vals[i] = vals[i] / sum;
        double *cdf = (double *)malloc(sizeof(double) * (N ? N : 1));
        int64_t *picks = (int64_t *)malloc(sizeof(int64_t) * (s + 1));
        int64_t tk = its_row(vals, cdf, N, s, NULL, seed, epoch, (uint64_t)d,
                             (uint64_t)(batch_offset + b), picks);
        qsort(picks, (size_t)tk, sizeof(int64_t), cmp_i64);
        S[b] = (int32_t *)malloc(sizeof(int32_t) * (tk ? tk : 1));
        for (int64_t t = 0; t < tk; ++t) S[b][t] = touched[picks[t]];
        take[b] = tk;
        free(touched); free(vals); free(cdf); free(picks);
      }
      free(cnt);
    }
    /* frontier: k rows, sorted picks */
    int64_t *fptr = (int64_t *)malloc(sizeof(int64_t) * (k + 1));
    fptr[0] = 0;
    for (int64_t b = 0; b < k; ++b) fptr[b + 1] = fptr[b] + take[b];
    int64_t F = fptr[k];
    int32_t *fcol = (int32_t *)malloc(sizeof(int32_t) * (F ? F : 1));
    for (int64_t b = 0; b < k; ++b) memcpy(fcol + fptr[b], S[b], sizeof(int32_t) * take[b]);
    Ly->frontier.n_rows = k; Ly->frontier.n_cols = n; Ly->frontier.nnz = F;
    Ly->frontier.ptr = fptr; Ly->frontier.col = fcol;
    /* ladies_assemble: shared layout iff every batch has the same width */
    int shared = 1;
    for (int64_t b = 1; b < k; ++b) if (take[b] != take[0]) shared = 0;
    int64_t *coloff = (int64_t *)malloc(sizeof(int64_t) * (k + 1));
    coloff[0] = 0;
    for (int64_t b = 0; b < k; ++b) coloff[b + 1] = coloff[b] + (shared ? 0 : take[b]);
    /* A_S rows: one per Q nonzero, in Q order; entries = ranks of A[u,:] ∩ S_b */
    int64_t AR = qoff[k];
    int64_t *aptr = (int64_t *)malloc(sizeof(int64_t) * (AR + 1));
    int64_t *rcnt = (int64_t *)calloc((size_t)(AR + 1), sizeof(int64_t));
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < k; ++b)
      for (int64_t i = qoff[b]; i < qoff[b + 1]; ++i) {
        int32_t u = q[i];
        int64_t c = 0;
        for (int64_t e = rowptr[u]; e < rowptr[u + 1]; ++e) {
          int64_t pos = lower_bound_i32(S[b], take[b], col[e]);
          if (pos < take[b] && S[b][pos] == col[e]) ++c;
        }
        rcnt[i] = c;
      }
    aptr[0] = 0;
    for (int64_t i = 0; i < AR; ++i) aptr[i + 1] = aptr[i] + rcnt[i];
    int32_t *acol = (int32_t *)malloc(sizeof(int32_t) * (aptr[AR] ? aptr[AR] : 1));
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < k; ++b)
      for (int64_t i = qoff[b]; i < qoff[b + 1]; ++i) {
        int32_t u = q[i];
        int64_t o = aptr[i];
        for (int64_t e = rowptr[u]; e < rowptr[u + 1]; ++e) {
          int64_t pos = lower_bound_i32(S[b], take[b], col[e]);
          if (pos < take[b] && S[b][pos] == col[e]) acol[o++] = (int32_t)(coloff[b] + pos);
        }
      }
    Ly->adj.n_rows = AR;
    Ly->adj.n_cols = k == 0 ? 0 : (shared ? take[0] : coloff[k]);
    Ly->adj.nnz = aptr[AR];
    Ly->adj.ptr = aptr; Ly->adj.col = acol;
    Ly->rowv_off = qoff; Ly->rowv = q;
    Ly->colv_off = (int64_t *)malloc(sizeof(int64_t) * (k + 1));
    memcpy(Ly->colv_off, fptr, sizeof(int64_t) * (k + 1));
    Ly->colv = (int32_t *)malloc(sizeof(int32_t) * (F ? F : 1));
    memcpy(Ly->colv, fcol, sizeof(int32_t) * F);
    Ly->sampv_off = (int64_t *)malloc(sizeof(int64_t) * (k + 1));
    memcpy(Ly->sampv_off, fptr, sizeof(int64_t) * (k + 1));
    Ly->sampv = (int32_t *)malloc(sizeof(int32_t) * (F ? F : 1));
    memcpy(Ly->sampv, fcol, sizeof(int32_t) * F);
    /* next Q = frontier */
    int64_t *nqoff = (int64_t *)malloc(sizeof(int64_t) * (k + 1));
    memcpy(nqoff, fptr, sizeof(int64_t) * (k + 1));
    int32_t *nq = (int32_t *)malloc(sizeof(int32_t) * (F ? F : 1));
    memcpy(nq, fcol, sizeof(int32_t) * F);
    qoff = nqoff; q = nq;
    for (int64_t b = 0; b < k; ++b) free(S[b]);
    free(S); free(take); free(coloff); free(rcnt);
  }
  free(q); free(qoff);
  return E;
}
