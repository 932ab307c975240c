/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.c).  Host restatement of the
 * synthetic-graph recipe of SURVEY.md Appendix B as the library builds it on
 * the device (paper_2311_02909_b200/csrc/gb_graphgen.cu, gb_rmat_graph), and
 * of the reference's Graph.from_edges (pkg/src/gnnbulk/sparse.py:82-103,
 * 211-216: sorted CSR, duplicates collapsed).  Used to check the device
 * ingestion bit for bit and to give bench.py's reference arm its input
 * graph without loading the product library.
 *
 *   candidates  draw e = 0, 1, 2, ...: Graph500 R-MAT quadrants over
 *               scale = ceil(log2 n) levels from Philox4x64-10 keyed by e
 *               (4 levels per block), ids >= n and self loops rejected,
 *               (min, max) when symmetric
 *   selection   the first m distinct pairs in draw order (hash set)
 *   relabel     v -> rank of ((hash63(v) >> sb) << sb | v)
 *   CSR         (label u, label v) [+ reverse], rows sorted
 */
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

void orc_philox4x64_10(const uint64_t in_ctr[4], const uint64_t in_key[2], uint64_t out[4]);

static int gen_bits(int64_t n) {
  int b = 1;
  while (b < 62 && ((int64_t)1 << b) < n) ++b;
  return b;
}

static int rmat_pair(uint64_t seed, int scale, int64_t n, uint64_t e, double a, double b,
                     double c, int64_t *u, int64_t *v) {
  int64_t x = 0, y = 0;
  for (int lvl = 0; lvl < scale; lvl += 4) {
    const uint64_t ctr[4] = {e, 0x524d4154ULL, (uint64_t)lvl, 0};
    const uint64_t key[2] = {seed, 0x67656e6572617465ULL};
    uint64_t w[4];
    orc_philox4x64_10(ctr, key, w);
    for (int q = 0; q < 4 && lvl + q < scale; ++q) {
      const double r = (double)(w[q] >> 11) * 0x1.0p-53;
      const int64_t bu = r >= a + b ? 1 : 0;
      const int64_t bv = ((r >= a && r < a + b) || r >= a + b + c) ? 1 : 0;
      x |= bu << (lvl + q);
      y |= bv << (lvl + q);
    }
  }
  *u = x;
  *v = y;
  return !(x == y || x >= n || y >= n);
}

static uint64_t hash63(uint64_t seed, uint64_t x) {
  const uint64_t ctr[4] = {x, 0x68617368ULL, 0, 0};
  const uint64_t key[2] = {seed, 0x72656c6162656cULL};
  uint64_t w[4];
  orc_philox4x64_10(ctr, key, w);
  return w[0] >> 1;
}

static int cmp_u64(const void *a, const void *b) {
  const uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
  return x < y ? -1 : x > y;
}

static int cmp_i32(const void *a, const void *b) {
  const int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return x < y ? -1 : x > y;
}

static uint64_t mix(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  return x;
}

/* Returns nnz (>= 0) and malloc'd *rowptr (n + 1) / *col (nnz); -1 on
 * allocation failure.  orc_free releases them. */
int64_t orc_rmat_graph(uint64_t seed, int64_t n, int64_t m, int symmetric, double a, double b,
                       double c, int64_t **rowptr_out, int32_t **col_out) {
  const int sb = gen_bits(n);
  int scale = 1;
  while (((int64_t)1 << scale) < n) ++scale;
  /* selection: open-addressing set of pair keys, filled in draw order */
  uint64_t cap = 1;
  while (cap < (uint64_t)(2 * m + 16)) cap <<= 1;
  uint64_t *set = (uint64_t *)malloc(sizeof(uint64_t) * cap);
  uint64_t *pairs = (uint64_t *)malloc(sizeof(uint64_t) * (m > 0 ? m : 1));
  if (!set || !pairs) { free(set); free(pairs); return -1; }
  memset(set, 0xff, sizeof(uint64_t) * cap);
  const int64_t blk = 1 << 20;
  uint64_t *cand = (uint64_t *)malloc(sizeof(uint64_t) * blk);
  if (!cand) { free(set); free(pairs); return -1; }
  int64_t found = 0;
  for (uint64_t e0 = 0; found < m; e0 += blk) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < blk; ++i) {
      int64_t u, v;
      if (rmat_pair(seed, scale, n, e0 + i, a, b, c, &u, &v)) {
        if (symmetric && u > v) { const int64_t t = u; u = v; v = t; }
        cand[i] = ((uint64_t)u << sb) | (uint64_t)v;
      } else {
        cand[i] = ~0ull;
      }
    }
    for (int64_t i = 0; i < blk && found < m; ++i) {
      const uint64_t k = cand[i];
      if (k == ~0ull) continue;
      uint64_t h = mix(k) & (cap - 1);
      while (set[h] != ~0ull && set[h] != k) h = (h + 1) & (cap - 1);
      if (set[h] == k) continue;
      set[h] = k;
      pairs[found++] = k;
    }
  }
  free(cand);
  free(set);
  /* relabel by hash rank */
  uint64_t *rk = (uint64_t *)malloc(sizeof(uint64_t) * n);
  int32_t *label = (int32_t *)malloc(sizeof(int32_t) * n);
  if (!rk || !label) { free(rk); free(label); free(pairs); return -1; }
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; ++v) rk[v] = ((hash63(seed + 2, (uint64_t)v) >> sb) << sb) | (uint64_t)v;
  qsort(rk, (size_t)n, sizeof(uint64_t), cmp_u64);
  const uint64_t mask = (1ull << sb) - 1ull;
  for (int64_t i = 0; i < n; ++i) label[rk[i] & mask] = (int32_t)i;
  free(rk);
  /* CSR: counting sort by source, rows sorted, duplicates collapsed */
  const int64_t E = symmetric ? 2 * m : m;
  int64_t *rowptr = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  int32_t *col = (int32_t *)malloc(sizeof(int32_t) * (E > 0 ? E : 1));
  int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
  if (!rowptr || !col || !cur) { free(rowptr); free(col); free(cur); free(label); free(pairs); return -1; }
  for (int64_t i = 0; i < m; ++i) {
    rowptr[label[pairs[i] >> sb] + 1]++;
    if (symmetric) rowptr[label[pairs[i] & mask] + 1]++;
  }
  for (int64_t v = 0; v < n; ++v) rowptr[v + 1] += rowptr[v];
  memcpy(cur, rowptr, sizeof(int64_t) * (n + 1));
  for (int64_t i = 0; i < m; ++i) {
    const int32_t lu = label[pairs[i] >> sb], lv = label[pairs[i] & mask];
    col[cur[lu]++] = lv;
    if (symmetric) col[cur[lv]++] = lu;
  }
  free(pairs);
  free(label);
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t v = 0; v < n; ++v)
    qsort(col + rowptr[v], (size_t)(rowptr[v + 1] - rowptr[v]), sizeof(int32_t), cmp_i32);
  /* compact duplicates (none for distinct pairs; kept for the contract) */
  int64_t o = 0;
  for (int64_t v = 0; v < n; ++v) {
    const int64_t a0 = rowptr[v], a1 = rowptr[v + 1];
    rowptr[v] = o;
    for (int64_t e = a0; e < a1; ++e)
      if (e == a0 || col[e] != col[e - 1]) col[o++] = col[e];
  }
  rowptr[n] = o;
  free(cur);
  *rowptr_out = rowptr;
  *col_out = col;
  return o;
}

void orc_free(void *p) { free(p); }
