// Synthetic OGB-shaped graphs on the device (SURVEY.md §8(d) inputs, §8(f)4),
// the canonical recipe of SURVEY.md Appendix B with counter-based draws:
//   candidates  Graph500 R-MAT (a, b, c) over scale = ceil(log2 n) levels,
//               Philox4x64-10 keyed by the draw index (deterministic on every
//               device); ids >= n and self loops rejected; undirected pairs
//               canonicalised to (min, max) for symmetric shapes
//   selection   the first m distinct pairs in draw order: stable radix sort
//               of (pair, draw index), run starts mark their first draw, a
//               scan over draw order ranks them
//   relabel     vertex v -> rank of its keyed 63-bit hash (ties by v)
//   CSR         (label u, label v) (+ reverse when symmetric) through the
//               device COO -> CSR builder (gb_csr.cu)
// oracle/csrc/gen.c builds the identical graph on the host.
#include "gb_common.cuh"
#include "gb_internal.h"
#include "gb_scan.cuh"

namespace gb {

// Candidate e: for each of `scale` levels draw u and pick a quadrant with
// probabilities (a, b, c, 1-a-b-c); bit l of (src, dst) is set for the
// lower/right halves.  false for rejected candidates (self loop, id >= n).
// oracle/csrc/gen.c restates it for the host.
__device__ __forceinline__ bool rmat_pair(uint64_t seed, int32_t scale, int64_t n, uint64_t e,
                                          double a, double b, double c, int64_t& u, int64_t& v) {
  u = 0;
  v = 0;
  for (int lvl = 0; lvl < scale; lvl += 4) {
    uint64_t c0 = e, c1 = 0x524d4154ULL /* "RMAT" */, c2 = (uint64_t)lvl, c3 = 0;
    philox4x64_10(c0, c1, c2, c3, seed, 0x67656e6572617465ULL);
    const uint64_t w[4] = {c0, c1, c2, c3};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (lvl + q >= scale) break;
      const double r = (double)(w[q] >> 11) * 0x1.0p-53;
      const int64_t bu = r >= a + b ? 1 : 0;
      const int64_t bv = ((r >= a && r < a + b) || r >= a + b + c) ? 1 : 0;
      u |= bu << (lvl + q);
      v |= bv << (lvl + q);
    }
  }
  return !(u == v || u >= n || v >= n);
}

__global__ void k_rmat(uint64_t seed, int32_t scale, int64_t n, int64_t first, int64_t count,
                       double a, double b, double c, int64_t* __restrict__ src,
                       int64_t* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t u, v;
    const bool ok = rmat_pair(seed, scale, n, (uint64_t)(first + i), a, b, c, u, v);
    src[i] = ok ? u : -1;
    dst[i] = ok ? v : -1;
  }
}

__device__ __forceinline__ uint64_t hash63(uint64_t seed, uint64_t x) {
  uint64_t c0 = x, c1 = 0x68617368ULL, c2 = 0, c3 = 0;
  philox4x64_10(c0, c1, c2, c3, seed, 0x72656c6162656cULL);
  return c0 >> 1;
}

__global__ void k_hash64(uint64_t seed, const int64_t* __restrict__ x, int64_t count,
                         int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    out[i] = (int64_t)hash63(seed, (uint64_t)x[i]);  // non-negative sort key
  }
}

// ------------------------------------------------------- full generator

__global__ void k_relabel_keys(uint64_t seed, int64_t n, int sb, uint64_t* __restrict__ keys) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    keys[v] = ((hash63(seed, (uint64_t)v) >> sb) << sb) | (uint64_t)v;
}

__global__ void k_relabel_table(const uint64_t* __restrict__ sorted, int64_t n, int sb,
                                int32_t* __restrict__ label) {
  const uint64_t mask = (1ull << sb) - 1ull;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    label[sorted[i] & mask] = (int32_t)i;
}

// pair key (lo << sb | hi, or src << sb | dst when directed), all ones for a
// rejected candidate (sorts last on the low 2 sb bits), payload = draw index
__global__ void k_rmat_keys(uint64_t seed, int32_t scale, int64_t n, int64_t C, double a,
                            double b, double c, int32_t symmetric, int sb,
                            uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < C;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t u, v;
    const bool ok = rmat_pair(seed, scale, n, (uint64_t)i, a, b, c, u, v);
    if (ok && symmetric && u > v) { const int64_t t = u; u = v; v = t; }
    keys[i] = ok ? ((uint64_t)u << sb) | (uint64_t)v : ~0ull;
    vals[i] = (uint32_t)i;
  }
}

// run starts of the sorted candidates mark their pair's first draw
__global__ void k_mark_first(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                             int64_t C, uint64_t end, uint8_t* __restrict__ mark) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < C;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t x = keys[i];
    if (x < end && (i == 0 || x != keys[i - 1])) mark[vals[i]] = 1;
  }
}

__global__ void k_csr_set_i64(int64_t* p, int64_t v) { *p = v; }

struct MarkF {
  const uint8_t* mark;
  __device__ int64_t operator()(int64_t i) const { return mark[i]; }
};

// the first m distinct pairs in draw order, relabelled, as CSR keys (and
// their reverses at [m, 2m) when symmetric)
// Block mode (row_hi > row_lo): an edge whose relabelled source lies outside
// [row_lo, row_hi) becomes ~0 (dropped by the CSR build), kept sources are
// shifted to block-local rows; *kept counts the block's edges.
__global__ void k_emit_pairs(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                             int64_t C, uint64_t end, const uint32_t* __restrict__ rank,
                             int64_t m, int sb, const int32_t* __restrict__ label,
                             int32_t symmetric, int64_t row_lo, int64_t row_hi,
                             uint64_t* __restrict__ out, unsigned long long* __restrict__ kept) {
  const uint64_t mask = (1ull << sb) - 1ull;
  const bool block = row_hi > row_lo;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < C;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t x = keys[i];
    if (x >= end || (i > 0 && x == keys[i - 1])) continue;
    const int64_t r = rank[vals[i]];
    if (r >= m) continue;
    const int64_t lu = label[x >> sb], lv = label[x & mask];
    if (!block) {
      out[r] = ((uint64_t)lu << sb) | (uint64_t)lv;
      if (symmetric) out[m + r] = ((uint64_t)lv << sb) | (uint64_t)lu;
      continue;
    }
    int nk = 0;
    const bool ku = lu >= row_lo && lu < row_hi;
    out[r] = ku ? ((uint64_t)(lu - row_lo) << sb) | (uint64_t)lv : ~0ull;
    nk += ku;
    if (symmetric) {
      const bool kv = lv >= row_lo && lv < row_hi;
      out[m + r] = kv ? ((uint64_t)(lv - row_lo) << sb) | (uint64_t)lu : ~0ull;
      nk += kv;
    }
    if (nk) atomicAdd(kept, (unsigned long long)nk);
  }
}

static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

struct GenLayout {
  size_t label, keysB, keysA, altA, valsA, valtA, mark, rank, scanws, tail, bytes;
};

static GenLayout gen_layout(int64_t n, int64_t m, int32_t symmetric, int64_t C) {
  GenLayout L{};
  const int64_t E = symmetric ? 2 * m : m;
  size_t off = 0;
  L.label = off; off += al256(sizeof(int32_t) * (n + 1));
  L.keysB = off; off += al256(sizeof(uint64_t) * (E + 1));
  const size_t uni = off;
  // phase A (candidates) — the relabel sort and the CSR build reuse it
  L.keysA = off; off += al256(sizeof(uint64_t) * (C + 1));
  L.altA = off; off += al256(sizeof(uint64_t) * (C + 1));
  L.valsA = off; off += al256(sizeof(uint32_t) * (C + 1));
  L.valtA = off; off += al256(sizeof(uint32_t) * (C + 1));
  L.mark = off; off += al256(C + 1);
  L.rank = off; off += al256(sizeof(uint32_t) * (C + 2));
  L.scanws = off; off += al256(sizeof(int64_t) * scan_workspace_elems<int64_t>(C + 1));
  L.tail = off; off += al256(radix_sort_ws(C > n ? C : n)) + 256;
  size_t need = off;
  const size_t relabel = uni + 2 * al256(sizeof(uint64_t) * (n + 1)) + al256(radix_sort_ws(n));
  const size_t csr = uni + csr_from_keys_ws(n, E);
  if (relabel > need) need = relabel;
  if (csr > need) need = csr;
  L.bytes = need;
  return L;
}

}  // namespace gb

using namespace gb;

extern "C" {

int gb_rmat_edges(uint64_t seed, int32_t scale, int64_t n, int64_t first, int64_t count, double a,
                  double b, double c, int64_t* d_src, int64_t* d_dst, void* stream) {
  if (scale < 1 || scale > 40 || count < 0 || a < 0 || b < 0 || c < 0 || a + b + c > 1.0) {
    set_error("rmat: bad parameters");
    return GB_ERR_CONTRACT;
  }
  if (count == 0) return GB_OK;
  int64_t g = (count + 255) / 256;
  if (g > 32 * kNumSMs) g = 32 * kNumSMs;
  k_rmat<<<(int)g, 256, 0, (cudaStream_t)stream>>>(seed, scale, n, first, count, a, b, c, d_src,
                                                   d_dst);
  GB_LAUNCH_CHECK("k_rmat");
  return GB_OK;
}

int gb_hash64(uint64_t seed, const int64_t* d_x, int64_t count, int64_t* d_out, void* stream) {
  if (count < 0) { set_error("hash64: count < 0"); return GB_ERR_CONTRACT; }
  if (count == 0) return GB_OK;
  int64_t g = (count + 255) / 256;
  if (g > 32 * kNumSMs) g = 32 * kNumSMs;
  k_hash64<<<(int)g, 256, 0, (cudaStream_t)stream>>>(seed, d_x, count, d_out);
  GB_LAUNCH_CHECK("k_hash64");
  return GB_OK;
}

size_t gb_rmat_graph_workspace(int64_t n, int64_t m, int32_t symmetric, int64_t candidates) {
  if (n < 2 || m < 0 || candidates < 0) return 0;
  return gen_layout(n, m, symmetric, candidates).bytes;
}

static int rmat_graph(uint64_t seed, int64_t n, int64_t m, int32_t symmetric, double a, double b,
                      double c, int64_t candidates, int64_t row_lo, int64_t row_hi,
                      int64_t* d_rowptr, int32_t* d_col, int64_t col_cap, int64_t* h_info,
                      void* d_ws, size_t ws_bytes, void* stream) {
  const int64_t E = symmetric ? 2 * m : m;
  const bool block = row_hi > row_lo;
  if (block && (row_lo < 0 || row_hi > n)) {
    set_error("rmat block: rows [%lld, %lld) outside [0, n)", (long long)row_lo,
              (long long)row_hi);
    return GB_ERR_CONTRACT;
  }
  if (n < 2 || n >= ((int64_t)1 << 31) || m < 0 || candidates < 0 ||
      candidates >= ((int64_t)1 << 32) || a < 0 || b < 0 || c < 0 || a + b + c > 1.0 ||
      !d_rowptr || !d_col || !h_info || (!block && col_cap < E + GB_COL_PAD)) {
    set_error("rmat graph: bad arguments");
    return GB_ERR_CONTRACT;
  }
  const GenLayout L = gen_layout(n, m, symmetric, candidates);
  if (L.bytes > ws_bytes) {
    set_error("rmat graph: workspace too small (%zu < %zu)", ws_bytes, L.bytes);
    return GB_ERR_CAPACITY;
  }
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)d_ws;
  int32_t* label = (int32_t*)(w + L.label);
  uint64_t* keysB = (uint64_t*)(w + L.keysB);
  const int sb = bits_for(n);
  int scale = 1;
  while (((int64_t)1 << scale) < n) ++scale;
  const uint64_t end = ((uint64_t)1 << (2 * sb)) - 1ull;
  auto grid = [](int64_t x) {
    const int64_t g = (x + 255) / 256;
    return (int)(g < 1 ? 1 : (g > 64 * kNumSMs ? 64 * kNumSMs : g));
  };
  // relabel table: label[v] = rank of (hash, v)
  {
    uint64_t* rk = (uint64_t*)(w + L.keysA);
    uint64_t* ra = rk + (n + 1);
    ra = (uint64_t*)(((uintptr_t)ra + 255) & ~(uintptr_t)255);
    char* rws = (char*)(((uintptr_t)(ra + n + 1) + 255) & ~(uintptr_t)255);
    k_relabel_keys<<<grid(n), 256, 0, st>>>(seed + 2, n, sb, rk);
    bool in_alt = false;
    int rc = radix_sort(rk, ra, nullptr, nullptr, n, 64, rws, radix_sort_ws(n), &in_alt, st);
    if (rc) return rc;
    k_relabel_table<<<grid(n), 256, 0, st>>>(in_alt ? ra : rk, n, sb, label);
    GB_LAUNCH_CHECK("relabel");
    count_launches(2);
  }
  // candidates, first m distinct pairs in draw order
  uint64_t* keysA = (uint64_t*)(w + L.keysA);
  uint64_t* altA = (uint64_t*)(w + L.altA);
  uint32_t* valsA = (uint32_t*)(w + L.valsA);
  uint32_t* valtA = (uint32_t*)(w + L.valtA);
  uint8_t* mark = (uint8_t*)(w + L.mark);
  uint32_t* rank = (uint32_t*)(w + L.rank);
  int64_t* scan_ws = (int64_t*)(w + L.scanws);
  int64_t* scal = (int64_t*)(w + L.tail);
  char* rws = w + L.tail + 256;
  const int64_t C = candidates;
  k_rmat_keys<<<grid(C), 256, 0, st>>>(seed, scale, n, C, a, b, c, symmetric, sb, keysA, valsA);
  GB_LAUNCH_CHECK("k_rmat_keys");
  bool in_alt = false;
  int rc = radix_sort(keysA, altA, valsA, valtA, C, 2 * sb, rws, radix_sort_ws(C > n ? C : n),
                      &in_alt, st);
  if (rc) return rc;
  const uint64_t* sk = in_alt ? altA : keysA;
  const uint32_t* sv = in_alt ? valtA : valsA;
  GB_CUDA(cudaMemsetAsync(mark, 0, C + 1, st));
  k_mark_first<<<grid(C), 256, 0, st>>>(sk, sv, C, end, mark);
  k_csr_set_i64<<<1, 1, 0, st>>>(scal, C);
  rc = device_exclusive_scan<int64_t>(scal, C, MarkF{mark}, rank, scan_ws, st);
  if (rc) return rc;
  uint32_t U = 0;
  GB_CUDA(cudaMemcpyAsync(&U, rank + C, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  GB_CUDA(cudaStreamSynchronize(st));
  h_info[0] = 0;
  h_info[1] = (int64_t)U;
  if ((int64_t)U < m) {
    set_error("rmat graph: %lld candidates gave %lld distinct pairs < m = %lld",
              (long long)C, (long long)U, (long long)m);
    return GB_ERR_CAPACITY;
  }
  unsigned long long* kept = (unsigned long long*)(scal + 1);
  GB_CUDA(cudaMemsetAsync(kept, 0, sizeof(unsigned long long), st));
  k_emit_pairs<<<grid(C), 256, 0, st>>>(sk, sv, C, end, rank, m, sb, label, symmetric, row_lo,
                                        row_hi, keysB, kept);
  GB_LAUNCH_CHECK("k_emit_pairs");
  count_launches(4);
  if (block) {
    unsigned long long h_kept = 0;
    GB_CUDA(cudaMemcpyAsync(&h_kept, kept, sizeof(h_kept), cudaMemcpyDeviceToHost, st));
    GB_CUDA(cudaStreamSynchronize(st));
    if ((int64_t)h_kept + GB_COL_PAD > col_cap) {
      h_info[0] = (int64_t)h_kept;
      set_error("rmat block: %lld edges need col_cap >= %lld", (long long)h_kept,
                (long long)h_kept + GB_COL_PAD);
      return GB_ERR_CAPACITY;
    }
  }
  int64_t* d_nnz = nullptr;
  rc = csr_from_keys(keysB, E, ~0ull, sb, block ? row_hi - row_lo : n, d_rowptr, d_col, &d_nnz,
                     w + L.keysA, ws_bytes - L.keysA, st);
  if (rc) return rc;
  int64_t nnz = 0;
  GB_CUDA(cudaMemcpyAsync(&nnz, d_nnz, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GB_CUDA(cudaStreamSynchronize(st));
  GB_CUDA(cudaMemsetAsync(d_col + nnz, 0, sizeof(int32_t) * GB_COL_PAD, st));
  GB_CUDA(cudaStreamSynchronize(st));
  h_info[0] = nnz;
  return GB_OK;
}

int gb_rmat_graph(uint64_t seed, int64_t n, int64_t m, int32_t symmetric, double a, double b,
                  double c, int64_t candidates, int64_t* d_rowptr, int32_t* d_col,
                  int64_t col_cap, int64_t* h_info, void* d_ws, size_t ws_bytes, void* stream) {
  return rmat_graph(seed, n, m, symmetric, a, b, c, candidates, 0, 0, d_rowptr, d_col, col_cap,
                    h_info, d_ws, ws_bytes, stream);
}

int gb_rmat_block(uint64_t seed, int64_t n, int64_t m, int32_t symmetric, double a, double b,
                  double c, int64_t candidates, int64_t row_lo, int64_t row_hi,
                  int64_t* d_rowptr, int32_t* d_col, int64_t col_cap, int64_t* h_info,
                  void* d_ws, size_t ws_bytes, void* stream) {
  if (row_hi <= row_lo) {
    set_error("rmat block: empty row range");
    return GB_ERR_CONTRACT;
  }
  return rmat_graph(seed, n, m, symmetric, a, b, c, candidates, row_lo, row_hi, d_rowptr, d_col,
                    col_cap, h_info, d_ws, ws_bytes, stream);
}

}  // extern "C"
