// Graph ingestion on the device (SURVEY.md §8(b) gb_csr_from_edges, §8(f)4):
// COO edge list -> canonical CSR with duplicates collapsed, i.e. reference
// Graph.from_edges = SparseMatrix.from_coo(..., dedup="first")
// (pkg/src/gnnbulk/sparse.py:82-103, 211-216) on 0/1 values.
//
//   pack     key = src << sb | dst (sb = bits of n - 1), range check
//   sort     stable LSD radix sort of the keys, 8-bit digits, only the
//            2 sb bits that vary: per pass a tile histogram (digit-major
//            counts), one exclusive scan, and a scatter where each warp
//            ranks its 512 keys in order with __match_any_sync and per-warp
//            digit counters in shared memory (stable: warp, item, lane
//            order = input order), optional 32-bit payload carried along
//   unique   run starts of the sorted keys, exclusive scan -> positions
//   emit     col[pos] = dst; rowptr filled over each gap of source ids
//            (long gaps by a CTA each)
// HBM-bound integer work (24 B per key per pass): no tensor cores.
#include "gb_common.cuh"
#include "gb_internal.h"
#include "gb_scan.cuh"

namespace gb {

constexpr int kRsThreads = 256;
constexpr int kRsItems = 16;
constexpr int kRsWarps = kRsThreads / 32;
constexpr int kRsWarpTile = 32 * kRsItems;           // 512 keys per warp
constexpr int64_t kRsTile = kRsThreads * kRsItems;   // 4096 keys per CTA
constexpr int kRsBins = 256;

__global__ void __launch_bounds__(kRsThreads) k_rs_hist(const uint64_t* __restrict__ keys,
                                                       int64_t m, int shift, int64_t nb,
                                                       uint32_t* __restrict__ counts) {
  __shared__ uint32_t h[kRsBins];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int lane = lane_id(), w = threadIdx.x >> 5;
  const int64_t base = (int64_t)blockIdx.x * kRsTile + w * kRsWarpTile + lane;
  uint32_t d[kRsItems];
#pragma unroll
  for (int j = 0; j < kRsItems; ++j) {
    const int64_t i = base + 32 * j;
    d[j] = i < m ? (uint32_t)(__ldg(keys + i) >> shift) & 255u : 0x100u;
  }
#pragma unroll
  for (int j = 0; j < kRsItems; ++j) {
    const unsigned peers = __match_any_sync(0xffffffffu, d[j]);
    if (d[j] < 0x100u && lane == __ffs(peers) - 1) atomicAdd(&h[d[j]], __popc(peers));
  }
  __syncthreads();
  counts[(int64_t)threadIdx.x * nb + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(kRsThreads) k_rs_scatter(
    const uint64_t* __restrict__ kin, uint64_t* __restrict__ kout,
    const uint32_t* __restrict__ vin, uint32_t* __restrict__ vout, int64_t m, int shift,
    int64_t nb, const int64_t* __restrict__ offs) {
  __shared__ uint32_t wc[kRsWarps][kRsBins];
  __shared__ int64_t wb[kRsWarps][kRsBins];
#pragma unroll
  for (int w = 0; w < kRsWarps; ++w) wc[w][threadIdx.x] = 0;
  __syncthreads();
  const int lane = lane_id(), w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t base = (int64_t)blockIdx.x * kRsTile + w * kRsWarpTile + lane;
  uint64_t k[kRsItems];
  uint32_t v[kRsItems], rk[kRsItems];
#pragma unroll
  for (int j = 0; j < kRsItems; ++j) {
    const int64_t i = base + 32 * j;
    k[j] = i < m ? __ldg(kin + i) : 0ull;
    v[j] = (vin && i < m) ? __ldg(vin + i) : 0u;
  }
#pragma unroll
  for (int j = 0; j < kRsItems; ++j) {
    const uint32_t d = base + 32 * j < m ? (uint32_t)(k[j] >> shift) & 255u : 0x100u;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const uint32_t dd = d & 255u;
    rk[j] = wc[w][dd] + __popc(peers & lt);
    __syncwarp();
    if (d < 0x100u && lane == __ffs(peers) - 1) wc[w][dd] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  {
    int64_t run = offs[(int64_t)threadIdx.x * nb + blockIdx.x];
#pragma unroll
    for (int ww = 0; ww < kRsWarps; ++ww) {
      wb[ww][threadIdx.x] = run;
      run += wc[ww][threadIdx.x];
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kRsItems; ++j) {
    if (base + 32 * j < m) {
      const int64_t pos = wb[w][(uint32_t)(k[j] >> shift) & 255u] + rk[j];
      kout[pos] = k[j];
      if (vout) vout[pos] = v[j];
    }
  }
}

struct CountF {
  const uint32_t* c;
  __device__ int64_t operator()(int64_t i) const { return c[i]; }
};

__global__ void k_csr_set(int64_t* p, int64_t v) { *p = v; }

size_t radix_sort_ws(int64_t m) {
  const int64_t nb = (m + kRsTile - 1) / kRsTile;
  const int64_t nc = kRsBins * (nb > 0 ? nb : 1);
  return 256 * 4 + ((sizeof(uint32_t) * nc + 255) & ~(size_t)255) +
         ((sizeof(int64_t) * (nc + 1) + 255) & ~(size_t)255) +
         ((sizeof(int64_t) * scan_workspace_elems<int64_t>(nc + 1) + 255) & ~(size_t)255);
}

// Stable LSD radix sort of keys[0, m) on bits [0, bits) with an optional
// 32-bit payload.  Ping-pongs between (keys, vals) and (alt, valt); *in_alt
// tells where the result ended.
int radix_sort(uint64_t* keys, uint64_t* alt, uint32_t* vals, uint32_t* valt, int64_t m,
               int bits, void* ws, size_t ws_bytes, bool* in_alt, cudaStream_t st) {
  *in_alt = false;
  if (m <= 1 || bits <= 0) return GB_OK;
  if (radix_sort_ws(m) > ws_bytes) {
    set_error("radix sort workspace too small");
    return GB_ERR_CAPACITY;
  }
  const int64_t nb = (m + kRsTile - 1) / kRsTile;
  const int64_t nc = kRsBins * nb;
  char* p = (char*)ws;
  int64_t* d_nc = (int64_t*)p;
  p += 256 * 4;
  uint32_t* counts = (uint32_t*)p;
  p += (sizeof(uint32_t) * nc + 255) & ~(size_t)255;
  int64_t* offs = (int64_t*)p;
  p += (sizeof(int64_t) * (nc + 1) + 255) & ~(size_t)255;
  int64_t* scan_ws = (int64_t*)p;
  k_csr_set<<<1, 1, 0, st>>>(d_nc, nc);
  count_launches(1);
  uint64_t *kin = keys, *kout = alt;
  uint32_t *vin = vals, *vout = valt;
  for (int shift = 0; shift < bits; shift += 8) {
    k_rs_hist<<<(unsigned)nb, kRsThreads, 0, st>>>(kin, m, shift, nb, counts);
    GB_LAUNCH_CHECK("k_rs_hist");
    int rc = device_exclusive_scan<int64_t>(d_nc, nc, CountF{counts}, offs, scan_ws, st);
    if (rc) return rc;
    k_rs_scatter<<<(unsigned)nb, kRsThreads, 0, st>>>(kin, kout, vin, vout, m, shift, nb, offs);
    GB_LAUNCH_CHECK("k_rs_scatter");
    count_launches(2);
    uint64_t* tk = kin; kin = kout; kout = tk;
    uint32_t* tv = vin; vin = vout; vout = tv;
    *in_alt = !*in_alt;
  }
  return GB_OK;
}

// ------------------------------------------------------------------- CSR

__global__ void k_csr_pack(int64_t m, const int64_t* __restrict__ src,
                           const int64_t* __restrict__ dst, int64_t n, int sb,
                           uint64_t* __restrict__ keys, int32_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = src[i], v = dst[i];
    int bad = (u < 0 || u >= n) ? 1 : 0;
    bad |= (v < 0 || v >= n) ? 2 : 0;
    if (bad) atomicOr(flag, bad);
    keys[i] = bad ? 0ull : ((uint64_t)u << sb) | (uint64_t)v;
  }
}

struct RunStartF {
  const uint64_t* k;
  uint64_t end;  // keys >= end are not emitted (invalid candidates)
  __device__ int64_t operator()(int64_t i) const {
    const uint64_t x = k[i];
    return x < end && (i == 0 || x != k[i - 1]) ? 1 : 0;
  }
};

constexpr int64_t kShortGap = 256;
struct Gap {
  int64_t lo, hi, val;  // rowptr[lo .. hi) = val
};

__device__ __forceinline__ void fill_gap(int64_t lo, int64_t hi, int64_t val,
                                         int64_t* __restrict__ rowptr, Gap* gaps,
                                         unsigned long long* ngaps) {
  if (hi - lo <= kShortGap) {
    for (int64_t x = lo; x < hi; ++x) rowptr[x] = val;
  } else {
    gaps[atomicAdd(ngaps, 1ull)] = Gap{lo, hi, val};
  }
}

// col[pos[i]] = dst of run start i; rowptr[v] = first position of a source
// >= v (v in (previous source, source] at each source change; the last key
// fills up to n)
__global__ void k_csr_emit(const uint64_t* __restrict__ keys, int64_t m, uint64_t end, int sb,
                           const int64_t* __restrict__ pos, int64_t n,
                           int64_t* __restrict__ rowptr, int32_t* __restrict__ col,
                           Gap* __restrict__ gaps, unsigned long long* __restrict__ ngaps) {
  const uint64_t mask = (1ull << sb) - 1ull;
  const int64_t nnz = pos[m];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t x = keys[i];
    if (x >= end) continue;
    const uint64_t prev = i ? keys[i - 1] : ~0ull;
    const int64_t s = (int64_t)(x >> sb);
    if (i == 0 || x != prev) {
      const int64_t p = pos[i];
      col[p] = (int32_t)(x & mask);
      const int64_t ps = i ? (int64_t)(prev >> sb) : -1;
      if (ps != s) fill_gap(ps + 1, s + 1, p, rowptr, gaps, ngaps);
    }
    const bool last = i + 1 == m || keys[i + 1] >= end;
    if (last) fill_gap(s + 1, n + 1, nnz, rowptr, gaps, ngaps);
  }
}

__global__ void k_csr_gaps(const Gap* __restrict__ gaps, const unsigned long long* __restrict__ ngaps,
                           int64_t* __restrict__ rowptr) {
  const int64_t ng = (int64_t)*ngaps;
  for (int64_t g = blockIdx.x; g < ng; g += gridDim.x) {
    const Gap gp = gaps[g];
    for (int64_t x = gp.lo + threadIdx.x; x < gp.hi; x += blockDim.x) rowptr[x] = gp.val;
  }
}

__global__ void k_csr_empty(int64_t n, int64_t* __restrict__ rowptr) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= n;
       v += (int64_t)gridDim.x * blockDim.x)
    rowptr[v] = 0;
}

int bits_for(int64_t n) {
  int b = 1;
  while (b < 62 && ((int64_t)1 << b) < n) ++b;
  return b;
}

static size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

size_t csr_from_keys_ws(int64_t n, int64_t m) {
  const int64_t gmax = (n + 1) / kShortGap + 4;
  return al(sizeof(uint64_t) * (m + 1)) + al(sizeof(int64_t) * (m + 1)) +
         al(sizeof(int64_t) * scan_workspace_elems<int64_t>(m + 1)) + al(sizeof(Gap) * gmax) +
         al(64) + radix_sort_ws(m);
}

// keys (and the first m entries of an alt buffer inside ws) -> CSR; keys >=
// end are dropped.  pos / gaps / scan scratch from ws.  Leaves *d_nnz on the
// device (pos[m]) and does not synchronise.
int csr_from_keys(uint64_t* keys, int64_t m, uint64_t end, int sb, int64_t n, int64_t* rowptr,
                  int32_t* col, int64_t** d_nnz, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (csr_from_keys_ws(n, m) > ws_bytes) {
    set_error("csr workspace too small");
    return GB_ERR_CAPACITY;
  }
  const int64_t gmax = (n + 1) / kShortGap + 4;
  char* p = (char*)ws;
  uint64_t* alt = (uint64_t*)p;
  p += al(sizeof(uint64_t) * (m + 1));
  int64_t* pos = (int64_t*)p;
  p += al(sizeof(int64_t) * (m + 1));
  int64_t* scan_ws = (int64_t*)p;
  p += al(sizeof(int64_t) * scan_workspace_elems<int64_t>(m + 1));
  Gap* gaps = (Gap*)p;
  p += al(sizeof(Gap) * gmax);
  int64_t* scal = (int64_t*)p;  // [0] m, [1] gap count
  p += al(64);
  *d_nnz = pos + m;
  if (m == 0) {
    k_csr_empty<<<(unsigned)((n + 256) / 256 < 4096 ? (n + 256) / 256 : 4096), 256, 0, st>>>(
        n, rowptr);
    GB_CUDA(cudaMemsetAsync(pos, 0, sizeof(int64_t), st));
    count_launches(1);
    return GB_OK;
  }
  GB_CUDA(cudaMemsetAsync(rowptr, 0, sizeof(int64_t) * (n + 1), st));  // no valid key at all
  bool in_alt = false;
  int rc = radix_sort(keys, alt, nullptr, nullptr, m, 2 * sb, p, ws_bytes - (p - (char*)ws),
                      &in_alt, st);
  if (rc) return rc;
  const uint64_t* sorted = in_alt ? alt : keys;
  k_csr_set<<<1, 1, 0, st>>>(scal, m);
  GB_CUDA(cudaMemsetAsync(scal + 1, 0, sizeof(int64_t), st));
  rc = device_exclusive_scan<int64_t>(scal, m, RunStartF{sorted, end}, pos, scan_ws, st);
  if (rc) return rc;
  const int grid = (int)((m + 255) / 256 < 64 * kNumSMs ? (m + 255) / 256 : 64 * kNumSMs);
  k_csr_emit<<<grid, 256, 0, st>>>(sorted, m, end, sb, pos, n, rowptr, col, gaps,
                                   (unsigned long long*)(scal + 1));
  GB_LAUNCH_CHECK("k_csr_emit");
  k_csr_gaps<<<4 * kNumSMs, 256, 0, st>>>(gaps, (const unsigned long long*)(scal + 1), rowptr);
  GB_LAUNCH_CHECK("k_csr_gaps");
  count_launches(3);
  return GB_OK;
}

}  // namespace gb

using namespace gb;

extern "C" {

size_t gb_csr_from_edges_workspace(int64_t n, int64_t m) {
  if (n < 0 || m < 0) return 0;
  return al(sizeof(uint64_t) * (m + 1)) + al(64) + csr_from_keys_ws(n, m);
}

int gb_csr_from_edges(int64_t n, int64_t m, const int64_t* d_src, const int64_t* d_dst,
                      int64_t* d_rowptr, int32_t* d_col, int64_t* h_nnz, void* d_ws,
                      size_t ws_bytes, void* stream) {
  if (n < 1 || n >= ((int64_t)1 << 31) || m < 0 || !d_rowptr || !h_nnz ||
      (m > 0 && (!d_src || !d_dst || !d_col))) {
    set_error("csr_from_edges: bad arguments");
    return GB_ERR_CONTRACT;
  }
  if (gb_csr_from_edges_workspace(n, m) > ws_bytes) {
    set_error("csr_from_edges: workspace too small");
    return GB_ERR_CAPACITY;
  }
  cudaStream_t st = (cudaStream_t)stream;
  char* p = (char*)d_ws;
  uint64_t* keys = (uint64_t*)p;
  p += al(sizeof(uint64_t) * (m + 1));
  int32_t* flag = (int32_t*)p;
  p += al(64);
  const int sb = bits_for(n);
  GB_CUDA(cudaMemsetAsync(flag, 0, sizeof(int32_t), st));
  if (m > 0) {
    const int grid = (int)((m + 255) / 256 < 64 * kNumSMs ? (m + 255) / 256 : 64 * kNumSMs);
    k_csr_pack<<<grid, 256, 0, st>>>(m, d_src, d_dst, n, sb, keys, flag);
    GB_LAUNCH_CHECK("k_csr_pack");
    count_launches(1);
  }
  int64_t* d_nnz = nullptr;
  int rc = csr_from_keys(keys, m, ~0ull, sb, n, d_rowptr, d_col, &d_nnz, p,
                         ws_bytes - (p - (char*)d_ws), st);
  if (rc) return rc;
  int32_t h_flag = 0;
  int64_t nnz = 0;
  GB_CUDA(cudaMemcpyAsync(&h_flag, flag, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  GB_CUDA(cudaMemcpyAsync(&nnz, d_nnz, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GB_CUDA(cudaStreamSynchronize(st));
  if (h_flag & 1) { set_error("row index out of range"); return GB_ERR_CONTRACT; }
  if (h_flag & 2) { set_error("column index out of range"); return GB_ERR_CONTRACT; }
  if (nnz > 0) GB_CUDA(cudaMemsetAsync(d_col + nnz, 0, sizeof(int32_t) * GB_COL_PAD, st));
  *h_nnz = nnz;
  return GB_OK;
}

}  // extern "C"
