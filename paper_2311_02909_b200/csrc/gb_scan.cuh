// Device-wide exclusive prefix sums with a device-resident length, so that
// every launch of a bulk has a host-known grid (upper bound) and no host
// synchronisation: the whole bulk can be captured in one CUDA graph.
//
// One single-pass kernel per scan (decoupled look-back), inputs produced by a
// functor so they are never materialised.  Output has n + 1 entries; out[n]
// is the total.
#pragma once
#include "gb_common.cuh"
#include "gb_internal.h"

namespace gb {

constexpr int kScanThreads = 256;
#ifndef GB_SCAN_ITEMS
#define GB_SCAN_ITEMS 8
#endif
constexpr int kScanItems = GB_SCAN_ITEMS;
constexpr int kScanTile = kScanThreads * kScanItems;

template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* smem_warp, T& total) {
  // v: per-thread value; returns exclusive prefix within the block.
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T inc = warp_incl_scan(v);
  if (lane == 31) smem_warp[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = lane < (int)(blockDim.x >> 5) ? smem_warp[lane] : T(0);
    T wi = warp_incl_scan(w);
    if (lane < (int)(blockDim.x >> 5)) smem_warp[lane] = wi - w;
    if (lane == 31) smem_warp[32] = wi;
  }
  __syncthreads();
  T res = inc - v + smem_warp[warp];
  total = smem_warp[32];
  __syncthreads();
  return res;
}

// Single pass with decoupled look-back: tiles are taken in ticket order; a
// tile publishes its aggregate, then warp 0 sums its predecessors' words
// 32 at a time back to the nearest one holding an inclusive prefix, and
// publishes its own inclusive prefix.  Status word: flag in bits 62-63
// (0 not ready, 1 aggregate, 2 inclusive prefix), the value below (counts
// are non-negative and far below 2^62).
constexpr unsigned long long kStAgg = 1ull << 62, kStInc = 2ull << 62;
constexpr unsigned long long kStVal = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long st_load(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_store(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Decoupled look-back for tile `tile` whose predecessors back to `first`
// (a segment start) are summed: publishes `total` (aggregate, then inclusive
// prefix) and returns the exclusive prefix.  Warp 0 only; st[1 + t] are the
// tile status words (zeroed before the launch).
__device__ __forceinline__ int64_t tile_lookback(unsigned long long* st, int64_t tile,
                                                 int64_t first, int64_t total) {
  const int lane = threadIdx.x & 31;
  int64_t prefix = 0;
  if (tile == first) {
    if (lane == 0) st_store(st + 1 + tile, kStInc | (unsigned long long)total);
    return 0;
  }
  if (lane == 0) st_store(st + 1 + tile, kStAgg | (unsigned long long)total);
  for (int64_t j = tile - 1;; j -= 32) {
    const int64_t idx = j - lane;  // lane 0: nearest predecessor
    unsigned long long w;
    do {
      w = idx >= first ? st_load(st + 1 + idx) : kStInc;
    } while (__any_sync(0xffffffffu, (w >> 62) == 0));
    const unsigned inc = __ballot_sync(0xffffffffu, (w >> 62) == 2);
    const int stop = inc ? __ffs(inc) - 1 : 31;
    prefix += warp_sum(lane <= stop ? (int64_t)(w & kStVal) : (int64_t)0);
    if (inc) break;
  }
  if (lane == 0) st_store(st + 1 + tile, kStInc | (unsigned long long)(prefix + total));
  return prefix;
}

template <typename OutT, typename F, int STRIDE = 1>
__global__ void __launch_bounds__(kScanThreads) scan_single_pass(const int64_t* n_ptr, F f,
                                                                 OutT* out,
                                                                 unsigned long long* st) {
  // st[0]: tile ticket; st[1 + t]: status of tile t (zeroed before launch)
  __shared__ int64_t sw[33];
  __shared__ int64_t s_tile, s_prefix;
  const int64_t n = *n_ptr;
  const int64_t ntiles = (n + kScanTile - 1) / kScanTile;
  if (ntiles == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (OutT)0;
    return;
  }
  const int lane = threadIdx.x & 31;
  for (;;) {
    if (threadIdx.x == 0) s_tile = (int64_t)atomicAdd(st, 1ull);
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile >= ntiles) return;
    const int64_t base = tile * kScanTile + (int64_t)threadIdx.x * kScanItems;
    int64_t vals[kScanItems];
    int64_t acc = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      vals[i] = base + i < n ? (int64_t)f(base + i) : 0;
      acc += vals[i];
    }
    int64_t total;
    int64_t ex = block_excl_scan(acc, sw, total);
    if (threadIdx.x < 32) {
      int64_t prefix = 0;
      if (tile == 0) {
        if (lane == 0) st_store(st + 1, kStInc | (unsigned long long)total);
      } else {
        if (lane == 0) st_store(st + 1 + tile, kStAgg | (unsigned long long)total);
        for (int64_t j = tile - 1;; j -= 32) {
          const int64_t idx = j - lane;  // lane 0: nearest predecessor
          unsigned long long w;
          do {
            w = idx >= 0 ? st_load(st + 1 + idx) : kStInc;
          } while (__any_sync(0xffffffffu, (w >> 62) == 0));
          const unsigned inc = __ballot_sync(0xffffffffu, (w >> 62) == 2);
          const int stop = inc ? __ffs(inc) - 1 : 31;
          prefix += warp_sum(lane <= stop ? (int64_t)(w & kStVal) : (int64_t)0);
          if (inc) break;
        }
        if (lane == 0) st_store(st + 1 + tile, kStInc | (unsigned long long)(prefix + total));
      }
      if (lane == 0) s_prefix = prefix;
    }
    __syncthreads();
    ex += s_prefix;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      if (base + i < n) out[(base + i) * STRIDE] = (OutT)ex;
      ex += vals[i];
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) out[n * STRIDE] = (OutT)(s_prefix + total);
    __syncthreads();  // s_tile / s_prefix reuse
  }
}

// Workspace: (max_n / tile + 2) 64-bit words.
template <typename T>
inline size_t scan_workspace_elems(int64_t max_n) {
  return (size_t)((max_n + kScanTile - 1) / kScanTile + 2);
}

// out[0..n) = exclusive prefix of f(0..n), out[n] = total; n = *d_n <= max_n.
// STRIDE > 1: element i lands at out[i * STRIDE] (prefixes interleaved with
// the data they count).
template <typename T, int STRIDE = 1, typename OutT, typename F>
inline int device_exclusive_scan(const int64_t* d_n, int64_t max_n, F f, OutT* out, T* ws,
                                 cudaStream_t st) {
  static_assert(sizeof(T) == 8, "64-bit scan workspace");
  const int64_t max_tiles = (max_n + kScanTile - 1) / kScanTile;
  const int grid = (int)(max_tiles < 8 * kNumSMs ? (max_tiles > 0 ? max_tiles : 1) : 8 * kNumSMs);
  GB_CUDA(cudaMemsetAsync(ws, 0, sizeof(unsigned long long) * (max_tiles + 1), st));
  scan_single_pass<OutT, F, STRIDE><<<grid, kScanThreads, 0, st>>>(d_n, f, out,
                                                           (unsigned long long*)ws);
  GB_LAUNCH_CHECK("device_exclusive_scan");
  count_launches(1);
  return GB_OK;
}

}  // namespace gb
