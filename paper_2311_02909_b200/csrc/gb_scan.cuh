// Device-wide exclusive prefix sums with a device-resident length, so that
// every launch of a bulk has a host-known grid (upper bound) and no host
// synchronisation: the whole bulk can be captured in one CUDA graph.
//
// Three phases (reduce tiles -> scan tile sums in one CTA -> rescan tiles),
// inputs produced by a functor so they are never materialised.  Output has
// n + 1 entries; out[n] is the total.
#pragma once
#include "gb_common.cuh"
#include "gb_internal.h"

namespace gb {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;  // 2048

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

template <typename T, typename F>
__global__ void __launch_bounds__(kScanThreads) scan_reduce_tiles(const int64_t* n_ptr, F f,
                                                                  T* tile_sums) {
  __shared__ T sw[33];
  const int64_t n = *n_ptr;
  const int64_t ntiles = (n + kScanTile - 1) / kScanTile;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t base = tile * kScanTile + (int64_t)threadIdx.x * kScanItems;
    T acc = T(0);
#pragma unroll
    for (int i = 0; i < kScanItems; ++i)
      if (base + i < n) acc += f(base + i);
    T total;
    block_excl_scan(acc, sw, total);
    if (threadIdx.x == 0) tile_sums[tile] = total;
  }
}

template <typename T>
__global__ void __launch_bounds__(1024) scan_tile_sums(const int64_t* n_ptr, T* tile_sums,
                                                       T* out_total) {
  __shared__ T sw[33];
  const int64_t n = *n_ptr;
  const int64_t ntiles = (n + kScanTile - 1) / kScanTile;
  T carry = T(0);
  for (int64_t b = 0; b < ntiles; b += blockDim.x) {
    const int64_t i = b + threadIdx.x;
    T v = i < ntiles ? tile_sums[i] : T(0);
    T total;
    T ex = block_excl_scan(v, sw, total);
    if (i < ntiles) tile_sums[i] = ex + carry;
    carry += total;
  }
  if (threadIdx.x == 0) *out_total = carry;
}

template <typename T, typename OutT, typename F>
__global__ void __launch_bounds__(kScanThreads) scan_tiles(const int64_t* n_ptr, F f,
                                                           const T* tile_offsets, OutT* out) {
  __shared__ T sw[33];
  const int64_t n = *n_ptr;
  const int64_t ntiles = (n + kScanTile - 1) / kScanTile;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t base = tile * kScanTile + (int64_t)threadIdx.x * kScanItems;
    T vals[kScanItems];
    T acc = T(0);
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      vals[i] = base + i < n ? f(base + i) : T(0);
      acc += vals[i];
    }
    T total;
    T ex = block_excl_scan(acc, sw, total) + tile_offsets[tile];
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      if (base + i < n) out[base + i] = (OutT)ex;
      ex += vals[i];
    }
  }
}

// Writes out[n] too: the total.
template <typename T, typename OutT>
__global__ void scan_write_total(const int64_t* n_ptr, const T* total, OutT* out) {
  out[*n_ptr] = (OutT)*total;
}

// Workspace: (max_n / tile + 2) elements of T.
template <typename T>
inline size_t scan_workspace_elems(int64_t max_n) {
  return (size_t)((max_n + kScanTile - 1) / kScanTile + 2);
}

template <typename T, typename OutT, typename F>
inline int device_exclusive_scan(const int64_t* d_n, int64_t max_n, F f, OutT* out, T* ws,
                                 cudaStream_t st) {
  const int64_t max_tiles = (max_n + kScanTile - 1) / kScanTile;
  const int grid = (int)(max_tiles < 4 * kNumSMs ? (max_tiles > 0 ? max_tiles : 1) : 4 * kNumSMs);
  T* tile_sums = ws;
  T* total = ws + max_tiles + 1;
  scan_reduce_tiles<T, F><<<grid, kScanThreads, 0, st>>>(d_n, f, tile_sums);
  scan_tile_sums<T><<<1, 1024, 0, st>>>(d_n, tile_sums, total);
  scan_tiles<T, OutT, F><<<grid, kScanThreads, 0, st>>>(d_n, f, tile_sums, out);
  scan_write_total<T, OutT><<<1, 1, 0, st>>>(d_n, total, out);
  GB_LAUNCH_CHECK("device_exclusive_scan");
  count_launches(4);
  return GB_OK;
}

}  // namespace gb
