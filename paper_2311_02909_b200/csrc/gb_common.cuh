// Shared device helpers for the B200 bulk sampler (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/gnnbulk_b200.h"

namespace gb {

constexpr int kWarp = 32;
constexpr int kNumSMs = 148;  // B200; persistent grids are multiples of this

// ---------------------------------------------------------------- errors
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);
#define GB_CUDA(call)                                    \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return gb::cuda_status(_e, #call); \
  } while (0)
// GB_SYNC_DEBUG=1 in the environment: every checked launch also
// synchronises the device and reports a fault against the launch that
// caused it (debugging only; breaks CUDA-graph capture).
bool sync_debug();
#define GB_LAUNCH_CHECK(what)                                      \
  do {                                                             \
    cudaError_t _e = cudaGetLastError();                           \
    if (_e == cudaSuccess && gb::sync_debug()) _e = cudaDeviceSynchronize(); \
    if (_e != cudaSuccess) return gb::cuda_status(_e, what);       \
  } while (0)

// ------------------------------------------------------------------ RNG
// Philox4x64-10 (Random123; numpy.random.Philox) and the keyed uniform
//   u(seed, epoch, depth, row, t) = (philox([row, depth, t>>2, 0],
//                                            [seed, epoch])[t&3] >> 11) * 2^-53
// that replaces reference RowRng.stream (pkg/src/gnnbulk/sampler.py:97-116);
// oracle/philox.py is the pinned CPU restatement.
__device__ __forceinline__ void philox4x64_10(uint64_t& c0, uint64_t& c1, uint64_t& c2,
                                              uint64_t& c3, uint64_t k0, uint64_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B97F4A7C15ULL;
      k1 += 0xBB67AE8584CAA73BULL;
    }
    const uint64_t lo0 = 0xD2E7470EE14C6C93ULL * c0;
    const uint64_t hi0 = __umul64hi(0xD2E7470EE14C6C93ULL, c0);
    const uint64_t lo1 = 0xCA5A826395121157ULL * c2;
    const uint64_t hi1 = __umul64hi(0xCA5A826395121157ULL, c2);
    const uint64_t n0 = hi1 ^ c1 ^ k0;
    const uint64_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
}

__device__ __forceinline__ uint64_t philox_word(uint64_t seed, uint64_t epoch, uint64_t depth,
                                                uint64_t row, uint64_t t) {
  uint64_t c0 = row, c1 = depth, c2 = t >> 2, c3 = 0;
  philox4x64_10(c0, c1, c2, c3, seed, epoch);
  const uint32_t w = (uint32_t)(t & 3);
  return w == 0 ? c0 : w == 1 ? c1 : w == 2 ? c2 : c3;
}

__device__ __forceinline__ double uniform53(uint64_t seed, uint64_t epoch, uint64_t depth,
                                            uint64_t row, uint64_t t) {
  return (double)(philox_word(seed, epoch, depth, row, t) >> 11) * 0x1.0p-53;
}

// Philox4x32-10 (Random123), used where 24-bit uniforms suffice (race keys)
__device__ __forceinline__ void philox4x32_10(uint32_t& c0, uint32_t& c1, uint32_t& c2,
                                              uint32_t& c3, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
}

// Exp(1) variate E = -log(1 - V) from a 32-bit word x, V = (x + 1/2) 2^-32.
// The race selects the SMALLEST keys E / e^2, so E must be accurate in
// relative terms near 0: V is formed exactly (relative rounding 2^-24 at
// most) and E = -log1p(-V) there; the upper half uses 1 - V formed exactly
// from the complement, so neither branch cancels.  Accurate libm log1pf /
// logf (a few ulp), never the __logf intrinsic (absolute error ~2^-21,
// which near the selection boundary is a large fraction of E).
__device__ __forceinline__ float race_exp(uint32_t x) {
  if (x < 0x80000000u) return -log1pf(-(((float)x + 0.5f) * 0x1.0p-32f));
  return -logf(((float)(0xffffffffu - x) + 0.5f) * 0x1.0p-32f);
}

// ------------------------------------------------------------ warp utils
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// first index i in [lo, hi) with a[i] > x (a sorted ascending), i.e.
// numpy searchsorted(side="right")
template <typename T>
__device__ __forceinline__ int64_t upper_bound(const T* a, int64_t lo, int64_t hi, T x) {
  while (lo < hi) {
    int64_t mid = lo + ((hi - lo) >> 1);
    if (a[mid] > x) hi = mid; else lo = mid + 1;
  }
  return lo;
}

__device__ __forceinline__ int grid_warps() { return (gridDim.x * blockDim.x) >> 5; }
__device__ __forceinline__ int global_warp() {
  return (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
}

}  // namespace gb
