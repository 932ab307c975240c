// Synthetic graph ingredients on the device (SURVEY.md §8(d) inputs, §8(f)4):
// Graph500 R-MAT edge candidates driven by the same Philox4x64-10 as the
// sampler (deterministic on every device), and a 64-bit keyed hash used to
// order / relabel vertices.  Sorting and de-duplication of the candidates is
// plumbing done by the caller (torch.sort / unique on the device).
#include "gb_common.cuh"
#include "gb_internal.h"

namespace gb {

// Candidate i: for each of `scale` levels draw u and pick a quadrant with
// probabilities (a, b, c, 1-a-b-c); bit l of (src, dst) is set for the
// lower/right halves.  Rejected (self loop or id >= n) candidates get -1.
__global__ void k_rmat(uint64_t seed, int32_t scale, int64_t n, int64_t first, int64_t count,
                       double a, double b, double c, int64_t* __restrict__ src,
                       int64_t* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t e = (uint64_t)(first + i);
    int64_t u = 0, v = 0;
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
    const bool bad = u == v || u >= n || v >= n;
    src[i] = bad ? -1 : u;
    dst[i] = bad ? -1 : v;
  }
}

__global__ void k_hash64(uint64_t seed, const int64_t* __restrict__ x, int64_t count,
                         int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t c0 = (uint64_t)x[i], c1 = 0x68617368ULL, c2 = 0, c3 = 0;
    philox4x64_10(c0, c1, c2, c3, seed, 0x72656c6162656cULL);
    out[i] = (int64_t)(c0 >> 1);  // non-negative sort key
  }
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

}  // extern "C"
