// Aggregation products of the epoch pipeline (reference pipeline.py:123-130
// forward_aggregate, 267-305 _propagate_batch), sm_100a:
//   * Y = A^l X over the stacked sampled adjacency of a bulk (A values 1.0,
//     fp32 features): warp per row, lanes across the feature width (16-B
//     loads when f % 4 == 0), entries summed in row order with the next
//     four X rows in flight;
//   * the first-occurrence map that carries a deeper layer's rows onto the
//     next shallower layer's column vertices.
// A row of batch b addresses X row col[e] + shift[b]: shift = 0 for the
// block-diagonal layout (SAGE), colv_off[b] for LADIES' shared layout.
#include "gb_common.cuh"
#include "gb_internal.h"

namespace gb {

__device__ __forceinline__ int64_t agg_batch_of(const int64_t* off, int64_t k, int64_t r) {
  int64_t lo = 0, hi = k;  // last b with off[b] <= r
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (off[mid] <= r) lo = mid; else hi = mid;
  }
  return lo;
}

template <bool V4>
__global__ void __launch_bounds__(256) k_spmm_rows(int64_t R, const int64_t* __restrict__ rowptr,
                                                   const int32_t* __restrict__ col,
                                                   const int64_t* __restrict__ rowb,
                                                   const int64_t* __restrict__ shift, int64_t k,
                                                   const float* __restrict__ X, int64_t f,
                                                   float* __restrict__ Y) {
  constexpr int W = V4 ? 128 : 32;  // features per warp pass
  const int lane = lane_id();
  for (int64_t r = global_warp(); r < R; r += grid_warps()) {
    const int64_t sh = shift ? shift[agg_batch_of(rowb, k, r)] : 0;
    const int64_t e0 = rowptr[r], e1 = rowptr[r + 1];
    for (int64_t f0 = 0; f0 < f; f0 += W) {
      const int64_t fl = f0 + (V4 ? 4 * lane : lane);
      const bool on = fl < f;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      int64_t e = e0;
      for (; e + 4 <= e1; e += 4) {
        float4 x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float* p = X + (int64_t)(__ldg(col + e + u) + sh) * f + fl;
          if (V4) x[u] = on ? __ldg((const float4*)p) : make_float4(0.f, 0.f, 0.f, 0.f);
          else x[u] = make_float4(on ? __ldg(p) : 0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          acc.x += x[u].x; acc.y += x[u].y; acc.z += x[u].z; acc.w += x[u].w;
        }
      }
      for (; e < e1; ++e) {
        const float* p = X + (int64_t)(__ldg(col + e) + sh) * f + fl;
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        if (V4) { if (on) x = __ldg((const float4*)p); }
        else if (on) x.x = __ldg(p);
        acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
      }
      if (on) {
        float* q = Y + r * f + fl;
        if (V4) *(float4*)q = acc;
        else *q = acc.x;
      }
    }
  }
}

// first[j] = smallest entry e whose column index is j (entry e of layer
// l - 1 is row e of layer l); colidx == nullptr: e itself (LADIES)
__global__ void k_first_occ(int64_t F, const int32_t* __restrict__ colidx,
                            const int64_t* __restrict__ eb, const int64_t* __restrict__ shift,
                            int64_t k, int32_t* __restrict__ first) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < F;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = e;
    if (colidx) j = colidx[e] + (shift ? shift[agg_batch_of(eb, k, e)] : 0);
    atomicMin(first + j, (int32_t)e);
  }
}

static int agg_grid(int64_t work, int threads) {
  int64_t g = (work + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 16 * kNumSMs) g = 16 * kNumSMs;
  return (int)g;
}

int spmm_rows(int64_t R, const int64_t* rowptr, const int32_t* col, const int64_t* rowb,
              const int64_t* shift, int64_t k, const float* X, int64_t f, float* Y,
              cudaStream_t st) {
  if (R == 0 || f == 0) return GB_OK;
  const bool v4 = (f % 4 == 0) && ((uintptr_t)X % 16 == 0) && ((uintptr_t)Y % 16 == 0);
  if (v4)
    k_spmm_rows<true><<<agg_grid(R * 32, 256), 256, 0, st>>>(R, rowptr, col, rowb, shift, k, X, f,
                                                             Y);
  else
    k_spmm_rows<false><<<agg_grid(R * 32, 256), 256, 0, st>>>(R, rowptr, col, rowb, shift, k, X,
                                                              f, Y);
  GB_LAUNCH_CHECK("k_spmm_rows");
  count_launches(1);
  return GB_OK;
}

// forward_aggregate (pipeline.py:123-130) = scipy `A.to_scipy() @ H` in
// float64 with A's values: warp per row, lanes over the feature columns,
// y[c] = y[c] + v_e * X[col_e, c] over the row's entries in order, the
// product and the sum rounded separately — scipy's csr_matvecs loop, so the
// result is bit-identical to the reference's.
__global__ void __launch_bounds__(256) k_spmm_f64(int64_t R, const int64_t* __restrict__ rowptr,
                                                const int32_t* __restrict__ col,
                                                const double* __restrict__ val,
                                                const double* __restrict__ X, int64_t f,
                                                double* __restrict__ Y) {
  const int lane = lane_id();
  for (int64_t r = global_warp(); r < R; r += grid_warps()) {
    const int64_t e0 = rowptr[r], e1 = rowptr[r + 1];
    for (int64_t c0 = 0; c0 < f; c0 += 32) {
      const int64_t c = c0 + lane;
      double y = 0.0;
      if (c < f)
        for (int64_t e = e0; e < e1; ++e)
          y = __dadd_rn(y, __dmul_rn(__ldg(val + e), __ldg(X + (int64_t)__ldg(col + e) * f + c)));
      if (c < f) Y[r * f + c] = y;
    }
  }
}

int spmm_f64(int64_t R, const int64_t* rowptr, const int32_t* col, const double* val,
             const double* X, int64_t f, double* Y, cudaStream_t st) {
  if (R == 0 || f == 0) return GB_OK;
  k_spmm_f64<<<agg_grid(R * 32, 256), 256, 0, st>>>(R, rowptr, col, val, X, f, Y);
  GB_LAUNCH_CHECK("k_spmm_f64");
  count_launches(1);
  return GB_OK;
}

int first_occurrence(int64_t F, const int32_t* colidx, const int64_t* eb, const int64_t* shift,
                     int64_t k, int64_t ncols, int32_t* first, cudaStream_t st) {
  GB_CUDA(cudaMemsetAsync(first, 0x7f, sizeof(int32_t) * (ncols > 0 ? ncols : 1), st));
  if (F == 0) return GB_OK;
  k_first_occ<<<agg_grid(F, 256), 256, 0, st>>>(F, colidx, eb, shift, k, first);
  GB_LAUNCH_CHECK("k_first_occ");
  count_launches(1);
  return GB_OK;
}

// dst[dst_off[row_i] + t] = src[src_off[i] + t] for t < len_i, warp per
// segment; row_i = rows[i] (identity when rows == nullptr), len_i = lens[i]
// or src_off[i + 1] - src_off[i].  Places the picks returned by block owners
// and packs slot-layout rows in the distributed executor.
__global__ void k_segment_copy(int64_t m, const int64_t* __restrict__ rows,
                               const int64_t* __restrict__ src_off,
                               const int32_t* __restrict__ lens, const int32_t* __restrict__ src,
                               const int64_t* __restrict__ dst_off, int32_t* __restrict__ dst) {
  const int lane = lane_id();
  for (int64_t i = global_warp(); i < m; i += grid_warps()) {
    const int64_t s0 = src_off[i];
    const int64_t len = lens ? (int64_t)lens[i] : src_off[i + 1] - s0;
    const int64_t d0 = dst_off[rows ? rows[i] : i];
    for (int64_t t = lane; t < len; t += 32) dst[d0 + t] = src[s0 + t];
  }
}

int segment_copy(int64_t m, const int64_t* rows, const int64_t* src_off, const int32_t* lens,
                 const int32_t* src, const int64_t* dst_off, int32_t* dst, cudaStream_t st) {
  if (m == 0) return GB_OK;
  k_segment_copy<<<agg_grid(m * 32, 256), 256, 0, st>>>(m, rows, src_off, lens, src, dst_off, dst);
  GB_LAUNCH_CHECK("k_segment_copy");
  count_launches(1);
  return GB_OK;
}

}  // namespace gb
