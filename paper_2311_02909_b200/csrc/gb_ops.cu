// Generic sparse operators of the reference API on the device (sm_100a):
//   spgemm          sparse.py:233-251  (scipy csr_matmat + drop |x| < 1e-12)
//   add             sparse.py:417-427  (scipy csr + csr, same drop policy)
//   norm_rows_*     sparse.py:254-286  (numpy add.reduceat order)
//   ITS sampling    sampler.py:157-207 (its_sample_row / sample_rows_ordered)
// used by the public operator API, the `prob_spgemm` hook of
// sample_epoch_bulk and the distributed multiply.  Bit-exact rules:
//   * spgemm accumulates every C[i, j] in the order of A's row i (ascending
//     k), starting from 0.0, with separate fp64 multiply and add — what
//     csr_matmat does; the hash accumulator processes one A entry per step,
//     so per-slot updates are ordered.
//   * row sums follow numpy's add.reduce: a[0] + pairwise(a[1:]) with the
//     8-accumulator blocks of 128 (numpy pairwise_sum).
//   * ITS is the literal remove-and-renormalise loop with keyed uniforms.
#include "gb_common.cuh"
#include "gb_internal.h"
#include "gb_scan.cuh"

namespace gb {

constexpr double kDropTol = 1e-12;  // sparse.py:25
constexpr int kSpThreads = 256;
constexpr int kSmemHash = 2048;     // shared-memory hash slots per CTA

struct UbF {
  const int64_t* a_ptr;
  const int32_t* a_col;
  const int64_t* b_ptr;
  __device__ int64_t operator()(int64_t i) const {
    int64_t s = 0;
    for (int64_t e = a_ptr[i]; e < a_ptr[i + 1]; ++e) {
      const int32_t k = a_col[e];
      s += b_ptr[k + 1] - b_ptr[k];
    }
    return s;
  }
};

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

__device__ __forceinline__ int hpow2(int64_t ub) {
  int64_t h = 1;
  while (h < 2 * ub) h <<= 1;
  return (int)h;
}

// in-place bitonic sort of (key, val) pairs, n = power of two, block-wide
template <typename V>
__device__ void block_bitonic(int32_t* key, V* val, int n) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool up = (i & k) == 0;
          if ((key[i] > key[ixj]) == up) {
            const int32_t tk = key[i]; key[i] = key[ixj]; key[ixj] = tk;
            const V tv = val[i]; val[i] = val[ixj]; val[ixj] = tv;
          }
        }
      }
      __syncthreads();
    }
  }
}

// One CTA per row of A (grid-stride).  Hash in shared memory when the
// row's product bound fits, else in the row's global slice (4 * ub slots).
// Sorted surviving entries go to tmp at ub-offset; counts to cnt.
__global__ void __launch_bounds__(kSpThreads) k_spgemm_rows(
    int64_t m, const int64_t* __restrict__ a_ptr, const int32_t* __restrict__ a_col,
    const double* __restrict__ a_val, const int64_t* __restrict__ b_ptr,
    const int32_t* __restrict__ b_col, const double* __restrict__ b_val,
    const int64_t* __restrict__ ub, int32_t* __restrict__ gkey, double* __restrict__ gval,
    int32_t* __restrict__ tmp_col, double* __restrict__ tmp_val, int64_t* __restrict__ cnt) {
  __shared__ int32_t skey[kSmemHash];
  __shared__ double sval[kSmemHash];
  __shared__ int s_c;
  for (int64_t i = blockIdx.x; i < m; i += gridDim.x) {
    const int64_t u0 = ub[i], u = ub[i + 1] - u0;
    if (u == 0) {
      if (threadIdx.x == 0) cnt[i] = 0;
      continue;
    }
    const int H = hpow2(u);
    const bool sm = H <= kSmemHash;
    int32_t* key = sm ? skey : gkey + 4 * u0;
    double* val = sm ? sval : gval + 4 * u0;
    for (int h = threadIdx.x; h < H; h += blockDim.x) { key[h] = -1; val[h] = 0.0; }
    __syncthreads();
    for (int64_t e = a_ptr[i]; e < a_ptr[i + 1]; ++e) {
      const int32_t kk = a_col[e];
      const double av = a_val[e];
      for (int64_t f = b_ptr[kk] + threadIdx.x; f < b_ptr[kk + 1]; f += blockDim.x) {
        const int32_t j = b_col[f];
        uint32_t h = hash32((uint32_t)j) & (uint32_t)(H - 1);
        while (true) {
          const int32_t prev = atomicCAS(&key[h], -1, j);
          if (prev == -1 || prev == j) break;
          h = (h + 1) & (uint32_t)(H - 1);
        }
        val[h] = __dadd_rn(val[h], __dmul_rn(av, b_val[f]));
      }
      __syncthreads();  // k-steps in order: C[i, j] accumulated as csr_matmat
    }
    // keep |x| >= drop tol (csr_matmat drops exact zeros, the wrapper < 1e-12)
    if (threadIdx.x == 0) s_c = 0;
    __syncthreads();
    for (int h = threadIdx.x; h < H; h += blockDim.x) {
      const bool keep = key[h] >= 0 && fabs(val[h]) >= kDropTol;
      if (!keep) key[h] = 0x7fffffff;
    }
    __syncthreads();
    block_bitonic<double>(key, val, H);
    for (int h = threadIdx.x; h < H; h += blockDim.x) {
      if (key[h] != 0x7fffffff) {
        tmp_col[u0 + h] = key[h];
        tmp_val[u0 + h] = val[h];
        atomicAdd(&s_c, 1);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) cnt[i] = s_c;
    __syncthreads();
  }
}

__global__ void k_rows_copy(int64_t m, const int64_t* __restrict__ src_off,
                            const int64_t* __restrict__ dst_ptr, const int32_t* __restrict__ sc,
                            const double* __restrict__ sv, int32_t* __restrict__ dc,
                            double* __restrict__ dv) {
  for (int64_t i = blockIdx.x; i < m; i += gridDim.x) {
    const int64_t s0 = src_off[i], d0 = dst_ptr[i], c = dst_ptr[i + 1] - d0;
    for (int64_t x = threadIdx.x; x < c; x += blockDim.x) {
      dc[d0 + x] = sc[s0 + x];
      dv[d0 + x] = sv[s0 + x];
    }
  }
}

struct CntF {
  const int64_t* c;
  __device__ int64_t operator()(int64_t i) const { return c[i]; }
};

// C = A + B (same shape): per-row merge of two sorted rows, thread per row
template <bool WRITE>
__global__ void k_add_rows(int64_t m, const int64_t* __restrict__ a_ptr,
                           const int32_t* __restrict__ a_col, const double* __restrict__ a_val,
                           const int64_t* __restrict__ b_ptr, const int32_t* __restrict__ b_col,
                           const double* __restrict__ b_val, int64_t* __restrict__ cnt,
                           const int64_t* __restrict__ c_ptr, int32_t* __restrict__ c_col,
                           double* __restrict__ c_val) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t x = a_ptr[i], xe = a_ptr[i + 1], y = b_ptr[i], ye = b_ptr[i + 1];
    int64_t o = WRITE ? c_ptr[i] : 0, c = 0;
    while (x < xe || y < ye) {
      int32_t col;
      double v;
      if (y >= ye || (x < xe && a_col[x] < b_col[y])) { col = a_col[x]; v = a_val[x++]; }
      else if (x >= xe || b_col[y] < a_col[x]) { col = b_col[y]; v = b_val[y++]; }
      else { col = a_col[x]; v = __dadd_rn(a_val[x++], b_val[y++]); }
      if (fabs(v) >= kDropTol) {
        if (WRITE) { c_col[o + c] = col; c_val[o + c] = v; }
        ++c;
      }
    }
    if (!WRITE) cnt[i] = c;
  }
}

// numpy pairwise_sum (numpy/core/src/umath/loops_utils.h.src): n < 8
// sequential, n <= 128 eight accumulators, else split at n/2 rounded down
// to a multiple of 8 (recursion depth <= log2(n / 128)).
template <bool SQUARE>
__device__ double np_pairwise(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, SQUARE ? __dmul_rn(a[i], a[i]) : a[i]);
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = SQUARE ? __dmul_rn(a[j], a[j]) : a[j];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], SQUARE ? __dmul_rn(a[i + j], a[i + j]) : a[i + j]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, SQUARE ? __dmul_rn(a[i], a[i]) : a[i]);
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise<SQUARE>(a, n2), np_pairwise<SQUARE>(a + n2, n - n2));
}

// norm_rows: out = v / (v[0] + pairwise(v[1:])) (SQUARE: v*v / same of v*v)
template <bool SQUARE>
__global__ void k_norm_rows(int64_t m, const int64_t* __restrict__ ptr,
                            const double* __restrict__ val, double* __restrict__ out,
                            int32_t* __restrict__ err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = ptr[i], n = ptr[i + 1] - a;
    if (n == 0) continue;
    const double first = SQUARE ? __dmul_rn(val[a], val[a]) : val[a];
    const double s = __dadd_rn(first, np_pairwise<SQUARE>(val + a + 1, n - 1));
    if (!(s > 0.0)) atomicExch(err, 2);
    for (int64_t x = 0; x < n; ++x) {
      if (val[a + x] < 0.0) atomicExch(err, 1);
      const double v = SQUARE ? __dmul_rn(val[a + x], val[a + x]) : val[a + x];
      out[a + x] = __ddiv_rn(v, s);
    }
  }
}

// Generic keyed ITS (its_sample_row over arbitrary positive weights), one
// thread per row; draws of row r use u(seed, epoch, depth, keys[r], t) or
// the injected inject[r * s + t].  picks[r*s + t] = picked index (draw order).
__global__ void k_its_rows(int64_t m, const int64_t* __restrict__ ptr,
                           const double* __restrict__ val, int32_t s,
                           const int64_t* __restrict__ keys, const double* __restrict__ inject,
                           uint64_t seed, uint64_t epoch, uint64_t depth,
                           double* __restrict__ w, double* __restrict__ cdf,
                           int32_t* __restrict__ picks, int32_t* __restrict__ take_out,
                           int32_t* __restrict__ err) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = ptr[r], n = ptr[r + 1] - a;
    const int64_t take = n < s ? n : s;
    take_out[r] = (int32_t)take;
    if (n == 0) continue;
    double* wr = w + a;
    double* cr = cdf + a;
    double mn = val[a];
    for (int64_t x = 0; x < n; ++x) {
      wr[x] = val[a + x];
      mn = fmin(mn, wr[x]);
    }
    if (mn <= 0.0) { atomicExch(err, 1); continue; }
    if (take == n) {
      for (int64_t x = 0; x < n; ++x) picks[r * s + x] = (int32_t)x;
      continue;
    }
    int64_t dirty = 0;
    for (int64_t t = 0; t < take; ++t) {
      double acc = dirty ? cr[dirty - 1] : 0.0;
      for (int64_t x = dirty; x < n; ++x) {
        acc = __dadd_rn(acc, wr[x]);
        cr[x] = acc;
      }
      const double u = inject ? inject[r * s + t]
                              : uniform53(seed, epoch, depth, (uint64_t)keys[r], (uint64_t)t);
      const double target = __dmul_rn(u, cr[n - 1]);
      int64_t idx = upper_bound(cr, 0, n, target);
      if (idx >= n) idx = n - 1;
      while (wr[idx] == 0.0) --idx;
      picks[r * s + t] = (int32_t)idx;
      wr[idx] = 0.0;
      dirty = idx;
    }
  }
}

static int ogrid(int64_t n, int t, int cap) {
  int64_t g = (n + t - 1) / t;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

}  // namespace gb

using namespace gb;

extern "C" {

int gb_spgemm_bound(int64_t m, const int64_t* d_a_ptr, const int32_t* d_a_col,
                    const int64_t* d_b_ptr, const int64_t* d_m, int64_t* d_ub, int64_t* d_scan_ws,
                    void* stream) {
  if (m < 0) { set_error("spgemm: m < 0"); return GB_ERR_CONTRACT; }
  return device_exclusive_scan<int64_t>(d_m, m, UbF{d_a_ptr, d_a_col, d_b_ptr}, d_ub, d_scan_ws,
                                        (cudaStream_t)stream);
}

size_t gb_scan_workspace_bytes(int64_t max_n) {
  return sizeof(int64_t) * scan_workspace_elems<int64_t>(max_n + 1);
}

int gb_spgemm(int64_t m, const int64_t* d_m, const int64_t* d_a_ptr, const int32_t* d_a_col,
              const double* d_a_val, const int64_t* d_b_ptr, const int32_t* d_b_col,
              const double* d_b_val, const int64_t* d_ub, int64_t ub_total, int32_t* d_gkey,
              double* d_gval, int32_t* d_tmp_col, double* d_tmp_val, int64_t* d_cnt,
              int64_t* d_c_ptr, int32_t* d_c_col, double* d_c_val, int64_t* d_scan_ws,
              void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (m < 0 || ub_total < 0) { set_error("spgemm: bad sizes"); return GB_ERR_CONTRACT; }
  k_spgemm_rows<<<ogrid(m, 1, 8 * kNumSMs), kSpThreads, 0, st>>>(
      m, d_a_ptr, d_a_col, d_a_val, d_b_ptr, d_b_col, d_b_val, d_ub, d_gkey, d_gval, d_tmp_col,
      d_tmp_val, d_cnt);
  GB_LAUNCH_CHECK("k_spgemm_rows");
  int rc = device_exclusive_scan<int64_t>(d_m, m, CntF{d_cnt}, d_c_ptr, d_scan_ws, st);
  if (rc) return rc;
  k_rows_copy<<<ogrid(m, 1, 8 * kNumSMs), 128, 0, st>>>(m, d_ub, d_c_ptr, d_tmp_col, d_tmp_val,
                                                       d_c_col, d_c_val);
  GB_LAUNCH_CHECK("k_rows_copy");
  count_launches(2);
  return GB_OK;
}

int gb_csr_add(int64_t m, const int64_t* d_m, const int64_t* d_a_ptr, const int32_t* d_a_col,
               const double* d_a_val, const int64_t* d_b_ptr, const int32_t* d_b_col,
               const double* d_b_val, int64_t* d_cnt, int64_t* d_c_ptr, int32_t* d_c_col,
               double* d_c_val, int64_t* d_scan_ws, int32_t phase, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (phase == 0) {
    k_add_rows<false><<<ogrid(m, 128, 16 * kNumSMs), 128, 0, st>>>(
        m, d_a_ptr, d_a_col, d_a_val, d_b_ptr, d_b_col, d_b_val, d_cnt, nullptr, nullptr, nullptr);
    GB_LAUNCH_CHECK("k_add_rows");
    count_launches(1);
    return device_exclusive_scan<int64_t>(d_m, m, CntF{d_cnt}, d_c_ptr, d_scan_ws, st);
  }
  k_add_rows<true><<<ogrid(m, 128, 16 * kNumSMs), 128, 0, st>>>(
      m, d_a_ptr, d_a_col, d_a_val, d_b_ptr, d_b_col, d_b_val, nullptr, d_c_ptr, d_c_col, d_c_val);
  GB_LAUNCH_CHECK("k_add_rows");
  count_launches(1);
  return GB_OK;
}

int gb_norm_rows(int64_t m, const int64_t* d_ptr, const double* d_val, int32_t square,
                 double* d_out, int32_t* d_err, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (square)
    k_norm_rows<true><<<ogrid(m, 128, 16 * kNumSMs), 128, 0, st>>>(m, d_ptr, d_val, d_out, d_err);
  else
    k_norm_rows<false><<<ogrid(m, 128, 16 * kNumSMs), 128, 0, st>>>(m, d_ptr, d_val, d_out, d_err);
  GB_LAUNCH_CHECK("k_norm_rows");
  count_launches(1);
  return GB_OK;
}

int gb_its_rows(int64_t m, const int64_t* d_ptr, const double* d_val, int32_t s,
                const int64_t* d_keys, const double* d_inject, uint64_t seed, uint64_t epoch,
                uint64_t depth, double* d_w, double* d_cdf, int32_t* d_picks, int32_t* d_take,
                int32_t* d_err, void* stream) {
  if (s < 1) { set_error("its: s must be >= 1"); return GB_ERR_CONTRACT; }
  k_its_rows<<<ogrid(m, 64, 64 * kNumSMs), 64, 0, (cudaStream_t)stream>>>(
      m, d_ptr, d_val, s, d_keys, d_inject, seed, epoch, depth, d_w, d_cdf, d_picks, d_take,
      d_err);
  GB_LAUNCH_CHECK("k_its_rows");
  count_launches(1);
  return GB_OK;
}

}  // extern "C"
