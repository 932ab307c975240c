// LADIES layer-wise bulk sampling (Alg. 1 with Q^l = one row per batch),
// sm_100a.  Reference: sample_epoch_bulk LADIES path
// (pkg/src/gnnbulk/sampler.py:325-387, 420-462, 475-483).
//
// Per layer, for the k batches at once:
//   P = Q^l A        row i = sum of A rows of batch i's vertex set -> counts
//                    e_v (spgemm sparse.py:233-251 on 0/1 values): dense
//                    per-batch count vectors fed by a warp per gathered row
//                    (atomic accumulate), first touches counted per batch.
//   NORM             w_v = fl(e_v^2 / sum e^2) (norm_rows_ladies
//                    sparse.py:263-286); the sum is an exact int64 reduce.
//   SAMPLE           min(s, N_i) distinct columns per batch:
//                    GB_LADIES_EXACT  — its_sample_row replayed literally
//                      (sequential fp64 cumsum per draw, searchsorted right,
//                      clamp, walk back; sampler.py:176-188) with the keyed
//                      uniforms: bit-exact, O(s N) per batch, small graphs;
//                    GB_LADIES_RACE   — exponential race / Gumbel top-s:
//                      key_v = -log(u_v) / e_v^2, the s smallest keys (radix
//                      select).  Same law as successive sampling without
//                      replacement; validated statistically.
//   EXTRACT          A_S = rows of Q^l (in order) x sampled columns: second
//                    streaming pass over the gathered rows with a per-batch
//                    rank marker (build_column_extraction sparse.py:430-446,
//                    ladies_assemble sampler.py:420-434: shared columns when
//                    every batch took the same count, else block diagonal).
#include "gb_common.cuh"
#include "gb_internal.h"
#include "gb_scan.cuh"

namespace gb {

constexpr int kLadiesThreads = 256;
constexpr int kLadiesSizes = 5;  // per layer: A_S rows, F, A_S nnz, A_S cols, nnz(P)

__device__ __forceinline__ int64_t last_le(const int64_t* a, int64_t n_plus1, int64_t x) {
  // last b in [0, n) with a[b] <= x, a has n+1 monotone entries
  int64_t lo = 0, hi = n_plus1 - 1;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid; else hi = mid;
  }
  return lo;
}

// counts: cnt[i * n + v] += 1 for every v in A[u,:], u in Q_i; nnz_b[i]
// counts first touches (= N_i).  One warp per Q entry.
__global__ void __launch_bounds__(kLadiesThreads) k_ladies_count(
    const int64_t* __restrict__ qoff, int64_t k, const int32_t* __restrict__ qcol,
    const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col, int64_t n,
    int32_t* __restrict__ cnt, int64_t* __restrict__ nnz_b) {
  const int lane = lane_id();
  const int64_t QN = qoff[k];
  for (int64_t q = global_warp(); q < QN; q += grid_warps()) {
    const int64_t i = last_le(qoff, k + 1, q);
    const int32_t u = qcol[q];
    const int64_t a0 = rowptr[u], a1 = rowptr[u + 1];
    int32_t* ci = cnt + i * n;
    int64_t first = 0;
    for (int64_t e = a0 + lane; e < a1; e += 32) {
      const int32_t v = __ldg(col + e);
      if (atomicAdd(ci + v, 1) == 0) ++first;
    }
    first = warp_sum(first);
    if (lane == 0 && first) atomicAdd((unsigned long long*)(nnz_b + i), (unsigned long long)first);
  }
}

// Compaction of the nonzeros of batch i (ascending v): one CTA per batch,
// block-scan over tiles of its n counters; writes (v, e) at poff[i] and
// clears the counters.  Also the exact int64 sum of e^2 per batch.
__global__ void __launch_bounds__(1024) k_ladies_compact(
    int64_t k, int64_t n, int32_t* __restrict__ cnt, const int64_t* __restrict__ poff,
    int32_t* __restrict__ pv, int32_t* __restrict__ pe, int64_t* __restrict__ sumsq) {
  __shared__ int64_t sw[33];
  for (int64_t i = blockIdx.x; i < k; i += gridDim.x) {
    int32_t* ci = cnt + i * n;
    int64_t base = poff[i];
    int64_t sq = 0;
    for (int64_t t0 = 0; t0 < n; t0 += blockDim.x) {
      const int64_t v = t0 + threadIdx.x;
      const int32_t e = v < n ? ci[v] : 0;
      int64_t total;
      const int64_t ex = block_excl_scan<int64_t>(e > 0 ? 1 : 0, sw, total);
      if (e > 0) {
        pv[base + ex] = (int32_t)v;
        pe[base + ex] = e;
        ci[v] = 0;
        sq += (int64_t)e * e;
      }
      base += total;
    }
    int64_t tot;
    block_excl_scan<int64_t>(sq, sw, tot);
    if (threadIdx.x == 0) sumsq[i] = tot;
  }
}

struct LadiesSampleArgs {
  const int64_t* poff;   // k+1 offsets of the P rows' nonzeros
  const int32_t* pv;
  const int32_t* pe;
  const int64_t* sumsq;
  int64_t k;
  int32_t s;
  int64_t batch_offset;
  uint64_t seed, epoch, depth;
  double* scratch_w;     // exact mode: weights / cdf scratch (same layout as pv)
  double* scratch_c;
  int32_t* sel;          // per batch up to s selected positions (k * s)
  int64_t* take;         // per batch count
};

// Exact replay of its_sample_row: one thread per batch (sequential fp64
// cumsum is inherently serial; small graphs only).  Writes the selected
// positions (draw order) into sel[i*s ...].
__global__ void k_ladies_sample_exact(LadiesSampleArgs A) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < A.k;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p0 = A.poff[i], N = A.poff[i + 1] - p0;
    const int64_t take = N < A.s ? N : A.s;
    A.take[i] = take;
    int32_t* sel = A.sel + i * A.s;
    if (N == 0) continue;
    if (take == N) {
      for (int64_t t = 0; t < N; ++t) sel[t] = (int32_t)t;
      continue;
    }
    double* w = A.scratch_w + p0;
    double* cdf = A.scratch_c + p0;
    const double S = (double)A.sumsq[i];
    for (int64_t j = 0; j < N; ++j) {
      const double e = (double)A.pe[p0 + j];
      w[j] = __ddiv_rn(__dmul_rn(e, e), S);
    }
    const uint64_t key = (uint64_t)(A.batch_offset + i);
    int64_t dirty = 0;  // cdf valid below this index
    for (int64_t t = 0; t < take; ++t) {
      double acc = dirty ? cdf[dirty - 1] : 0.0;
      for (int64_t j = dirty; j < N; ++j) {
        acc = __dadd_rn(acc, w[j]);
        cdf[j] = acc;
      }
      const double total = cdf[N - 1];
      const double u = uniform53(A.seed, A.epoch, A.depth, key, (uint64_t)t);
      const double target = __dmul_rn(u, total);
      int64_t idx = upper_bound(cdf, 0, N, target);
      if (idx >= N) idx = N - 1;
      while (w[idx] == 0.0) --idx;
      sel[t] = (int32_t)idx;
      w[idx] = 0.0;
      dirty = idx;
    }
  }
}

// Exponential race: the s smallest key_v = -log(u_v) / e_v^2 (ties by
// position).  Keys are computed once per P nonzero (k_ladies_race_keys);
// one CTA per batch then radix-selects the take smallest with three
// histogram passes (12 + 12 + 8 bits of the float key) and resolves exact
// key ties by position.
__global__ void k_ladies_race_keys(LadiesSampleArgs A, const int64_t* __restrict__ P_ptr,
                                   uint32_t* __restrict__ keys) {
  const int64_t P = *P_ptr;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < P;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = last_le(A.poff, A.k + 1, j);
    const double u = uniform53(A.seed, A.epoch, A.depth | (1ULL << 32),
                               (uint64_t)(A.batch_offset + i), (uint64_t)A.pv[j]);
    const float e = (float)A.pe[j];
    const float x = (float)(-log1p(-u)) / (e * e);  // Exp(1) / weight, non-negative
    keys[j] = __float_as_uint(x);  // non-negative floats order like their bit patterns
  }
}

constexpr int kRaceBins = 4096;
constexpr int kRaceTies = 2048;

__global__ void __launch_bounds__(1024) k_ladies_sample_race(LadiesSampleArgs A,
                                                           const uint32_t* __restrict__ keys,
                                                           int32_t* __restrict__ overflow) {
  __shared__ uint32_t hist[kRaceBins];
  __shared__ int32_t ties[kRaceTies];
  __shared__ int s_sel, s_bin, s_acc, s_tie;
  const int shifts[3] = {20, 8, 0};
  const int widths[3] = {12, 12, 8};
  for (int64_t i = blockIdx.x; i < A.k; i += gridDim.x) {
    const int64_t p0 = A.poff[i], N = A.poff[i + 1] - p0;
    const int64_t take = N < A.s ? N : A.s;
    int32_t* sel = A.sel + i * A.s;
    if (threadIdx.x == 0) A.take[i] = take;
    if (take == N) {
      for (int64_t t = threadIdx.x; t < N; t += blockDim.x) sel[t] = (int32_t)t;
      __syncthreads();
      continue;
    }
    const uint32_t* ki = keys + p0;
    uint32_t prefix = 0, pmask = 0;
    int64_t need = take;
    if (threadIdx.x == 0) s_sel = 0;
    for (int pass = 0; pass < 3; ++pass) {
      const int sh = shifts[pass];
      const uint32_t bm = (1u << widths[pass]) - 1u;
      for (int b = threadIdx.x; b < kRaceBins; b += blockDim.x) hist[b] = 0;
      __syncthreads();
      for (int64_t j = threadIdx.x; j < N; j += blockDim.x) {
        const uint32_t kk = ki[j];
        if ((kk & pmask) == prefix) atomicAdd(&hist[(kk >> sh) & bm], 1u);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        int64_t acc = 0;
        uint32_t b = 0;
        for (; b <= bm; ++b) {
          if (acc + hist[b] >= need) break;
          acc += hist[b];
        }
        s_bin = (int)b;
        s_acc = (int)acc;
      }
      __syncthreads();
      const uint32_t bin = (uint32_t)s_bin;
      for (int64_t j = threadIdx.x; j < N; j += blockDim.x) {
        const uint32_t kk = ki[j];
        if ((kk & pmask) == prefix && ((kk >> sh) & bm) < bin) sel[atomicAdd(&s_sel, 1)] = (int32_t)j;
      }
      need -= s_acc;
      prefix |= bin << sh;
      pmask |= bm << sh;
      __syncthreads();
    }
    // remaining `need` picks among keys exactly equal to prefix: smallest positions
    if (threadIdx.x == 0) s_tie = 0;
    __syncthreads();
    for (int64_t j = threadIdx.x; j < N; j += blockDim.x)
      if (ki[j] == prefix) {
        const int t = atomicAdd(&s_tie, 1);
        if (t < kRaceTies) ties[t] = (int32_t)j; else atomicExch(overflow, 1);
      }
    __syncthreads();
    const int m = min(s_tie, kRaceTies);
    const int base = s_sel;
    for (int a2 = threadIdx.x; a2 < m; a2 += blockDim.x) {
      int rank = 0;
      for (int b2 = 0; b2 < m; ++b2) rank += ties[b2] < ties[a2] ? 1 : 0;
      if (rank < need) sel[base + rank] = ties[a2];
    }
    __syncthreads();
  }
}

// Sort each batch's selected positions ascending (positions ascend with
// vertex id) and emit the frontier row: fcol[fptr[i] + r] = pv[p0 + pos].
__global__ void __launch_bounds__(256) k_ladies_emit(const int64_t* __restrict__ poff,
                                                   const int32_t* __restrict__ pv, int64_t k,
                                                   int32_t s, const int32_t* __restrict__ sel,
                                                   const int64_t* __restrict__ fptr,
                                                   int32_t* __restrict__ fcol) {
  for (int64_t i = blockIdx.x; i < k; i += gridDim.x) {
    const int64_t take = fptr[i + 1] - fptr[i];
    const int32_t* si = sel + i * s;
    for (int64_t a = threadIdx.x; a < take; a += blockDim.x) {
      const int32_t x = si[a];
      int64_t rank = 0;
      for (int64_t b = 0; b < take; ++b) rank += si[b] < x ? 1 : 0;
      fcol[fptr[i] + rank] = pv[poff[i] + x];
    }
  }
}

// marker[i*n + v] = rank + 1 for the sampled vertices (0 elsewhere)
__global__ void k_ladies_mark(const int64_t* __restrict__ fptr, int64_t k, int64_t n,
                              const int32_t* __restrict__ fcol, int32_t* __restrict__ marker,
                              int32_t clear) {
  const int64_t F = fptr[k];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < F;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = last_le(fptr, k + 1, e);
    marker[i * n + fcol[e]] = clear ? 0 : (int32_t)(e - fptr[i] + 1);
  }
}

// A_S row q (batch i, vertex u = qcol[q]): the marked ranks of A[u,:] in
// column order.  COUNT pass writes rcnt[q]; WRITE pass fills acol.
template <bool WRITE>
__global__ void __launch_bounds__(kLadiesThreads) k_ladies_extract(
    const int64_t* __restrict__ qoff, int64_t k, const int32_t* __restrict__ qcol,
    const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col, int64_t n,
    const int32_t* __restrict__ marker, const int64_t* __restrict__ coloff,
    int32_t* __restrict__ rcnt, const int64_t* __restrict__ aptr, int32_t* __restrict__ acol) {
  const unsigned FULL = 0xffffffffu;
  const int lane = lane_id();
  const int64_t QN = qoff[k];
  for (int64_t q = global_warp(); q < QN; q += grid_warps()) {
    const int64_t i = last_le(qoff, k + 1, q);
    const int32_t u = qcol[q];
    const int64_t a0 = rowptr[u], a1 = rowptr[u + 1];
    const int32_t* mi = marker + i * n;
    int64_t o = WRITE ? aptr[q] : 0;
    const int64_t cbase = WRITE ? coloff[i] : 0;
    for (int64_t e0 = a0; e0 < a1; e0 += 32) {
      const int64_t e = e0 + lane;
      const int32_t m = e < a1 ? mi[__ldg(col + e)] : 0;
      const unsigned bal = __ballot_sync(FULL, m > 0);
      if (WRITE && m > 0) acol[o + __popc(bal & ((1u << lane) - 1))] = (int32_t)(cbase + m - 1);
      o += __popc(bal);
    }
    if (!WRITE && lane == 0) rcnt[q] = (int32_t)o;
  }
}

struct RcntF {
  const int32_t* r;
  __device__ int64_t operator()(int64_t i) const { return r[i]; }
};
struct TakeLF {
  const int64_t* t;
  __device__ int64_t operator()(int64_t i) const { return t[i]; }
};
struct NnzF {
  const int64_t* t;
  __device__ int64_t operator()(int64_t i) const { return t[i]; }
};

// shared layout iff every batch took the same count (ladies_assemble)
__global__ void k_ladies_layout(const int64_t* __restrict__ fptr, int64_t k,
                                const int64_t* __restrict__ qoff, const int64_t* __restrict__ aptr,
                                const int64_t* __restrict__ poff,
                                int64_t* __restrict__ coloff, int64_t* __restrict__ sizes) {
  if (threadIdx.x == 0 && blockIdx.x == 0) sizes[4] = poff[k];  // nnz(P)
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  bool shared = true;
  for (int64_t i = 1; i < k; ++i)
    if (fptr[i + 1] - fptr[i] != fptr[1] - fptr[0]) shared = false;
  for (int64_t i = 0; i <= k; ++i) coloff[i] = shared ? 0 : fptr[i];
  const int64_t QN = qoff[k];
  sizes[0] = QN;                                              // A_S rows
  sizes[1] = fptr[k];                                         // F
  sizes[2] = aptr[QN];                                        // A_S nnz
  sizes[3] = k == 0 ? 0 : (shared ? fptr[1] - fptr[0] : fptr[k]);  // A_S cols
}

static int grid_cap(int64_t n, int threads, int cap) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

struct LadiesWs {
  int32_t* cnt;      // k * n
  int64_t* nnz_b;    // k + 1
  int64_t* poff;     // k + 1
  int32_t* pv;       // P nnz cap
  int32_t* pe;
  double* sw;        // exact scratch
  double* sc;
  int64_t* sumsq;    // k
  uint32_t* keys;    // race keys (P nnz cap)
  int32_t* sel;      // k * s_max
  int64_t* take;     // k
  int32_t* rcnt;     // Q cap
  int64_t* scan_ws;
  int64_t* d_k;      // device scalar k
  int32_t* overflow;
  size_t bytes;
};

static size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

static LadiesWs ladies_ws_layout(char* base, int64_t k, int64_t n, int64_t p_cap, int64_t q_cap,
                                 int64_t s_max, bool exact) {
  LadiesWs w{};
  size_t off = 0;
  auto take = [&](size_t bytes) { char* p = base ? base + off : nullptr; off += al(bytes); return p; };
  w.cnt = (int32_t*)take(sizeof(int32_t) * (size_t)(k * n + 1));
  w.nnz_b = (int64_t*)take(sizeof(int64_t) * (k + 1));
  w.poff = (int64_t*)take(sizeof(int64_t) * (k + 1));
  w.pv = (int32_t*)take(sizeof(int32_t) * (p_cap + 1));
  w.pe = (int32_t*)take(sizeof(int32_t) * (p_cap + 1));
  w.sw = (double*)take(exact ? sizeof(double) * (p_cap + 1) : 8);
  w.sc = (double*)take(exact ? sizeof(double) * (p_cap + 1) : 8);
  w.sumsq = (int64_t*)take(sizeof(int64_t) * (k + 1));
  w.keys = (uint32_t*)take(exact ? 8 : sizeof(uint32_t) * (p_cap + 1));
  w.sel = (int32_t*)take(sizeof(int32_t) * (k * s_max + 1));
  w.take = (int64_t*)take(sizeof(int64_t) * (k + 1));
  w.rcnt = (int32_t*)take(sizeof(int32_t) * (q_cap + 1));
  const int64_t sn = q_cap > k ? q_cap : k;
  w.scan_ws = (int64_t*)take(sizeof(int64_t) * scan_workspace_elems<int64_t>(sn + 1));
  w.d_k = (int64_t*)take(sizeof(int64_t));
  w.overflow = (int32_t*)take(sizeof(int32_t));
  w.bytes = off;
  return w;
}

// P nnz capacity: N_i <= min(n, sum of degrees of Q_i) <= n per batch.
static int64_t ladies_p_cap(int64_t k, int64_t n) { return k * n; }

int ladies_workspace(const Graph* g, int64_t k, int64_t q1_cap, int32_t layers,
                     const int64_t* fanouts, int32_t mode, size_t* bytes) {
  int64_t s_max = 1, q_cap = q1_cap;
  for (int32_t l = 0; l < layers; ++l) {
    if (fanouts[l] > s_max) s_max = fanouts[l];
    if (k * fanouts[l] > q_cap) q_cap = k * fanouts[l];
  }
  *bytes = ladies_ws_layout(nullptr, k, g->n, ladies_p_cap(k, g->n), q_cap, s_max,
                            mode == GB_LADIES_EXACT).bytes;
  return GB_OK;
}

__global__ void k_set_i64_l(int64_t* p, int64_t v) { *p = v; }

int ladies_bulk(const Graph* g, int64_t k, const int64_t* d_qoff, const int32_t* d_qverts,
                int64_t q1_cap, int32_t layers, const int64_t* fanouts, uint64_t seed,
                uint64_t epoch, int64_t batch_offset, int32_t mode, gb_ladies_layer_out* L,
                int64_t* d_sizes, void* d_ws, size_t ws_bytes, cudaStream_t st) {
  const bool exact = mode == GB_LADIES_EXACT;
  int64_t s_max = 1, q_cap = q1_cap;
  for (int32_t l = 0; l < layers; ++l) {
    if (fanouts[l] > s_max) s_max = fanouts[l];
    if (k * fanouts[l] > q_cap) q_cap = k * fanouts[l];
  }
  const int64_t n = g->n;
  LadiesWs ws = ladies_ws_layout((char*)d_ws, k, n, ladies_p_cap(k, n), q_cap, s_max, exact);
  if (ws.bytes > ws_bytes) {
    set_error("ladies workspace too small: need %zu bytes, got %zu", ws.bytes, ws_bytes);
    return GB_ERR_CAPACITY;
  }
  int64_t qc = q1_cap;
  for (int32_t l = 0; l < layers; ++l) {
    if (L[l].q_cap < qc || L[l].f_cap < k * fanouts[l] || L[l].a_cap < qc * fanouts[l]) {
      set_error("ladies layer %d output too small", (int)l + 1);
      return GB_ERR_CAPACITY;
    }
    qc = k * fanouts[l];
  }
  GB_CUDA(cudaMemsetAsync(ws.cnt, 0, sizeof(int32_t) * (size_t)(k * n + 1), st));
  GB_CUDA(cudaMemsetAsync(ws.overflow, 0, sizeof(int32_t), st));
  k_set_i64_l<<<1, 1, 0, st>>>(ws.d_k, k);
  count_launches(1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  if (sms <= 0) sms = kNumSMs;
  qc = q1_cap;
  for (int32_t l = 0; l < layers; ++l) {
    const int32_t s = (int32_t)fanouts[l];
    gb_ladies_layer_out& o = L[l];
    const int64_t* qoff = l == 0 ? d_qoff : L[l - 1].fptr;
    const int32_t* qcol = l == 0 ? d_qverts : L[l - 1].fcol;
    const int64_t* d_QN = qoff + k;
    // ---- P = Q A (counts) + first touches
    GB_CUDA(cudaMemsetAsync(ws.nnz_b, 0, sizeof(int64_t) * (k + 1), st));
    prof_mark(st);
    k_ladies_count<<<grid_cap(qc * 32, kLadiesThreads, 16 * sms), kLadiesThreads, 0, st>>>(
        qoff, k, qcol, g->rowptr, g->col, n, ws.cnt, ws.nnz_b);
    GB_LAUNCH_CHECK("k_ladies_count");
    prof_mark(st);
    int rc = device_exclusive_scan<int64_t>(ws.d_k, k, NnzF{ws.nnz_b}, ws.poff, ws.scan_ws, st);
    if (rc) return rc;
    k_ladies_compact<<<(int)(k < 4 * sms ? (k > 0 ? k : 1) : 4 * sms), 1024, 0, st>>>(
        k, n, ws.cnt, ws.poff, ws.pv, ws.pe, ws.sumsq);
    GB_LAUNCH_CHECK("k_ladies_compact");
    // ---- NORM + SAMPLE
    LadiesSampleArgs A{};
    A.poff = ws.poff; A.pv = ws.pv; A.pe = ws.pe; A.sumsq = ws.sumsq; A.k = k; A.s = s;
    A.batch_offset = batch_offset; A.seed = seed; A.epoch = epoch; A.depth = (uint64_t)(l + 1);
    A.scratch_w = ws.sw; A.scratch_c = ws.sc; A.sel = ws.sel; A.take = ws.take;
    if (exact)
      k_ladies_sample_exact<<<grid_cap(k, 32, 4 * sms), 32, 0, st>>>(A);
    else {
      k_ladies_race_keys<<<grid_cap(k * n, 256, 32 * sms), 256, 0, st>>>(A, ws.poff + k, ws.keys);
      k_ladies_sample_race<<<(int)(k < 4 * sms ? (k > 0 ? k : 1) : 4 * sms), 1024, 0, st>>>(
          A, ws.keys, ws.overflow);
      count_launches(1);
    }
    GB_LAUNCH_CHECK("k_ladies_sample");
    rc = device_exclusive_scan<int64_t>(ws.d_k, k, TakeLF{ws.take}, o.fptr, ws.scan_ws, st);
    if (rc) return rc;
    k_ladies_emit<<<(int)(k < 4 * sms ? (k > 0 ? k : 1) : 4 * sms), 256, 0, st>>>(
        ws.poff, ws.pv, k, s, ws.sel, o.fptr, o.fcol);
    GB_LAUNCH_CHECK("k_ladies_emit");
    // ---- EXTRACT A_S = Q_R A Q_C
    const int mgrid = grid_cap(k * s, 256, 16 * sms);
    k_ladies_mark<<<mgrid, 256, 0, st>>>(o.fptr, k, n, o.fcol, ws.cnt, 0);
    const int egrid = grid_cap(qc * 32, kLadiesThreads, 16 * sms);
    k_ladies_extract<false><<<egrid, kLadiesThreads, 0, st>>>(
        qoff, k, qcol, g->rowptr, g->col, n, ws.cnt, nullptr, ws.rcnt, nullptr, nullptr);
    rc = device_exclusive_scan<int64_t>(d_QN, qc, RcntF{ws.rcnt}, o.aptr, ws.scan_ws, st);
    if (rc) return rc;
    k_ladies_layout<<<1, 1, 0, st>>>(o.fptr, k, qoff, o.aptr, ws.poff, o.coloff,
                                     d_sizes + kLadiesSizes * l);
    k_ladies_extract<true><<<egrid, kLadiesThreads, 0, st>>>(
        qoff, k, qcol, g->rowptr, g->col, n, ws.cnt, o.coloff, nullptr, o.aptr, o.acol);
    k_ladies_mark<<<mgrid, 256, 0, st>>>(o.fptr, k, n, o.fcol, ws.cnt, 1);
    GB_LAUNCH_CHECK("k_ladies_extract");
    count_launches(10);
    qc = k * s;
  }
  return GB_OK;
}

}  // namespace gb
