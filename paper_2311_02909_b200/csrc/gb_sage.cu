// GraphSAGE node-wise bulk sampling, Alg. 1 of arXiv 2311.02909
// (P <- Q^l A; NORM; SAMPLE; EXTRACT) for k stacked minibatches, sm_100a.
//
// Reference behaviour reproduced bit for bit (with the injected uniforms of
// gb_common.cuh): sample_epoch_bulk SAGE path, pkg/src/gnnbulk/sampler.py:325-387.
//
//   * Q^l is never built: row r of Q^l is one-hot at rowv[r]
//     (sage_seed_matrix sampler.py:122-127, expand_row_extraction
//     sparse.py:360-370), so row r of P = Q^l A is row rowv[r] of A.
//   * NORM: every entry of P row r is fl(1/deg) (norm_rows_sage,
//     sparse.py:254-286; row sums of 1.0-valued rows are exact).
//   * SAMPLE: its_sample_row (sampler.py:157-189) replayed exactly.  With
//     equal weights w = fl(1/deg) and removed weights contributing exactly
//     0.0, the sequential fp64 cumsum over the live entries is the prefix
//     table S[j] = fl(S[j-1] + w) of the degree alone (SURVEY.md Appendix
//     A.2).  S is stored once per distinct degree as "runs" of constant
//     increment inside one binade, so S[j] and its inverse are O(1) exact
//     look-ups (replay tables, built by gb_graph_create).
//   * EXTRACT (sage_batch_blocks / compact_columns / block_diag,
//     sampler.py:390-417, sparse.py:321-357): per-batch sorted-unique
//     columns via one bit per (batch, vertex), a popcount prefix scan for
//     the block-diagonal renumbering, and an enumerate pass for
//     col_vertices.
//
// Two modes of the SAMPLE kernel, identical outputs:
//   GB_SAGE_STREAM: P row formed on chip — the warp streams the whole A row
//     (coalesced 16-B loads, merge-path balanced over rows+entries) and
//     catches the picked entries out of registers.  This is Alg. 1 with P
//     never written to HBM; its algorithmic bytes are SURVEY.md §8(d).
//   GB_SAGE_PFREE: the P-free fast path: only the picked
//     entries of A are read.
#include <stdarg.h>
#include <stdio.h>

#include "gb_common.cuh"
#include "gb_scan.cuh"
#include "gb_internal.h"

namespace gb {

// ============================================================ replay tables

__global__ void k_degree_max(const int64_t* __restrict__ rowptr, int64_t n,
                             unsigned long long* __restrict__ out_max) {
  int64_t best = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    best = max(best, rowptr[v + 1] - rowptr[v]);
  best = max(best, (int64_t)__reduce_max_sync(0xffffffffu, (unsigned)min(best, (int64_t)0x7fffffff)));
  if ((threadIdx.x & 31) == 0) atomicMax(out_max, (unsigned long long)best);
}

__global__ void k_degree_flags(const int64_t* __restrict__ rowptr, int64_t n,
                               int32_t* __restrict__ flags) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    int64_t d = rowptr[v + 1] - rowptr[v];
    if (d >= 2) flags[d] = 1;
  }
}

struct FlagF {
  const int32_t* flags;
  __device__ int64_t operator()(int64_t i) const { return flags[i]; }
};

__global__ void k_degree_slots(const int32_t* __restrict__ flags, const int64_t* __restrict__ pre,
                               int64_t nd, int32_t* __restrict__ deg_slot,
                               int32_t* __restrict__ slot_deg) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < nd;
       d += (int64_t)gridDim.x * blockDim.x) {
    if (flags[d]) {
      deg_slot[d] = (int32_t)pre[d];
      slot_deg[pre[d]] = (int32_t)d;
    } else {
      deg_slot[d] = -1;
    }
  }
}

__device__ __forceinline__ uint64_t binade(double x) {
  return (uint64_t)__double_as_longlong(x) >> 52;
}

// One thread per distinct degree m: walk S[j] = fl(S[j-1] + fl(1/m)),
// j = 1..m, exactly as numpy's sequential cumsum does, and cut it into runs
// of constant increment inside one binade.
// Also the binade index lower[b] = number of runs whose start lies more than
// b binades below the top run's binade, so the run holding a target value
// is found in O(1) (gt_first_gt).
__global__ void k_build_runs(const int32_t* __restrict__ slot_deg, int64_t slots,
                             int32_t* __restrict__ run_j0, double* __restrict__ run_s0,
                             double* __restrict__ run_d, int32_t* __restrict__ run_n,
                             int8_t* __restrict__ run_lower, int32_t* __restrict__ overflow) {
  for (int64_t sl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sl < slots;
       sl += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = slot_deg[sl];
    const double w = 1.0 / (double)m;
    int32_t* J = run_j0 + sl * (kMaxRuns + 1);
    double* S0 = run_s0 + sl * kMaxRuns;
    double* D = run_d + sl * kMaxRuns;
    int nr = 0;
    int64_t j0 = 1, len = 1;
    double s0 = w, d = 0.0, S = w;
    bool bad = false;
    for (int64_t j = 2; j <= m; ++j) {
      const double S2 = __dadd_rn(S, w);
      const double step = __dadd_rn(S2, -S);
      if (len == 1 && binade(S2) == binade(s0)) {
        d = step;
        len = 2;
      } else if (len >= 2 && step == d && binade(S2) == binade(s0)) {
        ++len;
      } else {
        if (nr < kMaxRuns) { J[nr] = (int32_t)j0; S0[nr] = s0; D[nr] = d; } else bad = true;
        ++nr;
        j0 = j; s0 = S2; len = 1; d = 0.0;
      }
      S = S2;
    }
    if (nr < kMaxRuns) { J[nr] = (int32_t)j0; S0[nr] = s0; D[nr] = d; } else bad = true;
    ++nr;
    if (nr <= kMaxRuns) J[nr] = (int32_t)(m + 1);  // sentinel
    run_n[sl] = nr;
    if (!bad) {
      const int64_t top = (int64_t)binade(S0[nr - 1]);
      int8_t* low = run_lower + sl * kBinades;
      for (int b = 0; b < kBinades; ++b) {
        int c = 0;
        for (int r = 0; r < nr; ++r) c += (top - (int64_t)binade(S0[r]) > b) ? 1 : 0;
        low[b] = (int8_t)c;
      }
    }
    if (bad) atomicExch(overflow, 1);
  }
}

// ============================================================ layer kernels

__global__ void k_sage_prep(const int64_t* __restrict__ R_ptr, const int32_t* __restrict__ rowv,
                            const int64_t* __restrict__ rowptr, int32_t* __restrict__ deg) {
  const int64_t R = *R_ptr;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = rowv[r];
    deg[r] = (int32_t)(rowptr[v + 1] - rowptr[v]);
  }
}

struct TakeF {
  const int32_t* deg;
  int32_t s;
  __device__ int64_t operator()(int64_t i) const { return min(deg[i], s); }
};
struct DegF {
  const int32_t* deg;
  __device__ int64_t operator()(int64_t i) const { return deg[i]; }
};

struct SageArgs {
  const int64_t* rowptr;
  const int32_t* col;
  const int32_t* deg_slot;
  const int32_t* run_j0;
  const double* run_s0;
  const double* run_d;
  const int32_t* run_n;
  const int8_t* run_lower;
  const int32_t* rowv;
  const int64_t* rowkeys;  // optional explicit global row keys (owner-computes 1.5D)
  const int32_t* deg;
  const int64_t* fptr;
  const int64_t* gstart;
  const int64_t* brow;   // k + 1
  int64_t k;
  int32_t s;
  int64_t stride;
  int64_t batch_offset;
  uint64_t seed, epoch, depth;
  uint32_t* bitmap;
  int64_t nwords;
  int32_t* fcol;         // frontier columns (output)
  int32_t* pidx;         // stream mode: row-relative pick indices (scratch)
  // dedup mode: pick records grouped by distinct row vertex
  const uint32_t* vbits;
  const int32_t* vpre;
  const int64_t* goff;
  int32_t* gcur;
  uint64_t* pk;
  int32_t* pkb;
};

__device__ __forceinline__ int32_t vrank(const uint32_t* vbits, const int32_t* vpre, int32_t v) {
  return vpre[v >> 5] + __popc(vbits[v >> 5] & ((1u << (v & 31)) - 1u));
}

constexpr int kPickThreads = 128;
constexpr int kStreamThreads = 256;
constexpr int kRowCost = 48;       // merge-path weight of one row (in entries)
constexpr int kStreamUnroll = 8;   // 16-B loads in flight per lane
constexpr int kBrowSmem = 1024;
constexpr int kMaxFan = 32;

__device__ __forceinline__ int4 ld_stream_v4(const int32_t* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ int64_t batch_of(const int64_t* sb, const int64_t* gb_, int64_t k,
                                            int64_t r) {
  // last b with brow[b] <= r
  const int64_t* a = k + 1 <= kBrowSmem ? sb : gb_;
  int64_t lo = 0, hi = k;
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] <= r) lo = mid; else hi = mid;
  }
  return lo;
}

// Replay table of one degree read through the read-only path (L1-resident:
// ~1.4 KB per hot degree) with its binade index.
struct GTable {
  const int32_t* j0;
  const double* s0;
  const double* d;
  const int8_t* lower;
  int nr;
  uint64_t top;  // binade of the last run's start
};

// S[n], 1 <= n <= m: n_live is near m, so scan back from the last run
__device__ __forceinline__ double gt_S(const GTable& t, int64_t n) {
  int r = t.nr - 1;
  int32_t j0 = __ldg(t.j0 + r);
  while (j0 > n) j0 = __ldg(t.j0 + --r);
  return __dadd_rn(__ldg(t.s0 + r), __dmul_rn((double)(n - j0), __ldg(t.d + r)));
}

// first j >= 1 with S[j] > target (m + 1 when none).  The run is located by
// the binade index (O(1)), the position inside it by a float estimate that
// the exact fp64 comparisons then correct.
__device__ __forceinline__ int64_t gt_first_gt(const GTable& t, double target) {
  if (target < __ldg(t.s0)) return 1;
  const int64_t off = (int64_t)t.top - (int64_t)binade(target);
  int r = off < 0 ? t.nr : (int)__ldg(t.lower + (off < kBinades ? off : kBinades - 1));
  // r = first run starting in target's binade or above; step back / forward
  if (r >= t.nr || __ldg(t.s0 + r) > target) {
    r = r - 1;
  } else {
    while (r + 1 < t.nr && __ldg(t.s0 + r + 1) <= target) ++r;
  }
  const int64_t j0 = __ldg(t.j0 + r);
  const int64_t len = (int64_t)__ldg(t.j0 + r + 1) - j0;
  if (len == 1) return j0 + 1;
  const double s0 = __ldg(t.s0 + r), d = __ldg(t.d + r);
  int64_t q = (int64_t)__fdividef((float)(target - s0), (float)d);
  q = q < 0 ? 0 : (q > len - 1 ? len - 1 : q);
  while (q > 0 && __dadd_rn(s0, __dmul_rn((double)q, d)) > target) --q;
  while (q + 1 < len && __dadd_rn(s0, __dmul_rn((double)(q + 1), d)) <= target) ++q;
  return j0 + q + 1;
}

// NORM + SAMPLE, one thread per P row.  Draw t of row r uses
// u = uniform53(seed, epoch, depth, key_r, t); n_live = deg - t live entries
// of weight fl(1/deg); target = u * S[n_live]; the draw selects the j-th live
// entry, j = first j with S[j] > target clamped to n_live — exactly
// its_sample_row's cumsum/searchsorted/clamp/walk-back (sampler.py:176-188).
// Picks are kept sorted (frontier_from_rows sorts, sampler.py:216) in
// registers (MAXF = fanout bucket, fully unrolled).
// OUT 1 (P-free): read the picked columns of A directly and finish the row;
// OUT 0: write the row-relative indices for the row-streaming kernel;
// OUT 2 (dedup): write pick records straight into the row's vertex group.
template <int OUT, int MAXF>
__global__ void __launch_bounds__(kPickThreads) k_sage_pick(SageArgs A,
                                                          const int64_t* __restrict__ R_ptr) {
  __shared__ int64_t s_brow[kBrowSmem];
  const int64_t R = *R_ptr;
  const bool keyed = A.rowkeys != nullptr;  // explicit keys: no batch structure
  const bool brow_in_smem = !keyed && A.k + 1 <= kBrowSmem;
  if (brow_in_smem)
    for (int64_t i = threadIdx.x; i <= A.k; i += blockDim.x) s_brow[i] = A.brow[i];
  __syncthreads();
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t deg = A.deg[r];
    if (deg == 0) continue;  // empty P row (sample_rows_ordered, sampler.py:202-204)
    const int32_t take = min(deg, A.s);
    const int64_t fp = A.fptr[r];
    const int64_t bb = keyed ? 0 : batch_of(s_brow, A.brow, A.k, r);
    int32_t sorted[MAXF];
#pragma unroll
    for (int q = 0; q < MAXF; ++q) sorted[q] = q;  // exhaustion: every index (sampler.py:172-174)
    if (take < deg) {
      // global_row_keys (sampler.py:309-322), or the requester's keys
      uint64_t key;
      if (keyed) {
        key = (uint64_t)A.rowkeys[r];
      } else {
        const int64_t b0 = brow_in_smem ? s_brow[bb] : A.brow[bb];
        key = (uint64_t)((A.batch_offset + bb) * A.stride + (r - b0));
      }
      const int32_t slot = __ldg(A.deg_slot + deg);
      GTable tab;
      tab.j0 = A.run_j0 + (int64_t)slot * (kMaxRuns + 1);
      tab.s0 = A.run_s0 + (int64_t)slot * kMaxRuns;
      tab.d = A.run_d + (int64_t)slot * kMaxRuns;
      tab.lower = A.run_lower + (int64_t)slot * kBinades;
      tab.nr = __ldg(A.run_n + slot);
      tab.top = binade(__ldg(tab.s0 + tab.nr - 1));
      uint64_t w0 = 0, w1 = 0, w2 = 0, w3 = 0;
      for (int t = 0; t < take; ++t) {
        if ((t & 3) == 0) {
          w0 = key; w1 = A.depth; w2 = (uint64_t)(t >> 2); w3 = 0;
          philox4x64_10(w0, w1, w2, w3, A.seed, A.epoch);
        }
        const uint64_t w = (t & 3) == 0 ? w0 : (t & 3) == 1 ? w1 : (t & 3) == 2 ? w2 : w3;
        const double u = (double)(w >> 11) * 0x1.0p-53;
        const int64_t n_live = deg - t;
        const double target = __dmul_rn(u, gt_S(tab, n_live));
        int64_t j = gt_first_gt(tab, target);
        if (j > n_live) j = n_live;
        // j-th live index: skip over the removed (sorted) ones, then insert
        int32_t x = (int32_t)(j - 1);
        int i = 0;
#pragma unroll
        for (int q = 0; q < MAXF; ++q)
          if (q < t && sorted[q] <= x) { ++x; ++i; }
#pragma unroll
        for (int q = MAXF - 1; q > 0; --q)
          if (q > i && q <= t) sorted[q] = sorted[q - 1];
#pragma unroll
        for (int q = 0; q < MAXF; ++q)
          if (q == i) sorted[q] = x;
      }
    }
    if (OUT == 1) {
      const int64_t rs = A.rowptr[A.rowv[r]];
      int32_t cv[MAXF];
#pragma unroll
      for (int q = 0; q < MAXF; ++q)
        if (q < take) cv[q] = __ldg(A.col + rs + sorted[q]);
#pragma unroll
      for (int q = 0; q < MAXF; ++q)
        if (q < take) A.fcol[fp + q] = cv[q];
      if (A.bitmap) {
        uint32_t* bm = A.bitmap + bb * A.nwords;
#pragma unroll
        for (int q = 0; q < MAXF; ++q)
          if (q < take) atomicOr(bm + (cv[q] >> 5), 1u << (cv[q] & 31));
      }
    } else if (OUT == 2) {
      const int32_t g = vrank(A.vbits, A.vpre, A.rowv[r]);
      // rows of one vertex have the same degree, hence the same take:
      // one cursor atomic per vertex per warp (hub groups are hot)
      const unsigned act = __activemask();
      const unsigned peers = __match_any_sync(act, g);
      const int lane = lane_id(), leader = __ffs(peers) - 1;
      int32_t cur = 0;
      if (lane == leader) cur = atomicAdd(A.gcur + g, take * __popc(peers));
      cur = __shfl_sync(peers, cur, leader);
      const int64_t base = A.goff[g] + cur + take * __popc(peers & ((1u << lane) - 1u));
#pragma unroll
      for (int q = 0; q < MAXF; ++q)
        if (q < take) {
          A.pk[base + q] = ((uint64_t)(uint32_t)sorted[q] << 32) | (uint64_t)(fp + q);
          A.pkb[base + q] = (int32_t)bb;
        }
    } else {
#pragma unroll
      for (int q = 0; q < MAXF; ++q)
        if (q < take) A.pidx[fp + q] = sorted[q];
    }
  }
}

template <int OUT>
static void launch_pick(int grid, const SageArgs& A, const int64_t* R_ptr, cudaStream_t st) {
  if (A.s <= 8)
    k_sage_pick<OUT, 8><<<grid, kPickThreads, 0, st>>>(A, R_ptr);
  else if (A.s <= 16)
    k_sage_pick<OUT, 16><<<grid, kPickThreads, 0, st>>>(A, R_ptr);
  else
    k_sage_pick<OUT, 32><<<grid, kPickThreads, 0, st>>>(A, R_ptr);
}

// Q^l A with the P row formed on chip: warps stream every A row of the
// layer (16-B coalesced loads, kStreamUnroll in flight per lane), balanced
// by merge path over (rows x kRowCost + gathered entries), and catch the
// picked entries (row-relative indices from k_sage_pick) out of registers.
__global__ void __launch_bounds__(kStreamThreads, 4) k_sage_stream(SageArgs A,
                                                              const int64_t* __restrict__ R_ptr) {
  __shared__ int64_t s_brow[kBrowSmem];
  const unsigned FULL = 0xffffffffu;
  const int64_t R = *R_ptr;
  const bool brow_in_smem = A.k + 1 <= kBrowSmem;
  if (brow_in_smem)
    for (int64_t i = threadIdx.x; i <= A.k; i += blockDim.x) s_brow[i] = A.brow[i];
  __syncthreads();
  const int lane = lane_id();
  const int64_t NW = grid_warps(), w = global_warp();
  const int64_t G = A.gstart[R];
  const int64_t total = R * kRowCost + G;
  const int64_t share = (total + NW - 1) / NW;
  const int64_t path_a = min(w * share, total);
  const int64_t path_b = min(path_a + share, total);
  if (path_a >= path_b) return;
  // last r with P_r <= path_a, P_r = r * kRowCost + gstart[r]
  int64_t lo = 0, hi = R;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (mid * kRowCost + A.gstart[mid] <= path_a) lo = mid; else hi = mid;
  }
  const int64_t r_begin = lo;
  lo = r_begin;
  hi = R;  // first r with P_r >= path_b
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (mid * kRowCost + A.gstart[mid] >= path_b) hi = mid; else lo = mid + 1;
  }
  const int64_t r_end = lo;
  for (int64_t rb = r_begin; rb < r_end; rb += 32) {
    const int64_t r = rb + lane;
    int32_t deg = 0;
    int64_t fp = 0, rs = 0, gs = 0, bb = 0;
    if (r < r_end) {
      deg = A.deg[r];
      fp = A.fptr[r];
      rs = A.rowptr[A.rowv[r]];
      gs = A.gstart[r];
      bb = batch_of(s_brow, A.brow, A.k, r);
    }
    const int nrows = (int)min((int64_t)32, r_end - rb);
    for (int i = 0; i < nrows; ++i) {
      const int32_t d_i = __shfl_sync(FULL, deg, i);
      if (d_i == 0) continue;
      const int64_t pe = (rb + i) * kRowCost + __shfl_sync(FULL, gs, i) + kRowCost;
      const int64_t e0 = max(path_a - pe, (int64_t)0);
      const int64_t e1 = min(path_b - pe, (int64_t)d_i);
      if (e0 >= e1) continue;
      const int32_t take = min(d_i, A.s);
      const int64_t fp_i = __shfl_sync(FULL, fp, i);
      const int64_t rs_i = __shfl_sync(FULL, rs, i);
      const int64_t b_i = __shfl_sync(FULL, bb, i);
      const int32_t myidx = lane < take ? A.pidx[fp_i + lane] : -1;
      const int64_t e_lo = rs_i + e0, e_hi = rs_i + e1;
      const int64_t pabs = rs_i + myidx;
      const bool want = lane < take && pabs >= e_lo && pabs < e_hi;
      int32_t c = 0;
      bool have = false;
      for (int64_t w0 = e_lo & ~3LL; w0 < e_hi; w0 += 128 * kStreamUnroll) {
        int4 vals[kStreamUnroll];
#pragma unroll
        for (int u = 0; u < kStreamUnroll; ++u) {
          const int64_t e = w0 + 128 * u + 4 * lane;
          vals[u] = e < e_hi ? ld_stream_v4(A.col + e) : make_int4(0, 0, 0, 0);
        }
        const int64_t off = pabs - w0;
        const bool mine = want && off >= 0 && off < 128 * kStreamUnroll;
        if (__any_sync(FULL, mine)) {
#pragma unroll
          for (int u = 0; u < kStreamUnroll; ++u) {
            const int64_t o = off - 128 * u;
            const bool in_u = mine && o >= 0 && o < 128;
            if (__any_sync(FULL, in_u)) {
              const int src = (int)((o >> 2) & 31);
              const int comp = (int)(o & 3);
              const int x = __shfl_sync(FULL, vals[u].x, src);
              const int y = __shfl_sync(FULL, vals[u].y, src);
              const int z = __shfl_sync(FULL, vals[u].z, src);
              const int ww = __shfl_sync(FULL, vals[u].w, src);
              if (in_u) {
                c = comp == 0 ? x : comp == 1 ? y : comp == 2 ? z : ww;
                have = true;
              }
            }
          }
        }
      }
      if (have) {
        A.fcol[fp_i + lane] = c;
        if (A.bitmap) atomicOr(&A.bitmap[b_i * A.nwords + (c >> 5)], 1u << (c & 31));
      }
    }
  }
}

// ============================================ deduplicated P rows (GB_SAGE_DEDUP)
// Frontier rows repeat vertices heavily (hub bias: 3.5M rows over 0.55M
// distinct vertices in layer 3 at products scale), and identical rows of
// Q^l give identical rows of P = Q^l A.  Each distinct P row is formed on
// chip once — the A row streamed through shared memory — and serves the
// picks of every frontier row that references it.

// one bit per vertex that some row of the layer references
__global__ void k_dd_mark(const int64_t* __restrict__ R_ptr, const int32_t* __restrict__ rowv,
                          const int32_t* __restrict__ deg, uint32_t* __restrict__ vbits) {
  const int64_t R = *R_ptr;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x)
    if (deg[r] > 0) {
      const int32_t v = rowv[r];
      atomicOr(vbits + (v >> 5), 1u << (v & 31));
    }
}

// distinct vertex list (ascending) and its degrees
__global__ void k_dd_list(int64_t nwords, const uint32_t* __restrict__ vbits,
                          const int32_t* __restrict__ vpre, const int64_t* __restrict__ rowptr,
                          int32_t* __restrict__ dv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nwords;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t x = vbits[i];
    int32_t o = vpre[i];
    while (x) {
      const int bit = __ffs(x) - 1;
      dv[o++] = (int32_t)(i * 32 + bit);
      x &= x - 1;
    }
  }
}

// picks per distinct vertex
__global__ void k_dd_count(const int64_t* __restrict__ R_ptr, const int32_t* __restrict__ rowv,
                           const int32_t* __restrict__ deg, int32_t s,
                           const uint32_t* __restrict__ vbits, const int32_t* __restrict__ vpre,
                           int32_t* __restrict__ gcnt) {
  const int64_t R = *R_ptr;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t d = deg[r];
    if (d > 0) {
      const int32_t g = vrank(vbits, vpre, rowv[r]);
      const unsigned act = __activemask();
      const unsigned peers = __match_any_sync(act, g);  // same vertex -> same take
      if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(gcnt + g, min(d, s) * __popc(peers));
    }
  }
}

struct GcntF {
  const int32_t* c;
  __device__ int64_t operator()(int64_t i) const { return c[i]; }
};

// pick records of every row into its vertex group: (row-relative index,
// frontier position), packed as idx << 32 | pos
__global__ void k_dd_scatter(const int64_t* __restrict__ R_ptr, const int32_t* __restrict__ rowv,
                             const int32_t* __restrict__ deg, int32_t s,
                             const int64_t* __restrict__ fptr, const int32_t* __restrict__ pidx,
                             const uint32_t* __restrict__ vbits, const int32_t* __restrict__ vpre,
                             const int64_t* __restrict__ goff, int32_t* __restrict__ gcur,
                             uint64_t* __restrict__ pk, int32_t* __restrict__ pkb,
                             const int64_t* __restrict__ brow, int64_t k) {
  const int64_t R = *R_ptr;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t d = deg[r];
    if (d <= 0) continue;
    const int32_t take = min(d, s);
    const int32_t g = vrank(vbits, vpre, rowv[r]);
    const int64_t base = goff[g] + atomicAdd(gcur + g, take);
    const int64_t fp = fptr[r];
    int64_t lo = 0, hi = k;  // batch of row r (carried with the picks)
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(brow + mid) <= r) lo = mid; else hi = mid;
    }
    for (int t = 0; t < take; ++t) {
      pk[base + t] = ((uint64_t)(uint32_t)pidx[fp + t] << 32) | (uint64_t)(fp + t);
      pkb[base + t] = (int32_t)lo;
    }
  }
}

// Size tiers of distinct rows (degree d): 0 warp per row (d <= 1K, 4 KB
// stage), 1 CTA-256 per row (d <= 8K, 32 KB stage), 2 CTA-1024 per row
// (hubs, 192 KB stage, <= 4 passes over the row's picks at products scale).
constexpr int kDdThreads = 256;
constexpr int kDdUnroll = 4;  // 16-B loads in flight per thread while staging
template <int T> struct DdTier;
template <> struct DdTier<0> {
  static constexpr int kChunk = 1024, kThreads = 256, kLo = 0, kHi = 1024, kPicks = 0;
  static constexpr bool kWarp = true;
};
template <> struct DdTier<1> {
  static constexpr int kChunk = 8192, kThreads = 256, kLo = 1024, kHi = 8192, kPicks = 2048;
  static constexpr bool kWarp = false;
};
template <> struct DdTier<2> {
  static constexpr int kChunk = 49152, kThreads = 1024, kLo = 8192, kHi = 0x7fffffff, kPicks = 8192;
  static constexpr bool kWarp = false;
};

// work items of a CTA tier: ceil(picks / kPicks) per distinct row of the tier
template <int T>
struct ItemF {
  const int32_t* dv;
  const int64_t* rowptr;
  const int64_t* goff;
  __device__ int64_t operator()(int64_t g) const {
    const int32_t v = dv[g];
    const int64_t d = rowptr[v + 1] - rowptr[v];
    if (d <= DdTier<T>::kLo || d > DdTier<T>::kHi) return 0;
    const int64_t p = goff[g + 1] - goff[g];
    return (p + DdTier<T>::kPicks - 1) / DdTier<T>::kPicks;
  }
};
constexpr int kDdWarpChunk = 1024;

__device__ __forceinline__ void dd_emit(int32_t c, uint64_t rec, int32_t batch, int32_t* fcol,
                                        uint32_t* bitmap, int64_t nwords) {
  fcol[(int64_t)(rec & 0xffffffffu)] = c;
  atomicOr(bitmap + (int64_t)batch * nwords + (c >> 5), 1u << (c & 31));
}

// Stream every distinct A row once and serve its picks; TIER selects the
// row sizes handled and warp / CTA granularity.
template <int TIER>
__global__ void __launch_bounds__(DdTier<TIER>::kThreads) k_dd_stream(
    const int64_t* __restrict__ D_ptr, const int32_t* __restrict__ dv,
    const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
    const int64_t* __restrict__ goff, const uint64_t* __restrict__ pk,
    const int32_t* __restrict__ pkb, int32_t* __restrict__ fcol,
    uint32_t* __restrict__ bitmap, int64_t nwords, const int64_t* __restrict__ ioff) {
  constexpr bool LARGE = !DdTier<TIER>::kWarp;
  constexpr int kChunk = DdTier<TIER>::kChunk;
  constexpr int kSlotLen = kChunk + 4;
  extern __shared__ __align__(16) int32_t sdyn[];  // [slots][kSlotLen]
  const int64_t D = *D_ptr;
  const int lane = lane_id();
  const int tid = LARGE ? threadIdx.x : lane;
  const int nthr = LARGE ? blockDim.x : 32;
  int32_t* buf = sdyn + (LARGE ? 0 : (threadIdx.x >> 5) * kSlotLen);
  const int64_t first = LARGE ? blockIdx.x : global_warp();
  const int64_t step = LARGE ? gridDim.x : grid_warps();
  // warp tier: one distinct row per warp; CTA tiers: work items of at most
  // kPicks picks of one row (item prefix ioff over the rows of the tier)
  const int64_t nitems = LARGE ? ioff[D] : D;
  for (int64_t it = first; it < nitems; it += step) {
    int64_t g = it, p0, p1;
    if (LARGE) {
      int64_t lo = 0, hi = D;  // last g with ioff[g] <= it
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (ioff[mid] <= it) lo = mid; else hi = mid;
      }
      g = lo;
      p0 = goff[g] + (it - ioff[g]) * DdTier<TIER>::kPicks;
      p1 = min(p0 + (int64_t)DdTier<TIER>::kPicks, goff[g + 1]);
    } else {
      p0 = goff[g];
      p1 = goff[g + 1];
    }
    const int32_t v = dv[g];
    const int64_t a0 = rowptr[v], d = rowptr[v + 1] - a0;
    if (d <= DdTier<TIER>::kLo || d > DdTier<TIER>::kHi) continue;
    for (int64_t c0 = 0; c0 < d; c0 += kChunk) {
      const int64_t c1 = min(c0 + (int64_t)kChunk, d);
      // stage entries [c0, c1) of A row v: the P row on chip (16-B aligned
      // vector loads, kDdUnroll in flight per thread)
      const int64_t e0 = a0 + c0, e1 = a0 + c1;
      const int64_t al0 = e0 & ~3LL;
      for (int64_t eb = al0 + 4 * tid; eb < e1; eb += 4 * nthr * kDdUnroll) {
        int4 x[kDdUnroll];
#pragma unroll
        for (int u = 0; u < kDdUnroll; ++u) {
          const int64_t e = eb + 4 * nthr * u;
          x[u] = e < e1 ? ld_stream_v4(col + e) : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < kDdUnroll; ++u) {
          const int64_t e = eb + 4 * nthr * u;
          const int64_t o = e - e0;  // may be -3..-1 for the aligned head
          if (o + 0 >= 0 && e + 0 < e1) buf[o + 0] = x[u].x;
          if (o + 1 >= 0 && e + 1 < e1) buf[o + 1] = x[u].y;
          if (o + 2 >= 0 && e + 2 < e1) buf[o + 2] = x[u].z;
          if (o + 3 >= 0 && e + 3 < e1) buf[o + 3] = x[u].w;
        }
      }
      if (LARGE) __syncthreads(); else __syncwarp();
      for (int64_t p = p0 + tid; p < p1; p += nthr) {
        const uint64_t rec = pk[p];
        const int64_t idx = (int64_t)(rec >> 32);
        if (idx >= c0 && idx < c1) dd_emit(buf[idx - c0], rec, pkb[p], fcol, bitmap, nwords);
      }
      if (LARGE) __syncthreads(); else __syncwarp();
    }
  }
}

// ============================================================== extraction

struct PopF {
  const uint32_t* bitmap;
  __device__ int64_t operator()(int64_t i) const { return __popc(bitmap[i]); }
};

// eoff[b] = fptr[brow[b]] (entry offsets per batch = next layer's batch row
// offsets); coloff[b] = wpre[b * nwords]; sizes = (R, F, U)
__global__ void k_sage_layer_meta(const int64_t* __restrict__ brow, int64_t k,
                                  const int64_t* __restrict__ fptr,
                                  const int32_t* __restrict__ wpre, int64_t nwords,
                                  int64_t* __restrict__ eoff, int64_t* __restrict__ coloff,
                                  int64_t* __restrict__ sizes) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b <= k;
       b += (int64_t)gridDim.x * blockDim.x) {
    eoff[b] = fptr[brow[b]];
    coloff[b] = wpre[b * nwords];
    if (b == k) {
      sizes[0] = brow[k];
      sizes[1] = fptr[brow[k]];
      sizes[2] = wpre[k * nwords];
    }
  }
}

// acol[e] = block-diagonal column of frontier entry e:
//   coloff[batch] + rank of fcol[e] among the batch's sorted unique columns
// (compact_columns sparse.py:352-357 + block_diag sparse.py:321-342)
__global__ void k_sage_rank(const int64_t* __restrict__ F_ptr, const int64_t* __restrict__ eoff,
                            int64_t k, const int32_t* __restrict__ fcol,
                            const uint32_t* __restrict__ bitmap, const int32_t* __restrict__ wpre,
                            int64_t nwords, int32_t* __restrict__ acol) {
  __shared__ int64_t s_eoff[kBrowSmem];
  const bool sm = k + 1 <= kBrowSmem;
  if (sm)
    for (int64_t i = threadIdx.x; i <= k; i += blockDim.x) s_eoff[i] = eoff[i];
  __syncthreads();
  const int64_t F = *F_ptr;
  const int64_t* eo = sm ? s_eoff : eoff;
  int64_t lo = -1;  // batch of e: binary search once, then walk forward (e increases)
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < F;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (lo < 0) {
      int64_t a = 0, b = k;
      while (b - a > 1) {
        const int64_t mid = (a + b) >> 1;
        if (eo[mid] <= e) a = mid; else b = mid;
      }
      lo = a;
    } else {
      while (lo + 1 < k && eo[lo + 1] <= e) ++lo;
    }
    const int32_t v = fcol[e];
    const int64_t wi = lo * nwords + (v >> 5);
    const uint32_t mask = (1u << (v & 31)) - 1u;
    acol[e] = wpre[wi] + __popc(bitmap[wi] & mask);
  }
}

// col_vertices: enumerate set bits in (batch, vertex) order; clears the map.
__global__ void k_sage_enumerate(int64_t W, int64_t nwords, uint32_t* __restrict__ bitmap,
                                 const int32_t* __restrict__ wpre, int32_t* __restrict__ colv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < W;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t x = bitmap[i];
    if (!x) continue;
    const int64_t b = i / nwords;
    const int32_t vb = (int32_t)((i - b * nwords) << 5);
    int32_t o = wpre[i];
    while (x) {
      const int bit = __ffs(x) - 1;
      colv[o++] = vb + bit;
      x &= x - 1;
    }
    bitmap[i] = 0;
  }
}

__global__ void k_set_i64(int64_t* p, int64_t v) { *p = v; }

// ===================================================================== host

static int grid_for(int64_t n, int threads, int cap_blocks) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap_blocks) g = cap_blocks;
  return (int)g;
}

int graph_build_tables(Graph* g, cudaStream_t st) {
  // max degree
  unsigned long long* d_max = nullptr;
  GB_CUDA(cudaMallocAsync(&d_max, sizeof(unsigned long long), st));
  GB_CUDA(cudaMemsetAsync(d_max, 0, sizeof(unsigned long long), st));
  k_degree_max<<<grid_for(g->n, 256, 4 * kNumSMs), 256, 0, st>>>(g->rowptr, g->n, d_max);
  GB_LAUNCH_CHECK("k_degree_max");
  unsigned long long h_max = 0;
  GB_CUDA(cudaMemcpyAsync(&h_max, d_max, sizeof(h_max), cudaMemcpyDeviceToHost, st));
  GB_CUDA(cudaStreamSynchronize(st));
  g->max_deg = (int64_t)h_max;
  const int64_t nd = g->max_deg + 1;
  int32_t* flags = nullptr;
  int64_t* pre = nullptr;
  int64_t* scan_ws = nullptr;
  int64_t* d_nd = nullptr;
  GB_CUDA(cudaMallocAsync(&flags, sizeof(int32_t) * nd, st));
  GB_CUDA(cudaMallocAsync(&pre, sizeof(int64_t) * (nd + 1), st));
  GB_CUDA(cudaMallocAsync(&scan_ws, sizeof(int64_t) * scan_workspace_elems<int64_t>(nd), st));
  GB_CUDA(cudaMallocAsync(&d_nd, sizeof(int64_t), st));
  GB_CUDA(cudaMemsetAsync(flags, 0, sizeof(int32_t) * nd, st));
  k_set_i64<<<1, 1, 0, st>>>(d_nd, nd);
  k_degree_flags<<<grid_for(g->n, 256, 8 * kNumSMs), 256, 0, st>>>(g->rowptr, g->n, flags);
  GB_LAUNCH_CHECK("k_degree_flags");
  int rc = device_exclusive_scan<int64_t>(d_nd, nd, FlagF{flags}, pre, scan_ws, st);
  if (rc) return rc;
  int64_t slots = 0;
  GB_CUDA(cudaMemcpyAsync(&slots, pre + nd, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GB_CUDA(cudaStreamSynchronize(st));
  g->slots = slots;
  GB_CUDA(cudaMalloc(&g->deg_slot, sizeof(int32_t) * nd));
  const int64_t sl = slots > 0 ? slots : 1;
  GB_CUDA(cudaMalloc(&g->slot_deg, sizeof(int32_t) * sl));
  GB_CUDA(cudaMalloc(&g->run_j0, sizeof(int32_t) * sl * (kMaxRuns + 1)));
  GB_CUDA(cudaMalloc(&g->run_s0, sizeof(double) * sl * kMaxRuns));
  GB_CUDA(cudaMalloc(&g->run_d, sizeof(double) * sl * kMaxRuns));
  GB_CUDA(cudaMalloc(&g->run_n, sizeof(int32_t) * sl));
  GB_CUDA(cudaMalloc(&g->run_lower, sizeof(int8_t) * sl * kBinades));
  int32_t* d_over = nullptr;
  GB_CUDA(cudaMallocAsync(&d_over, sizeof(int32_t), st));
  GB_CUDA(cudaMemsetAsync(d_over, 0, sizeof(int32_t), st));
  k_degree_slots<<<grid_for(nd, 256, 8 * kNumSMs), 256, 0, st>>>(flags, pre, nd, g->deg_slot,
                                                                  g->slot_deg);
  GB_LAUNCH_CHECK("k_degree_slots");
  if (slots > 0) {
    k_build_runs<<<grid_for(slots, 64, 1 << 20), 64, 0, st>>>(g->slot_deg, slots, g->run_j0,
                                                               g->run_s0, g->run_d, g->run_n,
                                                               g->run_lower, d_over);
    GB_LAUNCH_CHECK("k_build_runs");
  }
  int32_t h_over = 0;
  GB_CUDA(cudaMemcpyAsync(&h_over, d_over, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  GB_CUDA(cudaStreamSynchronize(st));
  GB_CUDA(cudaFreeAsync(d_max, st));
  GB_CUDA(cudaFreeAsync(flags, st));
  GB_CUDA(cudaFreeAsync(pre, st));
  GB_CUDA(cudaFreeAsync(scan_ws, st));
  GB_CUDA(cudaFreeAsync(d_nd, st));
  GB_CUDA(cudaFreeAsync(d_over, st));
  GB_CUDA(cudaStreamSynchronize(st));
  if (h_over) {
    set_error("replay table overflow: a degree needs more than %d runs", kMaxRuns);
    return GB_ERR_UNSUPPORTED;
  }
  return GB_OK;
}

// ---------------------------------------------------------- workspace plan
struct SageWs {
  int32_t* pidx;
  int32_t* deg;
  int64_t* gstart;
  int64_t* scan_ws;
  uint32_t* bitmap;
  int32_t* wpre;
  int64_t* d_W;
  // dedup mode
  uint32_t* vbits;   // one bit per vertex
  int32_t* vpre;     // popcount prefix of vbits
  int64_t* d_nw;     // device scalars: nwords, D
  int32_t* dv;       // distinct vertices
  int32_t* gcnt;     // picks per distinct vertex
  int32_t* gcur;
  int64_t* goff;
  uint64_t* pk;      // pick records grouped by vertex
  int32_t* pkb;      // batch of each pick record
  int64_t* ioff1;    // work-item prefixes of the CTA tiers
  int64_t* ioff2;
  size_t bytes;
};

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

static SageWs sage_ws_layout(char* base, int64_t k, int64_t n, int64_t r_cap_max,
                             int64_t f_cap_max) {
  SageWs w{};
  const int64_t nwords = (n + 31) / 32;
  const int64_t W = k * nwords;
  int64_t scan_n = r_cap_max > W ? r_cap_max : W;
  if (nwords > scan_n) scan_n = nwords;
  size_t off = 0;
  auto take = [&](size_t bytes) { char* p = base ? base + off : nullptr; off += align_up(bytes); return p; };
  w.pidx = (int32_t*)take(sizeof(int32_t) * (f_cap_max + 1));
  w.deg = (int32_t*)take(sizeof(int32_t) * (r_cap_max + 1));
  w.gstart = (int64_t*)take(sizeof(int64_t) * (r_cap_max + 1));
  w.scan_ws = (int64_t*)take(sizeof(int64_t) * scan_workspace_elems<int64_t>(scan_n + 1));
  w.bitmap = (uint32_t*)take(sizeof(uint32_t) * (W + 1));
  w.wpre = (int32_t*)take(sizeof(int32_t) * (W + 1));
  w.d_W = (int64_t*)take(sizeof(int64_t));
  w.vbits = (uint32_t*)take(sizeof(uint32_t) * (nwords + 1));
  w.vpre = (int32_t*)take(sizeof(int32_t) * (nwords + 1));
  w.d_nw = (int64_t*)take(sizeof(int64_t) * 2);
  w.dv = (int32_t*)take(sizeof(int32_t) * (r_cap_max + 1));
  w.gcnt = (int32_t*)take(sizeof(int32_t) * (r_cap_max + 1));
  w.gcur = (int32_t*)take(sizeof(int32_t) * (r_cap_max + 1));
  w.goff = (int64_t*)take(sizeof(int64_t) * (r_cap_max + 1));
  w.pk = (uint64_t*)take(sizeof(uint64_t) * (f_cap_max + 1));
  w.pkb = (int32_t*)take(sizeof(int32_t) * (f_cap_max + 1));
  w.ioff1 = (int64_t*)take(sizeof(int64_t) * (r_cap_max + 1));
  w.ioff2 = (int64_t*)take(sizeof(int64_t) * (r_cap_max + 1));
  w.bytes = off;
  return w;
}

__global__ void k_sage_eoff(const int64_t* __restrict__ brow, int64_t k,
                            const int64_t* __restrict__ fptr, int64_t* __restrict__ eoff);

template <typename K>
static int persistent_grid(K kernel, int threads);

__global__ void k_i32_to_i64(const int32_t* __restrict__ src, int64_t* __restrict__ dst) {
  *dst = *src;
}

struct VPopF {
  const uint32_t* b;
  __device__ int64_t operator()(int64_t i) const { return __popc(b[i]); }
};

template <int T>
static int launch_dd(SageWs& ws, const Graph* g, gb_sage_layer_out& o, int64_t k, int64_t nwords,
                     int64_t r_cap, cudaStream_t st) {
  using Tr = DdTier<T>;
  const size_t smem = sizeof(int32_t) * (Tr::kChunk + 4) * (Tr::kWarp ? Tr::kThreads / 32 : 1);
  static int grid = 0;
  if (!grid) {
    cudaFuncSetAttribute(k_dd_stream<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dd_stream<T>, Tr::kThreads, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    grid = (occ > 0 ? occ : 1) * (sms > 0 ? sms : kNumSMs);
  }
  int64_t* ioff = nullptr;
  if (!Tr::kWarp) {
    ioff = T == 1 ? ws.ioff1 : ws.ioff2;
    int rc = device_exclusive_scan<int64_t>(ws.d_nw + 1, r_cap, ItemF<T>{ws.dv, g->rowptr, ws.goff},
                                            ioff, ws.scan_ws, st);
    if (rc) return rc;
  }
  k_dd_stream<T><<<grid, Tr::kThreads, smem, st>>>(ws.d_nw + 1, ws.dv, g->rowptr, g->col,
                                                    ws.goff, ws.pk, ws.pkb, o.fcol, ws.bitmap,
                                                    nwords, ioff);
  GB_LAUNCH_CHECK("k_dd_stream");
  return GB_OK;
}

// Dedup stream step of one layer (pidx from k_sage_pick<false> in place).
// Dedup step 1 (before the pick kernel): distinct row vertices, picks per
// vertex (from the degrees alone) and the group offsets the pick kernel
// writes its records into.
static int dedup_prepare(const Graph* g, SageWs& ws, const int64_t* R_ptr, const int32_t* rowv,
                         int32_t s, int64_t r_cap, int64_t nwords, cudaStream_t st) {
  const int64_t gw = 16 * kNumSMs;
  GB_CUDA(cudaMemsetAsync(ws.vbits, 0, sizeof(uint32_t) * (nwords + 1), st));
  GB_CUDA(cudaMemsetAsync(ws.gcnt, 0, sizeof(int32_t) * (r_cap + 1), st));
  GB_CUDA(cudaMemsetAsync(ws.gcur, 0, sizeof(int32_t) * (r_cap + 1), st));
  k_dd_mark<<<grid_for(r_cap, 256, gw), 256, 0, st>>>(R_ptr, rowv, ws.deg, ws.vbits);
  int rc = device_exclusive_scan<int64_t>(ws.d_nw, nwords, VPopF{ws.vbits}, ws.vpre, ws.scan_ws,
                                          st);
  if (rc) return rc;
  k_i32_to_i64<<<1, 1, 0, st>>>(ws.vpre + nwords, ws.d_nw + 1);
  k_dd_list<<<grid_for(nwords, 256, gw), 256, 0, st>>>(nwords, ws.vbits, ws.vpre, g->rowptr, ws.dv);
  k_dd_count<<<grid_for(r_cap, 256, gw), 256, 0, st>>>(R_ptr, rowv, ws.deg, s, ws.vbits, ws.vpre,
                                                      ws.gcnt);
  rc = device_exclusive_scan<int64_t>(ws.d_nw + 1, r_cap, GcntF{ws.gcnt}, ws.goff, ws.scan_ws, st);
  if (rc) return rc;
  GB_LAUNCH_CHECK("dedup prepare");
  count_launches(5);
  return GB_OK;
}

// Dedup step 2 (after the pick kernel wrote the grouped records): stream
// every distinct row once, in three size tiers.
static int dedup_stream(const Graph* g, SageWs& ws, gb_sage_layer_out& o, int64_t k,
                        int64_t r_cap, int64_t nwords, cudaStream_t st) {
  prof_mark(st);
  int rc = launch_dd<0>(ws, g, o, k, nwords, r_cap, st);
  if (!rc) rc = launch_dd<1>(ws, g, o, k, nwords, r_cap, st);
  if (!rc) rc = launch_dd<2>(ws, g, o, k, nwords, r_cap, st);
  if (rc) return rc;
  prof_mark(st);
  count_launches(5);
  return GB_OK;
}

static int64_t sage_rcap_max(int64_t r1_cap, int32_t layers, const int64_t* fanouts) {
  int64_t r = r1_cap, mx = r1_cap;
  for (int32_t l = 0; l + 1 < layers; ++l) {
    r *= fanouts[l];
    if (r > mx) mx = r;
  }
  return mx;
}

static int64_t sage_fcap_max(int64_t r1_cap, int32_t layers, const int64_t* fanouts) {
  int64_t r = r1_cap, mx = 0;
  for (int32_t l = 0; l < layers; ++l) {
    r *= fanouts[l];
    if (r > mx) mx = r;
  }
  return mx;
}

int sage_workspace(const Graph* g, int64_t k, int64_t r1_cap, int32_t layers,
                   const int64_t* fanouts, size_t* bytes) {
  *bytes = sage_ws_layout(nullptr, k, g->n, sage_rcap_max(r1_cap, layers, fanouts),
                          sage_fcap_max(r1_cap, layers, fanouts)).bytes;
  return GB_OK;
}

template <typename K>
static int persistent_grid(K kernel, int threads) {
  int o = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kernel, threads, 0);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  return (o < 1 ? 1 : o) * (sms > 0 ? sms : kNumSMs);
}

static int stream_grid() {
  static int g = 0;
  if (!g) g = persistent_grid(k_sage_stream, kStreamThreads);
  return g;
}

int sage_bulk(const Graph* g, int64_t k, const int64_t* d_bptr, const int32_t* d_bverts,
              int64_t r1_cap, int64_t batch_size, int32_t layers, const int64_t* fanouts,
              uint64_t seed, uint64_t epoch, int64_t batch_offset, int32_t mode,
              gb_sage_layer_out* L, int64_t* d_sizes, void* d_ws, size_t ws_bytes,
              cudaStream_t st) {
  const bool stream = mode == GB_SAGE_STREAM;
  const bool dedup = mode == GB_SAGE_DEDUP;
  const int64_t nwords = (g->n + 31) / 32;
  const int64_t W = k * nwords;
  const int64_t rmax = sage_rcap_max(r1_cap, layers, fanouts);
  SageWs ws = sage_ws_layout((char*)d_ws, k, g->n, rmax, sage_fcap_max(r1_cap, layers, fanouts));
  if (ws.bytes > ws_bytes) {
    set_error("sage workspace too small: need %zu bytes, got %zu", ws.bytes, ws_bytes);
    return GB_ERR_CAPACITY;
  }
  int64_t r_cap = r1_cap;
  for (int32_t l = 0; l < layers; ++l) {
    const int64_t f_cap = r_cap * fanouts[l];
    if (L[l].r_cap < r_cap || L[l].f_cap < f_cap) {
      set_error("layer %d output too small: need rows %lld entries %lld", (int)l + 1,
                (long long)r_cap, (long long)f_cap);
      return GB_ERR_CAPACITY;
    }
    if (f_cap >= (int64_t)1 << 31) {
      set_error("layer %d bound %lld entries exceeds int32 indexing", (int)l + 1, (long long)f_cap);
      return GB_ERR_UNSUPPORTED;
    }
    r_cap = f_cap;
  }
  GB_CUDA(cudaMemsetAsync(ws.bitmap, 0, sizeof(uint32_t) * (W + 1), st));
  k_set_i64<<<1, 1, 0, st>>>(ws.d_W, W);
  k_set_i64<<<1, 1, 0, st>>>(ws.d_nw, nwords);
  count_launches(2);
  int64_t stride = batch_size;
  r_cap = r1_cap;
  for (int32_t l = 0; l < layers; ++l) {
    const int32_t d = l + 1;
    if (l > 0) stride *= fanouts[l - 1];
    gb_sage_layer_out& o = L[l];
    const int32_t* rowv = l == 0 ? d_bverts : L[l - 1].fcol;
    const int64_t* brow = l == 0 ? d_bptr : L[l - 1].eoff;
    const int64_t* R_ptr = brow + k;
    const int32_t s = (int32_t)fanouts[l];
    k_sage_prep<<<grid_for(r_cap, 256, 16 * kNumSMs), 256, 0, st>>>(R_ptr, rowv, g->rowptr, ws.deg);
    GB_LAUNCH_CHECK("k_sage_prep");
    int rc = device_exclusive_scan<int64_t>(R_ptr, r_cap, TakeF{ws.deg, s}, o.fptr, ws.scan_ws, st);
    if (rc) return rc;
    if (stream) {
      rc = device_exclusive_scan<int64_t>(R_ptr, r_cap, DegF{ws.deg}, ws.gstart, ws.scan_ws, st);
      if (rc) return rc;
    }
    SageArgs A{};
    A.rowptr = g->rowptr; A.col = g->col;
    A.deg_slot = g->deg_slot; A.run_j0 = g->run_j0; A.run_s0 = g->run_s0; A.run_d = g->run_d;
    A.run_n = g->run_n; A.run_lower = g->run_lower;
    A.rowv = rowv; A.deg = ws.deg; A.fptr = o.fptr; A.gstart = ws.gstart;
    A.brow = brow; A.k = k; A.s = s; A.stride = stride; A.batch_offset = batch_offset;
    A.seed = seed; A.epoch = epoch; A.depth = (uint64_t)d;
    A.bitmap = ws.bitmap; A.nwords = nwords; A.fcol = o.fcol; A.pidx = ws.pidx;
    const int pick_grid = grid_for(r_cap, kPickThreads, 64 * kNumSMs);
    if (dedup) {
      rc = dedup_prepare(g, ws, R_ptr, rowv, s, r_cap, nwords, st);
      if (rc) return rc;
      A.vbits = ws.vbits; A.vpre = ws.vpre; A.goff = ws.goff; A.gcur = ws.gcur;
      A.pk = ws.pk; A.pkb = ws.pkb;
    }
    prof_mark(st);
    if (dedup)
      launch_pick<2>(pick_grid, A, R_ptr, st);
    else if (stream)
      launch_pick<0>(pick_grid, A, R_ptr, st);
    else
      launch_pick<1>(pick_grid, A, R_ptr, st);
    GB_LAUNCH_CHECK("k_sage_pick");
    prof_mark(st);
    if (stream) {
      prof_mark(st);
      k_sage_stream<<<stream_grid(), kStreamThreads, 0, st>>>(A, R_ptr);
      GB_LAUNCH_CHECK("k_sage_stream");
      prof_mark(st);
      count_launches(1);
    }
    if (dedup) {
      rc = dedup_stream(g, ws, o, k, r_cap, nwords, st);
      if (rc) return rc;
    }
    rc = device_exclusive_scan<int64_t>(ws.d_W, W, PopF{ws.bitmap}, ws.wpre, ws.scan_ws, st);
    if (rc) return rc;
    int64_t* sizes = d_sizes + 3 * l;
    k_sage_layer_meta<<<grid_for(k + 1, 128, 64), 128, 0, st>>>(brow, k, o.fptr, ws.wpre, nwords,
                                                                 o.eoff, o.coloff, sizes);
    GB_LAUNCH_CHECK("k_sage_layer_meta");
    const int64_t f_cap = r_cap * s;
    k_sage_rank<<<grid_for(f_cap, 256, 16 * kNumSMs), 256, 0, st>>>(
        sizes + 1, o.eoff, k, o.fcol, ws.bitmap, ws.wpre, nwords, o.acol);
    GB_LAUNCH_CHECK("k_sage_rank");
    k_sage_enumerate<<<grid_for(W, 256, 16 * kNumSMs), 256, 0, st>>>(W, nwords, ws.bitmap, ws.wpre,
                                                                       o.colv);
    GB_LAUNCH_CHECK("k_sage_enumerate");
    count_launches(5);  // prep, sample, meta, rank, enumerate
    r_cap = f_cap;
  }
  return GB_OK;
}

// ====================================== per-layer pieces (distributed executor)

// eoff[b] = fptr[brow[b]]; then one bit per (batch, picked vertex)
__global__ void k_sage_eoff(const int64_t* __restrict__ brow, int64_t k,
                            const int64_t* __restrict__ fptr, int64_t* __restrict__ eoff) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b <= k;
       b += (int64_t)gridDim.x * blockDim.x)
    eoff[b] = fptr[brow[b]];
}

__global__ void k_sage_setbits(const int64_t* __restrict__ eoff, int64_t k,
                               const int32_t* __restrict__ fcol, uint32_t* __restrict__ bitmap,
                               int64_t nwords) {
  const int64_t F = eoff[k];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < F;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = k;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (eoff[mid] <= e) lo = mid; else hi = mid;
    }
    const int32_t v = fcol[e];
    atomicOr(bitmap + lo * nwords + (v >> 5), 1u << (v & 31));
  }
}

size_t sage_layer_sample_ws(int64_t r_cap, int64_t f_cap) {
  return align_up(sizeof(int32_t) * (f_cap + 1)) + align_up(sizeof(int64_t) * (r_cap + 1)) +
         align_up(sizeof(int64_t) * scan_workspace_elems<int64_t>(r_cap + 1));
}

// NORM + SAMPLE of the rows with deg[r] > 0 through the CSR (rowptr, col)
// addressed by rowv[r]; picks land at fptr[r] (caller-computed).  No bitmap:
// extraction runs separately once the frontier is complete.
int sage_layer_sample(const Graph* tables, int64_t k, const int64_t* brow, int64_t r_cap,
                      const int32_t* rowv, const int32_t* deg, const int64_t* fptr,
                      const int64_t* rowptr, const int32_t* col, int32_t s, int64_t stride,
                      int64_t batch_offset, uint64_t seed, uint64_t epoch, uint64_t depth,
                      int32_t mode, int32_t* fcol, void* d_ws, size_t ws_bytes, cudaStream_t st) {
  const int64_t f_cap = r_cap * s;
  if (sage_layer_sample_ws(r_cap, f_cap) > ws_bytes) {
    set_error("sage layer workspace too small");
    return GB_ERR_CAPACITY;
  }
  char* p = (char*)d_ws;
  int32_t* pidx = (int32_t*)p;
  p += align_up(sizeof(int32_t) * (f_cap + 1));
  int64_t* gstart = (int64_t*)p;
  p += align_up(sizeof(int64_t) * (r_cap + 1));
  int64_t* scan_ws = (int64_t*)p;
  const int64_t* R_ptr = brow + k;
  const bool stream = mode == GB_SAGE_STREAM;
  if (stream) {
    int rc = device_exclusive_scan<int64_t>(R_ptr, r_cap, DegF{deg}, gstart, scan_ws, st);
    if (rc) return rc;
  }
  SageArgs A{};
  A.rowptr = rowptr; A.col = col;
  A.deg_slot = tables->deg_slot; A.run_j0 = tables->run_j0; A.run_s0 = tables->run_s0;
  A.run_d = tables->run_d; A.run_n = tables->run_n; A.run_lower = tables->run_lower;
  A.rowv = rowv; A.deg = deg; A.fptr = fptr; A.gstart = gstart;
  A.brow = brow; A.k = k; A.s = s; A.stride = stride; A.batch_offset = batch_offset;
  A.seed = seed; A.epoch = epoch; A.depth = depth;
  A.bitmap = nullptr; A.nwords = 0; A.fcol = fcol; A.pidx = pidx;
  const int pick_grid = grid_for(r_cap, kPickThreads, 64 * kNumSMs);
  if (stream) {
    launch_pick<0>(pick_grid, A, R_ptr, st);
    k_sage_stream<<<stream_grid(), kStreamThreads, 0, st>>>(A, R_ptr);
    count_launches(2);
  } else {
    launch_pick<1>(pick_grid, A, R_ptr, st);
    count_launches(1);
  }
  GB_LAUNCH_CHECK("sage_layer_sample");
  return GB_OK;
}

// Owner-computes sampling (1.5D): rows given by (local row, degree, global
// row key, output offset) — the block owner samples requested rows with the
// requester's keys and returns only the picks.  P-free gather.
int sage_sample_keyed(const Graph* tables, int64_t R, const int64_t* d_R, const int32_t* rowv,
                      const int32_t* deg, const int64_t* fptr, const int64_t* rowkeys,
                      const int64_t* rowptr, const int32_t* col, int32_t s, uint64_t seed,
                      uint64_t epoch, uint64_t depth, int32_t* fcol, cudaStream_t st) {
  if (R == 0) return GB_OK;
  SageArgs A{};
  A.rowptr = rowptr; A.col = col;
  A.deg_slot = tables->deg_slot; A.run_j0 = tables->run_j0; A.run_s0 = tables->run_s0;
  A.run_d = tables->run_d; A.run_n = tables->run_n; A.run_lower = tables->run_lower;
  A.rowv = rowv; A.rowkeys = rowkeys; A.deg = deg; A.fptr = fptr;
  A.k = 0; A.s = s; A.seed = seed; A.epoch = epoch; A.depth = depth;
  A.bitmap = nullptr; A.fcol = fcol;
  launch_pick<1>(grid_for(R, kPickThreads, 64 * kNumSMs), A, d_R, st);
  GB_LAUNCH_CHECK("sage_sample_keyed");
  count_launches(1);
  return GB_OK;
}

size_t sage_layer_extract_ws(int64_t n, int64_t k) {
  const int64_t W = k * ((n + 31) / 32);
  return align_up(sizeof(uint32_t) * (W + 1)) + align_up(sizeof(int32_t) * (W + 1)) +
         align_up(sizeof(int64_t) * scan_workspace_elems<int64_t>(W + 1)) + align_up(8);
}

// EXTRACT of a complete frontier (fptr, fcol): sage_batch_blocks +
// block_diag (sampler.py:390-417): acol, colv, eoff, coloff, sizes (R, F, U)
int sage_layer_extract(int64_t n, int64_t k, const int64_t* brow, const int64_t* fptr,
                       const int32_t* fcol, int64_t f_cap, int32_t* acol, int32_t* colv,
                       int64_t* eoff, int64_t* coloff, int64_t* sizes, void* d_ws,
                       size_t ws_bytes, cudaStream_t st) {
  if (sage_layer_extract_ws(n, k) > ws_bytes) {
    set_error("sage extract workspace too small");
    return GB_ERR_CAPACITY;
  }
  const int64_t nwords = (n + 31) / 32, W = k * nwords;
  char* p = (char*)d_ws;
  uint32_t* bitmap = (uint32_t*)p;
  p += align_up(sizeof(uint32_t) * (W + 1));
  int32_t* wpre = (int32_t*)p;
  p += align_up(sizeof(int32_t) * (W + 1));
  int64_t* scan_ws = (int64_t*)p;
  p += align_up(sizeof(int64_t) * scan_workspace_elems<int64_t>(W + 1));
  int64_t* d_W = (int64_t*)p;
  GB_CUDA(cudaMemsetAsync(bitmap, 0, sizeof(uint32_t) * (W + 1), st));
  k_set_i64<<<1, 1, 0, st>>>(d_W, W);
  k_sage_eoff<<<grid_for(k + 1, 128, 64), 128, 0, st>>>(brow, k, fptr, eoff);
  k_sage_setbits<<<grid_for(f_cap, 256, 16 * kNumSMs), 256, 0, st>>>(eoff, k, fcol, bitmap, nwords);
  GB_LAUNCH_CHECK("k_sage_setbits");
  int rc = device_exclusive_scan<int64_t>(d_W, W, PopF{bitmap}, wpre, scan_ws, st);
  if (rc) return rc;
  k_sage_layer_meta<<<grid_for(k + 1, 128, 64), 128, 0, st>>>(brow, k, fptr, wpre, nwords, eoff,
                                                               coloff, sizes);
  k_sage_rank<<<grid_for(f_cap, 256, 16 * kNumSMs), 256, 0, st>>>(sizes + 1, eoff, k, fcol,
                                                                  bitmap, wpre, nwords, acol);
  k_sage_enumerate<<<grid_for(W, 256, 16 * kNumSMs), 256, 0, st>>>(W, nwords, bitmap, wpre, colv);
  GB_LAUNCH_CHECK("sage_layer_extract");
  count_launches(6);
  return GB_OK;
}

int take_scan(int64_t r_cap, const int64_t* R_ptr, const int32_t* deg, int32_t s, int64_t* fptr,
              int64_t* scan_ws, cudaStream_t st) {
  return device_exclusive_scan<int64_t>(R_ptr, r_cap, TakeF{deg, s}, fptr, scan_ws, st);
}

// gather rows `ids` of a CSR block (rows are ids[i] - row0) into a
// contiguous buffer at out_off[i] (caller-computed from known degrees)
__global__ void k_gather_rows(int64_t m, const int32_t* __restrict__ ids, int64_t row0,
                              const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                              const int64_t* __restrict__ out_off, int32_t* __restrict__ out) {
  const int lane = lane_id();
  for (int64_t i = global_warp(); i < m; i += grid_warps()) {
    const int64_t r = ids[i] - row0;
    const int64_t a = rowptr[r], d = rowptr[r + 1] - a, o = out_off[i];
    for (int64_t x = lane; x < d; x += 32) out[o + x] = col[a + x];
  }
}

int gather_rows(int64_t m, const int32_t* ids, int64_t row0, const int64_t* rowptr,
                const int32_t* col, const int64_t* out_off, int32_t* out, cudaStream_t st) {
  if (m == 0) return GB_OK;
  k_gather_rows<<<grid_for(m * 32, 256, 16 * kNumSMs), 256, 0, st>>>(m, ids, row0, rowptr, col,
                                                                     out_off, out);
  GB_LAUNCH_CHECK("k_gather_rows");
  count_launches(1);
  return GB_OK;
}

// dense feature rows: out[i, :] = H[ids[i] - row0, :] (fp32, f columns)
__global__ void k_gather_feat(int64_t m, const int32_t* __restrict__ ids, int64_t row0,
                              const float* __restrict__ H, int64_t f, float* __restrict__ out) {
  const int lane = lane_id();
  for (int64_t i = global_warp(); i < m; i += grid_warps()) {
    const float* src = H + (ids[i] - row0) * f;
    float* dst = out + i * f;
    for (int64_t x = lane; x < f; x += 32) dst[x] = src[x];
  }
}

int gather_features(int64_t m, const int32_t* ids, int64_t row0, const float* H, int64_t f,
                    float* out, cudaStream_t st) {
  if (m == 0) return GB_OK;
  k_gather_feat<<<grid_for(m * 32, 256, 16 * kNumSMs), 256, 0, st>>>(m, ids, row0, H, f, out);
  GB_LAUNCH_CHECK("k_gather_feat");
  count_launches(1);
  return GB_OK;
}

}  // namespace gb
