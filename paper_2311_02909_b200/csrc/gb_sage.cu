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
// Three modes of the SAMPLE kernels, identical outputs:
//   GB_SAGE_DEDUP (default): rows grouped by vertex, each distinct P row
//     sampled once per group; its picks read in place or the row staged
//     by TMA (below).
//   GB_SAGE_STREAM: P row formed on chip — the warp streams the whole A row
//     (coalesced 16-B loads, merge-path balanced over rows+entries) and
//     catches the picked entries out of registers.  This is Alg. 1 with P
//     never written to HBM; its algorithmic bytes are SURVEY.md §8(d).
//   GB_SAGE_PFREE: the P-free fast path: only the picked
//     entries of A are read.
// Extraction is dense (every bitmap record scanned) or, for n >= 2^23,
// over the touched records only (k_touch / k_rec_scan_touch /
// k_enum_touch).
#include <stdarg.h>
#include <stdlib.h>
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
                             int32_t* __restrict__ run_j0, double2* __restrict__ run_sd,
                             int32_t* __restrict__ run_n,
                             int8_t* __restrict__ run_lower, int32_t* __restrict__ overflow) {
  for (int64_t sl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sl < slots;
       sl += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = slot_deg[sl];
    const double w = 1.0 / (double)m;
    int32_t* J = run_j0 + sl * (kMaxRuns + 1);
    double2* SD = run_sd + sl * kMaxRuns;
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
        if (nr < kMaxRuns) { J[nr] = (int32_t)j0; SD[nr] = make_double2(s0, d); } else bad = true;
        ++nr;
        j0 = j; s0 = S2; len = 1; d = 0.0;
      }
      S = S2;
    }
    if (nr < kMaxRuns) { J[nr] = (int32_t)j0; SD[nr] = make_double2(s0, d); } else bad = true;
    ++nr;
    if (nr <= kMaxRuns) J[nr] = (int32_t)(m + 1);  // sentinel
    run_n[sl] = nr;
    if (!bad) {
      const int64_t top = (int64_t)binade(SD[nr - 1].x);
      int8_t* low = run_lower + sl * kBinades;
      for (int b = 0; b < kBinades; ++b) {
        int c = 0;
        for (int r = 0; r < nr; ++r) c += (top - (int64_t)binade(SD[r].x) > b) ? 1 : 0;
        low[b] = (int8_t)c;
      }
    }
    if (bad) atomicExch(overflow, 1);
  }
}

// ============================================================ layer kernels

// degrees of the layer's rows; vbits != nullptr (dedup): also one bit per
// vertex that some nonempty row references
__global__ void k_sage_prep(const int64_t* __restrict__ R_ptr, const int32_t* __restrict__ rowv,
                            const int64_t* __restrict__ rowptr, int32_t* __restrict__ deg,
                            uint32_t* __restrict__ vbits) {
  const int64_t R = *R_ptr;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = rowv[r];
    const int32_t d = (int32_t)(rowptr[v + 1] - rowptr[v]);
    deg[r] = d;
    if (vbits && d > 0) atomicOr(vbits + (v >> 5), 1u << (v & 31));
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

struct PeerRows {
  int nblk;
  const int64_t* bounds;
  const int64_t* const* brp;
  const int32_t* const* bcol;
};

struct SageArgs {
  const int64_t* rowptr;
  const int32_t* col;
  const int32_t* deg_slot;
  const int32_t* run_j0;
  const double2* run_sd;  // (run start S, increment) per run
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
  // dedup mode (OUT 2): frontier rows grouped by vertex, per grouped row its
  // frontier offset and batch, picks at pidx[q * s ..]
  const int64_t* D_ptr;
  const unsigned long long* grows;  // grouped rows in total (dedup)
  const int4* rrec;
  // P-free (OUT 1) extra destinations: peer frontiers written over NVLink
  int32_t* dst[8];
  int ndst;
  PeerRows peer;  // nblk > 0 (1.5D split): A rows live in the owners' block CSRs
};

__device__ __forceinline__ int32_t vrank(const uint32_t* vbits, const int32_t* vpre, int32_t v) {
  return vpre[v >> 5] + __popc(vbits[v >> 5] & ((1u << (v & 31)) - 1u));
}

// (batch, vertex) bitmap of the bulk: one 16-B record per 96 vertices —
// three bit words and, after the extraction scan, the number of set bits
// before the record in its batch row — so the block-diagonal rank of a
// picked vertex is one 16-B load and at most three popcounts.  uint32 index
// of vertex v's bit word inside its batch row:
__device__ __forceinline__ uint32_t pk_word(int32_t v) {
  const uint32_t w = (uint32_t)v >> 5, r = w / 3u;
  return (r << 2) + (w - 3u * r);
}

#ifndef GB_PICK_T
#define GB_PICK_T 128  // pick CTA (swept 64 / 128 / 256)
#endif
#ifndef GB_PICK_GRID
#define GB_PICK_GRID 64  // pick grid x SMs (swept 8 / 16 / 64 / 128 / 1024)
#endif
#ifndef GB_GRP_GRID
#define GB_GRP_GRID 16  // grouping grids x SMs (swept 8 / 16 / 32)
#endif
#ifndef GB_X_GRID
#define GB_X_GRID 32  // extraction grids x SMs (swept 8 / 16 / 32 / 64 / 128)
#endif
constexpr int kPickThreads = GB_PICK_T;
constexpr int kStreamThreads = 256;
constexpr int kRowCost = 48;       // merge-path weight of one row (in entries)
constexpr int kStreamUnroll = 8;   // 16-B loads in flight per lane
constexpr int kBrowSmem = 1024;

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

// Replay table of one degree with its binade index: read through the
// read-only path (L1-resident, ~1.4 KB per hot degree; SM = false) or from a
// shared-memory copy (SM = true, the fused dedup kernel).
struct GTable {
  const int32_t* j0;
  const double2* sd;  // (run start S, increment)
  const int8_t* lower;
  int nr;
  uint64_t top;  // binade of the last run's start
};

// first j >= 1 with S[j] > target (m + 1 when none).  The run is located by
// the binade index (O(1)), the position inside it by a float estimate that
// the exact fp64 comparisons then correct.
__device__ __forceinline__ int64_t gt_first_gt(const GTable& t, double target) {
  if (target < __ldg(&t.sd->x)) return 1;
  const int64_t off = (int64_t)t.top - (int64_t)binade(target);
  int r = off < 0 ? t.nr : (int)__ldg(t.lower + (off < kBinades ? off : kBinades - 1));
  // r = first run starting in target's binade or above; step back / forward
  double2 sd;
  if (r >= t.nr || (sd = __ldg(t.sd + r)).x > target) {
    sd = __ldg(t.sd + --r);
  } else {
    double2 nx;
    while (r + 1 < t.nr && (nx = __ldg(t.sd + r + 1)).x <= target) { ++r; sd = nx; }
  }
  const int64_t j0 = __ldg(t.j0 + r);
  const int64_t len = (int64_t)__ldg(t.j0 + r + 1) - j0;
  if (len == 1) return j0 + 1;
  const double s0 = sd.x, d = sd.y;
  int64_t q = (int64_t)__fdividef((float)(target - s0), (float)d);
  q = q < 0 ? 0 : (q > len - 1 ? len - 1 : q);
  while (q > 0 && __dadd_rn(s0, __dmul_rn((double)q, d)) > target) --q;
  while (q + 1 < len && __dadd_rn(s0, __dmul_rn((double)(q + 1), d)) <= target) ++q;
  return j0 + q + 1;
}

// Per-degree replay tables of the graph (gb_graph_create).
struct SageTabs {
  const int32_t* deg_slot;
  const int32_t* run_j0;
  const double2* run_sd;
  const int32_t* run_n;
  const int8_t* run_lower;
};

// NORM + SAMPLE of one P row: draw t uses u = uniform53(seed, epoch, depth,
// key, t); n_live = deg - t live entries of weight fl(1/deg); target =
// u * S[n_live]; the draw selects the j-th live entry, j = first j with
// S[j] > target clamped to n_live — exactly its_sample_row's
// cumsum/searchsorted/clamp/walk-back (sampler.py:176-188).  The picks are
// kept sorted (frontier_from_rows sorts, sampler.py:216) in registers (MAXF
// = fanout bucket, fully unrolled).  Requires take < deg (exhausted rows
// take every index, sampler.py:172-174, and consume no uniform).
template <int MAXF>
__device__ __forceinline__ void sage_draws(const SageTabs& T, uint64_t key, int32_t deg,
                                           int32_t take, uint64_t seed, uint64_t epoch,
                                           uint64_t depth, int32_t (&sorted)[MAXF]) {
  const int32_t slot = __ldg(T.deg_slot + deg);
  GTable tab;
  tab.j0 = T.run_j0 + (int64_t)slot * (kMaxRuns + 1);
  tab.sd = T.run_sd + (int64_t)slot * kMaxRuns;
  tab.lower = T.run_lower + (int64_t)slot * kBinades;
  tab.nr = __ldg(T.run_n + slot);
  // S[n_live] run cursor: n_live only falls, so the run of S[n_live] is
  // carried across draws and its (j0, s0, d) reloaded only when it moves
  int rS = tab.nr - 1;
  int32_t j0S = __ldg(tab.j0 + rS);
  double2 sdS = __ldg(tab.sd + rS);
  tab.top = binade(sdS.x);
  uint64_t w0 = 0, w1 = 0, w2 = 0, w3 = 0;
  auto draw = [&](int t) {
    if ((t & 3) == 0) {
      w0 = key; w1 = depth; w2 = (uint64_t)(t >> 2); w3 = 0;
      philox4x64_10(w0, w1, w2, w3, seed, epoch);
    }
    const uint64_t w = (t & 3) == 0 ? w0 : (t & 3) == 1 ? w1 : (t & 3) == 2 ? w2 : w3;
    const double u = (double)(w >> 11) * 0x1.0p-53;
    const int64_t n_live = deg - t;
    if (j0S > n_live) {
      do j0S = __ldg(tab.j0 + --rS); while (j0S > n_live);
      sdS = __ldg(tab.sd + rS);
    }
    const double target =
        __dmul_rn(u, __dadd_rn(sdS.x, __dmul_rn((double)(n_live - j0S), sdS.y)));
    int64_t j = gt_first_gt(tab, target);
    if (j > n_live) j = n_live;
    // j-th live index: skip over the removed (sorted) ones, then insert
    int32_t x = (int32_t)(j - 1);
    int i = 0;
#pragma unroll
    for (int z = 0; z < MAXF; ++z)
      if (z < t && sorted[z] <= x) { ++x; ++i; }
#pragma unroll
    for (int z = MAXF - 1; z > 0; --z)  // shift up and insert in one pass
      sorted[z] = (z > i && z <= t) ? sorted[z - 1] : (z == i ? x : sorted[z]);
    if (i == 0) sorted[0] = x;
  };
  if constexpr (MAXF <= 10) {
    // small buckets: unrolled, so draw t's Philox word, the skip over the t
    // removed indices and the insertion are all static
#pragma unroll
    for (int t = 0; t < MAXF; ++t)
      if (t < take) draw(t);
  } else {
    for (int t = 0; t < take; ++t) draw(t);
  }
}

// NORM + SAMPLE, one thread per P row (sage_draws).
// OUT 1 (P-free): read the picked columns of A directly and finish the row;
// OUT 0: write the row-relative indices for the row-streaming kernel.
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
  const SageTabs T{A.deg_slot, A.run_j0, A.run_sd, A.run_n, A.run_lower};
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t deg = A.deg[r];
    if (deg == 0) continue;  // empty P row (sample_rows_ordered, sampler.py:202-204)
    const int32_t take = min(deg, A.s);
    const int64_t fp = A.fptr[r];
    // P-free: the row's start in A, loaded before the draws so its latency
    // (rowv -> row_ptr, or the owner's block table) hides behind them
    const int32_t* rowp = nullptr;
    if (OUT == 1) {
      const int32_t v = A.rowv[r];
      if (A.peer.nblk) {
        int pb = 0;
        while (pb + 1 < A.peer.nblk && A.peer.bounds[pb + 1] <= v) ++pb;
        rowp = A.peer.bcol[pb] + A.peer.brp[pb][v - A.peer.bounds[pb]];
      } else {
        rowp = A.col + A.rowptr[v];
      }
    }
    const int64_t bb = keyed ? 0 : batch_of(s_brow, A.brow, A.k, r);
    int32_t sorted[MAXF];
#pragma unroll
    for (int z = 0; z < MAXF; ++z) sorted[z] = z;  // exhaustion: every index (sampler.py:172-174)
    if (take < deg) {
      // global_row_keys (sampler.py:309-322), or the requester's keys
      uint64_t key;
      if (keyed) {
        key = (uint64_t)A.rowkeys[r];
      } else {
        const int64_t b0 = brow_in_smem ? s_brow[bb] : A.brow[bb];
        key = (uint64_t)((A.batch_offset + bb) * A.stride + (r - b0));
      }
      sage_draws<MAXF>(T, key, deg, take, A.seed, A.epoch, A.depth, sorted);
    }
    if (OUT == 1) {
      int32_t cv[MAXF];
#pragma unroll
      for (int z = 0; z < MAXF; ++z)
        if (z < take) cv[z] = __ldg(rowp + sorted[z]);
      if (A.fcol) {
#pragma unroll
        for (int z = 0; z < MAXF; ++z)
          if (z < take) A.fcol[fp + z] = cv[z];
      }
      for (int m = 0; m < A.ndst; ++m) {
        int32_t* d = A.dst[m] + fp;
#pragma unroll
        for (int z = 0; z < MAXF; ++z)
          if (z < take) d[z] = cv[z];
      }
      if (A.bitmap) {
        uint32_t* bm = A.bitmap + bb * A.nwords;
#pragma unroll
        for (int z = 0; z < MAXF; ++z)
          if (z < take) atomicOr(bm + pk_word(cv[z]), 1u << (cv[z] & 31));
      }
    } else {
#pragma unroll
      for (int t = 0; t < MAXF; ++t)
        if (t < take) A.pidx[fp + t] = sorted[t];
    }
  }
}

template <int OUT>
static void launch_pick(int grid, const SageArgs& A, const int64_t* R_ptr, cudaStream_t st) {
  if (A.s <= 5)
    k_sage_pick<OUT, 5><<<grid, kPickThreads, 0, st>>>(A, R_ptr);
  else if (A.s <= 8)
    k_sage_pick<OUT, 8><<<grid, kPickThreads, 0, st>>>(A, R_ptr);
  else if (A.s <= 10)
    k_sage_pick<OUT, 10><<<grid, kPickThreads, 0, st>>>(A, R_ptr);
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
        if (A.bitmap) atomicOr(&A.bitmap[b_i * A.nwords + pk_word(c)], 1u << (c & 31));
      }
    }
  }
}

// ============================================ deduplicated P rows (GB_SAGE_DEDUP)
// Frontier rows repeat vertices heavily (hub bias: 3.5M rows over 0.55M
// distinct vertices in layer 3 at products scale), and identical rows of
// Q^l give identical rows of P = Q^l A.  Rows are grouped by vertex and a
// group's picks reach A one of two ways, chosen per vertex by bytes moved
// (k_grp_items): "direct" — every pick read in place by the pick kernel (a
// 32-B sector each; most vertices), or "staged" — the A row formed on chip
// once per work item by TMA bulk copies (cp.async.bulk + mbarrier) and the
// picks of every frontier row that references it served from there
// (heavily re-referenced rows).  The first layer (seed rows) is sampled
// P-free without grouping (dedup_from).
//
// Grouping (three passes over the layer's rows, no vertex bitmap):
//   k_grp_count  degree of each row; rows per vertex counted in a per-vertex
//                counter (the row keeps its slot); a vertex's first row
//                appends it to the distinct list (block-aggregated)
//   k_grp_items  per distinct vertex: its work items (tier by degree) and its
//                rows' range, reserved by block-aggregated atomics (item and
//                row order are free: every frontier row is independent);
//                clears the counter for the next layer
//   k_grp_rows   16-B record (local row, degree or ~vertex for a direct
//                row, frontier offset, batch) of each row at its group's
//                range + slot
// then NORM + SAMPLE per grouped row (k_dd_pick, whole-GPU thread per row,
// rows of one vertex in adjacent lanes share the replay-table loads; direct
// rows finish their frontier entries and batch bits there) and the serve
// tiers for the staged rows (k_dd_serve<0,1,2>).

constexpr int kGrpThreads = 256;
#ifndef GB_GRP_U
#define GB_GRP_U 2  // swept 1 / 2 / 4 / 8: 2 best
#endif
constexpr int kGrpU = GB_GRP_U;  // rows / distinct vertices per thread, gathers issued together
__global__ void __launch_bounds__(kGrpThreads) k_grp_count(
    const int64_t* __restrict__ R_ptr, const int32_t* __restrict__ rowv,
    const int64_t* __restrict__ rowptr, int32_t* __restrict__ deg, int32_t* __restrict__ vcnt,
    int32_t* __restrict__ rslot, int32_t* __restrict__ dv, unsigned long long* __restrict__ dcount) {
  __shared__ int32_t s_w[kGrpThreads / 32];
  __shared__ unsigned long long s_base;
  const int64_t R = *R_ptr;
  const int lane = lane_id(), wid = threadIdx.x >> 5;
  constexpr int64_t kBlk = (int64_t)kGrpThreads * kGrpU;
  for (int64_t r0 = (int64_t)blockIdx.x * kBlk; r0 < R; r0 += (int64_t)gridDim.x * kBlk) {
    int32_t v[kGrpU], d[kGrpU], slot[kGrpU];
#pragma unroll
    for (int u = 0; u < kGrpU; ++u) {
      const int64_t r = r0 + u * kGrpThreads + threadIdx.x;
      v[u] = r < R ? rowv[r] : -1;
    }
#pragma unroll
    for (int u = 0; u < kGrpU; ++u)
      d[u] = v[u] >= 0 ? (int32_t)(rowptr[v[u] + 1] - rowptr[v[u]]) : 0;
#pragma unroll
    for (int u = 0; u < kGrpU; ++u) slot[u] = d[u] > 0 ? atomicAdd(vcnt + v[u], 1) : -1;
    int nf = 0;
#pragma unroll
    for (int u = 0; u < kGrpU; ++u) {
      const int64_t r = r0 + u * kGrpThreads + threadIdx.x;
      if (r < R) {
        deg[r] = d[u];
        rslot[r] = slot[u];
      }
      nf += slot[u] == 0;
    }
    // distinct list: one atomic per block round
    const int incl = warp_incl_scan(nf);
    if (lane == 31) s_w[wid] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int w = 0; w < kGrpThreads / 32; ++w) { const int c = s_w[w]; s_w[w] = tot; tot += c; }
      s_base = tot ? atomicAdd(dcount, (unsigned long long)tot) : 0ull;
    }
    __syncthreads();
    int64_t o = (int64_t)s_base + s_w[wid] + incl - nf;
#pragma unroll
    for (int u = 0; u < kGrpU; ++u)
      if (slot[u] == 0) dv[o++] = v[u];
    __syncthreads();
  }
}

// Serve tiers by row degree d (DdTier below): 0 d <= hi0 (1.5K), 1 d <= hi1
// (4K), 2 hubs; bounds from the sweep in DESIGN.md §6.  An item serves at
// most rows_item(d) frontier rows (about 512 / 2048 / 8192 picks).
struct DdTiers {
  int32_t hi0, hi1;
};
__host__ __device__ __forceinline__ int dd_tier(int64_t d, DdTiers t) {
  return d <= t.hi0 ? 0 : d <= t.hi1 ? 1 : 2;
}
__host__ __device__ __forceinline__ int32_t rows_item(int64_t d, int32_t s, DdTiers t) {
  const int32_t p = d <= t.hi0 ? 512 : d <= t.hi1 ? 2048 : 8192;
  const int32_t r = p / s;
  return r < 1 ? 1 : r;
}

// Work-item descriptor: everything the serve kernels need before the first
// load, in one 32-B record.
struct __align__(16) DdItem {
  int64_t a0;     // A row start (index into col, or peer address / 4)
  int32_t d;      // A row length
  int32_t q0;     // first grouped row
  int32_t nrows;  // grouped rows served
  int32_t pad[3];
};

// row source of the 1.5D batch-split mode: rows of block b (vertices
// [bounds[b], bounds[b+1])) live in a peer's memory as CSR brp[b] / bcol[b]

// tier t's items live in [t * icap, t * icap + tcnt[t]) (t = serve tier by
// degree); tcnt[3] counts the grouped rows.  kGrpU distinct vertices per
// thread, their gathers issued together (the pass is latency-bound on
// random rowptr / counter loads).
constexpr int kItemThreads = 256;
__global__ void __launch_bounds__(kItemThreads) k_grp_items(
    const unsigned long long* __restrict__ dcount, const int32_t* __restrict__ dv,
    const int64_t* __restrict__ rowptr, int32_t* __restrict__ vcnt, int32_t* __restrict__ roff,
    int32_t s, int64_t icap, unsigned long long* __restrict__ tcnt, DdItem* __restrict__ items,
    PeerRows peer, DdTiers tiers, int32_t direct_ratio, bool peer_direct) {
  __shared__ int32_t s_wsum[4][kItemThreads / 32];
  __shared__ int64_t s_base[4];
  const int64_t D = (int64_t)*dcount;
  const int lane = lane_id(), wid = threadIdx.x >> 5;
  constexpr int64_t kBlk = (int64_t)kItemThreads * kGrpU;
  for (int64_t g0 = blockIdx.x * kBlk; g0 < D; g0 += (int64_t)gridDim.x * kBlk) {
    int32_t v[kGrpU], gc[kGrpU], n[kGrpU], t[kGrpU], per[kGrpU];
    int64_t a0[kGrpU], d[kGrpU];
#pragma unroll
    for (int u = 0; u < kGrpU; ++u) {
      const int64_t g = g0 + u * kItemThreads + threadIdx.x;
      v[u] = g < D ? dv[g] : -1;
    }
#pragma unroll
    for (int u = 0; u < kGrpU; ++u) {
      gc[u] = 0;
      a0[u] = d[u] = 0;
      if (v[u] >= 0) {
        a0[u] = rowptr[v[u]];
        d[u] = rowptr[v[u] + 1];
        gc[u] = vcnt[v[u]];
      }
    }
    int tot[4] = {0, 0, 0, 0};
    bool dir[kGrpU];
#pragma unroll
    for (int u = 0; u < kGrpU; ++u) {
      n[u] = 0;
      t[u] = 0;
      per[u] = 1;
      dir[u] = false;
      if (v[u] >= 0) {
        vcnt[v[u]] = 0;  // ready for the next layer
        d[u] -= a0[u];
        t[u] = dd_tier(d[u], tiers);
        per[u] = rows_item(d[u], s, tiers);
        // direct: the rows' picks cover so little of the A row that reading
        // them in place (a sector each) moves fewer bytes than staging it
        const int64_t take = d[u] < s ? d[u] : s;
        dir[u] = direct_ratio > 0 && (!peer.nblk || peer_direct) &&
                 (int64_t)gc[u] * take * direct_ratio < 8 * d[u];
        n[u] = dir[u] ? 0 : (gc[u] + per[u] - 1) / per[u];
        tot[0] += t[u] == 0 ? n[u] : 0;
        tot[1] += t[u] == 1 ? n[u] : 0;
        tot[2] += t[u] == 2 ? n[u] : 0;
        tot[3] += gc[u];
      }
    }
    // per-tier item offsets and the rows' range (z = 3) inside the block
    int incl[4];
#pragma unroll
    for (int z = 0; z < 4; ++z) {
      incl[z] = warp_incl_scan(tot[z]);
      if (lane == 31) s_wsum[z][wid] = incl[z];
    }
    __syncthreads();
    if (threadIdx.x < 4) {
      int all = 0;
      for (int w = 0; w < kItemThreads / 32; ++w) all += s_wsum[threadIdx.x][w];
      s_base[threadIdx.x] =
          all ? (int64_t)atomicAdd(tcnt + threadIdx.x, (unsigned long long)all) : 0;
    }
    __syncthreads();
    int64_t o[4];
#pragma unroll
    for (int z = 0; z < 4; ++z) {
      o[z] = s_base[z] + incl[z] - tot[z];
      for (int w = 0; w < wid; ++w) o[z] += s_wsum[z][w];
    }
#pragma unroll
    for (int u = 0; u < kGrpU; ++u) {
      if (!gc[u]) continue;
      const int64_t r0 = o[3];
      o[3] += gc[u];
      roff[v[u]] = dir[u] ? ~(int32_t)r0 : (int32_t)r0;  // < 0: direct rows
      if (!n[u]) continue;
      const int64_t oi = (t[u] == 0 ? o[0] : t[u] == 1 ? o[1] : o[2]) + (int64_t)t[u] * icap;
      if (t[u] == 0) o[0] += n[u]; else if (t[u] == 1) o[1] += n[u]; else o[2] += n[u];
      int64_t ad = a0[u];
      if (peer.nblk) {
        int b = 0;
        while (b + 1 < peer.nblk && peer.bounds[b + 1] <= v[u]) ++b;
        const int64_t* brp = peer.brp[b];
        ad = ((int64_t)(uintptr_t)(peer.bcol[b] + brp[v[u] - peer.bounds[b]])) >> 2;
      }
      const int64_t r1 = r0 + gc[u];
      for (int q = 0; q < n[u]; ++q) {
        DdItem it;
        it.a0 = ad;
        it.d = (int32_t)d[u];
        it.q0 = (int32_t)(r0 + (int64_t)q * per[u]);
        it.nrows = (int32_t)min((int64_t)per[u], r1 - it.q0);
        it.pad[0] = it.pad[1] = it.pad[2] = 0;
        items[oi + q] = it;
      }
    }
    __syncthreads();  // s_wsum / s_base reused by the next round
  }
}

// grouped row records: (row within its batch, degree — or ~vertex for a
// direct row —, frontier offset, batch)
__global__ void k_grp_rows(const int64_t* __restrict__ R_ptr, const int32_t* __restrict__ rowv,
                           const int32_t* __restrict__ deg, const int64_t* __restrict__ fptr,
                           const int64_t* __restrict__ brow, int64_t k,
                           const int32_t* __restrict__ rslot, const int32_t* __restrict__ roff,
                           int4* __restrict__ rrec) {
  __shared__ int64_t s_brow[kBrowSmem];
  const bool sm = k + 1 <= kBrowSmem;
  if (sm)
    for (int64_t i = threadIdx.x; i <= k; i += blockDim.x) s_brow[i] = brow[i];
  __syncthreads();
  const int64_t R = *R_ptr;
  const int64_t blk = (int64_t)blockDim.x * kGrpU;
  for (int64_t r0 = blockIdx.x * blk + threadIdx.x; r0 < R; r0 += (int64_t)gridDim.x * blk) {
    int32_t d[kGrpU], v[kGrpU], sl[kGrpU], pos[kGrpU];
#pragma unroll
    for (int u = 0; u < kGrpU; ++u) {
      const int64_t r = r0 + u * (int64_t)blockDim.x;
      d[u] = 0;
      if (r < R) {
        d[u] = deg[r];
        v[u] = rowv[r];
        sl[u] = rslot[r];
      }
    }
#pragma unroll
    for (int u = 0; u < kGrpU; ++u)
      if (d[u] > 0) pos[u] = roff[v[u]];
#pragma unroll
    for (int u = 0; u < kGrpU; ++u) {
      if (d[u] > 0) {
        const int64_t r = r0 + u * (int64_t)blockDim.x;
        const int64_t b = batch_of(s_brow, brow, k, r);
        const bool dir = pos[u] < 0;
        rrec[(dir ? ~pos[u] : pos[u]) + sl[u]] =
            make_int4((int32_t)(r - (sm ? s_brow[b] : brow[b])), dir ? ~v[u] : d[u],
                      (int32_t)fptr[r], (int32_t)b);
      }
    }
  }
}

// NORM + SAMPLE of every grouped row with take < d: sorted picks at
// pidx[q * s ..] (rows of one vertex sit in adjacent lanes and share their
// replay-table loads); exhausted rows are served in order without picks.
// Direct rows (record .y = ~vertex) read their picked columns in place and
// finish the frontier entries and batch bits here.
struct DdPickOut {
  int32_t* pidx;
  const int64_t* rowptr;
  const int32_t* col;
  int32_t* fcol;
  uint32_t* bitmap;
  int64_t nwords;
  PeerRows peer;  // nblk > 0: direct rows live in the owners' block CSRs
};
template <int MAXF>
__global__ void __launch_bounds__(kPickThreads) k_dd_pick(
    const unsigned long long* __restrict__ grows, const int4* __restrict__ rrec, SageTabs T,
    int32_t s, int64_t batch_offset, int64_t stride, uint64_t seed, uint64_t epoch,
    uint64_t depth, DdPickOut O) {
  const int64_t R = (int64_t)*grows;
  const int64_t gs = (int64_t)gridDim.x * blockDim.x;
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int4 rec_n = q < R ? rrec[q] : make_int4(0, 0, 0, 0);  // the next row's record in flight
  for (; q < R; q += gs) {
    const int4 rec = rec_n;
    if (q + gs < R) rec_n = rrec[q + gs];
    int32_t d = rec.y;
    int64_t a0 = -1;
    const int32_t* rowp = nullptr;  // the direct row's entries
    if (d < 0) {
      const int32_t v = ~d;
      if (O.peer.nblk) {
        int b = 0;
        while (b + 1 < O.peer.nblk && O.peer.bounds[b + 1] <= v) ++b;
        const int64_t* brp = O.peer.brp[b] + (v - O.peer.bounds[b]);
        a0 = brp[0];
        d = (int32_t)(brp[1] - a0);
        rowp = O.peer.bcol[b] + a0;
      } else {
        a0 = O.rowptr[v];
        d = (int32_t)(O.rowptr[v + 1] - a0);
        rowp = O.col + a0;
      }
    }
    const int32_t take = min(d, s);
    if (take == d && a0 < 0) continue;
    const uint64_t key = (uint64_t)((batch_offset + rec.w) * stride + rec.x);
    int32_t sorted[MAXF];
#pragma unroll
    for (int z = 0; z < MAXF; ++z) sorted[z] = z;
    if (take < d) sage_draws<MAXF>(T, key, d, take, seed, epoch, depth, sorted);
    if (a0 < 0) {
      int32_t* out = O.pidx + q * s;
#pragma unroll
      for (int z = 0; z < MAXF; ++z)
        if (z < take) out[z] = sorted[z];
    } else {
      int32_t cv[MAXF];
#pragma unroll
      for (int z = 0; z < MAXF; ++z)
        if (z < take) cv[z] = __ldg(rowp + sorted[z]);
      uint32_t* bm = O.bitmap + (int64_t)rec.w * O.nwords;
#pragma unroll
      for (int z = 0; z < MAXF; ++z)
        if (z < take) {
          O.fcol[rec.z + z] = cv[z];
          atomicOr(bm + pk_word(cv[z]), 1u << (cv[z] & 31));
        }
    }
  }
}

// ---------------------------------------------------------------- staging
// One-dimensional TMA: cp.async.bulk global -> shared, completion counted in
// bytes on an mbarrier (arrive.expect_tx by one thread, try_wait.parity by
// all).  Rows are staged from their 16-B aligned start to the 16-B aligned
// end (col arrays are 16-B aligned and padded by GB_COL_PAD).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_row(void* smem, const void* gmem, uint32_t bytes,
                                        uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(smem)),
      "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// staged entries of an A row (16-B granules from the aligned start)
__device__ __forceinline__ int dd_row_len(int64_t a0, int32_t d) {
  return (int)(((a0 + d) - (a0 & ~3LL) + 3) & ~3LL);
}

struct DdArgs {
  const int32_t* col;              // nullptr: item a0 is a peer address / 4
  const unsigned long long* tcnt;  // items per tier; tier t's at [t * icap, ..)
  int64_t icap;
  const DdItem* items;
  const int4* rrec;                // grouped rows: (local row, degree, frontier offset, batch)
  const int32_t* pidx;             // sorted picks of grouped row q at pidx[q * s ..]
  int32_t s;
  int32_t* fcol;
  uint32_t* bitmap;
  int64_t nwords;
  int32_t chunk;                   // staged entries per pass (tier 2), row buffer (tier 0 / 1)
};

// pick (row i of an item, draw t): entry index, frontier position, batch
__device__ __forceinline__ void dd_pair(const DdArgs& A, int32_t q, int32_t t, int32_t take,
                                        bool all, int32_t& idx, int32_t& fp, int32_t& bb) {
  idx = all ? t : A.pidx[(uint32_t)q * (uint32_t)A.s + (uint32_t)t];
  const int2 fb = reinterpret_cast<const int2*>(A.rrec)[2 * (uint32_t)q + 1];
  fp = fb.x + t;
  bb = fb.y;
}

__device__ __forceinline__ void dd_put(const DdArgs& A, int32_t fp, int32_t bb, int32_t cv) {
  A.fcol[(uint32_t)fp] = cv;
  atomicOr(A.bitmap + (uint32_t)bb * (uint32_t)A.nwords + pk_word(cv), 1u << (cv & 31));
}

// Serve, three size tiers of distinct rows (degree d, bounds DdTiers): 0
// warp-batched (a warp takes 32 work items, packs as many of their rows as
// fit its buffer, one TMA bulk copy per row, and serves all their picks
// lane-parallel), 1 CTA-256 per item (the row is one TMA bulk copy), 2
// CTA-1024 per item (hubs: TMA chunks as large as shared memory allows).
// The next item's descriptor and each pass's pick metadata load while the
// row lands.
template <int T> struct DdTier;
template <> struct DdTier<0> {
  static constexpr int kThreads = 256;
  static constexpr bool kWarp = true;
};
template <> struct DdTier<1> {
  static constexpr int kThreads = 256;
  static constexpr bool kWarp = false;
};
template <> struct DdTier<2> {
  static constexpr int kThreads = 1024;
  static constexpr bool kWarp = false;
};

constexpr int kGrpInts = 2;  // per-warp mbarrier of the warp tier (in ints)
#ifndef GB_DDU
#define GB_DDU 4  // swept 2 / 4 / 6 / 8: 4 best
#endif
constexpr int kDdU = GB_DDU;  // picks per lane whose loads are in flight together

// (frontier offset, batch) of grouped row q: the second half of its record
__device__ __forceinline__ int2 dd_fb(const DdArgs& A, int32_t q) {
  return reinterpret_cast<const int2*>(A.rrec)[2 * (uint32_t)q + 1];
}

// Warp tier.  A warp takes 32 work items (lane j holds item j) and packs as
// many of their rows as fit its buffer; every row is staged by its own lane
// with one bulk copy (TMA, completion counted on the warp's mbarrier; 16-B
// cp.async granules measured slower at every row length).  Pick p of the
// sub-group belongs to the item whose pick range holds it: found for 32
// consecutive picks at once by a ballot (items starting at or before the
// first) and an OR-reduction of the start bits inside the window, then the
// item's fields are shuffled from its lane — no tables, no searches.
__device__ void dd_serve_warp(const DdArgs& A, int32_t* buf, int B, uint64_t* bar) {
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = lane_id(), s = A.s;
  const uint32_t NW = (uint32_t)A.nwords;
  const int64_t it1 = (int64_t)A.tcnt[0];
  const int64_t nblk = (it1 + 31) / 32;
  if (lane == 0) mbar_init(bar, 1);
  __syncwarp();
  uint32_t phase = 0;
  for (int64_t blk = global_warp(); blk < nblk; blk += grid_warps()) {
    const int64_t it = blk * 32 + lane;
    const int nitems = (int)min((int64_t)32, it1 - blk * 32);
    DdItem c{};
    const bool valid = lane < nitems;
    if (valid) c = A.items[it];
    const int len = valid ? dd_row_len(c.a0, c.d) : 0;
    const int take = valid ? min(c.d, s) : 1;
    const int np = valid ? c.nrows * take : 0;
    const bool all = take == c.d;  // every entry, no picks stored
    const uint32_t mg = 0xffffffffu / (uint32_t)take + 1u;  // r / take = umulhi(r, mg)
    for (int j0 = 0; j0 < nitems;) {
      // sub-group [j0, j1): rows packed while they fit (always at least one)
      const int lz = lane >= j0 ? len : 0;
      const int incl = warp_incl_scan(lz);
      const unsigned fit = __ballot_sync(FULL, lane >= j0 && lane < nitems && incl <= B);
      const int j1 = fit ? 32 - __clz(fit) : j0 + 1;
      const bool in = lane >= j0 && lane < j1;
      const int pz = in ? np : 0;
      const int pinc = warp_incl_scan(pz);
      const int P = __shfl_sync(FULL, pinc, j1 - 1);
      const int pst = pinc - pz;                         // item's first pick
      const int rof = incl - lz + (int)(c.a0 & 3);       // item's row base in buf
      // every packed row: one bulk copy issued by its own lane
      const uint32_t bytes = warp_sum(in ? 4u * (uint32_t)len : 0u);
      if (lane == 0) mbar_expect_tx(bar, bytes);
      __syncwarp();
      if (in) {
        fence_async_smem();
        tma_row(buf + (incl - lz), A.col + (c.a0 & ~3LL), 4u * (uint32_t)len, bar);
      }
      // pick metadata of kDdU windows of 32 picks; the global loads are
      // issued here and first used in the serve loop below
      int32_t idx[kDdU], t[kDdU], ro[kDdU];
      int2 fb[kDdU];
      auto batch = [&](int p0) {
#pragma unroll
        for (int u = 0; u < kDdU; ++u) {
          const int base = p0 + 32 * u;
          const unsigned le = __ballot_sync(FULL, in && pst <= base);
          const bool st = in && pst > base && pst < base + 32;
          const unsigned M = __reduce_or_sync(FULL, st ? 1u << (pst - base) : 0u);
          const int item = j0 + __popc(le) - 1 + __popc(M & ((2u << lane) - 1u));
          const int ps = __shfl_sync(FULL, pst, item);
          const int tk = __shfl_sync(FULL, take, item);
          const uint32_t m = __shfl_sync(FULL, mg, item);
          const int q0 = __shfl_sync(FULL, c.q0, item);
          const int al = __shfl_sync(FULL, (int)all, item);
          ro[u] = __shfl_sync(FULL, rof, item);
          const int p = base + lane;
          if (p < P) {
            const int r = p - ps;
            const int i = tk == 1 ? r : (int)__umulhi((uint32_t)r, m);
            t[u] = r - i * tk;
            const int q = q0 + i;
            idx[u] = al ? t[u] : A.pidx[(uint32_t)q * (uint32_t)s + (uint32_t)t[u]];
            fb[u] = dd_fb(A, q);
          }
        }
      };
      batch(0);  // while the rows land
      mbar_wait(bar, phase);
      phase ^= 1u;
      for (int p0 = 0; p0 < P; p0 += 32 * kDdU) {
        if (p0) batch(p0);
#pragma unroll
        for (int u = 0; u < kDdU; ++u) {
          if (p0 + 32 * u + lane < P) {
            const int32_t cv = buf[ro[u] + idx[u]];
            A.fcol[(uint32_t)(fb[u].x + t[u])] = cv;
            atomicOr(A.bitmap + ((uint32_t)fb[u].y * NW + pk_word(cv)), 1u << (cv & 31));
          }
        }
      }
      __syncwarp();  // buffer free
      j0 = j1;
    }
  }
}

// CTA tiers: per work item the A row (tier 2: a chunk of it) lands by TMA
// while the first pass's pick metadata loads; every pick is served from
// shared memory.  Tier t's items live at [t * icap, t * icap + tcnt[t]).
template <int TIER>
__global__ void __launch_bounds__(DdTier<TIER>::kThreads) k_dd_serve(DdArgs A) {
  constexpr bool CTA = !DdTier<TIER>::kWarp;
  extern __shared__ __align__(128) int32_t sbuf[];
  if constexpr (!CTA) {
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    dd_serve_warp(A, sbuf + w * (A.chunk + 8), A.chunk + 8,
                  reinterpret_cast<uint64_t*>(sbuf + nw * (A.chunk + 8) + w * kGrpInts));
    return;
  } else {
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, nthr = blockDim.x;
    if (tid == 0) mbar_init(&bar, 1);
    __syncthreads();
    uint32_t phase = 0;
    const int chunk = A.chunk, s = A.s;
    const int64_t it1 = TIER * A.icap + (int64_t)A.tcnt[TIER];
    const int64_t step = gridDim.x;
    int64_t it = TIER * A.icap + blockIdx.x;
    DdItem cur;
    if (it < it1) cur = A.items[it];
    for (; it < it1; it += step) {
      DdItem nxt;
      if (it + step < it1) nxt = A.items[it + step];
      const int64_t a0 = cur.a0;
      const int32_t d = cur.d, nrows = cur.nrows;
      const int32_t q0 = cur.q0;
      const int32_t take = min(d, s);  // < d: CTA-tier rows are longer than any fanout
      const int npairs = nrows * take;
      for (int32_t c0 = 0; c0 < d; c0 += chunk) {
        const int32_t c1 = min(c0 + chunk, d);
        const int64_t al0 = (a0 + c0) & ~3LL;
        if (tid == 0) {
          const uint32_t bytes = 4u * (uint32_t)dd_row_len(a0 + c0, c1 - c0);
          fence_async_smem();
          mbar_expect_tx(&bar, bytes);
          tma_row(sbuf, A.col + al0, bytes, &bar);
        }
        // pick metadata, kDdU picks per thread in flight; the first batch
        // loads while the row lands
        int32_t idx[kDdU], t[kDdU];
        int2 fb[kDdU];
        auto batch = [&](int p0) {
#pragma unroll
          for (int u = 0; u < kDdU; ++u) {
            const int p = p0 + u * nthr + tid;
            if (p < npairs) {
              const int i = p / take;
              t[u] = p - i * take;
              idx[u] = A.pidx[(uint32_t)(q0 + i) * (uint32_t)s + (uint32_t)t[u]];
              fb[u] = dd_fb(A, q0 + i);
            }
          }
        };
        batch(0);
        mbar_wait(&bar, phase);
        phase ^= 1u;
        const int32_t sh = (int32_t)((a0 + c0) - al0 - c0);  // sbuf[idx + sh], idx in [c0, c1)
        for (int p0 = 0; p0 < npairs; p0 += kDdU * nthr) {
          if (p0) batch(p0);
#pragma unroll
          for (int u = 0; u < kDdU; ++u)
            if (p0 + u * nthr + tid < npairs && idx[u] >= c0 && idx[u] < c1)
              dd_put(A, fb[u].x + t[u], fb[u].y, sbuf[idx[u] + sh]);
        }
        __syncthreads();  // buffer free for the next chunk / item
      }
      cur = nxt;
    }
  }
}

// Fanouts above 32 (no register-resident pick list): thread per frontier
// row, the sorted picks kept in the row's own frontier slot (insertion,
// O(s^2) per row), then replaced by their columns — P-free, same output.
__global__ void __launch_bounds__(kPickThreads) k_sage_pick_big(SageArgs A,
                                                              const int64_t* __restrict__ R_ptr) {
  const int64_t R = *R_ptr;
  const SageTabs T{A.deg_slot, A.run_j0, A.run_sd, A.run_n, A.run_lower};
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t deg = A.deg[r];
    if (deg == 0) continue;
    const int32_t take = min(deg, A.s);
    int32_t* sl = A.fcol + A.fptr[r];
    if (take == deg) {
      for (int z = 0; z < take; ++z) sl[z] = z;
    } else {
      const int64_t b = batch_of(A.brow, A.brow, A.k, r);
      const uint64_t key = (uint64_t)((A.batch_offset + b) * A.stride + (r - A.brow[b]));
      const int32_t slot = __ldg(T.deg_slot + deg);
      GTable tab;
      tab.j0 = T.run_j0 + (int64_t)slot * (kMaxRuns + 1);
      tab.sd = T.run_sd + (int64_t)slot * kMaxRuns;
      tab.lower = T.run_lower + (int64_t)slot * kBinades;
      tab.nr = __ldg(T.run_n + slot);
      tab.top = binade(__ldg(tab.sd + tab.nr - 1).x);
      uint64_t w4[4] = {0, 0, 0, 0};
      for (int t = 0; t < take; ++t) {
        if ((t & 3) == 0) {
          w4[0] = key; w4[1] = A.depth; w4[2] = (uint64_t)(t >> 2); w4[3] = 0;
          philox4x64_10(w4[0], w4[1], w4[2], w4[3], A.seed, A.epoch);
        }
        const double u = (double)(w4[t & 3] >> 11) * 0x1.0p-53;
        const int64_t n_live = deg - t;
        // S[n_live] through the table (first j with S[j] > S[n_live] - 0 is
        // n_live + 1, so S[n_live] = value of run holding n_live)
        int rS = tab.nr - 1;
        while (__ldg(tab.j0 + rS) > n_live) --rS;
        const double2 sdS = __ldg(tab.sd + rS);
        const double target = __dmul_rn(
            u, __dadd_rn(sdS.x, __dmul_rn((double)(n_live - __ldg(tab.j0 + rS)), sdS.y)));
        int64_t j = gt_first_gt(tab, target);
        if (j > n_live) j = n_live;
        int32_t x = (int32_t)(j - 1);
        int i = 0;
        while (i < t && sl[i] <= x) { ++x; ++i; }
        for (int z = t; z > i; --z) sl[z] = sl[z - 1];
        sl[i] = x;
      }
    }
    const int64_t rs = A.rowptr[A.rowv[r]];
    const int64_t b = A.bitmap ? batch_of(A.brow, A.brow, A.k, r) : 0;
    for (int z = 0; z < take; ++z) {
      const int32_t cv = __ldg(A.col + rs + sl[z]);
      sl[z] = cv;
      if (A.bitmap) atomicOr(A.bitmap + b * A.nwords + pk_word(cv), 1u << (cv & 31));
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
  // F < 2^31 and k * nwords < 2^31 (checked by the host): 32-bit indexing.
  // U entries per thread per pass (coalesced, 2U independent gathers in
  // flight); batch by binary search for the first, a forward walk for the rest
  constexpr int U = 4;
  __shared__ int32_t s_eoff[kBrowSmem];
  const bool sm = k + 1 <= kBrowSmem;
  if (sm)
    for (int i = threadIdx.x; i <= k; i += blockDim.x) s_eoff[i] = (int32_t)eoff[i];
  __syncthreads();
  const int32_t F = (int32_t)*F_ptr;
  const int32_t K = (int32_t)k, NW = (int32_t)nwords;
  auto eo = [&](int32_t i) { return sm ? s_eoff[i] : (int32_t)eoff[i]; };
  for (int32_t e0 = blockIdx.x * blockDim.x * U + threadIdx.x; e0 < F;
       e0 += gridDim.x * blockDim.x * U) {
    int32_t v[U], wi[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int32_t e = e0 + u * (int32_t)blockDim.x;
      v[u] = e < F ? fcol[e] : 0;
    }
    int32_t a = 0, b = K;  // last batch with eoff <= e0
    while (b - a > 1) {
      const int32_t mid = (a + b) >> 1;
      if (eo(mid) <= e0) a = mid; else b = mid;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int32_t e = e0 + u * (int32_t)blockDim.x;
      while (a + 1 < K && eo(a + 1) <= e) ++a;
      wi[u] = a * NW + (v[u] >> 5);
    }
    uint32_t bm[U];
    int32_t wp[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (e0 + u * (int32_t)blockDim.x < F) { bm[u] = bitmap[wi[u]]; wp[u] = wpre[wi[u]]; }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int32_t e = e0 + u * (int32_t)blockDim.x;
      if (e < F) acol[e] = wp[u] + __popc(bm[u] & ((1u << (v[u] & 31)) - 1u));
    }
  }
}

// Record extraction (the bulk path, pk_word layout).  Per batch row one CTA
// scans its records (no cross-row look-back: rows are independent), writing
// each record's within-row prefix into its fourth word and the row total;
// the column offsets are the scan of the row totals.
#ifndef GB_RS_GRID
#define GB_RS_GRID 8  // record-scan grid x SMs (swept 4 / 8 / 16: flat)
#endif
#ifndef GB_RS_U
#define GB_RS_U 4  // swept 2 / 4 / 8 / 16: 4 best
#endif
constexpr int kRsThreads = 256, kRsU = GB_RS_U, kRsTile = kRsThreads * kRsU;
// tiles of kRsTile records never straddle a batch row: tile t is segment
// t % tpr of row t / tpr, and its look-back stops at the row's first tile,
// so the 64 rows' chains advance concurrently (st zeroed before the launch)
__global__ void __launch_bounds__(kRsThreads) k_rec_scan(uint4* __restrict__ rec, int64_t NR,
                                                       int64_t k, int64_t* __restrict__ tot,
                                                       unsigned long long* __restrict__ st) {
  __shared__ int64_t sw[33];
  __shared__ int64_t s_tile, s_prefix;
  const int64_t tpr = (NR + kRsTile - 1) / kRsTile;
  const int64_t ntiles = tpr * k;
  for (;;) {
    if (threadIdx.x == 0) s_tile = (int64_t)atomicAdd(st, 1ull);
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile >= ntiles) return;
    const int64_t row = tile / tpr, seg = tile - row * tpr;
    uint4* r = rec + row * NR;
    uint32_t* r32 = reinterpret_cast<uint32_t*>(r);
    const int64_t i0 = seg * kRsTile + (int64_t)threadIdx.x * kRsU;
    int c[kRsU];
    int tsum = 0;
#pragma unroll
    for (int u = 0; u < kRsU; ++u) {
      c[u] = 0;
      if (i0 + u < NR) {
        const uint4 x = r[i0 + u];
        c[u] = __popc(x.x) + __popc(x.y) + __popc(x.z);
      }
      tsum += c[u];
    }
    int64_t total;
    int64_t run = block_excl_scan<int64_t>(tsum, sw, total);
    if (threadIdx.x < 32) {
      const int64_t pre = tile_lookback(st, tile, row * tpr, total);
      if (threadIdx.x == 0) s_prefix = pre;
    }
    __syncthreads();
    run += s_prefix;
#pragma unroll
    for (int u = 0; u < kRsU; ++u) {
      if (i0 + u < NR) r32[4 * (i0 + u) + 3] = (uint32_t)run;
      run += c[u];
    }
    if (seg == tpr - 1 && threadIdx.x == 0) tot[row] = s_prefix + total;
    __syncthreads();
  }
}

// coloff[b] = sum of the row totals before b; sizes = (R, F, U).  One CTA.
// ---- sparse extraction (large n: the (batch, vertex) bit rows are almost
// empty, e.g. papers shape: 7.1 G bits for <= 6.4 M set).  One touch bit per
// 16-B record, set from the layer's picks; the scan and the enumeration then
// visit touched records only instead of streaming every record.
constexpr int kTouchB = 8;  // touched records whose loads are in flight together
// touch bit of every pick's record: batch row walked as in k_sage_rank128
__global__ void k_touch(const int64_t* __restrict__ brow, const int64_t* __restrict__ fptr,
                        const int64_t* __restrict__ eoff, int64_t k,
                        const int32_t* __restrict__ fcol, int64_t TW,
                        uint32_t* __restrict__ touch) {
  const int64_t F = fptr[brow[k]];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < F;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = 0, b = k;  // last batch with eoff <= e
    while (b - a > 1) {
      const int64_t mid = (a + b) >> 1;
      if (eoff[mid] <= e) a = mid; else b = mid;
    }
    const uint32_t r = (uint32_t)fcol[e] / 96u;  // record of the vertex in its batch row
    atomicOr(touch + a * TW + (r >> 5), 1u << (r & 31));
  }
}
#ifndef GB_TS_T
#define GB_TS_T 1024  // swept 128 / 256 / 512 / 1024 (papers: 1024 best)
#endif
#ifndef GB_ET_GRID
#define GB_ET_GRID 16  // swept 8 / 16 / 32 / 64 (flat)
#endif
#ifndef GB_TS_GRID
#define GB_TS_GRID 8
#endif
constexpr int kTsThreads = GB_TS_T;  // touched-record scan CTA = touch words per tile
// k_rec_scan over touched records only: tile = kTsThreads touch words of
// one batch row, look-back chained within the row
__global__ void __launch_bounds__(kTsThreads) k_rec_scan_touch(
    uint4* __restrict__ rec, int64_t NR, int64_t k, const uint32_t* __restrict__ touch,
    int64_t TW, int64_t* __restrict__ tot, unsigned long long* __restrict__ st) {
  __shared__ int64_t sw[33];
  __shared__ int64_t s_tile, s_prefix;
  __shared__ uint8_t s_c8[32 * kTsThreads];  // set bits of each touched record
  constexpr int64_t kTile = kTsThreads;  // touch words per tile
  const int64_t tpr = (TW + kTile - 1) / kTile;
  const int64_t ntiles = tpr * k;
  for (;;) {
    if (threadIdx.x == 0) s_tile = (int64_t)atomicAdd(st, 1ull);
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile >= ntiles) return;
    const int64_t row = tile / tpr, seg = tile - row * tpr;
    uint4* r = rec + row * NR;
    const uint32_t* tw = touch + row * TW;
    const int64_t w0 = seg * kTile + (int64_t)threadIdx.x;  // a touch word per thread
    const uint32_t t = w0 < TW ? tw[w0] : 0u;
    // the word's touched records in order, kTouchB at a time: their loads in
    // flight together (one record load per iteration would serialise)
    auto each = [&](auto&& fn) {
      for (uint32_t m = t; m;) {
        int32_t idx[kTouchB];
        int nb = 0;
#pragma unroll
        for (int z = 0; z < kTouchB; ++z)
          if (m) {
            idx[z] = (int32_t)(w0 * 32) + __ffs(m) - 1;
            m &= m - 1;
            nb = z + 1;
          }
        uint4 x[kTouchB];
#pragma unroll
        for (int z = 0; z < kTouchB; ++z)
          if (z < nb) x[z] = r[idx[z]];
#pragma unroll
        for (int z = 0; z < kTouchB; ++z)
          if (z < nb) fn(idx[z], __popc(x[z].x) + __popc(x[z].y) + __popc(x[z].z));
      }
    };
    int csum = 0, nt = 0;
    each([&](int32_t, int c) {
      s_c8[nt++ * kTsThreads + threadIdx.x] = (uint8_t)c;  // <= 96 per record
      csum += c;
    });
    int64_t total;
    int64_t run = block_excl_scan<int64_t>(csum, sw, total);
    if (threadIdx.x < 32) {
      const int64_t pre = tile_lookback(st, tile, row * tpr, total);
      if (threadIdx.x == 0) s_prefix = pre;
    }
    __syncthreads();
    run += s_prefix;
    // prefixes from the counts kept in shared memory (no record reloads)
    uint32_t* r32 = reinterpret_cast<uint32_t*>(r);
    int j = 0;
    for (uint32_t m = t; m; m &= m - 1, ++j) {
      const int64_t i = w0 * 32 + __ffs(m) - 1;
      r32[4 * i + 3] = (uint32_t)run;
      run += s_c8[j * kTsThreads + threadIdx.x];
    }
    if (seg == tpr - 1 && threadIdx.x == 0) tot[row] = s_prefix + total;
    __syncthreads();
  }
}
// k_sage_enumerate128 over touched records; clears their bits and the touch
// words (the workspace's clean state)
__global__ void k_enum_touch(int64_t k, int64_t NR, uint4* __restrict__ rec,
                             uint32_t* __restrict__ touch, int64_t TW,
                             const int64_t* __restrict__ coloff, int32_t* __restrict__ colv) {
  for (int64_t wi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; wi < k * TW;
       wi += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t t = touch[wi];
    if (!t) continue;
    const int64_t bt = wi / TW, wr = wi - bt * TW;
    const int64_t cb = coloff[bt];
    for (uint32_t m = t; m;) {
      // kTouchB touched records at a time, their loads in flight together
      int32_t ri[kTouchB];
      int nb = 0;
#pragma unroll
      for (int z = 0; z < kTouchB; ++z)
        if (m) {
          ri[z] = (int32_t)(wr * 32) + __ffs(m) - 1;  // record within the batch row
          m &= m - 1;
          nb = z + 1;
        }
      uint4 x[kTouchB];
#pragma unroll
      for (int z = 0; z < kTouchB; ++z)
        if (z < nb) x[z] = rec[bt * NR + ri[z]];
#pragma unroll
      for (int z = 0; z < kTouchB; ++z) {
        if (z >= nb) break;
        const int32_t vb = ri[z] * 96;
        int32_t o = (int32_t)(cb + x[z].w);
        const uint32_t w[3] = {x[z].x, x[z].y, x[z].z};
#pragma unroll
        for (int j = 0; j < 3; ++j)
          for (uint32_t b = w[j]; b; b &= b - 1) colv[o++] = vb + 32 * j + __ffs(b) - 1;
        rec[bt * NR + ri[z]] = make_uint4(0u, 0u, 0u, x[z].w);
      }
    }
    touch[wi] = 0u;
  }
}

__global__ void k_layer_cols(const int64_t* __restrict__ brow, int64_t k,
                             const int64_t* __restrict__ fptr, const int64_t* __restrict__ tot,
                             int64_t* __restrict__ coloff, int64_t* __restrict__ sizes) {
  __shared__ int64_t sw[33];
  int64_t base = 0;
  for (int64_t b0 = 0; b0 < k; b0 += blockDim.x) {
    const int64_t b = b0 + threadIdx.x;
    int64_t total;
    const int64_t ex = block_excl_scan<int64_t>(b < k ? tot[b] : 0, sw, total);
    if (b < k) coloff[b] = base + ex;
    base += total;
  }
  if (threadIdx.x == 0) {
    coloff[k] = base;
    sizes[0] = brow[k];
    sizes[1] = fptr[brow[k]];
    sizes[2] = base;
  }
}

// acol[e] = coloff[batch] + record prefix + rank inside the record
// (compact_columns sparse.py:352-357 + block_diag :321-342); U entries per
// thread, their record loads issued together
#ifndef GB_RANK_U
#define GB_RANK_U 4
#endif
__global__ void k_sage_rank128(const int64_t* __restrict__ F_ptr, const int64_t* __restrict__ eoff,
                               const int64_t* __restrict__ coloff, int64_t k,
                               const int32_t* __restrict__ fcol, const uint4* __restrict__ rec,
                               int64_t NR, int32_t* __restrict__ acol) {
  constexpr int U = GB_RANK_U;  // entries per thread, loads in flight together (swept 2 / 4 / 6 / 8 / 16: 4 best)
  __shared__ int32_t s_eoff[kBrowSmem], s_col[kBrowSmem];
  const bool sm = k + 1 <= kBrowSmem;
  if (sm)
    for (int i = threadIdx.x; i <= k; i += blockDim.x) {
      s_eoff[i] = (int32_t)eoff[i];
      s_col[i] = (int32_t)coloff[i];
    }
  __syncthreads();
  const int32_t F = (int32_t)*F_ptr;
  const int32_t K = (int32_t)k, nr = (int32_t)NR;
  auto eo = [&](int32_t i) { return sm ? s_eoff[i] : (int32_t)eoff[i]; };
  for (int32_t e0 = blockIdx.x * blockDim.x * U + threadIdx.x; e0 < F;
       e0 += gridDim.x * blockDim.x * U) {
    int32_t v[U], bt[U];
    uint4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int32_t e = e0 + u * (int32_t)blockDim.x;
      v[u] = e < F ? fcol[e] : 0;
    }
    int32_t a = 0, b = K;  // last batch with eoff <= e0
    while (b - a > 1) {
      const int32_t mid = (a + b) >> 1;
      if (eo(mid) <= e0) a = mid; else b = mid;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int32_t e = e0 + u * (int32_t)blockDim.x;
      while (a + 1 < K && eo(a + 1) <= e) ++a;
      bt[u] = a;
      if (e < F) x[u] = rec[a * nr + (int32_t)(((uint32_t)v[u] >> 5) / 3u)];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int32_t e = e0 + u * (int32_t)blockDim.x;
      if (e < F) {
        const uint32_t w = (uint32_t)v[u] >> 5, j = w - 3u * (w / 3u);
        const uint32_t m = (1u << (v[u] & 31)) - 1u;
        const uint32_t wj = j == 0 ? x[u].x : j == 1 ? x[u].y : x[u].z;
        const int32_t below = (j > 0 ? __popc(x[u].x) : 0) + (j > 1 ? __popc(x[u].y) : 0);
        acol[e] = (sm ? s_col[bt[u]] : (int32_t)coloff[bt[u]]) + (int32_t)x[u].w + below +
                  __popc(wj & m);
      }
    }
  }
}

// col_vertices from the records, thread per record; clears the bits (the
// prefix word is rewritten by the next scan)
__global__ void k_sage_enumerate128(int64_t NRt, int64_t NR, uint4* __restrict__ rec,
                                    const int64_t* __restrict__ coloff,
                                    int32_t* __restrict__ colv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < NRt;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 r = rec[i];
    if (!(r.x | r.y | r.z)) continue;
    const int64_t bt = i / NR;
    const int32_t vb = (int32_t)((i - bt * NR) * 96);
    int32_t o = (int32_t)(coloff[bt] + r.w);
    const uint32_t w[3] = {r.x, r.y, r.z};
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      uint32_t x = w[j];
      while (x) {
        colv[o++] = vb + 32 * j + __ffs(x) - 1;
        x &= x - 1;
      }
    }
    rec[i] = make_uint4(0u, 0u, 0u, r.w);
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
  GB_CUDA(cudaMalloc(&g->run_sd, sizeof(double2) * sl * kMaxRuns));
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
                                                               g->run_sd, g->run_n,
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
  int32_t* pidx;     // stream mode: row-relative picks
  int32_t* deg;
  int64_t* gstart;
  int64_t* scan_ws;
  uint32_t* bitmap;   // (batch, vertex) bits and their popcount prefix, two sets:
  uint32_t* bitmap2;  // layer l's extraction overlaps layer l + 1's sampling
  int64_t* scan_ws2;  // scans of the extraction stream
  int64_t* d_W;
  int64_t* clean;    // clean mark after a completed bulk (bit words, counters clear)
  int64_t* btot;     // set bits per batch row (extraction)
  // dedup mode
  int32_t* vcnt;     // [n] rows per vertex (zero between layers)
  int32_t* roff;     // [n] group row range start per vertex
  int32_t* rslot;    // per frontier row: slot in its vertex group
  int32_t* dv;       // distinct row vertices (unordered)
  unsigned long long* cnts;  // [0] distinct count, [1..3] tier items, grouped rows
  unsigned int* ticket;      // serve kernels' work counters
  int64_t icap;      // work-item capacity per tier
  DdItem* items;     // work-item descriptors
  int4* rrec;        // per grouped row: (local row, degree, frontier offset, batch)
  uint32_t* touch;   // sparse extraction: touch bit per record, one set per bitmap set
  uint32_t* touch2;
  int64_t TW;        // touch words per batch row
  size_t bytes;
};

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

static SageWs sage_ws_layout(char* base, int64_t k, int64_t n, int64_t r_cap_max,
                             int64_t f_cap_max) {
  SageWs w{};
  const int64_t nwords = (n + 31) / 32;
  const int64_t W = k * 4 * ((nwords + 2) / 3);  // pk_word records: 16 B per 96 vertices
  int64_t scan_n = 3 * r_cap_max > W ? 3 * r_cap_max : W;
  if (nwords > scan_n) scan_n = nwords;
  size_t off = 0;
  auto take = [&](size_t bytes) { char* p = base ? base + off : nullptr; off += align_up(bytes); return p; };
  w.pidx = (int32_t*)take(sizeof(int32_t) * (f_cap_max + 1));
  w.deg = (int32_t*)take(sizeof(int32_t) * (r_cap_max + 1));
  w.gstart = (int64_t*)take(sizeof(int64_t) * (r_cap_max + 1));
  w.scan_ws = (int64_t*)take(sizeof(int64_t) * scan_workspace_elems<int64_t>(scan_n + 1));
  w.bitmap = (uint32_t*)take(sizeof(uint32_t) * (W + 8));
  w.bitmap2 = (uint32_t*)take(sizeof(uint32_t) * (W + 8));
  const int64_t NRr = (nwords + 2) / 3;  // bitmap records per batch row
  const int64_t rs_tiles = k * ((NRr + kRsTile - 1) / kRsTile) + 2;
  const int64_t sw2 = scan_workspace_elems<int64_t>(W + 1);
  w.scan_ws2 = (int64_t*)take(sizeof(int64_t) * (sw2 > rs_tiles ? sw2 : rs_tiles));
  w.d_W = (int64_t*)take(sizeof(int64_t));
  w.clean = (int64_t*)take(sizeof(int64_t));
  w.btot = (int64_t*)take(sizeof(int64_t) * (k + 1));
  w.vcnt = (int32_t*)take(sizeof(int32_t) * (n + 1));
  w.roff = (int32_t*)take(sizeof(int32_t) * (n + 1));
  w.rslot = (int32_t*)take(sizeof(int32_t) * (r_cap_max + 1));
  w.dv = (int32_t*)take(sizeof(int32_t) * (r_cap_max + 1));
  w.cnts = (unsigned long long*)take(sizeof(unsigned long long) * 8);
  w.ticket = (unsigned int*)take(sizeof(unsigned int) * 8);
  // items <= groups + rows / rows_item(min) <= 2 * rows, per tier region
  w.icap = 2 * r_cap_max + 2;
  w.items = (DdItem*)take(sizeof(DdItem) * 3 * w.icap);
  w.rrec = (int4*)take(sizeof(int4) * (r_cap_max + 1));
  w.TW = (NRr + 31) / 32;
  w.touch = (uint32_t*)take(sizeof(uint32_t) * (k * w.TW + 1));
  w.touch2 = (uint32_t*)take(sizeof(uint32_t) * (k * w.TW + 1));
  w.bytes = off;
  return w;
}

__global__ void k_sage_eoff(const int64_t* __restrict__ brow, int64_t k,
                            const int64_t* __restrict__ fptr, int64_t* __restrict__ eoff);

constexpr int64_t kWsClean = 0x636c65616e6d6b31LL;
// the clean mark certifies one layout (bitmap and counter sizes)
__host__ __device__ __forceinline__ int64_t ws_clean_mark(int64_t nb, int64_t nv) {
  return kWsClean ^ (nb * 0x9E3779B97F4A7C15LL) ^ (nv << 17);
}
__global__ void k_ws_clear(const int64_t* __restrict__ clean, uint32_t* __restrict__ b1,
                           uint32_t* __restrict__ b2, int64_t nb, int32_t* __restrict__ vcnt,
                           int64_t nv, uint32_t* __restrict__ t1, uint32_t* __restrict__ t2,
                           int64_t nt) {
  if (*clean == ws_clean_mark(nb, nv)) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nb;
       i += (int64_t)gridDim.x * blockDim.x) {
    b1[i] = 0u;
    b2[i] = 0u;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nt;
       i += (int64_t)gridDim.x * blockDim.x) {
    t1[i] = 0u;
    t2[i] = 0u;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * blockDim.x)
    vcnt[i] = 0;
}

template <typename K>
static int persistent_grid(K kernel, int threads, size_t smem = 0) {
  int o = 0, dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kernel, threads, smem);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (o < 1 ? 1 : o) * (sms > 0 ? sms : kNumSMs);
}

// Per-device launch configuration of the dedup kernels (attributes are per
// device; grids from the occupancy of the current device).
constexpr int kMaxDevices = 16;
struct ServeCfg {
  bool init = false;
  DdTiers tiers{1536, 4096};
  // a vertex's rows read their picks in place when rows x take x ratio <
  // 8 d (0: always staged)
  // peer rows (1.5D split): direct rows read their picks from the owner's
  // memory over NVLink instead of staging the row (GB_PEER_DIRECT=0/1)
  bool peer_direct = true;
  int32_t direct_ratio = 2;  // swept 1 / 2 / 4 / 8
  int grid[3] = {0, 0, 0};
  int chunk[3] = {0, 0, 0};
  size_t smem[3] = {0, 0, 0};
};
static ServeCfg g_serve[kMaxDevices];

template <int T>
static void serve_tier_setup(ServeCfg& c, int max_smem) {
  using Tr = DdTier<T>;
  // tier 0: a row buffer (+ group table) per warp; tier 1: the whole row;
  // tier 2: all of shared memory (chunks) but the static mbarrier
  c.chunk[T] = T == 2 ? (((max_smem - 256) / 4 - 8) & ~3) : T == 0 ? c.tiers.hi0 : c.tiers.hi1;
  c.smem[T] = sizeof(int32_t) * (c.chunk[T] + 8 + (Tr::kWarp ? kGrpInts : 0)) *
              (Tr::kWarp ? Tr::kThreads / 32 : 1);
  cudaFuncSetAttribute(k_dd_serve<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)c.smem[T]);
  c.grid[T] = persistent_grid(k_dd_serve<T>, Tr::kThreads, c.smem[T]);
}

static ServeCfg& serve_cfg() {
  int dev = 0;
  cudaGetDevice(&dev);
  ServeCfg& c = g_serve[dev < kMaxDevices ? dev : 0];
  if (!c.init) {
    int max_smem = 0;
    cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (max_smem <= 0) max_smem = 227 * 1024;
    // tier bounds (GB_SERVE_TIERS="hi0,hi1" overrides, for tuning sweeps)
    if (const char* e = getenv("GB_SERVE_TIERS")) {
      int a = 0, b2 = 0;
      if (sscanf(e, "%d,%d", &a, &b2) == 2 && a >= 16 && b2 > a && b2 <= 16384) {
        c.tiers.hi0 = a & ~3;
        c.tiers.hi1 = b2 & ~3;
      }
    }
    if (const char* e = getenv("GB_PEER_DIRECT")) c.peer_direct = atoi(e) != 0;
    serve_tier_setup<0>(c, max_smem);
    serve_tier_setup<1>(c, max_smem);
    serve_tier_setup<2>(c, max_smem);
    c.init = true;
  }
  return c;
}

// staged/direct threshold: GB_DIRECT_RATIO read per bulk (tests force either)
static int32_t direct_ratio() {
  const char* e = getenv("GB_DIRECT_RATIO");
  if (!e) return serve_cfg().direct_ratio;
  const int v = atoi(e);
  return v > 0 ? v : 0;
}

// per distinct vertex: work items and group row ranges (k_grp_items); runs
// on its own stream next to the frontier-offset scan
static int launch_items(const Graph* g, SageWs& ws, int32_t s, int64_t r_cap,
                        const PeerRows& peer, cudaStream_t st) {
  const int64_t gw = GB_GRP_GRID * kNumSMs;
  k_grp_items<<<grid_for((r_cap < g->n ? r_cap : g->n + 0) / kGrpU + 1, kItemThreads, gw),
                kItemThreads, 0, st>>>(
      ws.cnts, ws.dv, g->rowptr, ws.vcnt, ws.roff, s, ws.icap, ws.cnts + 1, ws.items, peer,
      serve_cfg().tiers, direct_ratio(), serve_cfg().peer_direct);
  GB_LAUNCH_CHECK("k_grp_items");
  return GB_OK;
}

static int fan_bucket(int32_t s) { return s <= 5 ? 0 : s <= 8 ? 1 : s <= 10 ? 2 : s <= 16 ? 3 : 4; }

// One dedup layer: grouping (count already ran; items, rows), NORM + SAMPLE
// per grouped row, then the serve kernels (tier A bins, tier B chunks on a
// forked stream; they touch disjoint frontier entries and commutative
// bitmap ORs).
static int dedup_layer(const Graph* g, SageWs& ws, const int64_t* R_ptr, const int32_t* rowv,
                       const int64_t* fptr, const int64_t* brow, int64_t k, int32_t s,
                       int64_t stride, int64_t batch_offset, uint64_t seed, uint64_t epoch,
                       uint64_t depth, int64_t r_cap, const PeerRows& peer, int32_t* fcol,
                       uint32_t* bitmap, int64_t nwords8, cudaStream_t st) {
  const int64_t gw = GB_GRP_GRID * kNumSMs;
  k_grp_rows<<<grid_for(r_cap / kGrpU + 1, 256, gw), 256, 0, st>>>(R_ptr, rowv, ws.deg, fptr,
                                                                   brow, k, ws.rslot, ws.roff,
                                                                   ws.rrec);
  GB_LAUNCH_CHECK("k_grp_rows");
  const ServeCfg& c = serve_cfg();
  const SageTabs T{g->deg_slot, g->run_j0, g->run_sd, g->run_n, g->run_lower};
  const int b = fan_bucket(s);
  const int pgrid = grid_for(r_cap, kPickThreads, GB_PICK_GRID * kNumSMs);
  const unsigned long long* grows = ws.cnts + 4;
  prof_mark(st);
  const DdPickOut PO{ws.pidx, g->rowptr, g->col, fcol, bitmap, nwords8, peer};
#define GB_DD_PICK(MF)                                                                   \
  k_dd_pick<MF><<<pgrid, kPickThreads, 0, st>>>(grows, ws.rrec, T, s, batch_offset, stride, \
                                               seed, epoch, depth, PO)
  switch (b) {
    case 0: GB_DD_PICK(5); break;
    case 1: GB_DD_PICK(8); break;
    case 2: GB_DD_PICK(10); break;
    case 3: GB_DD_PICK(16); break;
    default: GB_DD_PICK(32); break;
  }
#undef GB_DD_PICK
  GB_LAUNCH_CHECK("k_dd_pick");
  prof_mark(st);
  DdArgs A{};
  A.col = peer.nblk ? nullptr : g->col;
  A.tcnt = ws.cnts + 1;
  A.icap = ws.icap;
  A.items = ws.items;
  A.rrec = ws.rrec;
  A.pidx = ws.pidx;
  A.s = s;
  A.fcol = fcol;
  A.bitmap = bitmap;
  A.nwords = nwords8;
  prof_mark(st);
  // the tiers touch disjoint frontier entries (and commutative bitmap ORs):
  // run them concurrently so each tier's tail overlaps the others
  fork_begin(st, 2);
  A.chunk = c.chunk[0];
  k_dd_serve<0><<<c.grid[0], DdTier<0>::kThreads, c.smem[0], st>>>(A);
  GB_LAUNCH_CHECK("k_dd_serve<0>");
  A.chunk = c.chunk[1];
  k_dd_serve<1><<<c.grid[1], DdTier<1>::kThreads, c.smem[1], fork_stream(0)>>>(A);
  GB_LAUNCH_CHECK("k_dd_serve<1>");
  A.chunk = c.chunk[2];
  k_dd_serve<2><<<c.grid[2], DdTier<2>::kThreads, c.smem[2], fork_stream(1)>>>(A);
  GB_LAUNCH_CHECK("k_dd_serve<2>");
  fork_join(st, 2);
  prof_mark(st);
  count_launches(6);  // items, rows, pick, serve x3
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

static int stream_grid() {
  static int g[kMaxDevices] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  int& x = g[dev < kMaxDevices ? dev : 0];
  if (!x) x = persistent_grid(k_sage_stream, kStreamThreads);
  return x;
}

// first layer sampled by the dedup kernels in dedup mode (GB_DEDUP_FROM
// overrides, for sweeps)
static int dedup_from() {
  const char* e = getenv("GB_DEDUP_FROM");  // read per bulk (tests force either way)
  const int v = e ? atoi(e) : 1;
  return v < 0 ? 0 : v;
}

// Grouping a layer's rows by vertex pays when they repeat vertices: when
// the layer's row bound reaches GB_GROUP_RATIO (default 0.25) x n.  Measured:
// products layer 3 (bound 4 n) grouped 0.58 vs 0.66 ms; papers layer 3
// (bound 0.09 n: 1.46M rows over 0.93M vertices) P-free 1.59 vs 1.89 ms
// per bulk.
static bool group_pays(int64_t r_cap, int64_t n) {
  const char* e = getenv("GB_GROUP_RATIO");  // read per bulk (tests force either way)
  const double ratio = e ? atof(e) : 0.25;
  return (double)r_cap >= ratio * (double)n;
}

int sage_bulk(const Graph* g, int64_t k, const int64_t* d_bptr, const int32_t* d_bverts,
              int64_t r1_cap, int64_t batch_size, int32_t layers, const int64_t* fanouts,
              uint64_t seed, uint64_t epoch, int64_t batch_offset, int32_t mode,
              gb_sage_layer_out* L, int64_t* d_sizes, void* d_ws, size_t ws_bytes,
              cudaStream_t st, const PeerRowsHost* peer_host) {
  const bool stream = mode == GB_SAGE_STREAM;
  const bool dedup = mode == GB_SAGE_DEDUP;
  PeerRows peer{0, nullptr, nullptr, nullptr};
  if (peer_host) {
    if (!dedup) {
      set_error("sage bulk: peer rows need the dedup mode");
      return GB_ERR_UNSUPPORTED;
    }
    peer = PeerRows{peer_host->nblk, peer_host->bounds, peer_host->brp, peer_host->bcol};
    for (int32_t l = 0; l < layers; ++l)
      if (fanouts[l] > 32) {
        set_error("sage bulk: peer rows support fanouts up to 32");
        return GB_ERR_UNSUPPORTED;
      }
  }
  const int64_t nwords = (g->n + 31) / 32;
  // (batch, vertex) bitmaps as pk_word records (3 bit words, prefix)
  const int64_t NR = (nwords + 2) / 3;  // records per batch row
  const int64_t nw8 = 4 * NR;           // uint32 per batch row
  const int64_t W = k * nw8, NS = k * NR;
  if (W >= ((int64_t)1 << 31)) {
    set_error("bulk: k * ceil(n / 32) = %lld (batch, vertex) words exceeds int32 indexing",
              (long long)W);
    return GB_ERR_UNSUPPORTED;
  }
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
  // the bit words and vertex counters are left clear by a completed bulk
  // (enumerate / items clear what they used): zero them only when the
  // workspace's clean mark is absent (first use, or an aborted bulk)
  k_ws_clear<<<4 * kNumSMs, 256, 0, st>>>(ws.clean, ws.bitmap, ws.bitmap2, W + 8, ws.vcnt,
                                         g->n + 1, ws.touch, ws.touch2, k * ws.TW + 1);
  GB_LAUNCH_CHECK("k_ws_clear");
  k_set_i64<<<1, 1, 0, st>>>(ws.d_W, NS);
  k_set_i64<<<1, 1, 0, st>>>(ws.clean, 0);
  count_launches(3);
  // sparse extraction (touched records only) when the (batch, vertex) bit
  // rows are long: n >= 2^23 (papers shape: 1.2 GB of records per layer for
  // a few million set bits); GB_SPARSE_EXTRACT=0/1 forces either
  bool sparse = g->n >= ((int64_t)1 << 23);
  if (const char* e = getenv("GB_SPARSE_EXTRACT")) sparse = atoi(e) != 0;
  // extraction of layer l (popcount scan, rank, enumerate) runs on a side
  // stream while layer l + 1 samples; layer l + 2 reuses layer l's bitmap
  // only after that extraction (ring events) — graph-capturable
  const cudaStream_t xs = fork_stream(2);
  int64_t stride = batch_size;
  r_cap = r1_cap;
  for (int32_t l = 0; l < layers; ++l) {
    const int32_t d = l + 1;
    if (l > 0) stride *= fanouts[l - 1];
    gb_sage_layer_out& o = L[l];
    const int32_t s = (int32_t)fanouts[l];
    // fanouts above 32 take the P-free thread-per-row kernel in every mode;
    // dedup mode samples its first dedup_from() layers P-free too (the seed
    // rows repeat little across batches, so the grouping pass costs more
    // than the shared rows save — measured)
    const bool big = s > 32;
    const bool ldedup = dedup && !big && l >= dedup_from() && group_pays(r_cap, g->n);
    const bool lstream = stream && !big;
    const int32_t* rowv = l == 0 ? d_bverts : L[l - 1].fcol;
    const int64_t* brow = l == 0 ? d_bptr : L[l - 1].eoff;
    const int64_t* R_ptr = brow + k;
    uint32_t* bm = (l & 1) ? ws.bitmap2 : ws.bitmap;
    if (l >= 2) GB_CUDA(cudaStreamWaitEvent(st, ring_event(l - 2), 0));
    if (ldedup) {
      GB_CUDA(cudaMemsetAsync(ws.cnts, 0, sizeof(unsigned long long) * 8, st));
      GB_CUDA(cudaMemsetAsync(ws.ticket, 0, sizeof(unsigned int) * 8, st));
      k_grp_count<<<grid_for(r_cap / kGrpU + 1, kGrpThreads, GB_GRP_GRID * kNumSMs), kGrpThreads, 0, st>>>(
          R_ptr, rowv, g->rowptr, ws.deg, ws.vcnt, ws.rslot, ws.dv, ws.cnts);
      GB_LAUNCH_CHECK("k_grp_count");
    } else {
      k_sage_prep<<<grid_for(r_cap, 256, 16 * kNumSMs), 256, 0, st>>>(R_ptr, rowv, g->rowptr,
                                                                       ws.deg, nullptr);
      GB_LAUNCH_CHECK("k_sage_prep");
    }
    // the distinct vertices' items (dedup) overlap the frontier-offset scan
    if (ldedup) {
      fork_begin(st, 1);
      int rc0 = launch_items(g, ws, s, r_cap, peer, fork_stream(0));
      if (rc0) return rc0;
    }
    int rc = device_exclusive_scan<int64_t>(R_ptr, r_cap, TakeF{ws.deg, s}, o.fptr, ws.scan_ws, st);
    if (rc) return rc;
    if (ldedup) fork_join(st, 1);
    if (lstream) {
      rc = device_exclusive_scan<int64_t>(R_ptr, r_cap, DegF{ws.deg}, ws.gstart, ws.scan_ws, st);
      if (rc) return rc;
    }
    if (ldedup) {
      rc = dedup_layer(g, ws, R_ptr, rowv, o.fptr, brow, k, s, stride, batch_offset, seed, epoch,
                       (uint64_t)d, r_cap, peer, o.fcol, bm, nw8, st);
      if (rc) return rc;
    } else {
      SageArgs A{};
      A.rowptr = g->rowptr; A.col = g->col; A.peer = peer;
      A.deg_slot = g->deg_slot; A.run_j0 = g->run_j0; A.run_sd = g->run_sd;
      A.run_n = g->run_n; A.run_lower = g->run_lower;
      A.rowv = rowv; A.deg = ws.deg; A.fptr = o.fptr; A.gstart = ws.gstart;
      A.brow = brow; A.k = k; A.s = s; A.stride = stride; A.batch_offset = batch_offset;
      A.seed = seed; A.epoch = epoch; A.depth = (uint64_t)d;
      A.bitmap = bm; A.nwords = nw8; A.fcol = o.fcol; A.pidx = ws.pidx;
      const int pick_grid = grid_for(r_cap, kPickThreads, GB_PICK_GRID * kNumSMs);
      prof_mark(st);
      if (big)
        k_sage_pick_big<<<pick_grid, kPickThreads, 0, st>>>(A, R_ptr);
      else if (lstream)
        launch_pick<0>(pick_grid, A, R_ptr, st);
      else
        launch_pick<1>(pick_grid, A, R_ptr, st);
      GB_LAUNCH_CHECK("k_sage_pick");
      prof_mark(st);
      if (lstream) {
        prof_mark(st);
        k_sage_stream<<<stream_grid(), kStreamThreads, 0, st>>>(A, R_ptr);
        GB_LAUNCH_CHECK("k_sage_stream");
        prof_mark(st);
        count_launches(1);
      } else if (dedup) {  // P-free layer of a dedup bulk: empty serve interval
        prof_mark(st);
        prof_mark(st);
      }
      count_launches(1);
    }
    // next layer's batch row offsets, on the sampling stream
    k_sage_eoff<<<grid_for(k + 1, 128, 64), 128, 0, st>>>(brow, k, o.fptr, o.eoff);
    GB_LAUNCH_CHECK("k_sage_eoff");
    stream_wait(xs, st);
    // per batch row: record prefixes and the row total; column offsets
    int64_t* sizes = d_sizes + 3 * l;
    uint32_t* tch = (l & 1) ? ws.touch2 : ws.touch;
    const int64_t f_cap0 = r_cap * s;
    if (k > 0 && sparse) {
      k_touch<<<grid_for(f_cap0, 256, 16 * kNumSMs), 256, 0, xs>>>(brow, o.fptr, o.eoff, k,
                                                                  o.fcol, ws.TW, tch);
      GB_LAUNCH_CHECK("k_touch");
      const int64_t ttiles = k * ((ws.TW + kTsThreads - 1) / kTsThreads);
      GB_CUDA(cudaMemsetAsync(ws.scan_ws2, 0, sizeof(int64_t) * (ttiles + 2), xs));
      k_rec_scan_touch<<<grid_for(ttiles, 1, GB_TS_GRID * kNumSMs), kTsThreads, 0, xs>>>(
          (uint4*)bm, NR, k, tch, ws.TW, ws.btot, (unsigned long long*)ws.scan_ws2);
      GB_LAUNCH_CHECK("k_rec_scan_touch");
      count_launches(2);
    } else if (k > 0) {
      const int64_t rtiles = k * ((NR + kRsTile - 1) / kRsTile);
      GB_CUDA(cudaMemsetAsync(ws.scan_ws2, 0, sizeof(int64_t) * (rtiles + 2), xs));
      k_rec_scan<<<grid_for(rtiles, 1, GB_RS_GRID * kNumSMs), kRsThreads, 0, xs>>>(
          (uint4*)bm, NR, k, ws.btot, (unsigned long long*)ws.scan_ws2);
      GB_LAUNCH_CHECK("k_rec_scan");
      count_launches(1);
    }
    k_layer_cols<<<1, 1024, 0, xs>>>(brow, k, o.fptr, ws.btot, o.coloff, sizes);
    GB_LAUNCH_CHECK("k_layer_cols");
    const int64_t f_cap = r_cap * s;
    k_sage_rank128<<<grid_for(f_cap / GB_RANK_U + 1, 256, GB_X_GRID * kNumSMs), 256, 0, xs>>>(
        sizes + 1, o.eoff, o.coloff, k, o.fcol, (const uint4*)bm, NR, o.acol);
    GB_LAUNCH_CHECK("k_sage_rank128");
    if (sparse) {
      k_enum_touch<<<grid_for(k * ws.TW, 256, GB_ET_GRID * kNumSMs), 256, 0, xs>>>(
          k, NR, (uint4*)bm, tch, ws.TW, o.coloff, o.colv);
      GB_LAUNCH_CHECK("k_enum_touch");
    } else {
      k_sage_enumerate128<<<grid_for(NS, 256, GB_X_GRID * kNumSMs), 256, 0, xs>>>(NS, NR, (uint4*)bm,
                                                                           o.coloff, o.colv);
      GB_LAUNCH_CHECK("k_sage_enumerate128");
    }
    GB_CUDA(cudaEventRecord(ring_event(l), xs));
    count_launches(5);  // prep/count, eoff, cols, rank, enumerate
    r_cap = f_cap;
  }
  stream_wait(st, xs);
  k_set_i64<<<1, 1, 0, st>>>(ws.clean, ws_clean_mark(W + 8, g->n + 1));
  count_launches(1);
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
  A.deg_slot = tables->deg_slot; A.run_j0 = tables->run_j0; A.run_sd = tables->run_sd;
  A.run_n = tables->run_n; A.run_lower = tables->run_lower;
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
  A.deg_slot = tables->deg_slot; A.run_j0 = tables->run_j0; A.run_sd = tables->run_sd;
  A.run_n = tables->run_n; A.run_lower = tables->run_lower;
  A.rowv = rowv; A.rowkeys = rowkeys; A.deg = deg; A.fptr = fptr;
  A.k = 0; A.s = s; A.seed = seed; A.epoch = epoch; A.depth = depth;
  A.bitmap = nullptr; A.fcol = fcol;
  launch_pick<1>(grid_for(R, kPickThreads, 64 * kNumSMs), A, d_R, st);
  GB_LAUNCH_CHECK("sage_sample_keyed");
  count_launches(1);
  return GB_OK;
}

// ------------------------------------------ owner sampling over peer memory
// 1.5D owner-computes with the exchange fused into the kernels: the owner of
// a block reads the requesting grid row's frontier, batch offsets and
// frontier offsets straight from that rank's memory (P2P loads over NVLink),
// keeps the rows whose vertex lies in its block, samples them from its local
// block with the requester's keys, and stores the picks into the frontier of
// every replica of that grid row (P2P stores) — no request / reply messages
// and no all-reduce.  Caller brackets it with device barriers.

// rows of a requester whose vertex lies in [lo, hi): block-local row,
// degree, global row key and frontier offset (order arbitrary)
__global__ void k_p2p_rows(const int32_t* __restrict__ rows, const int64_t* __restrict__ brow,
                           const int64_t* __restrict__ fptr, int64_t k, int64_t boff,
                           int64_t stride, int64_t lo, int64_t hi,
                           const int64_t* __restrict__ brp, int32_t* __restrict__ lrow,
                           int32_t* __restrict__ ldeg, int64_t* __restrict__ lkey,
                           int64_t* __restrict__ lpos, int64_t* __restrict__ count) {
  __shared__ int64_t s_brow[kBrowSmem];
  if (k + 1 <= kBrowSmem)
    for (int64_t i = threadIdx.x; i <= k; i += blockDim.x) s_brow[i] = brow[i];
  __syncthreads();
  const int64_t R = brow[k];
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = rows[r];
    if (v < lo || v >= hi) continue;
    const int64_t lr = v - lo;
    const int32_t d = (int32_t)(brp[lr + 1] - brp[lr]);
    if (d == 0) continue;
    const int64_t b = batch_of(s_brow, brow, k, r);
    const int64_t b0 = k + 1 <= kBrowSmem ? s_brow[b] : brow[b];
    const unsigned peers = __activemask();
    const int lane = lane_id(), leader = __ffs(peers) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd((unsigned long long*)count, (unsigned long long)__popc(peers));
    base = __shfl_sync(peers, base, leader);
    const int64_t o = (int64_t)base + __popc(peers & ((1u << lane) - 1u));
    lrow[o] = (int32_t)lr;
    ldeg[o] = d;
    lkey[o] = (boff + b) * stride + (r - b0);
    lpos[o] = fptr[r];
  }
}

size_t sage_owner_p2p_ws(int64_t r_cap) {
  return 2 * align_up(sizeof(int32_t) * (r_cap + 1)) + 2 * align_up(sizeof(int64_t) * (r_cap + 1)) +
         align_up(sizeof(int64_t) * 2);
}

int sage_owner_p2p(const Graph* tables, int64_t ngroups, const int32_t* const* rows,
                   const int64_t* const* brow, const int64_t* const* fptr, const int64_t* boff,
                   int64_t k, int64_t r_cap, int32_t ndst, int32_t* const* dst, int64_t lo,
                   int64_t hi, const int64_t* brp, const int32_t* bcol, int32_t s, int64_t stride,
                   uint64_t seed, uint64_t epoch, uint64_t depth, void* d_ws, size_t ws_bytes,
                   cudaStream_t st) {
  if (sage_owner_p2p_ws(r_cap) > ws_bytes) {
    set_error("owner p2p workspace too small");
    return GB_ERR_CAPACITY;
  }
  if (ndst < 1 || ndst > 8) {
    set_error("owner p2p: 1..8 destination frontiers per grid row");
    return GB_ERR_UNSUPPORTED;
  }
  char* p = (char*)d_ws;
  auto carve = [&](size_t bytes) { char* r = p; p += align_up(bytes); return r; };
  int32_t* lrow = (int32_t*)carve(sizeof(int32_t) * (r_cap + 1));
  int32_t* ldeg = (int32_t*)carve(sizeof(int32_t) * (r_cap + 1));
  int64_t* lkey = (int64_t*)carve(sizeof(int64_t) * (r_cap + 1));
  int64_t* lpos = (int64_t*)carve(sizeof(int64_t) * (r_cap + 1));
  int64_t* count = (int64_t*)carve(sizeof(int64_t) * 2);
  for (int64_t g = 0; g < ngroups; ++g) {
    GB_CUDA(cudaMemsetAsync(count, 0, sizeof(int64_t), st));
    k_p2p_rows<<<grid_for(r_cap, 256, 16 * kNumSMs), 256, 0, st>>>(
        rows[g], brow[g], fptr[g], k, boff[g], stride, lo, hi, brp, lrow, ldeg, lkey, lpos, count);
    GB_LAUNCH_CHECK("k_p2p_rows");
    SageArgs A{};
    A.rowptr = brp; A.col = bcol;
    A.deg_slot = tables->deg_slot; A.run_j0 = tables->run_j0; A.run_sd = tables->run_sd;
    A.run_n = tables->run_n; A.run_lower = tables->run_lower;
    A.rowv = lrow; A.rowkeys = lkey; A.deg = ldeg; A.fptr = lpos;
    A.k = 0; A.s = s; A.seed = seed; A.epoch = epoch; A.depth = depth;
    A.bitmap = nullptr; A.fcol = nullptr;
    A.ndst = ndst;
    for (int m = 0; m < ndst; ++m) A.dst[m] = dst[g * ndst + m];
    launch_pick<1>(grid_for(r_cap, kPickThreads, 64 * kNumSMs), A, count, st);
    GB_LAUNCH_CHECK("owner p2p pick");
    count_launches(2);
  }
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
  if (W >= ((int64_t)1 << 31) || f_cap >= ((int64_t)1 << 31)) {
    set_error("extract: k * ceil(n / 32) and the entry bound must stay below 2^31");
    return GB_ERR_UNSUPPORTED;
  }
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
// Rows ids[i] (block rows, row0-relative) copied to out[out_off[i] ..) (the
// block may live in a peer's memory: NVLink round trips).  Work items are
// chunks of at most kGatherChunk entries — their offsets an exclusive scan
// of the rows' chunk counts — so a hub row is copied by many warps instead
// of being walked by one (measured: one 148K-entry row set the whole
// fetch's time); a warp per item, 8 loads in flight per lane.
constexpr int kGatherChunk = 2048;
struct GatherChunksF {
  const int32_t* ids;
  int64_t row0;
  const int64_t* rowptr;
  __device__ int64_t operator()(int64_t i) const {
    const int64_t r = ids[i] - row0;
    const int64_t d = rowptr[r + 1] - rowptr[r];
    return d > 0 ? (d + kGatherChunk - 1) / kGatherChunk : 0;
  }
};
__global__ void k_gather_rows(int64_t m, const int32_t* __restrict__ ids, int64_t row0,
                              const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                              const int64_t* __restrict__ out_off, int32_t* __restrict__ out,
                              const int64_t* __restrict__ coff) {
  const int lane = lane_id();
  const int64_t nitems = coff[m];
  for (int64_t it = global_warp(); it < nitems; it += grid_warps()) {
    int64_t lo = 0, hi = m;  // last row with coff <= it
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (coff[mid] <= it) lo = mid; else hi = mid;
    }
    const int64_t r = ids[lo] - row0;
    const int64_t a = rowptr[r], d = rowptr[r + 1] - a, o = out_off[lo];
    const int64_t x0 = (it - coff[lo]) * kGatherChunk;
    const int64_t x1 = min(d, x0 + kGatherChunk);
    for (int64_t x = x0 + lane; x < x1; x += 256) {
      int32_t v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = x + 32 * u < x1 ? col[a + x + 32 * u] : 0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (x + 32 * u < x1) out[o + x + 32 * u] = v[u];
    }
  }
}
int gather_rows(int64_t m, const int32_t* ids, int64_t row0, const int64_t* rowptr,
                const int32_t* col, const int64_t* out_off, int32_t* out, cudaStream_t st) {
  if (m == 0) return GB_OK;
  // chunk offsets (m + 1), the scan length and its workspace from the
  // device's stream-ordered pool, which keeps its memory between calls
  static bool pool_set[16] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!pool_set[dev & 15]) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    pool_set[dev & 15] = true;
  }
  const size_t sw = scan_workspace_elems<int64_t>(m + 1);
  int64_t* scratch = nullptr;
  GB_CUDA(cudaMallocAsync((void**)&scratch, sizeof(int64_t) * (m + 2 + sw), st));
  int64_t* coff = scratch;
  int64_t* d_m = scratch + m + 1;
  k_set_i64<<<1, 1, 0, st>>>(d_m, m);
  int rc = device_exclusive_scan<int64_t>(d_m, m, GatherChunksF{ids, row0, rowptr}, coff,
                                          scratch + m + 2, st);
  if (rc) return rc;
  k_gather_rows<<<16 * kNumSMs, 256, 0, st>>>(m, ids, row0, rowptr, col, out_off, out, coff);
  GB_LAUNCH_CHECK("k_gather_rows");
  GB_CUDA(cudaFreeAsync(scratch, st));
  count_launches(2);
  return GB_OK;
}

// dense feature rows: out[i, :] = H[ids[i] - row0, :] (fp32, f columns)
// rows of H (fp32, f wide) for ids: a warp moves kGU rows per step with all
// their loads issued first (16-B vectors when f % 4 == 0 and aligned), so a
// remote (peer-memory) H keeps several NVLink requests in flight per warp
constexpr int kGU = 4;
template <bool V4>
__global__ void k_gather_feat(int64_t m, const int32_t* __restrict__ ids, int64_t row0,
                              const float* __restrict__ H, int64_t f, float* __restrict__ out) {
  const int lane = lane_id();
  constexpr int W = V4 ? 128 : 32;
  for (int64_t i0 = global_warp() * (int64_t)kGU; i0 < m; i0 += (int64_t)grid_warps() * kGU) {
    int64_t src[kGU];
#pragma unroll
    for (int u = 0; u < kGU; ++u) src[u] = i0 + u < m ? ((int64_t)ids[i0 + u] - row0) * f : -1;
    for (int64_t f0 = 0; f0 < f; f0 += W) {
      const int64_t x = f0 + (V4 ? 4 * lane : lane);
      float4 v[kGU];
#pragma unroll
      for (int u = 0; u < kGU; ++u) {
        v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (src[u] >= 0 && x < f) {
          if (V4) v[u] = __ldg((const float4*)(H + src[u] + x));
          else v[u].x = __ldg(H + src[u] + x);
        }
      }
#pragma unroll
      for (int u = 0; u < kGU; ++u)
        if (src[u] >= 0 && x < f) {
          float* d = out + (i0 + u) * f + x;
          if (V4) *(float4*)d = v[u];
          else *d = v[u].x;
        }
    }
  }
}

int gather_features(int64_t m, const int32_t* ids, int64_t row0, const float* H, int64_t f,
                    float* out, cudaStream_t st) {
  if (m == 0) return GB_OK;
  const bool v4 = f % 4 == 0 && (uintptr_t)H % 16 == 0 && (uintptr_t)out % 16 == 0;
  const int grid = grid_for((m + kGU - 1) / kGU * 32, 256, 16 * kNumSMs);
  if (v4)
    k_gather_feat<true><<<grid, 256, 0, st>>>(m, ids, row0, H, f, out);
  else
    k_gather_feat<false><<<grid, 256, 0, st>>>(m, ids, row0, H, f, out);
  GB_LAUNCH_CHECK("k_gather_feat");
  count_launches(1);
  return GB_OK;
}

}  // namespace gb
