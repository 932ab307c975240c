// LADIES layer-wise bulk sampling (Alg. 1 with Q^l = one row per batch),
// sm_100a.  Reference: sample_epoch_bulk LADIES path
// (pkg/src/gnnbulk/sampler.py:325-387, 420-462, 475-483).
//
// Per layer, for the k batches:
//   P = Q^l A   row i = sum of the A rows of batch i's vertex set: counts
//               e_v (spgemm sparse.py:233-251 on 0/1 values).  Batches are
//               processed in groups whose packed 16-bit count vectors stay
//               L2-resident (e_v <= |Q_i|); warps stream the gathered rows,
//               merge-path balanced over (rows, entries), and accumulate with
//               atomics on the packed counters.
//   NORM        w_v = fl(e_v^2 / sum e^2) (norm_rows_ladies sparse.py:263-286).
//   SAMPLE      min(s, N_i) distinct columns per batch:
//               GB_LADIES_EXACT — its_sample_row replayed literally
//                 (sequential fp64 cumsum per draw, searchsorted right, clamp,
//                 walk back; sampler.py:176-188) with the keyed uniforms:
//                 bit-exact, O(s N) serial per batch, small graphs;
//               GB_LADIES_RACE — exponential race (Gumbel top-s):
//                 key_v = E_v / e_v^2, E_v ~ Exp(1), the s smallest keys (multi-CTA
//                 histogram radix select).  Same law as successive sampling
//                 without replacement; validated statistically.
//   EXTRACT     A_S row (batch i, u) = sorted intersection A[u,:] ∩ S_i with
//               ranks (build_column_extraction sparse.py:430-446,
//               ladies_assemble sampler.py:420-434): one warp per row with S_i
//               in shared memory — short rows binary-search S_i per entry,
//               long (hub) rows binary-search A[u,:] per sampled vertex.
//               Shared column layout when every batch took the same count,
//               else block diagonal.
#include "gb_common.cuh"
#include "gb_internal.h"
#include "gb_scan.cuh"

namespace gb {

constexpr int kLadiesThreads = 256;
constexpr int kLadiesSizes = 5;     // per layer: A_S rows, F, A_S nnz, A_S cols, nnz(P)
constexpr int kLRowCost = 32;       // merge-path weight of one Q row
constexpr int kBins = 4096;         // radix-select histogram (12 bits)
constexpr int kTies = 2048;
constexpr int64_t kGroupBytes = 64ll << 20;  // packed counters of one group (L2-resident)
constexpr int kSmaxSmem = 1024;     // S_i staged in shared memory up to this size

__device__ __forceinline__ int64_t last_le(const int64_t* a, int64_t n_plus1, int64_t x) {
  int64_t lo = 0, hi = n_plus1 - 1;  // last b in [0, n) with a[b] <= x
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid; else hi = mid;
  }
  return lo;
}

// ---------------------------------------------------------------- P = Q A

struct QDegF {
  const int32_t* qcol;
  const int64_t* rowptr;
  __device__ int64_t operator()(int64_t q) const {
    const int32_t u = qcol[q];
    return rowptr[u + 1] - rowptr[u];
  }
};

// Counts for the batches [g0, g1): rows q in [qoff[g0], qoff[g1]), packed
// uint16 counters cnt16[(i - g0) * n + v]; first touches -> nnz_b[i].
__global__ void __launch_bounds__(kLadiesThreads) k_lad_count(
    const int64_t* __restrict__ qoff, int64_t k, int64_t g0, int64_t g1,
    const int32_t* __restrict__ qcol, const int64_t* __restrict__ qg,
    const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col, int64_t n,
    uint32_t* __restrict__ cnt32, int64_t* __restrict__ nnz_b) {
  const int lane = lane_id();
  const int64_t q0 = qoff[g0], q1 = qoff[g1];
  if (q1 <= q0) return;
  const int64_t base = q0 * kLRowCost + qg[q0];
  const int64_t total = q1 * kLRowCost + qg[q1] - base;
  const int64_t NW = grid_warps(), w = global_warp();
  const int64_t share = (total + NW - 1) / NW;
  const int64_t pa = min(w * share, total) + base, pb = min(w * share + share, total) + base;
  if (pa >= pb) return;
  int64_t lo = q0, hi = q1;  // last q with P_q <= pa
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (mid * kLRowCost + qg[mid] <= pa) lo = mid; else hi = mid;
  }
  for (int64_t q = lo; q < q1; ++q) {
    const int64_t pq = q * kLRowCost + qg[q];
    if (pq >= pb) break;
    const int64_t d = qg[q + 1] - qg[q];
    const int64_t e0 = max(pa - pq - kLRowCost, (int64_t)0), e1 = min(pb - pq - kLRowCost, d);
    if (e0 >= e1) continue;
    const int64_t i = last_le(qoff, k + 1, q);
    const int32_t u = qcol[q];
    const int64_t a0 = rowptr[u];
    uint32_t* ci = cnt32;
    const int64_t cb = (i - g0) * n;
    for (int64_t e = a0 + e0 + lane; e < a0 + e1; e += 32) {
      const int64_t v = cb + __ldg(col + e);
      atomicAdd(ci + (v >> 1), 1u << ((uint32_t)(v & 1) << 4));  // no return: RED
    }
  }
  (void)nnz_b;
}

// Group-local nonzero offsets: gpoff[j] = sum_{g0 <= i < g0 + j} nnz_b[i].
__global__ void k_lad_gpoff(const int64_t* __restrict__ nnz_b, int64_t g0, int64_t gn,
                            int64_t* __restrict__ gpoff) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int64_t acc = 0;
    for (int64_t j = 0; j < gn; ++j) { gpoff[j] = acc; acc += nnz_b[g0 + j]; }
    gpoff[gn] = acc;
  }
}

// Tile-parallel stream compaction of the group's counters in (batch, v)
// order.  Pass 1: nonzeros per tile.  Pass 2 (after a tile-sum scan): block
// scan + scatter (v, e) and clear the counters.
constexpr int kCompTile = 4096;  // counters per tile (256 threads x 16)

// Also N_i: nonzeros per batch (a thread's 16 counters straddle at most one
// batch boundary when n >= 16; otherwise counted one by one).
__global__ void __launch_bounds__(256) k_lad_compact_count(const uint32_t* __restrict__ cnt32,
                                                         int64_t words, int64_t n, int64_t g0,
                                                         int64_t* __restrict__ tile_cnt,
                                                         int64_t* __restrict__ nnz_b) {
  __shared__ int64_t sw[33];
  const int64_t ntiles = (2 * words + kCompTile - 1) / kCompTile;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t w0 = t * (kCompTile / 2) + threadIdx.x * 8;
    int64_t c = 0;
    // per-thread counts of its (at most two when n >= 16) batches; a third
    // segment (tiny n) goes straight to memory
    const int64_t ja = (2 * w0) / n;
    int64_t next = (ja + 1) * n, jcur = ja;
    uint32_t ca = 0, cb = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t wi = w0 + j;
      if (wi < words) {
        const uint32_t x = cnt32[wi];
        for (int h = 0; h < 2; ++h) {
          if ((x >> (16 * h)) & 0xffffu) {
            const int64_t f = 2 * wi + h;
            if (f >= next) {
              jcur = f / n;
              next = (jcur + 1) * n;
            }
            if (jcur == ja) ++ca;
            else if (jcur == ja + 1) ++cb;
            else atomicAdd((unsigned long long*)(nnz_b + g0 + jcur), 1ull);
            ++c;
          }
        }
      }
    }
    // warp-aggregate per batch id, one atomic per distinct batch per warp
    const unsigned FULL = 0xffffffffu;
    for (int part = 0; part < 2; ++part) {
      const int64_t jj = ja + part;
      const uint32_t cc = part ? cb : ca;
      const unsigned grp = __match_any_sync(FULL, jj);
      const uint32_t sum = __reduce_add_sync(grp, cc);
      if (sum && (threadIdx.x & 31) == __ffs(grp) - 1)
        atomicAdd((unsigned long long*)(nnz_b + g0 + jj), (unsigned long long)sum);
    }
    int64_t total;
    block_excl_scan<int64_t>(c, sw, total);
    if (threadIdx.x == 0) tile_cnt[t] = total;
  }
}

struct TileF {
  const int64_t* t;
  __device__ int64_t operator()(int64_t i) const { return t[i]; }
};

// race key of P entry (batch key, v, e): E / e^2 as float bits, E ~ Exp(1)
// from a full 32-bit Philox word (race_exp: accurate in relative terms near
// 0, where the s smallest keys are decided); non-negative floats order like
// their bit patterns; keyed by (batch key, v) in a domain disjoint from the
// ITS draws (depth | 2^31).  Equal keys are ordered by vertex id.
struct RaceKey {
  uint64_t seed, epoch, depth;
  int64_t key0;  // batch_offset + g0
  __device__ __forceinline__ uint32_t word(int64_t j, int32_t v) const {
    // Philox4x32-10, counter (v, batch key lo/hi, depth), key (seed ^ epoch mix)
    const uint64_t bk = (uint64_t)(key0 + j);
    uint32_t c0 = (uint32_t)v, c1 = (uint32_t)bk, c2 = (uint32_t)(bk >> 32),
             c3 = (uint32_t)depth | 0x80000000u;
    philox4x32_10(c0, c1, c2, c3, (uint32_t)seed ^ (uint32_t)(seed >> 32),
                  (uint32_t)epoch ^ (uint32_t)(epoch >> 32) ^ 0x6c616479u);
    return c0;
  }
  __device__ __forceinline__ uint32_t operator()(int64_t j, int32_t v, uint32_t e) const {
    return __float_as_uint(race_exp(word(j, v)) / ((float)e * (float)e));
  }
  // (exact histogram bin of the key) << 20 | e, e < 2^20, without the
  // accurate logarithm for almost every entry: E from the fast MUFU log
  // (relative error < 2^-15: |log2 x| >= 0.02 on the log branch, 2^-22.6
  // absolute error there; a 3-term series below V = 2^-6) brackets the key
  // within +-2^-12; only a bracket that straddles a bin edge (~0.1% of
  // entries) falls back to the exact key.  The exact key of an entry that
  // can be selected is formed later from (v, e) (k_lad_filter_tiles).
  __device__ __forceinline__ uint32_t bin_key(int64_t j, int32_t v, uint32_t e) const {
    const uint32_t x = word(j, v);
    float E;
    if (x < 0x80000000u) {
      const float V = ((float)x + 0.5f) * 0x1.0p-32f;
      E = V < 0x1.0p-6f ? V * (1.0f + V * (0.5f + V * (1.0f / 3.0f)))
                        : -__log2f(1.0f - V) * 0.69314718f;
    } else {
      E = -__log2f(((float)(0xffffffffu - x) + 0.5f) * 0x1.0p-32f) * 0.69314718f;
    }
    const float ka = __fdividef(E, (float)e * (float)e);
    const uint32_t lo = __float_as_uint(ka * (1.0f - 0x1.0p-12f)) >> 20;
    const uint32_t hi = __float_as_uint(ka * (1.0f + 0x1.0p-12f)) >> 20;
    const uint32_t bin =
        lo == hi ? lo : __float_as_uint(race_exp(x) / ((float)e * (float)e)) >> 20;
    return (bin << 20) | e;
  }
};

// obase != nullptr: outputs start at *obase (batch groups appended)
__global__ void __launch_bounds__(256) k_lad_compact_write(uint32_t* __restrict__ cnt32,
                                                         int64_t words, int64_t n,
                                                         const int64_t* __restrict__ tile_off,
                                                         int32_t* __restrict__ pv,
                                                         int32_t* __restrict__ pe,
                                                         const int64_t* __restrict__ obase,
                                                         int32_t vbase = 0) {
  __shared__ int64_t sw[33];
  if (obase) {
    pv += *obase;
    pe += *obase;
  }
  const int64_t ntiles = (2 * words + kCompTile - 1) / kCompTile;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t w0 = t * (kCompTile / 2) + threadIdx.x * 8;
    uint32_t x[8];
    int64_t c = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t wi = w0 + j;
      x[j] = wi < words ? cnt32[wi] : 0u;
      c += ((x[j] & 0xffffu) != 0) + ((x[j] >> 16) != 0);
    }
    int64_t total;
    int64_t o = block_excl_scan<int64_t>(c, sw, total) + tile_off[t];
    int64_t jb = (2 * w0) / n, base = jb * n;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (!x[j]) continue;
      const int64_t flat = 2 * (w0 + j);
      for (int h = 0; h < 2; ++h) {
        const uint32_t e = (x[j] >> (16 * h)) & 0xffffu;
        if (e) {
          int64_t v = flat + h - base;
          while (v >= n) { ++jb; base += n; v -= n; }
          pv[o] = (int32_t)v + vbase;
          pe[o] = (int32_t)e;
          ++o;
        }
      }
      cnt32[w0 + j] = 0u;
    }
  }
}

// ------------------------------------------- P = Q A by column tiles (race)
// GB_LADIES_RACE does not need the dense per-batch counter vectors: one CTA
// per (batch, column tile) counts e_v for its tile in shared memory, then
// compacts the tile's nonzeros straight into the P layout with their race
// keys and key histogram.  Tiles are at most kLTileW columns wide and cut by
// degree mass (columns near hubs are narrow) so CTAs carry similar work;
// CTAs take (batch, tile) tickets in order and chain their output offsets by
// decoupled look-back, so P comes out in (batch, v) order in one pass.
// Tile geometry and the sparse list (build-time knobs, swept round 2):
// 32K columns x 512 threads, 2048 listed columns keeps two CTAs per SM; 64K
// x 1024 with a 6144 list gained 5% on the papers shape and lost 7% on the
// products shape; a 4096 list alone drops to one CTA per SM (-30%).
#ifndef GB_LTILE_W
#define GB_LTILE_W 32768
#define GB_LTILE_T 512
#endif
constexpr int kLTileW = GB_LTILE_W;  // columns per tile (16-bit counters: 2 B each)
constexpr int kLTileThreads = GB_LTILE_T;
constexpr int kLMassTiles = 64;     // extra cuts by degree mass

// cut before v when v is a multiple of kLTileW or crosses a mass quantile
struct CutF {
  const int64_t* rowptr;
  int64_t n, mass;
  __device__ int64_t operator()(int64_t v) const {
    if (v == 0 || v >= n) return 0;
    return (v % kLTileW == 0) || (rowptr[v] / mass != rowptr[v - 1] / mass) ? 1 : 0;
  }
};

// tb[0] = 0, tb[c] = the c-th cut, tb[ntiles] = n; *ntiles
__global__ void k_lad_tiles(const int64_t* __restrict__ rowptr, int64_t n, int64_t mass,
                            const int64_t* __restrict__ cpre, int32_t* __restrict__ tb,
                            int64_t* __restrict__ ntiles) {
  const CutF f{rowptr, n, mass};
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= n;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (v == 0) tb[0] = 0;
    if (v == n) {
      tb[cpre[n] + 1] = (int32_t)n;
      *ntiles = cpre[n] + 1;
    }
    if (v < n && f(v)) tb[cpre[v] + 1] = (int32_t)v;
  }
}

// first index in col[a, b) with col >= x: 32-ary warp search
__device__ __forceinline__ int64_t warp_lower_bound(const int32_t* __restrict__ col, int64_t a,
                                                    int64_t b, int32_t x) {
  const int lane = lane_id();
  const unsigned FULL = 0xffffffffu;
  while (b - a > 32) {
    const int64_t step = (b - a + 31) >> 5;
    const int64_t p = a + (int64_t)lane * step;
    const bool lt = p < b && __ldg(col + p) < x;
    const int c = __popc(__ballot_sync(FULL, lt));  // lanes 0..c-1 below x
    if (c == 0) return a;
    a = a + (int64_t)(c - 1) * step + 1;
    const int64_t nb = a - 1 + step;
    if (nb < b) b = nb;
  }
  const int64_t p = a + lane;
  const bool lt = p < b && __ldg(col + p) < x;
  return a + __popc(__ballot_sync(FULL, lt));
}

struct LadTileArgs {
  const int64_t* qoff;     // batch row offsets (k + 1)
  const int32_t* qcol;
  const int64_t* rowptr;
  const int32_t* col;
  const int32_t* tb;       // tile bounds (ntiles + 1)
  const int64_t* ntiles;
  int64_t n;
  int64_t g0, gn;          // batches of this group
  RaceKey rk;
  unsigned long long* ticket;
  int32_t* pv;             // P columns: batch j, tile t at slot j * n + tb[t]
  uint32_t* keys;          // race keys, same slots
  int32_t* tcnt;           // nonzeros of (j, t), gn * ntiles
  uint32_t* hist;          // gn * kBins key histograms
  int64_t* nnz_b;          // nonzeros per batch
};

// build-time knobs, swept round 2 (cfg3 / papers minibatches/s): kLUnroll 2
// 12.8K, 4 13.0K, 8 12.8K; kLTileRun 8 12.7K / 2.24K, 16 13.0K / 2.36K, 32
// 11.7K / 2.35K; kLShort 8 12.8K / 2.22K, 16 13.0K / 2.36K, 32 13.1K / 1.95K
#ifndef GB_LTAIL
#define GB_LTAIL 16  // swept (tail, run): (0,-) 13.7K · (8,4) 13.7K · (16,2) 14.0K · (16,4) 14.1K · (24,4) 14.1K · (32,4) 14.0K · (16,8) 13.6K
#endif
#ifndef GB_LTAILRUN
#define GB_LTAILRUN 4
#endif
constexpr int kLTail = GB_LTAIL;        // last tiles of every batch in short runs
constexpr int kLTailRun = GB_LTAILRUN;  // their run length
#ifndef GB_LRUN
#define GB_LRUN 16
#endif
constexpr int kLTileRun = GB_LRUN;     // consecutive tiles per ticket (row cursors carried over)
constexpr int kLRowsSmem = 1024;  // rows whose cursors fit in shared memory
#ifndef GB_LUNROLL
#define GB_LUNROLL 4
#endif
constexpr int kLUnroll = GB_LUNROLL;       // 32-entry loads in flight per row
#ifndef GB_LLIST
#define GB_LLIST 2048
#endif
constexpr int kLList = GB_LLIST;  // touched offsets remembered per tile (sparse compaction)
#ifndef GB_LSHORT
#define GB_LSHORT 16
#endif
constexpr int kLShort = GB_LSHORT;       // expected entries per tile below which a row is "short"
constexpr int kLShortU = 8;        // entries of a short row loaded at once (thread per row)

// One ticket = batch j and a run of kLTileRun consecutive column tiles.  Per
// tile: counts in shared memory (warp per A row, from the row's cursor, which
// the scan leaves at the first column past the tile), then a warp-balanced
// compaction of the nonzeros into the tile's slot with their race keys.
__global__ void __launch_bounds__(kLTileThreads) k_lad_tile(LadTileArgs A) {
  extern __shared__ uint32_t s_cnt[];               // kLTileW / 2 packed 16-bit counters
  uint32_t* s_h = s_cnt + kLTileW / 2;               // kBins
  int64_t* s_ra = (int64_t*)(s_h + kBins);           // row start, kLRowsSmem
  int32_t* s_rl = (int32_t*)(s_ra + kLRowsSmem);     // row length
  int32_t* s_rc = s_rl + kLRowsSmem;                 // row cursor (relative)
  int32_t* s_nv = s_rc + kLRowsSmem;                 // column at the cursor (INT32_MAX: done)
  int16_t* s_act = (int16_t*)(s_nv + kLRowsSmem);    // rows with entries in the tile
  __shared__ int s_nact, s_lcnt, s_emit, s_rnext, s_nshort;
  __shared__ uint16_t s_list[kLList];               // column offsets touched (sparse tiles)
  __shared__ int32_t s_wcnt[kLTileThreads / 32 + 1];
  __shared__ uint32_t s_stage[kLTileThreads / 32 * 64];
  __shared__ int64_t s_ticket;
  __shared__ unsigned long long s_nnz;
  const unsigned FULL = 0xffffffffu;
  const int lane = lane_id(), warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int64_t ntiles = *A.ntiles;
  // tickets: every batch's first tiles in runs of kLTileRun (cursors carried
  // over a run), then — after all of those — its last kLTail tiles in runs
  // of kLTailRun, so the final round of tickets is fine-grained
  const int64_t tail = ntiles < kLTail ? ntiles : kLTail;
  const int64_t nlong = (ntiles - tail) / kLTileRun;
  const int64_t tail0 = nlong * kLTileRun;  // first tile of the short runs
  const int64_t nshortr = (ntiles - tail0 + kLTailRun - 1) / kLTailRun;
  const int64_t nt = A.gn * (nlong + nshortr);
  for (int w = threadIdx.x; w < kLTileW / 2; w += blockDim.x) s_cnt[w] = 0;
  // count column c (inside the tile when `in`) and, while the tile is sparse
  // (lc <= kLList, warp-uniform), list it for the sparse compaction — only
  // at its counter's 0 -> 1 step (`ft`; measured: papers-shape LADIES 1.3K
  // -> 2.4K minibatches/s, a sparse batch's tiles then list distinct
  // columns and stay within kLList), or every entry (`ft` false).  The
  // compaction reads and clears each listed counter, so repeats are
  // harmless; a list count past kLList marks the tile dense.
  // Warp-collective.
  auto count = [&](int32_t c, bool in, int lc, int32_t v0, bool ft) {
    const uint32_t off = (uint32_t)(c - v0), sh = (off & 1u) << 4;
    if (lc <= kLList) {
      bool first = in;
      if (in) {
        if (ft)
          first = ((atomicAdd(s_cnt + (off >> 1), 1u << sh) >> sh) & 0xffffu) == 0u;
        else
          atomicAdd(s_cnt + (off >> 1), 1u << sh);
      }
      const unsigned m = __ballot_sync(FULL, first);
      if (m) {
        int lb = 0;
        if (lane == 0) lb = atomicAdd(&s_lcnt, __popc(m));
        lb = __shfl_sync(FULL, lb, 0) + __popc(m & ((1u << lane) - 1u));
        if (first && lb < kLList) s_list[lb] = (uint16_t)off;
      }
    } else if (in) {
      atomicAdd(s_cnt + (off >> 1), 1u << sh);
    }
  };
  for (;;) {
    if (threadIdx.x == 0) {
      s_ticket = (int64_t)atomicAdd(A.ticket, 1ull);
      s_nnz = 0;
    }
    for (int b = threadIdx.x; b < kBins; b += blockDim.x) s_h[b] = 0;
    __syncthreads();
    const int64_t ticket = s_ticket;
    if (ticket >= nt) return;
    int64_t j, t0, t1;
    if (ticket < A.gn * nlong) {
      j = ticket / nlong;
      t0 = (ticket - j * nlong) * kLTileRun;
      t1 = t0 + kLTileRun;
    } else {
      const int64_t x = ticket - A.gn * nlong;
      j = x / nshortr;
      t0 = tail0 + (x - j * nshortr) * kLTailRun;
      t1 = min(t0 + kLTailRun, ntiles);
    }
    const int64_t q0 = A.qoff[A.g0 + j], q1 = A.qoff[A.g0 + j + 1];
    const bool cur = q1 - q0 <= kLRowsSmem;
    if (cur) {
      // cursors at the run's first column: a binary search per row, one row
      // per thread, so all rows' searches are in flight together
      const int32_t vs = A.tb[t0];
      for (int64_t q = q0 + threadIdx.x; q < q1; q += blockDim.x) {
        const int32_t u = A.qcol[q];
        const int64_t a = A.rowptr[u], b = A.rowptr[u + 1];
        int64_t lo = a, hi = vs > 0 ? b : a;
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (__ldg(A.col + mid) < vs) lo = mid + 1; else hi = mid;
        }
        s_ra[q - q0] = a;
        s_rl[q - q0] = (int32_t)(b - a);
        s_rc[q - q0] = (int32_t)(lo - a);
        s_nv[q - q0] = lo < b ? __ldg(A.col + lo) : 0x7fffffff;
      }
    }
    for (int64_t t = t0; t < t1; ++t) {
      const int32_t v0 = A.tb[t], v1 = A.tb[t + 1];
      const int nw2 = (v1 - v0 + 1) >> 1;
      // counters are zero here: cleared once at start, then by the compaction
      if (threadIdx.x == 0) {
        s_nact = 0;
        s_lcnt = 0;
        s_emit = 0;
        s_rnext = 0;
        s_nshort = 0;
      }
      __syncthreads();
      // rows whose next column falls in this tile (cursor mode): tiles a
      // row has no entries in cost one shared-memory read
      // Rows expected to hold few entries in the tile (deg * width / n <
      // kLShort, columns are spread uniformly by the relabel) are listed from
      // the back and counted a thread per row.
      int nact = (int)(q1 - q0), nshort = 0;
      if (cur) {
        const int64_t wn = (int64_t)(v1 - v0);
        for (int r = threadIdx.x; r < q1 - q0; r += blockDim.x)
          if (s_nv[r] < v1) {
            if ((int64_t)s_rl[r] * wn < (int64_t)kLShort * A.n)
              s_act[kLRowsSmem - 1 - atomicAdd(&s_nshort, 1)] = (int16_t)r;
            else
              s_act[atomicAdd(&s_nact, 1)] = (int16_t)r;
          }
        __syncthreads();
        nact = s_nact;
        nshort = s_nshort;
      }
      auto lcnow = [&]() { return __shfl_sync(FULL, s_lcnt, 0); };
      // ---- e_v for v in [v0, v1)
      // cursor mode: the first kLUnroll x 32 entries of the warp's next row
      // are loaded while the current row is counted (two rows in flight)
      if (cur) {
        auto row_at = [&](int ai, int64_t& q, int64_t& a, int64_t& b, int64_t& e0) {
          q = q0 + (int64_t)s_act[ai];
          a = s_ra[q - q0];
          b = a + s_rl[q - q0];
          e0 = a + s_rc[q - q0];
        };
        // rows taken dynamically (segment lengths vary widely per tile)
        auto grab = [&]() {
          int x = 0;
          if (lane == 0) x = atomicAdd(&s_rnext, 1);
          return __shfl_sync(FULL, x, 0);
        };
        int64_t qn = 0, an = 0, bn = 0, e0n = 0;
        int32_t cvn[kLUnroll];
        int ai = grab();
        if (ai < nact) {
          row_at(ai, qn, an, bn, e0n);
#pragma unroll
          for (int u = 0; u < kLUnroll; ++u) {
            const int64_t e = e0n + lane + 32 * u;
            cvn[u] = e < bn ? __ldg(A.col + e) : 0x7fffffff;
          }
        }
        while (ai < nact) {
          // the list state once per row (a stale count only lags: appends
          // past kLList are dropped and still mark the tile dense), so no
          // shared load sits in front of every step's atomic
          const int lcr = lcnow();
          const int64_t q = qn, a = an, b = bn, e0 = e0n;
          int32_t cv[kLUnroll];
#pragma unroll
          for (int u = 0; u < kLUnroll; ++u) cv[u] = cvn[u];
          const int anext = grab();
          if (anext < nact) {
            row_at(anext, qn, an, bn, e0n);
#pragma unroll
            for (int u = 0; u < kLUnroll; ++u) {
              const int64_t e = e0n + lane + 32 * u;
              cvn[u] = e < bn ? __ldg(A.col + e) : 0x7fffffff;
            }
          }
          bool done = false;
          for (int64_t e = e0 + lane;; e += 32 * kLUnroll) {
            if (e != e0 + lane) {
#pragma unroll
              for (int u = 0; u < kLUnroll; ++u)
                cv[u] = e + 32 * u < b ? __ldg(A.col + e + 32 * u) : 0x7fffffff;
            }
#pragma unroll
            for (int u = 0; u < kLUnroll; ++u) {
              if (done) break;
              const int32_t c = cv[u];
              const bool in = c < v1;
              count(c, in, lcr, v0, true);
              const unsigned out = __ballot_sync(FULL, !in);
              if (out) {
                const int src = __ffs(out) - 1;
                const int32_t nv = __shfl_sync(FULL, c, src);
                if (lane == 0) {
                  s_rc[q - q0] = (int32_t)(e + 32 * u - lane - a + src);
                  s_nv[q - q0] = nv;
                }
                done = true;
              }
            }
            if (done) break;
          }
          ai = anext;
        }
        // short rows: a thread per row, kLShortU of its entries loaded at
        // once — every short row's loads are in flight together, one memory
        // round trip per tile rather than one per warp step (the rows of a
        // sparse batch hold a few entries per tile: papers shape ~7)
        for (int si0 = 0; si0 < nshort; si0 += blockDim.x) {
          const int si = si0 + (int)threadIdx.x;
          bool live = si < nshort;
          int64_t q = q0, a = 0, b = 0, e = 0;
          if (live) {
            q = q0 + (int64_t)s_act[kLRowsSmem - 1 - si];
            a = s_ra[q - q0];
            b = a + s_rl[q - q0];
            e = a + s_rc[q - q0];
          }
          while (__any_sync(FULL, live)) {
            int32_t c[kLShortU];
#pragma unroll
            for (int z = 0; z < kLShortU; ++z)
              c[z] = live && e + z < b ? __ldg(A.col + e + z) : 0x7fffffff;
            int nin = 0;  // columns are sorted: the in-tile entries are a prefix
#pragma unroll
            for (int z = 0; z < kLShortU; ++z) nin += c[z] < v1 ? 1 : 0;
            const int lc = lcnow();
#pragma unroll
            for (int z = 0; z < kLShortU; ++z) count(c[z], live && z < nin, lc, v0, true);
            if (live) {
              if (nin < kLShortU) {  // the row leaves the tile (or ends) here
                int32_t nv = 0x7fffffff;
#pragma unroll
                for (int z = 0; z < kLShortU; ++z)
                  if (z == nin) nv = c[z];
                s_rc[q - q0] = (int32_t)(e + nin - a);
                s_nv[q - q0] = nv;
                live = false;
              } else {
                e += kLShortU;
              }
            }
          }
        }
      } else
      for (int ai = warp; ai < nact; ai += nwarps) {
        const int lcr = lcnow();
        const int64_t q = q0 + (cur ? (int64_t)s_act[ai] : (int64_t)ai);
        int64_t a, b, e0;
        if (cur) {
          a = s_ra[q - q0];
          b = a + s_rl[q - q0];
          e0 = a + s_rc[q - q0];
        } else {
          const int32_t u = A.qcol[q];
          a = A.rowptr[u];
          b = A.rowptr[u + 1];
          e0 = a < b && __ldg(A.col + a) < v0 ? warp_lower_bound(A.col, a, b, v0) : a;
        }
        if (e0 >= b) continue;
        // kLUnroll 32-entry steps per round: all loads in flight
        bool done = false;
        for (int64_t e = e0 + lane; !done; e += 32 * kLUnroll) {
          int32_t cv[kLUnroll];
#pragma unroll
          for (int u = 0; u < kLUnroll; ++u)
            cv[u] = e + 32 * u < b ? __ldg(A.col + e + 32 * u) : 0x7fffffff;
#pragma unroll
          for (int u = 0; u < kLUnroll; ++u) {
            if (done) break;
            const int32_t c = cv[u];
            const bool in = c < v1;
            count(c, in, lcr, v0, true);
            const unsigned out = __ballot_sync(FULL, !in);
            if (out) {
              const int src = __ffs(out) - 1;
              const int32_t nv = __shfl_sync(FULL, c, src);  // next column (or INT32_MAX)
              if (cur && lane == 0) {
                s_rc[q - q0] = (int32_t)(e + 32 * u - lane - a + src);
                s_nv[q - q0] = nv;
              }
              done = true;
            }
          }
        }
      }
      __syncthreads();
      const int64_t slot = j * A.n + v0;
      int total = 0;
      const int lcnt = s_lcnt;
      if (lcnt <= kLList) {
        // ---- sparse compaction: each touched counter read-and-cleared once
        for (int i = threadIdx.x; i < lcnt; i += blockDim.x) {
          const int off = s_list[i];
          const int sh = (off & 1) << 4;
          const uint32_t old = atomicAnd(s_cnt + (off >> 1), ~(0xffffu << sh));
          const uint32_t e = (old >> sh) & 0xffffu;
          if (e) {
            const int pos = atomicAdd(&s_emit, 1);
            const int32_t v = v0 + off;
            const uint32_t key = A.rk.bin_key(j, v, e);
            A.pv[slot + pos] = v;
            A.keys[slot + pos] = key;
            atomicAdd(s_h + (key >> 20), 1u);
          }
        }
        __syncthreads();
        total = s_emit;
      } else {
      // ---- compaction: warp w owns words [w * chunk, ...), counted then written
      const int chunk = (nw2 + nwarps - 1) / nwarps;
      const int wa = warp * chunk, wb = min(wa + chunk, nw2);
      int c = 0;
      for (int w = wa + lane; w < wb; w += 32) {
        const uint32_t x = s_cnt[w];
        c += ((x & 0xffffu) != 0) + ((x >> 16) != 0);
      }
      c = warp_sum(c);
      if (lane == 0) s_wcnt[warp] = c;
      __syncthreads();
      int base = 0;
      for (int w = 0; w < nwarps; ++w) {
        const int x = s_wcnt[w];
        base += w < warp ? x : 0;
        total += x;
      }
      // nonzeros of 32 words -> the warp's staging buffer (<= 64), then the
      // keys with all lanes busy and coalesced slot writes
      uint32_t* stg = s_stage + warp * 64;
      for (int w0 = wa; w0 < wb; w0 += 32) {
        const int w = w0 + lane;
        const uint32_t x = w < wb ? s_cnt[w] : 0u;
        if (x) s_cnt[w] = 0;  // ready for the next tile
        const int m = ((x & 0xffffu) != 0) + ((x >> 16) != 0);
        int inc = m;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(FULL, inc, o);
          if (lane >= o) inc += y;
        }
        int o = inc - m;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t e = (x >> (16 * h)) & 0xffffu;
          if (e) stg[o++] = ((uint32_t)(2 * w + h) << 16) | e;  // (tile offset, count)
        }
        const int cnt = __shfl_sync(FULL, inc, 31);
        __syncwarp();
        for (int p = lane; p < cnt; p += 32) {
          const uint32_t rec = stg[p];
          const int32_t v = v0 + (int32_t)(rec >> 16);
          const uint32_t key = A.rk.bin_key(j, v, rec & 0xffffu);
          A.pv[slot + base + p] = v;
          A.keys[slot + base + p] = key;
          atomicAdd(s_h + (key >> 20), 1u);
        }
        __syncwarp();
        base += cnt;
      }
      }
      if (threadIdx.x == 0) {
        A.tcnt[j * ntiles + t] = total;
        s_nnz += (unsigned long long)total;
      }
      __syncthreads();  // counters reused by the next tile
    }
    uint32_t* hj = A.hist + j * kBins;
    for (int b = threadIdx.x; b < kBins; b += blockDim.x)
      if (s_h[b]) atomicAdd(hj + b, s_h[b]);
    if (threadIdx.x == 0 && s_nnz)
      atomicAdd((unsigned long long*)(A.nnz_b + A.g0 + j), s_nnz);
    __syncthreads();
  }
}

// tiled P layout: every batch's slots start at j * n
__global__ void k_lad_slot_off(int64_t gn, int64_t n, int64_t* __restrict__ gpoff) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j <= gn;
       j += (int64_t)gridDim.x * blockDim.x)
    gpoff[j] = j * n;
}

// Block-wide search of the first bin where the running count reaches need:
// every thread owns kBins / blockDim consecutive bins.  Returns (bin, count
// strictly below it) through shared memory.
__device__ __forceinline__ void block_find_bin(const uint32_t* hist, int nbins, int64_t need,
                                               int64_t* sw, int* s_bin, int* s_acc) {
  const int per = (nbins + blockDim.x - 1) / blockDim.x;
  const int b0 = threadIdx.x * per;
  int64_t c = 0;
  for (int b = b0; b < b0 + per && b < nbins; ++b) c += hist[b];
  int64_t total;
  int64_t acc = block_excl_scan<int64_t>(c, sw, total);
  if (threadIdx.x == 0 && total < need) { *s_bin = nbins; *s_acc = (int)total; }
  if (acc < need && acc + c >= need) {
    for (int b = b0; b < b0 + per && b < nbins; ++b) {
      if (acc + hist[b] >= need) { *s_bin = b; *s_acc = (int)acc; break; }
      acc += hist[b];
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------- sampling

struct LadiesSampleArgs {
  const int64_t* gpoff;  // group-local offsets of the P rows' nonzeros (gn + 1)
  const int32_t* pv;
  const int32_t* pe;
  int64_t g0, gn;        // batches g0 .. g0+gn-1
  int32_t s;
  int64_t batch_offset;
  uint64_t seed, epoch, depth;
  double* sw;            // exact: weights, cdf scratch (P layout)
  double* sc;
  uint32_t* keys;        // race keys (P layout)
  int32_t* sel;          // per batch: up to s selected P positions (global batch index * s)
  int32_t* nsel;         // per batch selected count (atomic)
  int64_t* take;         // per batch
  const int64_t* nnzb;   // tiled layout: nonzeros per batch (P rows have slot gaps)
};

// Exact replay of its_sample_row: one thread per batch.
__global__ void k_lad_sample_exact(LadiesSampleArgs A) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < A.gn;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = A.g0 + j;
    const int64_t p0 = A.gpoff[j], N = A.gpoff[j + 1] - p0;
    const int64_t take = N < A.s ? N : A.s;
    A.take[i] = take;
    A.nsel[i] = (int32_t)take;
    int32_t* sel = A.sel + i * A.s;
    if (N == 0) continue;
    if (take == N) {
      for (int64_t t = 0; t < N; ++t) sel[t] = (int32_t)(p0 + t);
      continue;
    }
    double* w = A.sw + p0;
    double* cdf = A.sc + p0;
    // norm_rows_ladies: vals = e*e; sum = vals[0] + pairwise(vals[1:]) is
    // exact for integer values < 2^53, so an int64 sum gives the same double
    int64_t sq = 0;
    for (int64_t t = 0; t < N; ++t) sq += (int64_t)A.pe[p0 + t] * A.pe[p0 + t];
    const double S = (double)sq;
    for (int64_t t = 0; t < N; ++t) {
      const double e = (double)A.pe[p0 + t];
      w[t] = __ddiv_rn(__dmul_rn(e, e), S);
    }
    const uint64_t key = (uint64_t)(A.batch_offset + i);
    int64_t dirty = 0;  // cdf valid below this index
    for (int64_t t = 0; t < take; ++t) {
      double acc = dirty ? cdf[dirty - 1] : 0.0;
      for (int64_t x = dirty; x < N; ++x) {
        acc = __dadd_rn(acc, w[x]);
        cdf[x] = acc;
      }
      const double total = cdf[N - 1];
      const double u = uniform53(A.seed, A.epoch, A.depth, key, (uint64_t)t);
      const double target = __dmul_rn(u, total);
      int64_t idx = upper_bound(cdf, 0, N, target);
      if (idx >= N) idx = N - 1;
      while (w[idx] == 0.0) --idx;
      sel[t] = (int32_t)(p0 + idx);
      w[idx] = 0.0;
      dirty = idx;
    }
  }
}

// race keys of the group's P entries, one thread per entry
__global__ void __launch_bounds__(256) k_lad_keys(LadiesSampleArgs A, RaceKey rk) {
  __shared__ int64_t sp[kSmaxSmem + 1];
  const bool sm = A.gn + 1 <= kSmaxSmem;
  if (sm)
    for (int64_t j = threadIdx.x; j <= A.gn; j += blockDim.x) sp[j] = A.gpoff[j];
  __syncthreads();
  const int64_t* gp = sm ? sp : A.gpoff;
  const int64_t P = gp[A.gn];
  for (int64_t p = gp[0] + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = last_le(gp, A.gn + 1, p);
    A.keys[p] = rk(j, A.pv[p], (uint32_t)A.pe[p]);
  }
}

// histogram of the top 12 key bits per batch (smem-privatised per chunk)
constexpr int kHistChunk = 8192;
__global__ void __launch_bounds__(256) k_lad_hist(LadiesSampleArgs A, uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[kBins];
  const int64_t P = A.gpoff[A.gn];
  for (int64_t c0 = A.gpoff[0] + (int64_t)blockIdx.x * kHistChunk; c0 < P;
       c0 += (int64_t)gridDim.x * kHistChunk) {
    const int64_t c1 = min(c0 + kHistChunk, P);
    const int64_t j0 = last_le(A.gpoff, A.gn + 1, c0);
    const int64_t b1 = A.gpoff[j0 + 1];
    for (int b = threadIdx.x; b < kBins; b += blockDim.x) h[b] = 0;
    __syncthreads();
    for (int64_t p = c0 + threadIdx.x; p < c1; p += blockDim.x) {
      const uint32_t bin = A.keys[p] >> 20;
      if (p < b1) atomicAdd(&h[bin], 1u);
      else atomicAdd(&hist[last_le(A.gpoff, A.gn + 1, p) * kBins + bin], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < kBins; b += blockDim.x)
      if (h[b]) atomicAdd(&hist[j0 * kBins + b], h[b]);
    __syncthreads();
  }
}

// per batch: take, boundary bin, count strictly below it
__global__ void __launch_bounds__(256) k_lad_boundary(LadiesSampleArgs A,
                                                    const uint32_t* __restrict__ hist,
                                                    int32_t* __restrict__ bound) {
  __shared__ int64_t sw[33];
  __shared__ int s_bin, s_acc;
  const int j = blockIdx.x;
  if (j >= A.gn) return;
  const int64_t i = A.g0 + j;
  const int64_t N = A.nnzb ? A.nnzb[i] : A.gpoff[j + 1] - A.gpoff[j];
  const int64_t take = N < A.s ? N : A.s;
  if (take < N) {
    block_find_bin(hist + (int64_t)j * kBins, kBins, take, sw, &s_bin, &s_acc);
  } else if (threadIdx.x == 0) {
    s_bin = kBins;  // everything selected
    s_acc = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    A.take[i] = take;
    A.nsel[i] = 0;
    bound[2 * j] = s_bin;
    bound[2 * j + 1] = s_acc;
  }
}

// keys strictly below the boundary bin are selected; keys in it become
// candidates (stored at the batch's P offset)
__global__ void k_lad_filter(LadiesSampleArgs A, const int32_t* __restrict__ bound,
                             int32_t* __restrict__ cand, int32_t* __restrict__ ncand) {
  const int64_t P = A.gpoff[A.gn];
  for (int64_t p = A.gpoff[0] + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = last_le(A.gpoff, A.gn + 1, p);
    const int64_t i = A.g0 + j;
    const int b = bound[2 * j];
    const int bin = b == kBins ? -1 : (int)(A.keys[p] >> 20);
    if (b == kBins || bin < b) {
      A.sel[i * A.s + atomicAdd(A.nsel + i, 1)] = (int32_t)p;
    } else if (bin == b) {
      cand[A.gpoff[j] + atomicAdd(ncand + j, 1)] = (int32_t)p;
    }
  }
}

// k_lad_filter over the tiled layout: one CTA per (batch, tile) slot
// The tiled pass stores (exact bin, e) per entry (RaceKey::bin_key): every
// entry at or below the boundary bin gets its exact key here, before the
// refinement / emission read it.
__global__ void __launch_bounds__(256) k_lad_filter_tiles(LadiesSampleArgs A,
                                                        const int32_t* __restrict__ tb,
                                                        const int64_t* __restrict__ ntiles_p,
                                                        int64_t n, const int32_t* __restrict__ tcnt,
                                                        const int32_t* __restrict__ bound,
                                                        int32_t* __restrict__ cand,
                                                        int32_t* __restrict__ ncand,
                                                        RaceKey rk) {
  const int64_t ntiles = *ntiles_p;
  for (int64_t pr = blockIdx.x; pr < A.gn * ntiles; pr += gridDim.x) {
    const int32_t cnt = tcnt[pr];
    if (!cnt) continue;
    const int64_t j = pr / ntiles, t = pr - j * ntiles;
    const int64_t i = A.g0 + j;
    const int64_t slot = j * n + tb[t];
    const int b = bound[2 * j];
    for (int x = threadIdx.x; x < cnt; x += blockDim.x) {
      const int64_t p = slot + x;
      const uint32_t kb = A.keys[p];
      const int bin = (int)(kb >> 20);
      if (b == kBins || bin <= b) A.keys[p] = rk(j, A.pv[p], kb & 0xfffffu);
      if (b == kBins || bin < b)
        A.sel[i * A.s + atomicAdd(A.nsel + i, 1)] = (int32_t)p;
      else if (bin == b)
        cand[A.gpoff[j] + atomicAdd(ncand + j, 1)] = (int32_t)p;
    }
  }
}

// one CTA per batch: the need = take - below smallest candidates, two more
// histogram passes (12 + 8 bits) then ties by position
__global__ void __launch_bounds__(1024) k_lad_refine(LadiesSampleArgs A,
                                                   const int32_t* __restrict__ bound,
                                                   const int32_t* __restrict__ cand,
                                                   const int32_t* __restrict__ ncand,
                                                   int32_t* __restrict__ overflow) {
  __shared__ uint32_t hist[kBins];
  __shared__ int32_t ties[kTies];
  __shared__ int64_t sw[33];
  __shared__ int s_bin, s_acc, s_tie;
  const int shifts[2] = {8, 0};
  const int widths[2] = {12, 8};
  for (int64_t j = blockIdx.x; j < A.gn; j += gridDim.x) {
    const int64_t i = A.g0 + j;
    if (bound[2 * j] == kBins) continue;
    const int64_t take = A.take[i];
    int64_t need = take - bound[2 * j + 1];
    const int32_t* cj = cand + A.gpoff[j];
    const int m = ncand[j];
    uint32_t prefix = (uint32_t)bound[2 * j] << 20, pmask = 0xfff00000u;
    for (int pass = 0; pass < 2; ++pass) {
      const int sh = shifts[pass];
      const uint32_t bm = (1u << widths[pass]) - 1u;
      for (int b = threadIdx.x; b < kBins; b += blockDim.x) hist[b] = 0;
      __syncthreads();
      for (int a = threadIdx.x; a < m; a += blockDim.x) {
        const uint32_t kk = A.keys[cj[a]];
        if ((kk & pmask) == prefix) atomicAdd(&hist[(kk >> sh) & bm], 1u);
      }
      __syncthreads();
      block_find_bin(hist, (int)bm + 1, need, sw, &s_bin, &s_acc);
      const uint32_t bin = (uint32_t)s_bin;
      for (int a = threadIdx.x; a < m; a += blockDim.x) {
        const uint32_t kk = A.keys[cj[a]];
        if ((kk & pmask) == prefix && ((kk >> sh) & bm) < bin)
          A.sel[i * A.s + atomicAdd(A.nsel + i, 1)] = cj[a];
      }
      need -= s_acc;
      prefix |= bin << sh;
      pmask |= bm << sh;
      __syncthreads();
    }
    if (threadIdx.x == 0) s_tie = 0;
    __syncthreads();
    for (int a = threadIdx.x; a < m; a += blockDim.x)
      if (A.keys[cj[a]] == prefix) {
        const int t = atomicAdd(&s_tie, 1);
        if (t < kTies) ties[t] = cj[a]; else atomicOr(overflow, 1);
      }
    __syncthreads();
    const int mt = min(s_tie, kTies);
    const int base = A.nsel[i];
    for (int a = threadIdx.x; a < mt; a += blockDim.x) {
      int rank = 0;
      // ties by vertex (slot order need not follow v)
      const int32_t va = A.pv[ties[a]];
      for (int b2 = 0; b2 < mt; ++b2) rank += A.pv[ties[b2]] < va ? 1 : 0;
      if (rank < need) A.sel[i * A.s + base + rank] = ties[a];
    }
    __syncthreads();
    if (threadIdx.x == 0) A.nsel[i] = (int32_t)take;
    __syncthreads();
  }
}

// sorted sampled vertices of each batch of the group: Sfix[i*s + r]
// (and, for the distributed top-s merge, their race keys Kfix)
__global__ void __launch_bounds__(256) k_lad_emit(LadiesSampleArgs A, int32_t* __restrict__ Sfix,
                                                uint32_t* __restrict__ Kfix) {
  // the selected entries of a batch in vertex order: a bitonic sort of
  // (v, slot) pairs in shared memory when they fit, else rank by counting
  __shared__ unsigned long long s_kv[kSmaxSmem];
  for (int64_t j = blockIdx.x; j < A.gn; j += gridDim.x) {
    const int64_t i = A.g0 + j;
    const int64_t take = A.take[i];
    const int32_t* si = A.sel + i * A.s;
    if (take <= kSmaxSmem) {
      int np = 1;
      while (np < take) np <<= 1;
      for (int a = threadIdx.x; a < np; a += blockDim.x)
        s_kv[a] = a < take ? ((unsigned long long)(uint32_t)A.pv[si[a]] << 32) | (uint32_t)si[a]
                           : ~0ull;
      __syncthreads();
      for (int kk = 2; kk <= np; kk <<= 1)
        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
          for (int a = threadIdx.x; a < np; a += blockDim.x) {
            const int b = a ^ jj;
            if (b > a) {
              const unsigned long long x = s_kv[a], y = s_kv[b];
              if (((a & kk) == 0) == (x > y)) { s_kv[a] = y; s_kv[b] = x; }
            }
          }
          __syncthreads();
        }
      for (int a = threadIdx.x; a < take; a += blockDim.x) {
        const unsigned long long kv = s_kv[a];
        Sfix[i * A.s + a] = (int32_t)(kv >> 32);
        if (Kfix) Kfix[i * A.s + a] = A.keys[(uint32_t)kv];
      }
      __syncthreads();
      continue;
    }
    for (int64_t a = threadIdx.x; a < take; a += blockDim.x) {
      const int32_t x = si[a];
      const int32_t vx = A.pv[x];
      int64_t rank = 0;  // by vertex: slot order need not follow v
      for (int64_t b = 0; b < take; ++b) rank += A.pv[si[b]] < vx ? 1 : 0;
      Sfix[i * A.s + rank] = vx;
      if (Kfix) Kfix[i * A.s + rank] = A.keys[x];
    }
  }
}

__global__ void k_lad_pack_s(const int64_t* __restrict__ fptr, int64_t k, int32_t s,
                             const int32_t* __restrict__ Sfix, int32_t* __restrict__ fcol) {
  const int64_t F = fptr[k];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < F;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = last_le(fptr, k + 1, e);
    fcol[e] = Sfix[i * s + (e - fptr[i])];
  }
}

// ------------------------------------------------------------- extraction

// shared layout iff every batch took the same count (ladies_assemble)
__global__ void k_lad_layout(const int64_t* __restrict__ fptr, int64_t k,
                             int64_t* __restrict__ coloff, int64_t* __restrict__ sizes) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  bool shared = true;
  for (int64_t i = 1; i < k; ++i)
    if (fptr[i + 1] - fptr[i] != fptr[1] - fptr[0]) shared = false;
  for (int64_t i = 0; i <= k; ++i) coloff[i] = shared ? 0 : fptr[i];
  sizes[1] = fptr[k];
  sizes[3] = k == 0 ? 0 : (shared ? fptr[1] - fptr[0] : fptr[k]);
}

struct RcapF {
  const int32_t* qcol;
  const int64_t* rowptr;
  const int64_t* qoff;
  const int64_t* fptr;
  int64_t k;
  __device__ int64_t operator()(int64_t q) const {
    const int32_t u = qcol[q];
    const int64_t d = rowptr[u + 1] - rowptr[u];
    const int64_t i = last_le(qoff, k + 1, q);
    const int64_t t = fptr[i + 1] - fptr[i];
    return d < t ? d : t;
  }
};

// one warp per A_S row q: the ranks of A[u,:] ∩ S_i, ascending
__global__ void __launch_bounds__(kLadiesThreads) k_lad_extract(
    const int64_t* __restrict__ qoff, int64_t k, const int32_t* __restrict__ qcol,
    const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
    const int64_t* __restrict__ fptr, const int32_t* __restrict__ fcol,
    const int64_t* __restrict__ coloff, const int64_t* __restrict__ slot,
    int32_t* __restrict__ slots, int32_t* __restrict__ rcnt) {
  __shared__ int32_t sS[kLadiesThreads / 32][kSmaxSmem];
  const unsigned FULL = 0xffffffffu;
  const int lane = lane_id(), wib = threadIdx.x >> 5;
  const int64_t QN = qoff[k];
  int64_t staged = -1;
  for (int64_t q = global_warp(); q < QN; q += grid_warps()) {
    const int64_t i = last_le(qoff, k + 1, q);
    const int64_t f0 = fptr[i], take = fptr[i + 1] - f0;
    const bool in_smem = take <= kSmaxSmem;
    if (in_smem && staged != i) {
      __syncwarp();
      for (int64_t r = lane; r < take; r += 32) sS[wib][r] = fcol[f0 + r];
      __syncwarp();
      staged = i;
    }
    const int32_t* S = in_smem ? sS[wib] : fcol + f0;
    const int32_t u = qcol[q];
    const int64_t a0 = rowptr[u], d = rowptr[u + 1] - a0;
    const int64_t cb = coloff[i];
    int32_t* out = slots + slot[q];
    int64_t o = 0;
    if (d <= 16 * take) {
      // stream A[u,:]; binary search each entry in S_i
      for (int64_t e0 = 0; e0 < d; e0 += 32) {
        int rank = -1;
        if (e0 + lane < d) {
          const int32_t v = __ldg(col + a0 + e0 + lane);
          int lo = 0, hi = (int)take;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (S[mid] < v) lo = mid + 1; else hi = mid;
          }
          if (lo < take && S[lo] == v) rank = lo;
        }
        const unsigned bal = __ballot_sync(FULL, rank >= 0);
        if (rank >= 0) out[o + __popc(bal & ((1u << lane) - 1))] = (int32_t)(cb + rank);
        o += __popc(bal);
      }
    } else {
      // hub row: binary search each sampled vertex in A[u,:]
      for (int64_t r0 = 0; r0 < take; r0 += 32) {
        bool hit = false;
        if (r0 + lane < take) {
          const int32_t v = S[r0 + lane];
          int64_t lo = 0, hi = d;
          while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (__ldg(col + a0 + mid) < v) lo = mid + 1; else hi = mid;
          }
          hit = lo < d && __ldg(col + a0 + lo) == v;
        }
        const unsigned bal = __ballot_sync(FULL, hit);
        if (hit) out[o + __popc(bal & ((1u << lane) - 1))] = (int32_t)(cb + r0 + lane);
        o += __popc(bal);
      }
    }
    if (lane == 0) rcnt[q] = (int32_t)o;
  }
}

// A_S rows by hashing: CTA per (batch i, chunk of kXRows rows of Q_i); S_i
// goes into a shared-memory hash (vertex -> rank, 2·kSmaxSmem slots) once
// per item, then every A row of the chunk is streamed once (coalesced,
// kXUnroll loads in flight per lane) and probed — no per-entry binary search,
// hub rows read sequentially instead of searched per sampled vertex.  Hits
// come out in row order (ascending v), i.e. the sorted intersection.
#ifndef GB_XROWS
#define GB_XROWS 64  // swept 16 / 32 / 64 (flat above 16)
#endif
constexpr int kXRows = GB_XROWS;
constexpr int kXSlots = 2 * kSmaxSmem;  // 2048
constexpr int kXUnroll = 4;

#ifndef GB_LFILT_GRID
#define GB_LFILT_GRID 32  // filter grid x SMs (swept 8 / 16 / 32 / 64: 32-64 best)
#endif
#ifndef GB_XHUB
#define GB_XHUB 4  // hub rows (searched per sampled vertex) when d > GB_XHUB * take; swept 2 / 4 / 8 / 16
#endif
#ifndef GB_XSEARCH
#define GB_XSEARCH 4  // swept 2 / 4 / 8 / 16 (cfg3: 13.1 / 13.6 / 13.4 / 12.7K)
#endif
constexpr int kXSearch = GB_XSEARCH;  // hub-row binary searches in flight per lane

__device__ __forceinline__ uint32_t xhash(int32_t v) {
  return ((uint32_t)v * 0x9E3779B1u) >> (32 - 11);  // kXSlots = 2^11
}

__global__ void __launch_bounds__(kLadiesThreads) k_lad_extract_hash(
    const int64_t* __restrict__ qoff, int64_t k, int64_t chunks, const int32_t* __restrict__ qcol,
    const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
    const int64_t* __restrict__ fptr, const int32_t* __restrict__ fcol,
    const int64_t* __restrict__ coloff, const int64_t* __restrict__ slot,
    int32_t* __restrict__ slots, int32_t* __restrict__ rcnt) {
  __shared__ int32_t hkey[kXSlots];
  __shared__ int16_t hval[kXSlots];
  __shared__ int32_t sS[kSmaxSmem];
  __shared__ int s_next;
  const unsigned FULL = 0xffffffffu;
  const int lane = lane_id();
  for (int64_t item = blockIdx.x; item < k * chunks; item += gridDim.x) {
    const int64_t i = item / chunks, c = item - i * chunks;
    const int64_t q0 = qoff[i] + c * kXRows, q1 = min(q0 + kXRows, qoff[i + 1]);
    if (q0 >= q1) continue;  // uniform over the CTA
    const int64_t f0 = fptr[i], take = fptr[i + 1] - f0;
    for (int x = threadIdx.x; x < kXSlots; x += blockDim.x) hkey[x] = -1;
    if (threadIdx.x == 0) s_next = 0;
    __syncthreads();
    for (int64_t r = threadIdx.x; r < take; r += blockDim.x) {
      const int32_t v = fcol[f0 + r];
      sS[r] = v;
      uint32_t h = xhash(v);
      while (atomicCAS(&hkey[h], -1, v) != -1) h = (h + 1) & (kXSlots - 1);
      hval[h] = (int16_t)r;
    }
    __syncthreads();
    const int64_t cb = coloff[i];
    for (;;) {
      int r = 0;
      if (lane == 0) r = atomicAdd(&s_next, 1);
      r = __shfl_sync(FULL, r, 0);
      const int64_t q = q0 + r;
      if (q >= q1) break;
      const int32_t u = qcol[q];
      const int64_t a0 = rowptr[u], d = rowptr[u + 1] - a0;
      int32_t* out = slots + slot[q];
      int64_t o = 0;
      if (d > GB_XHUB * take) {
        // hub row: search each sampled vertex in A[u,:] (sorted), kXSearch
        // searches per lane in lock-step so their loads are in flight together
        // (log2 d round trips per kXSearch * 32 sampled vertices)
        const int nsteps = 32 - __clz((int)d);
        for (int64_t r0 = 0; r0 < take; r0 += 32 * kXSearch) {
          int32_t v[kXSearch], lo[kXSearch], hi[kXSearch];
#pragma unroll
          for (int j = 0; j < kXSearch; ++j) {
            const int64_t r = r0 + 32 * j + lane;
            v[j] = r < take ? sS[r] : 0;
            lo[j] = 0;
            hi[j] = r < take ? (int32_t)d : 0;
          }
          for (int step = 0; step < nsteps; ++step) {
            int32_t cm[kXSearch];
#pragma unroll
            for (int j = 0; j < kXSearch; ++j)
              cm[j] = lo[j] < hi[j] ? __ldg(col + a0 + ((lo[j] + hi[j]) >> 1)) : 0;
#pragma unroll
            for (int j = 0; j < kXSearch; ++j) {
              if (lo[j] < hi[j]) {
                const int32_t mid = (lo[j] + hi[j]) >> 1;
                if (cm[j] < v[j]) lo[j] = mid + 1; else hi[j] = mid;
              }
            }
          }
          int32_t at[kXSearch];
#pragma unroll
          for (int j = 0; j < kXSearch; ++j) {
            const int64_t r = r0 + 32 * j + lane;
            at[j] = r < take && lo[j] < d ? __ldg(col + a0 + lo[j]) : -1;
          }
#pragma unroll
          for (int j = 0; j < kXSearch; ++j) {
            const int64_t r = r0 + 32 * j + lane;
            const bool hit = r < take && at[j] == v[j];
            const unsigned bal = __ballot_sync(FULL, hit);
            if (hit) out[o + __popc(bal & ((1u << lane) - 1))] = (int32_t)(cb + r);
            o += __popc(bal);
          }
        }
        if (lane == 0) rcnt[q] = (int32_t)o;
        continue;
      }
      for (int64_t e0 = 0; e0 < d; e0 += 32 * kXUnroll) {
        int32_t vv[kXUnroll];
#pragma unroll
        for (int w = 0; w < kXUnroll; ++w) {
          const int64_t e = e0 + 32 * w + lane;
          vv[w] = e < d ? __ldg(col + a0 + e) : -1;
        }
#pragma unroll
        for (int w = 0; w < kXUnroll; ++w) {
          int rank = -1;
          const int32_t v = vv[w];
          if (v >= 0) {
            uint32_t h = xhash(v);
            int32_t kk;
            while ((kk = hkey[h]) != -1) {
              if (kk == v) { rank = hval[h]; break; }
              h = (h + 1) & (kXSlots - 1);
            }
          }
          const unsigned bal = __ballot_sync(FULL, rank >= 0);
          if (rank >= 0) out[o + __popc(bal & ((1u << lane) - 1))] = (int32_t)(cb + rank);
          o += __popc(bal);
        }
      }
      if (lane == 0) rcnt[q] = (int32_t)o;
    }
    __syncthreads();  // hash reused by the next item
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

__global__ void __launch_bounds__(kLadiesThreads) k_lad_pack_a(
    const int64_t* __restrict__ qoff, int64_t k, const int64_t* __restrict__ slot,
    const int32_t* __restrict__ slots, const int64_t* __restrict__ aptr,
    int32_t* __restrict__ acol) {
  const int lane = lane_id();
  const int64_t QN = qoff[k];
  for (int64_t q = global_warp(); q < QN; q += grid_warps()) {
    const int64_t o = aptr[q], c = aptr[q + 1] - o, s0 = slot[q];
    for (int64_t x = lane; x < c; x += 32) acol[o + x] = slots[s0 + x];
  }
}

__global__ void k_lad_sizes(const int64_t* __restrict__ qoff, int64_t k,
                            const int64_t* __restrict__ aptr, const int64_t* __restrict__ nnz_b,
                            int64_t* __restrict__ sizes) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int64_t QN = qoff[k];
  int64_t p = 0;
  for (int64_t i = 0; i < k; ++i) p += nnz_b[i];
  sizes[0] = QN;
  sizes[2] = aptr[QN];
  sizes[4] = p;
}

__global__ void k_lad_set(int64_t* p, int64_t v) { *p = v; }

__global__ void k_lad_flag(const int32_t* __restrict__ overflow, int64_t* __restrict__ size) {
  if (*overflow) *size = -(int64_t)*overflow;
}

// counts e_v <= |Q_i| live in packed 16-bit counters: a batch of more than
// 65535 rows is flagged (code 2) instead of silently carrying into the
// neighbouring counter (fanouts are checked on the host)
constexpr int64_t kMaxCount16 = 65535;
__global__ void k_lad_qcheck(const int64_t* __restrict__ qoff, int64_t k,
                             int32_t* __restrict__ overflow) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
       i += (int64_t)gridDim.x * blockDim.x)
    if (qoff[i + 1] - qoff[i] > kMaxCount16) atomicOr(overflow, 2);
}

// ============================================================== host side

static int gcap(int64_t n, int threads, int cap) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

struct LadiesWs {
  uint32_t* cnt32;   // packed uint16 counters of one group
  int64_t* nnz_b;    // k + 1
  int64_t* gpoff;    // group + 1
  int32_t* pv;       // group P cap
  int32_t* pe;
  double* sw;        // exact scratch
  double* sc;
  uint32_t* keys;    // race keys
  int32_t* cand;     // race candidates (P layout)
  int32_t* ncand;    // group
  uint32_t* hist;    // group * kBins
  int32_t* bound;    // group * 2
  int32_t* sel;      // k * s_max
  int32_t* nsel;     // k
  int64_t* take;     // k
  int32_t* Sfix;     // k * s_max
  int64_t* qg;       // Q cap + 1 (degree prefix of Q rows)
  int64_t* slot;     // Q cap + 1
  int32_t* slots;    // Q cap * s_max
  int32_t* rcnt;     // Q cap
  int64_t* tile_off; // compaction tiles + 1
  int64_t* scan_ws;
  int64_t* d_scalar; // 4 device scalars (k, words, tiles, n)
  int32_t* overflow;
  // race mode, column tiles
  int32_t* tb;       // tile bounds (ntiles_max + 1)
  int64_t* cpre;     // cut prefix (n + 1)
  int64_t* ntiles;   // device scalar
  unsigned long long* tst;  // tile ticket
  int32_t* tcnt;     // nonzeros per (batch, tile), gsize * ntiles_max
  size_t bytes;
};

static size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

struct LadiesPlan {
  int64_t gsize, words, tiles, p_cap, q_cap, s_max;
  bool tiled;          // race mode: column-tile counting, no dense counters
  int64_t ntiles_max;  // column tiles
  int64_t n;
};

constexpr int64_t kTiledGroupBytes = 16ll << 30;  // P layout (v, key, candidate) of one group

static LadiesPlan ladies_plan(int64_t k, int64_t n, int64_t q1_cap, int32_t layers,
                              const int64_t* fanouts, int32_t mode) {
  LadiesPlan p{};
  p.n = n;
  p.tiled = mode == GB_LADIES_RACE;
  p.s_max = 1;
  p.q_cap = q1_cap;
  for (int32_t l = 0; l < layers; ++l) {
    if (fanouts[l] > p.s_max) p.s_max = fanouts[l];
    if (k * fanouts[l] > p.q_cap) p.q_cap = k * fanouts[l];
  }
  p.gsize = n > 0 ? (p.tiled ? kTiledGroupBytes / (12 * n) : kGroupBytes / (2 * n)) : k;
  if (p.gsize < 1) p.gsize = 1;
  if (p.gsize > k) p.gsize = k > 0 ? k : 1;
  p.words = p.tiled ? 1 : (p.gsize * n + 1) / 2 + 1;
  p.tiles = p.tiled ? 1 : (2 * p.words + kCompTile - 1) / kCompTile;
  p.p_cap = p.gsize * n;
  p.ntiles_max = p.tiled ? n / kLTileW + kLMassTiles + 2 : 1;
  return p;
}

static LadiesWs ladies_ws_layout(char* base, int64_t k, const LadiesPlan& P, bool exact) {
  LadiesWs w{};
  size_t off = 0;
  auto take = [&](size_t bytes) { char* p = base ? base + off : nullptr; off += al(bytes); return p; };
  w.cnt32 = (uint32_t*)take(sizeof(uint32_t) * P.words);
  w.nnz_b = (int64_t*)take(sizeof(int64_t) * (k + 1));
  w.gpoff = (int64_t*)take(sizeof(int64_t) * (P.gsize + 1));
  w.pv = (int32_t*)take(sizeof(int32_t) * (P.p_cap + 1));
  w.pe = (int32_t*)take(P.tiled ? 8 : sizeof(int32_t) * (P.p_cap + 1));  // counts: exact only
  w.sw = (double*)take(exact ? sizeof(double) * (P.p_cap + 1) : 8);
  w.sc = (double*)take(exact ? sizeof(double) * (P.p_cap + 1) : 8);
  w.keys = (uint32_t*)take(exact ? 8 : sizeof(uint32_t) * (P.p_cap + 1));
  w.cand = (int32_t*)take(exact ? 8 : sizeof(int32_t) * (P.p_cap + 1));
  w.ncand = (int32_t*)take(sizeof(int32_t) * (P.gsize + 1));
  w.hist = (uint32_t*)take(sizeof(uint32_t) * P.gsize * kBins);
  w.bound = (int32_t*)take(sizeof(int32_t) * 2 * (P.gsize + 1));
  w.sel = (int32_t*)take(sizeof(int32_t) * (k * P.s_max + 1));
  w.nsel = (int32_t*)take(sizeof(int32_t) * (k + 1));
  w.take = (int64_t*)take(sizeof(int64_t) * (k + 1));
  w.Sfix = (int32_t*)take(sizeof(int32_t) * (k * P.s_max + 1));
  w.qg = (int64_t*)take(sizeof(int64_t) * (P.q_cap + 1));
  w.slot = (int64_t*)take(sizeof(int64_t) * (P.q_cap + 1));
  w.slots = (int32_t*)take(sizeof(int32_t) * (P.q_cap * P.s_max + 1));
  w.rcnt = (int32_t*)take(sizeof(int32_t) * (P.q_cap + 1));
  w.tile_off = (int64_t*)take(sizeof(int64_t) * (P.tiles + 1));
  int64_t sn = P.q_cap > k ? P.q_cap : k;
  if (P.tiles > sn) sn = P.tiles;
  if (P.tiled && P.n + 1 > sn) sn = P.n + 1;
  w.scan_ws = (int64_t*)take(sizeof(int64_t) * scan_workspace_elems<int64_t>(sn + 1));
  w.d_scalar = (int64_t*)take(sizeof(int64_t) * 4);
  w.overflow = (int32_t*)take(sizeof(int32_t));
  w.tb = (int32_t*)take(sizeof(int32_t) * (P.ntiles_max + 1));
  w.cpre = (int64_t*)take(P.tiled ? sizeof(int64_t) * (P.n + 2) : 8);
  w.ntiles = (int64_t*)take(sizeof(int64_t));
  w.tst = (unsigned long long*)take(sizeof(unsigned long long) * 2);
  w.tcnt = (int32_t*)take(sizeof(int32_t) * (P.gsize * P.ntiles_max + 1));
  w.bytes = off;
  return w;
}

int ladies_workspace(const Graph* g, int64_t k, int64_t q1_cap, int32_t layers,
                     const int64_t* fanouts, int32_t mode, size_t* bytes) {
  const LadiesPlan P = ladies_plan(k, g->n, q1_cap, layers, fanouts, mode);
  *bytes = ladies_ws_layout(nullptr, k, P, mode == GB_LADIES_EXACT).bytes;
  return GB_OK;
}

int ladies_bulk(const Graph* g, int64_t k, const int64_t* d_qoff, const int32_t* d_qverts,
                int64_t q1_cap, int32_t layers, const int64_t* fanouts, uint64_t seed,
                uint64_t epoch, int64_t batch_offset, int32_t mode, gb_ladies_layer_out* L,
                int64_t* d_sizes, void* d_ws, size_t ws_bytes, cudaStream_t st,
                const LadiesRows* src) {
  const bool exact = mode == GB_LADIES_EXACT;
  const int64_t n = g->n;
  // rows of Q: the graph's, or (one layer) a local CSR of the Q rows with
  // global column ids, Q given as local row indices (1.5D batch slices)
  if (src && layers != 1) {
    set_error("ladies: a local row source serves exactly one layer");
    return GB_ERR_CONTRACT;
  }
  const int64_t* RP = src ? src->rowptr : g->rowptr;
  const int32_t* CL = src ? src->col : g->col;
  const LadiesPlan P = ladies_plan(k, n, q1_cap, layers, fanouts, mode);
  LadiesWs ws = ladies_ws_layout((char*)d_ws, k, P, exact);
  if (ws.bytes > ws_bytes) {
    set_error("ladies workspace too small: need %zu bytes, got %zu", ws.bytes, ws_bytes);
    return GB_ERR_CAPACITY;
  }
  int64_t qc = q1_cap;
  for (int32_t l = 0; l < layers; ++l) {
    if (fanouts[l] < 1 || fanouts[l] > kMaxCount16) {
      set_error("ladies layer %d: fanout %lld outside 1..%lld (16-bit counts)", (int)l + 1,
                (long long)fanouts[l], (long long)kMaxCount16);
      return GB_ERR_UNSUPPORTED;
    }
    if (L[l].q_cap < qc || L[l].f_cap < k * fanouts[l] || L[l].a_cap < qc * fanouts[l]) {
      set_error("ladies layer %d output too small", (int)l + 1);
      return GB_ERR_CAPACITY;
    }
    qc = k * fanouts[l];
  }
  int sms = 0, cur_dev = 0;
  cudaGetDevice(&cur_dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cur_dev);
  if (sms <= 0) sms = kNumSMs;
  int64_t* d_k = ws.d_scalar;
  int64_t* d_tiles = ws.d_scalar + 1;
  GB_CUDA(cudaMemsetAsync(ws.cnt32, 0, sizeof(uint32_t) * P.words, st));
  GB_CUDA(cudaMemsetAsync(ws.overflow, 0, sizeof(int32_t), st));
  k_lad_set<<<1, 1, 0, st>>>(d_k, k);
  k_lad_set<<<1, 1, 0, st>>>(d_tiles, P.tiles);
  k_lad_qcheck<<<gcap(k, 256, 64), 256, 0, st>>>(d_qoff, k, ws.overflow);
  count_launches(3);
  int tile_grid = 0;
  const size_t tile_smem = sizeof(uint32_t) * (kLTileW / 2 + kBins) +
                           (sizeof(int64_t) + 3 * sizeof(int32_t) + sizeof(int16_t)) *
                               kLRowsSmem;
  if (P.tiled) {
    // column tiles of this graph: cuts every kLTileW columns and at
    // kLMassTiles quantiles of the degree mass
    int64_t* d_n = ws.d_scalar + 3;
    k_lad_set<<<1, 1, 0, st>>>(d_n, n);
    const int64_t mass = g->nnz / kLMassTiles + 1;
    int rc = device_exclusive_scan<int64_t>(d_n, n, CutF{g->rowptr, n, mass}, ws.cpre, ws.scan_ws,
                                            st);
    if (rc) return rc;
    k_lad_tiles<<<gcap(n + 1, 256, 16 * sms), 256, 0, st>>>(g->rowptr, n, mass, ws.cpre, ws.tb,
                                                          ws.ntiles);
    GB_LAUNCH_CHECK("k_lad_tiles");
    // the smem attribute and the occupancy are per device
    static int s_grid[16] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    int& grid_dev = s_grid[dev < 16 ? dev : 0];
    if (!grid_dev) {
      cudaFuncSetAttribute(k_lad_tile, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)tile_smem);
      int occ = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_lad_tile, kLTileThreads, tile_smem);
      grid_dev = (occ > 0 ? occ : 1) * sms;
    }
    tile_grid = grid_dev;
    count_launches(2);
  }
  qc = q1_cap;
  for (int32_t l = 0; l < layers; ++l) {
    const int32_t s = (int32_t)fanouts[l];
    gb_ladies_layer_out& o = L[l];
    const int64_t* qoff = l == 0 ? d_qoff : L[l - 1].fptr;
    const int32_t* qcol = l == 0 ? (src ? src->qrow : d_qverts) : L[l - 1].fcol;
    const int64_t* d_QN = qoff + k;
    int64_t* sizes = d_sizes + kLadiesSizes * l;
    int rc = GB_OK;
    if (!P.tiled) {
      rc = device_exclusive_scan<int64_t>(d_QN, qc, QDegF{qcol, RP}, ws.qg, ws.scan_ws, st);
      if (rc) return rc;
    }
    GB_CUDA(cudaMemsetAsync(ws.nnz_b, 0, sizeof(int64_t) * (k + 1), st));
    for (int64_t g0 = 0; g0 < k; g0 += P.gsize) {
      const int64_t g1 = g0 + P.gsize < k ? g0 + P.gsize : k;
      const int64_t gn = g1 - g0;
      const int64_t words = (gn * n + 1) / 2;
      const uint64_t depth = src ? (uint64_t)src->depth : (uint64_t)(l + 1);
      const RaceKey rk{seed, epoch, depth, batch_offset + g0};
      if (P.tiled) {
        // ---- P = Q A, race keys and key histograms for this group, one pass
        GB_CUDA(cudaMemsetAsync(ws.tst, 0, sizeof(unsigned long long), st));
        GB_CUDA(cudaMemsetAsync(ws.hist, 0, sizeof(uint32_t) * gn * kBins, st));
        LadTileArgs T{};
        T.qoff = qoff; T.qcol = qcol; T.rowptr = RP; T.col = CL; T.tb = ws.tb;
        T.ntiles = ws.ntiles; T.n = n; T.g0 = g0; T.gn = gn; T.rk = rk; T.ticket = ws.tst;
        T.pv = ws.pv; T.keys = ws.keys; T.tcnt = ws.tcnt; T.hist = ws.hist; T.nnz_b = ws.nnz_b;
        prof_mark(st);
        k_lad_tile<<<tile_grid, kLTileThreads, tile_smem, st>>>(T);
        GB_LAUNCH_CHECK("k_lad_tile");
        prof_mark(st);
        k_lad_slot_off<<<gcap(gn + 1, 128, 64), 128, 0, st>>>(gn, n, ws.gpoff);
        count_launches(2);
      } else {
        // ---- P = Q A for this group
        prof_mark(st);
        k_lad_count<<<4 * sms, kLadiesThreads, 0, st>>>(qoff, k, g0, g1, qcol, ws.qg, RP, CL, n,
                                                        ws.cnt32, ws.nnz_b);
        GB_LAUNCH_CHECK("k_lad_count");
        prof_mark(st);
        k_lad_compact_count<<<gcap(P.tiles, 1, 8 * sms), 256, 0, st>>>(ws.cnt32, words, n, g0,
                                                                      ws.tile_off, ws.nnz_b);
        k_lad_gpoff<<<1, 1, 0, st>>>(ws.nnz_b, g0, gn, ws.gpoff);
        rc = device_exclusive_scan<int64_t>(d_tiles, P.tiles, TileF{ws.tile_off}, ws.tile_off,
                                            ws.scan_ws, st);
        if (rc) return rc;
        k_lad_compact_write<<<gcap(P.tiles, 1, 8 * sms), 256, 0, st>>>(
            ws.cnt32, words, n, ws.tile_off, ws.pv, ws.pe, nullptr);
        GB_LAUNCH_CHECK("k_lad_compact");
      }
      // ---- NORM + SAMPLE
      LadiesSampleArgs A{};
      A.gpoff = ws.gpoff; A.pv = ws.pv; A.pe = ws.pe; A.g0 = g0; A.gn = gn; A.s = s;
      A.batch_offset = batch_offset; A.seed = seed; A.epoch = epoch; A.depth = depth;
      A.sw = ws.sw; A.sc = ws.sc; A.keys = ws.keys; A.sel = ws.sel; A.nsel = ws.nsel;
      A.take = ws.take;
      A.nnzb = P.tiled ? ws.nnz_b : nullptr;
      if (exact) {
        k_lad_sample_exact<<<gcap(gn, 32, 4 * sms), 32, 0, st>>>(A);
        count_launches(1);
      } else {
        GB_CUDA(cudaMemsetAsync(ws.ncand, 0, sizeof(int32_t) * (gn + 1), st));
        if (!P.tiled) {
          GB_CUDA(cudaMemsetAsync(ws.hist, 0, sizeof(uint32_t) * gn * kBins, st));
          k_lad_keys<<<16 * sms, 256, 0, st>>>(A, rk);
          k_lad_hist<<<4 * sms, 256, 0, st>>>(A, ws.hist);
        }
        k_lad_boundary<<<(int)gn, 256, 0, st>>>(A, ws.hist, ws.bound);
        if (P.tiled)
          k_lad_filter_tiles<<<GB_LFILT_GRID * sms, 256, 0, st>>>(A, ws.tb, ws.ntiles, n, ws.tcnt, ws.bound,
                                                       ws.cand, ws.ncand, rk);
        else
          k_lad_filter<<<16 * sms, 256, 0, st>>>(A, ws.bound, ws.cand, ws.ncand);
        k_lad_refine<<<(int)gn, 1024, 0, st>>>(A, ws.bound, ws.cand, ws.ncand, ws.overflow);
        count_launches(P.tiled ? 3 : 5);
      }
      GB_LAUNCH_CHECK("k_lad_sample");
      k_lad_emit<<<(int)gn, 256, 0, st>>>(A, ws.Sfix, nullptr);
      GB_LAUNCH_CHECK("k_lad_emit");
      count_launches(6);
    }
    rc = device_exclusive_scan<int64_t>(d_k, k, TakeLF{ws.take}, o.fptr, ws.scan_ws, st);
    if (rc) return rc;
    k_lad_pack_s<<<gcap(k * s, 256, 16 * sms), 256, 0, st>>>(o.fptr, k, s, ws.Sfix, o.fcol);
    k_lad_layout<<<1, 1, 0, st>>>(o.fptr, k, o.coloff, sizes);
    // ---- EXTRACT A_S = Q_R A Q_C
    rc = device_exclusive_scan<int64_t>(d_QN, qc, RcapF{qcol, RP, qoff, o.fptr, k},
                                        ws.slot, ws.scan_ws, st);
    if (rc) return rc;
    if (s <= kSmaxSmem) {
      // rows per batch: the batch sizes (layer 1, bounded by the Q rows) or s
      const int64_t rows_max = l == 0 ? q1_cap : fanouts[l - 1];
      const int64_t chunks = (rows_max + kXRows - 1) / kXRows;
      k_lad_extract_hash<<<gcap(k * chunks, 1, 8 * sms), kLadiesThreads, 0, st>>>(
          qoff, k, chunks, qcol, RP, CL, o.fptr, o.fcol, o.coloff, ws.slot, ws.slots,
          ws.rcnt);
    } else {
      k_lad_extract<<<8 * sms, kLadiesThreads, 0, st>>>(qoff, k, qcol, RP, CL, o.fptr,
                                                       o.fcol, o.coloff, ws.slot, ws.slots,
                                                       ws.rcnt);
    }
    rc = device_exclusive_scan<int64_t>(d_QN, qc, RcntF{ws.rcnt}, o.aptr, ws.scan_ws, st);
    if (rc) return rc;
    k_lad_pack_a<<<8 * sms, kLadiesThreads, 0, st>>>(qoff, k, ws.slot, ws.slots, o.aptr, o.acol);
    k_lad_sizes<<<1, 1, 0, st>>>(qoff, k, o.aptr, ws.nnz_b, sizes);
    GB_LAUNCH_CHECK("k_lad_extract");
    count_launches(5);
    qc = k * s;
  }
  // capacity overflow anywhere in the bulk (race tie list): the last layer's
  // nnz(P) size becomes -flag for the caller
  k_lad_flag<<<1, 1, 0, st>>>(ws.overflow, d_sizes + kLadiesSizes * (layers - 1) + 4);
  count_launches(1);
  return GB_OK;
}

// ======================================== pieces of the 1.5D LADIES executor

struct QDegMF {
  const int32_t* qdeg;
  __device__ int64_t operator()(int64_t q) const { return qdeg[q]; }
};

// global offsets of a group's batches: poff[g0 + j + 1] = poff[g0 + j] + nnz
__global__ void k_lad_poff(const int64_t* __restrict__ nnz_b, int64_t g0, int64_t gn,
                           int64_t* __restrict__ poff) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    if (g0 == 0) poff[0] = 0;
    for (int64_t j = 0; j < gn; ++j) poff[g0 + j + 1] = poff[g0 + j] + nnz_b[g0 + j];
  }
}

size_t ladies_counts_ws(int64_t k, int64_t n, int64_t q_cap) {
  int64_t gsize = n > 0 ? kGroupBytes / (2 * n) : k;
  if (gsize < 1) gsize = 1;
  if (gsize > k) gsize = k > 0 ? k : 1;
  const int64_t words = (gsize * n + 1) / 2 + 1;
  const int64_t tiles = (2 * words + kCompTile - 1) / kCompTile;
  int64_t sn = q_cap > tiles ? q_cap : tiles;
  return al(sizeof(uint32_t) * words) + al(sizeof(int64_t) * (k + 1)) +
         al(sizeof(int64_t) * (q_cap + 1)) + al(sizeof(int64_t) * (tiles + 1)) +
         al(sizeof(int64_t) * scan_workspace_elems<int64_t>(sn + 1)) + al(sizeof(int64_t) * 4);
}

// Partial P = Q A over the rows with qdeg[q] > 0, read through the CSR
// (rowptr, col) addressed by qcol[q]: per batch the sorted (v, e) nonzeros
// at poff[i] (k + 1 offsets).  Same grouped counters as ladies_bulk.
int ladies_counts(int64_t k, const int64_t* qoff, const int32_t* qcol, const int32_t* qdeg,
                  int64_t q_cap, const int64_t* rowptr, const int32_t* col, int64_t n,
                  int64_t* poff, int32_t* pv, int32_t* pe, void* d_ws, size_t ws_bytes,
                  cudaStream_t st) {
  if (ladies_counts_ws(k, n, q_cap) > ws_bytes) {
    set_error("ladies counts workspace too small");
    return GB_ERR_CAPACITY;
  }
  int64_t gsize = n > 0 ? kGroupBytes / (2 * n) : k;
  if (gsize < 1) gsize = 1;
  if (gsize > k) gsize = k > 0 ? k : 1;
  const int64_t pwords = (gsize * n + 1) / 2 + 1;
  const int64_t tiles = (2 * pwords + kCompTile - 1) / kCompTile;
  char* p = (char*)d_ws;
  auto carve = [&](size_t bytes) { char* r = p; p += al(bytes); return r; };
  uint32_t* cnt32 = (uint32_t*)carve(sizeof(uint32_t) * pwords);
  int64_t* nnz_b = (int64_t*)carve(sizeof(int64_t) * (k + 1));
  int64_t* qg = (int64_t*)carve(sizeof(int64_t) * (q_cap + 1));
  int64_t* tile_off = (int64_t*)carve(sizeof(int64_t) * (tiles + 1));
  int64_t sn = q_cap > tiles ? q_cap : tiles;
  int64_t* scan_ws = (int64_t*)carve(sizeof(int64_t) * scan_workspace_elems<int64_t>(sn + 1));
  int64_t* d_tiles = (int64_t*)carve(sizeof(int64_t) * 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  if (sms <= 0) sms = kNumSMs;
  GB_CUDA(cudaMemsetAsync(cnt32, 0, sizeof(uint32_t) * pwords, st));
  GB_CUDA(cudaMemsetAsync(nnz_b, 0, sizeof(int64_t) * (k + 1), st));
  k_lad_set<<<1, 1, 0, st>>>(d_tiles, tiles);
  int rc = device_exclusive_scan<int64_t>(qoff + k, q_cap, QDegMF{qdeg}, qg, scan_ws, st);
  if (rc) return rc;
  if (k == 0) k_lad_poff<<<1, 1, 0, st>>>(nnz_b, 0, 0, poff);
  for (int64_t g0 = 0; g0 < k; g0 += gsize) {
    const int64_t g1 = g0 + gsize < k ? g0 + gsize : k;
    const int64_t gn = g1 - g0;
    const int64_t words = (gn * n + 1) / 2;
    k_lad_count<<<4 * sms, kLadiesThreads, 0, st>>>(qoff, k, g0, g1, qcol, qg, rowptr, col, n,
                                                    cnt32, nnz_b);
    k_lad_compact_count<<<gcap(tiles, 1, 8 * sms), 256, 0, st>>>(cnt32, words, n, g0, tile_off,
                                                                nnz_b);
    k_lad_poff<<<1, 1, 0, st>>>(nnz_b, g0, gn, poff);
    rc = device_exclusive_scan<int64_t>(d_tiles, tiles, TileF{tile_off}, tile_off, scan_ws, st);
    if (rc) return rc;
    k_lad_compact_write<<<gcap(tiles, 1, 8 * sms), 256, 0, st>>>(cnt32, words, n, tile_off, pv,
                                                                pe, poff + g0);
    GB_LAUNCH_CHECK("ladies_counts");
    count_launches(4);
  }
  return GB_OK;
}

// Sum of partial (batch, v, e) triples for the vertex range [v0, v0 + nloc)
// (the sparse merge of the 1.5D LADIES counts): RED adds into the grouped
// packed 16-bit counters, then the same compaction as ladies_counts.
__global__ void k_lad_merge_add(int64_t m, const int32_t* __restrict__ trip, int64_t g0,
                                int64_t g1, int64_t v0, int64_t nloc,
                                uint32_t* __restrict__ cnt32) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = trip[3 * t];
    if (b < g0 || b >= g1) continue;
    const int64_t idx = (b - g0) * nloc + (trip[3 * t + 1] - v0);
    atomicAdd(cnt32 + (idx >> 1), (uint32_t)trip[3 * t + 2] << ((uint32_t)(idx & 1) << 4));
  }
}

size_t ladies_merge_ws(int64_t k, int64_t nloc) { return ladies_counts_ws(k, nloc, 1); }

int ladies_merge_counts(int64_t k, int64_t m, const int32_t* trip, int64_t v0, int64_t nloc,
                        int64_t* poff, int32_t* pv, int32_t* pe, void* d_ws, size_t ws_bytes,
                        cudaStream_t st) {
  if (ladies_merge_ws(k, nloc) > ws_bytes) {
    set_error("ladies merge workspace too small");
    return GB_ERR_CAPACITY;
  }
  int64_t gsize = nloc > 0 ? kGroupBytes / (2 * nloc) : k;
  if (gsize < 1) gsize = 1;
  if (gsize > k) gsize = k > 0 ? k : 1;
  const int64_t pwords = (gsize * nloc + 1) / 2 + 1;
  const int64_t tiles = (2 * pwords + kCompTile - 1) / kCompTile;
  char* p = (char*)d_ws;
  auto carve = [&](size_t bytes) { char* r = p; p += al(bytes); return r; };
  uint32_t* cnt32 = (uint32_t*)carve(sizeof(uint32_t) * pwords);
  int64_t* nnz_b = (int64_t*)carve(sizeof(int64_t) * (k + 1));
  carve(sizeof(int64_t) * 2);  // (q rows of ladies_counts_ws: unused here)
  int64_t* tile_off = (int64_t*)carve(sizeof(int64_t) * (tiles + 1));
  const int64_t sn = tiles > 1 ? tiles : 1;
  int64_t* scan_ws = (int64_t*)carve(sizeof(int64_t) * scan_workspace_elems<int64_t>(sn + 1));
  int64_t* d_tiles = (int64_t*)carve(sizeof(int64_t) * 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  if (sms <= 0) sms = kNumSMs;
  GB_CUDA(cudaMemsetAsync(cnt32, 0, sizeof(uint32_t) * pwords, st));
  GB_CUDA(cudaMemsetAsync(nnz_b, 0, sizeof(int64_t) * (k + 1), st));
  k_lad_set<<<1, 1, 0, st>>>(d_tiles, tiles);
  if (k == 0) k_lad_poff<<<1, 1, 0, st>>>(nnz_b, 0, 0, poff);
  for (int64_t g0 = 0; g0 < k; g0 += gsize) {
    const int64_t g1 = g0 + gsize < k ? g0 + gsize : k;
    const int64_t gn = g1 - g0;
    const int64_t words = (gn * nloc + 1) / 2;
    if (m > 0)
      k_lad_merge_add<<<gcap(m, 256, 16 * sms), 256, 0, st>>>(m, trip, g0, g1, v0, nloc, cnt32);
    k_lad_compact_count<<<gcap(tiles, 1, 8 * sms), 256, 0, st>>>(cnt32, words, nloc, g0,
                                                                tile_off, nnz_b);
    k_lad_poff<<<1, 1, 0, st>>>(nnz_b, g0, gn, poff);
    int rc = device_exclusive_scan<int64_t>(d_tiles, tiles, TileF{tile_off}, tile_off, scan_ws, st);
    if (rc) return rc;
    k_lad_compact_write<<<gcap(tiles, 1, 8 * sms), 256, 0, st>>>(cnt32, words, nloc, tile_off, pv,
                                                                pe, poff + g0, (int32_t)v0);
    GB_LAUNCH_CHECK("ladies_merge_counts");
    count_launches(5);
  }
  return GB_OK;
}

constexpr int64_t kSelGroup = 64;  // batches per race-select pass

size_t ladies_race_topk_ws(int64_t k, int64_t p_cap, int32_t s) {
  return al(sizeof(uint32_t) * (p_cap + 1)) + al(sizeof(int32_t) * (p_cap + 1)) +
         al(sizeof(int32_t) * (kSelGroup + 1)) + al(sizeof(uint32_t) * kSelGroup * kBins) +
         al(sizeof(int32_t) * 2 * (kSelGroup + 1)) + al(sizeof(int32_t) * (k * s + 1)) +
         al(sizeof(int32_t) * (k + 1)) + al(sizeof(int32_t));
}

// Exponential-race top-s of every batch's (v, e) list: take[i], the sorted
// selected vertices Sv[i*s ...] and their keys Sk (for a distributed merge).
int ladies_race_topk(int64_t k, const int64_t* poff, const int32_t* pv, const int32_t* pe,
                     int64_t p_cap, int32_t s, uint64_t seed, uint64_t epoch, uint64_t depth,
                     int64_t batch_offset, int64_t* take, int32_t* Sv, uint32_t* Sk, void* d_ws,
                     size_t ws_bytes, cudaStream_t st) {
  if (ladies_race_topk_ws(k, p_cap, s) > ws_bytes) {
    set_error("ladies race workspace too small");
    return GB_ERR_CAPACITY;
  }
  char* p = (char*)d_ws;
  auto carve = [&](size_t bytes) { char* r = p; p += al(bytes); return r; };
  uint32_t* keys = (uint32_t*)carve(sizeof(uint32_t) * (p_cap + 1));
  int32_t* cand = (int32_t*)carve(sizeof(int32_t) * (p_cap + 1));
  int32_t* ncand = (int32_t*)carve(sizeof(int32_t) * (kSelGroup + 1));
  uint32_t* hist = (uint32_t*)carve(sizeof(uint32_t) * kSelGroup * kBins);
  int32_t* bound = (int32_t*)carve(sizeof(int32_t) * 2 * (kSelGroup + 1));
  int32_t* sel = (int32_t*)carve(sizeof(int32_t) * (k * s + 1));
  int32_t* nsel = (int32_t*)carve(sizeof(int32_t) * (k + 1));
  int32_t* overflow = (int32_t*)carve(sizeof(int32_t));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  if (sms <= 0) sms = kNumSMs;
  for (int64_t g0 = 0; g0 < k; g0 += kSelGroup) {
    const int64_t gn = g0 + kSelGroup < k ? kSelGroup : k - g0;
    LadiesSampleArgs A{};
    A.gpoff = poff + g0; A.pv = pv; A.pe = pe; A.g0 = g0; A.gn = gn; A.s = s;
    A.batch_offset = batch_offset; A.seed = seed; A.epoch = epoch; A.depth = depth;
    A.keys = keys; A.sel = sel; A.nsel = nsel; A.take = take;
    const RaceKey rk{seed, epoch, depth, batch_offset + g0};
    GB_CUDA(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * gn * kBins, st));
    GB_CUDA(cudaMemsetAsync(ncand, 0, sizeof(int32_t) * (gn + 1), st));
    k_lad_keys<<<16 * sms, 256, 0, st>>>(A, rk);
    k_lad_hist<<<4 * sms, 256, 0, st>>>(A, hist);
    k_lad_boundary<<<(int)gn, 256, 0, st>>>(A, hist, bound);
    k_lad_filter<<<16 * sms, 256, 0, st>>>(A, bound, cand, ncand);
    k_lad_refine<<<(int)gn, 1024, 0, st>>>(A, bound, cand, ncand, overflow);
    k_lad_emit<<<(int)gn, 256, 0, st>>>(A, Sv, Sk);
    GB_LAUNCH_CHECK("ladies_race_topk");
    count_launches(6);
  }
  return GB_OK;
}

int ladies_extract_rows(int64_t k, const int64_t* qoff, const int32_t* qcol,
                        const int64_t* rowptr, const int32_t* col, const int64_t* fptr,
                        const int32_t* fcol, const int64_t* coloff, const int64_t* slot,
                        int32_t* slots, int32_t* rcnt, cudaStream_t st) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  if (sms <= 0) sms = kNumSMs;
  k_lad_extract<<<8 * sms, kLadiesThreads, 0, st>>>(qoff, k, qcol, rowptr, col, fptr, fcol, coloff,
                                                   slot, slots, rcnt);
  GB_LAUNCH_CHECK("ladies_extract_rows");
  count_launches(1);
  return GB_OK;
}

}  // namespace gb
