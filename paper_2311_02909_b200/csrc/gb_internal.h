// Internal (C++) declarations shared by the library translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/gnnbulk_b200.h"

namespace gb {

constexpr int kMaxRuns = 64;  // replay-table runs per degree (<= 33 + binades observed)
constexpr int kBinades = 64;  // binade index entries per degree

// Device CSR adjacency + exact-replay tables (opaque gb_graph).
struct Graph {
  int64_t n = 0, nnz = 0;
  const int64_t* rowptr = nullptr;  // caller-owned device memory
  const int32_t* col = nullptr;     // caller-owned, readable for nnz + GB_COL_PAD
  int64_t max_deg = 0, slots = 0;
  int32_t* deg_slot = nullptr;      // [max_deg + 1] -> table slot or -1
  int32_t* slot_deg = nullptr;      // [slots]
  int32_t* run_j0 = nullptr;        // [slots * (kMaxRuns + 1)]
  double2* run_sd = nullptr;        // [slots * kMaxRuns] (run start S, increment)
  int32_t* run_n = nullptr;         // [slots]
  int8_t* run_lower = nullptr;      // [slots * kBinades] binade index
};

// Launch accounting (gb_launch_counter) and optional CUDA-event marks around
// the dominant kernels (gb_profile_begin / gb_profile_end), host-thread local.
void count_launches(int n);
void prof_mark(cudaStream_t st);

// Fork n <= kForkStreams side streams off st (they wait for st's work so
// far), launch on fork_stream(i), then fork_join makes st wait for them.
constexpr int kForkStreams = 3;
cudaStream_t fork_begin(cudaStream_t st, int n);
cudaStream_t fork_stream(int i);
void fork_join(cudaStream_t st, int n);
// waiter continues only after src's work enqueued so far
void stream_wait(cudaStream_t waiter, cudaStream_t src);
// per-device event ring for ordering across streams (i mod kEventRing)
constexpr int kEventRing = 8;
cudaEvent_t ring_event(int i);

int graph_build_tables(Graph* g, cudaStream_t st);
// device COO -> CSR (gb_csr.cu)
int bits_for(int64_t n);
size_t radix_sort_ws(int64_t m);
int radix_sort(uint64_t* keys, uint64_t* alt, uint32_t* vals, uint32_t* valt, int64_t m,
               int bits, void* ws, size_t ws_bytes, bool* in_alt, cudaStream_t st);
size_t csr_from_keys_ws(int64_t n, int64_t m);
int csr_from_keys(uint64_t* keys, int64_t m, uint64_t end, int sb, int64_t n, int64_t* rowptr,
                  int32_t* col, int64_t** d_nnz, void* ws, size_t ws_bytes, cudaStream_t st);
int spmm_rows(int64_t R, const int64_t* rowptr, const int32_t* col, const int64_t* rowb,
              const int64_t* shift, int64_t k, const float* X, int64_t f, float* Y,
              cudaStream_t st);
int spmm_f64(int64_t R, const int64_t* rowptr, const int32_t* col, const double* val,
             const double* X, int64_t f, double* Y, cudaStream_t st);
int segment_copy(int64_t m, const int64_t* rows, const int64_t* src_off, const int32_t* lens,
                 const int32_t* src, const int64_t* dst_off, int32_t* dst, cudaStream_t st);
size_t sage_owner_p2p_ws(int64_t r_cap);
int sage_owner_p2p(const Graph* tables, int64_t ngroups, const int32_t* const* rows,
                   const int64_t* const* brow, const int64_t* const* fptr, const int64_t* boff,
                   int64_t k, int64_t r_cap, int32_t ndst, int32_t* const* dst, int64_t lo,
                   int64_t hi, const int64_t* brp, const int32_t* bcol, int32_t s, int64_t stride,
                   uint64_t seed, uint64_t epoch, uint64_t depth, void* d_ws, size_t ws_bytes,
                   cudaStream_t st);
int first_occurrence(int64_t F, const int32_t* colidx, const int64_t* eb, const int64_t* shift,
                     int64_t k, int64_t ncols, int32_t* first, cudaStream_t st);
int sage_workspace(const Graph* g, int64_t k, int64_t r1_cap, int32_t layers,
                   const int64_t* fanouts, size_t* bytes);
// rows held by peers (1.5D batch split): device arrays of the block bounds
// (nblk + 1) and of the blocks' CSR pointers in their owners' memory
struct PeerRowsHost {
  int nblk;
  const int64_t* bounds;
  const int64_t* const* brp;
  const int32_t* const* bcol;
};
int sage_bulk(const Graph* g, int64_t k, const int64_t* d_bptr, const int32_t* d_bverts,
              int64_t r1_cap, int64_t batch_size, int32_t layers, const int64_t* fanouts,
              uint64_t seed, uint64_t epoch, int64_t batch_offset, int32_t mode,
              gb_sage_layer_out* L, int64_t* d_sizes, void* d_ws, size_t ws_bytes,
              cudaStream_t st, const PeerRowsHost* peer = nullptr);
size_t sage_layer_sample_ws(int64_t r_cap, int64_t f_cap);
int sage_layer_sample(const Graph* tables, int64_t k, const int64_t* brow, int64_t r_cap,
                      const int32_t* rowv, const int32_t* deg, const int64_t* fptr,
                      const int64_t* rowptr, const int32_t* col, int32_t s, int64_t stride,
                      int64_t batch_offset, uint64_t seed, uint64_t epoch, uint64_t depth,
                      int32_t mode, int32_t* fcol, void* d_ws, size_t ws_bytes, cudaStream_t st);
int sage_sample_keyed(const Graph* tables, int64_t R, const int64_t* d_R, const int32_t* rowv,
                      const int32_t* deg, const int64_t* fptr, const int64_t* rowkeys,
                      const int64_t* rowptr, const int32_t* col, int32_t s, uint64_t seed,
                      uint64_t epoch, uint64_t depth, int32_t* fcol, cudaStream_t st);
size_t sage_layer_extract_ws(int64_t n, int64_t k);
int sage_layer_extract(int64_t n, int64_t k, const int64_t* brow, const int64_t* fptr,
                       const int32_t* fcol, int64_t f_cap, int32_t* acol, int32_t* colv,
                       int64_t* eoff, int64_t* coloff, int64_t* sizes, void* d_ws,
                       size_t ws_bytes, cudaStream_t st);
int take_scan(int64_t r_cap, const int64_t* R_ptr, const int32_t* deg, int32_t s, int64_t* fptr,
              int64_t* scan_ws, cudaStream_t st);
int gather_rows(int64_t m, const int32_t* ids, int64_t row0, const int64_t* rowptr,
                const int32_t* col, const int64_t* out_off, int32_t* out, cudaStream_t st);
int gather_features(int64_t m, const int32_t* ids, int64_t row0, const float* H, int64_t f,
                    float* out, cudaStream_t st);
size_t ladies_counts_ws(int64_t k, int64_t n, int64_t q_cap);
size_t ladies_merge_ws(int64_t k, int64_t nloc);
int ladies_merge_counts(int64_t k, int64_t m, const int32_t* trip, int64_t v0, int64_t nloc,
                        int64_t* poff, int32_t* pv, int32_t* pe, void* d_ws, size_t ws_bytes,
                        cudaStream_t st);
int ladies_counts(int64_t k, const int64_t* qoff, const int32_t* qcol, const int32_t* qdeg,
                  int64_t q_cap, const int64_t* rowptr, const int32_t* col, int64_t n,
                  int64_t* poff, int32_t* pv, int32_t* pe, void* d_ws, size_t ws_bytes,
                  cudaStream_t st);
size_t ladies_race_topk_ws(int64_t k, int64_t p_cap, int32_t s);
int ladies_race_topk(int64_t k, const int64_t* poff, const int32_t* pv, const int32_t* pe,
                     int64_t p_cap, int32_t s, uint64_t seed, uint64_t epoch, uint64_t depth,
                     int64_t batch_offset, int64_t* take, int32_t* Sv, uint32_t* Sk, void* d_ws,
                     size_t ws_bytes, cudaStream_t st);
int ladies_extract_rows(int64_t k, const int64_t* qoff, const int32_t* qcol,
                        const int64_t* rowptr, const int32_t* col, const int64_t* fptr,
                        const int32_t* fcol, const int64_t* coloff, const int64_t* slot,
                        int32_t* slots, int32_t* rcnt, cudaStream_t st);
int ladies_workspace(const Graph* g, int64_t k, int64_t q1_cap, int32_t layers,
                     const int64_t* fanouts, int32_t mode, size_t* bytes);
// local row source for one LADIES layer: Q's rows as a CSR with global
// column ids, Q given as local row indices qrow[q]
struct LadiesRows {
  const int64_t* rowptr;
  const int32_t* col;
  const int32_t* qrow;
  int32_t depth;  // layer index of the keys (1-based)
};
int ladies_bulk(const Graph* g, int64_t k, const int64_t* d_qoff, const int32_t* d_qverts,
                int64_t q1_cap, int32_t layers, const int64_t* fanouts, uint64_t seed,
                uint64_t epoch, int64_t batch_offset, int32_t mode, gb_ladies_layer_out* L,
                int64_t* d_sizes, void* d_ws, size_t ws_bytes, cudaStream_t st,
                const LadiesRows* src = nullptr);

}  // namespace gb
