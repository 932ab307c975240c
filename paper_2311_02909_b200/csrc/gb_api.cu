#include <stdlib.h>
// extern "C" boundary of libgnnbulk_b200.so (include/gnnbulk_b200.h).
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include "gb_common.cuh"
#include "gb_internal.h"

namespace gb {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static thread_local int64_t g_launches = 0;
void count_launches(int n) { g_launches += n; }

struct Profile {
  cudaEvent_t ev[256];
  int created = 0, used = 0;
  bool on = false;
};
static thread_local Profile g_prof;

void prof_mark(cudaStream_t st) {
  if (!g_prof.on || g_prof.used >= g_prof.created) return;
  cudaEventRecord(g_prof.ev[g_prof.used++], st);
}

// Side streams for independent launches inside one step (fork / join by
// events, so it also works under CUDA graph capture), per device.
struct Fork {
  cudaStream_t s[kForkStreams];
  cudaEvent_t ev[kForkStreams + 2];
  cudaEvent_t ring[kEventRing];
  bool ready = false;
};
static Fork g_fork[16];

static Fork& fork_state() {
  int dev = 0;
  cudaGetDevice(&dev);
  Fork& f = g_fork[dev & 15];
  if (!f.ready) {
    for (int i = 0; i < kForkStreams; ++i)
      cudaStreamCreateWithFlags(&f.s[i], cudaStreamNonBlocking);
    for (int i = 0; i < kForkStreams + 2; ++i)
      cudaEventCreateWithFlags(&f.ev[i], cudaEventDisableTiming);
    for (int i = 0; i < kEventRing; ++i)
      cudaEventCreateWithFlags(&f.ring[i], cudaEventDisableTiming);
    f.ready = true;
  }
  return f;
}

void stream_wait(cudaStream_t waiter, cudaStream_t src) {
  Fork& f = fork_state();
  cudaEventRecord(f.ev[kForkStreams + 1], src);
  cudaStreamWaitEvent(waiter, f.ev[kForkStreams + 1], 0);
}

cudaEvent_t ring_event(int i) { return fork_state().ring[((i % kEventRing) + kEventRing) % kEventRing]; }

cudaStream_t fork_begin(cudaStream_t st, int n) {
  Fork& f = fork_state();
  cudaEventRecord(f.ev[kForkStreams], st);
  for (int i = 0; i < n && i < kForkStreams; ++i) cudaStreamWaitEvent(f.s[i], f.ev[kForkStreams], 0);
  return f.s[0];
}

cudaStream_t fork_stream(int i) { return fork_state().s[i]; }

void fork_join(cudaStream_t st, int n) {
  Fork& f = fork_state();
  for (int i = 0; i < n && i < kForkStreams; ++i) {
    cudaEventRecord(f.ev[i], f.s[i]);
    cudaStreamWaitEvent(st, f.ev[i], 0);
  }
}

bool sync_debug() {
  static int flag = -1;
  if (flag < 0) {
    const char* v = getenv("GB_SYNC_DEBUG");
    flag = (v && v[0] == '1') ? 1 : 0;
  }
  return flag == 1;
}

int cuda_status(cudaError_t e, const char* what) {
  set_error("CUDA error in %s: %s", what, cudaGetErrorString(e));
  return GB_ERR_CUDA;
}

__global__ void k_uniforms(uint64_t seed, uint64_t epoch, uint64_t depth,
                           const int64_t* __restrict__ rows, const int64_t* __restrict__ t,
                           int64_t count, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = uniform53(seed, epoch, depth, (uint64_t)rows[i], (uint64_t)t[i]);
}

}  // namespace gb

using namespace gb;

struct gb_graph : public gb::Graph {};

extern "C" {

const char* gb_last_error(void) { return g_err; }

int64_t gb_launch_counter(int32_t reset) {
  int64_t v = g_launches;
  if (reset) g_launches = 0;
  return v;
}

int gb_profile_begin(int32_t max_marks) {
  if (max_marks < 0 || max_marks > 256) { set_error("profile: 0..256 marks"); return GB_ERR_CONTRACT; }
  while (g_prof.created < max_marks) GB_CUDA(cudaEventCreate(&g_prof.ev[g_prof.created++]));
  g_prof.used = 0;
  g_prof.on = true;
  return GB_OK;
}

int gb_profile_end(float* h_ms, int32_t cap, int32_t* h_pairs) {
  g_prof.on = false;
  const int pairs = g_prof.used / 2;
  if (pairs > 0) GB_CUDA(cudaEventSynchronize(g_prof.ev[2 * pairs - 1]));
  for (int i = 0; i < pairs && i < cap; ++i)
    GB_CUDA(cudaEventElapsedTime(&h_ms[i], g_prof.ev[2 * i], g_prof.ev[2 * i + 1]));
  if (h_pairs) *h_pairs = pairs;
  g_prof.used = 0;
  return GB_OK;
}
int gb_version(void) { return 1; }

int gb_uniforms(uint64_t seed, uint64_t epoch, uint64_t depth, const int64_t* d_rows,
                const int64_t* d_t, int64_t count, double* d_out, void* stream) {
  if (count < 0) { set_error("count must be >= 0"); return GB_ERR_CONTRACT; }
  if (count == 0) return GB_OK;
  int64_t g = (count + 255) / 256;
  if (g > 16 * kNumSMs) g = 16 * kNumSMs;
  k_uniforms<<<(int)g, 256, 0, (cudaStream_t)stream>>>(seed, epoch, depth, d_rows, d_t, count,
                                                       d_out);
  GB_LAUNCH_CHECK("k_uniforms");
  return GB_OK;
}

int gb_graph_create(int64_t n, int64_t nnz, const int64_t* d_rowptr, const int32_t* d_col,
                    void* stream, gb_graph** out) {
  if (!out || n < 0 || nnz < 0 || n >= ((int64_t)1 << 31)) {
    set_error("graph: need 0 <= n < 2^31 and nnz >= 0");
    return GB_ERR_CONTRACT;
  }
  if (((uintptr_t)d_col & 15) != 0) {
    set_error("graph: column array must be 16-byte aligned");
    return GB_ERR_CONTRACT;
  }
  gb_graph* g = new gb_graph();
  g->n = n;
  g->nnz = nnz;
  g->rowptr = d_rowptr;
  g->col = d_col;
  int rc = graph_build_tables(g, (cudaStream_t)stream);
  if (rc) {
    gb_graph_destroy(g);
    return rc;
  }
  *out = g;
  return GB_OK;
}

int gb_graph_destroy(gb_graph* g) {
  if (!g) return GB_OK;
  cudaFree(g->deg_slot);
  cudaFree(g->slot_deg);
  cudaFree(g->run_j0);
  cudaFree(g->run_sd);
  cudaFree(g->run_n);
  cudaFree(g->run_lower);
  delete g;
  return GB_OK;
}

int gb_graph_info(const gb_graph* g, int64_t* h_max_deg, int64_t* h_table_slots) {
  if (!g) { set_error("null graph"); return GB_ERR_CONTRACT; }
  if (h_max_deg) *h_max_deg = g->max_deg;
  if (h_table_slots) *h_table_slots = g->slots;
  return GB_OK;
}

int gb_sage_bulk_workspace(const gb_graph* g, int64_t k, int64_t r1_cap, int32_t layers,
                           const int64_t* h_fanouts, size_t* h_bytes) {
  if (!g || !h_bytes || k < 0 || layers < 1) {
    set_error("sage workspace: bad arguments");
    return GB_ERR_CONTRACT;
  }
  return sage_workspace(g, k, r1_cap, layers, h_fanouts, h_bytes);
}

int gb_sage_bulk(const gb_graph* g, int64_t k, const int64_t* d_bptr, const int32_t* d_bverts,
                 int64_t r1_cap, int64_t batch_size, int32_t layers, const int64_t* h_fanouts,
                 uint64_t seed, uint64_t epoch, int64_t batch_offset, int32_t mode,
                 gb_sage_layer_out* h_layers, int64_t* d_sizes, void* d_ws, size_t ws_bytes,
                 void* stream) {
  if (!g || k < 0 || layers < 1 || batch_size < 1 || !h_fanouts || !h_layers) {
    set_error("sage bulk: bad arguments");
    return GB_ERR_CONTRACT;
  }
  for (int32_t l = 0; l < layers; ++l)
    if (h_fanouts[l] < 1) {
      set_error("sage bulk: fanout %lld < 1", (long long)h_fanouts[l]);
      return GB_ERR_CONTRACT;
    }
  if (mode != GB_SAGE_STREAM && mode != GB_SAGE_PFREE && mode != GB_SAGE_DEDUP) {
    set_error("sage bulk: unknown mode %d", mode);
    return GB_ERR_CONTRACT;
  }
  return sage_bulk(g, k, d_bptr, d_bverts, r1_cap, batch_size, layers, h_fanouts, seed, epoch,
                   batch_offset, mode, h_layers, d_sizes, d_ws, ws_bytes, (cudaStream_t)stream);
}

int gb_sage_bulk_peer(const gb_graph* g, int64_t k, const int64_t* d_bptr,
                      const int32_t* d_bverts, int64_t r1_cap, int64_t batch_size, int32_t layers,
                      const int64_t* h_fanouts, uint64_t seed, uint64_t epoch,
                      int64_t batch_offset, gb_sage_layer_out* h_layers, int64_t* d_sizes,
                      void* d_ws, size_t ws_bytes, int32_t nblk, const int64_t* d_bounds,
                      const int64_t* const* d_brp, const int32_t* const* d_bcol, void* stream) {
  if (nblk < 1 || !d_bounds || !d_brp || !d_bcol) {
    set_error("sage bulk peer: need the block table");
    return GB_ERR_CONTRACT;
  }
  if (!g || k < 0 || layers < 1 || batch_size < 1 || !h_fanouts || !h_layers) {
    set_error("sage bulk: bad arguments");
    return GB_ERR_CONTRACT;
  }
  for (int32_t l = 0; l < layers; ++l)
    if (h_fanouts[l] < 1 || h_fanouts[l] > 32) {
      set_error("sage bulk: fanout %lld outside [1, 32]", (long long)h_fanouts[l]);
      return h_fanouts[l] < 1 ? GB_ERR_CONTRACT : GB_ERR_UNSUPPORTED;
    }
  const PeerRowsHost peer{nblk, d_bounds, d_brp, d_bcol};
  return sage_bulk(g, k, d_bptr, d_bverts, r1_cap, batch_size, layers, h_fanouts, seed, epoch,
                   batch_offset, GB_SAGE_DEDUP, h_layers, d_sizes, d_ws, ws_bytes,
                   (cudaStream_t)stream, &peer);
}

size_t gb_sage_layer_sample_workspace(int64_t r_cap, int64_t f_cap) {
  return sage_layer_sample_ws(r_cap, f_cap);
}

int gb_sage_layer_sample(const gb_graph* tables, int64_t k, const int64_t* d_brow, int64_t r_cap,
                         const int32_t* d_rowv, const int32_t* d_deg, const int64_t* d_fptr,
                         const int64_t* d_rowptr, const int32_t* d_col, int32_t s, int64_t stride,
                         int64_t batch_offset, uint64_t seed, uint64_t epoch, uint64_t depth,
                         int32_t mode, int32_t* d_fcol, void* d_ws, size_t ws_bytes,
                         void* stream) {
  if (!tables || k < 0 || s < 1 || s > 32 || (mode != GB_SAGE_STREAM && mode != GB_SAGE_PFREE)) {
    set_error("sage layer sample: bad arguments");
    return GB_ERR_CONTRACT;
  }
  return sage_layer_sample(tables, k, d_brow, r_cap, d_rowv, d_deg, d_fptr, d_rowptr, d_col, s,
                           stride, batch_offset, seed, epoch, depth, mode, d_fcol, d_ws, ws_bytes,
                           (cudaStream_t)stream);
}

int gb_sage_sample_keyed(const gb_graph* tables, int64_t R, const int64_t* d_R,
                         const int32_t* d_rowv, const int32_t* d_deg, const int64_t* d_fptr,
                         const int64_t* d_rowkeys, const int64_t* d_rowptr, const int32_t* d_col,
                         int32_t s, uint64_t seed, uint64_t epoch, uint64_t depth,
                         int32_t* d_fcol, void* stream) {
  if (!tables || R < 0 || s < 1 || s > 32) {
    set_error("sage keyed sample: bad arguments");
    return GB_ERR_CONTRACT;
  }
  return sage_sample_keyed(tables, R, d_R, d_rowv, d_deg, d_fptr, d_rowkeys, d_rowptr, d_col, s,
                           seed, epoch, depth, d_fcol, (cudaStream_t)stream);
}

size_t gb_sage_layer_extract_workspace(int64_t n, int64_t k) { return sage_layer_extract_ws(n, k); }

int gb_sage_layer_extract(int64_t n, int64_t k, const int64_t* d_brow, const int64_t* d_fptr,
                          const int32_t* d_fcol, int64_t f_cap, int32_t* d_acol, int32_t* d_colv,
                          int64_t* d_eoff, int64_t* d_coloff, int64_t* d_sizes, void* d_ws,
                          size_t ws_bytes, void* stream) {
  if (n < 0 || k < 0) { set_error("sage extract: bad arguments"); return GB_ERR_CONTRACT; }
  return sage_layer_extract(n, k, d_brow, d_fptr, d_fcol, f_cap, d_acol, d_colv, d_eoff, d_coloff,
                            d_sizes, d_ws, ws_bytes, (cudaStream_t)stream);
}

int gb_take_scan(int64_t r_cap, const int64_t* d_R, const int32_t* d_deg, int32_t s,
                 int64_t* d_fptr, int64_t* d_scan_ws, void* stream) {
  return take_scan(r_cap, d_R, d_deg, s, d_fptr, d_scan_ws, (cudaStream_t)stream);
}

int gb_gather_rows(int64_t m, const int32_t* d_ids, int64_t row0, const int64_t* d_rowptr,
                   const int32_t* d_col, const int64_t* d_out_off, int32_t* d_out, void* stream) {
  return gather_rows(m, d_ids, row0, d_rowptr, d_col, d_out_off, d_out, (cudaStream_t)stream);
}

int gb_gather_features(int64_t m, const int32_t* d_ids, int64_t row0, const float* d_H, int64_t f,
                       float* d_out, void* stream) {
  return gather_features(m, d_ids, row0, d_H, f, d_out, (cudaStream_t)stream);
}

int gb_spmm_rows(int64_t R, const int64_t* d_rowptr, const int32_t* d_col,
                 const int64_t* d_row_batch, const int64_t* d_shift, int64_t k, const float* d_X,
                 int64_t f, float* d_Y, void* stream) {
  if (R < 0 || f < 0 || k < 0 || (d_shift && !d_row_batch)) {
    set_error("spmm_rows: bad arguments");
    return GB_ERR_CONTRACT;
  }
  return spmm_rows(R, d_rowptr, d_col, d_row_batch, d_shift, k, d_X, f, d_Y, (cudaStream_t)stream);
}

int gb_spmm_f64(int64_t R, const int64_t* d_rowptr, const int32_t* d_col, const double* d_val,
                const double* d_X, int64_t f, double* d_Y, void* stream) {
  if (R < 0 || f < 0 || (R > 0 && (!d_rowptr || !d_Y))) {
    set_error("spmm_f64: bad arguments");
    return GB_ERR_CONTRACT;
  }
  return spmm_f64(R, d_rowptr, d_col, d_val, d_X, f, d_Y, (cudaStream_t)stream);
}

size_t gb_sage_owner_p2p_workspace(int64_t r_cap) { return sage_owner_p2p_ws(r_cap); }

int gb_sage_owner_p2p(const gb_graph* tables, int64_t ngroups, const int32_t* const* h_rows,
                      const int64_t* const* h_brow, const int64_t* const* h_fptr,
                      const int64_t* h_boff, int64_t k, int64_t r_cap, int32_t ndst,
                      int32_t* const* h_dst, int64_t lo, int64_t hi, const int64_t* d_brp,
                      const int32_t* d_bcol, int32_t s, int64_t stride, uint64_t seed,
                      uint64_t epoch, uint64_t depth, void* d_ws, size_t ws_bytes, void* stream) {
  if (!tables || ngroups < 0 || k < 1 || r_cap < 0 || lo < 0 || hi < lo || s < 1 || s > 32 ||
      (ngroups && (!h_rows || !h_brow || !h_fptr || !h_boff || !h_dst))) {
    set_error("owner p2p: bad arguments");
    return GB_ERR_CONTRACT;
  }
  return sage_owner_p2p(tables, ngroups, h_rows, h_brow, h_fptr, h_boff, k, r_cap, ndst, h_dst, lo,
                        hi, d_brp, d_bcol, s, stride, seed, epoch, depth, d_ws, ws_bytes,
                        (cudaStream_t)stream);
}

int gb_segment_copy(int64_t m, const int64_t* d_rows, const int64_t* d_src_off,
                    const int32_t* d_lens, const int32_t* d_src, const int64_t* d_dst_off,
                    int32_t* d_dst, void* stream) {
  if (m < 0 || (m > 0 && (!d_src_off || !d_src || !d_dst_off || !d_dst))) {
    set_error("segment_copy: bad arguments");
    return GB_ERR_CONTRACT;
  }
  return segment_copy(m, d_rows, d_src_off, d_lens, d_src, d_dst_off, d_dst, (cudaStream_t)stream);
}

int gb_first_occurrence(int64_t F, const int32_t* d_colidx, const int64_t* d_entry_batch,
                        const int64_t* d_shift, int64_t k, int64_t ncols, int32_t* d_first,
                        void* stream) {
  if (F < 0 || ncols < 0 || F >= ((int64_t)1 << 31) || (d_shift && !d_entry_batch)) {
    set_error("first_occurrence: bad arguments");
    return GB_ERR_CONTRACT;
  }
  return first_occurrence(F, d_colidx, d_entry_batch, d_shift, k, ncols, d_first,
                          (cudaStream_t)stream);
}

size_t gb_ladies_counts_workspace(int64_t k, int64_t n, int64_t q_cap) {
  return ladies_counts_ws(k, n, q_cap);
}

int gb_ladies_counts(int64_t k, const int64_t* d_qoff, const int32_t* d_qcol, const int32_t* d_qdeg,
                     int64_t q_cap, const int64_t* d_rowptr, const int32_t* d_col, int64_t n,
                     int64_t* d_poff, int32_t* d_pv, int32_t* d_pe, void* d_ws, size_t ws_bytes,
                     void* stream) {
  if (k < 0 || n < 0) { set_error("ladies counts: bad arguments"); return GB_ERR_CONTRACT; }
  return ladies_counts(k, d_qoff, d_qcol, d_qdeg, q_cap, d_rowptr, d_col, n, d_poff, d_pv, d_pe,
                       d_ws, ws_bytes, (cudaStream_t)stream);
}

size_t gb_ladies_merge_counts_workspace(int64_t k, int64_t nloc) {
  return ladies_merge_ws(k, nloc);
}

int gb_ladies_merge_counts(int64_t k, int64_t m, const int32_t* d_trip, int64_t v0, int64_t nloc,
                           int64_t* d_poff, int32_t* d_pv, int32_t* d_pe, void* d_ws,
                           size_t ws_bytes, void* stream) {
  if (k < 0 || m < 0 || v0 < 0 || nloc < 0) {
    set_error("ladies merge: bad arguments");
    return GB_ERR_CONTRACT;
  }
  return ladies_merge_counts(k, m, d_trip, v0, nloc, d_poff, d_pv, d_pe, d_ws, ws_bytes,
                             (cudaStream_t)stream);
}

size_t gb_ladies_race_topk_workspace(int64_t k, int64_t p_cap, int32_t s) {
  return ladies_race_topk_ws(k, p_cap, s);
}

int gb_ladies_race_topk(int64_t k, const int64_t* d_poff, const int32_t* d_pv, const int32_t* d_pe,
                        int64_t p_cap, int32_t s, uint64_t seed, uint64_t epoch, uint64_t depth,
                        int64_t batch_offset, int64_t* d_take, int32_t* d_Sv, uint32_t* d_Sk,
                        void* d_ws, size_t ws_bytes, void* stream) {
  if (k < 0 || s < 1) { set_error("ladies race: bad arguments"); return GB_ERR_CONTRACT; }
  return ladies_race_topk(k, d_poff, d_pv, d_pe, p_cap, s, seed, epoch, depth, batch_offset,
                          d_take, d_Sv, d_Sk, d_ws, ws_bytes, (cudaStream_t)stream);
}

int gb_ladies_extract_rows(int64_t k, const int64_t* d_qoff, const int32_t* d_qcol,
                           const int64_t* d_rowptr, const int32_t* d_col, const int64_t* d_fptr,
                           const int32_t* d_fcol, const int64_t* d_coloff, const int64_t* d_slot,
                           int32_t* d_slots, int32_t* d_rcnt, void* stream) {
  return ladies_extract_rows(k, d_qoff, d_qcol, d_rowptr, d_col, d_fptr, d_fcol, d_coloff, d_slot,
                             d_slots, d_rcnt, (cudaStream_t)stream);
}

int gb_ladies_bulk_workspace(const gb_graph* g, int64_t k, int64_t q1_cap, int32_t layers,
                             const int64_t* h_fanouts, int32_t mode, size_t* h_bytes) {
  if (!g || !h_bytes || k < 0 || layers < 1 || !h_fanouts) {
    set_error("ladies workspace: bad arguments");
    return GB_ERR_CONTRACT;
  }
  return ladies_workspace(g, k, q1_cap, layers, h_fanouts, mode, h_bytes);
}

int gb_ladies_bulk(const gb_graph* g, int64_t k, const int64_t* d_qoff, const int32_t* d_qverts,
                   int64_t q1_cap, int32_t layers, const int64_t* h_fanouts, uint64_t seed,
                   uint64_t epoch, int64_t batch_offset, int32_t mode,
                   gb_ladies_layer_out* h_layers, int64_t* d_sizes, void* d_ws, size_t ws_bytes,
                   void* stream) {
  if (!g || k < 0 || layers < 1 || !h_fanouts || !h_layers) {
    set_error("ladies bulk: bad arguments");
    return GB_ERR_CONTRACT;
  }
  for (int32_t l = 0; l < layers; ++l)
    if (h_fanouts[l] < 1) {
      set_error("ladies bulk: sample count must be >= 1");
      return GB_ERR_CONTRACT;
    }
  if (mode != GB_LADIES_EXACT && mode != GB_LADIES_RACE && mode != GB_LADIES_RACE_DENSE) {
    set_error("ladies bulk: unknown mode %d", mode);
    return GB_ERR_CONTRACT;
  }
  return ladies_bulk(g, k, d_qoff, d_qverts, q1_cap, layers, h_fanouts, seed, epoch,
                     batch_offset, mode, h_layers, d_sizes, d_ws, ws_bytes, (cudaStream_t)stream);
}

int gb_ladies_layer_rows(const gb_graph* g, int64_t k, const int64_t* d_qoff,
                         const int32_t* d_qrow, int64_t q_cap, const int64_t* d_lrowptr,
                         const int32_t* d_lcol, int64_t s, uint64_t seed, uint64_t epoch,
                         int32_t depth, int64_t batch_offset, int32_t mode,
                         gb_ladies_layer_out* h_layer, int64_t* d_sizes, void* d_ws,
                         size_t ws_bytes, void* stream) {
  if (!g || k < 0 || s < 1 || depth < 1 || !h_layer || !d_lrowptr || !d_lcol || !d_qrow) {
    set_error("ladies layer rows: bad arguments");
    return GB_ERR_CONTRACT;
  }
  if (mode != GB_LADIES_RACE && mode != GB_LADIES_RACE_DENSE) {
    set_error("ladies layer rows: race modes only");
    return GB_ERR_CONTRACT;
  }
  const LadiesRows src{d_lrowptr, d_lcol, d_qrow, depth};
  return ladies_bulk(g, k, d_qoff, nullptr, q_cap, 1, &s, seed, epoch, batch_offset, mode,
                     h_layer, d_sizes, d_ws, ws_bytes, (cudaStream_t)stream, &src);
}

}  // extern "C"
