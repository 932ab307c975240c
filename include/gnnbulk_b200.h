/*
 * gnnbulk_b200 — C ABI of the B200-native matrix-based bulk GNN sampler
 * (arXiv 2311.02909).  The reference (`gnnbulk`, pure Python + numpy/scipy)
 * has no FFI of its own; these are the entry points a ctypes/cffi binding of
 * its hot path binds.  Each entry point cites the
 * reference function it replaces.
 *
 * Conventions
 *   - Plain C types only; every array argument prefixed d_ is DEVICE memory,
 *     h_ is host memory.  `stream` is a cudaStream_t passed as void*.
 *   - Calls are stream-ordered and do not synchronise the host unless the
 *     comment says so (graph creation, size queries).
 *   - Return 0 (GB_OK) or a negative status; gb_last_error() describes the
 *     last failure of the calling thread.  GB_ERR_CONTRACT is what the
 *     Python shim maps to reference `ContractViolation`
 *     (pkg/src/gnnbulk/errors.py:4-11).
 *   - Vertex ids are int32 (n < 2^31), row offsets int64, keys int64.
 *   - The caller owns every buffer; sizes are obtained with the *_workspace
 *     queries.  Column arrays of a graph must be 16-byte aligned and readable
 *     for nnz + GB_COL_PAD entries (streaming loads are 16 B wide).
 */
#ifndef GNNBULK_B200_H
#define GNNBULK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GB_OK 0
#define GB_ERR_CONTRACT (-1)
#define GB_ERR_CUDA (-2)
#define GB_ERR_CAPACITY (-3)
#define GB_ERR_UNSUPPORTED (-4)

#define GB_COL_PAD 4

/* SAGE sample-kernel modes (identical outputs) */
#define GB_SAGE_STREAM 0 /* Alg. 1: P row formed on chip by streaming A rows */
#define GB_SAGE_PFREE 1  /* P-free fast path: read only the picked entries  */
#define GB_SAGE_DEDUP 2  /* Alg. 1 with duplicate-row elimination: every
                            distinct P row formed on chip once, serving the
                            picks of all frontier rows that reference it */

const char* gb_last_error(void);
int gb_version(void);

/* ------------------------------------------------------------------ RNG
 * u(seed, epoch, depth, row, t) for count (row, t) pairs — the injected
 * replacement of RowRng.stream(global_row).random() (sampler.py:97-116);
 * the t-th call of row `row`.  Known-answer tested against numpy Philox. */
int gb_uniforms(uint64_t seed, uint64_t epoch, uint64_t depth, const int64_t* d_rows,
                const int64_t* d_t, int64_t count, double* d_out, void* stream);

/* ---------------------------------------------------------------- graph
 * Graph (sparse.py:194-227) on the device: CSR rows = out-neighbours,
 * values implicitly 1.0.  Creation builds the per-degree exact-replay
 * tables of the SAGE sampler (synchronises `stream`). */
typedef struct gb_graph gb_graph;
int gb_graph_create(int64_t n, int64_t nnz, const int64_t* d_rowptr, const int32_t* d_col,
                    void* stream, gb_graph** out);
int gb_graph_destroy(gb_graph* g);
int gb_graph_info(const gb_graph* g, int64_t* h_max_deg, int64_t* h_table_slots);

/* ---------------------------------------------------------- SAGE bulk
 * sample_epoch_bulk with SamplerConfig.kind == SAGE (sampler.py:325-387):
 * all L layers for k stacked minibatches, entirely on the device.
 *
 * Per layer l the caller provides buffers with capacity r_cap rows and
 * f_cap = r_cap * fanouts[l] entries, r_cap(1) >= total batch vertices,
 * r_cap(l+1) = f_cap(l).  Outputs (device):
 *   fptr  [R+1]  frontier row offsets == adjacency row offsets
 *   fcol  [F]    frontier columns (sorted per row) == sampled_vertices, and
 *                the next layer's row vertices (expand_row_extraction)
 *   acol  [F]    block-diagonal adjacency columns (block_diag of
 *                compact_columns per batch, sparse.py:321-357)
 *   colv  [U]    col_vertices, per batch sorted unique, concatenated
 *   eoff  [k+1]  per-batch offsets into fcol (sampled_vertices) == next
 *                layer's batch row offsets
 *   coloff[k+1]  per-batch offsets into colv
 * d_sizes[3*l + {0,1,2}] = (R, F, U) of layer l.  Layer 1 rows are the batch
 * vertices d_bverts with batch offsets d_bptr (sage_seed_matrix). */
typedef struct {
  int64_t* fptr;
  int32_t* fcol;
  int32_t* acol;
  int32_t* colv;
  int64_t* eoff;
  int64_t* coloff;
  int64_t r_cap;
  int64_t f_cap;
} gb_sage_layer_out;

/* Workspace contract: d_ws is zero-filled before its first bulk and not
 * modified by the caller between bulks — a completed bulk leaves its bit
 * maps and vertex counters clear (and marks the workspace so), so the next
 * bulk on it skips clearing them.  A workspace the caller reused for other
 * data must be zero-filled again. */
int gb_sage_bulk_workspace(const gb_graph* g, int64_t k, int64_t r1_cap, int32_t layers,
                           const int64_t* h_fanouts, size_t* h_bytes);
int gb_sage_bulk(const gb_graph* g, int64_t k, const int64_t* d_bptr, const int32_t* d_bverts,
                 int64_t r1_cap, int64_t batch_size, int32_t layers, const int64_t* h_fanouts,
                 uint64_t seed, uint64_t epoch, int64_t batch_offset, int32_t mode,
                 gb_sage_layer_out* h_layers, int64_t* d_sizes, void* d_ws, size_t ws_bytes,
                 void* stream);

/* ------------------------------------- SAGE per-layer pieces (1.5D mode)
 * The distributed executor (one process per GPU) composes a layer from:
 *   gb_take_scan            fptr = exclusive scan of min(deg[r], s), r < *d_R
 *   gb_sage_layer_sample    NORM + SAMPLE of the rows with d_deg[r] > 0
 *                           through the CSR (d_rowptr, d_col) addressed by
 *                           d_rowv[r] (a local block of fetched A rows);
 *                           picks land at d_fptr[r] in d_fcol; replay
 *                           tables of `tables` (built on the global degrees)
 *   gb_sage_layer_extract   EXTRACT of the completed frontier (after the
 *                           grid-row exchange): acol, colv, eoff, coloff,
 *                           sizes (R, F, U) — sage_batch_blocks/block_diag
 *   gb_gather_rows          sparsity-aware row reply: rows ids[i] - row0 of a
 *                           CSR block packed at out_off[i] (rows_subset,
 *                           sparse.py:391-414 / dist.py:357-361)
 *   gb_gather_features      fp32 feature rows for the all-to-allv of
 *                           fetch_features (pipeline.py:78-120) */
int gb_take_scan(int64_t r_cap, const int64_t* d_R, const int32_t* d_deg, int32_t s,
                 int64_t* d_fptr, int64_t* d_scan_ws, void* stream);
size_t gb_sage_layer_sample_workspace(int64_t r_cap, int64_t f_cap);
int gb_sage_layer_sample(const gb_graph* tables, int64_t k, const int64_t* d_brow, int64_t r_cap,
                         const int32_t* d_rowv, const int32_t* d_deg, const int64_t* d_fptr,
                         const int64_t* d_rowptr, const int32_t* d_col, int32_t s, int64_t stride,
                         int64_t batch_offset, uint64_t seed, uint64_t epoch, uint64_t depth,
                         int32_t mode, int32_t* d_fcol, void* d_ws, size_t ws_bytes,
                         void* stream);
/* owner-computes variant: the block owner samples requested rows (local row
 * d_rowv[r], degree, explicit global row key d_rowkeys[r]) and writes the
 * sorted picks at d_fptr[r] — only s ids per row cross NVLink */
int gb_sage_sample_keyed(const gb_graph* tables, int64_t R, const int64_t* d_R,
                         const int32_t* d_rowv, const int32_t* d_deg, const int64_t* d_fptr,
                         const int64_t* d_rowkeys, const int64_t* d_rowptr, const int32_t* d_col,
                         int32_t s, uint64_t seed, uint64_t epoch, uint64_t depth,
                         int32_t* d_fcol, void* stream);
size_t gb_sage_layer_extract_workspace(int64_t n, int64_t k);
int gb_sage_layer_extract(int64_t n, int64_t k, const int64_t* d_brow, const int64_t* d_fptr,
                          const int32_t* d_fcol, int64_t f_cap, int32_t* d_acol, int32_t* d_colv,
                          int64_t* d_eoff, int64_t* d_coloff, int64_t* d_sizes, void* d_ws,
                          size_t ws_bytes, void* stream);
int gb_gather_rows(int64_t m, const int32_t* d_ids, int64_t row0, const int64_t* d_rowptr,
                   const int32_t* d_col, const int64_t* d_out_off, int32_t* d_out, void* stream);
int gb_gather_features(int64_t m, const int32_t* d_ids, int64_t row0, const float* d_H, int64_t f,
                       float* d_out, void* stream);

/* ------------------------------------------ epoch pipeline aggregation
 * Replaces forward_aggregate (pipeline.py:123-130) and the layer-to-layer
 * carry of _propagate_batch (pipeline.py:280-305) for a whole bulk.
 *   gb_spmm_rows        Y[r, :] = sum_e X[col[e] + shift[b(r)], :] over the
 *                       stacked sampled adjacency (values 1.0), fp32; b(r)
 *                       from d_row_batch[k+1] (rows of batch b); d_shift may
 *                       be NULL (block-diagonal columns address X directly)
 *   gb_first_occurrence first[j] = smallest entry e with column index j
 *                       (col[e] + shift[b(e)], batch offsets d_entry_batch),
 *                       or e itself when d_colidx is NULL; unset = INT32_MAX */
/* gb_spmm_f64 — forward_aggregate (pipeline.py:123-130): Y = A X in float64
 * with A's values (any, not only 0/1), the reference's scipy csr_matvecs
 * order (per row, entries in order, product then sum): bit-identical. */
int gb_spmm_f64(int64_t R, const int64_t* d_rowptr, const int32_t* d_col, const double* d_val,
                const double* d_X, int64_t f, double* d_Y, void* stream);
int gb_spmm_rows(int64_t R, const int64_t* d_rowptr, const int32_t* d_col,
                 const int64_t* d_row_batch, const int64_t* d_shift, int64_t k, const float* d_X,
                 int64_t f, float* d_Y, void* stream);
int gb_first_occurrence(int64_t F, const int32_t* d_colidx, const int64_t* d_entry_batch,
                        const int64_t* d_shift, int64_t k, int64_t ncols, int32_t* d_first,
                        void* stream);
/* Segmented copy of the distributed executor (placing picks returned by the
 * block owner into the frontier, dist.py:357-361 reply handling; packing
 * slot-layout A_S rows, dist.py:523-541):
 * d_dst[d_dst_off[row_i] + t] = d_src[d_src_off[i] + t], t < len_i, with
 * row_i = d_rows[i] (identity if NULL), len_i = d_lens[i] (or
 * d_src_off[i+1] - d_src_off[i] if NULL). */
int gb_segment_copy(int64_t m, const int64_t* d_rows, const int64_t* d_src_off,
                    const int32_t* d_lens, const int32_t* d_src, const int64_t* d_dst_off,
                    int32_t* d_dst, void* stream);

/* -------------------------------------------------------- LADIES bulk
 * sample_epoch_bulk with SamplerConfig.kind == LADIES (sampler.py:325-387,
 * 420-462, 475-483).  Layer-1 rows: the batches, each sorted and distinct
 * (ladies_seed_matrix), offsets d_qoff[k+1], vertices d_qverts.
 * Per layer (caller buffers; q_cap >= rows of Q, f_cap >= k*s,
 * a_cap >= q_cap*s):
 *   fptr  [k+1]   frontier row offsets; fcol [F] sorted sampled vertices
 *                 (== col_vertices == sampled_vertices == next layer's Q)
 *   aptr  [Q+1], acol [nnz]  A_S (one row per Q nonzero, ladies_assemble)
 *   coloff[k+1]   column offset of each batch's block (all 0 = shared layout)
 * d_sizes[5*l + {0,1,2,3,4}] = (A_S rows, F, A_S nnz, A_S cols, nnz(P)); a
 * negative last entry reports a capacity overflow inside the bulk (-1: race
 * tie list of more than 2048 equal keys).
 * mode GB_LADIES_EXACT replays its_sample_row bit for bit (sequential fp64
 * cumsum, small graphs); GB_LADIES_RACE draws the same law by an
 * exponential race (Gumbel top-s) for production sizes, counting P by
 * column tiles in shared memory; GB_LADIES_RACE_DENSE is the same race over
 * dense per-batch counters (identical output; kept as a cross-check). */
#define GB_LADIES_EXACT 0
#define GB_LADIES_RACE 1
#define GB_LADIES_RACE_DENSE 2

typedef struct {
  int64_t* fptr;
  int32_t* fcol;
  int64_t* aptr;
  int32_t* acol;
  int64_t* coloff;
  int64_t q_cap;
  int64_t f_cap;
  int64_t a_cap;
} gb_ladies_layer_out;

int gb_ladies_bulk_workspace(const gb_graph* g, int64_t k, int64_t q1_cap, int32_t layers,
                             const int64_t* h_fanouts, int32_t mode, size_t* h_bytes);
int gb_ladies_bulk(const gb_graph* g, int64_t k, const int64_t* d_qoff, const int32_t* d_qverts,
                   int64_t q1_cap, int32_t layers, const int64_t* h_fanouts, uint64_t seed,
                   uint64_t epoch, int64_t batch_offset, int32_t mode,
                   gb_ladies_layer_out* h_layers, int64_t* d_sizes, void* d_ws, size_t ws_bytes,
                   void* stream);

/* ------------------------------------------------- generic operators
 * Device CSR (int64 row offsets, int32 columns, f64 values) operators of
 * the reference API.  d_m points to the row count on the device (so the
 * calls can follow device-sized producers); d_scan_ws has
 * gb_scan_workspace_bytes(m) bytes.
 *   gb_spgemm_bound  d_ub[m+1] = exclusive prefix of per-row product bounds
 *   gb_spgemm        C = A B (spgemm, sparse.py:233-251): scipy csr_matmat
 *                    accumulation order, drop |x| < 1e-12; scratch: gkey /
 *                    gval 4*ub_total, tmp 1*ub_total, cnt m+1; C capacity
 *                    ub_total, nnz = d_c_ptr[m]
 *   gb_csr_add       C = A + B (add, sparse.py:417-427); phase 0 counts and
 *                    scans d_c_ptr, phase 1 writes
 *   gb_norm_rows     norm_rows_sage (square=0) / norm_rows_ladies (1)
 *                    (sparse.py:254-286), numpy add.reduce order; *d_err = 1
 *                    negative value, 2 zero-mass row
 *   gb_its_rows      its_sample_row for every row (sampler.py:157-207):
 *                    picks[r*s + t] in draw order, keyed uniforms or
 *                    d_inject[r*s + t]; *d_err = 1 non-positive weight */
size_t gb_scan_workspace_bytes(int64_t max_n);
int gb_spgemm_bound(int64_t m, const int64_t* d_a_ptr, const int32_t* d_a_col,
                    const int64_t* d_b_ptr, const int64_t* d_m, int64_t* d_ub, int64_t* d_scan_ws,
                    void* stream);
int gb_spgemm(int64_t m, const int64_t* d_m, const int64_t* d_a_ptr, const int32_t* d_a_col,
              const double* d_a_val, const int64_t* d_b_ptr, const int32_t* d_b_col,
              const double* d_b_val, const int64_t* d_ub, int64_t ub_total, int32_t* d_gkey,
              double* d_gval, int32_t* d_tmp_col, double* d_tmp_val, int64_t* d_cnt,
              int64_t* d_c_ptr, int32_t* d_c_col, double* d_c_val, int64_t* d_scan_ws,
              void* stream);
int gb_csr_add(int64_t m, const int64_t* d_m, const int64_t* d_a_ptr, const int32_t* d_a_col,
               const double* d_a_val, const int64_t* d_b_ptr, const int32_t* d_b_col,
               const double* d_b_val, int64_t* d_cnt, int64_t* d_c_ptr, int32_t* d_c_col,
               double* d_c_val, int64_t* d_scan_ws, int32_t phase, void* stream);
int gb_norm_rows(int64_t m, const int64_t* d_ptr, const double* d_val, int32_t square,
                 double* d_out, int32_t* d_err, void* stream);
int gb_its_rows(int64_t m, const int64_t* d_ptr, const double* d_val, int32_t s,
                const int64_t* d_keys, const double* d_inject, uint64_t seed, uint64_t epoch,
                uint64_t depth, double* d_w, double* d_cdf, int32_t* d_picks, int32_t* d_take,
                int32_t* d_err, void* stream);

/* Owner sampling over peer memory (1.5D SAGE, fused exchange): for each of
 * ngroups requesting grid rows g, read its frontier rows h_rows[g] (R =
 * h_brow[g][k]), batch offsets h_brow[g] (k+1) and frontier offsets
 * h_fptr[g] directly from that rank's memory (P2P), keep the rows whose
 * vertex is in [lo, hi) (this rank's block, CSR d_brp / d_bcol over the
 * block's rows), sample them with keys (h_boff[g] + batch) * stride + row,
 * and store the picks into h_dst[g * ndst + m] + fptr (the frontiers of the
 * grid row's ndst replicas, P2P).  Replaces the request / reply messages of
 * the owner-computes variant and the grid-row all-reduce (dist.py:349-378,
 * 469-484).  Host arrays of device pointers; caller brackets the call with
 * device barriers over the participating ranks. */
size_t gb_sage_owner_p2p_workspace(int64_t r_cap);
int gb_sage_owner_p2p(const gb_graph* tables, int64_t ngroups, const int32_t* const* h_rows,
                      const int64_t* const* h_brow, const int64_t* const* h_fptr,
                      const int64_t* h_boff, int64_t k, int64_t r_cap, int32_t ndst,
                      int32_t* const* h_dst, int64_t lo, int64_t hi, const int64_t* d_brp,
                      const int32_t* d_bcol, int32_t s, int64_t stride, uint64_t seed,
                      uint64_t epoch, uint64_t depth, void* d_ws, size_t ws_bytes, void* stream);

/* ------------------------------------ LADIES per-layer pieces (1.5D mode)
 *   gb_ladies_counts       partial P = Q A over the rows with d_qdeg[q] > 0
 *                          through a local CSR addressed by d_qcol[q]: per
 *                          batch the sorted (v, e) nonzeros at d_poff[i]
 *   gb_ladies_merge_counts sum of partial (batch, v, e) int32 triples d_trip
 *                          [3m] for v in [v0, v0 + nloc) (the sparse merge of
 *                          the grid row): per batch the sorted (v, e) at d_poff
 *   gb_ladies_race_topk    exponential-race top-s of every batch's (v, e)
 *                          list: d_take[i], sorted vertices d_Sv[i*s ...] and
 *                          their race keys d_Sk (for the grid-row merge)
 *   gb_ladies_extract_rows A_S rows of Q (ranks of A[u,:] ∩ S_i) into the
 *                          upper-bound slot layout d_slot / d_slots, counts
 *                          d_rcnt (ladies_assemble, sampler.py:420-434) */
size_t gb_ladies_counts_workspace(int64_t k, int64_t n, int64_t q_cap);
int gb_ladies_counts(int64_t k, const int64_t* d_qoff, const int32_t* d_qcol, const int32_t* d_qdeg,
                     int64_t q_cap, const int64_t* d_rowptr, const int32_t* d_col, int64_t n,
                     int64_t* d_poff, int32_t* d_pv, int32_t* d_pe, void* d_ws, size_t ws_bytes,
                     void* stream);
/* gb_sage_bulk (dedup mode) over rows held in other GPUs' memory (1.5D
 * batch split): the graph g supplies degrees and replay tables; the A rows of
 * block b (vertices [d_bounds[b], d_bounds[b+1])) are read from CSR
 * d_brp[b] / d_bcol[b] (device arrays of peer pointers, e.g. symmetric
 * memory) — the distinct rows are staged straight from the owners' memory
 * by the serve kernels (P2P cp.async over NVLink).  Same outputs as
 * gb_sage_bulk. */
int gb_sage_bulk_peer(const gb_graph* g, int64_t k, const int64_t* d_bptr,
                      const int32_t* d_bverts, int64_t r1_cap, int64_t batch_size, int32_t layers,
                      const int64_t* h_fanouts, uint64_t seed, uint64_t epoch,
                      int64_t batch_offset, gb_sage_layer_out* h_layers, int64_t* d_sizes,
                      void* d_ws, size_t ws_bytes, int32_t nblk, const int64_t* d_bounds,
                      const int64_t* const* d_brp, const int32_t* const* d_bcol, void* stream);

/* One LADIES race layer over a local row source (1.5D batch slices): Q's
 * rows as a CSR d_lrowptr / d_lcol (global column ids, e.g. gathered from
 * the block owners' memory), Q given as local row indices d_qrow under the
 * batch offsets d_qoff; keys use layer index `depth`.  Output and workspace
 * as gb_ladies_bulk with layers = 1 (gb_ladies_bulk_workspace(g, k, q_cap,
 * 1, &s, mode)); the graph g supplies the column count and degree prefix. */
int gb_ladies_layer_rows(const gb_graph* g, int64_t k, const int64_t* d_qoff,
                         const int32_t* d_qrow, int64_t q_cap, const int64_t* d_lrowptr,
                         const int32_t* d_lcol, int64_t s, uint64_t seed, uint64_t epoch,
                         int32_t depth, int64_t batch_offset, int32_t mode,
                         gb_ladies_layer_out* h_layer, int64_t* d_sizes, void* d_ws,
                         size_t ws_bytes, void* stream);
size_t gb_ladies_merge_counts_workspace(int64_t k, int64_t nloc);
int gb_ladies_merge_counts(int64_t k, int64_t m, const int32_t* d_trip, int64_t v0, int64_t nloc,
                           int64_t* d_poff, int32_t* d_pv, int32_t* d_pe, void* d_ws,
                           size_t ws_bytes, void* stream);
size_t gb_ladies_race_topk_workspace(int64_t k, int64_t p_cap, int32_t s);
int gb_ladies_race_topk(int64_t k, const int64_t* d_poff, const int32_t* d_pv, const int32_t* d_pe,
                        int64_t p_cap, int32_t s, uint64_t seed, uint64_t epoch, uint64_t depth,
                        int64_t batch_offset, int64_t* d_take, int32_t* d_Sv, uint32_t* d_Sk,
                        void* d_ws, size_t ws_bytes, void* stream);
int gb_ladies_extract_rows(int64_t k, const int64_t* d_qoff, const int32_t* d_qcol,
                           const int64_t* d_rowptr, const int32_t* d_col, const int64_t* d_fptr,
                           const int32_t* d_fcol, const int64_t* d_coloff, const int64_t* d_slot,
                           int32_t* d_slots, int32_t* d_rcnt, void* stream);

/* ----------------------------------------------------- synthetic inputs
 * R-MAT edge candidates first..first+count (Graph500 quadrant recursion over
 * `scale` levels with probabilities a, b, c; rejected candidates = -1) and
 * a keyed 64-bit hash for relabelling; the device side of the canonical
 * generator (graph_io.py:79-197 is the reference's
 * host-only ingestion). */
int gb_rmat_edges(uint64_t seed, int32_t scale, int64_t n, int64_t first, int64_t count,
                  double a, double b, double c, int64_t* d_src, int64_t* d_dst, void* stream);
int gb_hash64(uint64_t seed, const int64_t* d_x, int64_t count, int64_t* d_out, void* stream);

/* ---------------------------------------------------------- ingestion
 * gb_csr_from_edges — Graph.from_edges (sparse.py:211-216) =
 * SparseMatrix.from_coo(n, n, src, dst, ones, dedup="first")
 * (sparse.py:82-103) on the device: COO (int64 ids) -> canonical CSR
 * (rowptr int64[n+1], col int32, sorted and distinct per row), by a stable
 * LSD radix sort of the packed (src, dst) keys.  d_col needs m + GB_COL_PAD
 * entries; the padding is zeroed.  Ids outside [0, n) -> GB_ERR_CONTRACT
 * ("row/column index out of range", sparse.py:93-96).  Synchronises
 * `stream` (returns the distinct edge count in *h_nnz). */
size_t gb_csr_from_edges_workspace(int64_t n, int64_t m);
int gb_csr_from_edges(int64_t n, int64_t m, const int64_t* d_src, const int64_t* d_dst,
                      int64_t* d_rowptr, int32_t* d_col, int64_t* h_nnz, void* d_ws,
                      size_t ws_bytes, void* stream);

/* gb_rmat_graph — the synthetic OGB-shaped graphs of SURVEY.md §8(d) (the
 * canonical recipe of Appendix B with counter-based draws): `candidates`
 * R-MAT draws (Philox keyed by the draw index; ids >= n and self loops
 * rejected; (min, max) pairs when symmetric), the first m distinct pairs in
 * draw order, vertices relabelled by the rank of a keyed hash, reverse edges
 * added when symmetric, CSR built as above.  h_info = (nnz, distinct pairs
 * among the candidates); GB_ERR_CAPACITY when fewer than m distinct pairs
 * were drawn (retry with more candidates).  col_cap >= (symmetric ? 2m : m)
 * + GB_COL_PAD.  Synchronises `stream`.  oracle/csrc/gen.c is the host
 * restatement (bit-identical CSR). */
size_t gb_rmat_graph_workspace(int64_t n, int64_t m, int32_t symmetric, int64_t candidates);
int gb_rmat_graph(uint64_t seed, int64_t n, int64_t m, int32_t symmetric, double a, double b,
                  double c, int64_t candidates, int64_t* d_rowptr, int32_t* d_col,
                  int64_t col_cap, int64_t* h_info, void* d_ws, size_t ws_bytes, void* stream);
/* gb_rmat_block — rows [row_lo, row_hi) of the same graph as a block CSR
 * (local rows, global column ids): the 1.5D partition's block row
 * (partition_block_rows, dist.py:200-214) built without the other blocks
 * resident.  The candidate selection is global (transient workspace);
 * GB_ERR_CAPACITY with h_info[0] = block edges when col_cap is too small. */
int gb_rmat_block(uint64_t seed, int64_t n, int64_t m, int32_t symmetric, double a, double b,
                  double c, int64_t candidates, int64_t row_lo, int64_t row_hi,
                  int64_t* d_rowptr, int32_t* d_col, int64_t col_cap, int64_t* h_info,
                  void* d_ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------- instrumentation
 * gb_launch_counter: kernels this host thread has launched through the
 * library (optionally reset).  gb_profile_begin/end: CUDA events recorded
 * around every dominant-kernel launch (the SAGE sample kernel) until end;
 * end synchronises and returns the per-launch durations in ms. */
int64_t gb_launch_counter(int32_t reset);
int gb_profile_begin(int32_t max_marks);
int gb_profile_end(float* h_ms, int32_t cap, int32_t* h_pairs);

#ifdef __cplusplus
}
#endif
#endif /* GNNBULK_B200_H */
