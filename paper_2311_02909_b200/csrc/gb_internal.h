// Internal (C++) declarations shared by the library translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/gnnbulk_b200.h"

namespace gb {

constexpr int kMaxRuns = 64;  // replay-table runs per degree (<= 33 + binades observed)

// Device CSR adjacency + exact-replay tables (opaque gb_graph).
struct Graph {
  int64_t n = 0, nnz = 0;
  const int64_t* rowptr = nullptr;  // caller-owned device memory
  const int32_t* col = nullptr;     // caller-owned, readable for nnz + GB_COL_PAD
  int64_t max_deg = 0, slots = 0;
  int32_t* deg_slot = nullptr;      // [max_deg + 1] -> table slot or -1
  int32_t* slot_deg = nullptr;      // [slots]
  int32_t* run_j0 = nullptr;        // [slots * (kMaxRuns + 1)]
  double* run_s0 = nullptr;         // [slots * kMaxRuns]
  double* run_d = nullptr;          // [slots * kMaxRuns]
  int32_t* run_n = nullptr;         // [slots]
};

// Launch accounting (gb_launch_counter) and optional CUDA-event marks around
// the dominant kernels (gb_profile_begin / gb_profile_end), host-thread local.
void count_launches(int n);
void prof_mark(cudaStream_t st);

int graph_build_tables(Graph* g, cudaStream_t st);
int sage_workspace(const Graph* g, int64_t k, int64_t r1_cap, int32_t layers,
                   const int64_t* fanouts, size_t* bytes);
int sage_bulk(const Graph* g, int64_t k, const int64_t* d_bptr, const int32_t* d_bverts,
              int64_t r1_cap, int64_t batch_size, int32_t layers, const int64_t* fanouts,
              uint64_t seed, uint64_t epoch, int64_t batch_offset, int32_t mode,
              gb_sage_layer_out* L, int64_t* d_sizes, void* d_ws, size_t ws_bytes,
              cudaStream_t st);
int ladies_workspace(const Graph* g, int64_t k, int64_t q1_cap, int32_t layers,
                     const int64_t* fanouts, int32_t mode, size_t* bytes);
int ladies_bulk(const Graph* g, int64_t k, const int64_t* d_qoff, const int32_t* d_qverts,
                int64_t q1_cap, int32_t layers, const int64_t* fanouts, uint64_t seed,
                uint64_t epoch, int64_t batch_offset, int32_t mode, gb_ladies_layer_out* L,
                int64_t* d_sizes, void* d_ws, size_t ws_bytes, cudaStream_t st);

}  // namespace gb
