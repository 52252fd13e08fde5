// tc_host.h -- host side of the tensor-core (tcgen05) scan: plan + launch.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "remoe.h"

namespace remoe {

// Batches up to this size use the streaming CUDA-core scan when both are legal.
constexpr int kSimtMaxB = 0;  // the tensor-core scan is faster at every measured B (profiles/)

struct TcPlan {
  bool ok = false;            // tensor-core scan usable for this store
  const char* why = "not initialised";
  int grid = 0;               // persistent CTAs
  int threads_per_cta_queries = 0;  // per-CTA private top-k lanes
  alignas(64) unsigned char tmap_x[128];  // CUtensorMap of the store (bf16 [n][D], K-major)
  const uint16_t* x = nullptr;
  int64_t n_rows = 0;
  int dim = 0;
};

// row_stride: elements between consecutive rows (default dim; a multiple of dim selects
// every (row_stride/dim)-th row of the store, e.g. the threshold-seeding sample).
remoe_status_t tc_plan_create(TcPlan* t, const uint16_t* x, int64_t n_rows, int dim, int num_sms,
                              int max_k, int64_t row_stride = 0);
void tc_plan_destroy(TcPlan* t);
// Scores bc queries (any bc >= 1; 64 or 128 queries per pass) and writes sorted
// top-k key lists: *lists_per_query lists of k keys per query,
// lists[(b * lists_per_query + l) * k + i].
// gid_map (optional): global id of row r is gid_map[r] instead of gid_offset + r.
remoe_status_t tc_scan(TcPlan* t, const uint16_t* q, const float* qnorm, int bc, int k, float sigma,
                       const float* xnorm, int64_t n_rows, int64_t gid_offset, const int64_t* gid_map,
                       uint64_t* cand_buf, unsigned long long* gthr, uint64_t* lists, cudaStream_t st,
                       int* launches, int* lists_per_query);
// Large batches: the CTA-pair (cta_group::2) GEMM-tiled scan (k_scan_pair.cu), same
// output contract as tc_scan; 256 queries per pair.
bool tc_pair_usable(const TcPlan* t);
remoe_status_t tc_pair_scan(TcPlan* t, const uint16_t* q, const float* qnorm, int bc, int k, float sigma,
                            const float* xnorm, int64_t n_rows, int64_t gid_offset, const int64_t* gid_map,
                            uint64_t* cand_buf, unsigned long long* gthr, uint64_t* lists, cudaStream_t st,
                            int* launches, int* lists_per_query);
// Batches of at least this many queries use the pair scan (REMOE_PAIR_MIN_B overrides).
constexpr int kPairMinB = 128;

// Largest lists_per_query tc_scan can produce (workspace sizing).
constexpr int kTcMaxStatesPerCta = 2;
constexpr int kTcEpilogueThreads = 256;

}  // namespace remoe
