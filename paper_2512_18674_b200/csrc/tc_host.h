// tc_host.h -- host side of the tensor-core (tcgen05) scan: plan + launch.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdlib.h>
#include <stdint.h>

#include "remoe.h"

namespace remoe {

// Batches up to this size use the streaming CUDA-core scan when both are legal.
constexpr int kSimtMaxB = 0;  // the tensor-core scan is faster at every measured B (profiles/)

// Threshold seeding (runtime.cu): batches >= kSeedMinB (and every k > 32) first scan every
// kSeedStride-th row with a k_s-key register top-k per state.
constexpr int kSeedMinB = 32;
// ... and every batch from k = kSeedMinK on: a state's warm-up inserts grow with k (the c5
// sweep: k = 32 at B <= 16 ran at 0.71-0.82 of HBM unseeded, k = 64 seeded at 0.89-0.91)
constexpr int kSeedMinK = 16;
// Shards below kSeedSmallRows rows give each top-k state so few rows that the warm-up
// inserts dominate: seed from kSeedMinBSmall queries on (measured on the c2 store).
constexpr int64_t kSeedSmallRows = 512 * 1024;
constexpr int kSeedMinBSmall = 8;
constexpr int kSeedStride = 64;
// Experiment / debug knobs of the tensor-core scans, read from the environment ONCE when a
// plan is created (remoe_sps_build), never on the launch path.
struct TcKnobs {
  int promo = 3;             // REMOE_TC_PROMO: L2 promotion of TMA boxes (0 none, 1 64 B, 2 128 B, 3 256 B)
  bool full_slab = false;    // REMOE_TC_FULL_SLAB: always store M query rows per K-block
  bool global_bufs = false;  // REMOE_TC_GLOBAL_BUFS: LaneTopk buffers in global memory
  int stages = 0;            // REMOE_TC_STAGES: cap the stage ring (0: as many as fit)
  bool no_multicast = false; // REMOE_NO_MULTICAST: no cluster multicast of store tiles
  int epi_sleep = 0;         // REMOE_EPI_SLEEP: epilogue waits with a suspend-time hint
  int dbg = 0;               // REMOE_TC_DBG: experiment bits (wrong results)
  bool lockstep = false;     // REMOE_PAIR_LOCKSTEP=1: CTA-pair scan query groups in lockstep (k_scan_pair)
  bool stats = false;        // REMOE_TC_STATS: candidate / insert counters (prints, syncs)
  bool trace = false;        // REMOE_TC_TRACE: per-CTA phase stamps (prints, syncs)
  bool verbose = false;      // REMOE_VERBOSE
  static TcKnobs from_env() {
    TcKnobs k;
    auto ival = [](const char* n, int d) { const char* e = getenv(n); return e ? atoi(e) : d; };
    k.promo = ival("REMOE_TC_PROMO", 3);
    k.full_slab = getenv("REMOE_TC_FULL_SLAB") != nullptr;
    k.global_bufs = getenv("REMOE_TC_GLOBAL_BUFS") != nullptr;
    k.stages = ival("REMOE_TC_STAGES", 0);
    k.no_multicast = getenv("REMOE_NO_MULTICAST") != nullptr;
    k.epi_sleep = ival("REMOE_EPI_SLEEP", 0);
    k.dbg = ival("REMOE_TC_DBG", 0);
    k.lockstep = ival("REMOE_PAIR_LOCKSTEP", 0) != 0;
    k.stats = getenv("REMOE_TC_STATS") != nullptr;
    k.trace = getenv("REMOE_TC_TRACE") != nullptr;
    k.verbose = getenv("REMOE_VERBOSE") != nullptr;
    return k;
  }
  CUtensorMapL2promotion promotion() const {
    return promo == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
         : promo == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
         : promo == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }
};
inline int seed_ks_for(int k) { return k <= 32 ? 1 : k <= 64 ? 2 : 4; }

struct TcPlan {
  bool ok = false;            // tensor-core scan usable for this store
  int max_qps = 64;           // queries per resident slab (64; fewer for D > 1280)
  const char* why = "not initialised";
  int grid = 0;               // persistent CTAs (CTA-pair scan, workspaces): min(128-row tiles, SMs)
  int grid_units = 0;         // resident-slab scan CTAs: min(256-row units, SMs) <= grid
  int threads_per_cta_queries = 0;  // per-CTA private top-k lanes
  alignas(64) unsigned char tmap_x[128];  // CUtensorMap of the store (bf16 [n][D], K-major)
  const uint16_t* x = nullptr;
  int64_t n_rows = 0;
  int dim = 0;
  int64_t row_stride = 0;     // elements between rows
  // Tiled copy of the store (tc_tile_store), or nullptr: box (tile, kb) = 128 rows x 64
  // elements, pre-swizzled (SWIZZLE_128B) and contiguous, 16 KB at xt + (tile*nkb + kb)*8192.
  const uint16_t* xt = nullptr;
  TcKnobs kn;                 // read once at plan creation
  // debug buffers of this plan (REMOE_TC_STATS / REMOE_TC_TRACE), freed by tc_plan_destroy
  unsigned* pair_sync = nullptr;          // [17] CTA-pair scan group lockstep counters (zeroed, self-resetting)
  unsigned long long* stats_buf = nullptr;
  unsigned long long* trace_buf = nullptr;
};

// In-kernel threshold seeding (k_scan_tc): a tiled copy of every s-th store
// row (s = 64, 32, 16, 8 are prefixes of 1..4 segments), built once per handle.
struct TcSeed {
  int n_seg = 0;
  int seg_t0[5] = {0, 0, 0, 0, 0};   // first sample unit (256 rows) of segment g; seg_t0[n_seg] = units
  int64_t seg_count[4] = {0, 0, 0, 0}, seg_off[4] = {0, 0, 0, 0}, seg_stride[4] = {0, 0, 0, 0};
  uint16_t* xt = nullptr;            // tiled sample [tiles][D/64][16 KB]
  float* xn = nullptr;               // its norms [tiles * 128] (padding rows: 1)
  uint64_t* pub = nullptr;           // [max_batch][2 * grid] published (key >> 32) << 32 | epoch (zeroed at build)
  uint64_t* done = nullptr;          // [max_batch] (threshold score word) << 32 | epoch, once seeded
  unsigned* epoch = nullptr;         // current epoch (starts at 1; bumped by each chunk's merge)
  long long wait_ns = 200000;        // REMOE_SEED_WAIT_US: the seeding warp's wait bound
};
// One scan's use of the sample: the first n_stiles tiles; every state publishes its h-th
// best sample key and the threshold is the r-th largest published key minus one.
struct TcSeedUse {
  const TcSeed* store = nullptr;
  int n_stiles = 0, h = 1, r = 1;
};
// Builds the sample from x / xnorm (device) with `alloc(actx, bytes)` (returns nullptr on
// failure; the caller owns the memory).  Synchronous on st.
remoe_status_t tc_seed_build(TcSeed* sd, const uint16_t* x, const float* xnorm, int64_t n_rows, int dim,
                             cudaStream_t st, void* (*alloc)(void*, size_t), void* actx);

// Writes the tiled, pre-swizzled copy of x [n_rows x dim] (dim % 8 == 0; K zero-padded to a multiple of 64) into xt
// [ceil(n_rows/128) * 128 * dim] (rows past n_rows are zero).
cudaError_t tc_tile_store(const uint16_t* x, int64_t n_rows, int dim, uint16_t* xt, cudaStream_t st);
// 0 if dynamic shared memory starts 1024-byte aligned, else 1024 (probed once per process).
int dyn_smem_pad();
// D rounded up to whole 64-element K-blocks: the tensor-core scans zero-pad the
// contraction (D % 8 == 0 is all the API requires; the zeros add nothing to a dot product)
inline int tc_kpad(int dim) { return (dim + 63) & ~63; }
inline size_t tc_tiled_bytes(int64_t n_rows, int dim) { return (size_t)((n_rows + 127) / 128) * 128 * tc_kpad(dim) * 2; }

// row_stride: elements between consecutive rows (default dim; a multiple of dim selects
// every (row_stride/dim)-th row of the store, e.g. the threshold-seeding sample).
remoe_status_t tc_plan_create(TcPlan* t, const uint16_t* x, int64_t n_rows, int dim, int num_sms,
                              int max_k, int64_t row_stride = 0);
void tc_plan_destroy(TcPlan* t);
// Scores bc queries (any bc >= 1; 64 or 128 queries per pass) and writes sorted
// top-k key lists: *lists_per_query lists of k keys per query,
// lists[(b * lists_per_query + l) * k + i].
// gid_stride: global id of row r is gid_offset + r * gid_stride (1 for a shard, the
// sample stride for the seeding sample: an arithmetic id, no per-candidate id load).
remoe_status_t tc_scan(TcPlan* t, const uint16_t* q, const float* qnorm, int bc, int k, float sigma,
                       const float* xnorm, int64_t n_rows, int64_t gid_offset, int64_t gid_stride,
                       uint64_t* cand_buf, unsigned long long* gthr, uint64_t* lists, cudaStream_t st,
                       int* launches, int* lists_per_query, const TcSeedUse* seed = nullptr,
                       bool norms_in_kernel = false);
// Large batches: the CTA-pair (cta_group::2) GEMM-tiled scan (k_scan_pair.cu), same
// output contract as tc_scan; 256 queries per pair.
bool tc_pair_usable(const TcPlan* t);
// queries one resident-slab launch keeps in a single slab (128 for D <= 576, else max_qps)
int tc_single_slab_max(const TcPlan* t);
remoe_status_t tc_pair_scan(TcPlan* t, const uint16_t* q, const float* qnorm, int bc, int k, float sigma,
                            const float* xnorm, int64_t n_rows, int64_t gid_offset, int64_t gid_stride,
                            uint64_t* cand_buf, unsigned long long* gthr, uint64_t* lists, cudaStream_t st,
                            int* launches, int* lists_per_query);
// Batches of at least this many queries use the pair scan (REMOE_PAIR_MIN_B overrides).
constexpr int kPairMinB = 128;
// a shard of >= kPairLargeUnits 256-row units per CTA sends every multi-slab batch to the
// CTA-pair scan (c3 B = 72-120: 11% faster; on c2-size stores the pair's fixed costs lose)
constexpr int kPairLargeUnits = 16;

// Largest lists_per_query tc_scan can produce (workspace sizing).
constexpr int kTcMaxStatesPerCta = 2;
constexpr int kTcEpilogueThreads = 256;

}  // namespace remoe
