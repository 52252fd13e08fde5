// runtime.cu -- the C ABI (include/remoe.h): handle, validation, workspaces,
// kernel selection, the per-query launch sequence and the multi-rank exchange.
//
// Query sequence per chunk of <= max_batch queries:
//   k_norms(Q)                                     S1
//   k_scan_{simt|tc|pair}                          S2+S3  (per-CTA top-k lists)
//   k_merge(n_cta lists -> local top-k)            S4     (world == 1: + S6+S7 fused)
//   world > 1:
//     exchange 1: all-gather of the local top-k keys [G][B][k]
//     k_merge(G lists -> global top-k) + fused S6 + partial S7: every rank writes the
//       same ids/scores and P_g = sum over the winners it OWNS (r ascending)       S5-S7
//     exchange 2: all-gather of the partials [G][B][L*E] (small) or, above
//       xchg_ag_max bytes, an all-to-all by query slice + broadcast of the slices
//     k_psum: P = P_0 + P_1 + ... + P_{G-1} in rank order (identical bits on every rank
//       and at every batch position; ncclAllReduce's ring order would not give that)
// The exchanges run over NCCL between processes, or -- for a loopback group (test
// harness: G handles of one process on one device) -- as device copies; both drive
// the same stage functions below.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "remoe.h"
#include "tc_host.h"
#include "tree.h"

namespace {

thread_local std::string g_err;

remoe_status_t fail(remoe_status_t s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define CUDA_TRY(expr)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail(e_ == cudaErrorMemoryAllocation ? REMOE_ERR_OOM : REMOE_ERR_CUDA,        \
                  "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__);    \
  } while (0)

#define NCCL_TRY(expr)                                                                     \
  do {                                                                                     \
    ncclResult_t r_ = (expr);                                                              \
    if (r_ != ncclSuccess)                                                                 \
      return fail(REMOE_ERR_NCCL, "%s: %s (%s:%d)", #expr, ncclGetErrorString(r_),         \
                  __FILE__, __LINE__);                                                     \
  } while (0)

#define ST_TRY(expr)                       \
  do {                                     \
    remoe_status_t s_ = (expr);            \
    if (s_ != REMOE_OK) return s_;         \
  } while (0)

// Restores the caller's current device on scope exit.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// NVTX range for profiler timelines (header-only nvtx3; a no-op without a tool attached).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// Balanced contiguous slice g of n items over G owners: [lo, lo + cnt).
inline void slice_of(int n, int G, int g, int* lo, int* cnt) {
  const int a = (int)((int64_t)n * g / G), b = (int)((int64_t)n * (g + 1) / G);
  *lo = a;
  *cnt = b - a;
}

constexpr int kGraphCache = 8;  // cached device-query graphs per handle (distinct buffer sets)

}  // namespace

struct remoe_sps;

// A loopback group: `world` handles built in one process on one device that act as the
// ranks of one sharded store; their exchanges are device copies (remoe_sps_query_group).
struct remoe_group {
  int world = 0;
  std::vector<remoe_sps*> members;  // by rank; nullptr until that rank is built
  // CUDA graphs of whole group queries (fused exchange only: every step is a kernel), keyed
  // by the buffers; dropped when a member is destroyed
  struct Graph {
    const void* q = nullptr;
    std::vector<const void*> bufs;
    int B = -1, k = -1;
    cudaGraphExec_t exec = nullptr;
    int launches = 0;
  };
  std::vector<Graph> graphs;
  cudaStream_t gst = nullptr;
  cudaEvent_t gev = nullptr, gev_done = nullptr;
  void reset_graphs() {
    for (Graph& gr : graphs)
      if (gr.exec) cudaGraphExecDestroy(gr.exec);
    graphs.clear();
  }
  ~remoe_group() {
    reset_graphs();
    if (gev) cudaEventDestroy(gev);
    if (gev_done) cudaEventDestroy(gev_done);
    if (gst) cudaStreamDestroy(gst);
  }
};

struct remoe_sps {
  remoe_sps_config_t cfg{};
  int64_t n_total = 0;
  int64_t LE = 0;
  int num_sms = 0;
  int grid_simt = 0;
  int grid_tc = 0;
  int stage_rows = 0;
  remoe_group* group = nullptr;  // loopback group membership (world > 1 without NCCL)
  // store
  uint16_t* x = nullptr;
  uint16_t* xt = nullptr;  // tiled copy for the tensor-core scan (or nullptr)
  float* xnorm = nullptr;
  float* act = nullptr;
  // workspaces
  float* qnorm = nullptr;
  unsigned long long* gthr = nullptr;
  uint64_t* cand_buf = nullptr;
  uint64_t* lists = nullptr;
  uint64_t* local_top = nullptr;
  uint64_t* gathered = nullptr;    // [world][max_batch][max_k] (world > 1)
  uint64_t* global_top = nullptr;
  unsigned* split_cnt = nullptr;   // [max_batch] column-split counters of the merge (zeroed, self-resetting)
  float* part = nullptr;           // [max_batch][LE] this rank's partial prediction (world > 1)
  float* part_all = nullptr;       // gathered partials / all-to-all receive buffer (world > 1)
  size_t part_all_floats = 0;
  size_t xchg_ag_max = 32u << 20;  // exchange 2 by all-gather while world*B*LE*4 <= this
  // fused peer-memory exchange (REMOE_FUSED_COMM=1): gathered / part_all are
  // double-buffered by chunk parity; peers store into them directly and raise their flag
  bool fused = false;
  unsigned long long* xflag = nullptr;  // [2][world]: exchange-1 / exchange-2 flag of each rank
  unsigned* xcount = nullptr;           // [2] finished-CTA counters of the two producing kernels
  unsigned long long* d_xseq = nullptr; // chunks exchanged so far, on the device (identical on every rank)
  uint64_t* p_gathered[remoe::kMaxPeers] = {};
  float* p_part_all[remoe::kMaxPeers] = {};
  unsigned long long* p_xflag[remoe::kMaxPeers] = {};
  std::vector<void*> ipc_opened;        // peer allocations opened through CUDA IPC
  // host-path staging
  uint16_t* hq = nullptr;
  int64_t* hids = nullptr;
  float* hscores = nullptr;
  float* hpred = nullptr;
  // tensor-core path
  remoe::TcPlan tc{};
  // threshold seeding: a strided sample of S rows, scanned first; its
  // k-th best key - 1 is a strict lower bound that the full scan starts from
  struct SeedSample {
    int64_t stride = 0, rows = 0;  // rows j * stride, j < rows
    remoe::TcPlan tc{};            // strided tensor map over the store
    float* xns = nullptr;          // their norms
  };
  SeedSample seeds[4];  // strides 64, 32, 16, 8 (larger k takes a denser sample): CTA-pair scan
  int n_seeds = 0;
  // the tensor-core scan seeds inside the kernel from a tiled sample (TcSeed, k_scan_tc)
  remoe::TcSeed seed_store{};
  bool seed_inkernel = true;  // REMOE_SEED_INKERNEL=0: the separate seed-scan launch instead (A/B)
  int seed_segs = 0;          // REMOE_SEED_SEGS: sample segments used by the in-kernel seed (0: by k)
  int seed_units_per_k = 0;   // REMOE_SEED_UNITS_PER_K: sample units the in-kernel seed wants per k
                              // (0: 3 for k <= 64, 1 above -- c3 B = 16/64, k = 128: 0.90/0.83 -> 0.93/0.85
                              // with 1 instead of 2; c2 B = 16/64: 2 -> 3 is 2-3% faster)
  uint64_t* seed_top = nullptr;
  // -1 auto: seed when k >= kSeedMinK or B >= seed_min_b; 1 always (REMOE_SEED=1); 0 never
  // (REMOE_SEED=0).  Without a seed every top-k state (a CTA's rows for one query) starts
  // from nothing and inserts ~k(1 + ln(R/k)) keys, most of them in the first tiles, when
  // all SMs insert at once and the store stream stalls (ncu PM sampling, profiles/).
  int seed_mode = -1;
  int seed_min_b = remoe::kSeedMinB;
  int seed_ks = 0;       // per-state list length of the seed scan (0: seed_ks_for(k))
  ncclComm_t comm = nullptr;
  // NEXT-N2 clustering tree over this shard (remoe_sps_tree_build)
  remoe::Tree tree{};
  bool has_tree = false;
  int force_kernel = 0;
  int last_kernel = 0;
  int pair_min_b = remoe::kPairMinB;  // auto: batches >= this use the CTA-pair scan
  bool use_graphs = true;             // REMOE_NO_GRAPH=1 at build turns the query graphs off
  int last_launches = 0;
  size_t device_bytes = 0;
  std::vector<void*> allocs;
  // CUDA graph of the host-buffer query (remoe_sps_query_host), one cached shape: the
  // H2D copy, S1-S7 and the D2H copies replay as one launch; per call only the four
  // memcpy nodes are re-pointed at the caller's (pinned) buffers.
  struct HostGraph {
    int B = -1, k = -1;
    bool pred = false;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraphNode_t h2d = nullptr, d2h_ids = nullptr, d2h_sc = nullptr, d2h_pred = nullptr;
    int launches = 0;
    void reset() {
      if (exec) cudaGraphExecDestroy(exec);
      if (graph) cudaGraphDestroy(graph);
      exec = nullptr; graph = nullptr; B = -1; k = -1; pred = false;
      h2d = d2h_ids = d2h_sc = d2h_pred = nullptr; launches = 0;
    }
  } hg;
  // CUDA graphs of the device-buffer query (remoe_sps_query, world == 1, one chunk): one
  // per (buffers, B, k) with LRU replacement.  The caller's buffers are baked into the
  // kernel nodes, so a graph is reused only for the same pointers.
  struct DevGraph {
    const void* q = nullptr;
    const void* ids = nullptr;
    const void* scores = nullptr;
    const void* pred = nullptr;
    int B = -1, k = -1, kernel = -1;
    cudaGraphExec_t exec = nullptr;
    int launches = 0;
    int scan_kernel = 0;  // the scan kernel the captured query runs (get_info after a replay)
    uint64_t used = 0;
    void reset() {
      if (exec) cudaGraphExecDestroy(exec);
      exec = nullptr; q = ids = scores = pred = nullptr; B = k = kernel = -1; launches = 0; scan_kernel = 0; used = 0;
    }
  } dg[kGraphCache];
  uint64_t dg_clock = 0;
  void reset_graphs() {
    hg.reset();
    for (auto& g : dg) g.reset();
  }
  // the graphs are captured and replayed on a library stream (the caller's may be the legacy
  // default stream, which cannot be captured), ordered after / before the caller's stream
  // by events
  cudaStream_t gst = nullptr;
  cudaEvent_t gev = nullptr, gev_done = nullptr;
  // live scan timing (remoe_sps_profile)
  bool prof = false;
  std::vector<cudaEvent_t> prof_ev;  // pairs (start, end)
  size_t prof_used = 0;              // pairs recorded since the last read
  double prof_ms = 0.0;
  int64_t prof_launches = 0;

  cudaError_t prof_mark(cudaStream_t st, bool start) {
    if (!prof) return cudaSuccess;
    const size_t idx = 2 * prof_used + (start ? 0 : 1);
    while (prof_ev.size() <= idx) {
      cudaEvent_t e;
      cudaError_t r = cudaEventCreate(&e);
      if (r != cudaSuccess) return r;
      prof_ev.push_back(e);
    }
    cudaError_t r = cudaEventRecord(prof_ev[idx], st);
    if (!start) ++prof_used;
    return r;
  }
  cudaError_t prof_collect() {
    for (size_t i = 0; i < prof_used; ++i) {
      cudaError_t r = cudaEventSynchronize(prof_ev[2 * i + 1]);
      if (r != cudaSuccess) return r;
      float ms = 0.f;
      r = cudaEventElapsedTime(&ms, prof_ev[2 * i], prof_ev[2 * i + 1]);
      if (r != cudaSuccess) return r;
      prof_ms += ms;
    }
    prof_used = 0;
    return cudaSuccess;
  }

  remoe_status_t alloc(void** p, size_t bytes) {
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMalloc(p, bytes);
    if (e != cudaSuccess)
      return fail(e == cudaErrorMemoryAllocation ? REMOE_ERR_OOM : REMOE_ERR_CUDA,
                  "cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
    allocs.push_back(*p);
    device_bytes += bytes;
    return REMOE_OK;
  }
  void release() {
    reset_graphs();
    for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
    ipc_opened.clear();
    if (gev) { cudaEventDestroy(gev); gev = nullptr; }
    if (gev_done) { cudaEventDestroy(gev_done); gev_done = nullptr; }
    if (gst) { cudaStreamDestroy(gst); gst = nullptr; }
    for (void* p : allocs) cudaFree(p);
    allocs.clear();
    for (cudaEvent_t e : prof_ev) cudaEventDestroy(e);
    prof_ev.clear();
    remoe::tc_plan_destroy(&tc);
    for (int i = 0; i < n_seeds; ++i) remoe::tc_plan_destroy(&seeds[i].tc);
    n_seeds = 0;
    if (has_tree) { remoe::tree_free(&tree); has_tree = false; }
    if (comm) { ncclCommDestroy(comm); comm = nullptr; }
    if (group) {
      if (cfg.rank >= 0 && cfg.rank < (int)group->members.size() && group->members[cfg.rank] == this)
        group->members[cfg.rank] = nullptr;
      group->reset_graphs();  // captured with this member's buffers
      group = nullptr;
    }
  }
};

extern "C" {

void remoe_sps_config_default(remoe_sps_config_t* c) {
  if (!c) return;
  std::memset(c, 0, sizeof *c);
  c->sigma = 1e-6f;
  c->temperature = 1.0f;
  c->max_batch = 256;
  c->max_k = 128;
  c->world = 1;
  c->validate = 1;
}

const char* remoe_status_string(remoe_status_t s) {
  switch (s) {
    case REMOE_OK: return "ok";
    case REMOE_ERR_INVALID_ARG: return "invalid argument";
    case REMOE_ERR_CUDA: return "CUDA error";
    case REMOE_ERR_NCCL: return "NCCL error";
    case REMOE_ERR_OOM: return "out of device memory";
    case REMOE_ERR_UNSUPPORTED: return "unsupported";
    case REMOE_ERR_STATE: return "invalid state";
  }
  return "unknown status";
}

const char* remoe_last_error(void) { return g_err.c_str(); }

remoe_status_t remoe_nccl_unique_id(uint8_t out[128]) {
  if (!out) return fail(REMOE_ERR_INVALID_ARG, "out is NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  std::memcpy(out, &id, 128);
  return REMOE_OK;
}

remoe_status_t remoe_loopback_group_create(int32_t world, remoe_group_t* out) {
  if (!out) return fail(REMOE_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (world < 1 || world > 1024) return fail(REMOE_ERR_INVALID_ARG, "need 1 <= world <= 1024");
  remoe_group* g = new (std::nothrow) remoe_group();
  if (!g) return fail(REMOE_ERR_OOM, "host allocation failed");
  g->world = world;
  g->members.assign(world, nullptr);
  *out = g;
  return REMOE_OK;
}

remoe_status_t remoe_loopback_group_destroy(remoe_group_t g) {
  if (!g) return REMOE_OK;
  for (remoe_sps* m : g->members)
    if (m) return fail(REMOE_ERR_STATE, "destroy the group's handles first");
  delete g;
  return REMOE_OK;
}

// Checks that cannot wait for the multi-rank agreement (a rank failing them cannot even
// join the group).  Everything else is checked by check_local after the NCCL
// communicator exists, so that every rank fails together (remoe_sps_build's agreement).
static remoe_status_t check_join(const remoe_sps_config_t* c) {
  if (!c) return fail(REMOE_ERR_INVALID_ARG, "cfg is NULL");
  if (c->world < 1 || c->rank < 0 || c->rank >= c->world)
    return fail(REMOE_ERR_INVALID_ARG, "need 0 <= rank < world");
  const bool lb = c->loopback_group != nullptr;
  if (c->world == 1 && (c->nccl_unique_id != nullptr || lb))
    return fail(REMOE_ERR_INVALID_ARG, "world == 1 takes neither an NCCL id nor a loopback group");
  if (c->world > 1 && ((c->nccl_unique_id != nullptr) == lb))
    return fail(REMOE_ERR_INVALID_ARG, "world > 1 needs exactly one of nccl_unique_id / loopback_group");
  if (lb) {
    const remoe_group* g = static_cast<const remoe_group*>(c->loopback_group);
    if (g->world != c->world) return fail(REMOE_ERR_INVALID_ARG, "loopback group world %d != cfg world %d",
                                          g->world, c->world);
    if (g->members[c->rank] != nullptr) return fail(REMOE_ERR_STATE, "rank %d of the loopback group is taken", c->rank);
  }
  return REMOE_OK;
}

static remoe_status_t check_device(const remoe_sps_config_t* c) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(REMOE_ERR_CUDA, "no CUDA device visible");
  }
  if (c->device < 0 || c->device >= ndev) return fail(REMOE_ERR_INVALID_ARG, "device out of range");
  return REMOE_OK;
}

static remoe_status_t check_local(const remoe_sps_config_t* c, const void* emb, const void* act) {
  if (c->n_local < 1) return fail(REMOE_ERR_INVALID_ARG, "n_local must be >= 1");
  if (c->global_offset < 0) return fail(REMOE_ERR_INVALID_ARG, "global_offset must be >= 0");
  if (c->global_offset + c->n_local > 0xFFFFFFFELL)
    return fail(REMOE_ERR_UNSUPPORTED, "global ids must fit 32 bits");
  if (c->dim < 8 || c->dim % 8 != 0) return fail(REMOE_ERR_INVALID_ARG, "dim must be a positive multiple of 8");
  if (c->dim > 4096) return fail(REMOE_ERR_UNSUPPORTED, "dim > 4096");
  if (c->n_layers < 1) return fail(REMOE_ERR_INVALID_ARG, "n_layers must be >= 1");
  if (c->n_experts < 1) return fail(REMOE_ERR_INVALID_ARG, "n_experts must be >= 1");
  if (c->n_experts > 256) return fail(REMOE_ERR_UNSUPPORTED, "n_experts > 256");
  if (!(c->sigma > 0.f)) return fail(REMOE_ERR_INVALID_ARG, "sigma must be > 0 (Eq. 11)");
  if (!(c->temperature > 0.f)) return fail(REMOE_ERR_INVALID_ARG, "temperature must be > 0");
  if (c->max_batch < 1) return fail(REMOE_ERR_INVALID_ARG, "max_batch must be >= 1");
  if (c->max_k < 1) return fail(REMOE_ERR_INVALID_ARG, "max_k must be >= 1");
  if (c->max_k > 256) return fail(REMOE_ERR_UNSUPPORTED, "max_k > 256");
  if (!emb || !act) return fail(REMOE_ERR_INVALID_ARG, "emb/act is NULL");
  return REMOE_OK;
}

// Everything of the build that is local to this rank: the store, its norms and validation,
// the tensor-core plans and the workspaces.
static remoe_status_t build_local(remoe_sps* h, const uint16_t* emb, const float* act, cudaStream_t st) {
  const remoe_sps_config_t& c = h->cfg;
  ST_TRY(check_local(&c, emb, act));
  // ---- store
  const size_t xbytes = (size_t)c.n_local * c.dim * 2;
  const size_t abytes = (size_t)c.n_local * h->LE * 4;
  ST_TRY(h->alloc((void**)&h->x, xbytes));
  // + 4 floats: the tensor-core scan bulk-copies a tile's norms in 16-byte units
  ST_TRY(h->alloc((void**)&h->xnorm, (size_t)(c.n_local + 4) * 4));
  ST_TRY(h->alloc((void**)&h->act, abytes));
  const cudaMemcpyKind kind = c.inputs_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  CUDA_TRY(cudaMemcpyAsync(h->x, emb, xbytes, kind, st));
  CUDA_TRY(cudaMemcpyAsync(h->act, act, abytes, kind, st));
  CUDA_TRY(remoe::launch_norms(h->x, c.n_local, c.dim, h->xnorm, st));
  if (c.validate) {
    unsigned long long* bad = nullptr;
    ST_TRY(h->alloc((void**)&bad, 8));
    CUDA_TRY(cudaMemsetAsync(bad, 0, 8, st));
    CUDA_TRY(remoe::launch_validate(h->x, c.n_local, c.dim, h->act, c.n_local * c.n_layers,
                                    c.n_experts, bad, st));
    unsigned long long hb = 0;
    CUDA_TRY(cudaMemcpyAsync(&hb, bad, 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (hb) return fail(REMOE_ERR_INVALID_ARG, "validate: %llu non-finite embeddings or invalid activation rows", hb);
  }

  // ---- kernel geometry + workspaces
  h->grid_simt = h->num_sms;
  h->stage_rows = std::max(1, std::min(64, 65536 / (2 * c.dim)));  // 64 KB TMA stages
  const int capmax = 32 * remoe::topk_P(c.max_k);
  ST_TRY(remoe::tc_plan_create(&h->tc, h->x, c.n_local, c.dim, h->num_sms, c.max_k));
  h->grid_tc = h->tc.grid;
  // Tiled, pre-swizzled copy of the store for the tensor-core scan: every
  // 16 KB box the scan loads is one contiguous range of HBM.  REMOE_TC_TILED=0 keeps the
  // 2-D tensor-map loads of the row-major store (and saves the copy's memory).
  const char* tiled_env = getenv("REMOE_TC_TILED");
  if (h->tc.ok && !(tiled_env && atoi(tiled_env) == 0)) {
    ST_TRY(h->alloc((void**)&h->xt, remoe::tc_tiled_bytes(c.n_local, c.dim)));
    CUDA_TRY(remoe::tc_tile_store(h->x, c.n_local, c.dim, h->xt, st));
    h->tc.xt = h->xt;
  }
  const int lists_max = std::max(h->grid_simt, h->grid_tc * remoe::kTcMaxStatesPerCta);
  const size_t cand_lanes = std::max((size_t)h->grid_simt * 32,
                                     (size_t)h->grid_tc * h->tc.threads_per_cta_queries);
  const int mb = c.max_batch;
  ST_TRY(h->alloc((void**)&h->qnorm, (size_t)mb * 4));
  ST_TRY(h->alloc((void**)&h->gthr, (size_t)2 * mb * 8));  // [0, mb): main scan, [mb, 2mb): seed scan
  CUDA_TRY(cudaMemsetAsync(h->gthr, 0, (size_t)2 * mb * 8, st));  // kept zero between chunks (k_merge resets)
  // ---- seeding sample: S rows j * stride, S a multiple
  // of 128, only for large shards.  The sample is read in place through a strided tensor
  // map; only its norms and global ids are copied.
  std::vector<int64_t> strides = {remoe::kSeedStride, remoe::kSeedStride / 2, remoe::kSeedStride / 4,
                                  remoe::kSeedStride / 8};
  if (const char* e = getenv("REMOE_SEED_STRIDE")) strides = {std::max(2, atoi(e))};
  if (h->tc.ok && c.n_local >= 32 * 2048) {
    ST_TRY(h->alloc((void**)&h->seed_top, (size_t)mb * c.max_k * 8));
    for (int64_t want : strides) {
      const int64_t stride = std::max<int64_t>(2, std::min<int64_t>(want, c.n_local / 2048));
      if (h->n_seeds > 0 && h->seeds[h->n_seeds - 1].stride == stride) continue;
      remoe_sps::SeedSample& sd = h->seeds[h->n_seeds];
      const int64_t S = (c.n_local / stride) / 128 * 128;
      sd.stride = stride;
      sd.rows = S;
      ST_TRY(h->alloc((void**)&sd.xns, (size_t)S * 4));
      CUDA_TRY(cudaMemcpy2DAsync(sd.xns, 4, h->xnorm, (size_t)stride * 4, 4, S, cudaMemcpyDeviceToDevice, st));
      CUDA_TRY(cudaStreamSynchronize(st));
      ST_TRY(remoe::tc_plan_create(&sd.tc, h->x, S, c.dim, h->num_sms, c.max_k, stride * c.dim));
      if (sd.tc.ok) ++h->n_seeds;
    }
  }
  // in-kernel seeding sample of the tensor-core scan: every 64th/32nd/16th/8th row, tiled
  if (h->tc.ok && h->xt && c.n_local >= 32768) {
    auto al = [](void* ctx, size_t bytes) -> void* {
      void* p = nullptr;
      return static_cast<remoe_sps*>(ctx)->alloc(&p, bytes) == REMOE_OK ? p : nullptr;
    };
    ST_TRY(remoe::tc_seed_build(&h->seed_store, h->x, h->xnorm, c.n_local, c.dim, st, al, h));
    remoe::TcSeed& sd = h->seed_store;
    if (sd.n_seg > 0) {
      const size_t slots = (size_t)mb * 2 * std::max(1, h->grid_tc);
      ST_TRY(h->alloc((void**)&sd.pub, slots * 8));
      ST_TRY(h->alloc((void**)&sd.epoch, sizeof(unsigned)));
      ST_TRY(h->alloc((void**)&sd.done, (size_t)mb * 8));
      CUDA_TRY(cudaMemsetAsync(sd.pub, 0, slots * 8, st));
      CUDA_TRY(cudaMemsetAsync(sd.done, 0, (size_t)mb * 8, st));
      static const unsigned one = 1;  // epoch 0 would match the zeroed words
      CUDA_TRY(cudaMemcpyAsync(sd.epoch, &one, sizeof one, cudaMemcpyHostToDevice, st));
      if (const char* e = getenv("REMOE_SEED_WAIT_US")) sd.wait_ns = 1000LL * std::max(0, atoi(e));
    }
  }
  if (const char* e = getenv("REMOE_SEED")) h->seed_mode = atoi(e) != 0 ? 1 : 0;
  if (const char* e = getenv("REMOE_SEED_INKERNEL")) h->seed_inkernel = atoi(e) != 0;
  if (const char* e = getenv("REMOE_SEED_SEGS")) h->seed_segs = std::max(0, std::min(4, atoi(e)));
  if (const char* e = getenv("REMOE_SEED_UNITS_PER_K")) h->seed_units_per_k = std::max(1, std::min(8, atoi(e)));
  if (const char* e = getenv("REMOE_SEED_MIN_B")) h->seed_min_b = atoi(e);
  if (const char* e = getenv("REMOE_SEED_KS")) h->seed_ks = std::max(0, std::min(32, atoi(e)));
  if (const char* e = getenv("REMOE_PAIR_MIN_B")) {
    h->pair_min_b = atoi(e);
  } else if (h->tc.ok && h->tc.grid > 0 &&
             c.n_local >= (int64_t)remoe::kPairLargeUnits * 256 * h->tc.grid) {
    // a large shard: batches past one resident slab go to the CTA-pair scan
    h->pair_min_b = std::min(remoe::kPairMinB, remoe::tc_single_slab_max(&h->tc) + 1);
  }
  if (const char* e = getenv("REMOE_NO_GRAPH")) h->use_graphs = atoi(e) == 0;
  if (h->tc.kn.trace || h->tc.kn.stats) h->use_graphs = false;  // debug knobs read back and print per launch
  if (const char* e = getenv("REMOE_XCHG_AG_MAX")) h->xchg_ag_max = (size_t)std::max(0LL, atoll(e));
  ST_TRY(h->alloc((void**)&h->cand_buf, cand_lanes * capmax * 8));
  ST_TRY(h->alloc((void**)&h->lists, (size_t)mb * lists_max * c.max_k * 8));
  ST_TRY(h->alloc((void**)&h->local_top, (size_t)mb * c.max_k * 8));
  ST_TRY(h->alloc((void**)&h->global_top, (size_t)mb * c.max_k * 8));
  ST_TRY(h->alloc((void**)&h->split_cnt, (size_t)mb * sizeof(unsigned)));
  CUDA_TRY(cudaMemsetAsync(h->split_cnt, 0, (size_t)mb * sizeof(unsigned), st));
  if (c.world > 1) {
    // exchange workspaces: keys [G][mb][max_k]; this rank's partial P
    // [mb][LE]; the gathered partials [G][mb][LE] when they fit xchg_ag_max, and always
    // the all-to-all receive slices [G][ceil(mb / G)][LE]
    const size_t G = (size_t)c.world, LE = (size_t)h->LE;
    if (const char* e = getenv("REMOE_FUSED_COMM")) h->fused = atoi(e) != 0 && c.world <= remoe::kMaxPeers;
    const size_t nbuf = h->fused ? 2 : 1;  // fused: double-buffered by chunk parity
    ST_TRY(h->alloc((void**)&h->gathered, nbuf * G * mb * c.max_k * 8));
    ST_TRY(h->alloc((void**)&h->part, (size_t)mb * LE * 4));
    const size_t a2a = G * ((mb + G - 1) / G) * LE;
    const size_t ag = std::min(G * mb * LE, h->xchg_ag_max / 4);
    h->part_all_floats = std::max(a2a, ag);
    ST_TRY(h->alloc((void**)&h->part_all, nbuf * h->part_all_floats * 4));
    if (h->fused) {
      ST_TRY(h->alloc((void**)&h->xflag, 2 * G * sizeof(unsigned long long)));
      ST_TRY(h->alloc((void**)&h->xcount, 2 * sizeof(unsigned)));
      ST_TRY(h->alloc((void**)&h->d_xseq, sizeof(unsigned long long)));
      CUDA_TRY(cudaMemsetAsync(h->d_xseq, 0, sizeof(unsigned long long), st));
      CUDA_TRY(cudaMemsetAsync(h->xflag, 0, 2 * G * sizeof(unsigned long long), st));
      CUDA_TRY(cudaMemsetAsync(h->xcount, 0, 2 * sizeof(unsigned), st));
    }
  }
  ST_TRY(h->alloc((void**)&h->hq, (size_t)mb * c.dim * 2));
  ST_TRY(h->alloc((void**)&h->hids, (size_t)mb * c.max_k * 8));
  ST_TRY(h->alloc((void**)&h->hscores, (size_t)mb * c.max_k * 4));
  ST_TRY(h->alloc((void**)&h->hpred, (size_t)mb * h->LE * 4));
  CUDA_TRY(cudaStreamSynchronize(st));

  if (const char* f = getenv("REMOE_FORCE_KERNEL")) {
    if (!strcmp(f, "stream")) h->force_kernel = 1;
    else if (!strcmp(f, "tc")) h->force_kernel = 2;
    else if (!strcmp(f, "pair")) h->force_kernel = 3;
  }
  return REMOE_OK;
}

// NCCL ranks agree on the build: every rank contributes (offset, n_local, status); if any
// rank failed, every rank fails (none is left waiting in a later collective), otherwise
// the shards must tile [0, N) in rank order.
static remoe_status_t agree_build(remoe_sps* h, remoe_status_t local, cudaStream_t st) {
  const remoe_sps_config_t& c = h->cfg;
  const std::string local_err = g_err;
  int64_t* d = nullptr;
  const size_t bytes = sizeof(int64_t) * 4 * (c.world + 1);
  if (cudaMalloc(&d, bytes) != cudaSuccess) {
    cudaGetLastError();
    return fail(REMOE_ERR_OOM, "agreement buffer");  // cannot take part: peers will see NCCL errors
  }
  int64_t mine[4] = {c.global_offset, c.n_local, (int64_t)local, h->fused ? 1 : 0};
  std::vector<int64_t> all(4 * c.world);
  cudaError_t ce = cudaMemcpyAsync(d, mine, sizeof mine, cudaMemcpyHostToDevice, st);
  ncclResult_t nr = ce == cudaSuccess ? ncclAllGather(d, d + 4, 4, ncclInt64, h->comm, st) : ncclSuccess;
  if (ce == cudaSuccess && nr == ncclSuccess)
    ce = cudaMemcpyAsync(all.data(), d + 4, sizeof(int64_t) * 4 * c.world, cudaMemcpyDeviceToHost, st);
  if (ce == cudaSuccess && nr == ncclSuccess) ce = cudaStreamSynchronize(st);
  cudaFree(d);
  if (local != REMOE_OK) {
    g_err = local_err;
    return local;
  }
  if (nr != ncclSuccess) return fail(REMOE_ERR_NCCL, "build agreement: %s", ncclGetErrorString(nr));
  if (ce != cudaSuccess) return fail(REMOE_ERR_CUDA, "build agreement: %s", cudaGetErrorString(ce));
  for (int g = 0; g < c.world; ++g)
    if (all[4 * g + 2] != REMOE_OK)
      return fail((remoe_status_t)all[4 * g + 2], "rank %d failed its build (%s); every rank fails", g,
                  remoe_status_string((remoe_status_t)all[4 * g + 2]));
  int64_t expect = 0;
  bool fused_all = true;
  for (int g = 0; g < c.world; ++g) {
    if (all[4 * g] != expect)
      return fail(REMOE_ERR_INVALID_ARG, "shards do not tile [0, N): rank %d offset %lld, expected %lld",
                  g, (long long)all[4 * g], (long long)expect);
    expect += all[4 * g + 1];
    fused_all = fused_all && all[4 * g + 3] != 0;
  }
  h->n_total = expect;
  h->fused = fused_all;  // the fused exchange only if every rank asked for it
  return REMOE_OK;
}

// Fused exchange between NCCL ranks: every rank exports CUDA IPC handles of
// its receive buffers (gathered keys, partials, flags), the handles are all-gathered once,
// and every rank opens its peers' (NVLink peer mappings on one node).  The ranks agree
// (all-reduce MIN): if any rank cannot open every peer, none uses the fused path.
static remoe_status_t setup_peers_nccl(remoe_sps* h, cudaStream_t st) {
  const int G = h->cfg.world, r = h->cfg.rank;
  struct Handles { cudaIpcMemHandle_t gathered, part_all, xflag; };
  Handles mine{};
  int ok = cudaIpcGetMemHandle(&mine.gathered, h->gathered) == cudaSuccess &&
           cudaIpcGetMemHandle(&mine.part_all, h->part_all) == cudaSuccess &&
           cudaIpcGetMemHandle(&mine.xflag, h->xflag) == cudaSuccess;
  cudaGetLastError();
  std::vector<Handles> all(G);
  char* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, sizeof(Handles) * (G + 1) + sizeof(int)));
  struct Free { char* p; ~Free() { cudaFree(p); } } fr{d};
  int* dok = reinterpret_cast<int*>(d + sizeof(Handles) * (G + 1));
  CUDA_TRY(cudaMemcpyAsync(d, &mine, sizeof mine, cudaMemcpyHostToDevice, st));
  NCCL_TRY(ncclAllGather(d, d + sizeof(Handles), sizeof(Handles), ncclChar, h->comm, st));
  CUDA_TRY(cudaMemcpyAsync(all.data(), d + sizeof(Handles), sizeof(Handles) * G, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  for (int g = 0; g < G; ++g) {
    if (g == r) {
      h->p_gathered[g] = h->gathered; h->p_part_all[g] = h->part_all; h->p_xflag[g] = h->xflag;
      continue;
    }
    void* pg = nullptr; void* pp = nullptr; void* pf = nullptr;
    if (ok && cudaIpcOpenMemHandle(&pg, all[g].gathered, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess) h->ipc_opened.push_back(pg); else ok = 0;
    if (ok && cudaIpcOpenMemHandle(&pp, all[g].part_all, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess) h->ipc_opened.push_back(pp); else ok = 0;
    if (ok && cudaIpcOpenMemHandle(&pf, all[g].xflag, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess) h->ipc_opened.push_back(pf); else ok = 0;
    cudaGetLastError();
    h->p_gathered[g] = static_cast<uint64_t*>(pg);
    h->p_part_all[g] = static_cast<float*>(pp);
    h->p_xflag[g] = static_cast<unsigned long long*>(pf);
  }
  CUDA_TRY(cudaMemcpyAsync(dok, &ok, sizeof ok, cudaMemcpyHostToDevice, st));
  NCCL_TRY(ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, h->comm, st));
  CUDA_TRY(cudaMemcpyAsync(&ok, dok, sizeof ok, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (!ok) {  // every rank falls back to the NCCL exchanges
    for (void* p : h->ipc_opened) cudaIpcCloseMemHandle(p);
    h->ipc_opened.clear();
    h->fused = false;
  }
  return REMOE_OK;
}

// Fused exchange in a loopback group: the peers are the members' own device buffers.
static remoe_status_t setup_peers_loopback(remoe_sps* const* hs, int G) {
  bool all = true;
  for (int g = 0; g < G; ++g) all = all && hs[g]->fused;
  for (int m = 0; m < G; ++m) {
    if (!all) { hs[m]->fused = false; continue; }
    for (int g = 0; g < G; ++g) {
      hs[m]->p_gathered[g] = hs[g]->gathered;
      hs[m]->p_part_all[g] = hs[g]->part_all;
      hs[m]->p_xflag[g] = hs[g]->xflag;
    }
  }
  return REMOE_OK;
}

static remoe_status_t build_impl(remoe_sps* h, const uint16_t* emb, const float* act) {
  const remoe_sps_config_t& c = h->cfg;
  CUDA_TRY(cudaSetDevice(c.device));
  CUDA_TRY(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, c.device));
  h->LE = (int64_t)c.n_layers * c.n_experts;
  cudaStream_t st = nullptr;
  CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard { cudaStream_t s; ~StreamGuard() { cudaStreamDestroy(s); } } sg{st};
  if (c.world > 1 && c.loopback_group == nullptr) {
    // the communicator first: a rank whose local build fails below still takes part in
    // the agreement, so no peer is left blocked in a collective
    ncclUniqueId id;
    std::memcpy(&id, c.nccl_unique_id, sizeof id);
    NCCL_TRY(ncclCommInitRank(&h->comm, c.world, id, c.rank));
    ST_TRY(agree_build(h, build_local(h, emb, act, st), st));
    return h->fused ? setup_peers_nccl(h, st) : REMOE_OK;
  }
  ST_TRY(build_local(h, emb, act, st));
  if (c.loopback_group) {
    h->group = static_cast<remoe_group*>(const_cast<void*>(c.loopback_group));
    h->group->members[c.rank] = h;
    h->n_total = 0;  // known once every member is built (checked by remoe_sps_query_group)
  } else {
    h->n_total = c.n_local;
  }
  return REMOE_OK;
}

remoe_status_t remoe_sps_build(const remoe_sps_config_t* cfg, const uint16_t* emb_bf16,
                               const float* act, remoe_sps_t* out) {
  if (!out) return fail(REMOE_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  ST_TRY(check_join(cfg));
  // single-process builds check everything up front, before any CUDA call; NCCL ranks
  // check the rest after the communicator exists (build_impl's agreement)
  if (cfg->world == 1 || cfg->loopback_group) ST_TRY(check_local(cfg, emb_bf16, act));
  ST_TRY(check_device(cfg));
  remoe_sps* h = new (std::nothrow) remoe_sps();
  if (!h) return fail(REMOE_ERR_OOM, "host allocation failed");
  h->cfg = *cfg;
  DeviceGuard dg(cfg->device);
  remoe_status_t s = build_impl(h, emb_bf16, act);
  h->cfg.nccl_unique_id = nullptr;  // the caller owns those bytes; not kept past build
  if (s == REMOE_OK) {
    *out = h;
  } else {
    h->release();
    delete h;
  }
  return s;
}

}  // extern "C"

// ------------------------------------------------------------------ query stages

// S1-S4 on this rank's shard: query norms, [threshold seeding], the scan, and the merge of
// the per-CTA lists.  With `fin` (world == 1) the merge CTA goes on to S5-S7 itself (ids,
// scores, prediction); otherwise the local top-k keys land in h->local_top.
static remoe_status_t stage_scan(remoe_sps* h, const uint16_t* q, int bc, int k, const remoe::FinalizeArgs* fin,
                                 cudaStream_t st, int* launches, const remoe::PeerXchg* px = nullptr) {
  const remoe_sps_config_t& c = h->cfg;
  // ---- S2+S3
  int which = h->force_kernel;
  if (which == 0) {
    which = (bc <= remoe::kSimtMaxB || !h->tc.ok) ? 1 : 2;
    if (which == 2 && bc >= h->pair_min_b && remoe::tc_pair_usable(&h->tc)) which = 3;
  }
  if (which >= 2 && !h->tc.ok) return fail(REMOE_ERR_UNSUPPORTED, "tensor-core scan unavailable: %s", h->tc.why);
  if (which == 3 && !remoe::tc_pair_usable(&h->tc))
    return fail(REMOE_ERR_UNSUPPORTED, "CTA-pair tensor-core scan unavailable for this store");
  int grid = 0;  // sorted key lists per query produced by the scan
  remoe::TcSeedUse su;  // in-kernel seeding of the tensor-core scan (none: su.store == nullptr)
  // S1: the resident-slab tensor-core scan computes the query norms in its prologue (and the
  // previous chunk's merge left the shared thresholds at zero); the other paths launch
  // k_norms, which also zeroes the thresholds
  const bool fold_norms = which == 2 && (h->seed_inkernel || h->seed_mode == 0);
  if (!fold_norms) {
    CUDA_TRY(remoe::launch_norms(q, bc, c.dim, h->qnorm, st, h->gthr, c.max_batch));
    ++*launches;
  }
  CUDA_TRY(h->prof_mark(st, true));
  if (which == 1) {
    grid = h->grid_simt;
    int BQ = bc >= 8 ? 8 : bc >= 4 ? 4 : bc >= 2 ? 2 : 1;
    // the query slab (BQ x D fp32) and >= 2 stages must fit the opt-in shared memory
    while (BQ > 1 && remoe::simt_smem_bytes(BQ, c.dim, h->stage_rows, 2) > (size_t)remoe::kSimtMaxSmem) BQ >>= 1;
    if (remoe::simt_smem_bytes(BQ, c.dim, h->stage_rows, 2) > (size_t)remoe::kSimtMaxSmem)
      return fail(REMOE_ERR_UNSUPPORTED, "streaming scan: D = %d does not fit shared memory", c.dim);
    int NST = std::max(2, std::min(6, (int)((210 * 1024 - std::min<size_t>(210 * 1024, (size_t)BQ * c.dim * 4)) /
                                            ((size_t)h->stage_rows * c.dim * 2))));
    while (NST > 2 && remoe::simt_smem_bytes(BQ, c.dim, h->stage_rows, NST) > (size_t)remoe::kSimtMaxSmem) --NST;
    for (int s0 = 0; s0 < bc; s0 += BQ) {
      remoe::SimtScanParams p{};
      p.x = h->x; p.xnorm = h->xnorm; p.n_rows = c.n_local; p.gid_offset = c.global_offset;
      p.dim = c.dim; p.q = q + (size_t)s0 * c.dim; p.qnorm = h->qnorm + s0;
      p.nq = std::min(BQ, bc - s0); p.k = k; p.sigma = c.sigma;
      p.stage_rows = h->stage_rows; p.n_stages_ring = NST;
      p.cand_buf = h->cand_buf; p.gthr = h->gthr + s0; p.out = h->lists + (size_t)s0 * grid * k;
      CUDA_TRY(remoe::launch_scan_simt(p, BQ, grid, st));
      ++*launches;
    }
  } else {
    int nl = 0;
    const int seed_min_b = c.n_local < remoe::kSeedSmallRows ? std::min(h->seed_min_b, remoe::kSeedMinBSmall)
                                                              : h->seed_min_b;
    const bool seed = h->seed_mode == 1 || (h->seed_mode == -1 && (k >= remoe::kSeedMinK || bc >= seed_min_b));
    // Lists per query the seed scan will produce, at least: one per CTA of a query slab
    // (M >= 64 queries per slab) or per CTA pair of a 256-query group.
    // Sample density by k: the sample should hold ~k rows of a query's topic for its k-th
    // best to approach the final k-th best (stride 64 for k <= 16, 8 for k >= 128).
    int want_stride = remoe::kSeedStride;
    while (want_stride > remoe::kSeedStride / 8 && (int64_t)want_stride * k > 1024) want_stride /= 2;
    int si = 0;
    for (int i = 0; i < h->n_seeds; ++i)
      if (h->seeds[i].stride >= want_stride) si = i;
    const remoe_sps::SeedSample* sd = h->n_seeds > 0 ? &h->seeds[si] : nullptr;
    const int sg = sd ? (which == 3 ? sd->tc.grid : sd->tc.grid_units) : 0;  // the seed scan's CTAs
    const int lists_min = which == 3 ? std::max(1, (sg / 2) / std::max(1, std::min((bc + 255) / 256, sg / 2)))
                                     : std::max(1, sg / std::max(1, std::min((bc + 63) / 64, sg)));
    int ks_auto = remoe::seed_ks_for(k);
    while (ks_auto < 32 && (int64_t)lists_min * ks_auto < 4 * k) ks_auto *= 2;
    const int ks = h->seed_ks > 0 ? std::min(h->seed_ks, k) : std::min(ks_auto, k);
    // the tensor-core scan seeds inside the kernel (TcSeed): the first tiles of the sample
    // prefix with stride ~1024 / k, each state's h-th best key, threshold = the r-th largest
    const remoe::TcSeed& ss = h->seed_store;
    if (which == 2 && seed && ss.n_seg > 0 && h->seed_inkernel) {
      // Each state publishes its best sample key (h = 1) and the threshold is the k-th largest
      // of them (r = k): the sample needs >= k units (seed_units_per_k * k wanted), so the
      // prefix grows with k (every 64th row, then 32nd, 16th, 8th; REMOE_SEED_SEGS overrides
      // the segment count).  One key per 256-row unit of a random-order sample: the k-th
      // largest unit maximum is about the k-th best row of the sample.
      const int want = (h->seed_units_per_k > 0 ? h->seed_units_per_k : k <= 64 ? 3 : 1) * k;
      int nseg = 1;
      while (nseg < ss.n_seg && ss.seg_t0[nseg] < want) ++nseg;
      if (h->seed_segs > 0) nseg = std::min(h->seed_segs, ss.n_seg);
      const int ntl = ss.seg_t0[nseg];
      if (ntl >= k) {  // a smaller sample than wanted still seeds (k keys are enough)
        su.store = &ss;
        su.n_stiles = ntl;
        su.h = 1;
        su.r = k;
      }
    }
    // the separate seed-scan launch: the CTA-pair scan, and the tensor-core scan when in-kernel
    // seeding is off (it needs k_norms' query norms and zeroed seed thresholds)
    if ((which == 3 || (!su.store && !fold_norms)) && sd && seed && 8 * k <= sd->rows && (int64_t)lists_min * ks >= k) {
      // Scan the sample with a short register top-k (k_s keys per state, k_s = 1 for
      // k <= 32: a running max, no insertion work): the k-th best key of the union of the
      // per-CTA lists is a real key of the store, hence a lower bound of the final k-th
      // best; minus one it seeds the thresholds (strict bound).
      int sl = 0;
      const remoe_status_t ss =
          which == 3 ? remoe::tc_pair_scan(const_cast<remoe::TcPlan*>(&sd->tc), q, h->qnorm, bc, ks, c.sigma, sd->xns,
                                           sd->rows, c.global_offset, sd->stride, h->cand_buf, h->gthr + c.max_batch, h->lists, st,
                                           &nl, &sl)
                     : remoe::tc_scan(const_cast<remoe::TcPlan*>(&sd->tc), q, h->qnorm, bc, ks, c.sigma, sd->xns,
                                      sd->rows, c.global_offset, sd->stride, h->cand_buf, h->gthr + c.max_batch, h->lists, st, &nl,
                                      &sl);
      if (ss != REMOE_OK)
        return fail(ss, "seed scan launch failed: %s", cudaGetErrorString(cudaGetLastError()));
      if ((int64_t)sl * ks < k) return fail(REMOE_ERR_STATE, "seed sample too small for k=%d", k);
      CUDA_TRY(remoe::launch_merge(h->lists, bc, sl, (int64_t)sl * ks, ks, k, h->seed_top, st, h->gthr, nullptr,
                                   nullptr, ks));
      ++nl;
    }
    const remoe_status_t ts =
        which == 3 ? remoe::tc_pair_scan(&h->tc, q, h->qnorm, bc, k, c.sigma, h->xnorm, c.n_local, c.global_offset,
                                         1, h->cand_buf, h->gthr, h->lists, st, &nl, &grid)
                   : remoe::tc_scan(&h->tc, q, h->qnorm, bc, k, c.sigma, h->xnorm, c.n_local, c.global_offset,
                                    1, h->cand_buf, h->gthr, h->lists, st, &nl, &grid, su.store ? &su : nullptr,
                                    fold_norms);
    if (ts != REMOE_OK)
      return fail(ts, "tensor-core scan launch failed: %s", cudaGetErrorString(cudaGetLastError()));
    *launches += nl;
  }
  CUDA_TRY(h->prof_mark(st, false));
  ++h->prof_launches;  // one S2+S3 phase per query chunk
  h->last_kernel = which;
  // ---- S4 (+ S5..S7 fused when world == 1).  gthr[b] holds a lower bound of the
  // final k-th best key (every published value is some state's own k-th best or a
  // seeded strict bound), so the merge drops every key below it.
  const cudaError_t me = remoe::launch_merge(h->lists, bc, grid, (int64_t)grid * k, k, k, h->local_top, st, nullptr,
                                             h->gthr, fin, -1, su.store ? h->seed_store.epoch : nullptr, true, px,
                                             h->split_cnt);
  if (me != cudaSuccess) {
    // nothing resets the thresholds / retires the published seed keys now: do it here, so a
    // later chunk starts clean
    cudaMemsetAsync(h->gthr, 0, (size_t)2 * c.max_batch * 8, st);
    if (su.store) {
      cudaMemsetAsync(h->seed_store.pub, 0, (size_t)c.max_batch * 2 * std::max(1, h->grid_tc) * 8, st);
      cudaMemsetAsync(h->seed_store.done, 0, (size_t)c.max_batch * 8, st);
    }
  }
  CUDA_TRY(me);
  ++*launches;
  return REMOE_OK;
}

// S5 + S6 + partial S7 (world > 1): merge the G gathered key lists into the global top-k
// (every rank runs the same merge on the same keys, so every rank writes the same ids and
// scores), softmax weights, and this rank's partial prediction from the winners it owns.
static remoe_status_t stage_merge(remoe_sps* h, int bc, int k, int64_t* ids, float* scores, bool want_pred,
                                  cudaStream_t st, int* launches) {
  const remoe_sps_config_t& c = h->cfg;
  const remoe::FinalizeArgs f{h->act, c.global_offset, c.n_local, 2, h->LE, c.temperature, ids, scores,
                              want_pred ? h->part : nullptr};
  CUDA_TRY(remoe::launch_merge(h->gathered, bc, c.world, k, (int64_t)bc * k, k, h->global_top, st, nullptr,
                               nullptr, &f, -1, nullptr, false, nullptr, h->split_cnt));
  ++*launches;
  return REMOE_OK;
}

// Exchange-2 layout: all-gather of whole partials while world * B * LE * 4 <= xchg_ag_max.
static bool xchg_allgather(const remoe_sps* h, int bc) {
  const size_t n = (size_t)h->cfg.world * bc * h->LE;
  return n * 4 <= h->xchg_ag_max && n <= h->part_all_floats;
}

// S7 combine: pred = sum of the G partials in rank order.  All-gather layout: the whole
// batch; all-to-all layout: this rank's query slice (broadcast afterwards).
static remoe_status_t stage_combine(remoe_sps* h, int bc, float* pred, cudaStream_t st, int* launches) {
  const int G = h->cfg.world;
  const int64_t LE = h->LE;
  if (xchg_allgather(h, bc)) {
    CUDA_TRY(remoe::launch_psum(h->part_all, G, (int64_t)bc * LE, (int64_t)bc * LE, pred, st));
  } else {
    int lo, cnt;
    slice_of(bc, G, h->cfg.rank, &lo, &cnt);
    const int cap = (bc + G - 1) / G;
    CUDA_TRY(remoe::launch_psum(h->part_all, G, (int64_t)cap * LE, (int64_t)cnt * LE, pred + (int64_t)lo * LE, st));
  }
  ++*launches;
  return REMOE_OK;
}

enum class Xchg { Keys, PartsAllGather, PartsAllToAll, SlicesBroadcast };

// One exchange step for the ranks in hs[0..nh): over NCCL (one handle of this process,
// nh == 1) or, for a loopback group (all world handles, nh == world), as device copies
// of exactly the bytes NCCL would move.
static remoe_status_t exchange(remoe_sps* const* hs, int nh, Xchg x, int bc, int k, float* const* pred,
                               cudaStream_t st) {
  remoe_sps* h0 = hs[0];
  const int G = h0->cfg.world;
  const int64_t LE = h0->LE;
  const int cap = (bc + G - 1) / G;
  if (h0->comm) {
    remoe_sps* h = h0;
    switch (x) {
      case Xchg::Keys:
        NCCL_TRY(ncclAllGather(h->local_top, h->gathered, (size_t)bc * k, ncclUint64, h->comm, st));
        break;
      case Xchg::PartsAllGather:
        NCCL_TRY(ncclAllGather(h->part, h->part_all, (size_t)bc * LE, ncclFloat, h->comm, st));
        break;
      case Xchg::PartsAllToAll: {
        int lo_me, cnt_me;
        slice_of(bc, G, h->cfg.rank, &lo_me, &cnt_me);
        NCCL_TRY(ncclGroupStart());
        for (int g = 0; g < G; ++g) {
          int lo, cnt;
          slice_of(bc, G, g, &lo, &cnt);
          if (cnt > 0) NCCL_TRY(ncclSend(h->part + (size_t)lo * LE, (size_t)cnt * LE, ncclFloat, g, h->comm, st));
          if (cnt_me > 0)
            NCCL_TRY(ncclRecv(h->part_all + (size_t)g * cap * LE, (size_t)cnt_me * LE, ncclFloat, g, h->comm, st));
        }
        NCCL_TRY(ncclGroupEnd());
        break;
      }
      case Xchg::SlicesBroadcast:
        NCCL_TRY(ncclGroupStart());
        for (int g = 0; g < G; ++g) {
          int lo, cnt;
          slice_of(bc, G, g, &lo, &cnt);
          if (cnt > 0)
            NCCL_TRY(ncclBroadcast(pred[0] + (size_t)lo * LE, pred[0] + (size_t)lo * LE, (size_t)cnt * LE, ncclFloat,
                                   g, h->comm, st));
        }
        NCCL_TRY(ncclGroupEnd());
        break;
    }
    return REMOE_OK;
  }
  if (nh != G) return fail(REMOE_ERR_STATE, "loopback exchange needs all %d ranks", G);
  const cudaMemcpyKind dd = cudaMemcpyDeviceToDevice;
  for (int m = 0; m < G; ++m) {
    remoe_sps* hm = hs[m];
    for (int p = 0; p < G; ++p) {
      const remoe_sps* hp = hs[p];
      switch (x) {
        case Xchg::Keys:
          CUDA_TRY(cudaMemcpyAsync(hm->gathered + (size_t)p * bc * k, hp->local_top, (size_t)bc * k * 8, dd, st));
          break;
        case Xchg::PartsAllGather:
          CUDA_TRY(cudaMemcpyAsync(hm->part_all + (size_t)p * bc * LE, hp->part, (size_t)bc * LE * 4, dd, st));
          break;
        case Xchg::PartsAllToAll: {
          int lo, cnt;
          slice_of(bc, G, m, &lo, &cnt);  // rank m receives its slice from every rank p
          if (cnt > 0)
            CUDA_TRY(cudaMemcpyAsync(hm->part_all + (size_t)p * cap * LE, hp->part + (size_t)lo * LE,
                                     (size_t)cnt * LE * 4, dd, st));
          break;
        }
        case Xchg::SlicesBroadcast: {
          int lo, cnt;
          slice_of(bc, G, p, &lo, &cnt);  // rank p's finished slice to rank m
          if (p != m && cnt > 0)
            CUDA_TRY(cudaMemcpyAsync(pred[m] + (size_t)lo * LE, pred[p] + (size_t)lo * LE, (size_t)cnt * LE * 4, dd, st));
          break;
        }
      }
    }
  }
  return REMOE_OK;
}

// Fused exchange (h->fused): the PeerXchg of each producing kernel.  Exchange 1:
// the S4 merge stores the local keys into every rank's gathered[par][rank]; exchange 2
// (all-gather layout): the S5 merge stores the partial rows into every rank's
// part_all[par][rank]; each raises this rank's flag in every rank.  The chunk's sequence
// number (and with it the parity par) is read on the device from d_xseq and advanced by
// k_seq_bump after the chunk, so the whole sequence can be captured once in a CUDA graph.
static size_t gathered_par_stride(const remoe_sps* h) {
  return (size_t)h->cfg.world * h->cfg.max_batch * h->cfg.max_k;
}
static remoe::PeerXchg fused_keys(const remoe_sps* h, int bc, int k) {
  remoe::PeerXchg px{};
  px.G = h->cfg.world;
  for (int g = 0; g < px.G; ++g) {
    px.key_dst[g] = h->p_gathered[g] + (size_t)h->cfg.rank * bc * k;  // parity 0 (key_par: parity 1)
    px.flag_dst[g] = h->p_xflag[g] + h->cfg.rank;                     // exchange-1 flags: [0, G)
  }
  px.counter = h->xcount;
  px.seq_ptr = h->d_xseq;
  px.key_par = (int64_t)gathered_par_stride(h);
  return px;
}
static remoe_status_t stage_merge_fused(remoe_sps* h, int bc, int k, int64_t* ids, float* scores, bool want_pred,
                                        bool ag, cudaStream_t st, int* launches) {
  const remoe_sps_config_t& c = h->cfg;
  remoe::FinalizeArgs f{h->act, c.global_offset, c.n_local, 2, h->LE, c.temperature, ids, scores,
                        want_pred ? h->part : nullptr};
  remoe::PeerXchg px{};
  px.G = c.world;
  px.wait_flags = h->xflag;  // every rank's exchange-1 flag
  px.seq_ptr = h->d_xseq;
  px.in_par = (int64_t)gathered_par_stride(h);
  if (want_pred && ag) {
    f.n_pred_peer = c.world;
    for (int g = 0; g < c.world; ++g) {
      f.pred_peer[g] = h->p_part_all[g] + (size_t)c.rank * bc * h->LE;  // parity 0 (pred_par: parity 1)
      px.flag_dst[g] = h->p_xflag[g] + c.world + c.rank;                 // exchange-2 flags: [G, 2G)
    }
    px.counter = h->xcount + 1;
    px.pred_par = (int64_t)h->part_all_floats;
  }
  CUDA_TRY(remoe::launch_merge(h->gathered, bc, c.world, k, (int64_t)bc * k, k, h->global_top, st, nullptr, nullptr,
                               &f, -1, nullptr, false, &px));
  ++*launches;
  return REMOE_OK;
}

// The multi-rank pipeline for the handles in hs[0..nh) (NCCL: this process's handle;
// loopback: every rank of the group).  local(h, px) runs S1-S4 (or the tree search) into
// h->local_top -- and, fused, into every rank's receive buffer (px); then exchange 1,
// S5-S7 and exchange 2.  ids/scores/pred are per handle.  `fusable`: the local stage
// honours px (the brute-force scan; the tree search does not).
template <class LocalStage>
static remoe_status_t query_ranks(remoe_sps* const* hs, int nh, int bc, int k, int64_t* const* ids,
                                  float* const* scores, float* const* pred, cudaStream_t st, int* launches,
                                  LocalStage&& local, bool fusable) {
  const bool want = pred != nullptr && pred[0] != nullptr;
  const bool ag = xchg_allgather(hs[0], bc);
  if (fusable && hs[0]->fused) {
    auto bump = [&]() -> remoe_status_t {  // the chunk is over on this rank: advance its sequence
      for (int i = 0; i < nh; ++i) {
        CUDA_TRY(remoe::launch_seq_bump(hs[i]->d_xseq, st));
        ++*launches;
      }
      return REMOE_OK;
    };
    for (int i = 0; i < nh; ++i) {
      const remoe::PeerXchg px = fused_keys(hs[i], bc, k);
      ST_TRY(local(hs[i], &px));
    }
    for (int i = 0; i < nh; ++i) ST_TRY(stage_merge_fused(hs[i], bc, k, ids[i], scores[i], want, ag, st, launches));
    if (!want) return bump();
    if (ag) {
      for (int i = 0; i < nh; ++i) {
        remoe_sps* h = hs[i];
        CUDA_TRY(remoe::launch_psum(h->part_all, h->cfg.world, (int64_t)bc * h->LE, (int64_t)bc * h->LE, pred[i], st,
                                    h->xflag + h->cfg.world, 0, h->d_xseq, (int64_t)h->part_all_floats));
        ++*launches;
      }
      return bump();
    }
    // all-to-all layout: the partials (h->part) go through the collectives below
    ST_TRY(bump());
  } else {
    for (int i = 0; i < nh; ++i) ST_TRY(local(hs[i], nullptr));
    ST_TRY(exchange(hs, nh, Xchg::Keys, bc, k, pred, st));
    for (int i = 0; i < nh; ++i) ST_TRY(stage_merge(hs[i], bc, k, ids[i], scores[i], want, st, launches));
    if (!want) return REMOE_OK;
  }
  ST_TRY(exchange(hs, nh, ag ? Xchg::PartsAllGather : Xchg::PartsAllToAll, bc, k, pred, st));
  for (int i = 0; i < nh; ++i) ST_TRY(stage_combine(hs[i], bc, pred[i], st, launches));
  if (!ag) ST_TRY(exchange(hs, nh, Xchg::SlicesBroadcast, bc, k, pred, st));
  return REMOE_OK;
}

static remoe_status_t query_chunk(remoe_sps* h, const uint16_t* q, int bc, int k, int64_t* ids,
                                  float* scores, float* pred, cudaStream_t st, int* launches) {
  const remoe_sps_config_t& c = h->cfg;
  if (c.world == 1) {
    const remoe::FinalizeArgs fin{h->act, c.global_offset, c.n_local, 0, h->LE, c.temperature, ids, scores, pred};
    return stage_scan(h, q, bc, k, &fin, st, launches);
  }
  remoe_sps* hs[1] = {h};
  return query_ranks(
      hs, 1, bc, k, &ids, &scores, &pred, st, launches,
      [&](remoe_sps* hh, const remoe::PeerXchg* px) { return stage_scan(hh, q, bc, k, nullptr, st, launches, px); },
      true);
}

static bool aligned(const void* p, size_t a) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) % a) == 0; }

static remoe_status_t check_query(remoe_sps* h, const uint16_t* q, int32_t B, int32_t k,
                                  const int64_t* ids, const float* scores, const float* pred,
                                  bool device_bufs = true) {
  if (!h) return fail(REMOE_ERR_STATE, "handle is NULL");
  if (B < 0) return fail(REMOE_ERR_INVALID_ARG, "B must be >= 0");
  if (k < 1) return fail(REMOE_ERR_INVALID_ARG, "k must be >= 1");
  if (k > h->cfg.max_k) return fail(REMOE_ERR_INVALID_ARG, "k=%d exceeds max_k=%d", k, h->cfg.max_k);
  if (k > h->n_total)
    return fail(REMOE_ERR_INVALID_ARG, "k=%d exceeds the history size %lld (SPEC S:227)", k,
                (long long)h->n_total);
  if (B > 0 && (!q || !ids || !scores)) return fail(REMOE_ERR_INVALID_ARG, "q/ids/scores is NULL");
  // the kernels read q with 16-byte vector loads / cp.async and write pred with float4 stores
  if (device_bufs && (!aligned(q, 16) || !aligned(pred, 16) || !aligned(ids, 8) || !aligned(scores, 4)))
    return fail(REMOE_ERR_INVALID_ARG, "misaligned buffer: q and pred need 16 bytes, ids 8, scores 4");
  return REMOE_OK;
}

// The device-buffer query of one chunk through a cached CUDA graph: captured once per
// (buffers, B, k, kernel choice) on the library stream, replayed as one launch on the
// caller's stream.
static remoe_status_t query_device_graph(remoe_sps* h, const uint16_t* q, int B, int k, int64_t* ids,
                                         float* scores, float* pred, cudaStream_t caller) {
  if (!h->gst) {
    CUDA_TRY(cudaStreamCreateWithFlags(&h->gst, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&h->gev, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&h->gev_done, cudaEventDisableTiming));
  }
  remoe_sps::DevGraph* g = nullptr;
  for (auto& e : h->dg)
    if (e.exec && e.q == q && e.ids == ids && e.scores == scores && e.pred == pred && e.B == B && e.k == k &&
        e.kernel == h->force_kernel) { g = &e; break; }
  const cudaStream_t st = h->gst;  // capture only (nothing runs during a capture)
  if (!g) {
    g = &h->dg[0];
    for (auto& e : h->dg)
      if (e.used < g->used) g = &e;  // least recently used (or empty) slot
    g->reset();
    CUDA_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
    int launches = 0;
    const remoe_status_t qs = query_chunk(h, q, B, k, ids, scores, pred, st, &launches);
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(st, &graph);
    if (qs != REMOE_OK || ce != cudaSuccess || !graph) {
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();
      if (qs != REMOE_OK) return qs;
      return fail(REMOE_ERR_CUDA, "graph capture failed: %s", cudaGetErrorString(ce));
    }
    const cudaError_t ie = cudaGraphInstantiate(&g->exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) {
      g->reset();
      return fail(REMOE_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(ie));
    }
    g->q = q; g->ids = ids; g->scores = scores; g->pred = pred;
    g->B = B; g->k = k; g->kernel = h->force_kernel; g->launches = launches;
    g->scan_kernel = h->last_kernel;
  }
  g->used = ++h->dg_clock;
  // replayed on the caller's stream itself: ordered with its earlier and later work without
  // the two cross-stream events per query of a launch on a library stream
  CUDA_TRY(cudaGraphLaunch(g->exec, caller));
  h->last_launches = g->launches;
  h->last_kernel = g->scan_kernel;
  return REMOE_OK;
}

extern "C" {

remoe_status_t remoe_sps_query(remoe_sps_t h, const uint16_t* q, int32_t B, int32_t k,
                               int64_t* ids, float* scores, float* pred, void* stream) {
  if (h && h->group) return fail(REMOE_ERR_STATE, "a loopback group member is queried with remoe_sps_query_group");
  ST_TRY(check_query(h, q, B, k, ids, scores, pred));
  if (B == 0) return REMOE_OK;
  DeviceGuard dg(h->cfg.device);
  NvtxRange nr("remoe_sps_query");
  cudaStream_t st = (cudaStream_t)stream;
  const int mb = h->cfg.max_batch;
  // one GPU, or world > 1 with the fused exchange in the all-gather layout (every step of
  // the chunk is then a kernel of this library -- no NCCL call -- and graph-capturable)
  const bool graphable = h->cfg.world == 1 || (h->fused && !h->group && (!pred || xchg_allgather(h, B)));
  if (B <= mb && graphable && !h->prof && h->use_graphs)
    return query_device_graph(h, q, B, k, ids, scores, pred, st);
  int launches = 0;
  for (int b0 = 0; b0 < B; b0 += mb) {
    const int bc = std::min(mb, B - b0);
    ST_TRY(query_chunk(h, q + (size_t)b0 * h->cfg.dim, bc, k, ids + (size_t)b0 * k,
                       scores + (size_t)b0 * k, pred ? pred + (size_t)b0 * h->LE : nullptr, st,
                       &launches));
  }
  h->last_launches = launches;
  return REMOE_OK;
}

// Loopback group query (test harness of the multi-rank path on one device).
remoe_status_t remoe_sps_query_group(remoe_group_t g, const uint16_t* q, int32_t B, int32_t k,
                                     int64_t* const* ids, float* const* scores, float* const* pred, void* stream) {
  if (!g) return fail(REMOE_ERR_STATE, "group is NULL");
  const int G = g->world;
  if (!ids || !scores) return fail(REMOE_ERR_INVALID_ARG, "ids/scores arrays are NULL");
  for (int r = 0; r < G; ++r)
    if (!g->members[r]) return fail(REMOE_ERR_STATE, "rank %d of the loopback group is not built", r);
  remoe_sps* const* hs = g->members.data();
  const int dev = hs[0]->cfg.device;
  int64_t expect = 0;
  for (int r = 0; r < G; ++r) {
    const remoe_sps_config_t& c = hs[r]->cfg;
    if (c.device != dev) return fail(REMOE_ERR_STATE, "loopback ranks must share one device");
    if (c.global_offset != expect)
      return fail(REMOE_ERR_INVALID_ARG, "shards do not tile [0, N): rank %d offset %lld, expected %lld", r,
                  (long long)c.global_offset, (long long)expect);
    expect += c.n_local;
    if (c.dim != hs[0]->cfg.dim || hs[r]->LE != hs[0]->LE || c.max_batch != hs[0]->cfg.max_batch)
      return fail(REMOE_ERR_INVALID_ARG, "loopback ranks differ in dim, table shape or max_batch");
  }
  for (int r = 0; r < G; ++r) hs[r]->n_total = expect;
  ST_TRY(setup_peers_loopback(hs, G));
  const bool want = pred != nullptr && pred[0] != nullptr;
  for (int r = 0; r < G; ++r) {
    ST_TRY(check_query(hs[r], q, B, k, ids[r], scores[r], want ? pred[r] : nullptr));
    if (want && !pred[r]) return fail(REMOE_ERR_INVALID_ARG, "pred must be given for every rank or none");
  }
  if (B == 0) return REMOE_OK;
  DeviceGuard dgd(dev);
  cudaStream_t st = (cudaStream_t)stream;
  const int mb = hs[0]->cfg.max_batch;
  const int64_t LE = hs[0]->LE;
  int launches = 0;
  if (B <= mb && hs[0]->fused && (!want || xchg_allgather(hs[0], B)) && hs[0]->use_graphs && !hs[0]->prof) {
    // the whole G-rank sequence as one cached CUDA graph (captured on the group's stream,
    // replayed on the caller's)
    if (!g->gst) {
      CUDA_TRY(cudaStreamCreateWithFlags(&g->gst, cudaStreamNonBlocking));
      CUDA_TRY(cudaEventCreateWithFlags(&g->gev, cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&g->gev_done, cudaEventDisableTiming));
    }
    std::vector<const void*> bufs;
    for (int r = 0; r < G; ++r) {
      bufs.push_back(ids[r]);
      bufs.push_back(scores[r]);
      bufs.push_back(want ? pred[r] : nullptr);
    }
    remoe_group::Graph* gr = nullptr;
    for (auto& e : g->graphs)
      if (e.exec && e.q == q && e.B == B && e.k == k && e.bufs == bufs) { gr = &e; break; }
    if (!gr) {
      if (g->graphs.size() >= 8) g->reset_graphs();
      g->graphs.emplace_back();
      gr = &g->graphs.back();
      CUDA_TRY(cudaStreamBeginCapture(g->gst, cudaStreamCaptureModeRelaxed));
      int nl = 0;
      std::vector<float*> pc(G);
      for (int r = 0; r < G; ++r) pc[r] = want ? pred[r] : nullptr;
      const remoe_status_t qs = query_ranks(
          hs, G, B, k, ids, scores, want ? pc.data() : nullptr, g->gst, &nl,
          [&](remoe_sps* hh, const remoe::PeerXchg* px) { return stage_scan(hh, q, B, k, nullptr, g->gst, &nl, px); },
          true);
      cudaGraph_t graph = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(g->gst, &graph);
      if (qs != REMOE_OK || ce != cudaSuccess || !graph) {
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();
        g->graphs.pop_back();
        if (qs != REMOE_OK) return qs;
        return fail(REMOE_ERR_CUDA, "group graph capture failed: %s", cudaGetErrorString(ce));
      }
      const cudaError_t ie = cudaGraphInstantiate(&gr->exec, graph, 0);
      cudaGraphDestroy(graph);
      if (ie != cudaSuccess) {
        g->graphs.pop_back();
        return fail(REMOE_ERR_CUDA, "group graph instantiate: %s", cudaGetErrorString(ie));
      }
      gr->q = q; gr->bufs = bufs; gr->B = B; gr->k = k; gr->launches = nl;
    }
    CUDA_TRY(cudaGraphLaunch(gr->exec, st));  // on the caller's stream (captured on the group's)
    for (int r = 0; r < G; ++r) hs[r]->last_launches = gr->launches;
    return REMOE_OK;
  }
  std::vector<int64_t*> ic(G);
  std::vector<float*> sc(G), pc(G);
  for (int b0 = 0; b0 < B; b0 += mb) {
    const int bc = std::min(mb, B - b0);
    for (int r = 0; r < G; ++r) {
      ic[r] = ids[r] + (size_t)b0 * k;
      sc[r] = scores[r] + (size_t)b0 * k;
      pc[r] = want ? pred[r] + (size_t)b0 * LE : nullptr;
    }
    const uint16_t* qc = q + (size_t)b0 * hs[0]->cfg.dim;
    ST_TRY(query_ranks(
        hs, G, bc, k, ic.data(), sc.data(), want ? pc.data() : nullptr, st, &launches,
        [&](remoe_sps* hh, const remoe::PeerXchg* px) { return stage_scan(hh, qc, bc, k, nullptr, st, &launches, px); },
        true));
  }
  for (int r = 0; r < G; ++r) hs[r]->last_launches = launches;
  return REMOE_OK;
}

static bool is_pinned(const void* p) {
  if (!p) return true;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return a.type == cudaMemoryTypeHost;
}

// One batch (B <= max_batch, world == 1) through the cached CUDA graph; captured on the
// first call of a (B, k, pred) shape.  Returns UNSUPPORTED (nothing enqueued) when a host
// buffer is pageable, which stream capture cannot copy from.
static remoe_status_t query_host_graph(remoe_sps* h, const uint16_t* q, int B, int k, int64_t* ids,
                                       float* scores, float* pred, cudaStream_t st) {
  if (!is_pinned(q) || !is_pinned(ids) || !is_pinned(scores) || !is_pinned(pred)) return REMOE_ERR_UNSUPPORTED;
  const size_t qb = (size_t)B * h->cfg.dim * 2, ib = (size_t)B * k * 8, sb = (size_t)B * k * 4,
               pb = (size_t)B * h->LE * 4;
  auto& g = h->hg;
  const cudaStream_t caller = st;
  if (!h->gst) {
    CUDA_TRY(cudaStreamCreateWithFlags(&h->gst, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&h->gev, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&h->gev_done, cudaEventDisableTiming));
  }
  st = h->gst;  // capture only; the graph is replayed on the caller's stream
  if (!(g.exec && g.B == B && g.k == k && g.pred == (pred != nullptr))) {
    g.reset();
    CUDA_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
    int launches = 0;
    cudaMemcpyAsync(h->hq, q, qb, cudaMemcpyHostToDevice, st);
    const remoe_status_t qs = query_chunk(h, h->hq, B, k, h->hids, h->hscores, pred ? h->hpred : nullptr, st,
                                          &launches);
    cudaMemcpyAsync(ids, h->hids, ib, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(scores, h->hscores, sb, cudaMemcpyDeviceToHost, st);
    if (pred) cudaMemcpyAsync(pred, h->hpred, pb, cudaMemcpyDeviceToHost, st);
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(st, &graph);
    if (qs != REMOE_OK || ce != cudaSuccess || !graph) {
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();
      if (qs != REMOE_OK) return qs;
      return fail(REMOE_ERR_CUDA, "graph capture failed: %s", cudaGetErrorString(ce));
    }
    g.graph = graph;
    size_t n = 0;
    CUDA_TRY(cudaGraphGetNodes(graph, nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n);
    CUDA_TRY(cudaGraphGetNodes(graph, nodes.data(), &n));
    for (cudaGraphNode_t nd : nodes) {
      cudaGraphNodeType ty;
      if (cudaGraphNodeGetType(nd, &ty) != cudaSuccess || ty != cudaGraphNodeTypeMemcpy) continue;
      cudaMemcpy3DParms mp{};
      if (cudaGraphMemcpyNodeGetParams(nd, &mp) != cudaSuccess) continue;
      if (mp.dstPtr.ptr == h->hq) g.h2d = nd;
      else if (mp.srcPtr.ptr == h->hids) g.d2h_ids = nd;
      else if (mp.srcPtr.ptr == h->hscores) g.d2h_sc = nd;
      else if (mp.srcPtr.ptr == h->hpred) g.d2h_pred = nd;
    }
    if (!g.h2d || !g.d2h_ids || !g.d2h_sc || (pred && !g.d2h_pred)) {
      g.reset();
      return fail(REMOE_ERR_CUDA, "graph capture: copy nodes not found");
    }
    CUDA_TRY(cudaGraphInstantiate(&g.exec, graph, 0));
    g.B = B; g.k = k; g.pred = pred != nullptr; g.launches = launches;
  }
  CUDA_TRY(cudaGraphExecMemcpyNodeSetParams1D(g.exec, g.h2d, h->hq, q, qb, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaGraphExecMemcpyNodeSetParams1D(g.exec, g.d2h_ids, ids, h->hids, ib, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaGraphExecMemcpyNodeSetParams1D(g.exec, g.d2h_sc, scores, h->hscores, sb, cudaMemcpyDeviceToHost));
  if (pred)
    CUDA_TRY(cudaGraphExecMemcpyNodeSetParams1D(g.exec, g.d2h_pred, pred, h->hpred, pb, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaGraphLaunch(g.exec, caller));  // after the caller's earlier work on the handle
  CUDA_TRY(cudaStreamSynchronize(caller));
  h->last_launches = g.launches;
  return REMOE_OK;
}

remoe_status_t remoe_sps_query_host(remoe_sps_t h, const uint16_t* q, int32_t B, int32_t k,
                                    int64_t* ids, float* scores, float* pred, void* stream) {
  if (!h) return fail(REMOE_ERR_STATE, "handle is NULL");
  if (h->group) return fail(REMOE_ERR_STATE, "a loopback group member is queried with remoe_sps_query_group");
  ST_TRY(check_query(h, q, B, k, ids, scores, pred, false));  // host buffers: staged, any alignment
  if (B == 0) return REMOE_OK;
  DeviceGuard dg(h->cfg.device);
  NvtxRange nr("remoe_sps_query_host");
  cudaStream_t st = (cudaStream_t)stream;
  const int mb = h->cfg.max_batch;
  const int D = h->cfg.dim;
  int launches = 0;
  const bool graphable = h->cfg.world == 1 || (h->fused && !h->group && (!pred || xchg_allgather(h, B)));
  if (B <= mb && graphable && !h->prof && h->use_graphs) {
    remoe_status_t gs = query_host_graph(h, q, B, k, ids, scores, pred, st);
    if (gs != REMOE_ERR_UNSUPPORTED) return gs;  // UNSUPPORTED: pageable buffers -> direct path
  }
  for (int b0 = 0; b0 < B; b0 += mb) {
    const int bc = std::min(mb, B - b0);
    CUDA_TRY(cudaMemcpyAsync(h->hq, q + (size_t)b0 * D, (size_t)bc * D * 2, cudaMemcpyHostToDevice, st));
    ST_TRY(query_chunk(h, h->hq, bc, k, h->hids, h->hscores, pred ? h->hpred : nullptr, st, &launches));
    CUDA_TRY(cudaMemcpyAsync(ids + (size_t)b0 * k, h->hids, (size_t)bc * k * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(scores + (size_t)b0 * k, h->hscores, (size_t)bc * k * 4, cudaMemcpyDeviceToHost, st));
    if (pred)
      CUDA_TRY(cudaMemcpyAsync(pred + (size_t)b0 * h->LE, h->hpred, (size_t)bc * h->LE * 4,
                               cudaMemcpyDeviceToHost, st));
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  h->last_launches = launches;
  return REMOE_OK;
}

// ---------------------------------------------------------------- NEXT-N2 clustering tree
remoe_status_t remoe_sps_tree_build(remoe_sps_t h, int32_t beta, int32_t branching, int32_t max_iter,
                                    uint64_t seed) {
  if (!h) return fail(REMOE_ERR_STATE, "handle is NULL");
  if (beta < 1) return fail(REMOE_ERR_INVALID_ARG, "beta must be >= 1");
  if (branching < 2 || branching > remoe::kTreeCMax)
    return fail(REMOE_ERR_INVALID_ARG, "branching must be in [2, %d]", remoe::kTreeCMax);
  if (max_iter < 0) return fail(REMOE_ERR_INVALID_ARG, "max_iter must be >= 0");
  if ((int64_t)beta + h->cfg.max_k - 1 > remoe::kTreeCandCap)
    return fail(REMOE_ERR_UNSUPPORTED, "beta + max_k - 1 = %lld exceeds %d candidates per query",
                (long long)beta + h->cfg.max_k - 1, remoe::kTreeCandCap);
  DeviceGuard dg(h->cfg.device);
  cudaStream_t st = nullptr;
  CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  remoe::Tree t;
  std::string err;
  const remoe_status_t s = remoe::tree_build(h->x, h->cfg.n_local, h->cfg.dim, beta, branching, max_iter, seed,
                                             st, &t, &err);
  cudaStreamDestroy(st);
  if (s != REMOE_OK) return fail(s, "tree build: %s", err.c_str());
  if (h->has_tree) remoe::tree_free(&h->tree);
  h->tree = std::move(t);
  h->has_tree = true;
  return REMOE_OK;
}

remoe_status_t remoe_sps_tree_info(remoe_sps_t h, remoe_sps_tree_info_t* info) {
  if (!h) return fail(REMOE_ERR_STATE, "handle is NULL");
  if (!info) return fail(REMOE_ERR_INVALID_ARG, "info is NULL");
  if (!h->has_tree) return fail(REMOE_ERR_STATE, "no tree: call remoe_sps_tree_build first");
  const remoe::Tree& t = h->tree;
  info->n_nodes = t.n_nodes;
  info->n_leaves = t.n_leaves;
  info->depth = t.depth;
  info->max_leaf = t.max_leaf;
  info->beta = t.beta;
  info->branching = t.branching;
  info->build_ms = t.build_ms;
  return REMOE_OK;
}

remoe_status_t remoe_sps_tree_export(remoe_sps_t h, int64_t* perm, int64_t* begin, int64_t* end, int32_t* parent,
                                     int32_t* child0, int32_t* nchild, int64_t* medoid) {
  if (!h) return fail(REMOE_ERR_STATE, "handle is NULL");
  if (!h->has_tree) return fail(REMOE_ERR_STATE, "no tree: call remoe_sps_tree_build first");
  const remoe::Tree& t = h->tree;
  DeviceGuard dg(h->cfg.device);
  if (perm) CUDA_TRY(cudaMemcpy(perm, t.perm, (size_t)h->cfg.n_local * 8, cudaMemcpyDeviceToHost));
  auto cp = [&](auto* dst, const auto& src) { if (dst) std::copy(src.begin(), src.end(), dst); };
  cp(begin, t.h_begin);
  cp(end, t.h_end);
  cp(parent, t.h_parent);
  cp(child0, t.h_child0);
  cp(nchild, t.h_nchild);
  cp(medoid, t.h_medoid);
  return REMOE_OK;
}

remoe_status_t remoe_sps_tree_query(remoe_sps_t h, const uint16_t* q, int32_t B, int32_t k, int64_t* ids,
                                    float* scores, float* pred, int32_t* leaf, int32_t* n_eval, void* stream) {
  ST_TRY(check_query(h, q, B, k, ids, scores, pred));
  if (!h->has_tree) return fail(REMOE_ERR_STATE, "no tree: call remoe_sps_tree_build first");
  if (h->group) return fail(REMOE_ERR_UNSUPPORTED, "tree queries over a loopback group");
  if (B == 0) return REMOE_OK;
  DeviceGuard dg(h->cfg.device);
  NvtxRange nr("remoe_sps_tree_query");
  cudaStream_t st = (cudaStream_t)stream;
  const remoe_sps_config_t& c = h->cfg;
  const int mb = c.max_batch;
  int launches = 0;
  for (int b0 = 0; b0 < B; b0 += mb) {
    const int bc = std::min(mb, B - b0);
    const uint16_t* qc = q + (size_t)b0 * c.dim;
    int64_t* ic = ids + (size_t)b0 * k;
    float* sc = scores + (size_t)b0 * k;
    float* pc = pred ? pred + (size_t)b0 * h->LE : nullptr;
    auto local = [&](remoe_sps* hh, const remoe::PeerXchg*) -> remoe_status_t {
      CUDA_TRY(remoe::launch_norms(qc, bc, c.dim, hh->qnorm, st));
      CUDA_TRY(remoe::launch_tree_search(hh->tree, hh->x, hh->xnorm, c.dim, qc, hh->qnorm, bc, k, c.sigma,
                                         c.global_offset, hh->local_top, leaf ? leaf + b0 : nullptr,
                                         n_eval ? n_eval + b0 : nullptr, st));
      launches += 2;
      return REMOE_OK;
    };
    if (c.world == 1) {
      ST_TRY(local(h, nullptr));
      const remoe::FinalizeArgs f{h->act, c.global_offset, c.n_local, 0, h->LE, c.temperature, ic, sc, pc};
      CUDA_TRY(remoe::launch_finalize(h->local_top, bc, k, f, st));
      ++launches;
    } else {
      remoe_sps* hs[1] = {h};
      ST_TRY(query_ranks(hs, 1, bc, k, &ic, &sc, &pc, st, &launches, local, false));
    }
  }
  h->last_launches = launches;
  return REMOE_OK;
}

remoe_status_t remoe_expert_plan(const float* pred, int32_t B, int32_t L, int32_t E, int32_t n_cold,
                                 uint8_t* cold_mask, void* stream) {
  if (B < 0 || L < 1 || E < 1) return fail(REMOE_ERR_INVALID_ARG, "need B >= 0, L >= 1, E >= 1");
  if (E > 256) return fail(REMOE_ERR_UNSUPPORTED, "E > 256");
  if (n_cold < 0 || n_cold > E) return fail(REMOE_ERR_INVALID_ARG, "need 0 <= n_cold <= E");
  if (B == 0) return REMOE_OK;
  if (!pred || !cold_mask) return fail(REMOE_ERR_INVALID_ARG, "pred/cold_mask is NULL");
  CUDA_TRY(remoe::launch_plan(pred, B, L, E, n_cold, cold_mask, (cudaStream_t)stream));
  return REMOE_OK;
}

remoe_status_t remoe_sps_embed(const uint16_t* tokens_bf16, const int64_t* offsets, int32_t n_prompts,
                               int32_t dim, uint16_t* out_bf16, float* out_f32, void* stream) {
  if (n_prompts < 0) return fail(REMOE_ERR_INVALID_ARG, "n_prompts must be >= 0");
  if (dim < 8 || dim % 8 != 0) return fail(REMOE_ERR_INVALID_ARG, "dim must be a positive multiple of 8");
  if (dim > 4096) return fail(REMOE_ERR_UNSUPPORTED, "dim > 4096");
  if (n_prompts == 0) return REMOE_OK;
  if (!offsets || (!out_bf16 && !out_f32)) return fail(REMOE_ERR_INVALID_ARG, "offsets/outputs are NULL");
  CUDA_TRY(remoe::launch_embed(tokens_bf16, offsets, n_prompts, dim, out_bf16, out_f32, (cudaStream_t)stream));
  return REMOE_OK;
}

remoe_status_t remoe_js_divergence(const float* P, const float* Q, int32_t shared_q, int32_t B, int32_t L,
                                   int32_t E, float* out, void* stream) {
  if (B < 0 || L < 1 || E < 1) return fail(REMOE_ERR_INVALID_ARG, "need B >= 0, L >= 1, E >= 1");
  if (B == 0) return REMOE_OK;
  if (!P || !Q || !out) return fail(REMOE_ERR_INVALID_ARG, "P/Q/out is NULL");
  if ((int64_t)L * 4 > 200 * 1024) return fail(REMOE_ERR_UNSUPPORTED, "L too large");
  CUDA_TRY(remoe::launch_js(P, Q, shared_q ? 0 : (int64_t)L * E, B, L, E, out, (cudaStream_t)stream));
  return REMOE_OK;
}

remoe_status_t remoe_sps_sync(remoe_sps_t h) {
  if (!h) return fail(REMOE_ERR_STATE, "handle is NULL");
  DeviceGuard dg(h->cfg.device);
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaGetLastError());
  if (h->comm) {
    ncclResult_t ar = ncclSuccess;
    NCCL_TRY(ncclCommGetAsyncError(h->comm, &ar));
    if (ar != ncclSuccess) return fail(REMOE_ERR_NCCL, "async NCCL error: %s", ncclGetErrorString(ar));
  }
  return REMOE_OK;
}

remoe_status_t remoe_sps_get_info(remoe_sps_t h, remoe_sps_info_t* info) {
  if (!h) return fail(REMOE_ERR_STATE, "handle is NULL");
  if (!info) return fail(REMOE_ERR_INVALID_ARG, "info is NULL");
  info->n_total = h->n_total;
  info->n_local = h->cfg.n_local;
  info->global_offset = h->cfg.global_offset;
  info->dim = h->cfg.dim;
  info->n_layers = h->cfg.n_layers;
  info->n_experts = h->cfg.n_experts;
  info->rank = h->cfg.rank;
  info->world = h->cfg.world;
  info->last_scan_kernel = h->last_kernel;
  info->last_launches = h->last_launches;
  info->scan_ctas = h->last_kernel >= 2 ? h->grid_tc : h->grid_simt;
  info->device_bytes = (int64_t)h->device_bytes;
  info->fused_exchange = h->fused ? 1 : 0;
  return REMOE_OK;
}

remoe_status_t remoe_sps_set_kernel(remoe_sps_t h, int32_t which) {
  if (!h) return fail(REMOE_ERR_STATE, "handle is NULL");
  if (which < 0 || which > 3) return fail(REMOE_ERR_INVALID_ARG, "which must be 0, 1, 2 or 3");
  if (which >= 2 && !h->tc.ok) return fail(REMOE_ERR_UNSUPPORTED, "tensor-core scan unavailable: %s", h->tc.why);
  if (which == 3 && !remoe::tc_pair_usable(&h->tc))
    return fail(REMOE_ERR_UNSUPPORTED, "CTA-pair tensor-core scan unavailable for this store");
  if (h->force_kernel != which) {
    DeviceGuard dg(h->cfg.device);
    h->hg.reset();  // the cached host-query graph baked in the previous kernel choice
  }
  h->force_kernel = which;
  return REMOE_OK;
}

remoe_status_t remoe_sps_profile(remoe_sps_t h, int32_t enable, double* scan_ms, int64_t* launches) {
  if (!h) return fail(REMOE_ERR_STATE, "handle is NULL");
  DeviceGuard dg(h->cfg.device);
  CUDA_TRY(h->prof_collect());
  if (scan_ms) *scan_ms = h->prof_ms;
  if (launches) *launches = h->prof_launches;
  h->prof_ms = 0.0;
  h->prof_launches = 0;
  h->prof = enable != 0;
  return REMOE_OK;
}

void remoe_sps_destroy(remoe_sps_t h) {
  if (!h) return;
  {
    DeviceGuard dg(h->cfg.device);
    cudaDeviceSynchronize();
    h->release();
  }
  delete h;
}

}  // extern "C"
