/*
 * remoe.h -- C ABI of the B200-native Similar Prompts Searching (SPS) predictor.
 *
 * Paper: "Remoe: Towards Efficient and Low-Cost MoE Inference in Serverless
 * Computing", arXiv 2512.18674.  Line citations "P:n" are PAPER.md
 * lines; "S:n" are SPEC.md lines; "DESIGN R<n>" are the readings listed in
 * DESIGN.md where the paper is silent or ambiguous.
 *
 * What the library computes (the data-parallel hot path):
 *
 *   score(q, x_j) = (q . x_j) / (|q| |x_j| + sigma)                     (S1-S2)
 *       Eq. 11.  The paper's SCS on token matrices equals the
 *       cosine of the summed L2-normalised token rows (DESIGN R2), so a
 *       "prompt embedding" here is that sum (or any positive rescaling).
 *   top-k over all stored prompts, ordered by score descending, then global
 *       id ascending (DESIGN R5)                                          (S3-S5)
 *       Exact brute force, the paper's "BF"; k is the paper's alpha.
 *   w_r = softmax(s_r / T) over the k retrieved scores                   (S6)
 *       P:421 "converted into probability weights via softmax" (T=1, DESIGN R4).
 *   P[l][e] = sum_r w_r * S~_{id_r}[l][e], r = 0..k-1 ascending           (S7)
 *       P:421 "weighted-summed to predict the result"; S~ rows are the
 *       "linear scaling activation frequencies" of P:420.
 *   cold[l][e] = 1 for the n_cold experts of layer l with the smallest P   (S8)
 *       P:504 remote-expert selection: u_{l,k} = N_in s~ + N_out N_topk s~
 *       is a positive multiple of s~, so argmin of sum u over |R_l| = b K_l
 *       picks the n_cold smallest s~ (ties: lower expert index, DESIGN R12).
 *
 * Precision: embeddings and queries are bf16; dot products accumulate in fp32
 * (tensor-core or FMA) in an order fixed per (query, row) and independent of
 * the query's batch position and of the sharding; norms, scores, weights and
 * predictions are fp32.  Selection is exact with respect to the fp32 scores
 * and the key order above.
 *
 * Conventions (all functions):
 *   - C linkage, no exception or abort crosses the boundary.
 *   - Argument errors are detected synchronously, before any launch, and
 *     return REMOE_ERR_INVALID_ARG (or REMOE_ERR_UNSUPPORTED for legal but
 *     unimplemented shapes); outputs are then untouched.
 *   - Device work is asynchronous on the caller's stream; asynchronous CUDA /
 *     NCCL faults surface at the next call or at remoe_sps_sync().
 *   - remoe_last_error() returns a thread-local description of the last failure.
 *   - A handle is not safe for concurrent calls from several threads.
 */
#ifndef REMOE_H_
#define REMOE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define REMOE_API __attribute__((visibility("default")))
#else
#define REMOE_API
#endif

typedef enum {
  REMOE_OK = 0,
  REMOE_ERR_INVALID_ARG = 1, /* bad pointer, size, shard tiling, k > N_total, ... */
  REMOE_ERR_CUDA = 2,        /* a CUDA runtime/driver call failed */
  REMOE_ERR_NCCL = 3,        /* an NCCL call failed (multi-GPU only) */
  REMOE_ERR_OOM = 4,         /* device allocation failed */
  REMOE_ERR_UNSUPPORTED = 5, /* legal but not implemented (e.g. k > 256, D > 4096) */
  REMOE_ERR_STATE = 6        /* handle misuse (NULL handle, destroyed, wrong device) */
} remoe_status_t;

typedef struct remoe_sps* remoe_sps_t; /* opaque, library-owned */
typedef struct remoe_group* remoe_group_t; /* opaque loopback group (see remoe_loopback_group_create) */

/*
 * Build configuration.  One per rank; the store is sharded row-wise into
 * contiguous ranges: rank g owns global rows [global_offset, global_offset +
 * n_local), and the ranges of ranks 0..world-1 must tile [0, N_total) in rank
 * order (checked at build when world > 1; INVALID_ARG otherwise).
 */
typedef struct {
  int64_t n_local;        /* rows on this rank (>= 1) */
  int64_t global_offset;  /* global id of this rank's first row */
  int32_t dim;            /* D: embedding dimension, D % 8 == 0, 8 <= D <= 4096 */
  int32_t n_layers;       /* L: MoE layers of the activation table (>= 1) */
  int32_t n_experts;      /* E: routed experts per layer, 1 <= E <= 256 */
  float sigma;            /* Eq. 11 guard sigma > 0; DESIGN R3 default 1e-6 */
  float temperature;      /* softmax temperature T > 0 (DESIGN R4 default 1) */
  int32_t max_batch;      /* workspace sizing: largest B per internal chunk (>= 1) */
  int32_t max_k;          /* largest k ever queried, 1 <= max_k <= 256 */
  int32_t device;         /* CUDA device ordinal this handle lives on */
  int32_t rank, world;    /* 0 <= rank < world; world == 1 => no NCCL */
  const void* nccl_unique_id; /* 128-byte ncclUniqueId identical on all ranks; NULL iff world == 1 */
  int32_t inputs_on_device;   /* 1: emb/act passed to build are device pointers on `device`; 0: host */
  int32_t validate;       /* 1: reject non-finite embeddings, act < 0, |row sum - 1| > 1e-3 */
  const void* loopback_group; /* world > 1 without NCCL: the remoe_group_t this rank joins (all
                                 ranks in this process, on one device; exchanges are device copies).
                                 NULL otherwise.  Exactly one of nccl_unique_id / loopback_group
                                 is non-NULL when world > 1. */
} remoe_sps_config_t;

/* Fill *cfg with defaults (sigma 1e-6, T 1, max_batch 256, max_k 128, world 1,
 * validate 1); the caller then sets n_local, dim, n_layers, n_experts, ... */
REMOE_API void remoe_sps_config_default(remoe_sps_config_t* cfg);

/*
 * S0: ingest this rank's shard of the history.
 *   emb_bf16: [n_local x dim] row-major bf16 bit patterns (prompt vectors,
 *             P:374-385).  Copied; the caller keeps ownership.
 *   act:      [n_local x L x E] fp32 row-stochastic per (prompt, layer) activation
 *             frequencies S~.  Copied; the caller keeps ownership.
 *   out:      receives the handle on success, NULL on failure.
 * Collective over `world` ranks (all ranks must call it).  Synchronous: returns
 * after the device copies and the |x_j| pass have completed.
 * Multi-rank builds agree on the outcome: once the NCCL communicator exists, every
 * rank contributes (offset, n_local, local status) to one all-gather, and if any rank
 * failed (bad shard, validation, OOM, ...) every rank returns an error (the failing
 * rank its own; the others that rank's status), so no rank is left blocked in a later
 * collective.  Shards must tile [0, N_total) in rank order and hold >= 1 row each
 * (the balanced split offset_g = floor(N g / G) does for N >= G).
 */
REMOE_API remoe_status_t remoe_sps_build(const remoe_sps_config_t* cfg, const uint16_t* emb_bf16,
                                         const float* act, remoe_sps_t* out);

/*
 * S1-S7: score B queries against the whole (sharded) store, return the global
 * top-k and the predicted activation matrix.
 *   q_bf16: device [B x dim] bf16 bits, identical on every rank (SPMD).
 *   B >= 0 (B == 0 is a no-op), 1 <= k <= min(N_total, max_k).  B > max_batch
 *   is processed in internal chunks of max_batch.
 *   ids:    device [B x k] int64 global ids, by score desc then id asc.
 *   scores: device [B x k] fp32 scores (Eq. 11).
 *   pred:   device [B x L x E] fp32 prediction, or NULL to skip S6-S7.
 *   stream: the caller's stream; all work is enqueued there.
 * Collective when world > 1: every rank must call with the same B, k and
 * queries, and every rank receives identical outputs.
 */
REMOE_API remoe_status_t remoe_sps_query(remoe_sps_t h, const uint16_t* q_bf16, int32_t B,
                                         int32_t k, int64_t* ids, float* scores, float* pred,
                                         void* stream);

/*
 * Alignment (checked synchronously, INVALID_ARG): q_bf16 and pred must be 16-byte
 * aligned (16-byte vector loads / cp.async of the query rows, float4 stores of the
 * prediction), ids 8 bytes, scores 4 bytes.
 *
 * Multi-rank data path (world > 1, "top-alpha" over all history):
 * each rank scans its shard (S1-S4); its B x k local keys are all-gathered; every rank
 * merges the G lists with the same deterministic merge (S5: identical ids and scores on
 * every rank); each rank then reduces only the winners it OWNS into a partial
 * P_g = sum over owned r of w_r S~_{id_r} ("reduction on the owning ranks",
 * BASELINE north_star); the partials are exchanged (all-gather of [G][B][L*E] while that
 * is <= 32 MiB, REMOE_XCHG_AG_MAX at build; otherwise an all-to-all of query slices plus
 * a broadcast of the finished slices) and summed in rank order g = 0..G-1, so every rank
 * and every batch position gets the same bits.  Versus world == 1 the ids and scores are
 * bit-identical; pred differs only by fp32 re-association (<= ~1e-7).
 */

/*
 * Same as remoe_sps_query, but q/ids/scores/pred are HOST buffers (pinned or
 * pageable).  Copies in, runs, copies out and synchronizes the stream before
 * returning.  This is the end-to-end entry point a serving front end calls.
 */
REMOE_API remoe_status_t remoe_sps_query_host(remoe_sps_t h, const uint16_t* q_bf16, int32_t B,
                                              int32_t k, int64_t* ids, float* scores, float* pred,
                                              void* stream);

/*
 * S8: remote-expert selection.  For each (query b, layer l), the n_cold
 * experts with the smallest pred[b][l][e] (ties -> lower e) get mask 1 (cold /
 * remote, x_{l,k} = 1), the rest 0 (hot / local).
 *   pred: device [B x L x E] fp32; cold_mask: device [B x L x E] uint8.
 *   0 <= n_cold <= E (n_cold = floor(b * E) for MMP's remote ratio b).
 * Stateless; no communication.
 */
REMOE_API remoe_status_t remoe_expert_plan(const float* pred, int32_t B, int32_t L, int32_t E,
                                           int32_t n_cold, uint8_t* cold_mask, void* stream);

/*
 * NEXT-N1, the Eq. 11 front end: turn the pre-processing layer's
 * token embeddings into the prompt vectors the store and the queries hold.  SCS
 * normalises every token row and sums the rows of a prompt (V1^T X with V1 the
 * ownership vector), so for prompt p with token rows [offsets[p], offsets[p+1]):
 *     a_p = sum_t x_t / |x_t|      (fp32; a zero token contributes 0, DESIGN R17)
 *   tokens_bf16: device [T x dim] bf16 bits, T = offsets[n_prompts];
 *   offsets:     device [n_prompts + 1] int64, non-decreasing, offsets[0] = 0;
 *   out_bf16:    device [n_prompts x dim] bf16 (round to nearest even), or NULL;
 *   out_f32:     device [n_prompts x dim] fp32, or NULL (at least one non-NULL).
 *   dim % 8 == 0, 8 <= dim <= 4096.  Stateless; async on `stream`.
 */
REMOE_API remoe_status_t remoe_sps_embed(const uint16_t* tokens_bf16, const int64_t* offsets,
                                         int32_t n_prompts, int32_t dim, uint16_t* out_bf16,
                                         float* out_f32, void* stream);

/*
 * NEXT-N4, prediction quality: the paper scores its predictor by the
 * Jensen-Shannon divergence between predicted and true expert-activation
 * distributions.  out[b] = (1/L) sum_l JS_2(P[b][l][:], Q[b][l][:]), log base 2 (so
 * 0 <= JS <= 1, DESIGN R18), 0 log 0 = 0.
 *   P: device [B x L x E] fp32 (e.g. remoe_sps_query's pred);
 *   Q: device [B x L x E] fp32, or one [L x E] matrix for every b if shared_q != 0;
 *   out: device [B] fp32.  Rows are expected to be distributions (not checked).
 */
REMOE_API remoe_status_t remoe_js_divergence(const float* P, const float* Q, int32_t shared_q,
                                             int32_t B, int32_t L, int32_t E, float* out, void* stream);

/*
 * NEXT-N2, the clustering-tree SPS (Algorithm 1) -- the paper's
 * approximate search, next to the exact brute force of remoe_sps_query.
 *
 * remoe_sps_tree_build: builds the multi-fork clustering tree over this handle's store
 * shard: every node with more than beta prompts is split by k-medoids with
 * similarity 1 - cos (DESIGN R25), roulette-wheel centroid initialisation (R24, draws
 * from a counter-based generator keyed by seed, node, draw) and subcluster-level
 * centroid updates (at most max_iter updates per node; 0 keeps the initial draw).
 * 2 <= branching <= 16, beta >= 1, beta + max_k - 1 <= 2048 (candidates per query),
 * depth <= 63.  Synchronous; replaces a previous tree; runs on the GPU (fp64).
 * Collective-free: with world > 1 every rank builds the tree of its own shard.
 */
REMOE_API remoe_status_t remoe_sps_tree_build(remoe_sps_t h, int32_t beta, int32_t branching, int32_t max_iter,
                                              uint64_t seed);

typedef struct {
  int32_t n_nodes, n_leaves, depth, max_leaf, beta, branching;
  double build_ms;           /* host wall time of remoe_sps_tree_build */
} remoe_sps_tree_info_t;
REMOE_API remoe_status_t remoe_sps_tree_info(remoe_sps_t h, remoe_sps_tree_info_t* info);

/* Copies the tree to HOST buffers (each may be NULL): perm [n_local] local rows, node i
 * owns perm[begin[i], end[i]); children child0[i] .. child0[i] + nchild[i] - 1 (nodes
 * numbered breadth-first, root 0, parent[0] = -1); medoid[i] = local row of node i's
 * centroid (-1 for the root).  Node arrays have remoe_sps_tree_info().n_nodes entries. */
REMOE_API remoe_status_t remoe_sps_tree_export(remoe_sps_t h, int64_t* perm, int64_t* begin, int64_t* end,
                                               int32_t* parent, int32_t* child0, int32_t* nchild,
                                               int64_t* medoid);

/*
 * Algorithm 1 for B queries (same buffers and semantics as remoe_sps_query): descend by
 * the child centroid with the best Eq. 11 key, take the leaf's prompts, supplement from
 * sibling subtrees (best first, each explored depth-first in key order, whole leaves,
 * climbing a level when the siblings run out) until >= k candidates (R28), return the
 * exact top-k of the candidates by key, then the same
 * softmax-weighted prediction (S6+S7).  leaf [B] (the leaf the descent reached) and
 * n_eval [B] (Eq. 11 evaluations: centroids + candidates) are device outputs or NULL;
 * with world > 1 they describe the local tree and the k winners are merged across ranks
 * exactly as in remoe_sps_query.  REMOE_ERR_STATE before remoe_sps_tree_build.
 */
REMOE_API remoe_status_t remoe_sps_tree_query(remoe_sps_t h, const uint16_t* q_bf16, int32_t B, int32_t k,
                                              int64_t* ids, float* scores, float* pred, int32_t* leaf,
                                              int32_t* n_eval, void* stream);

/*
 * Loopback groups: the multi-rank path (S5 exchange + merge, the owner-side partial S7
 * and its exchange) run inside ONE process on ONE device, for testing and for emulating
 * a G-GPU partition on one GPU.  remoe_loopback_group_create makes an empty group of
 * `world` ranks; each rank's handle is built with remoe_sps_build (cfg.world = world,
 * cfg.rank, cfg.loopback_group = the group, nccl_unique_id = NULL); the exchanges are
 * device-to-device copies of exactly the bytes the NCCL collectives would move.
 * remoe_loopback_group_destroy returns REMOE_ERR_STATE while handles are still built.
 *
 * Fused exchange (environment REMOE_FUSED_COMM=1 at build, world <= 8):
 * instead of collectives, the merge kernels store their outputs (local top-k keys,
 * exchange 1; partial predictions, exchange 2 in the all-gather layout) straight into
 * every rank's receive buffer and raise a per-rank flag; the consuming kernels wait on
 * the flags (bounded: a trap after 120 s instead of a silent hang).  Between NCCL ranks
 * the receive buffers are mapped through CUDA IPC (NVLink peer access on one node; the
 * ranks agree at build, and all fall back to NCCL if any cannot map its peers); in a
 * loopback group they are the members' own buffers.  remoe_sps_get_info reports which
 * path a handle uses (fused_exchange).  The chunk sequence numbers live on the device, so
 * fused multi-rank queries (all-gather layout, B <= max_batch) are captured once as a CUDA
 * graph per buffer set and replayed, like one-GPU queries; loopback group queries too.
 */
REMOE_API remoe_status_t remoe_loopback_group_create(int32_t world, remoe_group_t* out);
REMOE_API remoe_status_t remoe_loopback_group_destroy(remoe_group_t g);

/*
 * remoe_sps_query for every rank of a loopback group at once: ids[r], scores[r], pred[r]
 * are rank r's device output buffers (the same shapes as remoe_sps_query; pred NULL, or
 * an array of `world` buffers).  Every rank's outputs are written; they are identical.
 * REMOE_ERR_STATE if a rank is missing; INVALID_ARG if the shards do not tile [0, N).
 * remoe_sps_query on a group member returns REMOE_ERR_STATE.
 */
REMOE_API remoe_status_t remoe_sps_query_group(remoe_group_t g, const uint16_t* q_bf16, int32_t B, int32_t k,
                                               int64_t* const* ids, float* const* scores, float* const* pred,
                                               void* stream);

/* Rank 0 calls this, then broadcasts the 128 bytes to all ranks (e.g. as a uint8
 * tensor over a torch.distributed group) before remoe_sps_build. */
REMOE_API remoe_status_t remoe_nccl_unique_id(uint8_t out[128]);

/* Synchronize the handle's device work and surface asynchronous CUDA/NCCL errors. */
REMOE_API remoe_status_t remoe_sps_sync(remoe_sps_t h);

/* Introspection: N_total, the kernel the last query used, and workspace bytes. */
typedef struct {
  int64_t n_total, n_local, global_offset;
  int32_t dim, n_layers, n_experts, rank, world;
  int32_t last_scan_kernel;   /* 0 none, 1 streaming (CUDA cores), 2 tensor core (tcgen05, resident
                                 query slab), 3 tensor core on CTA pairs (tcgen05 cta_group::2) */
  int32_t last_launches;      /* kernels launched by the last query (all chunks) */
  int32_t scan_ctas;          /* grid of the scan kernel */
  int64_t device_bytes;       /* store + table + workspaces */
  int32_t fused_exchange;     /* 1: world > 1 exchanges run as peer-memory stores fused into the
                                 merge kernels (REMOE_FUSED_COMM=1 at build, every rank agreed);
                                 0: NCCL collectives (or device copies in a loopback group) */
  int32_t reserved_;
} remoe_sps_info_t;
REMOE_API remoe_status_t remoe_sps_get_info(remoe_sps_t h, remoe_sps_info_t* info);

/* Force the scan kernel: 0 auto (default), 1 streaming, 2 tensor core (resident query slab),
 * 3 tensor core on CTA pairs (the large-batch GEMM tiling).  Auto picks 3 for batches of
 * at least 128 queries -- on a shard of >= 16 x 256 rows per SM already for any batch past
 * one resident slab (65 at D = 1024) -- (REMOE_PAIR_MIN_B overrides), else 2 (above
 * D = 1280 the resident slab holds fewer queries -- 48 at D = 1536, 40 at 2048, 16 at
 * 4096 -- and larger batches take several slabs; D % 64 != 0 zero-pads the last K-block).
 * 1 runs only when forced.
 * Also settable with the environment variable REMOE_FORCE_KERNEL=stream|tc|pair.
 * INVALID_ARG for other values, UNSUPPORTED when the kernel cannot serve this store. */
REMOE_API remoe_status_t remoe_sps_set_kernel(remoe_sps_t h, int32_t which);

/*
 * Live kernel timing for benchmarks.  enable = 1 starts recording CUDA events on
 * the query stream around the S2+S3 phase of every query chunk (the scan kernel
 * launches of that chunk, including the threshold-seeding scan when it runs); each
 * call returns (after synchronizing those events) the accumulated phase time in ms
 * and the number of phases since the previous call, then resets them.
 * enable = 0 stops recording.  scan_ms / launches may be NULL.
 */
REMOE_API remoe_status_t remoe_sps_profile(remoe_sps_t h, int32_t enable, double* scan_ms,
                                           int64_t* launches);

/* Collective when world > 1.  NULL-safe. */
REMOE_API void remoe_sps_destroy(remoe_sps_t h);

REMOE_API const char* remoe_status_string(remoe_status_t s);
REMOE_API const char* remoe_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* REMOE_H_ */
