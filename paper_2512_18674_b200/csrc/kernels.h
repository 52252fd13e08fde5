// kernels.h -- launch interface of the SPS device kernels (internal to libremoe).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace remoe {

// S2+S3, streaming (CUDA-core) variant.  Scores nq <= BQ queries against rows
// [0, n_rows) of the shard; writes per-CTA sorted top-k key lists to
// out[(query * grid + cta) * k + i] (zero padded).
struct SimtScanParams {
  const uint16_t* x;      // [n_rows][dim] bf16
  const float* xnorm;     // [n_rows]
  int64_t n_rows;
  int64_t gid_offset;     // global id of row 0
  int dim;
  const uint16_t* q;      // [nq][dim] bf16
  const float* qnorm;     // [nq]
  int nq;
  int k;
  float sigma;
  int stage_rows;         // rows per TMA stage
  int n_stages_ring;      // ring depth
  uint64_t* cand_buf;     // [grid][32][CAP] private lane buffers
  unsigned long long* gthr;  // [nq] shared per-query thresholds (zeroed by launch_norms)
  uint64_t* out;          // [nq][grid][k]
};
size_t simt_smem_bytes(int BQ, int dim, int stage_rows, int n_stages_ring);
constexpr int kSimtMaxSmem = 232448;  // opt-in dynamic shared memory per CTA (227 KB)
cudaError_t launch_scan_simt(const SimtScanParams& p, int BQ, int grid, cudaStream_t st);

// S2+S3, tensor-core (tcgen05) variant; see k_scan_tc.cu.

// S1 / S0: L2 norms of bf16 rows (fp32, fixed order).  If zero_u64 is non-null,
// zero_u64[row] = 0 as well (resets the per-query shared thresholds for free).
cudaError_t launch_norms(const uint16_t* x, int64_t n, int dim, float* out, cudaStream_t st,
                         unsigned long long* zero_u64 = nullptr, int64_t zero_stride = 0);

// S6 + S7 arguments.  mode 0: every winner's row comes from the local table
// act[(gid - offset) * LE] (one GPU: this rank holds every row).  mode 2 (multi-GPU
// partial prediction): only the winners this rank owns (offset <= gid < offset + n_local)
// contribute, in r-ascending order; the others are skipped, so pred receives this rank's
// partial P_g = sum over owned r of w_r S~_{id_r} (SURVEY §8(e) exchange 2).
constexpr int kMaxPeers = 8;  // ranks of one NVLink/NVSwitch node
struct FinalizeArgs {
  const float* act;
  int64_t offset;
  int64_t n_local;
  int mode;
  int64_t LE;
  float T;
  int64_t* ids;
  float* scores;
  float* pred;  // may be null: ids and scores only
  // fused exchange 2 (PeerXchg): the rows go to pred_peer[g] + b * LE for every rank g
  // instead of pred (pred stays non-null: "a prediction is wanted")
  int n_pred_peer;
  float* pred_peer[kMaxPeers];
};

// Fused peer-memory exchange (world > 1, REMOE_FUSED_COMM=1): the producing
// kernel stores its outputs straight into every rank's receive buffer (peer pointers:
// CUDA IPC over NVLink between processes, plain device pointers in a loopback group), and
// its last CTA raises this rank's flag in every rank to `seq` (release, system scope).  The
// consuming kernel first waits until every rank's flag is >= seq (acquire, bounded: a
// trap instead of a silent hang).  Receive buffers are double-buffered by seq parity.
struct PeerXchg {
  int G;                                     // ranks; 0 = off
  uint64_t* key_dst[kMaxPeers];              // S4 output: this rank's [B][k] slot in rank g
  unsigned long long* flag_dst[kMaxPeers];   // this rank's flag in rank g (null: no signal)
  unsigned* counter;                         // finished CTAs (the last one signals, resets it)
  const unsigned long long* wait_flags;      // [G] flags to wait for before reading (or null)
  unsigned long long seq;                    // the chunk's sequence number (when seq_ptr is null)
  // Graph-replayable form: the chunk's sequence number is read on the device (*seq_ptr + 1;
  // k_seq_bump advances it after the chunk), and odd chunks use the parity-1 halves of the
  // double-buffered receive buffers: input lists at in + in_par, key_dst[g] + key_par,
  // the partial rows at fin.pred_peer[g] + pred_par.
  const unsigned long long* seq_ptr;
  int64_t in_par, key_par, pred_par;
};

// S4 / S5: per query, merge n_lists sorted key lists of length list_len (default k) into
// the best k.
// key(b, l, i) = in[b * qstride + l * lstride + i].  Keys below lower[b] (a known lower
// bound of the final k-th best key) are dropped.  If set_thr is non-null, also
// set_thr[b] = (k-th best key) - 1 (threshold seeding from a row sample).  If fin is
// non-null the same CTA then runs S6 + S7 for the query (fused finalize).  If bump is
// non-null, *bump += 1 once (after the previous kernel completed): the seeding epoch.
// reset_lower: lower[b] = 0 once read (the scan that follows starts from no threshold,
// without a k_norms launch to zero it).
cudaError_t launch_merge(const uint64_t* in, int B, int n_lists, int64_t qstride, int64_t lstride,
                         int k, uint64_t* out, cudaStream_t st, unsigned long long* set_thr = nullptr,
                         unsigned long long* lower = nullptr, const FinalizeArgs* fin = nullptr,
                         int list_len = -1, unsigned* bump = nullptr, bool reset_lower = false,
                         const PeerXchg* px = nullptr, unsigned* split_cnt = nullptr);
// (split_cnt: [B] zeroed counters; when given with a prediction to compute, the merge runs
// as (B, n_split) CTAs that split the finalize's columns -- see k_merge)

// S6 + S7 as a separate kernel (tree search path with world == 1).
cudaError_t launch_finalize(const uint64_t* top, int B, int k, const FinalizeArgs& f, cudaStream_t st);

// Multi-GPU S7 combine: out[i] = sum_{g = 0..G-1} parts[g * part_stride + i] for i < n, g
// ascending (a fixed order: every rank and every batch position gets the same bits).
// wait_flags (fused exchange 2): first wait until wait_flags[g] >= seq for every g < G;
// with seq_ptr, seq = *seq_ptr + 1 and odd chunks read parts + parts_par.
cudaError_t launch_psum(const float* parts, int G, int64_t part_stride, int64_t n, float* out, cudaStream_t st,
                        const unsigned long long* wait_flags = nullptr, unsigned long long seq = 0,
                        const unsigned long long* seq_ptr = nullptr, int64_t parts_par = 0);
// *seq += 1 (one thread): ends a fused-exchange chunk (graph-replayable sequence numbers).
cudaError_t launch_seq_bump(unsigned long long* seq, cudaStream_t st);

// S8: cold mask of the n_cold smallest entries per (query, layer).
cudaError_t launch_plan(const float* pred, int B, int L, int E, int n_cold, uint8_t* mask,
                        cudaStream_t st);

// NEXT-N1: prompt vectors a_p = sum_t x_t / |x_t| over the token rows [off[p], off[p+1]).
cudaError_t launch_embed(const uint16_t* tok, const int64_t* off, int n_prompts, int dim, uint16_t* out_bf16,
                         float* out_f32, cudaStream_t st);

// NEXT-N4: out[b] = mean over layers of JS_2(P[b][l], Q[b][l]); Q[b] = Q + b * q_stride
// (q_stride = 0: one reference matrix for every b).
cudaError_t launch_js(const float* P, const float* Q, int64_t q_stride, int B, int L, int E, float* out,
                      cudaStream_t st);

// Build-time validation: counts non-finite embeddings and bad activation rows.
cudaError_t launch_validate(const uint16_t* x, int64_t n, int dim, const float* act, int64_t LE_rows,
                            int E, unsigned long long* bad, cudaStream_t st);

}  // namespace remoe
