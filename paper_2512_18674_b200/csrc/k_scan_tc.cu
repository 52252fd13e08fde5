// k_scan_tc.cu -- S2+S3 on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// score_ij = (q_i . x_j) / (|q_i||x_j| + sigma)  (Eq. 11, DESIGN R2),
// exact per-CTA running top-k per query (BF top-alpha).
//
// Shape (DESIGN.md §7 "k_scan_tc"): D[q, j] = sum_k Q[q, k] X[j, k], a bf16 x bf16 -> fp32
// contraction with M = queries (64, or 128 when D <= 576), N = 256 store rows per scan
// unit (two consecutive 128-row tiles of the tiled copy: half the MMA instructions per
// store byte of N = 128, whose issue loop co-limited the stream), K = D.  Both operands
// are K-major.  One persistent CTA per SM, 11 warps:
//   * The query slab (A) is written into shared memory ONCE per CTA in the 128-byte-
//     swizzled K-major layout and stays resident (only the 8-row atoms a single slab needs;
//     max_qps rows when D > 1536): the only HBM stream is the store itself.  The query
//     norms (S1) are computed from it in the prologue.
//   * Warp 0: producer.  The build-time tiled copy of the store (16 KB boxes already in the
//     UMMA layout) streams through an NST-deep ring of 32 KB stages (a unit's K-block: its
//     two tiles' boxes back to back) with 1-D cp.async.bulk (multicast across a cluster of
//     query slabs); seeding sample units come first.
//   * Warp 1: one thread issues tcgen05.mma.cta_group::1.kind::f16 (4 per K-block) into one
//     of two TMEM accumulators (256 fp32 columns each), bulk-copies the unit's x-norms next
//     to it, and tcgen05.commit's the smem slot / the finished accumulator to mbarriers.
//   * Warps 2-9: epilogue, one thread per (query, tile parity).  tcgen05.ld.32x32b.x32 gives
//     thread (quarter w, lane t) its query's dots for 32 consecutive store rows (8 chunks
//     per unit); a branch-free
//     conservative prefilter against the state's threshold, exact keys and inserts only for
//     the rare candidates (RegTopk for k <= 32, LaneTopk buffers above; common.cuh).
//   * Warp 10: threshold seeding (the r-th largest published sample key per query, a strict
//     lower bound of the final k-th best), then the broker that mirrors the shared global
//     thresholds into shared memory for the epilogue.
// The dot for (q, row) accumulates K-blocks in ascending order inside the tensor core;
// it does not depend on the query's batch position, on M, or on the sharding.
#include <cuda.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <type_traits>
#include <vector>

#include "common.cuh"

#include "host_util.h"
#include "kernels.h"
#include "tc_host.h"
#include "tcgen05.cuh"

namespace remoe {

namespace {
constexpr int kTileN = 128;          // store rows per tile of the tiled copy (k_tile_store)
constexpr int kUnitN = 256;          // store rows per scan unit = UMMA N: two consecutive tiles
constexpr int kBlockK = 64;          // bf16 elements per 128-byte swizzle row
constexpr int kTileBytes = kTileN * kBlockK * 2;   // 16 KB: one tile's K-block
constexpr int kStageBytes = kUnitN * kBlockK * 2;  // 32 KB: one unit's K-block (its two tiles' boxes)
constexpr int kThreads = 352;        // 11 warps: TMA, MMA, 8 epilogue, seeding
constexpr int kSeedWarp = 10;        // computes the seeded thresholds (idle without seeding)
constexpr int kEpiWarps = 8;
constexpr int kAcc = 2;              // TMEM accumulator stages (256 fp32 columns each)
constexpr int kTmemCols = kAcc * kUnitN;
constexpr int kMaxSmem = 232448;     // 227 KB opt-in
constexpr int kTraceSlots = 32;     // REMOE_TC_TRACE stamps per CTA
constexpr int kMaxStages = 4;        // stage ring depth cap: 4 x 32 KB measured best (6: -3..7%, 3: -2%, 2: -12%)

struct TcArgs {
  const float* xnorm;
  int64_t n_rows;
  int64_t gid_offset;
  int dim;
  const uint16_t* q;
  const float* qnorm;
  int nq;
  int k;
  float sigma;
  int n_stages;
  uint64_t* cand_buf;
  unsigned long long* gthr;  // [nq] shared thresholds (zeroed before the launch)
  uint64_t* out;
  int smem_bufs;  // candidate buffers in shared memory (else cand_buf in global memory)
  int64_t gid_stride;      // global id of row r = gid_offset + r * gid_stride (seed samples: stride)
  int merge_in_cta;        // register top-k: merge the two parity states into one list per CTA
  int cluster;             // CTAs per cluster along y (multicast of the store tiles), 1 = none
  int epi_sleep;           // epilogue waits with a suspend-time hint (REMOE_EPI_SLEEP=1)
  const uint16_t* xt;      // tiled store (TcPlan::xt): 1-D bulk copies, else the tensor map
  int dbg;                 // REMOE_TC_DBG bits (experiments only; 1 = skip the MMA)
  int slab_rows;           // query rows stored per K-block (multiple of 8, <= M): a single
                           // slab of nq queries stores only ceil(nq/8) 8-row atoms
  int qps;                 // queries per slab (M, or fewer when D is too large for an M-row
                           // slab: D > 1536 keeps qps rows resident, the MMA still runs M)
  unsigned long long* trace;  // REMOE_TC_TRACE: [grid][16] globaltimer stamps
  unsigned long long* stats;  // REMOE_TC_STATS: [0] candidate columns, [1] inserts, [2] chunks with a candidate
  // ---- in-kernel threshold seeding (DESIGN.md §7 "threshold seeding"): each CTA first
  // scans its share of the sample tiles (a tiled copy of every s-th store row, TcSeed)
  // with a small register tracker per state and publishes the state's h-th best sample
  // key, tagged with this launch's epoch; the seeding warp of CTA c then waits for every
  // state's key of the queries m = c (mod grid.x) and raises their shared thresholds to
  // (the r-th largest published key) - 1, r * h >= k: at least k real keys of the store
  // are >= that key, so it is a lower bound of the final k-th best (strict after -1).
  // The epilogue never waits for it: the thresholds are read again every tile.
  const uint16_t* seed_xt;   // tiled sample (nullptr: no seeding)
  const float* seed_xn;      // sample norms [n units * 256]
  int seed_n_stiles;         // sample units scanned (a prefix of the segments)
  int seed_nseg;
  int seed_t0[5];            // first sample unit of segment g (seed_t0[nseg] = total)
  int64_t seed_count[4];     // rows of segment g: store rows off + i * stride, i < count
  int64_t seed_off[4];
  int64_t seed_stride[4];
  int seed_h, seed_r;
  uint64_t* seed_pub;        // [nq][2 * gridDim.x] published words: (h-th key >> 32) << 32 | epoch
  uint64_t* seed_done;       // [nq] the query's seed word: (threshold score word) << 32 | epoch
  const unsigned* seed_epoch;  // the epoch of this query chunk (bumped by its merge kernel)
  long long seed_wait_ns;    // how long the seeding warp waits for all keys (then: the subset)
  int norms_in_kernel;       // S1 in the prologue (no k_norms launch; qnorm unused)
};
}  // namespace

// M = queries per pass (UMMA M, 64 or 128).  For M = 64 the accumulator rows live in
// lanes 0-15 of each 32-lane TMEM quarter (row r -> lane 32*(r/16) + r%16); slab row m
// holds query m, so query m is read by the epilogue warps of quarter m/16 (a batch of
// <= 16 uses quarter 0's two warps: the epilogue is busy ~25% of the stream time at c3 --
// REMOE_TC_TRACE -- and spreading the queries would need the full 64-row slab).
#define TRACE(idx)                                                                              \
  do {                                                                                          \
    if (p.trace && (threadIdx.x & 31) == 0) {                                                   \
      unsigned long long t_;                                                                    \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                    \
      p.trace[(blockIdx.y * gridDim.x + blockIdx.x) * kTraceSlots + (idx)] = t_;                         \
    }                                                                                           \
  } while (0)

template <int M, int P, int KR>
__global__ void __launch_bounds__(kThreads, 1)
    k_scan_tc(const __grid_constant__ CUtensorMap tmap_x, TcArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int D = p.dim;
  const int nkb = (D + kBlockK - 1) / kBlockK;  // the last K-block is zero-padded when D % 64 != 0
  const int NST = p.n_stages;
  uint8_t* sA = smem;                                   // [nkb][M rows][128 B] swizzled
  const int SR = p.slab_rows;
  uint8_t* sB = sA + (size_t)nkb * SR * 128;            // [NST][128 rows][128 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + (size_t)NST * kStageBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + NST;
  uint64_t* tfull = bars + 2 * NST;
  uint64_t* tempty = bars + 2 * NST + kAcc;
  uint64_t* cempty = bars + 2 * NST + 2 * kAcc;  // [NST] cluster-wide "slot free" (leader CTA)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * NST + 2 * kAcc);
  volatile unsigned& s_epoch = *reinterpret_cast<unsigned*>(bars + 3 * NST + 2 * kAcc + 1);  // free slot before sXn
  unsigned* s_epi_done = reinterpret_cast<unsigned*>(bars + 3 * NST + 2 * kAcc + 1) + 1;  // epilogue warps finished
  // [kAcc][256] x-norms of the unit in accumulator acc: bulk-copied by the MMA warp with the
  // unit (completing on tfull[acc]), so the epilogue never waits on a global load for them
  float* sXn = reinterpret_cast<float*>(bars + ((3 * NST + 2 * kAcc + 2 + 1) & ~1));
  // [M] per-query threshold shared by the two parity states of the CTA (register top-k)
  unsigned long long* pair_thr = reinterpret_cast<unsigned long long*>(sXn + kAcc * kUnitN);  // [M]
  float* sQn = reinterpret_cast<float*>(pair_thr + M);  // [M] query norms (p.norms_in_kernel)
  uint64_t* sBuf = reinterpret_cast<uint64_t*>(sQn + M);  // [256][CAP] if p.smem_bufs

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t n_tiles = (p.n_rows + kTileN - 1) / kTileN;  // 128-row tiles of the tiled copy
  const int64_t n_units = (p.n_rows + kUnitN - 1) / kUnitN;  // 256-row scan units (tiles 2u, 2u + 1)
  // This CTA's unit sequence: its sample units (threshold seeding) first, then its store
  // units; the TMA producer, the MMA issuer and the epilogue walk the same sequence.
  const bool seeding = p.seed_xt != nullptr;
  // Store unit u goes to CTA u mod grid, so the first n_units mod grid CTAs hold one unit
  // more; sample unit j goes to CTA (n_units + j) mod grid, i.e. to the others first, which
  // evens the CTAs' total work (c3: 28 -> 27 units on the busiest CTAs).  (REMOE_TC_DBG bit
  // 512, experiment: sample unit j on CTA j.)
  const int G = (int)gridDim.x;
  const int srot = (p.dbg & 512) ? 0 : (int)(n_units % G);
  const int sidx = ((int)blockIdx.x - srot + G) % G;  // this CTA's first sample unit
  const int64_t ns_cta = (seeding && p.seed_n_stiles > sidx) ? (p.seed_n_stiles - 1 - sidx) / G + 1 : 0;
  const int64_t n_it = ns_cta + (n_units - 1 - (int64_t)blockIdx.x) / G + 1;  // grid.x <= n_units
  auto tile_of = [&](int64_t i) -> int64_t {
    return i < ns_cta ? (int64_t)sidx + i * G : (int64_t)blockIdx.x + (i - ns_cta) * G;
  };
  TRACE(0);
  if (p.trace && threadIdx.x == 0) p.trace[(blockIdx.y * gridDim.x + blockIdx.x) * kTraceSlots + 11] = clock64();
  pdl_trigger();  // the merge kernel may be scheduled as SMs free up
  // Query slab of this CTA (blockIdx.y).  With several slabs, the CTAs of every slab walk
  // the store tiles in the same order (tile = blockIdx.x + j * gridDim.x), so the slabs
  // read each tile at about the same time: HBM once, the other slabs hit L2.
  const int slab = blockIdx.y;
  const int QS = p.qps;
  const int nq = min(QS, p.nq - slab * QS);
  const uint16_t* qsl = p.q + (size_t)slab * QS * D;
  const float* qnorm_sl = p.qnorm + slab * QS;
  unsigned long long* gthr_sl = p.gthr + slab * QS;
  const int lists_per_cta = p.merge_in_cta ? 1 : 2;
  uint64_t* out_sl = p.out + (size_t)slab * QS * gridDim.x * lists_per_cta * p.k;
  const size_t cta_lin = (size_t)blockIdx.y * gridDim.x + blockIdx.x;

  // Cluster of C = p.cluster CTAs along y (consecutive slabs, same tile sequence): the
  // leader (rank 0) multicasts every store tile into all C CTAs' shared memory, so one
  // L2 read feeds C query slabs.  Every CTA's MMA commit frees the slot in its own ring
  // (empty: pacing its expect_tx) and in the leader's (cempty, count C: pacing the load).
  const int C = p.cluster;
  uint32_t crank = 0;
  if (C > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));

  // ---- one-time setup: barriers, TMEM, the resident query slab
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&cempty[s], C);
    }
    // tfull: the x-norm copy's arrive.expect_tx + the accumulator commit
    for (int s = 0; s < kAcc; ++s) { mbar_init(&tfull[s], 2); mbar_init(&tempty[s], 4); }
    for (int s = 0; s < M; ++s) pair_thr[s] = 0ull;
    *s_epi_done = 0;
    if (seeding) s_epoch = *reinterpret_cast<const volatile unsigned*>(p.seed_epoch);
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_x) : "memory");
  }
  if (C > 1) {  // every CTA's barriers exist before any peer multicasts or arrives
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  TRACE(1);
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (warp != 0) {
    // Warps 1-9 write the resident query slab while warp 0 already streams the store:
    // Q[m][kb*64 + c*8 .. +8] -> sA + kb*SR*128 + m*128 + ((c ^ (m & 7)) * 16)  (SWIZZLE_128B).
    // With SR < M the UMMA's rows SR .. M-1 read past the K-block (other K-blocks or the
    // stage ring): garbage accumulator rows of queries >= nq, which no lane reads.
    const int cpk = nkb * 8;  // 16-byte chunks per slab row, K-padding included
    const int chunks = SR * cpk;
    const uint32_t a_s = smem_u32(sA);
    for (int i = threadIdx.x - 32; i < chunks; i += blockDim.x - 32) {
      const int m = i / cpk;  // slab row = query
      const int cc = i - m * cpk;
      const int kb = cc >> 3, c = cc & 7;
      const uint32_t dst = a_s + (uint32_t)(kb * SR * 128 + m * 128 + ((c ^ (m & 7)) << 4));
      const bool real = m < nq && cc < (D >> 3);
      const uint16_t* src = qsl + (size_t)(real ? m : 0) * D + (real ? cc * 8 : 0);
      const uint32_t bytes = real ? 16u : 0u;  // src-size 0 -> zero fill (padding rows / columns)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes)
                   : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("bar.sync 1, %0;" ::"n"(kThreads - 32) : "memory");  // warps 1-10 only
    TRACE(2);
  }
  if (p.norms_in_kernel && warp >= 2 && warp < 2 + kEpiWarps) {
    // S1 from the resident slab: |q_m| = sqrt(sum_d q_md^2), one warp per query in the
    // k_norms order (lane partial sums over 16-byte chunks cc = lane, lane + 32, ...;
    // fixed xor butterfly), so the bits equal launch_norms' on every CTA and position
    for (int mm = warp - 2; mm < nq; mm += kEpiWarps) {
      float acc2 = 0.f;
      for (int cc = lane; cc < (D >> 3); cc += 32) {
        const int kb = cc >> 3, c = cc & 7;
        const uint4 w = lds128(sA + (size_t)kb * SR * 128 + mm * 128 + ((c ^ (mm & 7)) << 4));
        const float vv[8] = {bf_lo(w.x), bf_hi(w.x), bf_lo(w.y), bf_hi(w.y),
                             bf_lo(w.z), bf_hi(w.z), bf_lo(w.w), bf_hi(w.w)};
#pragma unroll
        for (int u = 0; u < 8; ++u) acc2 = __fmaf_rn(vv[u], vv[u], acc2);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc2 += __shfl_xor_sync(kFull, acc2, off);
      if (lane == 0) sQn[mm] = __fsqrt_rn(acc2);
    }
    asm volatile("bar.sync 11, %0;" ::"n"(kEpiWarps * 32) : "memory");  // the epilogue warps
  }

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    // The whole warp walks the loop (warp-uniform control flow keeps the loop state in
    // uniform registers); lane 0 issues the copies.
    int s = 0;
    uint32_t ph = 0;
    for (int64_t i = 0; i < n_it; ++i) {
      const bool smp = i < ns_cta;
      const int64_t u = tile_of(i);
      // tiled store / sample: box (tile, kb) is 16 KB contiguous in HBM, already in the
      // swizzled UMMA layout, so 1-D bulk copies stream it (no 128 B-per-row DRAM pattern).
      // Unit u's K-block kb = the boxes (2u, kb) and (2u + 1, kb) back to back: one 256-row
      // B operand (the sample is padded to whole units; the store's last unit may hold one tile)
      const uint16_t* tsrc = smp ? p.seed_xt + (size_t)(2 * u) * nkb * (kTileBytes / 2)
                                 : p.xt ? p.xt + (size_t)(2 * u) * nkb * (kTileBytes / 2) : nullptr;
      const bool two = smp || 2 * u + 1 < n_tiles;
      const size_t second = (size_t)nkb * (kTileBytes / 2);  // tile 2u + 1 in the tiled copy
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&empty[s], ph ^ 1u);  // this CTA's MMA is done with the slot
        if (lane == 0) {
          if (p.dbg & 32) {  // debug (REMOE_TC_DBG bit 32): no load, the slot is "full" at once (wrong results)
            mbar_arrive(&full[s]);
          } else {
            uint8_t* dst = sB + (size_t)s * kStageBytes;
            mbar_arrive_expect_tx(&full[s], two ? kStageBytes : kTileBytes);
            const uint16_t* src = tsrc ? tsrc + (size_t)kb * (kTileBytes / 2) : nullptr;
            const int r0 = (int)(u * kUnitN);
            if (C == 1) {
              if (src) {
                bulk_g2s(dst, src, kTileBytes, &full[s]);
                if (two) bulk_g2s(dst + kTileBytes, src + second, kTileBytes, &full[s]);
              } else {
                tma_load_2d(dst, &tmap_x, kb * kBlockK, r0, &full[s]);
                if (two) tma_load_2d(dst + kTileBytes, &tmap_x, kb * kBlockK, r0 + kTileN, &full[s]);
              }
            } else if (crank == 0) {
              mbar_wait(&cempty[s], ph ^ 1u);  // every CTA of the cluster is done with the slot
              const uint16_t mc = (uint16_t)((1u << C) - 1u);
              if (src) {
                bulk_g2s_mc(dst, src, kTileBytes, &full[s], mc);
                if (two) bulk_g2s_mc(dst + kTileBytes, src + second, kTileBytes, &full[s], mc);
              } else {
                tma_load_2d_mc(dst, &tmap_x, kb * kBlockK, r0, &full[s], mc);
                if (two) tma_load_2d_mc(dst + kTileBytes, &tmap_x, kb * kBlockK, r0 + kTileN, &full[s], mc);
              }
            }
          }
        }
        __syncwarp();
        if (++s == NST) { s = 0; ph ^= 1u; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    // The whole warp walks the loop; lane 0 issues.  The per-K-block work is kept minimal --
    // descriptors advanced by constants, no division -- because the issuing thread's own
    // instruction latency, not the tensor pipe, bounded the stream (REMOE_TC_TRACE cycle
    // split: ~90% of the issuer's time was issue work with an index/division-heavy loop).
    // kind::f16: D fp32 (bit 4), A bf16 (bits 7-9 = 1), B bf16 (bits 10-12 = 1),
    // both K-major, N >> 3 at bit 17, M >> 4 at bit 24
    // (debug REMOE_TC_DBG bit 4: N = 32, a quarter of the MMA work; wrong results)
    const uint32_t nn = (p.dbg & 4) ? 32u : (uint32_t)kUnitN;
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((nn >> 3) << 17) |
                           ((uint32_t)(M >> 4) << 24);
    // descriptor = ((address >> 4) & 0x3FFF) | constant bits: offsets add in 16-byte units
    const uint64_t da0 = umma_desc(smem_u32(sA)), db0 = umma_desc(smem_u32(sB));
    const uint64_t da_kb = (uint64_t)(SR * 128) >> 4, db_st = (uint64_t)kStageBytes >> 4;
    const bool skip_mma = (p.dbg & 1) != 0;
    int s = 0;
    uint32_t ph = 0;
    long long w_full = 0, w_tempty = 0, t_loop0 = p.trace ? clock64() : 0;  // REMOE_TC_TRACE cycle split
    for (int64_t i = 0; i < n_it; ++i) {
      const int acc = (int)(i & (kAcc - 1));
      const uint32_t aph = (uint32_t)(i / kAcc) & 1u;
      long long c0 = p.trace ? clock64() : 0;
      mbar_wait(&tempty[acc], aph ^ 1u);
      if (p.trace) w_tempty += clock64() - c0;
      tc_fence_after();
      if (lane == 0) {
        // the tile's |x_j| into sXn[acc] (the epilogue released acc, so also its norms):
        // 16-byte multiple of the valid rows (the norm arrays are padded for the rounding)
        const bool smp = i < ns_cta;
        const int64_t t = tile_of(i);
        int nv;
        const float* src;
        if (smp) {
          src = p.seed_xn + t * kUnitN;
          nv = kUnitN;  // the sample's norms are padded to whole units
        } else {
          src = p.xnorm + t * kUnitN;
          nv = (int)min((int64_t)kUnitN, p.n_rows - t * kUnitN);
        }
        const uint32_t nb = (uint32_t)((nv * 4 + 15) & ~15);
        mbar_arrive_expect_tx(&tfull[acc], nb);
        bulk_g2s(sXn + acc * kUnitN, src, nb, &tfull[acc]);
      }
      const uint32_t d_tmem = tmem_base + (uint32_t)(acc * kUnitN);
      uint64_t da = da0;
      for (int kb = 0; kb < nkb; ++kb) {
        c0 = p.trace ? clock64() : 0;
        mbar_wait(&full[s], ph);
        if (p.trace) w_full += clock64() - c0;
        tc_fence_after();
        if (lane == 0) {
          if (skip_mma) {  // debug (REMOE_TC_DBG=1): no MMA, free the slot at once (wrong results)
            mbar_arrive(&empty[s]);
          } else {
            const uint64_t db = db0 + (uint64_t)s * db_st;
            umma_bf16(d_tmem, da, db, idesc, kb != 0);
            umma_bf16(d_tmem, da + 2, db + 2, idesc, 1);
            umma_bf16(d_tmem, da + 4, db + 4, idesc, 1);
            umma_bf16(d_tmem, da + 6, db + 6, idesc, 1);
            umma_commit(&empty[s]);
            if (C > 1) umma_commit_mc(&cempty[s], 1);  // the leader's slot-free barrier
          }
        }
        __syncwarp();
        da += da_kb;
        if (++s == NST) { s = 0; ph ^= 1u; }
      }
      if (lane == 0) umma_commit(&tfull[acc]);
      __syncwarp();
      if (i == 0) TRACE(5);
    }
    if (p.trace && lane == 0) {
      unsigned long long* tr = p.trace + (blockIdx.y * gridDim.x + blockIdx.x) * kTraceSlots;
      tr[13] = (unsigned long long)(clock64() - t_loop0);
      tr[14] = (unsigned long long)w_full;
      tr[15] = (unsigned long long)w_tempty;
    }
  } else if (warp == kSeedWarp) {
    // ------------------------------------------------ seeding warp
    // For the queries m = blockIdx.x (mod grid.x) of this slab: wait until every state of
    // every CTA has published its sample key for m with this launch's epoch (bounded: on a
    // timeout the keys published so far are used -- the r-th largest of any subset of
    // published keys is still a lower bound), take the r-th largest key T, raise the
    // query's shared threshold to T - 1.  Keys are distinct (each sample row belongs to one
    // state) or 0 (no key).
    if (seeding) {
      pdl_wait();  // k_norms zeroes the shared thresholds first
      TRACE(18);
      const int G2 = 2 * (int)gridDim.x;
      const unsigned ep = s_epoch;
      for (int mm = blockIdx.x; mm < nq; mm += gridDim.x) {
        const size_t base = (size_t)(slab * QS + mm) * G2;
        const long long t0 = clock64();  // SM cycle counter: cheap (a %globaltimer read is not)
        unsigned ready = 0;  // bit u: slot lane + 32 u has this epoch's word
        // the published keys' score words (key >> 32; 0 = no key).  Each word carries its
        // epoch in the low half, so one relaxed 64-bit load (single-copy atomic) gives the
        // key and its validity together: no fences, no second load.  Under a full-bandwidth
        // store stream every L2 round trip costs microseconds (REMOE_TC_TRACE: key + fence +
        // tag, then fence + key load, took ~9 us from the last publish to the threshold).
        uint32_t hi[10];
#pragma unroll
        for (int u = 0; u < 10; ++u) hi[u] = 0u;
        for (;;) {
#pragma unroll
          for (int u = 0; u < 10; ++u) {
            const int idx = lane + 32 * u;
            if (idx < G2 && !((ready >> u) & 1u)) {
              unsigned long long w;
              asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p.seed_pub + base + idx) : "memory");
              if ((unsigned)w == ep) { ready |= 1u << u; hi[u] = (uint32_t)(w >> 32); }
            } else if (idx >= G2) {
              ready |= 1u << u;
            }
          }
          if (__all_sync(kFull, ready == 0x3FFu)) break;
          if (clock64() - t0 > 2 * p.seed_wait_ns) break;  // ~ns at <= 2 GHz
          __nanosleep(64);
        }
        if (mm == blockIdx.x) TRACE(19);
        // T = the r-th largest score word, by a 32-step radix select with warp-wide counts
        // (cost independent of r).  At least r published keys -- r distinct real keys of the
        // store -- are >= T << 32, so T << 32 - 1 is a strict lower bound of the k-th best
        // (r * h >= k).
        uint32_t pre = 0;
#pragma unroll 1
        for (int b = 31; b >= 0; --b) {
          const uint32_t cand = pre | (1u << b);
          int cnt = 0;
#pragma unroll
          for (int u = 0; u < 10; ++u) cnt += hi[u] >= cand ? 1 : 0;
          if (__reduce_add_sync(kFull, (unsigned)cnt) >= (unsigned)p.seed_r) pre = cand;
        }
        const uint64_t T = (uint64_t)pre << 32;
        if (lane == 0) {
          // the epilogues take the threshold from the done word itself (no ordering against
          // the shared threshold needed); the atomic only feeds later readers of gthr
          const unsigned long long dw = ((unsigned long long)pre << 32) | ep;
          asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p.seed_done + slab * QS + mm), "l"(dw) : "memory");
          if (T != 0) atomicMax(gthr_sl + mm, (unsigned long long)(T - 1));
        }
        if (mm == blockIdx.x) TRACE(20);
      }
    }
    // Threshold broker (then, or from the start without seeding): copy every query's
    // shared threshold gthr (raised by all states of all CTAs) into pair_thr about every
    // 0.3 us, until the last epilogue warp is done; the epilogue reads only pair_thr.
    pdl_wait();  // gthr zeroed by k_norms (no-op if already waited)
    for (;;) {
      for (int mm = lane; mm < nq; mm += 32) {
        unsigned long long v;
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(gthr_sl + mm) : "memory");
        if (v > *reinterpret_cast<volatile unsigned long long*>(pair_thr + mm)) atomicMax(pair_thr + mm, v);
      }
      if (*reinterpret_cast<volatile unsigned*>(s_epi_done) >= (unsigned)kEpiWarps) break;
      __nanosleep(256);
    }
  } else {
    // ------------------------------------------------ epilogue warps 2..9
    // Two warps per TMEM lane quarter (quarter = warp % 4 is the hardware rule); the
    // pair alternates tiles (parity = tile index % 2), so each warp has two tiles' time
    // for one tile and the pair hides each other's latency.  One thread per (query,
    // parity): thread (quarter, t) owns query m and sees all 128 columns of its tiles,
    // i.e. two top-k states per query per CTA.  For M = 64 the queries sit in lanes
    // 0-15 of a quarter and lanes 16-31 idle.
    //
    // Per 32-column chunk the common path is branch-free: x-norms come from a per-parity
    // shared-memory copy (ld.shared.v4 broadcasts), and a conservative fp32 test
    // dot >= tlim * (|q||x| + sigma) builds a 32-bit candidate mask; only columns in
    // the mask (rare once the threshold has settled) get the IEEE division, the key
    // and the push.
    const int e = warp - 2;
    const int quarter = warp & 3;
    const int parity = e >> 2;
    const int m = (M == 128) ? quarter * 32 + lane : quarter * 16 + lane;
    const bool active = (M == 128 || lane < 16) && m < nq;
    pdl_wait();  // k_norms: query norms and zeroed shared thresholds
    TRACE(6);
    const float qn = active ? (p.norms_in_kernel ? sQn[m] : qnorm_sl[m]) : 0.f;
    const int slot = e * 32 + lane;
    constexpr int kCap = 32 * (P > 0 ? P : 2);
    uint64_t* buf = p.smem_bufs ? sBuf + (size_t)slot * kCap
                                : p.cand_buf + (cta_lin * kTcEpilogueThreads + slot) * kCap;
    // KR > 0: register top-KR (k <= KR <= 16); otherwise buffer + compaction (any k <= 256)
    using Topk = typename std::conditional<(KR > 0), RegTopk<(KR > 0 ? KR : 1)>, LaneTopk<(P > 0 ? P : 2)>>::type;
    Topk tk;
    if constexpr (KR > 0) tk.init(p.k, active ? gthr_sl + m : nullptr);
    else tk.init(buf, active ? gthr_sl + m : nullptr);
    if (!active) tk.tlim = __int_as_float(0x7f800000);  // +inf: never a candidate
    // Seeding tracker: the kHS best per-chunk maxima of this state's sample tiles, as (dot,
    // den, gid) ranked by cross-multiplication (no division, no key, no 64-bit compares);
    // at the hand-off the exact keys of the first h of them are computed and their minimum
    // is published: h real keys of this state are >= it, which is all the seed needs (an
    // fp32 cross-multiplied ranking only makes the published key smaller, never invalid).  The sample
    // tiles deliberately do NOT feed the real top-k state: from an empty list every column
    // is an insert (~450 cycles of dependent latency each), ~30 us per 128-row tile.
    constexpr int kHS = 1;  // h = 1: each state publishes its best sample key (runtime.cu)
    float tr_dot[kHS], tr_den[kHS];
    uint32_t tr_gid[kHS];
#pragma unroll
    for (int j = 0; j < kHS; ++j) {
      tr_dot[j] = -__int_as_float(0x7f800000); tr_den[j] = 1.f;
      tr_gid[j] = 0xFFFFFFFFu;
    }
    auto seed_key = [&]() -> uint64_t {
      uint64_t kmin = ~0ull;
#pragma unroll
      for (int j = 0; j < kHS; ++j) {
        if (j < p.seed_h) {
          const uint64_t key = tr_gid[j] == 0xFFFFFFFFu ? 0ull : make_key(__fdiv_rn(tr_dot[j], tr_den[j]), (int64_t)tr_gid[j]);
          kmin = umin64(kmin, key);
        }
      }
      return kmin == ~0ull ? 0ull : kmin;
    };

    // tile i of the sequence: x-norm source, valid rows, global id of column j = gbase + j * gstride
    struct TileInfo { const float* xn; int nvalid; int64_t gbase, gstride; };
    auto tile_info = [&](int64_t i) -> TileInfo {
      TileInfo ti;
      const int64_t t = tile_of(i);
      if (i < ns_cta) {
        // the tile's segment, by selects over the (parameter-space) segment arrays: a
        // run-time index would copy them to the local stack
        int64_t t0 = 0, cnt = 0, off = 0, str = 1;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          if (g < p.seed_nseg && t >= p.seed_t0[g]) {
            t0 = p.seed_t0[g]; cnt = p.seed_count[g]; off = p.seed_off[g]; str = p.seed_stride[g];
          }
        }
        const int64_t li = (t - t0) * kUnitN;
        ti.xn = p.seed_xn + t * kUnitN;
        ti.nvalid = (int)min((int64_t)kUnitN, cnt - li);
        ti.gstride = str;
        ti.gbase = p.gid_offset + off + li * str;
      } else {
        const int64_t row0 = t * kUnitN;
        ti.xn = p.xnorm + row0;
        ti.nvalid = (int)min((int64_t)kUnitN, p.n_rows - row0);
        ti.gstride = p.gid_stride;
        ti.gbase = p.gid_offset + row0 * p.gid_stride;
      }
      return ti;
    };
    // Seeding hand-off, once per state, before its first store tile (or at the end when it
    // has none): publish the state's h-th best sample key with this launch's epoch.
    auto seed_publish = [&](uint64_t kh) {
      if (!active) return;
      const size_t slot = (size_t)(slab * QS + m) * (2 * gridDim.x) + 2 * blockIdx.x + parity;
      const unsigned long long w = (kh & 0xFFFFFFFF00000000ull) | s_epoch;  // one 64-bit store: key word + epoch
      asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p.seed_pub + slot), "l"(w) : "memory");
    };
    bool synced = !seeding;
    uint64_t pair_pub = 0;  // last value this state shared with its parity partner
    // The epilogue issues no global load per tile: the x-norms arrive with the tile
    // (sXn[acc]), the query's shared threshold through pair_thr (the broker warp copies
    // gthr there).  Under a full-bandwidth stream an L2 round trip takes microseconds, and
    // a per-tile load one tile ahead stalled the catch-up after the seed (~3 us per tile).
    long long ep_wait = 0, ep_t0 = 0;  // REMOE_TC_TRACE: tfull wait cycles of the store tiles' loop
    const bool warp_has_query = __any_sync(kFull, active);
    for (int64_t i = parity; i < n_it; i += 2) {
      const bool smp = i < ns_cta;
      if (p.trace && !smp && ep_t0 == 0) { ep_t0 = clock64(); ep_wait = 0; }
      if (!smp && !synced) {
        TRACE(3);
        seed_publish(seed_key());
        synced = true;
        // wait (bounded) for this query's seeded threshold: the TMA producer and the MMA run
        // on meanwhile (four accumulators of slack), and the first store tiles are then
        // filtered by the seed instead of inserting from an empty list
        uint64_t seeded = 0;
        if (active) {
          const long long t0 = clock64();
          for (;;) {
            unsigned long long dw;
            asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(dw) : "l"(p.seed_done + slab * QS + m) : "memory");
            if ((unsigned)dw == s_epoch) {
              if (dw >> 32) seeded = (dw & 0xFFFFFFFF00000000ull) - 1ull;  // strict lower bound
              break;
            }
            if (clock64() - t0 > 2 * p.seed_wait_ns) break;
            __nanosleep(128);
          }
        }
        if (seeded) atomicMax(pair_thr + m, (unsigned long long)seeded);
        __syncwarp();  // reconverge before the warp-collective barrier / tcgen05.ld below
        TRACE(10);
      }
      const int acc = (int)(i % kAcc);
      const uint32_t aph = (uint32_t)(i / kAcc) & 1u;
      const TileInfo ti = tile_info(i);
      const long long tw0 = p.trace ? clock64() : 0;
      if (p.epi_sleep) mbar_wait_sleep(&tfull[acc], aph);
      else mbar_wait(&tfull[acc], aph);
      if (p.trace) ep_wait += clock64() - tw0;
      const float* xs = sXn + acc * kUnitN;  // landed with the unit (tfull)
      if (i < 2) TRACE(7);
      if (active && !smp) tk.raise(*reinterpret_cast<volatile unsigned long long*>(pair_thr + m));
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * kUnitN);
      // A warp with no query of this launch (batches of <= 48 leave whole lane quarters
      // empty) releases the accumulator unread: no tcgen05.ld, no prefilter -- its issue
      // slots go to the warps it shares a scheduler with (the MMA issuer among them).
      // (REMOE_TC_DBG bit 2, experiment: every warp does so -- wrong results)
      if (!warp_has_query || (p.dbg & 2)) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        continue;
      }
      if (smp) {
        // ---- a sample tile: only the tracker (the store pass scans these rows again)
        if (i < 2) TRACE(16);
#pragma unroll 1
        for (int c = 0; c < kUnitN / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(tbase + c * 32, v);
          tmem_wait_ld();
          // no per-lane early exit here: the next chunk's tcgen05.ld is warp-collective
          const float* xc = xs + c * 32;
          const int left = active ? ti.nvalid - c * 32 : 0;
          {
            // the chunk's best column by an argmax tree on (dot, den) pairs compared by
            // cross-multiplication (den > 0): no division, five levels of independent compares
            float bd[32], bn[32];
            int bi[32];
#pragma unroll
            for (int j4 = 0; j4 < 8; ++j4) {
              const float4 x4 = lds128f(xc + 4 * j4);
              const float xx[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int j = 4 * j4 + u;
                bd[j] = j < left ? __uint_as_float(v[j]) : -__int_as_float(0x7f800000);
                bn[j] = __fmaf_rn(qn, xx[u], p.sigma);
                bi[j] = j;
              }
            }
#pragma unroll
            for (int w = 16; w > 0; w >>= 1) {
#pragma unroll
              for (int j = 0; j < w; ++j) {
                const bool up = bd[j + w] * bn[j] > bd[j] * bn[j + w];
                bd[j] = up ? bd[j + w] : bd[j];
                bn[j] = up ? bn[j + w] : bn[j];
                bi[j] = up ? bi[j + w] : bi[j];
              }
            }
            // ... kept in a sorted list of the kHS best chunk maxima (h of them are published:
            // each is a real key of this state, so its h-th is still a valid bound)
            float nd = bd[0], nn = bn[0];
            uint32_t ng = (uint32_t)(ti.gbase + (int64_t)(c * 32 + bi[0]) * ti.gstride);
            if (left > 0 && nd * tr_den[kHS - 1] > tr_dot[kHS - 1] * nn) {
#pragma unroll
              for (int q = 0; q < kHS; ++q) {
                const bool up = nd * tr_den[q] > tr_dot[q] * nn;
                const float d0 = tr_dot[q], n0 = tr_den[q];
                const uint32_t g0 = tr_gid[q];
                tr_dot[q] = up ? nd : d0; tr_den[q] = up ? nn : n0; tr_gid[q] = up ? ng : g0;
                nd = up ? d0 : nd; nn = up ? n0 : nn; ng = up ? g0 : ng;
              }
            }
          }
        }
        // release the accumulator -- and with it sXn[acc] -- only after the last chunk's
        // norms were read (the MMA warp refills both for tile i + kAcc)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        if (i < 2) TRACE(17);
        continue;
      }
#pragma unroll 1
      for (int c = 0; c < kUnitN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tbase + c * 32, v);
        tmem_wait_ld();
        if constexpr (KR > 0) {
          // the other parity state of this query lives in the same CTA: share its k-th best
          // through shared memory every chunk (exact: disjoint rows, own k-th best keys)
          if (active) tk.raise(*reinterpret_cast<volatile unsigned long long*>(pair_thr + m));
        }
        const float* xc = xs + c * 32;
        unsigned mask = 0;
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          const float4 x4 = lds128f(xc + 4 * j4);
          const float xx[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = 4 * j4 + u;
            const float den = __fmaf_rn(qn, xx[u], p.sigma);
            mask |= (tk.may_pass(__uint_as_float(v[j]), den) ? 1u : 0u) << j;
          }
        }
        const int left = ti.nvalid - c * 32;
        if (left < 32) mask &= left > 0 ? ((1u << left) - 1u) : 0u;
        if constexpr (KR > 0) {
          if (__any_sync(kFull, mask != 0)) {
            const int64_t gbase = ti.gbase + (int64_t)(c * 32) * ti.gstride;
            if (p.stats) {
              atomicAdd(p.stats + 0, (unsigned long long)__popc(mask));
              if (lane == 0) atomicAdd(p.stats + 2, 1ull);
            }
            while (mask) {  // per lane: insertion network, no warp synchronisation
              const int j = __ffs(mask) - 1;
              mask &= mask - 1;
              const float den = __fmaf_rn(qn, xc[j], p.sigma);
              const float vj = __uint_as_float(sel32(v, j));
              if (vj >= tk.tlim * den) {
                const int64_t gid = gbase + j * ti.gstride;
                const uint64_t key = make_key(__fdiv_rn(vj, den), gid);
                if (p.stats && key > tk.thr) atomicAdd(p.stats + 1, 1ull);
                tk.insert(key);
              }
            }
            if (active && tk.thr > pair_pub) {
              atomicMax(pair_thr + m, (unsigned long long)tk.thr);
              pair_pub = tk.thr;
            }
          }
        } else {
          const int pc = __popc(mask);
          if (__any_sync(kFull, pc >= 4)) {
            // many candidates (the first tiles, before the thresholds settle): compute all
            // keys of the chunk at once and append them (room for 32 guaranteed first)
            tk.ensure_room(32, p.k);
            const int64_t gbase = ti.gbase + (int64_t)(c * 32) * ti.gstride;
#pragma unroll
            for (int j4 = 0; j4 < 8; ++j4) {
              const float4 x4 = lds128f(xc + 4 * j4);
              const float xx[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int j = 4 * j4 + u;
                if ((mask >> j) & 1u) {
                  const float den = __fmaf_rn(qn, xx[u], p.sigma);
                  const int64_t gid = gbase + j * ti.gstride;
                  tk.append(make_key(__fdiv_rn(__uint_as_float(v[j]), den), gid));
                }
              }
            }
          } else if (__any_sync(kFull, mask != 0)) {
            const int64_t gbase = ti.gbase + (int64_t)(c * 32) * ti.gstride;
            while (__any_sync(kFull, mask != 0)) {
              uint64_t key = 0;
              if (mask) {
                const int j = __ffs(mask) - 1;
                mask &= mask - 1;
                const float den = __fmaf_rn(qn, xc[j], p.sigma);
                const int64_t gid = gbase + j * ti.gstride;
                key = make_key(__fdiv_rn(__uint_as_float(sel32(v, j)), den), gid);
              }
              tk.push(key, p.k);
            }
          }
        }
      }
      // every tcgen05.ld of the tile completed and its last norms were read: release
      // the accumulator and sXn[acc]
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if constexpr (KR > 0) tk.publish();
    }
    if (lane == 0) atomicAdd(s_epi_done, 1u);  // the broker warp stops after the last one
    if (p.trace && lane == 0 && warp == 4) {  // quarter 0, parity 0: store-loop cycles, tfull waits
      unsigned long long* tr = p.trace + (blockIdx.y * gridDim.x + blockIdx.x) * kTraceSlots;
      tr[21] = (unsigned long long)(clock64() - ep_t0);
      tr[22] = (unsigned long long)ep_wait;
    }
    if (!synced) seed_publish(seed_key());  // this parity had no store tile
    TRACE(8);
    if (KR > 0 && p.merge_in_cta) {
      // Merge the two parity states of each query inside the CTA (one list per CTA per
      // query halves the merge kernel's input).  The TMA stage ring is idle now (every
      // tile has been consumed), so it serves as scratch: state (slot) -> KR keys.
      uint64_t* scratch = reinterpret_cast<uint64_t*>(sB);
      // every epilogue warp has consumed its last accumulator, so every MMA has completed
      // and every TMA load has landed: only then is the ring free
      asm volatile("bar.sync 2, %0;" ::"n"(kEpiWarps * 32) : "memory");
      if constexpr (KR > 0) tk.flush(scratch + (size_t)slot * KR);  // all KR slots (k <= KR)
      asm volatile("bar.sync %0, 64;" ::"r"(3 + quarter) : "memory");  // the quarter's two warps
      if (parity == 0 && active) {
        const uint64_t* a = scratch + (size_t)slot * (KR > 0 ? KR : 1);
        const uint64_t* b = scratch + (size_t)(slot + 128) * (KR > 0 ? KR : 1);  // warp e + 4, same lane
        uint64_t* o = out_sl + ((size_t)m * gridDim.x + blockIdx.x) * (size_t)p.k;
        int ia = 0, ib = 0;
        for (int r = 0; r < p.k; ++r) {  // two-pointer merge of two descending lists
          const uint64_t x = a[ia], y = b[ib];
          if (x >= y) { o[r] = x; ++ia; } else { o[r] = y; ++ib; }
        }
      }
    } else {
      uint64_t* out =
          active ? out_sl + (((size_t)m * gridDim.x + blockIdx.x) * 2 + parity) * (size_t)p.k : nullptr;
      if constexpr (KR > 0) {
        tk.flush(out);
      } else {
        // buffers in global memory: sort in the (now idle) TMA ring, 32 keys per lane --
        // once every epilogue warp consumed its last accumulator, every MMA has read the ring
        uint64_t* scratch = nullptr;
        if (!p.smem_bufs && (size_t)NST * kStageBytes >= (size_t)kEpiWarps * 32 * 32 * 8) {
          asm volatile("bar.sync 2, %0;" ::"n"(kEpiWarps * 32) : "memory");
          scratch = reinterpret_cast<uint64_t*>(sB) + (size_t)slot * 32;
        }
        tk.flush(out, p.k, scratch);
      }
    }
  }
  __syncthreads();
  TRACE(9);
  if (p.trace && threadIdx.x == 0) p.trace[(blockIdx.y * gridDim.x + blockIdx.x) * kTraceSlots + 12] = clock64();
  if (C > 1) {  // no CTA leaves while a peer may still arrive on its barriers
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(kTmemCols));
  }
}

// ------------------------------------------------------------------ tiled store
// xt box (tile, kb) = rows tile*128 .. +127, elements kb*64 .. +63, laid out exactly as
// the UMMA reads a SWIZZLE_128B K-major operand from a 1024-byte aligned stage: row r at
// r*128 bytes, its 16-byte chunk c at ((c ^ (r & 7)) * 16).  One thread per 16-byte chunk.
// Columns past D (when D % 64 != 0) and rows past n_rows are zero.
__global__ void k_tile_store(const uint4* __restrict__ x, int64_t n_rows, int dim, uint4* __restrict__ xt) {
  const int cpr = dim / 8;                  // 16-byte chunks per source row
  const int cpk = ((dim + 63) / 64) * 8;    // ... per tiled row, K-padding included
  const int64_t n_tiles = (n_rows + kTileN - 1) / kTileN;
  const int64_t total = n_tiles * kTileN * cpk;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / cpk;
    const int cc = (int)(i - row * cpk);
    const int kb = cc >> 3, c = cc & 7, r = (int)(row % kTileN);
    const int64_t tile = row / kTileN;
    const uint4 v = (row < n_rows && cc < cpr) ? x[row * cpr + cc] : make_uint4(0u, 0u, 0u, 0u);
    xt[((tile * (cpk >> 3) + kb) * kTileN + r) * 8 + (c ^ (r & 7))] = v;
  }
}

cudaError_t tc_tile_store(const uint16_t* x, int64_t n_rows, int dim, uint16_t* xt, cudaStream_t st) {
  if (dim % 8 != 0 || n_rows <= 0) return cudaErrorInvalidValue;
  k_tile_store<<<1184, 256, 0, st>>>(reinterpret_cast<const uint4*>(x), n_rows, dim, reinterpret_cast<uint4*>(xt));
  return cudaGetLastError();
}

// ------------------------------------------------------------------ seeding sample
// out row i = x[src[i]] (src[i] < 0: a zero row), its norm xn[src[i]] (1 for padding).
__global__ void k_gather_sample(const uint4* __restrict__ x, const float* __restrict__ xnorm,
                                const int64_t* __restrict__ src, int64_t n, int dim, uint4* __restrict__ out,
                                float* __restrict__ out_norm) {
  const int cpr = dim / 8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * cpr; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / cpr;
    const int c = (int)(i - row * cpr);
    const int64_t r = src[row];
    out[i] = r >= 0 ? x[r * cpr + c] : make_uint4(0u, 0u, 0u, 0u);
    if (c == 0) out_norm[row] = r >= 0 ? xnorm[r] : 1.f;
  }
}

remoe_status_t tc_seed_build(TcSeed* sd, const uint16_t* x, const float* xnorm, int64_t n_rows, int dim,
                             cudaStream_t st, void* (*alloc)(void*, size_t), void* actx) {
  // segments: rows 64j, 64j+32, 32j+16, 16j+8 (a prefix of g + 1 segments = every
  // (64 >> g)-th row), each padded to whole 256-row scan units
  static const int64_t off[4] = {0, 32, 16, 8}, stride[4] = {64, 64, 32, 16};
  sd->n_seg = 0;
  int64_t units = 0;
  std::vector<int64_t> src;
  for (int g = 0; g < 4; ++g) {
    const int64_t cnt = n_rows > off[g] ? (n_rows - off[g] + stride[g] - 1) / stride[g] : 0;
    if (cnt == 0) break;
    sd->seg_t0[g] = (int)units;
    sd->seg_count[g] = cnt;
    sd->seg_off[g] = off[g];
    sd->seg_stride[g] = stride[g];
    const int64_t nt = (cnt + kUnitN - 1) / kUnitN;  // whole scan units (two tiled-copy tiles each)
    for (int64_t i = 0; i < nt * kUnitN; ++i) src.push_back(i < cnt ? off[g] + i * stride[g] : -1);
    units += nt;
    sd->n_seg = g + 1;
  }
  sd->seg_t0[sd->n_seg] = (int)units;
  if (sd->n_seg == 0) return REMOE_OK;
  const int64_t rows = units * kUnitN;
  int64_t* d_src = static_cast<int64_t*>(alloc(actx, rows * 8));
  uint16_t* tmp = static_cast<uint16_t*>(alloc(actx, (size_t)rows * dim * 2));
  sd->xt = static_cast<uint16_t*>(alloc(actx, (size_t)rows * tc_kpad(dim) * 2));
  sd->xn = static_cast<float*>(alloc(actx, (size_t)rows * 4));
  if (!d_src || !tmp || !sd->xt || !sd->xn) return REMOE_ERR_OOM;
  if (cudaMemcpyAsync(d_src, src.data(), rows * 8, cudaMemcpyHostToDevice, st) != cudaSuccess) return REMOE_ERR_CUDA;
  k_gather_sample<<<1184, 256, 0, st>>>(reinterpret_cast<const uint4*>(x), xnorm, d_src, rows, dim,
                                        reinterpret_cast<uint4*>(tmp), sd->xn);
  if (cudaGetLastError() != cudaSuccess) return REMOE_ERR_CUDA;
  if (tc_tile_store(tmp, rows, dim, sd->xt, st) != cudaSuccess) return REMOE_ERR_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return REMOE_ERR_CUDA;
  return REMOE_OK;
}

// ------------------------------------------------------------------ host side

// Offset of dynamic shared memory from a 1024-byte boundary (kernels without static shared
// memory): probed once; the scans align their base up to 1024, so they reserve 1024 bytes
// of slack only if the base is not already aligned (the slack is worth a stage at D=1024).
__global__ void k_probe_dyn_smem(unsigned* out) {
  extern __shared__ uint8_t s_probe[];
  if (threadIdx.x == 0) *out = smem_u32(s_probe) & 1023u;
}

int dyn_smem_pad() {
  static int pad = -1;
  if (pad >= 0) return pad;
  int result = 1024;
  unsigned* d = nullptr;
  unsigned h = 1;
  const int bytes = kMaxSmem - 4096;
  if (cudaFuncSetAttribute((const void*)k_probe_dyn_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) ==
          cudaSuccess &&
      cudaMalloc(&d, sizeof(unsigned)) == cudaSuccess) {
    k_probe_dyn_smem<<<1, 32, bytes>>>(d);
    if (cudaMemcpy(&h, d, sizeof(unsigned), cudaMemcpyDeviceToHost) == cudaSuccess && h == 0) result = 0;
    cudaFree(d);
  }
  cudaGetLastError();
  pad = result;
  return pad;
}

// REMOE_TC_MAX_STAGES (read at plan creation): cap of the stage ring depth.
static int g_max_stages = 0;

// slab_rows: query rows stored per K-block (M for a full slab).
static size_t tc_smem(int M, int slab_rows, int D, int nst, int buf_bytes) {
  return (size_t)dyn_smem_pad() + (size_t)(tc_kpad(D) / kBlockK) * slab_rows * 128 + (size_t)nst * kStageBytes +
         (3 * (size_t)nst + 2 * kAcc + 4) * 8 + (size_t)kAcc * kUnitN * 4 + (size_t)M * 12 + (size_t)buf_bytes;
}

static int tc_stages(int M, int D, int buf_bytes, int slab_rows = 0) {
  const long avail = (long)kMaxSmem - (long)tc_smem(M, slab_rows > 0 ? slab_rows : M, D, 0, buf_bytes);
  const long n = avail / (kStageBytes + 24);  // a stage: its 32 KB + three mbarriers (full, empty, cempty)
  const int cap = g_max_stages > 0 ? g_max_stages : kMaxStages;
  return (int)(n > cap ? cap : n);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);

remoe_status_t tc_plan_create(TcPlan* t, const uint16_t* x, int64_t n_rows, int dim, int num_sms,
                              int max_k, int64_t row_stride) {
  if (row_stride <= 0) row_stride = dim;
  (void)max_k;
  t->ok = false;
  t->x = x;
  t->n_rows = n_rows;
  t->dim = dim;
  t->row_stride = row_stride;
  t->grid = t->grid_units = 0;
  t->threads_per_cta_queries = kTcEpilogueThreads;
  if (dim % 8 != 0) { t->why = "D % 8 != 0"; return REMOE_OK; }  // D % 64 != 0: the last K-block is zero-padded
  // the resident slab holds max_qps query rows: 64 while that leaves >= 2 stages of 32 KB
  // (D <= 1280), else the largest multiple of 8 that does (D = 1536: 48, 2048: 40, 4096: 16);
  // larger batches take several slabs (or the CTA-pair scan)
  t->max_qps = 0;
  for (int sr = 64; sr >= 8 && t->max_qps == 0; sr -= 8)
    if (tc_stages(64, dim, 0, sr) >= 2) t->max_qps = sr;
  if (t->max_qps == 0) { t->why = "even an 8-query slab does not fit shared memory"; return REMOE_OK; }
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q{};
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      fn == nullptr || q != cudaDriverEntryPointSuccess) {
    cudaGetLastError();
    t->why = "cuTensorMapEncodeTiled unavailable";
    return REMOE_OK;
  }
  t->kn = TcKnobs::from_env();
  if (const char* e = getenv("REMOE_TC_MAX_STAGES")) g_max_stages = atoi(e);
  const cuuint64_t gdim[2] = {(cuuint64_t)dim, (cuuint64_t)n_rows};
  const cuuint64_t gstride[1] = {(cuuint64_t)row_stride * 2};
  const cuuint32_t box[2] = {(cuuint32_t)kBlockK, (cuuint32_t)kTileN};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = ((EncodeTiledFn)fn)(reinterpret_cast<CUtensorMap*>(t->tmap_x), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                                   const_cast<uint16_t*>(x), gdim, gstride, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   t->kn.promotion(),
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { t->why = "cuTensorMapEncodeTiled failed"; return REMOE_OK; }
  const int64_t n_tiles = (n_rows + kTileN - 1) / kTileN, n_units = (n_rows + kUnitN - 1) / kUnitN;
  t->grid = (int)(n_tiles < num_sms ? n_tiles : num_sms);
  t->grid_units = (int)(n_units < num_sms ? n_units : num_sms);
  if (!t->pair_sync) {
    if (cudaMalloc(&t->pair_sync, 17 * sizeof(unsigned)) != cudaSuccess ||
        cudaMemset(t->pair_sync, 0, 17 * sizeof(unsigned)) != cudaSuccess) {
      cudaGetLastError();
      t->pair_sync = nullptr;  // the pair scan's groups then run without lockstep
    }
  }
  t->ok = true;
  t->why = "";
  return REMOE_OK;
}

void tc_plan_destroy(TcPlan* t) {
  t->ok = false;
  if (t->stats_buf) cudaFree(t->stats_buf);
  if (t->trace_buf) cudaFree(t->trace_buf);
  t->stats_buf = t->trace_buf = nullptr;
  if (t->pair_sync) cudaFree(t->pair_sync);
  t->pair_sync = nullptr;
}

template <int M, int P, int KR = 0>
static cudaError_t launch_tc_t(const TcPlan* t, const TcArgs& a, dim3 grid, cudaStream_t st) {
  const size_t smem = tc_smem(M, a.slab_rows, a.dim, a.n_stages, a.smem_bufs ? kTcEpilogueThreads * 32 * P * 8 : 0);
  static_assert(P >= 0, "P");
  auto kern = k_scan_tc<M, P, KR>;
  cudaError_t e = set_smem_attrs_once((const void*)kern, kMaxSmem);
  if (e != cudaSuccess) return e;
  if (a.cluster > 1) {
    // largest cluster size (<= requested) that divides the slabs and keeps every cluster
    // co-resident (tiles are assigned statically: a second wave would double the time)
    TcArgs& aa = const_cast<TcArgs&>(a);
    while (aa.cluster > 1 && ((grid.y % aa.cluster) != 0 ||
                              (int)(grid.x * grid.y / aa.cluster) >
                                  max_active_clusters_cached((const void*)kern, dim3(kThreads), smem, aa.cluster)))
      aa.cluster >>= 1;
    if (t->kn.verbose)
      fprintf(stderr, "[remoe] tc scan grid (%u,%u) cluster %d (max active clusters of 8/4/2: %d/%d/%d)\n",
              grid.x, grid.y, aa.cluster, max_active_clusters((const void*)kern, dim3(kThreads), smem, 8),
              max_active_clusters((const void*)kern, dim3(kThreads), smem, 4),
              max_active_clusters((const void*)kern, dim3(kThreads), smem, 2));
  }
  // PDL: the prologue (barriers, TMEM, query slab, first TMA loads) overlaps the tail of
  // k_norms; the epilogue waits for it (query norms, zeroed thresholds)
  if (a.cluster > 1)
    return launch_pdl_cluster(kern, grid, dim3(kThreads), smem, st, (unsigned)a.cluster,
                              *reinterpret_cast<const CUtensorMap*>(t->tmap_x), a);
  return launch_pdl(kern, grid, dim3(kThreads), smem, st,
                    *reinterpret_cast<const CUtensorMap*>(t->tmap_x), a);
}

template <int M>
static cudaError_t launch_tc_m(const TcPlan* t, const TcArgs& a, dim3 g, cudaStream_t st) {
  // register top-k for k <= 32 (list length pow2ceil(k))
  if (a.k <= 1) return launch_tc_t<M, 0, 1>(t, a, g, st);
  if (a.k <= 2) return launch_tc_t<M, 0, 2>(t, a, g, st);
  if (a.k <= 4) return launch_tc_t<M, 0, 4>(t, a, g, st);
  if (a.k <= 8) return launch_tc_t<M, 0, 8>(t, a, g, st);
  if (a.k <= 16) return launch_tc_t<M, 0, 16>(t, a, g, st);
  if (a.k <= 32) return launch_tc_t<M, 0, 32>(t, a, g, st);
  switch (topk_P(a.k)) {
    case 2: return launch_tc_t<M, 2>(t, a, g, st);
    case 4: return launch_tc_t<M, 4>(t, a, g, st);
    case 8: return launch_tc_t<M, 8>(t, a, g, st);
    case 16: return launch_tc_t<M, 16>(t, a, g, st);
  }
  return cudaErrorInvalidValue;
}

int tc_single_slab_max(const TcPlan* t) {
  return !t->ok ? 0 : tc_stages(128, t->dim, 0) >= 2 ? 128 : t->max_qps;
}

remoe_status_t tc_scan(TcPlan* t, const uint16_t* q, const float* qnorm, int bc, int k, float sigma,
                       const float* xnorm, int64_t n_rows, int64_t gid_offset, int64_t gid_stride,
                       uint64_t* cand_buf, unsigned long long* gthr, uint64_t* lists, cudaStream_t st,
                       int* launches, int* lists_per_query, const TcSeedUse* seed, bool norms_in_kernel) {
  if (!t->ok) return REMOE_ERR_UNSUPPORTED;
  // M = 128 when the 128-query slab still leaves >= 2 stages (64 KB), else 64.  Candidate
  // buffers go to shared memory when that still leaves >= 2 stages.
  const int QS = tc_single_slab_max(t);  // queries per slab
  const int M = QS == 128 ? 128 : 64;    // max_qps <= 64
  const int buf_bytes = k <= 32 ? 0 : kTcEpilogueThreads * 32 * topk_P(k) * 8;
  // a single slab stores only the 8-row atoms its queries need (more stages for small B)
  const int n_slabs_all = (bc + QS - 1) / QS;
  const TcKnobs& kn = t->kn;
  const int SR = (n_slabs_all == 1 && !(kn.full_slab && QS == M)) ? ((bc + 7) / 8) * 8 : QS;
  const bool smem_bufs = k > 32 && tc_stages(M, t->dim, buf_bytes, SR) >= 2 && !kn.global_bufs;
  int nst = tc_stages(M, t->dim, smem_bufs ? buf_bytes : 0, SR);
  if (kn.stages >= 2 && kn.stages < nst) nst = kn.stages;
  // register top-k merges its two parity states in-CTA when the stage ring can hold them
  const int KR = k <= 1 ? 1 : k <= 2 ? 2 : k <= 4 ? 4 : k <= 8 ? 8 : k <= 16 ? 16 : 32;
  const bool in_cta = k <= 32 && (size_t)nst * kStageBytes >= (size_t)kTcEpilogueThreads * KR * 8;
  const int lists_per_cta = in_cta ? 1 : 2;
  // Query slabs of M: one launch covers up to grid slabs, each slab on grid / slabs CTAs
  // walking the store in the same tile order (L2 sharing of every tile across slabs).
  const int n_slabs = n_slabs_all;
  const int slabs_per_launch = n_slabs < t->grid_units ? n_slabs : t->grid_units;
  const int ctas_per_slab = t->grid_units / slabs_per_launch;
  *lists_per_query = ctas_per_slab * lists_per_cta;
  for (int sl0 = 0; sl0 < n_slabs; sl0 += slabs_per_launch) {
    const int ns = n_slabs - sl0 < slabs_per_launch ? n_slabs - sl0 : slabs_per_launch;
    const int s0 = sl0 * QS;
    TcArgs a{};
    a.xnorm = xnorm;
    a.n_rows = n_rows;
    a.gid_offset = gid_offset;
    a.dim = t->dim;
    a.q = q + (size_t)s0 * t->dim;
    a.qnorm = qnorm + s0;
    a.nq = bc - s0;  // queries of this launch; slab y takes [y*M, y*M + M)
    a.k = k;
    a.sigma = sigma;
    a.n_stages = nst;
    a.cand_buf = cand_buf;
    a.gthr = gthr + s0;
    a.gid_stride = gid_stride;
    a.out = lists + (size_t)s0 * ctas_per_slab * lists_per_cta * k;
    a.merge_in_cta = in_cta ? 1 : 0;
    a.smem_bufs = smem_bufs ? 1 : 0;
    a.cluster = kn.no_multicast ? 1 : 8;  // reduced to what fits in launch_tc_t
    a.epi_sleep = kn.epi_sleep;
    a.xt = t->xt;
    a.slab_rows = SR;
    a.qps = QS;
    a.dbg = kn.dbg;
    a.norms_in_kernel = norms_in_kernel ? 1 : 0;
    if (seed && t->xt && 2 * ctas_per_slab <= 320 && seed->store->pub && seed->store->done) {
      const TcSeed& sd = *seed->store;
      a.seed_xt = sd.xt;
      a.seed_xn = sd.xn;
      a.seed_n_stiles = seed->n_stiles;
      a.seed_nseg = sd.n_seg;
      for (int g = 0; g <= sd.n_seg; ++g) a.seed_t0[g] = sd.seg_t0[g];
      for (int g = 0; g < sd.n_seg; ++g) {
        a.seed_count[g] = sd.seg_count[g];
        a.seed_off[g] = sd.seg_off[g];
        a.seed_stride[g] = sd.seg_stride[g];
      }
      a.seed_h = seed->h;
      a.seed_r = seed->r;
      a.seed_pub = sd.pub + (size_t)s0 * 2 * ctas_per_slab;
      a.seed_done = sd.done + s0;
      a.seed_epoch = sd.epoch;
      a.seed_wait_ns = sd.wait_ns;
    }
    if (kn.stats) {  // debug counters (this plan's buffer)
      if (!t->stats_buf && cudaMalloc(&t->stats_buf, 3 * 8) != cudaSuccess) return REMOE_ERR_OOM;
      cudaMemsetAsync(t->stats_buf, 0, 3 * 8, st);
      a.stats = t->stats_buf;
    }
    const int n_cta = ctas_per_slab * ns;
    if (kn.trace) {  // debug: per-CTA globaltimer stamps of the launch phases (this plan's buffer)
      if (!t->trace_buf && cudaMalloc(&t->trace_buf, (size_t)t->grid * kTraceSlots * 8) != cudaSuccess) return REMOE_ERR_OOM;
      cudaMemsetAsync(t->trace_buf, 0, (size_t)n_cta * kTraceSlots * 8, st);
      a.trace = t->trace_buf;
    }
    const dim3 g((unsigned)ctas_per_slab, (unsigned)ns);
    cudaError_t e = (M == 128) ? launch_tc_m<128>(t, a, g, st) : launch_tc_m<64>(t, a, g, st);
    if (e != cudaSuccess) return REMOE_ERR_CUDA;
    if (a.trace) {
      std::vector<unsigned long long> h((size_t)n_cta * kTraceSlots);
      cudaMemcpyAsync(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      unsigned long long t0 = ~0ull;
      for (int c = 0; c < n_cta; ++c) if (h[c * kTraceSlots] && h[c * kTraceSlots] < t0) t0 = h[c * kTraceSlots];
      fprintf(stderr, "[remoe] tc trace (us from first CTA start; CTA 0 | max over CTAs): nq %d k %d units %lld\n",
              a.nq, k, (long long)((n_rows + kUnitN - 1) / kUnitN));
      const char* names[22] = {"start", "setup", "slab", "seed publish", "", "mma tile0 commit",
                               "epi pdl_wait", "epi first tfull", "epi loop done", "end", "seed ready", "", "", "", "",
                               "", "sample tile start", "sample tile end", "seedw pdl_wait", "seedw keys seen", "seedw done", ""};
      for (int i = 0; i < 21; ++i) {
        if (!names[i][0]) continue;
        unsigned long long mx = 0;
        for (int c = 0; c < n_cta; ++c) if (h[c * kTraceSlots + i] > mx) mx = h[c * kTraceSlots + i];
        fprintf(stderr, "  %-18s %9.2f | %9.2f\n", names[i], h[i] ? (h[i] - t0) / 1e3 : -1.0,
                mx ? (mx - t0) / 1e3 : -1.0);
      }
      const int cyc[5] = {13, 14, 15, 21, 22};
      const char* cn[5] = {"mma loop cyc", "mma full wait", "mma tempty wait", "epi4 loop cyc", "epi4 tfull wait"};
      for (int j = 0; j < 5; ++j) {
        unsigned long long mx = 0, sum = 0;
        for (int c = 0; c < n_cta; ++c) { mx = std::max(mx, h[c * kTraceSlots + cyc[j]]); sum += h[c * kTraceSlots + cyc[j]]; }
        fprintf(stderr, "  %-18s %9llu | max %9llu | mean %9llu\n", cn[j], h[cyc[j]], mx, sum / n_cta);
      }
    }
    if (a.stats) {
      unsigned long long h[3];
      cudaMemcpyAsync(h, a.stats, 24, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      fprintf(stderr, "[remoe] tc stats: candidates %llu inserts %llu candidate-chunks %llu (queries %d, k %d)\n",
              h[0], h[1], h[2], a.nq, k);
    }
    ++*launches;
  }
  return REMOE_OK;
}

}  // namespace remoe
