// k_scan_pair.cu -- S2+S3 for large query batches on CTA pairs (tcgen05 cta_group::2).
//
// score_ij = (q_i . x_j) / (|q_i||x_j| + sigma)  (Eq. 11, DESIGN R2), exact
// per-CTA running top-k per query (BF top-alpha) -- the same arithmetic, keys and
// top-k states as k_scan_tc, on a different tiling.
//
// Why a second tensor-core scan: k_scan_tc keeps an M = 64 query slab resident in shared
// memory and streams only the store; that is right while the path is HBM-bound (B below
// the ridge, ~214), but every slab re-ingests the whole store, so at large B the SMs
// ingest B/64 copies of it and the tensor pipe idles.  Here the contraction is tiled as a
// GEMM on CTA pairs: UMMA M = 256 queries (128 per CTA), N = 256 store rows (128 loaded
// by each CTA), K = D in 64-element blocks, both operands streamed by TMA.  Per CTA a
// K-block moves 32 KB into shared memory for 2*128*256*64 flops (128 flop/byte, twice the
// slab kernel), and the pair shares both operands through the cta_group::2 MMA.
//   * Warp 0 (both CTAs): TMA producer.  A box [128 queries x 64] and B box [128 rows x
//     64] (SWIZZLE_128B) per K-block into an NST-deep ring; completion is counted on the
//     LEADER's full barrier (.cta_group::2 TMA), which expects both CTAs' 64 KB.
//   * Warp 1 (leader only): one thread issues tcgen05.mma.cta_group::2 (M=256, N=256,
//     K=16) x 4 per K-block into one of two TMEM accumulators (2 x 256 fp32 columns =
//     all 512), and commits (multicast to both CTAs) to the slot-free and
//     accumulator-full barriers.
//   * Warps 2-9 (both CTAs): epilogue.  Each CTA's TMEM holds its own 128 queries x 256
//     store rows.  Warps alternate tiles by parity (accumulator = tile parity); thread
//     (quarter, lane) owns query quarter*32 + lane and walks the 256 columns in 32-column
//     tcgen05.ld chunks: branch-free conservative prefilter, exact key + insert for the
//     rare candidates, shared per-query thresholds (all exactly as in k_scan_tc).  The
//     accumulator is released to the leader's tempty barrier (remote arrive from CTA 1).
// The dot for (q, row) accumulates K-blocks in ascending order in the tensor core; it does
// not depend on the batch position or the tiling (same fp32 sum order as k_scan_tc).
#include <cuda.h>
#include <stdio.h>
#include <stdlib.h>

#include <type_traits>

#include "common.cuh"
#include "host_util.h"
#include "kernels.h"
#include "tc_host.h"
#include "tcgen05.cuh"

namespace remoe {

namespace {
constexpr int kQPerCta = 128;            // A rows per CTA (UMMA M = 256 per pair)
constexpr int kPairN = 256;              // store rows per tile (UMMA N), 128 per CTA
constexpr int kPBK = 64;                 // bf16 elements per 128-byte swizzle row
constexpr int kBox = 128 * kPBK * 2;     // 16 KB: one operand box
constexpr int kPThreads = 320;           // TMA, MMA, 8 epilogue warps
constexpr int kPEpiWarps = 8;
constexpr int kPAcc = 2;                 // TMEM accumulators (= tile parities)
constexpr int kPTmemCols = kPAcc * kPairN;  // 512
constexpr int kPMaxSmem = 232448;

struct PairArgs {
  const float* xnorm;
  int64_t n_rows;
  int64_t gid_offset;
  int64_t gid_stride;      // global id of row r = gid_offset + r * gid_stride (seed samples: stride)
  int dim;
  const float* qnorm;      // [nq] of this launch
  int nq;                  // queries of this launch; group y, CTA rank r: [256 y + 128 r, +128)
  int k;
  float sigma;
  int n_stages;
  uint64_t* cand_buf;      // LaneTopk buffers in global memory (when not in shared memory)
  unsigned long long* gthr;  // [nq] shared thresholds (zeroed by k_norms)
  uint64_t* out;           // lists[(q * lists_per_query + l) * k + i]
  int smem_bufs;
  int merge_in_cta;
  int dbg;                 // REMOE_TC_DBG experiment bits (wrong results): 128 = load the query
                           // box only for the first tile, 256 = the store box only for the first
  // Group lockstep (REMOE_PAIR_LOCKSTEP=1, several query groups per launch): a pair starts
  // loading tile round r only once the groups have issued round r - kLockWindow on average,
  // so they read each store tile within a few rounds of each other and the later ones hit L2.
  // Measured at c3 B = 1024 (4 groups): DRAM 1.03-1.05x the algorithmic bytes instead of
  // 1.11-1.36x, but the scan ~2% slower (pairs wait for the slowest group; at 8 groups -8%,
  // at a 6-round window the live set thrashes L2) -- off by default: time is the metric.
  unsigned* prog;          // [gridDim.y] rounds issued per group (zeroed; reset by the last CTA)
  unsigned* exit_cnt;      // CTAs finished (the last one resets prog and itself)
};
constexpr int kLockWindow = 3;
constexpr int kLockMaxGroups = 4;  // more groups: waiting for the slowest of them costs more than the re-reads
}  // namespace

template <int P, int KR>
__global__ void __launch_bounds__(kPThreads, 1)
    k_scan_pair(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_q,
                PairArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int NST = p.n_stages;
  const int nkb = (p.dim + kPBK - 1) / kPBK;  // the last K-block's columns past D are TMA zero fill
  uint8_t* sA = smem;                              // [NST][128 queries][128 B] swizzled
  uint8_t* sB = sA + (size_t)NST * kBox;           // [NST][128 rows][128 B] swizzled
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + (size_t)NST * kBox);
  uint64_t* empty = full + NST;
  uint64_t* tfull = empty + NST;
  uint64_t* tempty = tfull + kPAcc;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + kPAcc);
  float* sXn = reinterpret_cast<float*>(tempty + kPAcc + 2);  // [8 warps][256], 16-byte aligned
  unsigned long long* pair_thr = reinterpret_cast<unsigned long long*>(sXn + kPEpiWarps * kPairN);  // [128]
  uint64_t* sBuf = reinterpret_cast<uint64_t*>(pair_thr + kQPerCta);  // [256][CAP] if p.smem_bufs

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  uint32_t crank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  const int pair = blockIdx.x >> 1;
  const int npairs = gridDim.x >> 1;
  const int qrow0 = blockIdx.y * (2 * kQPerCta) + (int)crank * kQPerCta;  // this CTA's first query
  const int nq = max(0, min(kQPerCta, p.nq - qrow0));
  const int64_t n_tiles = (p.n_rows + kPairN - 1) / kPairN;
  const int lists_per_cta = p.merge_in_cta ? 1 : 2;
  pdl_trigger();

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < kPAcc; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 2 * 4); }
    for (int s = 0; s < kQPerCta; ++s) pair_thr[s] = 0ull;
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_x) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_q) : "memory");
  }
  cluster_sync_all();  // the peer's barriers exist before any remote arrive, TMA or commit
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(kPTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer (both CTAs)
    // Warp-uniform loop (loop state in uniform registers), lane 0 issues; no division per
    // K-block (the issuing thread's instruction latency bounds these loops, k_scan_tc).
    const uint32_t full0 = mapa_shared(smem_u32(full), 0);  // the leader's full barriers
    int s = 0;
    uint32_t ph = 0;
    const bool lock = p.prog != nullptr && gridDim.y > 1 && crank == 0;
    const int64_t min_rounds = n_tiles / npairs;  // every pair has at least this many rounds
    int64_t r = 0;
    for (int64_t t = pair; t < n_tiles; t += npairs, ++r) {
      if (lock && r >= kLockWindow && r - kLockWindow < min_rounds) {
        if (lane == 0) {
          const unsigned need = (unsigned)((r - kLockWindow + 1) * npairs);  // rounds issued per group
          for (unsigned g = 0; g < gridDim.y; ++g) {
            for (;;) {
              unsigned v;
              asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.prog + g) : "memory");
              if (v >= need) break;
              __nanosleep(100);
            }
          }
        }
        __syncwarp();
      }
      const int xrow = (int)(t * kPairN) + (int)crank * 128;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&empty[s], ph ^ 1u);  // the pair's MMA is done with this CTA's slot
        if (lane == 0) {
          const bool first = t == pair;
          const bool la = first || !(p.dbg & 128), lb = first || !(p.dbg & 256);
          if (crank == 0) mbar_arrive_expect_tx(&full[s], (la ? 2 : 0) * kBox + (lb ? 2 : 0) * kBox);  // both CTAs' boxes
          if (la) tma_load_2d_pair(sA + (size_t)s * kBox, &tmap_q, kb * kPBK, qrow0, full0 + 8u * (uint32_t)s);
          if (lb) tma_load_2d_pair(sB + (size_t)s * kBox, &tmap_x, kb * kPBK, xrow, full0 + 8u * (uint32_t)s);
        }
        __syncwarp();
        if (++s == NST) { s = 0; ph ^= 1u; }
      }
      if (lock && lane == 0) atomicAdd(p.prog + blockIdx.y, 1u);  // this pair issued round r
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (leader CTA)
    if (crank == 0) {
      // kind::f16: D fp32 (bit 4), A bf16 (bits 7-9 = 1), B bf16 (bits 10-12 = 1), both
      // K-major, N >> 3 at bit 17, M >> 4 at bit 24 (M = 256: the pair)
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kPairN >> 3) << 17) |
                             ((uint32_t)(256 >> 4) << 24);
      const uint64_t da0 = umma_desc(smem_u32(sA)), db0 = umma_desc(smem_u32(sB));
      const uint64_t dst = (uint64_t)kBox >> 4;  // one stage, in descriptor address units
      int s = 0;
      uint32_t ph = 0;
      int i = 0;
      for (int64_t t = pair; t < n_tiles; t += npairs, ++i) {
        const int acc = i & 1;
        const uint32_t aph = (uint32_t)(i >> 1) & 1u;
        mbar_wait(&tempty[acc], aph ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * kPairN);
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          if (lane == 0) {
            const uint64_t da = da0 + (uint64_t)s * dst, db = db0 + (uint64_t)s * dst;
            umma_bf16_pair(d_tmem, da, db, idesc, kb != 0);
            umma_bf16_pair(d_tmem, da + 2, db + 2, idesc, 1);
            umma_bf16_pair(d_tmem, da + 4, db + 4, idesc, 1);
            umma_bf16_pair(d_tmem, da + 6, db + 6, idesc, 1);
            umma_commit_pair(&empty[s], 3);  // frees slot s in both CTAs
          }
          __syncwarp();
          if (++s == NST) { s = 0; ph ^= 1u; }
        }
        if (lane == 0) umma_commit_pair(&tfull[acc], 3);  // accumulator ready in both CTAs
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------ epilogue warps 2..9 (both CTAs)
    const int e = warp - 2;
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int parity = e >> 2;     // tiles (and accumulator) of this warp
    const int m = quarter * 32 + lane;
    const bool active = m < nq;
    pdl_wait();  // k_norms: query norms and zeroed shared thresholds
    const float qn = active ? p.qnorm[qrow0 + m] : 0.f;
    const int slot = e * 32 + lane;
    float* xs = sXn + e * kPairN;
    constexpr int kCap = 32 * (P > 0 ? P : 2);
    const size_t cta_lin = (size_t)blockIdx.y * gridDim.x + blockIdx.x;
    uint64_t* buf = p.smem_bufs ? sBuf + (size_t)slot * kCap
                                : p.cand_buf + (cta_lin * kTcEpilogueThreads + slot) * kCap;
    using Topk = typename std::conditional<(KR > 0), RegTopk<(KR > 0 ? KR : 1)>, LaneTopk<(P > 0 ? P : 2)>>::type;
    Topk tk;
    if constexpr (KR > 0) tk.init(p.k, active ? p.gthr + qrow0 + m : nullptr);
    else tk.init(buf, active ? p.gthr + qrow0 + m : nullptr);
    if (!active) tk.tlim = __int_as_float(0x7f800000);  // +inf: never a candidate
    const uint32_t tempty0 = mapa_shared(smem_u32(tempty), 0);
    // the tile's |x_j|: lane l holds rows 8l .. 8l+7, loaded one tile ahead
    auto load_xn = [&](int64_t t, float4& x0, float4& x1) {
      x0 = make_float4(1.f, 1.f, 1.f, 1.f);
      x1 = x0;
      if (t >= n_tiles) return;
      const int64_t r0 = t * kPairN;
      const int nv = (int)((p.n_rows - r0) < kPairN ? (p.n_rows - r0) : kPairN);
      const float* src = p.xnorm + r0 + 8 * lane;
      if (8 * lane + 7 < nv) {
        x0 = __ldg(reinterpret_cast<const float4*>(src));
        x1 = __ldg(reinterpret_cast<const float4*>(src) + 1);
      } else {
        float tmp[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) tmp[u] = (8 * lane + u < nv) ? __ldg(src + u) : 1.f;
        x0 = make_float4(tmp[0], tmp[1], tmp[2], tmp[3]);
        x1 = make_float4(tmp[4], tmp[5], tmp[6], tmp[7]);
      }
    };
    const int64_t tstep = 2 * (int64_t)npairs;
    float4 xa, xb;
    load_xn(pair + parity * (int64_t)npairs, xa, xb);
    uint64_t pair_pub = 0;
    uint64_t gt_next = tk.peek_shared();
    const int acc = parity;
    int i = parity;
    for (int64_t t = pair + parity * (int64_t)npairs; t < n_tiles; t += tstep, i += 2) {
      const uint32_t aph = (uint32_t)(i >> 1) & 1u;
      const int64_t row0 = t * kPairN;
      const int nvalid = (int)((p.n_rows - row0) < kPairN ? (p.n_rows - row0) : kPairN);
      const uint64_t gt = gt_next;
      __syncwarp();
      reinterpret_cast<float4*>(xs)[2 * lane] = xa;
      reinterpret_cast<float4*>(xs)[2 * lane + 1] = xb;
      __syncwarp();
      load_xn(t + tstep, xa, xb);
      gt_next = tk.peek_shared();
      mbar_wait(&tfull[acc], aph);
      if (active) tk.raise(gt);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * kPairN);
#pragma unroll 1
      for (int c = 0; c < kPairN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tbase + c * 32, v);
        tmem_wait_ld();
        if (c == kPairN / 32 - 1) {  // every load of this accumulator has completed
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(tempty0 + 8u * (uint32_t)acc);
        }
        if constexpr (KR > 0) {
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
        const int left = nvalid - c * 32;
        if (left < 32) mask &= left > 0 ? ((1u << left) - 1u) : 0u;
        const int64_t gbase = p.gid_offset + (row0 + c * 32) * p.gid_stride;
        if constexpr (KR > 0) {
          if (__any_sync(kFull, mask != 0)) {
            while (mask) {  // per lane: insertion network, no warp synchronisation
              const int j = __ffs(mask) - 1;
              mask &= mask - 1;
              const float den = __fmaf_rn(qn, xc[j], p.sigma);
              const float vj = __uint_as_float(sel32(v, j));
              if (vj >= tk.tlim * den) {
                const int64_t gid = gbase + j * p.gid_stride;
                tk.insert(make_key(__fdiv_rn(vj, den), gid));
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
            tk.ensure_room(32, p.k);
#pragma unroll
            for (int j4 = 0; j4 < 8; ++j4) {
              const float4 x4 = lds128f(xc + 4 * j4);
              const float xx[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int j = 4 * j4 + u;
                if ((mask >> j) & 1u) {
                  const float den = __fmaf_rn(qn, xx[u], p.sigma);
                  const int64_t gid = gbase + j * p.gid_stride;
                  tk.append(make_key(__fdiv_rn(__uint_as_float(v[j]), den), gid));
                }
              }
            }
          } else if (__any_sync(kFull, mask != 0)) {
            while (__any_sync(kFull, mask != 0)) {
              uint64_t key = 0;
              if (mask) {
                const int j = __ffs(mask) - 1;
                mask &= mask - 1;
                const float den = __fmaf_rn(qn, xc[j], p.sigma);
                const int64_t gid = gbase + j * p.gid_stride;
                key = make_key(__fdiv_rn(__uint_as_float(sel32(v, j)), den), gid);
              }
              tk.push(key, p.k);
            }
          }
        }
      }
      if constexpr (KR > 0) tk.publish();
    }
    const int npl = npairs * lists_per_cta;  // lists per query
    if (KR > 0 && p.merge_in_cta) {
      // Merge the two parity states of each query in the CTA, with the (now idle) stage
      // ring as scratch: every epilogue warp has consumed its last accumulator, so every
      // MMA of the pair -- and with it every read of this CTA's ring -- has completed.
      uint64_t* scratch = reinterpret_cast<uint64_t*>(sA);
      asm volatile("bar.sync 2, %0;" ::"n"(kPEpiWarps * 32) : "memory");
      if constexpr (KR > 0) tk.flush(scratch + (size_t)slot * KR);
      asm volatile("bar.sync %0, 64;" ::"r"(3 + quarter) : "memory");  // the quarter's two warps
      if (parity == 0 && active) {
        const uint64_t* a = scratch + (size_t)slot * (KR > 0 ? KR : 1);
        const uint64_t* b = scratch + (size_t)(slot + 128) * (KR > 0 ? KR : 1);  // warp e + 4, same lane
        uint64_t* o = p.out + ((size_t)(qrow0 + m) * npl + pair) * (size_t)p.k;
        int ia = 0, ib = 0;
        for (int r = 0; r < p.k; ++r) {
          const uint64_t x = a[ia], y = b[ib];
          if (x >= y) { o[r] = x; ++ia; } else { o[r] = y; ++ib; }
        }
      }
    } else {
      uint64_t* out = active ? p.out + ((size_t)(qrow0 + m) * npl + (size_t)pair * 2 + parity) * (size_t)p.k
                             : nullptr;
      if constexpr (KR > 0) {
        tk.flush(out);
      } else {
        // buffers in global memory: sort in the idle stage ring (see k_scan_tc)
        uint64_t* scratch = nullptr;
        if (!p.smem_bufs && (size_t)NST * kBox >= (size_t)kPEpiWarps * 32 * 32 * 8) {
          asm volatile("bar.sync 2, %0;" ::"n"(kPEpiWarps * 32) : "memory");
          scratch = reinterpret_cast<uint64_t*>(sA) + (size_t)slot * 32;
        }
        tk.flush(out, p.k, scratch);
      }
    }
  }
  __syncthreads();
  cluster_sync_all();  // no CTA leaves (or frees TMEM) while its peer may still signal it
  if (p.prog && threadIdx.x == 0) {  // the last CTA of the launch resets the lockstep counters
    if (atomicAdd(p.exit_cnt, 1u) == gridDim.x * gridDim.y - 1) {
      for (unsigned g = 0; g < gridDim.y; ++g) p.prog[g] = 0u;
      __threadfence();
      *p.exit_cnt = 0u;
    }
  }
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(kPTmemCols));
  }
}

// ------------------------------------------------------------------ host side

static size_t pair_smem(int nst, int buf_bytes) {
  return (size_t)dyn_smem_pad() + (size_t)nst * 2 * kBox + (2 * (size_t)nst + 2 * kPAcc + 2) * 8 + kPEpiWarps * kPairN * 4 +
         kQPerCta * 8 + (size_t)buf_bytes;
}

static int pair_stages(int buf_bytes) {
  const long avail = (long)kPMaxSmem - (long)pair_smem(0, buf_bytes);
  const long n = avail / (2 * kBox + 16);
  return (int)(n > 8 ? 8 : n);
}

typedef CUresult (*EncodeTiledFnP)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFnP encode_fn() {
  static EncodeTiledFnP fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    fn = (EncodeTiledFnP)f;
  }
  return fn;
}

template <int P, int KR>
static cudaError_t launch_pair_t(const TcPlan* t, const CUtensorMap& tq, const PairArgs& a, dim3 grid,
                                 cudaStream_t st) {
  const size_t smem = pair_smem(a.n_stages, a.smem_bufs ? kTcEpilogueThreads * 32 * P * 8 : 0);
  auto kern = k_scan_pair<P, KR>;
  cudaError_t e = set_smem_attrs_once((const void*)kern, kPMaxSmem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kPThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 2;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, *reinterpret_cast<const CUtensorMap*>(t->tmap_x), tq, a);
}

static cudaError_t launch_pair(const TcPlan* t, const CUtensorMap& tq, const PairArgs& a, dim3 g, cudaStream_t st) {
  if (a.k <= 1) return launch_pair_t<0, 1>(t, tq, a, g, st);
  if (a.k <= 2) return launch_pair_t<0, 2>(t, tq, a, g, st);
  if (a.k <= 4) return launch_pair_t<0, 4>(t, tq, a, g, st);
  if (a.k <= 8) return launch_pair_t<0, 8>(t, tq, a, g, st);
  if (a.k <= 16) return launch_pair_t<0, 16>(t, tq, a, g, st);
  if (a.k <= 32) return launch_pair_t<0, 32>(t, tq, a, g, st);
  switch (topk_P(a.k)) {
    case 2: return launch_pair_t<2, 0>(t, tq, a, g, st);
    case 4: return launch_pair_t<4, 0>(t, tq, a, g, st);
    case 8: return launch_pair_t<8, 0>(t, tq, a, g, st);
    case 16: return launch_pair_t<16, 0>(t, tq, a, g, st);
  }
  return cudaErrorInvalidValue;
}

bool tc_pair_usable(const TcPlan* t) { return t->ok && t->grid >= 2 && encode_fn() != nullptr; }

remoe_status_t tc_pair_scan(TcPlan* t, const uint16_t* q, const float* qnorm, int bc, int k, float sigma,
                            const float* xnorm, int64_t n_rows, int64_t gid_offset, int64_t gid_stride,
                            uint64_t* cand_buf, unsigned long long* gthr, uint64_t* lists, cudaStream_t st,
                            int* launches, int* lists_per_query) {
  if (!tc_pair_usable(t)) return REMOE_ERR_UNSUPPORTED;
  const int D = t->dim;
  const int buf_bytes = k <= 32 ? 0 : kTcEpilogueThreads * 32 * topk_P(k) * 8;
  const bool smem_bufs = k > 32 && pair_stages(buf_bytes) >= 4;
  int nst = pair_stages(smem_bufs ? buf_bytes : 0);
  if (t->kn.stages >= 2 && t->kn.stages < nst) nst = t->kn.stages;  // REMOE_TC_STAGES (experiments)
  const int KR = k <= 1 ? 1 : k <= 2 ? 2 : k <= 4 ? 4 : k <= 8 ? 8 : k <= 16 ? 16 : 32;
  const bool in_cta = k <= 32 && (size_t)nst * kBox >= (size_t)kTcEpilogueThreads * KR * 8;
  const int lists_per_cta = in_cta ? 1 : 2;
  // Query groups of 256 (one per pair); every group's pairs walk the store tiles in the
  // same order, so a tile is read from HBM once per launch and by the other groups from
  // L2.  Groups per launch g: minimise launches x (one store read + the launch's MMA time
  // on g * floor(pairs / g) pairs), with one group's MMA time ~ one store read (the ridge,
  // B ~ 254, is about one group of 256); overlap is not assumed.
  const int pairs_max = t->grid / 2;
  const int n_groups = (bc + 2 * kQPerCta - 1) / (2 * kQPerCta);
  int best_g = 1;
  double best_cost = 1e300;
  for (int g = 1; g <= (n_groups < pairs_max ? n_groups : pairs_max); ++g) {
    const int nl = (n_groups + g - 1) / g;
    const double cost = nl * (1.0 + (double)g * pairs_max / (double)(g * (pairs_max / g)));
    if (cost < best_cost - 1e-9) { best_cost = cost; best_g = g; }
  }
  const int gpl = best_g;
  const int ppg = pairs_max / gpl;  // pairs per group
  *lists_per_query = ppg * lists_per_cta;
  EncodeTiledFnP enc = encode_fn();
  for (int g0 = 0; g0 < n_groups; g0 += gpl) {
    const int ng = n_groups - g0 < gpl ? n_groups - g0 : gpl;
    const int s0 = g0 * 2 * kQPerCta;
    const int nq = bc - s0 < ng * 2 * kQPerCta ? bc - s0 : ng * 2 * kQPerCta;
    alignas(64) CUtensorMap tq;
    const cuuint64_t gdim[2] = {(cuuint64_t)D, (cuuint64_t)nq};
    const cuuint64_t gstride[1] = {(cuuint64_t)D * 2};
    const cuuint32_t box[2] = {(cuuint32_t)kPBK, 128u};
    const cuuint32_t estr[2] = {1, 1};
    if (enc(&tq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(q + (size_t)s0 * D), gdim, gstride,
            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, t->kn.promotion(),
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return REMOE_ERR_CUDA;
    PairArgs a{};
    a.xnorm = xnorm;
    a.n_rows = n_rows;
    a.gid_offset = gid_offset;
    a.gid_stride = gid_stride;
    a.dim = D;
    a.qnorm = qnorm + s0;
    a.nq = nq;
    a.k = k;
    a.sigma = sigma;
    a.n_stages = nst;
    a.cand_buf = cand_buf;
    a.gthr = gthr + s0;
    a.out = lists + (size_t)s0 * (*lists_per_query) * k;
    a.smem_bufs = smem_bufs ? 1 : 0;
    a.merge_in_cta = in_cta ? 1 : 0;
    a.dbg = t->kn.dbg;
    if (ng > 1 && ng <= kLockMaxGroups && t->pair_sync && t->kn.lockstep) {
      a.prog = t->pair_sync;
      a.exit_cnt = t->pair_sync + 16;
    }
    if (t->kn.verbose)
      fprintf(stderr, "[remoe] pair scan grid (%d,%d) stages %d lists/query %d\n", 2 * ppg, ng, nst,
              *lists_per_query);
    if (launch_pair(t, tq, a, dim3((unsigned)(2 * ppg), (unsigned)ng), st) != cudaSuccess) return REMOE_ERR_CUDA;
    ++*launches;
  }
  return REMOE_OK;
}

}  // namespace remoe
