// k_scan_simt.cu -- S2+S3 for few queries: TMA-staged streaming scan on CUDA cores.
//
// score_ij = (q_i . x_j) / (|q_i||x_j| + sigma)  (Eq. 11, reduced per DESIGN R2)
// followed by an exact per-CTA running top-k per query (BF top-alpha).
//
// Design:
//   * persistent grid, one CTA per SM; CTA c owns the contiguous rows
//     [c*R, (c+1)*R) of this rank's shard, so its whole input is one contiguous
//     byte range streamed by the TMA engine with 1-D bulk copies
//     (cp.async.bulk ... mbarrier::complete_tx) into an NST-deep ring of
//     32 KB stages -- no per-thread address generation, ~128 KB in flight per SM;
//   * warps 0-7 compute: lanes split D into 16-byte chunks (ld.shared.v4, bank
//     conflict free), bf16 -> fp32 is a shift, fp32 FMA chains, a fixed xor
//     butterfly across lanes.  The summation order depends only on D, never on
//     the batch position of the query or on sharding;
//   * warp 8 is the epilogue: lane b owns query b's running top-k (LaneTopk,
//     common.cuh): one 64-bit compare per score against a register threshold;
//   * warp 9 lane 0 is the TMA producer.
#include "common.cuh"
#include "host_util.h"
#include "kernels.h"

namespace remoe {

namespace {
constexpr int kComputeWarps = 8;
constexpr int kThreads = (kComputeWarps + 2) * 32;
constexpr int kRB = 4;  // rows per compute step per warp
}  // namespace

template <int BQ, int P>
__global__ void __launch_bounds__(kThreads, 1) k_scan_simt(SimtScanParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int D = p.dim;
  const int D8 = D >> 3;
  const int SR = p.stage_rows;
  const int NST = p.n_stages_ring;
  const size_t stage_bytes = (size_t)SR * D * 2;

  uint8_t* stages = smem;
  float* qs = reinterpret_cast<float*>(smem + (size_t)NST * stage_bytes);       // [BQ][D]
  float* S = qs + (size_t)BQ * D;                                               // [2][SR][BQ]
  float* qn = S + 2 * SR * BQ;                                                  // [BQ]
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(qn + BQ) + 7) & ~uintptr_t(7));
  uint64_t* full = bars;
  uint64_t* empty = bars + NST;
  uint64_t* sfull = bars + 2 * NST;
  uint64_t* sempty = bars + 2 * NST + 2;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  const int64_t per = (p.n_rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = (int64_t)cta * per < p.n_rows ? (int64_t)cta * per : p.n_rows;
  const int64_t r1 = r0 + per < p.n_rows ? r0 + per : p.n_rows;
  const int n_iter = (int)((r1 - r0 + SR - 1) / SR);

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], kComputeWarps); }
    for (int s = 0; s < 2; ++s) { mbar_init(&sfull[s], kComputeWarps); mbar_init(&sempty[s], 1); }
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < BQ * D; i += blockDim.x) {
    const int b = i / D, d = i - b * D;
    const uint16_t bits = b < p.nq ? p.q[(size_t)b * D + d] : (uint16_t)0;
    qs[i] = __uint_as_float((uint32_t)bits << 16);
  }
  if (threadIdx.x < BQ) qn[threadIdx.x] = threadIdx.x < p.nq ? p.qnorm[threadIdx.x] : 0.f;
  __syncthreads();

  if (warp < kComputeWarps) {
    // ------------------------------------------------ compute warps
    for (int it = 0; it < n_iter; ++it) {
      const int st = it % NST;
      const uint32_t ph = (uint32_t)(it / NST) & 1u;
      const int64_t rbase = r0 + (int64_t)it * SR;
      const int rows = (int)((r1 - rbase) < SR ? (r1 - rbase) : SR);
      const int sb = it & 1;
      const uint32_t sph = (uint32_t)(it >> 1) & 1u;
      const uint8_t* stg = stages + (size_t)st * stage_bytes;
      float* Sb = S + sb * SR * BQ;
      mbar_wait(&full[st], ph);
      mbar_wait(&sempty[sb], sph ^ 1u);
      const uint32_t stg_s = smem_u32(stg), qs_s = smem_u32(qs);
      for (int i = warp * kRB; i < rows; i += kComputeWarps * kRB) {
        float acc[kRB][BQ];
#pragma unroll
        for (int r = 0; r < kRB; ++r)
#pragma unroll
          for (int b = 0; b < BQ; ++b) acc[r][b] = 0.f;
        for (int c = lane; c < D8; c += 32) {
          float xf[kRB][8];
#pragma unroll
          for (int r = 0; r < kRB; ++r) {
            uint4 w = make_uint4(0, 0, 0, 0);
            if (i + r < rows)
              asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                           : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                           : "r"(stg_s + (uint32_t)(((i + r) * D + c * 8) * 2)));
            xf[r][0] = bf_lo(w.x); xf[r][1] = bf_hi(w.x);
            xf[r][2] = bf_lo(w.y); xf[r][3] = bf_hi(w.y);
            xf[r][4] = bf_lo(w.z); xf[r][5] = bf_hi(w.z);
            xf[r][6] = bf_lo(w.w); xf[r][7] = bf_hi(w.w);
          }
#pragma unroll
          for (int b = 0; b < BQ; ++b) {
            float4 qa, qb;
            const uint32_t qaddr = qs_s + (uint32_t)((b * D + c * 8) * 4);
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                         : "=f"(qa.x), "=f"(qa.y), "=f"(qa.z), "=f"(qa.w) : "r"(qaddr));
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                         : "=f"(qb.x), "=f"(qb.y), "=f"(qb.z), "=f"(qb.w) : "r"(qaddr + 16));
#pragma unroll
            for (int r = 0; r < kRB; ++r) {
              float a = acc[r][b];
              a = __fmaf_rn(xf[r][0], qa.x, a); a = __fmaf_rn(xf[r][1], qa.y, a);
              a = __fmaf_rn(xf[r][2], qa.z, a); a = __fmaf_rn(xf[r][3], qa.w, a);
              a = __fmaf_rn(xf[r][4], qb.x, a); a = __fmaf_rn(xf[r][5], qb.y, a);
              a = __fmaf_rn(xf[r][6], qb.z, a); a = __fmaf_rn(xf[r][7], qb.w, a);
              acc[r][b] = a;
            }
          }
        }
        // fixed xor butterfly: every lane ends with the full sums
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)
#pragma unroll
          for (int r = 0; r < kRB; ++r)
#pragma unroll
            for (int b = 0; b < BQ; ++b) acc[r][b] += __shfl_xor_sync(kFull, acc[r][b], off);
        // lane j < kRB*BQ computes the score of (row j / BQ, query j % BQ): one division
        // per lane, all in parallel
        float mine = 0.f;
#pragma unroll
        for (int r = 0; r < kRB; ++r)
#pragma unroll
          for (int b = 0; b < BQ; ++b)
            if (lane == r * BQ + b) mine = acc[r][b];
        const int rr = lane / BQ, bb = lane % BQ;
        if (lane < kRB * BQ && i + rr < rows)
          Sb[(i + rr) * BQ + bb] = eq11(mine, qn[bb], __ldg(p.xnorm + rbase + i + rr), p.sigma);
      }
      __syncwarp();
      if (lane == 0) { mbar_arrive(&empty[st]); mbar_arrive(&sfull[sb]); }
    }
  } else if (warp == kComputeWarps) {
    // ------------------------------------------------ epilogue: lane b owns query b
    LaneTopk<P> tk;
    tk.init(p.cand_buf + ((size_t)cta * 32 + lane) * LaneTopk<P>::CAP,
            lane < p.nq ? p.gthr + lane : nullptr);
    for (int it = 0; it < n_iter; ++it) {
      const int sb = it & 1;
      const uint32_t sph = (uint32_t)(it >> 1) & 1u;
      const int64_t rbase = r0 + (int64_t)it * SR;
      const int rows = (int)((r1 - rbase) < SR ? (r1 - rbase) : SR);
      const float* Sb = S + sb * SR * BQ;
      const uint64_t gt = tk.peek_shared();
      mbar_wait(&sfull[sb], sph);
      tk.raise(gt);
      for (int r = 0; r < rows; ++r) {
        // host guarantees nq <= BQ
        const uint64_t key = lane < p.nq ? make_key(Sb[r * BQ + lane], p.gid_offset + rbase + r) : 0ull;
        tk.push(key, p.k);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sempty[sb]);
    }
    uint64_t* out = lane < p.nq
                        ? p.out + ((size_t)lane * gridDim.x + cta) * (size_t)p.k
                        : nullptr;
    tk.flush(out, p.k);
  } else if (lane == 0) {
    // ------------------------------------------------ TMA producer
    for (int it = 0; it < n_iter; ++it) {
      const int st = it % NST;
      const uint32_t ph = (uint32_t)(it / NST) & 1u;
      const int64_t rbase = r0 + (int64_t)it * SR;
      const int rows = (int)((r1 - rbase) < SR ? (r1 - rbase) : SR);
      const uint32_t bytes = (uint32_t)rows * (uint32_t)D * 2u;
      mbar_wait(&empty[st], ph ^ 1u);
      mbar_arrive_expect_tx(&full[st], bytes);
      bulk_g2s(stages + (size_t)st * stage_bytes, p.x + (size_t)rbase * D, bytes, &full[st]);
    }
  }
}

size_t simt_smem_bytes(int BQ, int dim, int stage_rows, int n_stages_ring) {
  size_t s = (size_t)n_stages_ring * stage_rows * dim * 2;
  s += (size_t)BQ * dim * 4 + 2 * (size_t)stage_rows * BQ * 4 + (size_t)BQ * 4;
  s = (s + 7) & ~size_t(7);
  s += (2 * (size_t)n_stages_ring + 4) * 8;
  return s;
}

template <int BQ, int P>
static cudaError_t launch_t(const SimtScanParams& p, int grid, size_t smem, cudaStream_t st) {
  auto kern = k_scan_simt<BQ, P>;
  cudaError_t e = set_smem_attrs_once((const void*)kern, kSimtMaxSmem);
  if (e != cudaSuccess) return e;
  kern<<<grid, kThreads, smem, st>>>(p);
  return cudaGetLastError();
}

template <int BQ>
static cudaError_t launch_bq(const SimtScanParams& p, int P, int grid, size_t smem, cudaStream_t st) {
  switch (P) {
    case 2: return launch_t<BQ, 2>(p, grid, smem, st);
    case 4: return launch_t<BQ, 4>(p, grid, smem, st);
    case 8: return launch_t<BQ, 8>(p, grid, smem, st);
    case 16: return launch_t<BQ, 16>(p, grid, smem, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_scan_simt(const SimtScanParams& p, int BQ, int grid, cudaStream_t st) {
  const int P = topk_P(p.k);
  const size_t smem = simt_smem_bytes(BQ, p.dim, p.stage_rows, p.n_stages_ring);
  switch (BQ) {
    case 1: return launch_bq<1>(p, P, grid, smem, st);
    case 2: return launch_bq<2>(p, P, grid, smem, st);
    case 4: return launch_bq<4>(p, P, grid, smem, st);
    case 8: return launch_bq<8>(p, P, grid, smem, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace remoe
