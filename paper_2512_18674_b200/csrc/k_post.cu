// k_post.cu -- the small kernels around the scan (sm_100a):
//   S0/S1 row norms, S4/S5 key-list merge with fused S6+S7 (softmax + gather + weighted
//   reduce; merge.cuh), the multi-GPU partial-prediction sum in rank order, the fused
//   exchange's sequence counter, S8 expert plan, build validation.
#include "common.cuh"
#include "host_util.h"
#include "kernels.h"
#include "merge.cuh"

#include <algorithm>

namespace remoe {

// ---------------------------------------------------------------- S0 / S1 norms
// |x| = sqrt(sum_d x_d^2) (Eq. 11 denominator).  One warp per row; lane
// partial sums over 16-byte chunks in ascending chunk order, fixed xor butterfly.
__global__ void k_norms(const uint16_t* __restrict__ x, int64_t n, int dim, float* __restrict__ out,
                        unsigned long long* __restrict__ zero_u64, int64_t zero_stride) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  if (zero_u64 && lane == 0) zero_u64[row] = 0ull;
  if (zero_u64 && zero_stride && lane == 1) zero_u64[row + zero_stride] = 0ull;
  const uint16_t* xr = x + row * dim;
  float s = 0.f;
  for (int c = lane; c < (dim >> 3); c += 32) {
    const uint4 w = *reinterpret_cast<const uint4*>(xr + c * 8);
    const float v[8] = {bf_lo(w.x), bf_hi(w.x), bf_lo(w.y), bf_hi(w.y),
                        bf_lo(w.z), bf_hi(w.z), bf_lo(w.w), bf_hi(w.w)};
#pragma unroll
    for (int j = 0; j < 8; ++j) s = __fmaf_rn(v[j], v[j], s);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(kFull, s, off);
  if (lane == 0) out[row] = __fsqrt_rn(s);
}

cudaError_t launch_norms(const uint16_t* x, int64_t n, int dim, float* out, cudaStream_t st,
                         unsigned long long* zero_u64, int64_t zero_stride) {
  if (n <= 0) return cudaSuccess;
  const int wpb = 8;
  const int64_t grid = (n + wpb - 1) / wpb;
  cudaError_t e = set_smem_attrs_once((const void*)k_norms, 0);
  if (e != cudaSuccess) return e;
  k_norms<<<(unsigned)grid, wpb * 32, 0, st>>>(x, n, dim, out, zero_u64, zero_stride);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(256) k_merge(const uint64_t* __restrict__ in, int n_lists,
                                               int64_t qstride, int64_t lstride, int list_len, int k,
                                               uint64_t* __restrict__ out,
                                               unsigned long long* __restrict__ set_thr,
                                               unsigned long long* __restrict__ lower,
                                               FinalizeArgs fin, unsigned* __restrict__ bump, int reset_lower,
                                               PeerXchg px, unsigned* __restrict__ split_cnt) {
  __shared__ MergeScratch S;
  pdl_wait();  // the scan's lists and thresholds
  // the chunk's sequence number and buffer parity, on the device (offsets, not edits of the
  // pointer arrays: indexing a modified parameter array would move it to the local stack)
  unsigned long long seq = px.seq;
  int64_t key_off = 0, pred_off = 0;
  if (px.G > 0 && px.seq_ptr) {
    seq = *px.seq_ptr + 1;
    if (seq & 1) {
      in += px.in_par;
      key_off = px.key_par;
      pred_off = px.pred_par;
    }
  }
  // (key loads are ld.global.cg: L2-coherent, so keys a peer stored over NVLink during
  // this kernel's lifetime -- fused exchange 1 -- are never read through a stale L1 line)
  if (px.G > 0 && px.wait_flags) peer_wait(px.wait_flags, px.G, seq);  // fused exchange 1: every rank's keys
  // the scan is complete: a new seeding epoch for the next chunk (stale published keys of
  // this one can never be taken for the next one's)
  if (bump && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) atomicAdd(bump, 1u);
  // grid (B, n_split): split y redoes the (cheap) selection and reduces columns
  // [y * chunk, (y + 1) * chunk) of the prediction -- the gather of the k activation rows,
  // latency-bound in one CTA, spreads over n_split SMs; split 0 writes the keys, ids, scores
  const int n_split = (int)gridDim.y;
  const int64_t chunk = ((fin.LE + n_split - 1) / n_split + 3) & ~int64_t(3);
  const int64_t j0 = (int64_t)blockIdx.y * chunk;
  const int64_t j1 = j0 + chunk < fin.LE ? j0 + chunk : fin.LE;
  merge_query(in, blockIdx.x, n_lists, qstride, lstride, list_len, k, out, set_thr, lower, fin, reset_lower, &px,
              threadIdx.x, [] { __syncthreads(); }, S, j0, j1, blockIdx.y == 0, split_cnt, n_split, key_off, pred_off);
  if (px.G > 0 && px.flag_dst[0]) peer_signal(px, seq);
}

cudaError_t launch_merge(const uint64_t* in, int B, int n_lists, int64_t qstride, int64_t lstride,
                         int k, uint64_t* out, cudaStream_t st, unsigned long long* set_thr,
                         unsigned long long* lower, const FinalizeArgs* fin, int list_len,
                         unsigned* bump, bool reset_lower, const PeerXchg* px, unsigned* split_cnt) {
  if (B <= 0) return cudaSuccess;
  if (k > 256) return cudaErrorInvalidValue;
  if (list_len <= 0) list_len = k;
  FinalizeArgs f{};
  if (fin) f = *fin;
  PeerXchg x{};
  if (px) x = *px;
  cudaError_t e = set_smem_attrs_once((const void*)k_merge, 0);
  if (e != cudaSuccess) return e;
  // column splits of the finalize: ~2 CTAs per SM in total, >= 256 columns per split
  int n_split = 1;
  if (split_cnt && fin && f.pred && f.n_pred_peer == 0 && x.G == 0 && !set_thr) {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
      cudaGetLastError();
      sms = 148;
    }
    n_split = (int)std::max<int64_t>(1, std::min<int64_t>({8, (2 * (int64_t)sms) / B, f.LE / 256}));
  }
  return launch_pdl(k_merge, dim3(B, n_split), dim3(256), 0, st, in, n_lists, qstride, lstride, list_len, k, out,
                    set_thr, lower, f, bump, reset_lower ? 1 : 0, x, split_cnt);
}

// Grid (B, ceil(LE / 256)): every CTA recomputes its query's k weights (k <= 256
// exps, cheap) and produces 256 outputs; chunk 0 also writes ids and scores.
__global__ void __launch_bounds__(256) k_finalize(const uint64_t* __restrict__ top, int k, FinalizeArgs f) {
  __shared__ MergeScratch S;
  const int b = blockIdx.x;
  const int64_t j0 = (int64_t)blockIdx.y * blockDim.x;
  pdl_wait();
  finalize_query(top + (int64_t)b * k, k, b, f, j0, j0 + blockDim.x < f.LE ? j0 + blockDim.x : f.LE,
                 blockIdx.y == 0, threadIdx.x, [] { __syncthreads(); }, S);
}

cudaError_t launch_finalize(const uint64_t* top, int B, int k, const FinalizeArgs& f, cudaStream_t st) {
  if (B <= 0) return cudaSuccess;
  if (k > 256) return cudaErrorInvalidValue;
  const unsigned chunks = f.pred ? (unsigned)((f.LE + 255) / 256) : 1u;
  cudaError_t e = set_smem_attrs_once((const void*)k_finalize, 0);
  if (e != cudaSuccess) return e;
  return launch_pdl(k_finalize, dim3((unsigned)B, chunks), dim3(256), 0, st, top, k, f);
}

// ---------------------------------------------------------------- multi-GPU S7 combine
// out[i] = parts[0][i] + parts[1][i] + ... + parts[G-1][i], g ascending: every rank sums
// the same gathered partials in the same order, so all ranks (and every batch position)
// get identical bits (ncclAllReduce's ring order would not guarantee that).
__global__ void k_psum(const float* parts, int G, int64_t stride, int64_t n, float* __restrict__ out,
                       const unsigned long long* __restrict__ wait_flags, unsigned long long seq,
                       const unsigned long long* __restrict__ seq_ptr, int64_t parts_par) {
  pdl_wait();
  if (seq_ptr) {
    seq = *seq_ptr + 1;
    if (seq & 1) parts += parts_par;
  }
  if (wait_flags) peer_wait(wait_flags, G, seq);  // fused exchange 2: every rank's partial landed
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  if ((stride & 3) == 0 && (n & 3) == 0 && ((reinterpret_cast<uintptr_t>(parts) | reinterpret_cast<uintptr_t>(out)) & 15) == 0) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n >> 2); i += step) {
      float4 acc = __ldcg(reinterpret_cast<const float4*>(parts) + i);
      for (int g = 1; g < G; ++g) {
        const float4 v = __ldcg(reinterpret_cast<const float4*>(parts + g * stride) + i);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      reinterpret_cast<float4*>(out)[i] = acc;
    }
    return;
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += step) {
    float acc = parts[i];
    for (int g = 1; g < G; ++g) acc += parts[g * stride + i];
    out[i] = acc;
  }
}

cudaError_t launch_psum(const float* parts, int G, int64_t part_stride, int64_t n, float* out, cudaStream_t st,
                        const unsigned long long* wait_flags, unsigned long long seq,
                        const unsigned long long* seq_ptr, int64_t parts_par) {
  if (n <= 0) return cudaSuccess;
  const int64_t units = (n + 3) / 4;
  const unsigned grid = (unsigned)std::min<int64_t>((units + 255) / 256, 148 * 8);
  cudaError_t e = set_smem_attrs_once((const void*)k_psum, 0);
  if (e != cudaSuccess) return e;
  return launch_pdl(k_psum, dim3(grid), dim3(256), 0, st, parts, G, part_stride, n, out, wait_flags, seq, seq_ptr,
                    parts_par);
}

__global__ void k_seq_bump(unsigned long long* seq) {
  pdl_wait();
  *seq += 1ull;
}

cudaError_t launch_seq_bump(unsigned long long* seq, cudaStream_t st) {
  return launch_pdl(k_seq_bump, dim3(1), dim3(1), 0, st, seq);
}

// ---------------------------------------------------------------- S8 plan
// Remote-expert selection: expert e of (b, l) is cold iff its rank under
// (value asc, index asc) is < n_cold.  One warp per (b, l); E <= 256.
__global__ void __launch_bounds__(128) k_plan(const float* __restrict__ pred, int64_t n_rows, int E,
                                              int n_cold, uint8_t* __restrict__ mask) {
  __shared__ float v[4][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 4 + warp;
  if (row >= n_rows) return;
  const float* pr = pred + row * E;
  for (int e = lane; e < E; e += 32) v[warp][e] = pr[e];
  __syncwarp();
  for (int e = lane; e < E; e += 32) {
    const float x = v[warp][e];
    int rank = 0;
    for (int f = 0; f < E; ++f) {
      const float y = v[warp][f];
      rank += (y < x) || (y == x && f < e);
    }
    mask[row * E + e] = rank < n_cold ? 1 : 0;
  }
}

cudaError_t launch_plan(const float* pred, int B, int L, int E, int n_cold, uint8_t* mask,
                        cudaStream_t st) {
  const int64_t rows = (int64_t)B * L;
  if (rows <= 0) return cudaSuccess;
  k_plan<<<(unsigned)((rows + 3) / 4), 128, 0, st>>>(pred, rows, E, n_cold, mask);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- build validation
__global__ void k_validate(const uint16_t* __restrict__ x, int64_t nx, const float* __restrict__ act,
                           int64_t n_act_rows, int E, unsigned long long* bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long cnt = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nx; i += stride)
    cnt += ((x[i] & 0x7F80u) == 0x7F80u);  // inf / nan exponent
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_act_rows; r += stride) {
    const float* a = act + r * E;
    float s = 0.f;
    bool neg = false;
    for (int e = 0; e < E; ++e) { s += a[e]; neg |= !(a[e] >= 0.f) || isinf(a[e]); }
    cnt += neg || !(fabsf(s - 1.f) <= 1e-3f);
  }
  if (cnt) atomicAdd(bad, cnt);
}

cudaError_t launch_validate(const uint16_t* x, int64_t n, int dim, const float* act, int64_t LE_rows,
                            int E, unsigned long long* bad, cudaStream_t st) {
  k_validate<<<148 * 4, 256, 0, st>>>(x, n * dim, act, LE_rows, E, bad);
  return cudaGetLastError();
}

}  // namespace remoe
