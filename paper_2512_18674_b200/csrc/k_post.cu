// k_post.cu -- the small kernels around the scan (sm_100a):
//   S0/S1 row norms, S4/S5 key-list merge, S6+S7 softmax + gather + weighted
//   reduce, the multi-GPU winner-row gather, S8 expert plan, build validation.
#include "common.cuh"
#include "kernels.h"

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
  k_norms<<<(unsigned)grid, wpb * 32, 0, st>>>(x, n, dim, out, zero_u64, zero_stride);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- S4 / S5 merge
// One CTA per query: 8 warps each keep a warp-shared top-k over a subset of the
// lists, then warp 0 merges the 8 partial results.  Exact.
template <int P>
__global__ void __launch_bounds__(256) k_merge(const uint64_t* __restrict__ in, int n_lists,
                                               int64_t qstride, int64_t lstride, int k,
                                               uint64_t* __restrict__ out,
                                               unsigned long long* __restrict__ set_thr) {
  constexpr int CAP = 32 * P;
  extern __shared__ __align__(16) uint64_t msm[];
  uint64_t* buf = msm;               // [8][CAP]
  uint64_t* part = msm + 8 * CAP;    // [8][k]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x;
  const uint64_t* base = in + (int64_t)b * qstride;
  WarpTopk<P> tk;
  tk.init(buf + warp * CAP);
  for (int l = warp; l < n_lists; l += 8) {
    const uint64_t* li = base + (int64_t)l * lstride;
    for (int i0 = 0; i0 < k; i0 += 32) {
      const uint64_t key = (i0 + lane < k) ? li[i0 + lane] : 0ull;
      // lists are sorted descending: once a chunk has nothing above the
      // threshold, the rest of the list cannot contribute either
      if (!__any_sync(kFull, key > tk.thr)) break;
      tk.push(key, k);
    }
  }
  tk.finish(part + warp * k, k);
  __syncthreads();
  if (warp == 0) {
    tk.init(buf);
    for (int w = 0; w < 8; ++w)
      for (int i0 = 0; i0 < k; i0 += 32) {
        const uint64_t key = (i0 + lane < k) ? part[w * k + i0 + lane] : 0ull;
        tk.push(key, k);
      }
    tk.finish(out + (int64_t)b * k, k);
    if (set_thr) {
      // seeding: the k-th best key of a subset of rows, minus one (strict lower bound,
      // the subset's own rows stay admissible in the full scan)
      __syncwarp();
      if (lane == 0) {
        const uint64_t kth = out[(int64_t)b * k + k - 1];
        set_thr[b] = kth ? kth - 1 : 0ull;
      }
    }
  }
}

template <int P>
static cudaError_t merge_t(const uint64_t* in, int B, int n_lists, int64_t qstride, int64_t lstride,
                           int k, uint64_t* out, unsigned long long* set_thr, cudaStream_t st) {
  const size_t smem = (size_t)8 * (32 * P + k) * sizeof(uint64_t);
  cudaError_t e = cudaFuncSetAttribute(k_merge<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_merge<P><<<B, 256, smem, st>>>(in, n_lists, qstride, lstride, k, out, set_thr);
  return cudaGetLastError();
}

cudaError_t launch_merge(const uint64_t* in, int B, int n_lists, int64_t qstride, int64_t lstride,
                         int k, uint64_t* out, cudaStream_t st, unsigned long long* set_thr) {
  if (B <= 0) return cudaSuccess;
  switch (topk_P(k)) {  // WarpTopk needs CAP = 32*P >= k + 32: topk_P guarantees it
    case 2: return merge_t<2>(in, B, n_lists, qstride, lstride, k, out, set_thr, st);
    case 4: return merge_t<4>(in, B, n_lists, qstride, lstride, k, out, set_thr, st);
    case 8: return merge_t<8>(in, B, n_lists, qstride, lstride, k, out, set_thr, st);
    case 16: return merge_t<16>(in, B, n_lists, qstride, lstride, k, out, set_thr, st);
    case 32: return merge_t<32>(in, B, n_lists, qstride, lstride, k, out, set_thr, st);
  }
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------- S6 + S7
// w_r = softmax(s_r / T), max-subtracted: s_0 is the largest score of the
// sorted list.  exp in parallel, the normaliser by a fixed xor tree (order
// independent of batch position).  P[e] = sum_r w_r A_r[e], r ascending.
__global__ void __launch_bounds__(256) k_finalize(const uint64_t* __restrict__ top, int k,
                                                  const float* __restrict__ act, int64_t offset,
                                                  const float* __restrict__ rows, int mode,
                                                  int64_t LE, float T, int64_t* __restrict__ ids,
                                                  float* __restrict__ scores,
                                                  float* __restrict__ pred) {
  __shared__ float w[256];
  __shared__ const float* src[256];
  __shared__ float red[8];
  const int b = blockIdx.x;
  const int t = threadIdx.x;
  const uint64_t* tb = top + (int64_t)b * k;
  const float s0 = key_score(tb[0]);
  float e = 0.f;
  if (t < k) {
    const uint64_t key = tb[t];
    const float s = key_score(key);
    const int64_t gid = key_gid(key);
    ids[(int64_t)b * k + t] = gid;
    scores[(int64_t)b * k + t] = s;
    e = expf(__fdiv_rn(s - s0, T));
    src[t] = mode == 0 ? act + (gid - offset) * LE : rows + ((int64_t)b * k + t) * LE;
  }
  if (pred == nullptr) return;
  float z = e;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) z += __shfl_xor_sync(kFull, z, off);
  if ((t & 31) == 0) red[t >> 5] = z;
  __syncthreads();
  float Z = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) Z += red[i];
  if (t < k) w[t] = __fdiv_rn(e, Z);
  __syncthreads();
  float* pb = pred + (int64_t)b * LE;
  for (int64_t j = t; j < LE; j += blockDim.x) {
    float acc = 0.f;
    for (int r = 0; r < k; ++r) acc = __fmaf_rn(w[r], src[r][j], acc);
    pb[j] = acc;
  }
}

cudaError_t launch_finalize(const uint64_t* top, int B, int k, const float* act, int64_t offset,
                            const float* rows, int mode, int64_t LE, float temperature,
                            int64_t* ids, float* scores, float* pred, cudaStream_t st) {
  if (B <= 0) return cudaSuccess;
  if (k > 256) return cudaErrorInvalidValue;
  k_finalize<<<B, 256, 0, st>>>(top, k, act, offset, rows, mode, LE, temperature, ids, scores, pred);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- multi-GPU row gather
__global__ void k_gather_rows(const uint64_t* __restrict__ top, int k, const float* __restrict__ act,
                              int64_t offset, int64_t n_local, int64_t LE, float* __restrict__ rows) {
  const int64_t br = blockIdx.x;  // b * k + r
  const int64_t gid = key_gid(top[br]);
  const int64_t j = gid - offset;
  const bool own = j >= 0 && j < n_local;
  float* dst = rows + br * LE;
  const float* s = act + (own ? j : 0) * LE;
  for (int64_t e = threadIdx.x; e < LE; e += blockDim.x) dst[e] = own ? s[e] : 0.f;
}

cudaError_t launch_gather_rows(const uint64_t* top, int B, int k, const float* act, int64_t offset,
                               int64_t n_local, int64_t LE, float* rows, cudaStream_t st) {
  if (B <= 0) return cudaSuccess;
  k_gather_rows<<<(unsigned)((int64_t)B * k), 256, 0, st>>>(top, k, act, offset, n_local, LE, rows);
  return cudaGetLastError();
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
