// k_post.cu -- the small kernels around the scan (sm_100a):
//   S0/S1 row norms, S4/S5 key-list merge, S6+S7 softmax + gather + weighted
//   reduce, the multi-GPU winner-row gather, S8 expert plan, build validation.
#include "common.cuh"
#include "host_util.h"
#include "kernels.h"

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

__device__ __forceinline__ void finalize_query(const uint64_t* tb, int k, int b, const FinalizeArgs& f,
                                               int64_t j0, int64_t j1, bool write_ids);

// ---------------------------------------------------------------- S4 / S5 merge
// One CTA per query.  The answer is the k largest keys of the union of the lists
// (keys are unique: they carry the global id).  Exact selection:
//   1. every warp streams whole lists (4 loads in flight), and keys >= lb -- a known
//      lower bound of the final k-th key (the scan's shared threshold; 1 = "any real
//      key") -- are appended to shared memory with one atomic per warp;
//   2. n <= kRankMax survivors: each survivor's rank = #{survivors > it} (broadcast
//      reads of shared memory, O(n^2 / 256) compares per thread), rank < k -> out[rank];
//      kRankMax < n <= kSelCap: block bitonic sort; n > kSelCap: an MSB-first 8-bit
//      radix select finds the k-th largest key T exactly, and keys >= T are re-collected.
constexpr int kSelCap = 2048;
constexpr int kRankMax = 512;
constexpr int kItemCap = 4096;

__device__ __forceinline__ void block_sort_desc(uint64_t* a, int np2) {
  for (int size = 2; size <= np2; size <<= 1) {
    for (int j = size >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < (np2 >> 1); i += blockDim.x) {
        const int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1)), hi = lo + j;  // j is a power of 2
        const uint64_t x = a[lo], y = a[hi];
        const bool desc = (lo & size) == 0;
        if (desc ? x < y : x > y) { a[lo] = y; a[hi] = x; }
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------- fused peer exchange
// Thread 0 waits until flags[g] >= seq for every g (acquire, system scope: the data the
// peers stored before raising their flag is visible), then the CTA proceeds.  Bounded by
// kPeerWaitNs: a peer that never signals traps the kernel (an error, not a hung GPU).
constexpr unsigned long long kPeerWaitNs = 120000000000ull;  // 120 s: ranks may be seconds apart at their first query
__device__ __forceinline__ void peer_wait(const unsigned long long* flags, int G, unsigned long long seq) {
  if (threadIdx.x == 0) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int g = 0; g < G; ++g) {
      for (;;) {
        unsigned long long v;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + g) : "memory");
        if (v >= seq) break;
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (t1 - t0 > kPeerWaitNs) __trap();
        __nanosleep(64);
      }
    }
  }
  __syncthreads();
}
// Whole CTA, after its peer stores: the last CTA of the grid raises this rank's flag in
// every rank (release, system scope) and resets the counter for the next exchange.
__device__ __forceinline__ void peer_signal(const PeerXchg& px) {
  __threadfence_system();  // this CTA's peer stores before its arrival
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned done = atomicAdd(px.counter, 1u);
    if (done == gridDim.x - 1) {
      atomicExch(px.counter, 0u);
      __threadfence_system();  // every CTA's stores (seen through the counter) before the flags
      for (int g = 0; g < px.G; ++g)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(px.flag_dst[g]), "l"(px.seq) : "memory");
    }
  }
}

__global__ void __launch_bounds__(256) k_merge(const uint64_t* __restrict__ in, int n_lists,
                                               int64_t qstride, int64_t lstride, int list_len, int k,
                                               uint64_t* __restrict__ out,
                                               unsigned long long* __restrict__ set_thr,
                                               unsigned long long* __restrict__ lower,
                                               FinalizeArgs fin, unsigned* __restrict__ bump, int reset_lower,
                                               PeerXchg px) {
  __shared__ uint64_t cand[kSelCap];
  __shared__ uint64_t topk[256];
  __shared__ unsigned hist[256];
  __shared__ int cnt;
  __shared__ uint64_t prefix_s;
  __shared__ int need_s;
  __shared__ uint32_t items_s[kItemCap];  // (list << 3) | chunk
  __shared__ int n_items_s;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int b = blockIdx.x;
  pdl_wait();  // the scan's lists and thresholds
  // (key loads are ld.global.cg: L2-coherent, so keys a peer stored over NVLink during
  // this kernel's lifetime -- fused exchange 1 -- are never read through a stale L1 line)
  if (px.G > 0 && px.wait_flags) peer_wait(px.wait_flags, px.G, px.seq);  // fused exchange 1: every rank's keys
  // the scan is complete: a new seeding epoch for the next chunk (stale published keys of
  // this one can never be taken for the next one's)
  if (bump && b == 0 && t == 0) atomicAdd(bump, 1u);
  const uint64_t* base = in + (int64_t)b * qstride;
  const int nch = (list_len + 31) >> 5;
  const int items = n_lists * nch;
  uint64_t lb = lower ? lower[b] : 0ull;
  if (lower && reset_lower) {
    __syncthreads();                 // every thread has read it
    if (t == 0) lower[b] = 0ull;     // the next chunk's scan starts from no threshold
  }
  if (lb == 0) lb = 1;  // sentinel keys (0) never count
  auto item_key = [&](int it) -> uint64_t {
    if (it >= items) return 0ull;
    const int l = nch == 1 ? it : it / nch, c = it - l * nch;
    const int i = c * 32 + lane;
    return i < list_len ? __ldcg(base + (int64_t)l * lstride + i) : 0ull;
  };
  // flat key f = l * list_len + i: the whole block reads 8 keys per thread per round
  // (one L2 round trip per 2048 keys, instead of one per 32 lists of a warp)
  const int64_t n_keys = (int64_t)n_lists * list_len;
  auto flat_key = [&](int64_t f) -> uint64_t {
    if (f >= n_keys) return 0ull;
    const int64_t l = f / list_len, i = f - l * list_len;
    return __ldcg(base + l * lstride + i);
  };
  auto append = [&](uint64_t key, uint64_t thr_lo) {  // whole warp; keys >= thr_lo to cand
    const unsigned m = __ballot_sync(kFull, key >= thr_lo);
    if (m) {
      int pos0 = 0;
      if (lane == 0) pos0 = atomicAdd(&cnt, __popc(m));
      pos0 = __shfl_sync(kFull, pos0, 0);
      const int pos = pos0 + __popc(m & ((1u << lane) - 1u));
      if (key >= thr_lo && pos < kSelCap) cand[pos] = key;
    }
  };
  auto collect = [&](uint64_t thr_lo) {  // append keys >= thr_lo to cand (warp-aggregated)
    for (int64_t f0 = (int64_t)warp * 32 + lane; f0 - lane < n_keys; f0 += 8 * 256) {
      uint64_t kk[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) kk[u] = flat_key(f0 + 256 * u);
#pragma unroll
      for (int u = 0; u < 8; ++u) append(kk[u], thr_lo);
    }
  };
  // Lists are sorted descending: chunk c + 1 of a list (32 keys) can hold a key >= thr_lo
  // only if the last key of chunk c does.  With seeded thresholds most lists of a large
  // k end after their first chunk, so only the needed (list, chunk) items are read.
  auto collect_lists = [&](uint64_t thr_lo) {
    if (t == 0) n_items_s = 0;
    __syncthreads();
    for (int l = t; l < n_lists; l += blockDim.x) {
      const uint64_t* lp = base + (int64_t)l * lstride;
      int need = 1;
      while (need < nch && __ldcg(lp + 32 * need - 1) >= thr_lo) ++need;
      const int pos = atomicAdd(&n_items_s, need);
      for (int c = 0; c < need; ++c) items_s[pos + c] = ((uint32_t)l << 3) | (uint32_t)c;
    }
    __syncthreads();
    const int ni = n_items_s;
    for (int i0 = warp; i0 < ni; i0 += 8 * 4) {
      uint64_t kk[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int it = i0 + 8 * u;
        kk[u] = 0ull;
        if (it < ni) {
          const uint32_t w = items_s[it];
          const int i = (int)(w & 7u) * 32 + lane;
          if (i < list_len) kk[u] = __ldcg(base + (int64_t)(w >> 3) * lstride + i);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) append(kk[u], thr_lo);
    }
  };
  // Lists are sorted: the k-th largest list head is a real key <= the final k-th key,
  // a much tighter bound than lb when the state lists are many (S4: 2 per CTA).
  if (n_lists >= k && n_lists <= kSelCap) {
    if (t == 0) prefix_s = 0ull;
    for (int l = t; l < n_lists; l += blockDim.x) cand[l] = __ldcg(base + (int64_t)l * lstride);
    __syncthreads();
    for (int i = t; i < n_lists; i += blockDim.x) {
      const uint64_t x = cand[i];
      if (x == 0) continue;  // empty list; real keys are distinct
      int r = 0;
      for (int j = 0; j < n_lists; ++j) r += cand[j] > x;
      if (r == k - 1) prefix_s = x;
    }
    __syncthreads();
    if (prefix_s > lb) lb = prefix_s;
    __syncthreads();
  }
  if (t == 0) cnt = 0;
  __syncthreads();
  if (nch >= 2 && nch <= 8 && (int64_t)n_lists * nch <= kItemCap) collect_lists(lb);
  else collect(lb);
  __syncthreads();
  int n = cnt;
  if (n > kSelCap) {
    // radix select of the k-th largest key among keys >= lb
    uint64_t prefix = 0, pmask = 0;
    int need = k;
    for (int shift = 56; shift >= 0; shift -= 8) {
      hist[t] = 0;
      __syncthreads();
      for (int it0 = warp; it0 < items; it0 += 8) {
        const uint64_t key = item_key(it0);
        if (key >= lb && (key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
      }
      __syncthreads();
      if (warp == 0) {  // suffix sums over the 256 bins: lane l owns bins 255-8l .. 248-8l
        int h[8], tot = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) { h[u] = hist[255 - 8 * lane - u]; tot += h[u]; }
        int incl = tot;  // inclusive prefix over lanes (higher bins first)
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int o = __shfl_up_sync(kFull, incl, off);
          if (lane >= off) incl += o;
        }
        int c = incl - tot;  // keys in higher bins than this lane's
        const bool mine = c < need && incl >= need;
        if (mine) {
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (c + h[u] >= need) {
              prefix_s = prefix | ((uint64_t)(255 - 8 * lane - u) << shift);
              need_s = need - c;
              break;
            }
            c += h[u];
          }
        }
      }
      __syncthreads();
      prefix = prefix_s;
      need = need_s;
      pmask |= (uint64_t)255 << shift;
      __syncthreads();
    }
    if (t == 0) cnt = 0;
    __syncthreads();
    collect(prefix);  // exactly k keys: keys are unique and prefix is the k-th largest
    __syncthreads();
    n = cnt;
  }
  const int nout = n < k ? n : k;
  if (n <= kRankMax) {
    for (int i = t; i < n; i += blockDim.x) {
      const uint64_t x = cand[i];
      int r = 0;
      for (int j = 0; j < n; ++j) r += cand[j] > x;
      if (r < k) topk[r] = x;
    }
  } else {
    int np2 = 1;
    while (np2 < n) np2 <<= 1;
    for (int i = n + t; i < np2; i += blockDim.x) cand[i] = 0ull;
    __syncthreads();
    block_sort_desc(cand, np2);
    for (int i = t; i < nout; i += blockDim.x) topk[i] = cand[i];
  }
  __syncthreads();
  for (int i = t; i < k; i += blockDim.x) {
    const uint64_t v = i < nout ? topk[i] : 0ull;
    out[(int64_t)b * k + i] = v;
    if (px.G > 0 && px.key_dst[0])  // fused exchange 1: straight into every rank's gathered slot
      for (int g = 0; g < px.G; ++g) px.key_dst[g][(int64_t)b * k + i] = v;
  }
  if (set_thr && t == 0) {
    // seeding: the k-th best key of a subset of rows, minus one (strict lower bound,
    // the subset's own rows stay admissible in the full scan)
    const uint64_t kth = k <= nout ? topk[k - 1] : 0ull;
    set_thr[b] = kth ? kth - 1 : 0ull;
  }
  if (fin.act != nullptr) {  // fused S6 + S7 (one GPU) or S6 + partial S7 (multi-GPU)
    if (nout < k)
      for (int i = nout + t; i < k; i += blockDim.x) topk[i] = 0ull;
    __syncthreads();
    finalize_query(topk, k, b, fin, 0, fin.LE, true);
  }
  if (px.G > 0 && px.flag_dst[0]) peer_signal(px);
}

cudaError_t launch_merge(const uint64_t* in, int B, int n_lists, int64_t qstride, int64_t lstride,
                         int k, uint64_t* out, cudaStream_t st, unsigned long long* set_thr,
                         unsigned long long* lower, const FinalizeArgs* fin, int list_len,
                         unsigned* bump, bool reset_lower, const PeerXchg* px) {
  if (B <= 0) return cudaSuccess;
  if (k > 256) return cudaErrorInvalidValue;
  if (list_len <= 0) list_len = k;
  FinalizeArgs f{};
  if (fin) f = *fin;
  PeerXchg x{};
  if (px) x = *px;
  cudaError_t e = set_smem_attrs_once((const void*)k_merge, 0);
  if (e != cudaSuccess) return e;
  return launch_pdl(k_merge, dim3(B), dim3(256), 0, st, in, n_lists, qstride, lstride, list_len, k, out, set_thr,
                    lower, f, bump, reset_lower ? 1 : 0, x);
}

// ---------------------------------------------------------------- S6 + S7
// w_r = softmax(s_r / T), max-subtracted: s_0 is the largest score of the
// sorted list.  exp in parallel, the normaliser by a fixed xor tree (order
// independent of batch position).  P[e] = sum_r w_r A_r[e], r ascending over the rows
// that contribute (all k on one GPU; the owned ones for a multi-GPU partial, mode 2).
// Whole CTA (256 threads); outputs j = j0 + t, j0 + t + 256, ... < j1.
__device__ __forceinline__ void finalize_query(const uint64_t* tb, int k, int b, const FinalizeArgs& f,
                                               int64_t j0, int64_t j1, bool write_ids) {
  __shared__ float w[256];
  __shared__ const float* src[256];
  __shared__ float red[8];
  __shared__ int wcnt[8];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const float s0 = key_score(tb[0]);
  float e = 0.f;
  const float* my_src = nullptr;
  if (t < k) {
    const uint64_t key = tb[t];
    if (key != 0) {
      const float s = key_score(key);
      const int64_t gid = key_gid(key);
      if (write_ids) {
        f.ids[(int64_t)b * k + t] = gid;
        f.scores[(int64_t)b * k + t] = s;
      }
      e = expf(__fdiv_rn(s - s0, f.T));
      const int64_t j = gid - f.offset;
      if (j >= 0 && j < f.n_local) my_src = f.act + j * f.LE;  // a row this rank holds
    } else if (write_ids) {  // fewer than k candidates (cannot happen for k <= N_total): empty slot
      f.ids[(int64_t)b * k + t] = -1;
      f.scores[(int64_t)b * k + t] = -__int_as_float(0x7f800000);
    }
  }
  if (f.pred == nullptr) return;
  // destinations of the rows: pred, or (fused exchange 2) this rank's slot in every rank
  const int no = f.n_pred_peer > 0 ? f.n_pred_peer : 1;
  float* const* outs = f.n_pred_peer > 0 ? f.pred_peer : &f.pred;
  float z = e;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) z += __shfl_xor_sync(kFull, z, off);
  // compaction of the contributing rows, r ascending (warp ballots + an 8-entry scan)
  const unsigned keep = __ballot_sync(kFull, my_src != nullptr);
  if (lane == 0) { red[warp] = z; wcnt[warp] = __popc(keep); }
  __syncthreads();
  float Z = 0.f;
  int before = 0, nr = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    Z += red[i];
    before += i < warp ? wcnt[i] : 0;
    nr += wcnt[i];
  }
  if (my_src != nullptr) {
    const int pos = before + __popc(keep & ((1u << lane) - 1u));
    w[pos] = __fdiv_rn(e, Z);
    src[pos] = my_src;
  }
  __syncthreads();
  if ((f.LE & 3) == 0 && (j0 & 3) == 0 && ((j1 & 3) == 0 || j1 == f.LE)) {
    // float4 columns, two per thread per step, 8 rows at a time (16 x 16-byte loads in
    // flight): per element the same r-ascending FMA chain as the scalar path below
    const int64_t c0 = j0 >> 2, c1 = (j1 + 3) >> 2;
    for (int64_t ca = c0 + t; ca < c1; ca += 2 * (int64_t)blockDim.x) {
      const int64_t cb = ca + blockDim.x;
      const bool vb = cb < c1;
      float4 acc_a = make_float4(0.f, 0.f, 0.f, 0.f), acc_b = acc_a;
      for (int r0 = 0; r0 < nr; r0 += 8) {
        float4 xa[8], xb[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const bool vr = r0 + u < nr;
          const float4 zz = make_float4(0.f, 0.f, 0.f, 0.f);
          xa[u] = vr ? __ldg(reinterpret_cast<const float4*>(src[r0 + u]) + ca) : zz;
          xb[u] = (vr && vb) ? __ldg(reinterpret_cast<const float4*>(src[r0 + u]) + cb) : zz;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (r0 + u < nr) {  // r ascending
            const float wr = w[r0 + u];
            acc_a.x = __fmaf_rn(wr, xa[u].x, acc_a.x); acc_a.y = __fmaf_rn(wr, xa[u].y, acc_a.y);
            acc_a.z = __fmaf_rn(wr, xa[u].z, acc_a.z); acc_a.w = __fmaf_rn(wr, xa[u].w, acc_a.w);
            acc_b.x = __fmaf_rn(wr, xb[u].x, acc_b.x); acc_b.y = __fmaf_rn(wr, xb[u].y, acc_b.y);
            acc_b.z = __fmaf_rn(wr, xb[u].z, acc_b.z); acc_b.w = __fmaf_rn(wr, xb[u].w, acc_b.w);
          }
        }
      }
      for (int o = 0; o < no; ++o) {
        reinterpret_cast<float4*>(outs[o] + (int64_t)b * f.LE)[ca] = acc_a;
        if (vb) reinterpret_cast<float4*>(outs[o] + (int64_t)b * f.LE)[cb] = acc_b;
      }
    }
    return;
  }
  // two outputs per thread per step, 8 rows at a time: 16 independent loads in flight
  for (int64_t ja = j0 + t; ja < j1; ja += 2 * (int64_t)blockDim.x) {
    const int64_t jb = ja + blockDim.x;
    const bool vb = jb < j1;
    float acc_a = 0.f, acc_b = 0.f;
    for (int r0 = 0; r0 < nr; r0 += 8) {
      float xa[8], xb[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool vr = r0 + u < nr;
        xa[u] = vr ? __ldg(src[r0 + u] + ja) : 0.f;
        xb[u] = (vr && vb) ? __ldg(src[r0 + u] + jb) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (r0 + u < nr) {  // r ascending
          acc_a = __fmaf_rn(w[r0 + u], xa[u], acc_a);
          acc_b = __fmaf_rn(w[r0 + u], xb[u], acc_b);
        }
      }
    }
    for (int o = 0; o < no; ++o) {
      outs[o][(int64_t)b * f.LE + ja] = acc_a;
      if (vb) outs[o][(int64_t)b * f.LE + jb] = acc_b;
    }
  }
}

// Grid (B, ceil(LE / 256)): every CTA recomputes its query's k weights (k <= 256
// exps, cheap) and produces 256 outputs; chunk 0 also writes ids and scores.
__global__ void __launch_bounds__(256) k_finalize(const uint64_t* __restrict__ top, int k, FinalizeArgs f) {
  const int b = blockIdx.x;
  const int64_t j0 = (int64_t)blockIdx.y * blockDim.x;
  pdl_wait();
  finalize_query(top + (int64_t)b * k, k, b, f, j0, j0 + blockDim.x < f.LE ? j0 + blockDim.x : f.LE,
                 blockIdx.y == 0);
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
                       const unsigned long long* __restrict__ wait_flags, unsigned long long seq) {
  pdl_wait();
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
                        const unsigned long long* wait_flags, unsigned long long seq) {
  if (n <= 0) return cudaSuccess;
  const int64_t units = (n + 3) / 4;
  const unsigned grid = (unsigned)std::min<int64_t>((units + 255) / 256, 148 * 8);
  cudaError_t e = set_smem_attrs_once((const void*)k_psum, 0);
  if (e != cudaSuccess) return e;
  return launch_pdl(k_psum, dim3(grid), dim3(256), 0, st, parts, G, part_stride, n, out, wait_flags, seq);
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
