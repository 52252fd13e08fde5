// k_tree.cu -- NEXT-N2: the clustering-tree SPS of PAPER.md §IV-B.
//
// Build: "any node (cluster) with more than beta prompts is recursively
// partitioned ... customized k-medoids clustering algorithm using prompt-level semantic
// similarity as distance metric, where roulette wheel sampling-based centroid
// initialization and subcluster-level centroid updating are conducted."  Readings
// R24-R28 (oracle/tree.py states the same algorithm in numpy).  The host
// walks the tree level by level; every splitting node of a level is processed by the
// same kernels at once (one segment per node over the flat member permutation).  All
// build arithmetic is fp64 with fixed reduction orders, so every integer decision
// (draw, assignment, centroid) is reproducible and matches an fp64 reference except at
// exact ties:
//   roulette init   k_cos_update (best cosine to the chosen medoids, distance mass d)
//                   + k_pick (one warp per node: u * sum(d) on the running prefix)
//   assignment      k_assign (warp per member, cosines to <= 16 medoids in registers)
//   stable split    k_chunk_count / k_chunk_scan / k_scatter (counting sort by label)
//   centroid update k_cluster_partial / k_cluster_sum (S_j = sum x^ over the subcluster,
//                   chunked, fixed order) + k_obj (x^_i . S_j, the summed cosine) +
//                   k_obj_pick (tie window: keep the current medoid, else the
//                   earliest maximiser) + k_commit_medoid
// Search (Algorithm 1): k_tree_search, one CTA per query: descend by the best child
// centroid (Eq. 11, fp32, the BF path's formula and key order), gather the leaf (and
// sibling subtrees depth-first while < alpha), exact top-alpha by key; S6+S7 reuse
// k_finalize.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "host_util.h"
#include "tree.h"

namespace remoe {
namespace {

constexpr int C = kTreeCMax;

// ------------------------------------------------------------------ device helpers
__device__ __forceinline__ double bfd(uint16_t h) { return (double)__uint_as_float((uint32_t)h << 16); }
__device__ __forceinline__ double lo64(uint32_t w) { return (double)bf_lo(w); }
__device__ __forceinline__ double hi64(uint32_t w) { return (double)bf_hi(w); }

__device__ __forceinline__ double warp_sum64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__device__ __forceinline__ uint64_t ord64(double v) {
  const uint64_t u = (uint64_t)__double_as_longlong(v);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ULL);
}

// largest s with off[s] <= a (off ascending, off[0] = 0)
__device__ __forceinline__ int seg_of(const int64_t* __restrict__ off, int S, int64_t a) {
  int lo = 0, hi = S - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (off[mid] <= a) lo = mid; else hi = mid - 1;
  }
  return lo;
}

struct Level {
  // segments (splitting nodes of the level)
  int S;
  const int64_t* seg_begin;  // [S] position of the node's range in perm
  const int64_t* seg_off;    // [S+1] flat offsets of the active members
  const int32_t* seg_c;      // [S] target medoid count min(branching, n)
  int32_t* med_cnt;          // [S]
  int64_t* med_row;          // [S][C] local rows
  int64_t* med_pos;          // [S][C] relative positions (roulette only)
  const double* u;           // [S] this draw's uniforms
  int32_t* cnt;              // [S][C] members per slot (after k_chunk_scan)
  // members
  int64_t A;
  int64_t* perm;
  const uint16_t* x;
  const double* rn;          // [n] 1 / |x_row| (0 for a zero row)
  int dim;
  double* best;              // [A]
  double* d;                 // [A]
  uint8_t* lab;              // [A]
  int64_t* sorted_row;       // [A]
  double* obj;               // [A]
  int32_t* cl_of;            // [A]
  // 1024-member chunks
  const int32_t* ch_seg;     // [nch]
  const int64_t* ch_a0;
  const int64_t* ch_a1;
  const int32_t* seg_ch0;    // [S]
  const int32_t* seg_ch1;
  int32_t* ccnt;             // [nch][C]
  int32_t* cpre;             // [nch][C]
};

__global__ void k_rnorm64(const uint16_t* __restrict__ x, int64_t n, int dim, double* __restrict__ rn) {
  const int lane = threadIdx.x & 31;
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= n) return;
  const uint16_t* xr = x + row * dim;
  double acc = 0.0;
  for (int c = lane; c < dim / 8; c += 32) {
    const uint4 v = *reinterpret_cast<const uint4*>(xr + c * 8);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double a = lo64(w[i]), b = hi64(w[i]);
      acc = fma(a, a, acc);
      acc = fma(b, b, acc);
    }
  }
  acc = warp_sum64(acc);
  if (lane == 0) rn[row] = acc > 0.0 ? 1.0 / sqrt(acc) : 0.0;
}

__global__ void k_fill(double* p, int64_t n, double v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

__global__ void k_iota(int64_t* p, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = i;
}

// cosines of `row` against medoid rows m[0..nm) (fp64, warp-wide; every lane gets all)
template <int NM>
__device__ __forceinline__ void warp_cos(const Level& L, int64_t row, const int64_t* m, int nm, double (&out)[NM]) {
  const int lane = threadIdx.x & 31;
  double acc[NM];
#pragma unroll
  for (int j = 0; j < NM; ++j) acc[j] = 0.0;
  const uint16_t* xr = L.x + row * L.dim;
  for (int c = lane; c < L.dim / 8; c += 32) {
    const uint4 v = *reinterpret_cast<const uint4*>(xr + c * 8);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < NM; ++j) {
      if (j < nm) {
        const uint4 mv = *reinterpret_cast<const uint4*>(L.x + m[j] * L.dim + c * 8);
        const uint32_t mw[4] = {mv.x, mv.y, mv.z, mv.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          acc[j] = fma(lo64(w[i]), lo64(mw[i]), acc[j]);
          acc[j] = fma(hi64(w[i]), hi64(mw[i]), acc[j]);
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < NM; ++j)
    if (j < nm) out[j] = warp_sum64(acc[j]) * L.rn[row] * L.rn[m[j]];
}

// R24: after medoid jm was drawn, best = max(best, cos(x, m_jm)); d = max(0, 1 - best),
// 0 for the chosen medoids.
__global__ void k_cos_update(Level L, int jm) {
  const int64_t a = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (a >= L.A) return;
  const int s = seg_of(L.seg_off, L.S, a);
  const int mc = L.med_cnt[s];
  if (mc <= jm) return;  // this node's init stopped early (no distance mass left)
  const int64_t rel = a - L.seg_off[s];
  const int64_t row = L.perm[L.seg_begin[s] + rel];
  double c1[1];
  warp_cos<1>(L, row, L.med_row + (int64_t)s * C + jm, 1, c1);
  if ((threadIdx.x & 31) == 0) {
    const double b = fmax(L.best[a], c1[0]);
    L.best[a] = b;
    bool chosen = false;
    for (int j = 0; j < mc; ++j) chosen |= L.med_pos[(int64_t)s * C + j] == rel;
    L.d[a] = chosen ? 0.0 : fmax(0.0, 1.0 - b);
  }
}

// R24: draw medoid j of every node (one warp per node).  j = 0: position floor(u n).
// j > 0: the first position whose running sum of d exceeds u * sum(d) (sum in a fixed
// order); sum(d) == 0 stops the node's init.
__global__ void k_pick(Level L, int j) {
  const int s = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (s >= L.S) return;
  if (j >= L.seg_c[s] || L.med_cnt[s] != j) return;
  const int64_t a0 = L.seg_off[s], n = L.seg_off[s + 1] - a0;
  int64_t p = -1;
  if (j == 0) {
    p = (int64_t)floor(L.u[s] * (double)n);
    if (p > n - 1) p = n - 1;
  } else {
    double part = 0.0;
    for (int64_t i = lane; i < n; i += 32) part += L.d[a0 + i];
    const double total = warp_sum64(part);
    if (!(total > 0.0)) return;
    const double t = L.u[s] * total;
    double run = 0.0;
    int64_t last_pos = -1;
    for (int64_t base = 0; base < n && p < 0; base += 32) {
      const int64_t i = base + lane;
      const double v = i < n ? L.d[a0 + i] : 0.0;
      double incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      incl += run;
      const unsigned hit = __ballot_sync(kFull, i < n && incl > t);
      const unsigned pos = __ballot_sync(kFull, i < n && v > 0.0);
      if (hit) p = base + __ffs(hit) - 1;
      if (pos) last_pos = base + 31 - __clz(pos);
      run = __shfl_sync(kFull, incl, 31);
    }
    if (p < 0) p = last_pos;  // rounding left t just above the running total
    if (p < 0) return;
  }
  if (lane == 0) {
    L.med_pos[(int64_t)s * C + j] = p;
    L.med_row[(int64_t)s * C + j] = L.perm[L.seg_begin[s] + p];
    L.med_cnt[s] = j + 1;
  }
}

// R25: label = most similar medoid (first max -> lower slot)
__global__ void k_assign(Level L) {
  const int64_t a = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (a >= L.A) return;
  const int s = seg_of(L.seg_off, L.S, a);
  const int mc = L.med_cnt[s];
  const int64_t row = L.perm[L.seg_begin[s] + (a - L.seg_off[s])];
  double cs[C];
  warp_cos<C>(L, row, L.med_row + (int64_t)s * C, mc, cs);
  if ((threadIdx.x & 31) == 0) {
    int best = 0;
    double bv = cs[0];
#pragma unroll
    for (int j = 1; j < C; ++j)
      if (j < mc && cs[j] > bv) { bv = cs[j]; best = j; }
    L.lab[a] = (uint8_t)best;
  }
}

__global__ void __launch_bounds__(1024) k_chunk_count(Level L) {
  __shared__ int cnt[C];
  const int c = blockIdx.x;
  if (threadIdx.x < C) cnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t a = L.ch_a0[c] + threadIdx.x;
  if (a < L.ch_a1[c]) atomicAdd(&cnt[L.lab[a]], 1);
  __syncthreads();
  if (threadIdx.x < C) L.ccnt[(int64_t)c * C + threadIdx.x] = cnt[threadIdx.x];
}

// exclusive prefix of the chunk counts per (segment, slot); totals -> cnt
__global__ void k_chunk_scan(Level L) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)L.S * C) return;
  const int s = (int)(i / C), l = (int)(i % C);
  int run = 0;
  for (int c = L.seg_ch0[s]; c < L.seg_ch1[s]; ++c) {
    L.cpre[(int64_t)c * C + l] = run;
    run += L.ccnt[(int64_t)c * C + l];
  }
  L.cnt[(int64_t)s * C + l] = run;
}

// stable counting sort by label: sorted_row[seg_off + slot_off(l) + rank] = member row
__global__ void __launch_bounds__(1024) k_scatter(Level L) {
  __shared__ int wcnt[32][C];
  const int c = blockIdx.x;
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
  for (int i = t; i < 32 * C; i += blockDim.x) wcnt[i / C][i % C] = 0;
  __syncthreads();
  const int64_t a = L.ch_a0[c] + t;
  const bool valid = a < L.ch_a1[c];
  const int l = valid ? L.lab[a] : 255;
  const unsigned peers = __match_any_sync(kFull, l);
  const int rw = __popc(peers & ((1u << lane) - 1u));
  if (valid && lane == __ffs(peers) - 1) wcnt[w][l] = __popc(peers);
  __syncthreads();
  if (!valid) return;
  int r = rw;
  for (int v = 0; v < w; ++v) r += wcnt[v][l];
  const int s = L.ch_seg[c];
  int slot_off = 0;
  for (int v = 0; v < l; ++v) slot_off += L.cnt[(int64_t)s * C + v];
  const int64_t dst = L.seg_off[s] + slot_off + L.cpre[(int64_t)c * C + l] + r;
  L.sorted_row[dst] = L.perm[L.seg_begin[s] + (a - L.seg_off[s])];
}

// S_j partial sums of x^ over <= 256 consecutive sorted members, in order
__global__ void __launch_bounds__(256) k_cluster_partial(const uint16_t* __restrict__ x, const double* __restrict__ rn,
                                                         int dim, const int64_t* __restrict__ sorted_row,
                                                         const int64_t* __restrict__ cc_a0,
                                                         const int64_t* __restrict__ cc_a1, double* __restrict__ part) {
  const int64_t cc = blockIdx.x;
  const int64_t a0 = cc_a0[cc], a1 = cc_a1[cc];
  for (int d = threadIdx.x; d < dim; d += blockDim.x) {
    double acc = 0.0;
    int64_t i = a0;
    for (; i + 4 <= a1; i += 4) {
      int64_t r[4];
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) r[u] = sorted_row[i + u];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = bfd(x[r[u] * dim + d]) * rn[r[u]];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc += v[u];
    }
    for (; i < a1; ++i) {
      const int64_t r = sorted_row[i];
      acc += bfd(x[r * dim + d]) * rn[r];
    }
    part[cc * dim + d] = acc;
  }
}

__global__ void __launch_bounds__(256) k_cluster_sum(int dim, const int32_t* __restrict__ cl_c0,
                                                     const int32_t* __restrict__ cl_c1,
                                                     const double* __restrict__ part, double* __restrict__ ssum) {
  const int64_t cl = blockIdx.x;
  for (int d = threadIdx.x; d < dim; d += blockDim.x) {
    double acc = 0.0;
    for (int cc = cl_c0[cl]; cc < cl_c1[cl]; ++cc) acc += part[(int64_t)cc * dim + d];
    ssum[cl * dim + d] = acc;
  }
}

// summed cosine of every member to its subcluster: x^_i . S_j (R25)
__global__ void k_obj(Level L, const int32_t* __restrict__ cl_index, const double* __restrict__ ssum,
                      unsigned long long* __restrict__ best_bits) {
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= L.A) return;
  const int s = seg_of(L.seg_off, L.S, i);
  int64_t rel = i - L.seg_off[s];
  int l = 0;
  while (rel >= L.cnt[(int64_t)s * C + l]) rel -= L.cnt[(int64_t)s * C + l++];
  const int cl = cl_index[(int64_t)s * C + l];
  const int64_t row = L.sorted_row[i];
  const uint16_t* xr = L.x + row * L.dim;
  const double* sv = ssum + (int64_t)cl * L.dim;
  double acc = 0.0;
  for (int c = lane; c < L.dim / 8; c += 32) {
    const uint4 v = *reinterpret_cast<const uint4*>(xr + c * 8);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      acc = fma(lo64(w[e]), sv[c * 8 + 2 * e], acc);
      acc = fma(hi64(w[e]), sv[c * 8 + 2 * e + 1], acc);
    }
  }
  acc = warp_sum64(acc) * L.rn[row];
  if (lane == 0) {
    L.obj[i] = acc;
    L.cl_of[i] = cl;
    atomicMax(best_bits + cl, (unsigned long long)ord64(acc));
  }
}

__device__ __forceinline__ double unord64(uint64_t u) {
  return __longlong_as_double((long long)((u >> 63) ? (u & 0x7FFFFFFFFFFFFFFFULL) : ~u));
}

// maximisers within kTieTol * |cluster| of the maximum (R25): the earliest one, and
// whether the current medoid is one
constexpr double kTieTol = 1e-10;
__global__ void k_obj_pick(Level L, const unsigned long long* __restrict__ best_bits,
                           unsigned long long* __restrict__ best_i, const int32_t* __restrict__ cl_seg,
                           const int32_t* __restrict__ cl_slot, int* __restrict__ keep) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L.A) return;
  const int cl = L.cl_of[i];
  const int s = cl_seg[cl], l = cl_slot[cl];
  const double n = (double)max(1, L.cnt[(int64_t)s * C + l]);
  if (L.obj[i] >= unord64(best_bits[cl]) - kTieTol * n) {
    atomicMin(best_i + cl, (unsigned long long)i);
    if (L.sorted_row[i] == L.med_row[(int64_t)s * C + l]) keep[cl] = 1;
  }
}

__global__ void k_commit_medoid(Level L, int ncl, const int32_t* __restrict__ cl_seg,
                                const int32_t* __restrict__ cl_slot, const unsigned long long* __restrict__ best_i,
                                const int* __restrict__ keep, int* __restrict__ changed) {
  const int cl = blockIdx.x * blockDim.x + threadIdx.x;
  if (cl >= ncl || keep[cl]) return;
  const int64_t nr = L.sorted_row[best_i[cl]];
  int64_t* m = L.med_row + (int64_t)cl_seg[cl] * C + cl_slot[cl];
  if (*m != nr) {
    *m = nr;
    *changed = 1;
  }
}

__global__ void k_commit_perm(Level L, const uint8_t* __restrict__ commit) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= L.A) return;
  const int s = seg_of(L.seg_off, L.S, a);
  if (commit[s]) L.perm[L.seg_begin[s] + (a - L.seg_off[s])] = L.sorted_row[a];
}

// ------------------------------------------------------------------ host side
uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
// u(seed, node, j) in [0, 1), 53 bits (R24); the oracle implements the same generator.
double uniform01(uint64_t seed, uint64_t node, uint64_t j) {
  const uint64_t h = splitmix64(seed ^ (node * 0x9E3779B97F4A7C15ULL + j));
  return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

struct DevArena {
  std::vector<void*> ptrs;
  cudaError_t err = cudaSuccess;
  template <typename T>
  T* get(size_t n) {
    void* p = nullptr;
    if (err == cudaSuccess) err = cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T));
    if (err == cudaSuccess) ptrs.push_back(p);
    return (T*)p;
  }
  ~DevArena() {
    for (void* p : ptrs) cudaFree(p);
  }
};

inline unsigned blocks_for(int64_t threads, int bs) { return (unsigned)((threads + bs - 1) / bs); }

template <typename T>
cudaError_t up(T* d, const std::vector<T>& h, cudaStream_t st) {
  if (h.empty()) return cudaSuccess;
  return cudaMemcpyAsync(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, st);
}
template <typename T>
cudaError_t down(std::vector<T>& h, const T* d, size_t n, cudaStream_t st) {
  h.resize(n);
  if (n == 0) return cudaSuccess;
  cudaError_t e = cudaMemcpyAsync(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(st);
}

}  // namespace

void tree_free(Tree* t) {
  for (void* p : {(void*)t->perm, (void*)t->begin, (void*)t->end, (void*)t->child0, (void*)t->nchild,
                  (void*)t->medoid})
    if (p) cudaFree(p);
  *t = Tree{};
}

#define TB_TRY(expr)                                                                           \
  do {                                                                                         \
    cudaError_t e_ = (expr);                                                                   \
    if (e_ != cudaSuccess) {                                                                   \
      *err = std::string(#expr) + ": " + cudaGetErrorString(e_);                               \
      return e_ == cudaErrorMemoryAllocation ? REMOE_ERR_OOM : REMOE_ERR_CUDA;                 \
    }                                                                                          \
  } while (0)

remoe_status_t tree_build(const uint16_t* x, int64_t n, int dim, int beta, int branching, int max_iter,
                          uint64_t seed, cudaStream_t st, Tree* out, std::string* err) {
  const auto t0 = std::chrono::steady_clock::now();
  Tree T;
  T.beta = beta;
  T.branching = branching;
  TB_TRY(cudaMalloc(&T.perm, std::max<int64_t>(n, 1) * 8));
  struct Guard {
    Tree* t;
    bool keep = false;
    ~Guard() { if (!keep) tree_free(t); }
  } guard{&T};
  const int bs = 256;
  k_iota<<<blocks_for(n, bs), bs, 0, st>>>(T.perm, n);
  TB_TRY(cudaGetLastError());

  DevArena ar;
  const int64_t Smax = n / (beta + 1) + 1;
  const int64_t chmax = n / 1024 + Smax + 1;
  double* rn = ar.get<double>(n);
  double* best = ar.get<double>(n);
  double* dd = ar.get<double>(n);
  uint8_t* lab = ar.get<uint8_t>(n);
  int64_t* sorted_row = ar.get<int64_t>(n);
  double* obj = ar.get<double>(n);
  int32_t* cl_of = ar.get<int32_t>(n);
  int64_t* d_seg_begin = ar.get<int64_t>(Smax);
  int64_t* d_seg_off = ar.get<int64_t>(Smax + 1);
  int32_t* d_seg_c = ar.get<int32_t>(Smax);
  int32_t* d_med_cnt = ar.get<int32_t>(Smax);
  int64_t* d_med_row = ar.get<int64_t>(Smax * C);
  int64_t* d_med_pos = ar.get<int64_t>(Smax * C);
  double* d_u = ar.get<double>(Smax);
  int32_t* d_cnt = ar.get<int32_t>(Smax * C);
  int32_t* d_ch_seg = ar.get<int32_t>(chmax);
  int64_t* d_ch_a0 = ar.get<int64_t>(chmax);
  int64_t* d_ch_a1 = ar.get<int64_t>(chmax);
  int32_t* d_seg_ch0 = ar.get<int32_t>(Smax);
  int32_t* d_seg_ch1 = ar.get<int32_t>(Smax);
  int32_t* d_ccnt = ar.get<int32_t>(chmax * C);
  int32_t* d_cpre = ar.get<int32_t>(chmax * C);
  int32_t* d_cl_index = ar.get<int32_t>(Smax * C);
  uint8_t* d_commit = ar.get<uint8_t>(Smax);
  int* d_changed = ar.get<int>(1);
  TB_TRY(ar.err);
  // cluster-sized buffers grow on demand
  struct Grow {
    void* p = nullptr;
    size_t cap = 0;
    ~Grow() { if (p) cudaFree(p); }
    cudaError_t need(size_t bytes) {
      if (bytes <= cap) return cudaSuccess;
      if (p) cudaFree(p);
      p = nullptr;
      cap = 0;
      cudaError_t e = cudaMalloc(&p, bytes);
      if (e == cudaSuccess) cap = bytes;
      return e;
    }
  } g_part, g_ssum, g_cc_a0, g_cc_a1, g_cl_c0, g_cl_c1, g_cl_seg, g_cl_slot, g_best_bits, g_best_i, g_keep;

  k_rnorm64<<<blocks_for(n * 32, bs), bs, 0, st>>>(x, n, dim, rn);
  TB_TRY(cudaGetLastError());

  std::vector<int64_t> hb{0}, he{n}, hm{-1};
  std::vector<int32_t> hp{-1}, hc0{-1}, hnc{0};
  int64_t lvl_lo = 0, lvl_hi = 1;
  int depth = 0;
  while (true) {
    std::vector<int> segs;
    for (int64_t i = lvl_lo; i < lvl_hi; ++i)
      if (he[i] - hb[i] > beta) segs.push_back((int)i);
    if (segs.empty()) break;
    if (depth + 1 >= kTreeMaxDepth) {
      *err = "tree deeper than " + std::to_string(kTreeMaxDepth) + " levels";
      return REMOE_ERR_UNSUPPORTED;
    }
    const int S = (int)segs.size();
    std::vector<int64_t> seg_begin(S), seg_off(S + 1, 0);
    std::vector<int32_t> seg_c(S), seg_ch0(S), seg_ch1(S), ch_seg;
    std::vector<int64_t> ch_a0, ch_a1;
    int cmax = 0;
    for (int s = 0; s < S; ++s) {
      const int64_t nb = he[segs[s]] - hb[segs[s]];
      seg_begin[s] = hb[segs[s]];
      seg_off[s + 1] = seg_off[s] + nb;
      seg_c[s] = (int32_t)std::min<int64_t>(branching, nb);
      cmax = std::max(cmax, seg_c[s]);
      seg_ch0[s] = (int32_t)ch_seg.size();
      for (int64_t a = seg_off[s]; a < seg_off[s + 1]; a += 1024) {
        ch_seg.push_back(s);
        ch_a0.push_back(a);
        ch_a1.push_back(std::min(a + 1024, seg_off[s + 1]));
      }
      seg_ch1[s] = (int32_t)ch_seg.size();
    }
    const int64_t A = seg_off[S];
    const int nch = (int)ch_seg.size();
    TB_TRY(up(d_seg_begin, seg_begin, st));
    TB_TRY(up(d_seg_off, seg_off, st));
    TB_TRY(up(d_seg_c, seg_c, st));
    TB_TRY(up(d_seg_ch0, seg_ch0, st));
    TB_TRY(up(d_seg_ch1, seg_ch1, st));
    TB_TRY(up(d_ch_seg, ch_seg, st));
    TB_TRY(up(d_ch_a0, ch_a0, st));
    TB_TRY(up(d_ch_a1, ch_a1, st));
    TB_TRY(cudaMemsetAsync(d_med_cnt, 0, S * 4, st));
    k_fill<<<blocks_for(A, bs), bs, 0, st>>>(best, A, -2.0);
    TB_TRY(cudaGetLastError());

    Level L{};
    L.S = S; L.seg_begin = d_seg_begin; L.seg_off = d_seg_off; L.seg_c = d_seg_c; L.med_cnt = d_med_cnt;
    L.med_row = d_med_row; L.med_pos = d_med_pos; L.u = d_u; L.cnt = d_cnt; L.A = A; L.perm = T.perm;
    L.x = x; L.rn = rn; L.dim = dim; L.best = best; L.d = dd; L.lab = lab; L.sorted_row = sorted_row;
    L.obj = obj; L.cl_of = cl_of; L.ch_seg = d_ch_seg; L.ch_a0 = d_ch_a0; L.ch_a1 = d_ch_a1;
    L.seg_ch0 = d_seg_ch0; L.seg_ch1 = d_seg_ch1; L.ccnt = d_ccnt; L.cpre = d_cpre;

    // ---- roulette-wheel initialisation (R24)
    std::vector<double> u(S);
    for (int j = 0; j < cmax; ++j) {
      for (int s = 0; s < S; ++s) u[s] = uniform01(seed, (uint64_t)segs[s], (uint64_t)j);
      TB_TRY(up(d_u, u, st));
      if (j > 0) {
        k_cos_update<<<blocks_for(A * 32, bs), bs, 0, st>>>(L, j - 1);
        TB_TRY(cudaGetLastError());
      }
      k_pick<<<blocks_for((int64_t)S * 32, bs), bs, 0, st>>>(L, j);
      TB_TRY(cudaGetLastError());
    }

    const bool dbg = getenv("REMOE_TREE_DEBUG") != nullptr;
    auto dump = [&](const char* tag) -> cudaError_t {
      if (!dbg) return cudaSuccess;
      std::vector<int64_t> mr;
      std::vector<int32_t> mc;
      cudaError_t e = down(mr, d_med_row, (size_t)S * C, st);
      if (e == cudaSuccess) e = down(mc, d_med_cnt, (size_t)S, st);
      for (int s2 = 0; s2 < S && e == cudaSuccess; ++s2) {
        fprintf(stderr, "TREE %s node %d:", tag, segs[s2]);
        for (int j = 0; j < mc[s2]; ++j) fprintf(stderr, " %lld", (long long)mr[(size_t)s2 * C + j]);
        fprintf(stderr, "\n");
      }
      return e;
    };
    TB_TRY(dump("init"));
    auto assign_and_sort = [&]() -> cudaError_t {
      k_assign<<<blocks_for(A * 32, bs), bs, 0, st>>>(L);
      k_chunk_count<<<nch, 1024, 0, st>>>(L);
      k_chunk_scan<<<blocks_for((int64_t)S * C, bs), bs, 0, st>>>(L);
      k_scatter<<<nch, 1024, 0, st>>>(L);
      return cudaGetLastError();
    };
    std::vector<int32_t> cnt;
    // ---- k-medoids iterations (R25)
    for (int it = 0; it < max_iter; ++it) {
      TB_TRY(assign_and_sort());
      TB_TRY(down(cnt, d_cnt, (size_t)S * C, st));
      std::vector<int32_t> cl_index((size_t)S * C, -1), cl_c0, cl_c1, cl_seg, cl_slot;
      std::vector<int64_t> cc_a0, cc_a1;
      for (int s = 0; s < S; ++s) {
        int64_t at = seg_off[s];
        for (int l = 0; l < C; ++l) {
          const int64_t cn = cnt[(size_t)s * C + l];
          if (cn == 0) continue;
          cl_index[(size_t)s * C + l] = (int32_t)cl_seg.size();
          cl_seg.push_back(s);
          cl_slot.push_back(l);
          cl_c0.push_back((int32_t)cc_a0.size());
          for (int64_t a = at; a < at + cn; a += 256) {
            cc_a0.push_back(a);
            cc_a1.push_back(std::min(a + 256, at + cn));
          }
          cl_c1.push_back((int32_t)cc_a0.size());
          at += cn;
        }
      }
      const int ncl = (int)cl_seg.size();
      const int ncc = (int)cc_a0.size();
      TB_TRY(g_part.need((size_t)ncc * dim * 8));
      TB_TRY(g_ssum.need((size_t)ncl * dim * 8));
      TB_TRY(g_cc_a0.need((size_t)ncc * 8));
      TB_TRY(g_cc_a1.need((size_t)ncc * 8));
      TB_TRY(g_cl_c0.need((size_t)ncl * 4));
      TB_TRY(g_cl_c1.need((size_t)ncl * 4));
      TB_TRY(g_cl_seg.need((size_t)ncl * 4));
      TB_TRY(g_cl_slot.need((size_t)ncl * 4));
      TB_TRY(g_best_bits.need((size_t)ncl * 8));
      TB_TRY(g_best_i.need((size_t)ncl * 8));
      TB_TRY(g_keep.need((size_t)ncl * 4));
      TB_TRY(up((int64_t*)g_cc_a0.p, cc_a0, st));
      TB_TRY(up((int64_t*)g_cc_a1.p, cc_a1, st));
      TB_TRY(up((int32_t*)g_cl_c0.p, cl_c0, st));
      TB_TRY(up((int32_t*)g_cl_c1.p, cl_c1, st));
      TB_TRY(up((int32_t*)g_cl_seg.p, cl_seg, st));
      TB_TRY(up((int32_t*)g_cl_slot.p, cl_slot, st));
      TB_TRY(up(d_cl_index, cl_index, st));
      TB_TRY(cudaMemsetAsync(g_best_bits.p, 0, (size_t)ncl * 8, st));
      TB_TRY(cudaMemsetAsync(g_best_i.p, 0xFF, (size_t)ncl * 8, st));
      TB_TRY(cudaMemsetAsync(g_keep.p, 0, (size_t)ncl * 4, st));
      TB_TRY(cudaMemsetAsync(d_changed, 0, 4, st));
      k_cluster_partial<<<ncc, 256, 0, st>>>(x, rn, dim, sorted_row, (int64_t*)g_cc_a0.p, (int64_t*)g_cc_a1.p,
                                             (double*)g_part.p);
      k_cluster_sum<<<ncl, 256, 0, st>>>(dim, (int32_t*)g_cl_c0.p, (int32_t*)g_cl_c1.p, (double*)g_part.p,
                                         (double*)g_ssum.p);
      k_obj<<<blocks_for(A * 32, bs), bs, 0, st>>>(L, d_cl_index, (double*)g_ssum.p,
                                                   (unsigned long long*)g_best_bits.p);
      k_obj_pick<<<blocks_for(A, bs), bs, 0, st>>>(L, (unsigned long long*)g_best_bits.p,
                                                   (unsigned long long*)g_best_i.p, (int32_t*)g_cl_seg.p,
                                                   (int32_t*)g_cl_slot.p, (int*)g_keep.p);
      k_commit_medoid<<<blocks_for(ncl, bs), bs, 0, st>>>(L, ncl, (int32_t*)g_cl_seg.p, (int32_t*)g_cl_slot.p,
                                                          (unsigned long long*)g_best_i.p, (int*)g_keep.p,
                                                          d_changed);
      TB_TRY(cudaGetLastError());
      std::vector<int> changed;
      TB_TRY(down(changed, d_changed, 1, st));
      TB_TRY(dump("iter"));
      if (!changed[0]) break;
    }
    // ---- final assignment to the final medoids, stable split (R26)
    TB_TRY(assign_and_sort());
    TB_TRY(down(cnt, d_cnt, (size_t)S * C, st));
    std::vector<int64_t> med_row;
    TB_TRY(down(med_row, d_med_row, (size_t)S * C, st));
    std::vector<uint8_t> commit(S, 0);
    const int64_t first_child = (int64_t)hb.size();
    for (int s = 0; s < S; ++s) {
      const int node = segs[s];
      const int64_t nb = seg_off[s + 1] - seg_off[s];
      int nonempty = 0;
      for (int l = 0; l < C; ++l) nonempty += cnt[(size_t)s * C + l] > 0;
      hc0[node] = (int32_t)hb.size();
      if (nonempty >= 2) {
        commit[s] = 1;
        int64_t at = seg_begin[s];
        for (int l = 0; l < C; ++l) {
          const int64_t cn = cnt[(size_t)s * C + l];
          if (cn == 0) continue;
          hb.push_back(at); he.push_back(at + cn); hp.push_back(node); hc0.push_back(-1); hnc.push_back(0);
          hm.push_back(med_row[(size_t)s * C + l]);
          at += cn;
        }
        hnc[node] = nonempty;
      } else {  // duplicates: c equal contiguous chunks, centroid = first member
        const int c = seg_c[s];
        for (int j = 0; j < c; ++j) {
          const int64_t b0 = seg_begin[s] + nb * j / c, b1 = seg_begin[s] + nb * (j + 1) / c;
          int64_t r = 0;
          TB_TRY(cudaMemcpyAsync(&r, T.perm + b0, 8, cudaMemcpyDeviceToHost, st));
          TB_TRY(cudaStreamSynchronize(st));
          hb.push_back(b0); he.push_back(b1); hp.push_back(node); hc0.push_back(-1); hnc.push_back(0);
          hm.push_back(r);
        }
        hnc[node] = c;
      }
    }
    TB_TRY(up(d_commit, commit, st));
    k_commit_perm<<<blocks_for(A, bs), bs, 0, st>>>(L, d_commit);
    TB_TRY(cudaGetLastError());
    lvl_lo = first_child;
    lvl_hi = (int64_t)hb.size();
    ++depth;
  }
  TB_TRY(cudaStreamSynchronize(st));

  T.n_nodes = (int)hb.size();
  T.depth = depth;
  for (int i = 0; i < T.n_nodes; ++i)
    if (hnc[i] == 0) {
      ++T.n_leaves;
      T.max_leaf = std::max<int>(T.max_leaf, (int)(he[i] - hb[i]));
    }
  TB_TRY(cudaMalloc(&T.begin, T.n_nodes * 8));
  TB_TRY(cudaMalloc(&T.end, T.n_nodes * 8));
  TB_TRY(cudaMalloc(&T.medoid, T.n_nodes * 8));
  TB_TRY(cudaMalloc(&T.child0, T.n_nodes * 4));
  TB_TRY(cudaMalloc(&T.nchild, T.n_nodes * 4));
  TB_TRY(up(T.begin, hb, st));
  TB_TRY(up(T.end, he, st));
  TB_TRY(up(T.medoid, hm, st));
  TB_TRY(up(T.child0, hc0, st));
  TB_TRY(up(T.nchild, hnc, st));
  TB_TRY(cudaStreamSynchronize(st));
  T.bytes = (size_t)n * 8 + (size_t)T.n_nodes * 32;
  T.h_begin = std::move(hb);
  T.h_end = std::move(he);
  T.h_medoid = std::move(hm);
  T.h_parent = std::move(hp);
  T.h_child0 = std::move(hc0);
  T.h_nchild = std::move(hnc);
  T.build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  guard.keep = true;
  *out = std::move(T);
  return REMOE_OK;
}

// ------------------------------------------------------------------ Algorithm 1
namespace {

struct SearchArgs {
  const uint16_t* x;
  const float* xnorm;
  int dim;
  const uint16_t* q;
  const float* qnorm;
  int k;
  float sigma;
  int64_t gid_offset;
  const int64_t* perm;
  const int64_t* begin;
  const int64_t* end;
  const int32_t* child0;
  const int32_t* nchild;
  const int64_t* medoid;
  uint64_t* top;
  int32_t* leaf;
  int32_t* n_eval;
};

// Eq. 11 of query (fp32 copy in shared memory) vs local row, fp32, warp-wide
__device__ __forceinline__ float warp_dot32(const float* __restrict__ qf, const uint16_t* __restrict__ xr, int dim) {
  const int lane = threadIdx.x & 31;
  float acc = 0.f;
  for (int c = lane; c < dim / 8; c += 32) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(xr + c * 8));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      acc = __fmaf_rn(qf[c * 8 + 2 * i], bf_lo(w[i]), acc);
      acc = __fmaf_rn(qf[c * 8 + 2 * i + 1], bf_hi(w[i]), acc);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
  return acc;
}

// Score the children of `node`, write them to `sorted` by key descending.  Block-wide.
__device__ int rank_children(const SearchArgs& a, const float* qf, float qn, int node, int* sorted, uint64_t* keys) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nc = a.nchild[node], c0 = a.child0[node];
  for (int i = warp; i < nc; i += blockDim.x >> 5) {
    const int64_t row = a.medoid[c0 + i];
    const float dot = warp_dot32(qf, a.x + row * a.dim, a.dim);
    if (lane == 0) keys[i] = make_key(eq11(dot, qn, a.xnorm[row], a.sigma), row + a.gid_offset);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < nc; ++i) {  // insertion sort by key, descending
      int j = i;
      const uint64_t kk = keys[i];
      while (j > 0 && keys[sorted[j - 1] - c0] < kk) {
        sorted[j] = sorted[j - 1];
        --j;
      }
      sorted[j] = c0 + i;
    }
  }
  __syncthreads();
  return nc;
}

__global__ void __launch_bounds__(256) k_tree_search(SearchArgs a) {
  extern __shared__ float qf[];
  __shared__ uint64_t cand[kTreeCandCap];
  __shared__ int path_node[kTreeMaxDepth];
  __shared__ int path_sorted[kTreeMaxDepth][kTreeCMax];
  __shared__ int dfs_sorted[kTreeMaxDepth][kTreeCMax];
  __shared__ uint64_t keys[kTreeCMax];
  __shared__ int leaves[257];
  __shared__ int64_t leaf_cum[258];
  const int b = blockIdx.x, t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const uint16_t* qb = a.q + (int64_t)b * a.dim;
  for (int i = t; i < a.dim / 2; i += blockDim.x) {
    const uint32_t w = reinterpret_cast<const uint32_t*>(qb)[i];
    qf[2 * i] = bf_lo(w);
    qf[2 * i + 1] = bf_hi(w);
  }
  const float qn = a.qnorm[b];
  __syncthreads();
  int ne = 0;
  // descent (Alg. 1 line 4): successively the closest subcluster centroid
  int node = 0, depth = 0;
  while (a.nchild[node] > 0) {
    ne += rank_children(a, qf, qn, node, path_sorted[depth], keys);
    path_node[depth] = node;
    node = path_sorted[depth][0];
    ++depth;
  }
  const int leaf = node;
  int nl = 0;
  int64_t count = 0;
  if (t == 0) {
    leaves[0] = leaf;
    leaf_cum[0] = 0;
  }
  nl = 1;
  count = a.end[leaf] - a.begin[leaf];
  // supplement from siblings (Alg. 1 lines 6-9, R28): each sibling subtree depth-first,
  // children in key order, whole leaves, until >= alpha candidates; then one level up
  int stk_node[kTreeMaxDepth], stk_pos[kTreeMaxDepth];
  int cur = leaf;
  for (int lvl = depth - 1; lvl >= 0 && count < a.k; --lvl) {
    const int parent = path_node[lvl];
    const int nc = a.nchild[parent];
    for (int i = 0; i < nc && count < a.k; ++i) {
      const int c = path_sorted[lvl][i];
      if (c == cur) continue;
      int sp = 0;
      stk_node[0] = c;
      stk_pos[0] = -1;
      while (sp >= 0 && count < a.k) {
        const int nd = stk_node[sp];
        if (a.nchild[nd] == 0) {
          if (t == 0) leaves[nl] = nd;
          ++nl;
          count += a.end[nd] - a.begin[nd];
          --sp;
          continue;
        }
        if (stk_pos[sp] < 0) {
          ne += rank_children(a, qf, qn, nd, dfs_sorted[sp], keys);
          stk_pos[sp] = 0;
        }
        if (stk_pos[sp] >= a.nchild[nd]) {
          --sp;
          continue;
        }
        const int child = dfs_sorted[sp][stk_pos[sp]++];
        ++sp;
        stk_node[sp] = child;
        stk_pos[sp] = -1;
      }
    }
    cur = parent;
  }
  __syncthreads();
  if (t == 0) {
    int64_t run = 0;
    for (int i = 0; i < nl; ++i) {
      leaf_cum[i] = run;
      run += a.end[leaves[i]] - a.begin[leaves[i]];
    }
    leaf_cum[nl] = run;
  }
  __syncthreads();
  const int R = (int)count;  // <= k - 1 + beta <= kTreeCandCap (checked at build)
  // leaf brute force (Alg. 1 line 5): every gathered member, warp per row
  for (int r = warp; r < R; r += blockDim.x >> 5) {
    int li = 0;
    while (leaf_cum[li + 1] <= r) ++li;
    const int64_t row = a.perm[a.begin[leaves[li]] + (r - leaf_cum[li])];
    const float dot = warp_dot32(qf, a.x + row * a.dim, a.dim);
    if (lane == 0) cand[r] = make_key(eq11(dot, qn, a.xnorm[row], a.sigma), row + a.gid_offset);
  }
  ne += R;
  int np2 = 1;
  while (np2 < R) np2 <<= 1;
  if (np2 < 2) np2 = 2;
  for (int i = R + t; i < np2; i += blockDim.x) cand[i] = 0;
  __syncthreads();
  // exact top-alpha: block bitonic sort, descending
  for (int size = 2; size <= np2; size <<= 1) {
    for (int j = size >> 1; j > 0; j >>= 1) {
      for (int i = t; i < (np2 >> 1); i += blockDim.x) {
        const int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1)), hi = lo + j;
        const uint64_t x0 = cand[lo], x1 = cand[hi];
        const bool desc = (lo & size) == 0;
        if (desc ? x0 < x1 : x0 > x1) {
          cand[lo] = x1;
          cand[hi] = x0;
        }
      }
      __syncthreads();
    }
  }
  for (int i = t; i < a.k; i += blockDim.x) a.top[(int64_t)b * a.k + i] = i < R ? cand[i] : 0;
  if (t == 0) {
    if (a.leaf) a.leaf[b] = leaf;
    if (a.n_eval) a.n_eval[b] = ne;
  }
}

}  // namespace

cudaError_t launch_tree_search(const Tree& t, const uint16_t* x, const float* xnorm, int dim, const uint16_t* q,
                               const float* qnorm, int B, int k, float sigma, int64_t gid_offset, uint64_t* top,
                               int32_t* leaf, int32_t* n_eval, cudaStream_t st) {
  if (B <= 0) return cudaSuccess;
  SearchArgs a{x, xnorm, dim, q, qnorm, k, sigma, gid_offset, t.perm, t.begin, t.end, t.child0, t.nchild,
               t.medoid, top, leaf, n_eval};
  const size_t smem = (size_t)dim * 4;
  cudaError_t e = set_smem_attrs_once((const void*)k_tree_search, 4096 * 4);  // max dim
  if (e != cudaSuccess) return e;
  k_tree_search<<<B, 256, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace remoe
