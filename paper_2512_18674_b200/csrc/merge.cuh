// merge.cuh -- S4/S5 key-list merge and S6+S7 finalize as device functions of a
// 256-thread group with a caller-supplied barrier and shared-memory scratch, so that the
// same code runs as the stand-alone kernels (k_post.cu: __syncthreads, one CTA per query)
// and fused into the tail of the tensor-core scan (k_scan_tc.cu: the 8 epilogue warps of
// the last CTAs to finish, a named barrier, the idle TMA ring as scratch).
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace remoe {

// ---------------------------------------------------------------- S4 / S5 merge
// One 256-thread group per query.  The answer is the k largest keys of the union of the
// lists (keys are unique: they carry the global id).  Exact selection:
//   1. the k-th largest list head (lists are sorted) is a real key <= the final k-th key:
//      it raises the lower bound lb (the scan's shared threshold; 1 = "any real key");
//   2. keys >= lb are appended to shared memory with one atomic per warp (lists longer
//      than 32 keys: only the (list, 32-key chunk) items that can hold a survivor);
//   3. n <= kRankMax survivors: each survivor's rank = #{survivors > it} (broadcast reads
//      of shared memory, O(n^2 / 256) compares per thread), rank < k -> out[rank];
//      kRankMax < n <= kSelCap: bitonic sort; n > kSelCap: an MSB-first 8-bit radix
//      select finds the k-th largest key T exactly, and keys >= T are re-collected.
constexpr int kSelCap = 2048;
constexpr int kRankMax = 512;
constexpr int kItemCap = 4096;
constexpr int kMergeThreads = 256;

// Shared-memory scratch of one merge + finalize (~38 KB, 16-byte aligned).
struct MergeScratch {
  uint64_t cand[kSelCap];
  uint64_t topk[256];
  uint32_t items[kItemCap];  // (list << 3) | chunk
  unsigned hist[256];
  float w[256];
  const float* src[256];
  float red[8];
  int wcnt[8];
  uint64_t prefix;
  int cnt, need, n_items;
};

template <class Bar>
__device__ __forceinline__ void block_sort_desc(uint64_t* a, int np2, int t, Bar bar) {
  for (int size = 2; size <= np2; size <<= 1) {
    for (int j = size >> 1; j > 0; j >>= 1) {
      for (int i = t; i < (np2 >> 1); i += kMergeThreads) {
        const int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1)), hi = lo + j;  // j is a power of 2
        const uint64_t x = a[lo], y = a[hi];
        const bool desc = (lo & size) == 0;
        if (desc ? x < y : x > y) { a[lo] = y; a[hi] = x; }
      }
      bar();
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
__device__ __forceinline__ void peer_signal(const PeerXchg& px, unsigned long long seq) {
  __threadfence_system();  // this CTA's peer stores before its arrival
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned done = atomicAdd(px.counter, 1u);
    if (done == gridDim.x - 1) {
      atomicExch(px.counter, 0u);
      __threadfence_system();  // every CTA's stores (seen through the counter) before the flags
      for (int g = 0; g < px.G; ++g)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(px.flag_dst[g]), "l"(seq) : "memory");
    }
  }
}

// ---------------------------------------------------------------- S6 + S7
// w_r = softmax(s_r / T), max-subtracted: s_0 is the largest score of the
// sorted list.  exp in parallel, the normaliser by a fixed xor tree (order
// independent of batch position).  P[e] = sum_r w_r A_r[e], r ascending over the rows
// that contribute (all k on one GPU; the owned ones for a multi-GPU partial, mode 2).
// 256 threads (t = 0..255); outputs j = j0 + t, j0 + t + 256, ... < j1.
template <class Bar>
__device__ __forceinline__ void finalize_query(const uint64_t* tb, int k, int b, const FinalizeArgs& f,
                                               int64_t j0, int64_t j1, bool write_ids, int t, Bar bar,
                                               MergeScratch& S, int64_t pred_off = 0) {
  const int lane = t & 31, warp = t >> 5;
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
  if (lane == 0) { S.red[warp] = z; S.wcnt[warp] = __popc(keep); }
  bar();
  float Z = 0.f;
  int before = 0, nr = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    Z += S.red[i];
    before += i < warp ? S.wcnt[i] : 0;
    nr += S.wcnt[i];
  }
  if (my_src != nullptr) {
    const int pos = before + __popc(keep & ((1u << lane) - 1u));
    S.w[pos] = __fdiv_rn(e, Z);
    S.src[pos] = my_src;
  }
  bar();
  if ((f.LE & 3) == 0 && (j0 & 3) == 0 && ((j1 & 3) == 0 || j1 == f.LE)) {
    // float4 columns, two per thread per step, 8 rows at a time (16 x 16-byte loads in
    // flight): per element the same r-ascending FMA chain as the scalar path below
    const int64_t c0 = j0 >> 2, c1 = (j1 + 3) >> 2;
    for (int64_t ca = c0 + t; ca < c1; ca += 2 * (int64_t)kMergeThreads) {
      const int64_t cb = ca + kMergeThreads;
      const bool vb = cb < c1;
      float4 acc_a = make_float4(0.f, 0.f, 0.f, 0.f), acc_b = acc_a;
      for (int r0 = 0; r0 < nr; r0 += 8) {
        float4 xa[8], xb[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const bool vr = r0 + u < nr;
          const float4 zz = make_float4(0.f, 0.f, 0.f, 0.f);
          xa[u] = vr ? __ldg(reinterpret_cast<const float4*>(S.src[r0 + u]) + ca) : zz;
          xb[u] = (vr && vb) ? __ldg(reinterpret_cast<const float4*>(S.src[r0 + u]) + cb) : zz;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (r0 + u < nr) {  // r ascending
            const float wr = S.w[r0 + u];
            acc_a.x = __fmaf_rn(wr, xa[u].x, acc_a.x); acc_a.y = __fmaf_rn(wr, xa[u].y, acc_a.y);
            acc_a.z = __fmaf_rn(wr, xa[u].z, acc_a.z); acc_a.w = __fmaf_rn(wr, xa[u].w, acc_a.w);
            acc_b.x = __fmaf_rn(wr, xb[u].x, acc_b.x); acc_b.y = __fmaf_rn(wr, xb[u].y, acc_b.y);
            acc_b.z = __fmaf_rn(wr, xb[u].z, acc_b.z); acc_b.w = __fmaf_rn(wr, xb[u].w, acc_b.w);
          }
        }
      }
      for (int o = 0; o < no; ++o) {
        reinterpret_cast<float4*>(outs[o] + pred_off + (int64_t)b * f.LE)[ca] = acc_a;
        if (vb) reinterpret_cast<float4*>(outs[o] + pred_off + (int64_t)b * f.LE)[cb] = acc_b;
      }
    }
    return;
  }
  // two outputs per thread per step, 8 rows at a time: 16 independent loads in flight
  for (int64_t ja = j0 + t; ja < j1; ja += 2 * (int64_t)kMergeThreads) {
    const int64_t jb = ja + kMergeThreads;
    const bool vb = jb < j1;
    float acc_a = 0.f, acc_b = 0.f;
    for (int r0 = 0; r0 < nr; r0 += 8) {
      float xa[8], xb[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool vr = r0 + u < nr;
        xa[u] = vr ? __ldg(S.src[r0 + u] + ja) : 0.f;
        xb[u] = (vr && vb) ? __ldg(S.src[r0 + u] + jb) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (r0 + u < nr) {  // r ascending
          acc_a = __fmaf_rn(S.w[r0 + u], xa[u], acc_a);
          acc_b = __fmaf_rn(S.w[r0 + u], xb[u], acc_b);
        }
      }
    }
    for (int o = 0; o < no; ++o) {
      outs[o][pred_off + (int64_t)b * f.LE + ja] = acc_a;
      if (vb) outs[o][pred_off + (int64_t)b * f.LE + jb] = acc_b;
    }
  }
}

// Merge for query b: key(l, i) = in[b * qstride + l * lstride + i] (n_lists sorted lists
// of list_len keys) -> out[b * k + i]; see launch_merge (kernels.h) for set_thr / lower /
// fin / reset_lower and px (nullable; its key_dst stores only -- waiting and signalling
// are the caller's).  All 256 threads of the group call it; bar() synchronises them.
template <class Bar>
__device__ __forceinline__ void merge_query(const uint64_t* __restrict__ in, int b, int n_lists, int64_t qstride,
                                            int64_t lstride, int list_len, int k, uint64_t* __restrict__ out,
                                            unsigned long long* __restrict__ set_thr,
                                            unsigned long long* __restrict__ lower, const FinalizeArgs& fin,
                                            int reset_lower, const PeerXchg* px, int t, Bar bar,
                                            MergeScratch& S, int64_t j0 = 0, int64_t j1 = -1,
                                            bool primary = true, unsigned* split_cnt = nullptr,
                                            int n_split = 1, int64_t key_off = 0, int64_t pred_off = 0) {
  const int warp = t >> 5, lane = t & 31;
  const uint64_t* base = in + (int64_t)b * qstride;
  const int nch = (list_len + 31) >> 5;
  const int items = n_lists * nch;
  // Short contiguous lists (<= 32 keys each, <= 8 keys per thread in all): ONE round trip --
  // every key of the query is loaded here, together with lb, and the list heads (key f is
  // the head of list f / list_len when f % list_len == 0) come from the same registers.
  const int64_t n_keys = (int64_t)n_lists * list_len;
  const bool one_trip = nch == 1 && lstride == (int64_t)list_len && n_keys <= 8 * kMergeThreads &&
                        n_lists >= k && n_lists <= kSelCap;
  uint64_t kk1[8];
  if (one_trip) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int f = t + kMergeThreads * u;
      kk1[u] = f < n_keys ? __ldcg(base + f) : 0ull;
    }
  }
  uint64_t lb = lower ? lower[b] : 0ull;
  if (t == 0) S.cnt = 0;
  bar();  // every thread has read lb; cnt is zero
  // the next chunk's scan starts from no threshold: reset once every column split of this
  // query has read it (the last of n_split CTAs to arrive)
  if (lower && reset_lower && t == 0) {
    if (n_split <= 1) lower[b] = 0ull;
    else if (atomicAdd(split_cnt + b, 1u) == (unsigned)n_split - 1) { lower[b] = 0ull; split_cnt[b] = 0u; }
  }
  if (lb == 0) lb = 1;  // sentinel keys (0) never count
  // the lists of one query are usually contiguous (lstride == list_len): flat key f is base[f]
  const bool contiguous = lstride == (int64_t)list_len;
  auto item_key = [&](int it) -> uint64_t {
    if (it >= items) return 0ull;
    const int l = nch == 1 ? it : it / nch, c = it - l * nch;
    const int i = c * 32 + lane;
    return i < list_len ? __ldcg(base + (int64_t)l * lstride + i) : 0ull;
  };
  // flat key f = l * list_len + i: the whole block reads 8 keys per thread per round
  // (one L2 round trip per 2048 keys, instead of one per 32 lists of a warp)
  auto flat_key = [&](int64_t f) -> uint64_t {
    if (f >= n_keys) return 0ull;
    if (contiguous) return __ldcg(base + f);
    const int64_t l = f / list_len, i = f - l * list_len;
    return __ldcg(base + l * lstride + i);
  };
  auto append = [&](uint64_t key, uint64_t thr_lo) {  // whole warp; keys >= thr_lo to cand
    const unsigned m = __ballot_sync(kFull, key >= thr_lo);
    if (m) {
      int pos0 = 0;
      if (lane == 0) pos0 = atomicAdd(&S.cnt, __popc(m));
      pos0 = __shfl_sync(kFull, pos0, 0);
      const int pos = pos0 + __popc(m & ((1u << lane) - 1u));
      if (key >= thr_lo && pos < kSelCap) S.cand[pos] = key;
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
    if (t == 0) S.n_items = 0;
    bar();
    for (int l = t; l < n_lists; l += kMergeThreads) {
      const uint64_t* lp = base + (int64_t)l * lstride;
      int need = 1;
      while (need < nch && __ldcg(lp + 32 * need - 1) >= thr_lo) ++need;
      const int pos = atomicAdd(&S.n_items, need);
      for (int c = 0; c < need; ++c) S.items[pos + c] = ((uint32_t)l << 3) | (uint32_t)c;
    }
    bar();
    const int ni = S.n_items;
    for (int i0 = warp; i0 < ni; i0 += 8 * 4) {
      uint64_t kk[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int it = i0 + 8 * u;
        kk[u] = 0ull;
        if (it < ni) {
          const uint32_t w = S.items[it];
          const int i = (int)(w & 7u) * 32 + lane;
          if (i < list_len) kk[u] = __ldcg(base + (int64_t)(w >> 3) * lstride + i);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) append(kk[u], thr_lo);
    }
  };
  // Lists are sorted: the k-th largest list head is a real key <= the final k-th key,
  // a much tighter bound than lb when the state lists are many (S4: 1 or 2 per CTA).
  if (n_lists >= k && n_lists <= kSelCap) {
    if (t == 0) S.prefix = 0ull;
    if (one_trip) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int f = t + kMergeThreads * u;
        if (f < n_keys && f % list_len == 0) S.cand[f / list_len] = kk1[u];
      }
    } else {
      for (int l = t; l < n_lists; l += kMergeThreads) S.cand[l] = __ldcg(base + (int64_t)l * lstride);
    }
    bar();
    for (int i = t; i < n_lists; i += kMergeThreads) {
      const uint64_t x = S.cand[i];
      if (x == 0) continue;  // empty list; real keys are distinct
      int r = 0;
      for (int j = 0; j < n_lists; ++j) r += S.cand[j] > x;
      if (r == k - 1) S.prefix = x;
    }
    bar();
    if (S.prefix > lb) lb = S.prefix;
    bar();
  }
  if (one_trip) {
#pragma unroll
    for (int u = 0; u < 8; ++u) append(kk1[u], lb);  // the keys are already in registers
  } else if (nch >= 2 && nch <= 8 && (int64_t)n_lists * nch <= kItemCap) {
    collect_lists(lb);
  } else {
    collect(lb);
  }
  bar();
  int n = S.cnt;
  if (n > kSelCap) {
    // radix select of the k-th largest key among keys >= lb
    uint64_t prefix = 0, pmask = 0;
    int need = k;
    for (int shift = 56; shift >= 0; shift -= 8) {
      S.hist[t] = 0;
      bar();
      for (int it0 = warp; it0 < items; it0 += 8) {
        const uint64_t key = item_key(it0);
        if (key >= lb && (key & pmask) == prefix) atomicAdd(&S.hist[(key >> shift) & 255u], 1u);
      }
      bar();
      if (warp == 0) {  // suffix sums over the 256 bins: lane l owns bins 255-8l .. 248-8l
        int h[8], tot = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) { h[u] = S.hist[255 - 8 * lane - u]; tot += h[u]; }
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
              S.prefix = prefix | ((uint64_t)(255 - 8 * lane - u) << shift);
              S.need = need - c;
              break;
            }
            c += h[u];
          }
        }
      }
      bar();
      prefix = S.prefix;
      need = S.need;
      pmask |= (uint64_t)255 << shift;
      bar();
    }
    if (t == 0) S.cnt = 0;
    bar();
    collect(prefix);  // exactly k keys: keys are unique and prefix is the k-th largest
    bar();
    n = S.cnt;
  }
  const int nout = n < k ? n : k;
  if (n <= kRankMax) {
    for (int i = t; i < n; i += kMergeThreads) {
      const uint64_t x = S.cand[i];
      int r = 0;
      for (int j = 0; j < n; ++j) r += S.cand[j] > x;
      if (r < k) S.topk[r] = x;
    }
  } else {
    int np2 = 1;
    while (np2 < n) np2 <<= 1;
    for (int i = n + t; i < np2; i += kMergeThreads) S.cand[i] = 0ull;
    bar();
    block_sort_desc(S.cand, np2, t, bar);
    for (int i = t; i < nout; i += kMergeThreads) S.topk[i] = S.cand[i];
  }
  bar();
  for (int i = t; primary && i < k; i += kMergeThreads) {
    const uint64_t v = i < nout ? S.topk[i] : 0ull;
    out[(int64_t)b * k + i] = v;
    if (px && px->G > 0 && px->key_dst[0])  // fused exchange 1: straight into every rank's gathered slot
      for (int g = 0; g < px->G; ++g) px->key_dst[g][key_off + (int64_t)b * k + i] = v;
  }
  if (set_thr && primary && t == 0) {
    // seeding: the k-th best key of a subset of rows, minus one (strict lower bound,
    // the subset's own rows stay admissible in the full scan)
    const uint64_t kth = k <= nout ? S.topk[k - 1] : 0ull;
    set_thr[b] = kth ? kth - 1 : 0ull;
  }
  if (fin.act != nullptr) {  // fused S6 + S7 (one GPU) or S6 + partial S7 (multi-GPU)
    if (nout < k)
      for (int i = nout + t; i < k; i += kMergeThreads) S.topk[i] = 0ull;
    bar();
    finalize_query(S.topk, k, b, fin, j0, j1 < 0 ? fin.LE : j1, primary, t, bar, S, pred_off);
  }
}

}  // namespace remoe
