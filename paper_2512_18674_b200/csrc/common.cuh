// common.cuh -- device primitives shared by the SPS kernels (sm_100a).
//
// * Candidate keys: u64 = ordf(fp32 score) << 32 | (0xFFFFFFFF - gid).
//   The larger key is the better candidate: score descending, then global id
//   ascending (DESIGN R5).  Key 0 is the "no candidate" sentinel; every real key
//   is >= 1.  -0.0 is canonicalised to +0.0 before packing.
// * Warp bitonic sort of 32*P keys held P per lane (index i = lane*P + p).
// * Thread-private top-k ("one lane owns one query"): a threshold in a register
//   plus an append-only buffer of CAP = 32*P keys in global memory (L2); when a
//   lane's buffer is full the whole warp sorts it and keeps the best k.  Exact:
//   nothing better than the k-th kept key is ever discarded.
// * mbarrier / bulk-copy (TMA) PTX wrappers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace remoe {

constexpr uint32_t kFull = 0xFFFFFFFFu;

// ---------------------------------------------------------------- keys
__device__ __forceinline__ uint32_t ordf(float f) {
  uint32_t u = __float_as_uint(f);
  if ((u & 0x7FFFFFFFu) == 0) u = 0;  // -0 -> +0
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unordf(uint32_t o) {
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o);
}
__device__ __forceinline__ uint64_t make_key(float s, int64_t gid) {
  return ((uint64_t)ordf(s) << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)gid);
}
__device__ __forceinline__ int64_t key_gid(uint64_t k) {
  return (int64_t)(0xFFFFFFFFu - (uint32_t)(k & 0xFFFFFFFFull));
}
__device__ __forceinline__ float key_score(uint64_t k) { return unordf((uint32_t)(k >> 32)); }

// Eq. 11 on fp32 pieces: dot / (|q| |x| + sigma).  One fused multiply-add
// for the denominator and one IEEE division; identical in every kernel.
__device__ __forceinline__ float eq11(float dot, float qn, float xn, float sigma) {
  return __fdiv_rn(dot, __fmaf_rn(qn, xn, sigma));
}

// v[j] for a run-time j in [0, 32) as a 5-level select tree over registers.  Indexing a
// register array with a run-time j makes nvcc copy the whole array to the local stack
// (ncu: ~57 MB of local-store write-back to DRAM per 1M-row scan launch); 31 SELs per
// candidate keep it in registers.
__device__ __forceinline__ uint32_t sel32(const uint32_t (&v)[32], int j) {
  uint32_t a[16], b[8], c[4], d[2];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = (j & 16) ? v[i + 16] : v[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) b[i] = (j & 8) ? a[i + 8] : a[i];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i] = (j & 4) ? b[i + 4] : b[i];
#pragma unroll
  for (int i = 0; i < 2; ++i) d[i] = (j & 2) ? c[i + 2] : c[i];
  return (j & 1) ? d[1] : d[0];
}

// bf16 bit pairs packed in a 32-bit word -> fp32 (exact)
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

__device__ __forceinline__ uint64_t umax64(uint64_t a, uint64_t b) { return a > b ? a : b; }
__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// ---------------------------------------------------------------- warp bitonic sort
// Sorts the 32*P keys of the warp in DESCENDING order; element i = lane*P + p.
template <int P>
__device__ __forceinline__ void warp_sort_desc(uint64_t (&v)[P]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int size = 2; size <= 32 * P; size <<= 1) {
#pragma unroll
    for (int j = size >> 1; j > 0; j >>= 1) {
      if (j >= P) {
        const int lj = j / P;
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const int i = lane * P + p;
          const uint64_t o = __shfl_xor_sync(kFull, v[p], lj);
          const bool up = (i & size) == 0;
          const bool lower = (i & j) == 0;
          v[p] = (lower == up) ? umax64(v[p], o) : umin64(v[p], o);
        }
      } else {
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const int q = p ^ j;
          if (q > p) {
            const int i = lane * P + p;
            const uint64_t a = v[p], b = v[q];
            if ((i & size) == 0) { v[p] = umax64(a, b); v[q] = umin64(a, b); }
            else                 { v[p] = umin64(a, b); v[q] = umax64(a, b); }
          }
        }
      }
    }
  }
}

// Key at sorted position `pos` (warp-uniform), broadcast to all lanes.
template <int P>
__device__ __forceinline__ uint64_t warp_key_at(const uint64_t (&v)[P], int pos) {
  uint64_t mine = 0;
#pragma unroll
  for (int p = 0; p < P; ++p)
    if (p == (pos % P)) mine = v[p];
  return __shfl_sync(kFull, mine, pos / P);
}

// Sort the first `cnt` keys of buf (others read as 0) and write the best `k`
// back to buf[0..k) (or to `out` if non-null).  Returns the k-th best key
// (0 if cnt < k).  Whole warp, warp-uniform arguments.  Out of line: one copy of
// the unrolled network per kernel keeps the instruction footprint small (a cold
// instruction cache, not the sort, dominated small merges when it was inlined).
template <int P>
__device__ __noinline__ uint64_t warp_compact(uint64_t* buf, int cnt, int k, uint64_t* out) {
  const int lane = threadIdx.x & 31;
  uint64_t v[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const int i = lane * P + p;
    v[p] = i < cnt ? buf[i] : 0ull;
  }
  warp_sort_desc<P>(v);
  __syncwarp();
  uint64_t* dst = out ? out : buf;
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const int i = lane * P + p;
    if (i < k) dst[i] = v[p];
  }
  __syncwarp();
  return cnt >= k ? warp_key_at<P>(v, k - 1) : 0ull;
}

// Slow path of LaneTopk::push (rare, kept out of line): compact the full buffer of
// every lane named in `full` (warp-uniform); returns this lane's new threshold.
template <int P>
__device__ __noinline__ uint64_t lane_compact_slow(unsigned full, uint64_t* mybuf, int mycnt, int k) {
  const int lane = threadIdx.x & 31;
  uint64_t mine = 0;
  while (full) {
    const int L = __ffs(full) - 1;
    full &= full - 1;
    uint64_t* b = (uint64_t*)__shfl_sync(kFull, (unsigned long long)mybuf, L);
    const int c = __shfl_sync(kFull, mycnt, L);
    const uint64_t t = warp_compact<P>(b, c, k, nullptr);
    if (lane == L) mine = t;
  }
  return mine;
}

// Thread-private top-k state of one lane (one query per lane).
//
// Threshold sharing: every state of query q (other lanes, warps and CTAs) publishes
// its k-th best key to gthr[q] with atomicMax, and reads it back now and then.  Any
// state's k-th best is a lower bound of the final k-th best of the whole shard, so
// discarding keys <= max(published) is exact and cuts inserts to ~the single-state
// rate no matter how the rows are split across threads.
template <int P>
struct LaneTopk {
  static constexpr int CAP = 32 * P;
  uint64_t thr;   // discard keys <= thr
  float tlim;     // conservative score pre-filter: key > thr implies dot >= tlim * den
  int cnt;        // keys in buf
  uint64_t* buf;  // CAP keys, private to this lane
  unsigned long long* g;  // shared threshold of this lane's query (nullptr: none)

  __device__ __forceinline__ void init(uint64_t* b, unsigned long long* gt) {
    thr = 0; tlim = -__int_as_float(0x7f800000); cnt = 0; buf = b; g = gt;
  }

  __device__ __forceinline__ void raise(uint64_t t) {
    if (t > thr) {
      thr = t;
      // a score s = RN(dot / den) (den > 0) can beat thr only if dot >= tlim * den:
      // tlim sits 2^-18 (relative) below thr's score, far more than the few-ulp
      // rounding of the division and of tlim * den
      const float ts = key_score(t);
      tlim = ts - fabsf(ts) * 3.814697265625e-06f - 1e-30f;
    }
  }

  __device__ __forceinline__ uint64_t peek_shared() const {
    return g ? *reinterpret_cast<volatile unsigned long long*>(g) : 0ull;
  }

  __device__ __forceinline__ bool may_pass(float dot, float den) const { return dot >= tlim * den; }

  // Whole warp: compact the lanes in `full` (warp-uniform mask) down to their best k.
  __device__ __forceinline__ void compact(unsigned full, int k) {
    const uint64_t t = lane_compact_slow<P>(full, buf, cnt, k);
    if ((full >> (threadIdx.x & 31)) & 1u) {
      cnt = cnt < k ? cnt : k;
      if (t) {
        if (g) atomicMax(g, (unsigned long long)t);
        raise(t);
      }
    }
  }

  // Whole warp: make room for `need` more keys in every lane's buffer (need <= CAP - k).
  __device__ __forceinline__ void ensure_room(int need, int k) {
    const unsigned full = __ballot_sync(kFull, cnt + need > CAP);
    if (full) compact(full, k);
  }

  // Append without a capacity check (after ensure_room).
  __device__ __forceinline__ void append(uint64_t key) {
    if (key > thr) buf[cnt++] = key;
  }

  // Whole warp calls with one key per lane (0 = nothing to offer).
  __device__ __forceinline__ void push(uint64_t key, int k) {
    const unsigned full = __ballot_sync(kFull, key > thr && cnt == CAP);
    if (full) compact(full, k);
    if (key > thr) buf[cnt++] = key;
  }

  // Out-of-line push for hot loops (keeps the unrolled common path small): the
  // state travels by value in registers.
  struct State { uint64_t thr; float tlim; int cnt; };
  __device__ __forceinline__ State save() const { return State{thr, tlim, cnt}; }
  __device__ __forceinline__ void load(const State& s) { thr = s.thr; tlim = s.tlim; cnt = s.cnt; }
  static __device__ __noinline__ State push_call(State st, uint64_t key, int k, uint64_t* b,
                                                 unsigned long long* gt) {
    LaneTopk t;
    t.thr = st.thr; t.tlim = st.tlim; t.cnt = st.cnt; t.buf = b; t.g = gt;
    t.push(key, k);
    return t.save();
  }
  __device__ __forceinline__ void push_ool(uint64_t key, int k) { load(push_call(save(), key, k, buf, g)); }

  // Whole warp: write each lane's sorted best k to out_of(lane) (k keys, zero padded).
  // The sort network is sized to the lane's fill, not to CAP: with seeded thresholds a
  // buffer usually holds a handful of keys, and sorting all CAP = 512 slots of 32 lanes
  // one after another cost ~0.5 ms per scan at k = 128.
  // scratch (optional): 32 keys of shared memory private to this lane -- a buffer in global
  // memory (k > 32 with large CAP) is then sorted there instead of in place: the in-place
  // insertion sort's dependent global loads and stores cost ~20-30 us per k = 64/128 scan.
  __device__ __forceinline__ void flush(uint64_t* my_out, int k, uint64_t* scratch = nullptr) {
    const int lane = threadIdx.x & 31;
    // lanes holding at most 32 keys sort their own buffer (insertion sort, all lanes at
    // once) and write their list themselves; only fuller buffers take the warp network
    const bool self = my_out != nullptr && cnt <= 32;
    if (self) {
      uint64_t* sb = buf;
      if (scratch) {
        for (int i = 0; i < cnt; ++i) scratch[i] = buf[i];  // independent loads, in flight together
        sb = scratch;
      }
      for (int i = 1; i < cnt; ++i) {
        const uint64_t x = sb[i];
        int j = i - 1;
        while (j >= 0 && sb[j] < x) { sb[j + 1] = sb[j]; --j; }
        sb[j + 1] = x;
      }
      for (int i = 0; i < k; ++i) my_out[i] = i < cnt ? sb[i] : 0ull;
    }
    const unsigned rest = __ballot_sync(kFull, my_out != nullptr && !self);
    for (int L = 0; L < 32; ++L) {
      if (!((rest >> L) & 1u)) continue;
      uint64_t* b = (uint64_t*)__shfl_sync(kFull, (unsigned long long)buf, L);
      uint64_t* o = (uint64_t*)__shfl_sync(kFull, (unsigned long long)my_out, L);
      const int c = __shfl_sync(kFull, cnt, L);
      if (o == nullptr) continue;
      int n;  // slots the network sorts and writes (those past c read as 0)
      if (c <= 64 || P <= 2) { warp_compact<2>(b, c, k, o); n = 64; }
      else if (c <= 128 || P <= 4) { warp_compact<(P < 4 ? P : 4)>(b, c, k, o); n = 128; }
      else if (c <= 256 || P <= 8) { warp_compact<(P < 8 ? P : 8)>(b, c, k, o); n = 256; }
      else { warp_compact<P>(b, c, k, o); n = CAP; }
      for (int i = n + lane; i < k; i += 32) o[i] = 0ull;
      __syncwarp();
    }
  }
};

// Register-resident top-K of one lane (K = pow2ceil(k) <= 16): a descending list
// updated by an unrolled insertion network (~4 instructions per slot, no memory, no
// warp sync).  The threshold is the K-th best seen (<= the k-th best: a valid, slightly
// conservative bound) or the shared one, if higher; inserts stay near the
// K(1 + ln(R/K)) rate of an exact running top-K.
template <int K>
struct RegTopk {
  uint64_t L[K];
  uint64_t thr;        // discard keys <= thr
  uint64_t published;  // last value sent to g
  float tlim;
  int k;
  unsigned long long* g;

  __device__ __forceinline__ void init(int kk, unsigned long long* gt) {
#pragma unroll
    for (int j = 0; j < K; ++j) L[j] = 0;
    thr = 0; published = 0; tlim = -__int_as_float(0x7f800000); k = kk; g = gt;
  }
  __device__ __forceinline__ void raise(uint64_t t) {
    if (t > thr) {
      thr = t;
      const float ts = key_score(t);
      tlim = ts - fabsf(ts) * 3.814697265625e-06f - 1e-30f;  // see LaneTopk::raise
    }
  }
  __device__ __forceinline__ uint64_t peek_shared() const {
    return g ? *reinterpret_cast<volatile unsigned long long*>(g) : 0ull;
  }
  __device__ __forceinline__ bool may_pass(float dot, float den) const { return dot >= tlim * den; }

  // Per lane (no warp sync); key 0 or key <= thr is a no-op.
  __device__ __forceinline__ void insert(uint64_t x) {
    if (x <= thr) return;
#pragma unroll
    for (int j = K - 1; j > 0; --j) {
      const bool above_prev = x > L[j - 1];
      L[j] = above_prev ? L[j - 1] : (x > L[j] ? x : L[j]);
    }
    L[0] = x > L[0] ? x : L[0];
    raise(L[K - 1]);
  }
  // Share this lane's k-th best with the other states of its query (exact lower bound).
  __device__ __forceinline__ void publish() {
    if (g && thr > published) {
      atomicMax(g, (unsigned long long)thr);
      published = thr;
    }
  }
  // Per lane: the sorted best k (zero padded) to out.
  __device__ __forceinline__ void flush(uint64_t* out) const {
    if (!out) return;
#pragma unroll
    for (int j = 0; j < K; ++j)
      if (j < k) out[j] = L[j];
  }
};

// Warp-shared top-k over a stream of keys for ONE query (all lanes feed it).
// Buffer in shared memory; CAP = 32*P >= k + 32.
template <int P>
struct WarpTopk {
  static constexpr int CAP = 32 * P;
  uint64_t thr;
  int cnt;
  uint64_t* buf;
  __device__ __forceinline__ void init(uint64_t* b) { thr = 0; cnt = 0; buf = b; }
  __device__ __forceinline__ void push(uint64_t key, int k) {
    const int lane = threadIdx.x & 31;
    unsigned m = __ballot_sync(kFull, key > thr);
    if (!m) return;
    if (cnt + __popc(m) > CAP) {
      thr = warp_compact<P>(buf, cnt, k, nullptr);
      cnt = k < cnt ? k : cnt;
      m = __ballot_sync(kFull, key > thr);
    }
    if (key > thr) buf[cnt + __popc(m & ((1u << lane) - 1u))] = key;
    cnt += __popc(m);
    __syncwarp();
  }
  __device__ __forceinline__ void finish(uint64_t* out, int k) {
    warp_compact<P>(buf, cnt, k, out);
  }
};

// ---------------------------------------------------------------- programmatic dependent launch
// Wait until the previous kernel on the stream has completed and its writes are
// visible (no-op when the kernel was not launched with PDL).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Allow the next (PDL-launched) kernel to be scheduled before this one completes.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------------------- mbarrier + bulk copy
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Waiting variant for threads with nothing else to do (epilogue warps): the suspend-time
// hint lets the hardware park the warp until the phase completes instead of re-issuing
// try_wait, so idle waiters do not steal issue slots from the MMA / TMA threads.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAITS_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000)
      : "memory");
}
// 1-D bulk copy global -> shared, completion counted on `bar` (TMA engine).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ uint4 lds128(const void* p) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(smem_u32(p)));
  return r;
}
// A plain C++ shared-memory load (not volatile asm): the compiler may batch the eight
// loads of a chunk ahead of the arithmetic; barriers (asm with "memory" clobbers) still
// order it.  The volatile asm form serialised load -> FMA -> compare chains per column
// (~100 cycles per column in the seeding pass, REMOE_TC_TRACE cycle counters).
__device__ __forceinline__ float4 lds128f(const void* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ uint4 ldg_nc128(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// CAP selection shared by host and device: CAP = 32*P >= max(64, pow2ceil(2k)), which
// keeps CAP - k >= 32 (room for a chunk after a compaction) for every k <= 256.  (CAP =
// pow2ceil(4k) made the k > 64 scans spill: the P = 16 sort network needs more registers
// than the epilogue has, and seeded thresholds leave the buffers nearly empty anyway.)
// (k <= 256 = the API maximum gives P <= 16; the kernels instantiate P in {2, 4, 8, 16})
__host__ __device__ constexpr int topk_P(int k) {
  return (2 * k <= 64) ? 2 : (2 * k <= 128) ? 4 : (2 * k <= 256) ? 8 : (2 * k <= 512) ? 16 : 32;
}

}  // namespace remoe
