// Micro-benchmark (development tool; not part of the library): issue rate of
// tcgen05.mma.cta_group::1.kind::f16 (bf16 x bf16 -> fp32) by UMMA shape, one CTA per SM,
// operands resident in shared memory (K-major, SWIZZLE_128B), chains of MMAs into one
// TMEM accumulator, committed to an mbarrier.  Reports cycles per MMA and the store bytes
// (N rows x 32 B per K=16 step) the scan could consume per cycle at that rate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2512_18674_b200/csrc -o /tmp/bu bench_umma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "tcgen05.cuh"

using namespace remoe;

__device__ __forceinline__ bool mbar_try_wait_once(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}

__global__ void __launch_bounds__(128, 1) k_umma(int M, int N, int n_mma, int per_commit, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;                 // 128 rows x 128 B (16 KB)
  uint8_t* sB = smem + 16384;         // 256 rows x 128 B (32 KB)
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + 32768);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < (16384 + 32768) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    uint32_t ph = 0;
    // warm-up
    for (int i = 0; i < 64; ++i) umma_bf16(tmem, umma_desc(a0 + (i & 3) * 32), umma_desc(b0 + (i & 3) * 32), idesc, i != 0);
    umma_commit(bar);
    mbar_wait(bar, ph); ph ^= 1u;
    const long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      umma_bf16(tmem, umma_desc(a0 + (i & 3) * 32), umma_desc(b0 + (i & 3) * 32), idesc, 1);
      if ((i + 1) % per_commit == 0) {  // like the scan: a commit per K-block
        umma_commit(bar);
        mbar_wait(bar, ph); ph ^= 1u;
      }
    }
    umma_commit(bar);
    mbar_wait(bar, ph);
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// Same, but the commit does not wait (fire-and-forget per K-block, as the scan's slot
// release): only the final commit is waited on.
__global__ void __launch_bounds__(128, 1) k_umma_async(int M, int N, int n_mma, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + 16384;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + 32768);
  uint64_t* bar2 = bar + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < (16384 + 32768) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(bar, 1); mbar_init(bar2, 1 << 20); fence_mbar_init(); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    for (int i = 0; i < 64; ++i) umma_bf16(tmem, umma_desc(a0 + (i & 3) * 32), umma_desc(b0 + (i & 3) * 32), idesc, i != 0);
    umma_commit(bar);
    mbar_wait(bar, 0);
    const long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      umma_bf16(tmem, umma_desc(a0 + (i & 3) * 32), umma_desc(b0 + (i & 3) * 32), idesc, 1);
      if ((i & 3) == 3) umma_commit(bar2);  // arrivals never complete the phase: no waiter
    }
    umma_commit(bar);
    mbar_wait(bar, 1);
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// The scan's MMA-issuer loop shape: per K-block [wait on an already-completed mbarrier]
// [tcgen05.fence::after_thread_sync] 4 MMAs, commit to a slot barrier nobody waits on.
__global__ void __launch_bounds__(128, 1) k_umma_loop(int M, int N, int n_kb, int variant, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + 16384;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + 32768);
  uint64_t* bar2 = bar + 2;
  uint64_t* ready = bar + 3;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < (16384 + 32768) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1); mbar_init(bar2, 1 << 20); mbar_init(ready, 1);
    fence_mbar_init();
    mbar_arrive(ready);  // phase 0 complete: waits on parity 0 return at once
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    const long long t0 = clock64();
    for (int j = 0; j < n_kb; ++j) {
      if (variant & 1) mbar_wait(ready, 0);
      if (variant & 2) tc_fence_after();
      const uint32_t acc = (variant & 4) ? tmem + (uint32_t)((j >> 4) & 1) * 256 : tmem;  // bit 4: alternate accumulators per 16 K-blocks
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        umma_bf16(acc, umma_desc(a0 + kk * 32), umma_desc(b0 + kk * 32), idesc, (j | kk) != 0);
      umma_commit(bar2);
    }
    umma_commit(bar);
    mbar_wait(bar, 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// Operands that move like the scan's: A from a [nkb][M rows][128 B] slab (a new 8 KB block
// every K-block), B from an NST-deep ring of 16 KB stages; nothing is loaded (timing of the
// MMA operand fetch from fresh shared-memory addresses).
__global__ void __launch_bounds__(128, 1) k_umma_fresh(int M, int N, int n_kb, int nkb, int nst, int a_fixed,
                                                       unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;                              // nkb * M * 128 B
  uint8_t* sB = smem + (size_t)nkb * M * 128;      // nst * 16 KB (N = 128 rows x 128 B)
  uint64_t* bar = reinterpret_cast<uint64_t*>(sB + (size_t)nst * 16384);
  uint64_t* bar2 = bar + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int total = nkb * M * 128 + nst * 16384;
  for (int i = threadIdx.x; i < total / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(bar, 1); mbar_init(bar2, 1 << 20); fence_mbar_init(); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    const long long t0 = clock64();
    int s = 0;
    for (int j = 0; j < n_kb; ++j) {
      const int kb = j % nkb;
      const uint32_t abase = a0 + (a_fixed ? 0u : (uint32_t)(kb * M * 128));
      const uint32_t bbase = b0 + (uint32_t)(s * 16384);
      if (++s == nst) s = 0;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        umma_bf16(tmem, umma_desc(abase + kk * 32), umma_desc(bbase + kk * 32), idesc, (j | kk) != 0);
      umma_commit(bar2);
    }
    umma_commit(bar);
    mbar_wait(bar, 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// The scan's situation: thread 0 issues MMAs (async commits per 4) while the other warps of the
// CTA wait on an mbarrier that completes only at the end -- polling with try_wait (mode 0),
// try_wait + nanosleep back-off (mode 1), or parked on a named barrier (mode 2).
__global__ void __launch_bounds__(352, 1) k_umma_poll(int M, int N, int n_mma, int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + 16384;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + 32768);
  uint64_t* bar2 = bar + 2;
  uint64_t* gate = bar + 3;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < (16384 + 32768) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(bar, 1); mbar_init(bar2, 1 << 20); mbar_init(gate, 1); fence_mbar_init(); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    const long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      umma_bf16(tmem, umma_desc(a0 + (i & 3) * 32), umma_desc(b0 + (i & 3) * 32), idesc, 1);
      if ((i & 3) == 3) umma_commit(bar2);
    }
    umma_commit(bar);
    mbar_wait(bar, 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
    mbar_arrive(gate);
    if (mode == 2) asm volatile("bar.arrive 3, 352;" ::: "memory");
  } else if (threadIdx.x >= 64) {  // warps 2..10 wait, as the scan's epilogue / seeding warps do
    if (mode == 0) mbar_wait(gate, 0);
    else if (mode == 1) { while (!mbar_try_wait_once(gate, 0)) __nanosleep(200); }
    else asm volatile("bar.sync 3, 352;" ::: "memory");
  } else if (threadIdx.x >= 32 && threadIdx.x < 33 && mode != 2) {
    mbar_wait(gate, 0);  // warp 1 lane 0 (the scan's producer lane) polls too
  }
  if (mode == 2 && threadIdx.x > 0 && threadIdx.x < 64) asm volatile("bar.sync 3, 352;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int smem = 16384 + 32768 + 64;
  cudaFuncSetAttribute(k_umma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_umma_async, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int shapes[][2] = {{64, 64}, {64, 128}, {64, 256}, {128, 64}, {128, 128}, {128, 256}};
  const int n = 8192;
  printf("SMs %d, clock attr %d kHz; %d MMAs per CTA, all SMs busy\n", sms, clk, n);
  for (auto& sh : shapes) {
    const int M = sh[0], N = sh[1];
    for (int pc : {4, 1 << 30}) {
      unsigned long long h = 0;
      k_umma<<<sms, 128, smem>>>(M, N, n, pc, d);
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      const double cyc = (double)h / n;
      printf("M=%3d N=%3d %-22s: %7.1f cycles/MMA  %7.1f MAC/clk  %6.1f store B/clk (N*32/cyc)\n", M, N,
             pc == 4 ? "commit+wait per 4" : "one commit at end", cyc, (double)M * N * 16 / cyc, N * 32.0 / cyc);
    }
    unsigned long long h = 0;
    k_umma_async<<<sms, 128, smem>>>(M, N, n, d);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double cyc = (double)h / n;
    printf("M=%3d N=%3d %-22s: %7.1f cycles/MMA  %7.1f MAC/clk  %6.1f store B/clk\n", M, N, "async commit per 4", cyc,
           (double)M * N * 16 / cyc, N * 32.0 / cyc);
  }
  cudaFuncSetAttribute(k_umma_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (auto& sh : shapes) {
    const int M = sh[0], N = sh[1];
    for (int v = 0; v < 8; ++v) {
      unsigned long long h = 0;
      k_umma_loop<<<sms, 128, smem>>>(M, N, n / 4, v, d);
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      const double cyc = (double)h / n;
      printf("loop M=%3d N=%3d wait=%d fence=%d altacc=%d: %7.1f cycles/MMA %6.1f store B/clk\n", M, N, v & 1, (v >> 1) & 1,
             (v >> 2) & 1, cyc, N * 32.0 / cyc);
    }
  }
  cudaFuncSetAttribute(k_umma_poll, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 3; ++mode) {
    unsigned long long h = 0;
    k_umma_poll<<<sms, 352, smem>>>(64, 128, n, mode, d);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("poll M= 64 N=128 with 10 waiting warps, %s: %7.1f cycles/MMA\n",
           mode == 0 ? "try_wait spin      " : mode == 1 ? "test_wait+nanosleep" : "named barrier      ", (double)h / n);
  }
  cudaFuncSetAttribute(k_umma_fresh, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  for (int M : {64, 128}) {
    for (int nst : {1, 2, 6}) {
      for (int af : {0, 1}) {
        const int nkb = 16;
        const int sm = nkb * M * 128 + nst * 16384 + 64;
        if (sm > 227 * 1024) continue;
        unsigned long long h = 0;
        k_umma_fresh<<<sms, 128, sm>>>(M, 128, n / 4, nkb, nst, af, d);
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        const double cyc = (double)h / n;
        printf("fresh M=%3d N=128 stages=%d A %s: %7.1f cycles/MMA %6.1f store B/clk\n", M, nst,
               af ? "fixed      " : "per K-block", cyc, 128 * 32.0 / cyc);
      }
    }
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
