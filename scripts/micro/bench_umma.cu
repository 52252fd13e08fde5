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
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
