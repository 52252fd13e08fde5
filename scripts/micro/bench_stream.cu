// Micro-benchmark (development tool; not part of the library): the read-bandwidth ceiling
// of the scan's access pattern.  A persistent grid (one CTA per SM) streams a buffer in
// contiguous chunks with 1-D bulk copies (cp.async.bulk) into an NST-deep mbarrier ring;
// a consumer warp only waits and frees the slot.  Sweeps chunk size x stages x grid.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bs bench_stream.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(su32(bar)), "r"(ph) : "memory");
}

__global__ void __launch_bounds__(64, 1) k_stream(const uint8_t* src, int64_t bytes, int chunk, int nst, unsigned long long* sink, int tile_chunks) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)nst * chunk);
  uint64_t* empty = full + nst;
  const int64_t n_chunks = bytes / chunk;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // producer
    int it = 0;
    const int64_t per_cta = (n_chunks / ((int64_t)gridDim.x * tile_chunks)) * tile_chunks;
    for (int64_t j = 0; j < per_cta; ++j, ++it) {
      // tile_chunks == 1: chunk-interleaved across CTAs; else CTA-private tiles of tile_chunks chunks
      const int64_t c = tile_chunks == 1 ? blockIdx.x + j * gridDim.x
                                          : ((j / tile_chunks) * gridDim.x + blockIdx.x) * tile_chunks + j % tile_chunks;
      const int s = it % nst;
      wait(&empty[s], ((it / nst) & 1) ^ 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(smem + (size_t)s * chunk)), "l"(src + c * chunk), "r"(chunk), "r"(su32(&full[s]))
                   : "memory");
    }
  } else if (threadIdx.x == 32) {  // consumer
    int it = 0;
    unsigned long long acc = 0;
    const int64_t per_cta = (n_chunks / ((int64_t)gridDim.x * tile_chunks)) * tile_chunks;
    for (int64_t j = 0; j < per_cta; ++j, ++it) {
      const int s = it % nst;
      wait(&full[s], (it / nst) & 1);
      acc += smem[(size_t)s * chunk + (it & 127)];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    }
    if (acc == 0x123456789ull) *sink = acc;
  }
}

int main(int argc, char** argv) {
  const int64_t bytes = (int64_t)(argc > 1 ? atof(argv[1]) : 4.0) * (1ll << 30);
  uint8_t* buf;
  unsigned long long* sink;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&sink, 8);
  cudaMemset(buf, 1, bytes);
  uint8_t* flush;
  cudaMalloc(&flush, 256 << 20);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int chunks[] = {16384};
  const int grids[] = {1};  // CTAs per SM
  const int tcs[] = {1, 16, 4, 64};
  for (int tc : tcs)
  for (int gm : grids)
    for (int chunk : chunks)
      for (int nst = 4; nst <= 8; nst += 2) {
        const size_t sm = (size_t)nst * chunk + 2 * nst * 8;
        if (sm > (size_t)(gm == 1 ? 227 : 113) * 1024) continue;
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
          cudaMemset(flush, r, 256 << 20);
          cudaEventRecord(e0);
          k_stream<<<sms * gm, 64, sm>>>(buf, bytes, chunk, nst, sink, tc);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (ms < best) best = ms;
        }
        const int64_t moved = (bytes / chunk / ((int64_t)sms * gm * tc)) * tc * (sms * gm) * chunk;
        printf("tile %2d chunks, ctas/SM %d chunk %6d KB x %2d stages (%4zu KB in flight/SM): %7.1f GB/s\n", tc, gm,
               chunk >> 10, nst, (size_t)gm * nst * chunk >> 10, moved / (best / 1e3) / 1e9);
      }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
