// k_embed.cu -- NEXT-N1: the Eq. 11 front end, token matrices -> prompt vectors.
//
// SCS (Eq. 11) normalises every token embedding row and sums the rows of a
// prompt (V1^T X); the path scores those sums (DESIGN R2).  This kernel produces them
// from the pre-processing layer's token embeddings: for prompt p with tokens
// [off[p], off[p+1]):  a_p = sum_t x_t / |x_t|  (a zero token contributes 0).
//
// One CTA per prompt; warp w takes tokens t = off + w, off + w + 8, ...; lanes split
// D into 16-byte chunks; a token's norm is a fixed xor butterfly; each warp accumulates
// into its own fp32 row in shared memory, and the 8 rows are summed in warp order at the
// end -- the summation order depends only on the prompt, never on its batch position.
#include "common.cuh"
#include "host_util.h"
#include "kernels.h"

namespace remoe {

__global__ void __launch_bounds__(256) k_embed(const uint16_t* __restrict__ tok, const int64_t* __restrict__ off,
                                               int dim, uint16_t* __restrict__ out_bf16,
                                               float* __restrict__ out_f32) {
  extern __shared__ __align__(16) float acc[];  // [8][dim]
  const int p = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int D8 = dim >> 3;
  float* mine = acc + (size_t)warp * dim;
  for (int i = lane; i < dim; i += 32) mine[i] = 0.f;
  __syncwarp();
  const int64_t t0 = off[p], t1 = off[p + 1];
  for (int64_t t = t0 + warp; t < t1; t += 8) {
    const uint16_t* row = tok + t * dim;
    float ss = 0.f;
    for (int c = lane; c < D8; c += 32) {
      const uint4 w = __ldg(reinterpret_cast<const uint4*>(row) + c);
      const float v[8] = {bf_lo(w.x), bf_hi(w.x), bf_lo(w.y), bf_hi(w.y),
                          bf_lo(w.z), bf_hi(w.z), bf_lo(w.w), bf_hi(w.w)};
#pragma unroll
      for (int j = 0; j < 8; ++j) ss = __fmaf_rn(v[j], v[j], ss);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(kFull, ss, o);
    if (ss == 0.f) continue;  // a zero token has no direction: contributes nothing
    const float nrm = __fsqrt_rn(ss);
    for (int c = lane; c < D8; c += 32) {
      const uint4 w = __ldg(reinterpret_cast<const uint4*>(row) + c);
      const float v[8] = {bf_lo(w.x), bf_hi(w.x), bf_lo(w.y), bf_hi(w.y),
                          bf_lo(w.z), bf_hi(w.z), bf_lo(w.w), bf_hi(w.w)};
#pragma unroll
      for (int j = 0; j < 8; ++j) mine[c * 8 + j] += __fdiv_rn(v[j], nrm);
    }
  }
  __syncthreads();
  for (int d = threadIdx.x; d < dim; d += blockDim.x) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += acc[(size_t)w * dim + d];
    if (out_f32) out_f32[(size_t)p * dim + d] = s;
    if (out_bf16) {  // round to nearest even
      const uint32_t u = __float_as_uint(s);
      out_bf16[(size_t)p * dim + d] = (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
    }
  }
}

cudaError_t launch_embed(const uint16_t* tok, const int64_t* off, int n_prompts, int dim, uint16_t* out_bf16,
                         float* out_f32, cudaStream_t st) {
  if (n_prompts <= 0) return cudaSuccess;
  const size_t smem = (size_t)8 * dim * sizeof(float);
  cudaError_t e = set_smem_attrs_once((const void*)k_embed, 232448);
  if (e != cudaSuccess) return e;
  k_embed<<<n_prompts, 256, smem, st>>>(tok, off, dim, out_bf16, out_f32);
  return cudaGetLastError();
}

}  // namespace remoe
