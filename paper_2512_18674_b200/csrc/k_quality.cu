// k_quality.cu -- NEXT-N4: prediction quality.  Jensen-Shannon divergence (log base 2)
// between predicted and reference activation matrices, averaged over the L layers --
// the metric of the paper's prediction-accuracy study (fig
// predict_method_compare).  JS(p,q) = KL(p||m)/2 + KL(q||m)/2, m = (p+q)/2, 0 log 0 = 0.
#include "common.cuh"
#include "host_util.h"
#include "kernels.h"

namespace remoe {

// One CTA per matrix pair; warp w takes layers w, w+8, ...; the L row values are summed
// in layer order by one thread (deterministic).
__global__ void __launch_bounds__(256) k_js(const float* __restrict__ P, const float* __restrict__ Q,
                                            int64_t q_stride, int L, int E, float* __restrict__ out) {
  extern __shared__ float rowjs[];  // [L]
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* pb = P + (int64_t)b * L * E;
  const float* qb = Q + (int64_t)b * q_stride;
  for (int l = warp; l < L; l += 8) {
    float s = 0.f;
    for (int e = lane; e < E; e += 32) {
      const float p = pb[l * E + e], q = qb[l * E + e], m = 0.5f * (p + q);
      if (p > 0.f) s += 0.5f * p * log2f(p / m);
      if (q > 0.f) s += 0.5f * q * log2f(q / m);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    if (lane == 0) rowjs[l] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int l = 0; l < L; ++l) t += rowjs[l];
    out[b] = t / (float)L;
  }
}

cudaError_t launch_js(const float* P, const float* Q, int64_t q_stride, int B, int L, int E, float* out,
                      cudaStream_t st) {
  if (B <= 0) return cudaSuccess;
  // remoe_js_divergence admits L * 4 <= 200 KB of per-layer values: opt in to that much
  cudaError_t e = set_smem_attrs_once((const void*)k_js, 200 * 1024);
  if (e != cudaSuccess) return e;
  k_js<<<B, 256, (size_t)L * sizeof(float), st>>>(P, Q, q_stride, L, E, out);
  return cudaGetLastError();
}

}  // namespace remoe
