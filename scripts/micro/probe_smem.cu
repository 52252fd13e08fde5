#include <cstdio>
#include <cstdint>
__global__ void k(unsigned* out) {
  extern __shared__ uint8_t s[];
  if (threadIdx.x == 0) { *out = (unsigned)__cvta_generic_to_shared(s); }
}
int main() {
  unsigned* d; unsigned h = 7;
  cudaMalloc(&d, 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  k<<<1, 32, 232448>>>(d);
  cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
  printf("dyn smem base %u (mod 1024 = %u) err %s\n", h, h & 1023, cudaGetErrorString(cudaGetLastError()));
}
