// Micro-benchmark of the S4 merge kernel (development tool; not part of the library).
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>
#include "../../paper_2512_18674_b200/csrc/kernels.h"

int main(int argc, char** argv) {
  int B = argc > 1 ? atoi(argv[1]) : 1;
  int nl = argc > 2 ? atoi(argv[2]) : 296;
  int k = argc > 3 ? atoi(argv[3]) : 10;
  int LE = 1728;
  std::vector<uint64_t> h((size_t)B * nl * k);
  std::mt19937_64 rng(1);
  for (size_t i = 0; i < h.size(); i += k) {
    std::vector<uint64_t> v(k);
    for (auto& x : v) x = ((rng() >> 33) | 0x80000000ull) << 32 | (0xFFFFFFFFull - (rng() % 100000));
    std::sort(v.rbegin(), v.rend());
    std::copy(v.begin(), v.end(), h.begin() + i);
  }
  uint64_t *d, *o; unsigned long long* lb; float *act, *pred, *sc; int64_t* ids;
  cudaMalloc(&d, h.size() * 8); cudaMalloc(&o, (size_t)B * k * 8); cudaMalloc(&lb, B * 8);
  cudaMalloc(&act, (size_t)100000 * LE * 4); cudaMalloc(&pred, (size_t)B * LE * 4);
  cudaMalloc(&sc, B * k * 4); cudaMalloc(&ids, B * k * 8);
  cudaMemset(act, 0, (size_t)100000 * LE * 4);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  {  // lower bound = the 300th largest key of each query (what a good shared threshold gives)
    std::vector<unsigned long long> hl(B);
    for (int b = 0; b < B; ++b) {
      std::vector<uint64_t> v(h.begin() + (size_t)b * nl * k, h.begin() + (size_t)(b + 1) * nl * k);
      std::sort(v.rbegin(), v.rend());
      hl[b] = v[std::min<size_t>(300, v.size() - 1)];
    }
    cudaMemcpy(lb, hl.data(), B * 8, cudaMemcpyHostToDevice);
  }
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  remoe::FinalizeArgs fin{act, 0, nullptr, 0, LE, 1.f, ids, sc, pred};
  for (int mode = 0; mode < 3; ++mode) {
    float best = 1e9;
    for (int rep = 0; rep < 20; ++rep) {
      cudaEventRecord(a, st);
      cudaError_t e = remoe::launch_merge(d, B, nl, (int64_t)nl * k, k, k, o, st, nullptr,
                                          mode >= 1 ? lb : nullptr, mode == 2 ? &fin : nullptr);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
      best = std::min(best, ms);
    }
    printf("B=%d lists=%d k=%d mode=%d (0 plain, 1 +lower, 2 +fused finalize): %.2f us\n", B, nl, k, mode, best * 1e3);
  }
  // empty kernel-launch baseline
  float best = 1e9;
  for (int rep = 0; rep < 20; ++rep) {
    cudaEventRecord(a, st);
    remoe::launch_norms(nullptr, 0, 8, nullptr, st);
    cudaEventRecord(b, st); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms);
  }
  printf("event pair baseline: %.2f us\n", best * 1e3);
  return 0;
}
