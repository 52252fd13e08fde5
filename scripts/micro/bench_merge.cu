// Micro-benchmark (development tool): k_merge (S4 + fused S6/S7) on synthetic per-CTA lists,
// as the scan leaves them: B queries x L lists x k sorted keys, lower bound = a real key near
// the final k-th (seeded/shared threshold) or 0; with and without the finalize (LE columns).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../include
//        -I../../paper_2512_18674_b200/csrc -o /tmp/bm bench_merge.cu ../../build/k_post.o
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include "kernels.h"

static uint64_t mkkey(float s, uint32_t gid) {
  uint32_t u; memcpy(&u, &s, 4);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((uint64_t)u << 32) | (0xFFFFFFFFu - gid);
}

int main(int argc, char** argv) {
  const int B = argc > 1 ? atoi(argv[1]) : 16, L = argc > 2 ? atoi(argv[2]) : 148, k = argc > 3 ? atoi(argv[3]) : 10;
  const int LE = argc > 4 ? atoi(argv[4]) : 1728;
  const int N = 100000;
  std::vector<uint64_t> h((size_t)B * L * k);
  std::vector<uint64_t> lb(B);
  srand(1);
  for (int b = 0; b < B; ++b) {
    std::vector<uint64_t> all;
    for (int l = 0; l < L; ++l) {
      std::vector<uint64_t> v;
      for (int i = 0; i < k; ++i) v.push_back(mkkey((float)rand() / RAND_MAX * 0.3f, (uint32_t)(l * 1000 + i)));
      std::sort(v.rbegin(), v.rend());
      for (int i = 0; i < k; ++i) { h[((size_t)b * L + l) * k + i] = v[i]; all.push_back(v[i]); }
    }
    std::sort(all.rbegin(), all.rend());
    lb[b] = all[std::min((int)all.size() - 1, 3 * k)];  // a real key a little below the k-th
  }
  uint64_t *d_in, *d_out; unsigned long long* d_lb; float *d_act, *d_pred, *d_sc; int64_t* d_ids;
  cudaMalloc(&d_in, h.size() * 8); cudaMemcpy(d_in, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&d_out, (size_t)B * k * 8); cudaMalloc(&d_lb, B * 8);
  cudaMalloc(&d_act, (size_t)N * LE * 4); cudaMemset(d_act, 0, (size_t)N * LE * 4);
  cudaMalloc(&d_pred, (size_t)B * LE * 4); cudaMalloc(&d_sc, (size_t)B * k * 4); cudaMalloc(&d_ids, (size_t)B * k * 8);
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  unsigned* d_split; cudaMalloc(&d_split, B * 4); cudaMemset(d_split, 0, B * 4);
  for (int variant = 0; variant < 8; ++variant) {
    const bool use_lb = variant & 1, use_fin = variant & 2, use_split = variant & 4;
    if (use_split && !use_fin) continue;
    remoe::FinalizeArgs f{d_act, 0, N, 0, LE, 1.f, d_ids, d_sc, d_pred};
    float best = 1e9;
    for (int rep = 0; rep < 50; ++rep) {
      if (use_lb) cudaMemcpyAsync(d_lb, lb.data(), B * 8, cudaMemcpyHostToDevice, st);
      cudaEventRecord(e0, st);
      remoe::launch_merge(d_in, B, L, (int64_t)L * k, k, k, d_out, st, nullptr, use_lb ? d_lb : nullptr,
                          use_fin ? &f : nullptr, k, nullptr, use_lb, nullptr, use_split ? d_split : nullptr);
      cudaEventRecord(e1, st);
      cudaStreamSynchronize(st);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      best = std::min(best, ms);
    }
    printf("B=%d L=%d k=%d LE=%d lower=%d finalize=%d split=%d: best %.2f us (%s)\n", B, L, k, LE, use_lb, use_fin, use_split, best * 1e3,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
