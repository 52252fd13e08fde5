// tree.h -- NEXT-N2: the multi-fork clustering tree and Algorithm 1
// (P:391-415), internal interface of libremoe (see k_tree.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "remoe.h"

namespace remoe {

constexpr int kTreeCMax = 16;      // branching limit (register accumulators in k_assign)
constexpr int kTreeMaxDepth = 128;  // path storage in the search kernel (the synthetic stores reach ~70 levels: noise outliers peel off one at a time)
constexpr int kTreeCandCap = 2048; // candidate keys per query in shared memory

// Flat tree, breadth-first node numbering (root 0).  Node i owns perm[begin[i], end[i]);
// its children are child0[i] .. child0[i] + nchild[i] - 1; medoid[i] is the local row
// of its centroid (-1 for the root).  Device arrays + host copies.
struct Tree {
  int n_nodes = 0, n_leaves = 0, depth = 0, max_leaf = 0;
  int beta = 0, branching = 0;
  double build_ms = 0.0;
  int64_t* perm = nullptr;   // device [n]
  int64_t* begin = nullptr;  // device [n_nodes]
  int64_t* end = nullptr;
  int32_t* child0 = nullptr;
  int32_t* nchild = nullptr;
  int64_t* medoid = nullptr;
  size_t bytes = 0;
  std::vector<int64_t> h_begin, h_end, h_medoid;
  std::vector<int32_t> h_parent, h_child0, h_nchild;
};

// Build over the n rows of x (bf16 [n][dim]) on `st` (synchronous: returns when done).
remoe_status_t tree_build(const uint16_t* x, int64_t n, int dim, int beta, int branching, int max_iter,
                          uint64_t seed, cudaStream_t st, Tree* out, std::string* err);
void tree_free(Tree* t);

// Algorithm 1 for B queries: per query the sorted top-k keys (zero padded) to
// top[b * k ...], optionally the leaf reached by the descent and the number of Eq. 11
// evaluations.  xnorm/qnorm are the fp32 norms the BF path uses.
cudaError_t launch_tree_search(const Tree& t, const uint16_t* x, const float* xnorm, int dim, const uint16_t* q,
                               const float* qnorm, int B, int k, float sigma, int64_t gid_offset, uint64_t* top,
                               int32_t* leaf, int32_t* n_eval, cudaStream_t st);

}  // namespace remoe
