// Sparse approximate ideal interpolation and coarse gradient on the GPU.
#pragma once

#include "giant.cuh"
#include "split.cuh"

namespace hcamg {

struct InterpResult {
  DCsr R;    // n_c x n, rows +-1/sqrt(2)
  DCsr P;    // n x n_c   (canonical CSR)
  DCsr Pt;   // n_c x n   (transpose, for restriction and the Galerkin product)
  DCsr Gc;   // next-level gradient, sign-normalised (multilevel.py:71-75)
  std::vector<int64_t> gc_cols;  // nodal columns of R G kept (coarse_node_cols)
  int64_t ncomp = 0, max_comp = 0, ncomp_large = 0;
  // dense-interpolation regime: one component above kGiantMin is kept as the
  // dense block Z (P = P - S_G Z with P above holding only the sparse part)
  HybridP hp;
};

// transfer.py:77-122 (+ coarse_gradient 55-74).  mode: 0 = refinement, 1 = algebraic.
// Throws Error(ENOTSPD_, ..., pivot) on a breakdown in a component solve.
void build_interp(const DCsr& A, const DCsr& G, const SplitResult& sp, int mode, InterpResult& out, cudaStream_t s);

// Connected components of the graph of M (square, symmetric pattern):
// label[v] = component index, components numbered by their smallest vertex.
int64_t connected_components(const DCsr& M, DBuf<int32_t>& label, cudaStream_t s);

}  // namespace hcamg
