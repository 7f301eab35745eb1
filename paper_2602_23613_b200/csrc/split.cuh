// Coarse/fine splitting on the GPU (see split.cu).
#pragma once
#include <vector>

#include "sparse.cuh"

namespace hcamg {

struct SplitResult {
  int64_t n = 0;
  // 7 int64 per pair: dof1, dof2, sign1, sign2, tail(i), mid(k), head(j)
  std::vector<int64_t> pairs;
  std::vector<int64_t> interior;         // ascending unpaired DoFs
  std::vector<int64_t> coarse_nodes;     // algebraic route: c_G (sorted)
  std::vector<int64_t> pair_mesh_edges;  // refinement route
  int64_t n_triples = 0;                 // diagnostic: statically valid (i,j,k) candidates
  int64_t n_pairs() const { return (int64_t)pairs.size() / 7; }
};

// Gt = [G | -delta e_r for single-entry rows]; returns #appended columns (B).
int64_t augment_gradient(const DCsr& G, DCsr& Gt, cudaStream_t s);

// Neighbour (off-diagonal) and strong patterns of the nodal dual.
void nodal_graph(const DCsr& An, double theta, DCsr& nbr, DCsr& strong, cudaStream_t s);

// Compact indices r with flag[r] != 0 (ascending); returns the count.
int64_t compact_flags(const int64_t* flag, int64_t n, DBuf<int64_t>& out, cudaStream_t s);

// Greedy C/F of the nodal dual with B prescribed coarse (state: 1 = C, 2 = F).
void nodal_cf(const DCsr& An, const DBuf<int64_t>& bcols, double theta, DCsr& nbr,
              DBuf<int8_t>& state, cudaStream_t s);

void algebraic_splitting(const DCsr& A, const DCsr& G, double theta, SplitResult& out, cudaStream_t s);

void refinement_splitting(const int64_t* h_cedges, int64_t nec, const int64_t* h_fedges, int64_t nef,
                          const int64_t* h_children, const int64_t* h_e2d, int64_t n, SplitResult& out,
                          cudaStream_t s);

}  // namespace hcamg
