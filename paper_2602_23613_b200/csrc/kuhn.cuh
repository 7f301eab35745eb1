// GPU assembly of the 3D Kuhn-cube curl-curl systems (see kuhn.cu).
#pragma once
#include <vector>

#include "common.cuh"

namespace hcamg {

// n^3 hexes x 6 Kuhn tets, lexicographic vertex numbering; muinv per tet
// (cube-major, permutation-minor); S6, M6: the 6 x 36 element matrices of the
// six tet shapes (row-major 6x6 each).  A, G as canonical CSR on the device;
// free_edges / free_nodes: full index -> free index or -1 (host).
void kuhn_assemble(int64_t n, const double* h_muinv, double beta, const double* h_S6, const double* h_M6, DCsr& A,
                   DCsr& G, std::vector<int64_t>& free_edges, std::vector<int64_t>& free_nodes, cudaStream_t s);

}  // namespace hcamg
