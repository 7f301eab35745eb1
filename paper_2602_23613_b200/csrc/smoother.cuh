// OSS-l1 smoother setup (see smoother.cu).
#pragma once
#include "level.cuh"

namespace hcamg {

// Patches, patch inverses, wavefront schedule and gather lists for one level.
void build_smoother(const DCsr& A, const DCsr& G, Smoother& sm, cudaStream_t s);

// l1 diagonal d_i = sum_j |a_ij| (sequential row sum).
void build_l1(const DCsr& A, DBuf<double>& l1, cudaStream_t s);

}  // namespace hcamg
