// Sparse primitives for the setup phase.  Every product reproduces scipy's
// csr_matmat arithmetic exactly (sequential sum over the inner index in
// ascending order, starting at +0.0, separate multiply and add roundings — no
// FMA), so integer decisions taken on the results (patterns, C/F split,
// matching) are bit-for-bit those of the reference.
#pragma once
#include "common.cuh"

namespace hcamg {

// Exclusive prefix sum of n int64 counts into out[0..n] (out[n] = total).
// Returns the total (synchronises the stream).
int64_t exclusive_scan(const int64_t* counts, int64_t* out, int64_t n, cudaStream_t s);

// Canonical transpose: rows of At list source rows in ascending order.
void csr_transpose(const DCsr& A, DCsr& At, cudaStream_t s);

// C = A * B in scipy's order; structural zeros kept (dropped by the callers'
// canonicalisation, which never changes values).  Output columns sorted.
void spgemm(const DCsr& A, const DCsr& B, DCsr& C, cudaStream_t s);
// Every entry stored and in canonical order (val[i * ncols + j] = A[i, j]): the
// dense-regime coarse operator kept as CSR.
bool csr_is_dense_canonical(const DCsr& A, cudaStream_t s);

// S = canon(0.5 (M + M^T)) for square, sorted M (sparse.py:122, splitting.py:133).
void symmetrize(const DCsr& M, DCsr& S, cudaStream_t s);

// Drop stored exact zeros (csr() eliminate_zeros, sparse.py:64).
void drop_zeros(const DCsr& M, DCsr& out, cudaStream_t s);

// out = M[rows, :] with columns remapped by colmap (colmap[j] < 0 drops column
// j); colmap == nullptr keeps all columns.  ncols_out is the new column count.
// colmap must be monotone on kept columns so sortedness is preserved.
void csr_extract(const DCsr& M, const int32_t* rows, int64_t nrows_out, const int32_t* colmap,
                 int64_t ncols_out, DCsr& out, cudaStream_t s);

// Deep copy.
void csr_copy(const DCsr& M, DCsr& out, cudaStream_t s);

// Upload host CSR (int64 indptr, int32 indices).
void csr_upload(const int64_t* indptr, const int32_t* indices, const double* data, int64_t nrows,
                int64_t ncols, DCsr& out, cudaStream_t s);

// y = A x (plain, one value per row; used by setup checks and utilities).
void spmv(const DCsr& A, const double* x, double* y, cudaStream_t s);

// max |a_ij| and max |a_ij - a_ji| (exact symmetric check helper).
double max_abs(const DCsr& A, cudaStream_t s);

}  // namespace hcamg
