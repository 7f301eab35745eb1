// Dense SPD kernels: batched small Cholesky solves (harmonic-extension
// components, patch blocks) and a blocked right-looking Cholesky for large
// components / the coarsest operator.  Breakdown follows the reference's
// dense_cholesky (sparse.py:188-209): pivot floor 1e-13 * max|diag|; if a
// pivot is <= 0 the first pivot under the floor is reported (the slow column
// loop's answer), otherwise the smallest pivot if it is under the floor.
#pragma once

#include <vector>

#include "common.cuh"

namespace hcamg {

constexpr double kPivotRtol = 1e-13;  // sparse.py:30

// One problem of a batch: column-major k x k SPD matrix at a_off, k x nrhs
// right-hand side at b_off (solved in place), pivots written at piv_off.
struct DenseJob {
  int64_t a_off, b_off, piv_off;
  int32_t k, nrhs;
};

// Batched small solves (k <= 32): factor + two triangular solves per job.
// status[job] = -1 on success, else the failing pivot index.
void batched_small_spd_solve(const DenseJob* d_jobs, int64_t njobs, double* A, double* B, double* piv,
                             int64_t* status, cudaStream_t s);

// Batched small inverses (k <= 32): B_job := A_job^{-1} (k x k), via Cholesky.
void batched_small_spd_inverse(const DenseJob* d_jobs, int64_t njobs, double* A, double* B, double* piv,
                               int64_t* status, cudaStream_t s);

// Large SPD factor in place (column-major, lower, leading dim ld).  Returns
// -1 on success or the failing pivot index (reference semantics).
int64_t dense_cholesky(double* A, int64_t k, int64_t ld, cudaStream_t s);

// Factor in place and write the pivots; returns the index of the first
// non-positive / non-finite pivot, or k.  No verdict.  One host sync at the end.
int64_t dense_cholesky_raw(double* A, int64_t k, int64_t ld, double* piv, cudaStream_t s);
// The same without any host sync: *bad (device, -1 initially) receives base +
// the first failing pivot; later calls sharing `bad` become no-ops.
void dense_cholesky_async(double* A, int64_t k, int64_t ld, double* piv, long long* bad, int64_t base,
                          cudaStream_t s);
// The same, and Li (k x k, ld ldi) receives L^{-1} (lower triangular, zeros above): the panel
// solves of the recursion become products with the inverse, so there are no latency-bound
// triangular leaves, and a caller that needs L^{-1} anyway (block-column panel solves) has it.
void dense_cholesky_inv_async(double* A, int64_t k, int64_t ld, double* Li, int64_t ldi, double* piv, long long* bad,
                              int64_t base, cudaStream_t s);
// Reference breakdown verdict from the pivots (-1: fine).
int64_t pivot_verdict(const std::vector<double>& hp, int64_t k, int64_t j0, double scale);

// B := A^{-1} B using the factor produced by dense_cholesky.
// A^{-1} (exactly symmetric, n x n into Ainv) from the lower Cholesky factor in Lbuf (ld n;
// overwritten).
void dense_spd_inverse(double* Lbuf, int64_t n, double* Ainv, cudaStream_t s);
void dense_cholesky_solve(const double* L, int64_t k, int64_t ld, double* B, int64_t nrhs, int64_t ldb,
                          cudaStream_t s);

}  // namespace hcamg
