// FP64 level-3 kernels of the dense setup work (sm_100a, DMMA m8n8k4 tensor-core
// instructions): GEMM (also batched over pointer arrays and restricted to the
// lower triangle for SYRK), triangular solves and the triangular inverse.
// Column-major with cuBLAS's argument conventions, so each call site in
// dense.cu / giant.cu reads like the BLAS call it replaces.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace hcamg {
namespace dblas {

enum Op : int { N = 0, T = 1 };
enum Side : int { Left = 0, Right = 1 };

// C = alpha op(A) op(B) + beta C   (m x n, inner k).  lower: only C's entries
// with row >= col are computed / written (SYRK: op(B) = op(A)^T).
void gemm(Op ta, Op tb, int64_t m, int64_t n, int64_t k, double alpha, const double* A, int64_t lda, const double* B,
          int64_t ldb, double beta, double* C, int64_t ldc, cudaStream_t s, bool lower = false);
// the same for `batch` independent products given by device pointer arrays
void gemm_batched(Op ta, Op tb, int64_t m, int64_t n, int64_t k, double alpha, const double* const* A, int64_t lda,
                  const double* const* B, int64_t ldb, double beta, double* const* C, int64_t ldc, int64_t batch,
                  cudaStream_t s);
// C (n x n, lower triangle) = alpha A A^T + beta C  (A n x k), cublasDsyrk(LOWER, N)
void syrk_ln(int64_t n, int64_t k, double alpha, const double* A, int64_t lda, double beta, double* C, int64_t ldc,
             cudaStream_t s);

// lower(C) = Y^T Y for a lower-triangular n x n Y (the inner sum of entry
// (i, j), i >= j, runs over k >= i only; n^3/3 flops)
void gemm_tri_lower_tn(int64_t n, const double* Y, int64_t ldy, double* C, int64_t ldc, cudaStream_t s);

// Triangular solves with a lower-triangular, non-unit L (cublasDtrsm with
// FILL_MODE_LOWER, DIAG_NON_UNIT, alpha = 1):
//   Left:  op(L) X = B  (B m x n, L m x m);   Right: X op(L) = B  (L n x n).
// Recursive: halves of L down to 64 x 64 diagonal blocks applied as their
// explicit inverses; everything else is GEMM.
void trsm(Side side, Op op, int64_t m, int64_t n, const double* L, int64_t ldl, double* B, int64_t ldb,
          cudaStream_t s);
// Batched right-side solve X L^T = B for pairs (L[i], B[i]) of nb x nb tiles
// (m rows of B), host pointer lists: the distinct L are inverted once, then one
// batched GEMM.
void trsm_rlt_batched(int64_t m, int64_t nb, const std::vector<const double*>& L, int64_t ldl,
                      const std::vector<double*>& B, int64_t ldb, cudaStream_t s);
// Li = L^{-1} for a lower-triangular n x n L (Li lower, ld ldi; the strict upper part is zeroed).
void trtri_lower(int64_t n, const double* L, int64_t ldl, double* Li, int64_t ldi, cudaStream_t s);
// While a scope is alive (per thread), the inverse of a full 64 x 64 diagonal
// leaf is computed once per leaf address: the recursive triangular solves of a
// Cholesky factorisation revisit the same (final) leaves of L at every level of
// the recursion, and the triangular inverse after it visits them once more
// (config 2's coarsest operator: ~1,900 single-CTA leaf inversions of 77 us
// become 410).  Only for factors that are not modified inside the scope.
struct LeafCacheScope {
  LeafCacheScope();
  ~LeafCacheScope();
  LeafCacheScope(const LeafCacheScope&) = delete;
  void* prev;
  static bool active();
};
// Batched inverses of `batch` nb x nb lower-triangular tiles.
void copy_block(int64_t rows, int64_t cols, const double* src, int64_t lds, double* dst, int64_t ldd, cudaStream_t s);
// B_b := B_b Li^T for every tile of the batch (host pointer list), Li = L^{-1} given (nb x nb, ld nb)
// C = X Li^T with Li lower triangular (n x n, given explicitly): a product whose inner range per tile is cut to Li's nonzeros
void gemm_rinv_t(int64_t m, int64_t n, const double* X, int64_t ldx, const double* Li, int64_t ldi, double* C,
                 int64_t ldc, cudaStream_t s);
void apply_rinv_t_batched(int64_t m, int64_t nb, const double* Li, const std::vector<double*>& hb, int64_t ldb,
                          cudaStream_t s);
// inverses of many n x n lower-triangular matrices (host pointer lists), level-synchronous
void trtri_lower_many(int64_t n, const std::vector<const double*>& L, int64_t ldl, const std::vector<double*>& Li,
                      int64_t ldi, cudaStream_t s);
void trtri_lower_batched(int64_t nb, const double* const* L, int64_t ldl, double* const* Li, int64_t ldi, int64_t batch,
                         cudaStream_t s);

}  // namespace dblas
}  // namespace hcamg
