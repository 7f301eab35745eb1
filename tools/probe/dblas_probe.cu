// Correctness + speed of the own FP64 level-3 kernels (csrc/dblas.cu) against
// cuBLAS.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I../../paper_2602_23613_b200/csrc dblas_probe.cu ../../paper_2602_23613_b200/csrc/dblas.cu
//   ../../paper_2602_23613_b200/csrc/options.cu -lcublas -o dblas_probe
#include <cublas_v2.h>

#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "common.cuh"
#include "dblas.cuh"

using namespace hcamg;

static double maxdiff(const std::vector<double>& a, const std::vector<double>& b) {
  double m = 0, s = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    m = std::max(m, std::fabs(a[i] - b[i]));
    s = std::max(s, std::fabs(b[i]));
  }
  return m / std::max(s, 1e-300);
}

int main() {
  cudaStream_t s;
  cudaStreamCreate(&s);
  cublasHandle_t h;
  cublasCreate(&h);
  cublasSetStream(h, s);
  std::mt19937_64 rng(1);
  std::uniform_real_distribution<double> U(-1, 1);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // GEMM variants vs cuBLAS
  for (int ta = 0; ta < 2; ++ta)
    for (int tb = 0; tb < 2; ++tb) {
      const int64_t m = 1000, n = 777, k = 513;
      const int64_t lda = ta ? k + 3 : m + 5, ldb = tb ? n + 1 : k + 2, ldc = m + 7;
      std::vector<double> hA(lda * (ta ? m : k)), hB(ldb * (tb ? k : n)), hC(ldc * n);
      for (auto& v : hA) v = U(rng);
      for (auto& v : hB) v = U(rng);
      for (auto& v : hC) v = U(rng);
      DBuf<double> A, B, C1, C2;
      A.upload(hA.data(), hA.size(), s);
      B.upload(hB.data(), hB.size(), s);
      C1.upload(hC.data(), hC.size(), s);
      C2.upload(hC.data(), hC.size(), s);
      const double al = 1.3, be = -0.7;
      dblas::gemm((dblas::Op)ta, (dblas::Op)tb, m, n, k, al, A.p, lda, B.p, ldb, be, C1.p, ldc, s);
      cublasDgemm(h, ta ? CUBLAS_OP_T : CUBLAS_OP_N, tb ? CUBLAS_OP_T : CUBLAS_OP_N, m, n, k, &al, A.p, lda, B.p, ldb,
                  &be, C2.p, ldc);
      printf("gemm %c%c rel diff %.3e\n", ta ? 'T' : 'N', tb ? 'T' : 'N', maxdiff(C1.download(), C2.download()));
    }
  // speed: 8192^3 NN and NT
  {
    const int64_t n = 8192;
    DBuf<double> A(n * n, s), B(n * n, s), C(n * n, s);
    std::vector<double> hA(n * n);
    for (auto& v : hA) v = U(rng);
    HC_CUDA(cudaMemcpy(A.p, hA.data(), 8 * n * n, cudaMemcpyHostToDevice));
    HC_CUDA(cudaMemcpy(B.p, hA.data(), 8 * n * n, cudaMemcpyHostToDevice));
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0, s);
      dblas::gemm(dblas::N, dblas::T, n, n, n, 1.0, A.p, n, B.p, n, 0.0, C.p, n, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double one = 1.0, zero = 0.0;
      cudaEventRecord(e0, s);
      cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, n, n, n, &one, A.p, n, B.p, n, &zero, C.p, n);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms2;
      cudaEventElapsedTime(&ms2, e0, e1);
      printf("8192^3 NT: own %.1f TF/s, cuBLAS %.1f TF/s\n", 2.0 * n * n * n / (ms * 1e-3) / 1e12,
             2.0 * n * n * n / (ms2 * 1e-3) / 1e12);
    }
  }
  // setup shapes: forward-solve GEMM (m x 1024 x 1024, NT) and the staircase SYRK (n x n, k 1024)
  {
    const int64_t m = 26236, kk = 1024;
    DBuf<double> A(m * kk, s), B(kk * kk, s), C(m * m, s);
    std::vector<double> h1(m * kk);
    for (auto& v : h1) v = U(rng);
    HC_CUDA(cudaMemcpy(A.p, h1.data(), 8 * m * kk, cudaMemcpyHostToDevice));
    HC_CUDA(cudaMemcpy(B.p, h1.data(), 8 * kk * kk, cudaMemcpyHostToDevice));
    const double one = 1.0, mone = -1.0;
    float ms, ms2;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0, s);
      dblas::gemm(dblas::N, dblas::T, m, kk, kk, -1.0, A.p, m, B.p, kk, 1.0, C.p, m, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      cudaEventRecord(e0, s);
      cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, m, kk, kk, &mone, A.p, m, B.p, kk, &one, C.p, m);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms2, e0, e1);
    }
    printf("gemm %lldx1024x1024 NT: own %.1f TF/s, cuBLAS %.1f TF/s\n", (long long)m, 2.0 * m * kk * kk / (ms * 1e-3) / 1e12,
           2.0 * m * kk * kk / (ms2 * 1e-3) / 1e12);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0, s);
      dblas::syrk_ln(m, kk, 1.0, A.p, m, 1.0, C.p, m, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      cudaEventRecord(e0, s);
      cublasDsyrk(h, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, m, kk, &one, A.p, m, &one, C.p, m);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms2, e0, e1);
    }
    printf("syrk %lld k 1024: own %.1f TF/s, cuBLAS %.1f TF/s\n", (long long)m, 1.0 * m * m * kk / (ms * 1e-3) / 1e12,
           1.0 * m * m * kk / (ms2 * 1e-3) / 1e12);
  }
  // TRSM variants vs cuBLAS (well-conditioned L)
  for (int side = 0; side < 2; ++side)
    for (int op = 0; op < 2; ++op) {
      const int64_t m = side ? 1500 : 1100, n = side ? 1100 : 1500, d = side ? n : m;
      std::vector<double> hL(d * d, 0.0), hB(m * n);
      for (int64_t j = 0; j < d; ++j)
        for (int64_t i = j; i < d; ++i) hL[i + j * d] = i == j ? 2.0 + std::fabs(U(rng)) : 0.05 * U(rng) / std::sqrt((double)d);
      for (auto& v : hB) v = U(rng);
      DBuf<double> L, B1, B2;
      L.upload(hL.data(), hL.size(), s);
      B1.upload(hB.data(), hB.size(), s);
      B2.upload(hB.data(), hB.size(), s);
      dblas::trsm((dblas::Side)side, (dblas::Op)op, m, n, L.p, d, B1.p, m, s);
      const double one = 1.0;
      cublasDtrsm(h, side ? CUBLAS_SIDE_RIGHT : CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, op ? CUBLAS_OP_T : CUBLAS_OP_N,
                  CUBLAS_DIAG_NON_UNIT, m, n, &one, L.p, d, B2.p, m);
      printf("trsm %s %c rel diff %.3e\n", side ? "right" : "left", op ? 'T' : 'N',
             maxdiff(B1.download(), B2.download()));
    }
  // TRTRI
  {
    const int64_t d = 1300;
    std::vector<double> hL(d * d, 0.0);
    for (int64_t j = 0; j < d; ++j)
      for (int64_t i = j; i < d; ++i) hL[i + j * d] = i == j ? 2.0 + std::fabs(U(rng)) : 0.05 * U(rng) / std::sqrt((double)d);
    DBuf<double> L, Li, I2;
    L.upload(hL.data(), hL.size(), s);
    Li.alloc(d * d, s);
    I2.alloc(d * d, s);
    dblas::trtri_lower(d, L.p, d, Li.p, d, s);
    dblas::gemm(dblas::N, dblas::N, d, d, d, 1.0, L.p, d, Li.p, d, 0.0, I2.p, d, s);
    std::vector<double> hI = I2.download();
    double e = 0;
    for (int64_t j = 0; j < d; ++j)
      for (int64_t i = 0; i < d; ++i) e = std::max(e, std::fabs(hI[i + j * d] - (i == j ? 1.0 : 0.0)));
    printf("trtri: max |L Li - I| = %.3e\n", e);
  }
  return 0;
}
