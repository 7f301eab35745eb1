// Dense SPD kernels (see dense.cuh).
#include <cmath>
#include <vector>

#include "dblas.cuh"
#include <memory>

#include "dense.cuh"

namespace hcamg {

namespace {

constexpr int kSmallWarps = 4;

// Reference breakdown rule given the pivots computed so far (j0 = index of the
// first non-positive / non-finite pivot, or k if none).
__device__ int64_t breakdown_index(const double* piv, int k, int j0, double floor_) {
  if (j0 < k) {
    for (int j = 0; j <= j0; ++j)
      if (!(piv[j] > floor_) || !isfinite(piv[j])) return j;
    return j0;
  }
  int am = -1;
  double mn = INFINITY;
  for (int j = 0; j < k; ++j)
    if (piv[j] < mn) { mn = piv[j]; am = j; }
  if (am >= 0 && mn <= floor_) return am;
  return -1;
}

template <bool kInverse>
__global__ void __launch_bounds__(32 * kSmallWarps) k_small_spd(const DenseJob* __restrict__ jobs, int64_t njobs,
                                                                const double* __restrict__ A, double* __restrict__ B,
                                                                double* __restrict__ piv, int64_t* __restrict__ status) {
  __shared__ double T[kSmallWarps][32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double(*t)[33] = T[w];
  for (int64_t jb = (int64_t)blockIdx.x * kSmallWarps + w; jb < njobs; jb += (int64_t)gridDim.x * kSmallWarps) {
    const DenseJob jobv = jobs[jb];
    const int k = jobv.k;
    const double* a = A + jobv.a_off;
    double* pv = piv + jobv.piv_off;
    for (int c = 0; c < k; ++c)
      if (lane < k) t[lane][c] = a[lane + (int64_t)c * k];
    __syncwarp();
    double sc = lane < k ? fabs(t[lane][lane]) : 0.0;
    for (int o = 16; o; o >>= 1) sc = fmax(sc, __shfl_xor_sync(0xffffffffu, sc, o));
    const double floor_ = kPivotRtol * sc;
    int j0 = k;
    for (int j = 0; j < k; ++j) {
      double d = t[j][j];
      if (lane == 0) pv[j] = d;
      if (!(d > 0.0) || !isfinite(d)) { j0 = j; break; }
      double ljj = sqrt(d);
      __syncwarp();
      if (lane > j && lane < k) t[lane][j] = t[lane][j] / ljj;
      if (lane == j) t[j][j] = ljj;
      __syncwarp();
      for (int l = j + 1; l < k; ++l)
        if (lane >= l && lane < k) t[lane][l] = t[lane][l] - t[lane][j] * t[l][j];
      __syncwarp();
    }
    __syncwarp();
    int64_t bad = -1;
    if (lane == 0) bad = breakdown_index(pv, k, j0, floor_);
    bad = __shfl_sync(0xffffffffu, bad, 0);
    if (lane == 0) status[jb] = bad;
    if (bad >= 0) continue;
    double* b = B + jobv.b_off;
    const int nrhs = kInverse ? k : jobv.nrhs;
    for (int c = lane; c < nrhs; c += 32) {
      double y[32];
      for (int i = 0; i < k; ++i) {
        double v = kInverse ? (i == c ? 1.0 : 0.0) : b[i + (int64_t)c * k];
        for (int p = 0; p < i; ++p) v -= t[i][p] * y[p];
        y[i] = v / t[i][i];
      }
      for (int i = k - 1; i >= 0; --i) {
        double v = y[i];
        for (int p = i + 1; p < k; ++p) v -= t[p][i] * y[p];
        y[i] = v / t[i][i];
      }
      for (int i = 0; i < k; ++i) b[i + (int64_t)c * k] = y[i];
    }
    __syncwarp();
  }
}

constexpr int kTile = 128;
constexpr int kTileThreads = 512;

// Unblocked Cholesky of one nb x nb diagonal tile in shared memory.
// `bad` holds the first failing pivot index (-1: none so far); a tile after a
// failure returns at once, so a whole factorisation runs without host syncs.
// The trailing update of a column is spread over all threads element by
// element (round 2 first half: one thread per row walked its row serially,
// 150 us per 96-row tile; the envelope factorisation spent 0.9 of its 1.5 s
// in these leaves).  Every element still receives its updates in column
// order with the same expression, so the factor is bit-identical.
__global__ void __launch_bounds__(kTileThreads) k_potrf_tile(double* __restrict__ A, int64_t ld, int nb,
                                                             double* __restrict__ piv, long long* __restrict__ bad,
                                                             long long base, double* __restrict__ Li, int64_t ldi) {
  extern __shared__ double T[];  // nb x (nb+1), row-major T[i*(nb+1)+j]
  const int ldt = nb + 1;
  if (*(volatile long long*)bad >= 0) return;
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    int i = e % nb, j = e / nb;
    if (i >= j) T[i * ldt + j] = A[i + (int64_t)j * ld];
  }
  __syncthreads();
  __shared__ int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    double d = T[j * ldt + j];
    if (threadIdx.x == 0) {
      piv[j] = d;
      if (!(d > 0.0) || !isfinite(d)) { stop = 1; *bad = base + j; }
    }
    __syncthreads();
    if (stop) return;
    double ljj = sqrt(d);
    for (int i = j + 1 + threadIdx.x; i < nb; i += blockDim.x) T[i * ldt + j] /= ljj;
    __syncthreads();
    if (threadIdx.x == 0) T[j * ldt + j] = ljj;
    for (int i = j + 1 + (int)(threadIdx.x >> 5); i < nb; i += kTileThreads / 32) {  // a warp per row, lanes along it
      const double lij = T[i * ldt + j];
      for (int l = j + 1 + (int)(threadIdx.x & 31); l <= i; l += 32) T[i * ldt + l] -= lij * T[l * ldt + j];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    int i = e % nb, j = e / nb;
    if (i >= j) A[i + (int64_t)j * ld] = T[i * ldt + j];
  }
  if (!Li) return;
  // X = L^{-1} in place (L X = I, rows final from the top): at step p row p is
  // scaled by 1 / L[p][p], then every row below takes -L[i][p] X[p][.]; column
  // p of L is staged first because its positions receive X[.][p]
  __shared__ double col[kTile];
  for (int p = 0; p < nb; ++p) {
    const double lpp = T[p * ldt + p];
    __syncthreads();
    for (int i = p + 1 + threadIdx.x; i < nb; i += blockDim.x) col[i] = T[i * ldt + p];
    for (int j = threadIdx.x; j <= p; j += blockDim.x) T[p * ldt + j] = (j == p ? 1.0 : T[p * ldt + j]) / lpp;
    __syncthreads();
    for (int i = p + 1 + (int)(threadIdx.x >> 5); i < nb; i += kTileThreads / 32) {
      const double ci = col[i];
      for (int j = (int)(threadIdx.x & 31); j <= p; j += 32)
        T[i * ldt + j] = (j == p ? 0.0 : T[i * ldt + j]) - ci * T[p * ldt + j];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    int i = e % nb, j = e / nb;
    Li[i + (int64_t)j * ldi] = i >= j ? T[i * ldt + j] : 0.0;
  }
}

__global__ void k_diag_absmax(const double* __restrict__ A, int64_t k, int64_t ld, unsigned long long* out) {
  double m = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(A[i + i * ld]));
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

}  // namespace

void batched_small_spd_solve(const DenseJob* d_jobs, int64_t njobs, double* A, double* B, double* piv,
                             int64_t* status, cudaStream_t s) {
  if (!njobs) return;
  unsigned g = (unsigned)std::min<int64_t>((njobs + kSmallWarps - 1) / kSmallWarps, kSMs * 16);
  k_small_spd<false><<<g, 32 * kSmallWarps, 0, s>>>(d_jobs, njobs, A, B, piv, status);
  HC_CHECK_LAUNCH();
}

void batched_small_spd_inverse(const DenseJob* d_jobs, int64_t njobs, double* A, double* B, double* piv,
                               int64_t* status, cudaStream_t s) {
  if (!njobs) return;
  unsigned g = (unsigned)std::min<int64_t>((njobs + kSmallWarps - 1) / kSmallWarps, kSMs * 16);
  k_small_spd<true><<<g, 32 * kSmallWarps, 0, s>>>(d_jobs, njobs, A, B, piv, status);
  HC_CHECK_LAUNCH();
}

namespace {
// Recursive right-looking Cholesky: L11 = chol(A11); A21 := A21 L11^{-T};
// A22 -= A21 A21^T; L22 = chol(A22) -- leaves of <= kTile on one CTA, the
// updates on the own FP64 kernels (the trailing matrix is touched O(log n)
// times instead of once per 96-column panel)
void chol_rec(double* A, int64_t k, int64_t ld, double* piv, long long* bad, int64_t base, cudaStream_t s,
              double* Li = nullptr, int64_t ldi = 0) {
  static const int leaf = getenv("HCAMG_POTRF_TILE") ? std::max(32, std::min(kTile, atoi(getenv("HCAMG_POTRF_TILE")))) : 64;
  if (k <= leaf) {
    const size_t smem = sizeof(double) * kTile * (kTile + 1);
    static bool init = false;
    if (!init) {
      HC_CUDA(cudaFuncSetAttribute(k_potrf_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      init = true;
    }
    k_potrf_tile<<<1, kTileThreads, smem, s>>>(A, ld, (int)k, piv, bad, (long long)base, Li, ldi);
    HC_CHECK_LAUNCH();
    count_flops((double)k * k * k / 3.0 * (Li ? 2.0 : 1.0));
    return;
  }
  const int64_t k1 = std::min<int64_t>(k - 1, std::max<int64_t>(leaf, (k / 2 + leaf - 1) / leaf * leaf)), k2 = k - k1;
  double* A21 = A + k1;
  double* A22 = A + k1 + k1 * ld;
  if (!Li) {
    chol_rec(A, k1, ld, piv, bad, base, s);
    dblas::trsm(dblas::Right, dblas::T, k2, k1, A, ld, A21, ld, s);
    dblas::syrk_ln(k2, k1, -1.0, A21, ld, 1.0, A22, ld, s);
    chol_rec(A22, k2, ld, piv + k1, bad, base + k1, s);
    return;
  }
  // with the inverse of the factor alongside: the panel solve is a product with
  // L11^{-T} (no latency-bound triangular leaves), and L^{-1} is assembled as
  // [Li11 0; -Li22 L21 Li11, Li22]
  double* Li21 = Li + k1;
  double* Li22 = Li + k1 + k1 * ldi;
  chol_rec(A, k1, ld, piv, bad, base, s, Li, ldi);
  dblas::gemm(dblas::N, dblas::T, k2, k1, k1, 1.0, A21, ld, Li, ldi, 0.0, Li21, ldi, s);  // A21 L11^{-T} (Li21 as scratch)
  dblas::copy_block(k2, k1, Li21, ldi, A21, ld, s);
  dblas::syrk_ln(k2, k1, -1.0, A21, ld, 1.0, A22, ld, s);
  chol_rec(A22, k2, ld, piv + k1, bad, base + k1, s, Li22, ldi);
  DBuf<double> Tm(k2 * k1, s);
  dblas::gemm(dblas::N, dblas::N, k2, k1, k1, 1.0, A21, ld, Li, ldi, 0.0, Tm.p, k2, s);       // L21 Li11
  dblas::gemm(dblas::N, dblas::N, k2, k1, k2, -1.0, Li22, ldi, Tm.p, k2, 0.0, Li21, ldi, s);  // -Li22 (L21 Li11)
  HC_CUDA(cudaMemset2DAsync(Li + k1 * ldi, sizeof(double) * ldi, 0, sizeof(double) * k1, k2, s));
}
}  // namespace

void dense_cholesky_inv_async(double* A, int64_t k, int64_t ld, double* Li, int64_t ldi, double* piv, long long* bad,
                              int64_t base, cudaStream_t s) {
  if (k > 0) chol_rec(A, k, ld, piv, bad, base, s, Li, ldi);
}

void dense_cholesky_async(double* A, int64_t k, int64_t ld, double* piv, long long* bad, int64_t base,
                          cudaStream_t s) {
  if (k > 0) chol_rec(A, k, ld, piv, bad, base, s);
}

int64_t dense_cholesky_raw(double* A, int64_t k, int64_t ld, double* piv, cudaStream_t s) {
  if (k == 0) return 0;
  // leaf inverses of the panel solves cached for this factorisation (unless the caller's scope also spans its next step)
  std::unique_ptr<dblas::LeafCacheScope> leaves;
  if (!dblas::LeafCacheScope::active()) leaves.reset(new dblas::LeafCacheScope);
  DBuf<long long> bad(1, s);
  bad.fill_bytes(0xff);
  chol_rec(A, k, ld, piv, bad.p, 0, s);
  const long long b = read_scalar(bad.p, s);
  return b >= 0 ? (int64_t)b : k;
}

int64_t pivot_verdict(const std::vector<double>& hp, int64_t k, int64_t j0, double scale) {
  const double floor_ = kPivotRtol * scale;
  if (j0 < k) {
    for (int64_t j = 0; j <= j0; ++j)
      if (!(hp[(size_t)j] > floor_) || !std::isfinite(hp[(size_t)j])) return j;
    return j0;
  }
  if (k == 0) return -1;
  int64_t am = 0;
  for (int64_t j = 1; j < k; ++j)
    if (hp[(size_t)j] < hp[(size_t)am]) am = j;
  return hp[(size_t)am] <= floor_ ? am : -1;
}

int64_t dense_cholesky(double* A, int64_t k, int64_t ld, cudaStream_t s) {
  if (k == 0) return -1;
  DBuf<unsigned long long> mx(1, s);
  mx.zero();
  k_diag_absmax<<<grid_for(k, 256), 256, 0, s>>>(A, k, ld, mx.p);
  HC_CHECK_LAUNCH();
  DBuf<double> piv(k, s);
  const int64_t j0 = dense_cholesky_raw(A, k, ld, piv.p, s);
  unsigned long long hm = read_scalar(mx.p, s);
  double scale;
  memcpy(&scale, &hm, 8);
  std::vector<double> hp = piv.download();
  return pivot_verdict(hp, k, j0, scale);
}

namespace {
__global__ void k_sym_from_lower(const double* __restrict__ Lw, int64_t n, double* __restrict__ out) {
  // out (n x n, symmetric) from the lower triangle of Lw (column-major)
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % n, j = t / n;
    out[t] = i >= j ? Lw[i + j * n] : Lw[j + i * n];
  }
}
}  // namespace

// A^{-1} from its Cholesky factor L (lower, column-major in Lbuf, ld = n),
// exactly symmetric: Y = L^{-1} (recursive triangular inverse, n^3/3 flops),
// then the lower triangle of Y^T Y by GEMM tiles that start their inner
// dimension at their first row (Y is lower triangular: another n^3/3), written
// over Lbuf; the full symmetric inverse goes to Ainv.
void dense_spd_inverse(double* Lbuf, int64_t n, double* Ainv, cudaStream_t s) {
  if (n == 0) return;
  StageTimer st(s);
  dblas::trtri_lower(n, Lbuf, n, Ainv, n, s);
  st.mark("    inverse: Y = L^-1");
  dblas::gemm_tri_lower_tn(n, Ainv, n, Lbuf, n, s);
  st.mark("    inverse: lower(Y^T Y)");
  k_sym_from_lower<<<grid_for(n * n, 256, kSMs * 32), 256, 0, s>>>(Lbuf, n, Ainv);
  HC_CHECK_LAUNCH();
}

void dense_cholesky_solve(const double* L, int64_t k, int64_t ld, double* B, int64_t nrhs, int64_t ldb,
                          cudaStream_t s) {
  if (k == 0 || nrhs == 0) return;
  dblas::trsm(dblas::Left, dblas::N, k, nrhs, L, ld, B, ldb, s);
  dblas::trsm(dblas::Left, dblas::T, k, nrhs, L, ld, B, ldb, s);
}

}  // namespace hcamg
