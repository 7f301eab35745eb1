// FP64 level-3 kernels (see dblas.cuh).
//
// GEMM: 128 x 64 CTA tile, 8 warps of 32 x 32, each a 4 x 4 grid of DMMA
// m8n8k4 fragments (mma.sync ... .f64, FP64 tensor cores); operands staged
// through a 3-stage cp.async ring in shared memory with row strides = 4 (mod
// 16) doubles, so the fragment loads (lane -> (k = lane & 3, m = lane >> 2))
// are bank-conflict free.  Out-of-range elements are zero-filled by the copy.
// Triangular solves and inverses are recursive: halves down to 64 x 64
// diagonal blocks, inverted explicitly by one CTA each; everything else is GEMM.
#include <algorithm>
#include <unordered_map>
#include <vector>

#include "common.cuh"
#include "dblas.cuh"

namespace hcamg {
namespace dblas {

namespace {

#ifndef DBLAS_BN
#define DBLAS_BN 64
#endif
#ifndef DBLAS_STAGES
#define DBLAS_STAGES 3
#endif
constexpr int BM = 128, BN = DBLAS_BN, BK = 16, STAGES = DBLAS_STAGES, THREADS = 256;
constexpr int WNF = BN / 16;  // n fragments per warp (warps: 4 along m x 2 along n)
constexpr int LDA_S = BM + 4, LDB_S = BN + 4;
constexpr int STAGE_DOUBLES = BK * LDA_S + BK * LDB_S;
constexpr size_t SMEM = sizeof(double) * STAGES * STAGE_DOUBLES;
constexpr int NB0 = 64;  // recursion leaf of the triangular routines

struct GemmArgs {
  int64_t m, n, k, lda, ldb, ldc;
  double alpha, beta;
  const double* A;
  const double* B;
  double* C;
  const double* const* Ab;
  const double* const* Bb;
  double* const* Cb;
  int lower;     // only C entries with row >= col
  int kfromrow;  // op(A) is upper triangular in (row, k): k starts at the tile's first row
  int kfromcol;  // op(B) is lower triangular in (k, col): k starts at the tile's first column
  int ktorow;    // op(A) is lower triangular in (row, k): k ends with the tile's last row
  int ktocol;    // op(B) is upper triangular in (k, col) (B = Li^T, Li lower): k ends with the tile's last column
};

__device__ __forceinline__ void cp8(double* dst, const double* src, bool ok) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(ok ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp16(double* dst, const double* src, int bytes) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int kN>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(kN) : "memory");
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int TA, int TB>
__global__ void __launch_bounds__(THREADS) k_dgemm(GemmArgs g) {
  extern __shared__ __align__(16) double smem[];
  const int64_t bz = blockIdx.z;
  const double* A = g.Ab ? g.Ab[bz] : g.A;
  const double* B = g.Bb ? g.Bb[bz] : g.B;
  double* C = g.Cb ? g.Cb[bz] : g.C;
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  if (g.lower && m0 + BM <= n0) return;  // tile strictly above the diagonal
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int wm = w & 3, wn = w >> 2;
  // (the skipped products are exact zeros of a triangular factor: the sums are unchanged bit for bit)
  const int64_t kbeg = g.kfromrow ? (m0 / BK) * BK : g.kfromcol ? (n0 / BK) * BK : 0;
  const int64_t kend = g.ktorow ? (g.k < m0 + BM ? g.k : m0 + BM) : g.ktocol ? (g.k < n0 + BN ? g.k : n0 + BN) : g.k;
  const int64_t ktiles = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;

  // 16-byte copies along the contiguous global dimension when it is also the
  // contiguous shared dimension (op(A) = A, op(B) = B^T) and alignment allows
  const bool va = TA == 0 && ((reinterpret_cast<uintptr_t>(A) | (uintptr_t)(g.lda * 8)) & 15) == 0;
  const bool vb = TB == 1 && ((reinterpret_cast<uintptr_t>(B) | (uintptr_t)(g.ldb * 8)) & 15) == 0;
  auto load = [&](int64_t kt, int st) {
    double* As = smem + (size_t)st * STAGE_DOUBLES;
    double* Bs = As + BK * LDA_S;
    const int64_t k0 = kbeg + kt * BK;
    if (va) {
#pragma unroll
      for (int r = 0; r < (BM * BK) / (2 * THREADS); ++r) {
        const int idx = t + THREADS * r;
        const int il = 2 * (idx % (BM / 2)), kl = idx / (BM / 2);
        const int64_t i = m0 + il, kk = k0 + kl;
        const int bytes = kk < g.k ? (int)(8 * (g.m - i >= 2 ? 2 : (g.m - i > 0 ? g.m - i : 0))) : 0;
        cp16(As + kl * LDA_S + il, bytes ? A + i + kk * g.lda : A, bytes);
      }
    } else {
#pragma unroll
      for (int r = 0; r < (BM * BK) / THREADS; ++r) {
        const int idx = t + THREADS * r;
        int il, kl;
        if (TA == 0) { il = idx % BM; kl = idx / BM; }
        else { kl = idx % BK; il = idx / BK; }
        const int64_t i = m0 + il, kk = k0 + kl;
        const bool ok = i < g.m && kk < g.k;
        const double* src = ok ? (TA == 0 ? A + i + kk * g.lda : A + kk + i * g.lda) : A;
        cp8(As + kl * LDA_S + il, src, ok);
      }
    }
    if (vb) {
#pragma unroll
      for (int r = 0; r < (BN * BK) / (2 * THREADS); ++r) {
        const int idx = t + THREADS * r;
        const int jl = 2 * (idx % (BN / 2)), kl = idx / (BN / 2);
        const int64_t j = n0 + jl, kk = k0 + kl;
        const int bytes = kk < g.k ? (int)(8 * (g.n - j >= 2 ? 2 : (g.n - j > 0 ? g.n - j : 0))) : 0;
        cp16(Bs + kl * LDB_S + jl, bytes ? B + j + kk * g.ldb : B, bytes);
      }
    } else {
#pragma unroll
      for (int r = 0; r < (BN * BK) / THREADS; ++r) {
        const int idx = t + THREADS * r;
        int jl, kl;
        if (TB == 0) { kl = idx % BK; jl = idx / BK; }
        else { jl = idx % BN; kl = idx / BN; }
        const int64_t j = n0 + jl, kk = k0 + kl;
        const bool ok = j < g.n && kk < g.k;
        const double* src = ok ? (TB == 0 ? B + kk + j * g.ldb : B + j + kk * g.ldb) : B;
        cp8(Bs + kl * LDB_S + jl, src, ok);
      }
    }
  };

  double acc[4][WNF][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < WNF; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load(s, s);
    cp_commit();
  }
  for (int64_t kt = 0; kt < ktiles; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    if (kt + STAGES - 1 < ktiles) load(kt + STAGES - 1, (int)((kt + STAGES - 1) % STAGES));
    cp_commit();
    const double* As = smem + (size_t)(kt % STAGES) * STAGE_DOUBLES;
    const double* Bs = As + BK * LDA_S;
#pragma unroll
    for (int k4 = 0; k4 < BK / 4; ++k4) {
      const int kr = k4 * 4 + (lane & 3);
      double a[4], b[WNF];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = As[kr * LDA_S + wm * 32 + mi * 8 + (lane >> 2)];
#pragma unroll
      for (int ni = 0; ni < WNF; ++ni) b[ni] = Bs[kr * LDB_S + wn * (BN / 2) + ni * 8 + (lane >> 2)];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < WNF; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
    }
  }
  cp_wait<0>();
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < WNF; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t i = m0 + wm * 32 + mi * 8 + (lane >> 2);
        const int64_t j = n0 + wn * (BN / 2) + ni * 8 + 2 * (lane & 3) + h;
        if (i >= g.m || j >= g.n || (g.lower && i < j)) continue;
        double* c = C + i + j * g.ldc;
        const double v = g.alpha * acc[mi][ni][h];
        *c = g.beta == 0.0 ? v : fma(g.beta, *c, v);
      }
}

void launch(const GemmArgs& g, Op ta, Op tb, int64_t batch, cudaStream_t s) {
  if (g.m <= 0 || g.n <= 0 || batch <= 0) return;
  static bool init = false;
  if (!init) {
    HC_CUDA(cudaFuncSetAttribute(k_dgemm<0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    HC_CUDA(cudaFuncSetAttribute(k_dgemm<0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    HC_CUDA(cudaFuncSetAttribute(k_dgemm<1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    HC_CUDA(cudaFuncSetAttribute(k_dgemm<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    init = true;
  }
  const dim3 grid((unsigned)((g.m + BM - 1) / BM), (unsigned)((g.n + BN - 1) / BN), (unsigned)batch);
  require(grid.y <= 65535 && grid.z <= 65535, "dblas::gemm: grid too large");
  if (ta == N && tb == N) k_dgemm<0, 0><<<grid, THREADS, SMEM, s>>>(g);
  else if (ta == N && tb == T) k_dgemm<0, 1><<<grid, THREADS, SMEM, s>>>(g);
  else if (ta == T && tb == N) k_dgemm<1, 0><<<grid, THREADS, SMEM, s>>>(g);
  else k_dgemm<1, 1><<<grid, THREADS, SMEM, s>>>(g);
  HC_CHECK_LAUNCH();
}

// Inverse of the lower-triangular nb x nb blocks (nb <= 64) of a batch: one
// CTA of 64 threads per block, column j of the inverse by thread j
// (forward substitution on e_j), L staged in shared memory.
__global__ void __launch_bounds__(64) k_trtri_leaf(int nb, const double* const* Lp, const double* L0, int64_t ldl,
                                                   double* const* Lip, double* Li0, int64_t ldi, int64_t stride) {
  extern __shared__ double leaf_smem[];
  double(*Ls)[NB0 + 1] = reinterpret_cast<double(*)[NB0 + 1]>(leaf_smem);
  double(*X)[NB0 + 1] = reinterpret_cast<double(*)[NB0 + 1]>(leaf_smem + NB0 * (NB0 + 1));
  const int64_t bz = blockIdx.x;
  const double* L = Lp ? Lp[bz] : L0 + bz * stride * (ldl + 1);
  double* Li = Lip ? Lip[bz] : Li0 + bz * stride * (ldi + 1);
  const int j = threadIdx.x;
  for (int c = 0; c < nb; ++c)
    if (j < nb) Ls[j][c] = j >= c ? L[j + (int64_t)c * ldl] : 0.0;
  __syncthreads();
  if (j < nb) {
    for (int i = 0; i < nb; ++i) {
      double v = i == j ? 1.0 : 0.0;
      for (int p = j; p < i; ++p) v = fma(-Ls[i][p], X[p][j], v);
      X[i][j] = i >= j ? v / Ls[i][i] : 0.0;
    }
  }
  __syncthreads();
  for (int c = 0; c < nb; ++c)
    if (j < nb) Li[j + (int64_t)c * ldi] = X[j][c];
}

// dst (rows x cols, ld ldd) = src (ld lds)
__global__ void k_copy2d(int64_t rows, int64_t cols, const double* __restrict__ src, int64_t lds,
                         double* __restrict__ dst, int64_t ldd) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * cols; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % rows, c = t / rows;
    dst[i + c * ldd] = src[i + c * lds];
  }
}

void copy2d(int64_t rows, int64_t cols, const double* src, int64_t lds, double* dst, int64_t ldd, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return;
  k_copy2d<<<grid_for(rows * cols, 256, kSMs * 16), 256, 0, s>>>(rows, cols, src, lds, dst, ldd);
  HC_CHECK_LAUNCH();
}

constexpr size_t LEAF_SMEM = sizeof(double) * 2 * NB0 * (NB0 + 1);

void leaf_init() {
  static bool init = false;
  if (!init) {
    HC_CUDA(cudaFuncSetAttribute(k_trtri_leaf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LEAF_SMEM));
    init = true;
  }
}

int64_t split_at(int64_t m) {  // first half, a multiple of the leaf size
  const int64_t h = (m / 2 + NB0 - 1) / NB0 * NB0;
  return std::min<int64_t>(std::max<int64_t>(h, NB0), m - 1);
}

}  // namespace

void gemm(Op ta, Op tb, int64_t m, int64_t n, int64_t k, double alpha, const double* A, int64_t lda, const double* B,
          int64_t ldb, double beta, double* C, int64_t ldc, cudaStream_t s, bool lower) {
  GemmArgs g{m, n, k, lda, ldb, ldc, alpha, beta, A, B, C, nullptr, nullptr, nullptr, lower ? 1 : 0, 0};
  launch(g, ta, tb, 1, s);
  count_flops(2.0 * m * n * k * (lower ? 0.5 : 1.0));
}

void gemm_batched(Op ta, Op tb, int64_t m, int64_t n, int64_t k, double alpha, const double* const* A, int64_t lda,
                  const double* const* B, int64_t ldb, double beta, double* const* C, int64_t ldc, int64_t batch,
                  cudaStream_t s) {
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
    const int64_t nb = std::min<int64_t>(65535, batch - b0);
    GemmArgs g{m, n, k, lda, ldb, ldc, alpha, beta, nullptr, nullptr, nullptr, A + b0, B + b0, C + b0, 0, 0};
    launch(g, ta, tb, nb, s);
  }
  count_flops(2.0 * m * n * k * batch);
}

// batched product with a triangular factor: tri = 1: op(B) lower triangular (L21 Li11), tri = 2: op(A) lower
// triangular (Li22 X); the inner range of every tile is cut to the factor's nonzeros
static void gemm_batched_tri(int tri, int64_t m, int64_t n, int64_t k, double alpha, const double* const* A, int64_t lda,
                             const double* const* B, int64_t ldb, double* const* C, int64_t ldc, int64_t batch,
                             cudaStream_t s) {
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
    const int64_t nb = std::min<int64_t>(65535, batch - b0);
    GemmArgs g{m, n, k, lda, ldb, ldc, alpha, 0.0, nullptr, nullptr, nullptr, A + b0, B + b0, C + b0, 0, 0,
               tri == 1 ? 1 : 0, tri == 2 ? 1 : 0};
    launch(g, N, N, nb, s);
  }
  count_flops(1.0 * m * n * k * batch);
}

// C = X Li^T for a lower-triangular Li (n x n): the inner range of a tile ends with its last column
void gemm_rinv_t(int64_t m, int64_t n, const double* X, int64_t ldx, const double* Li, int64_t ldi, double* C,
                 int64_t ldc, cudaStream_t s) {
  GemmArgs g{m, n, n, ldx, ldi, ldc, 1.0, 0.0, X, Li, C, nullptr, nullptr, nullptr, 0, 0, 0, 0, 1};
  launch(g, N, T, 1, s);
  count_flops(1.0 * m * n * n);
}

void gemm_tri_lower_tn(int64_t n, const double* Y, int64_t ldy, double* C, int64_t ldc, cudaStream_t s) {
  GemmArgs g{n, n, n, ldy, ldy, ldc, 1.0, 0.0, Y, Y, C, nullptr, nullptr, nullptr, 1, 1};
  launch(g, T, N, 1, s);
  count_flops(2.0 * n * n * n / 6.0);
}

void syrk_ln(int64_t n, int64_t k, double alpha, const double* A, int64_t lda, double beta, double* C, int64_t ldc,
             cudaStream_t s) {
  gemm(N, T, n, n, k, alpha, A, lda, A, lda, beta, C, ldc, s, true);
}

namespace {
struct LeafCache {
  std::unordered_map<const double*, const double*> map;
  std::vector<DBuf<double>> store;
};
thread_local LeafCache* t_leaf = nullptr;
}  // namespace
LeafCacheScope::LeafCacheScope() : prev(t_leaf) { t_leaf = new LeafCache; }
LeafCacheScope::~LeafCacheScope() {
  delete t_leaf;
  t_leaf = static_cast<LeafCache*>(prev);
}
bool LeafCacheScope::active() { return t_leaf != nullptr; }

// the d x d inverse (ld d) of the diagonal leaf at L: cached per address inside a LeafCacheScope
static const double* leaf_inverse(int64_t d, const double* L, int64_t ldl, DBuf<double>& tmp, cudaStream_t s) {
  if (t_leaf && d == NB0) {
    auto it = t_leaf->map.find(L);
    if (it != t_leaf->map.end()) return it->second;
    t_leaf->store.emplace_back(d * d, s);
    double* p = t_leaf->store.back().p;
    leaf_init();
    k_trtri_leaf<<<1, NB0, LEAF_SMEM, s>>>((int)d, nullptr, L, ldl, nullptr, p, d, 0);
    HC_CHECK_LAUNCH();
    count_flops((double)d * d * d / 3.0);
    t_leaf->map[L] = p;
    return p;
  }
  tmp.alloc(d * d, s);
  trtri_lower(d, L, ldl, tmp.p, d, s);
  return tmp.p;
}

namespace {
__global__ void k_zero_upper(double* const* P, int64_t n, int64_t ld);  // (below)

// The recursion of trtri_lower on ONE large matrix of any size, level by level:
// every diagonal leaf in one launch per leaf size, then the nodes of each depth,
// deepest first, as two batched products per (m1, m2) shape.  Same tree
// (split_at), same products per node: the same inverse, bit for bit, in ~40
// launches instead of the ~2,500 dependent ones of the recursion (n = 26,236).
struct TriNode {
  int64_t off, m1, m2;
};
void tri_tree(int64_t off, int64_t n, int depth, std::vector<std::vector<TriNode>>& nodes,
              std::vector<std::pair<int64_t, int64_t>>& leaves) {
  if (n <= NB0) {
    leaves.emplace_back(off, n);
    return;
  }
  const int64_t m1 = split_at(n);
  if ((int)nodes.size() <= depth) nodes.resize((size_t)depth + 1);
  nodes[(size_t)depth].push_back(TriNode{off, m1, n - m1});
  tri_tree(off, m1, depth + 1, nodes, leaves);
  tri_tree(off + m1, n - m1, depth + 1, nodes, leaves);
}
}  // namespace

static void trtri_lower_levels(int64_t n, const double* L, int64_t ldl, double* Li, int64_t ldi, cudaStream_t s) {
  std::vector<std::vector<TriNode>> nodes;
  std::vector<std::pair<int64_t, int64_t>> leaves;
  tri_tree(0, n, 0, nodes, leaves);
  {
    DBuf<double*> one;
    one.upload(&Li, 1, s);
    k_zero_upper<<<dim3(kSMs * 4, 1), 256, 0, s>>>(one.p, n, ldi);
    HC_CHECK_LAUNCH();
    HC_CUDA(cudaStreamSynchronize(s));
  }
  // leaves, grouped by size
  std::sort(leaves.begin(), leaves.end(), [](auto& a, auto& b) { return a.second != b.second ? a.second > b.second : a.first < b.first; });
  leaf_init();
  for (size_t i = 0; i < leaves.size();) {
    size_t j = i;
    while (j < leaves.size() && leaves[j].second == leaves[i].second) ++j;
    std::vector<const double*> hl;
    std::vector<double*> hi;
    for (size_t t = i; t < j; ++t) {
      hl.push_back(L + leaves[t].first * (ldl + 1));
      hi.push_back(Li + leaves[t].first * (ldi + 1));
    }
    DBuf<const double*> dl;
    DBuf<double*> di;
    dl.upload(hl.data(), (int64_t)hl.size(), s);
    di.upload(hi.data(), (int64_t)hi.size(), s);
    const int64_t nb = leaves[i].second;
    for (int64_t b0 = 0; b0 < (int64_t)hl.size(); b0 += 65535) {
      const int64_t cnt = std::min<int64_t>(65535, (int64_t)hl.size() - b0);
      k_trtri_leaf<<<(unsigned)cnt, NB0, LEAF_SMEM, s>>>((int)nb, dl.p + b0, nullptr, ldl, di.p + b0, nullptr, ldi, 0);
      HC_CHECK_LAUNCH();
    }
    count_flops((double)nb * nb * nb / 3.0 * (double)hl.size());
    HC_CUDA(cudaStreamSynchronize(s));  // the host pointer lists are staged
    i = j;
  }
  for (int d = (int)nodes.size() - 1; d >= 0; --d) {
    std::vector<TriNode>& nd = nodes[(size_t)d];
    std::sort(nd.begin(), nd.end(), [](const TriNode& a, const TriNode& b) {
      return a.m1 != b.m1 ? a.m1 > b.m1 : a.m2 != b.m2 ? a.m2 > b.m2 : a.off < b.off;
    });
    int64_t scratch = 0;
    for (const TriNode& q : nd) scratch += q.m1 * q.m2;
    DBuf<double> Tm(scratch, s);
    int64_t used = 0;
    for (size_t i = 0; i < nd.size();) {
      size_t j = i;
      while (j < nd.size() && nd[j].m1 == nd[i].m1 && nd[j].m2 == nd[i].m2) ++j;
      const int64_t m1 = nd[i].m1, m2 = nd[i].m2;
      std::vector<const double*> a1, b1, a2, b2;
      std::vector<double*> c1, c2;
      for (size_t t = i; t < j; ++t) {
        const int64_t o = nd[t].off;
        double* tm = Tm.p + used;
        used += m1 * m2;
        a1.push_back(L + (o + m1) + o * ldl);           // L21
        b1.push_back(Li + o * (ldi + 1));               // Li11
        c1.push_back(tm);
        a2.push_back(Li + (o + m1) * (ldi + 1));        // Li22
        b2.push_back(tm);
        c2.push_back(Li + (o + m1) + o * ldi);          // Li21
      }
      DBuf<const double*> da1, db1, da2, db2;
      DBuf<double*> dc1, dc2;
      da1.upload(a1.data(), (int64_t)a1.size(), s);
      db1.upload(b1.data(), (int64_t)b1.size(), s);
      dc1.upload(c1.data(), (int64_t)c1.size(), s);
      da2.upload(a2.data(), (int64_t)a2.size(), s);
      db2.upload(b2.data(), (int64_t)b2.size(), s);
      dc2.upload(c2.data(), (int64_t)c2.size(), s);
      gemm_batched_tri(1, m2, m1, m1, 1.0, da1.p, ldl, db1.p, ldi, dc1.p, m2, (int64_t)a1.size(), s);   // L21 Li11
      gemm_batched_tri(2, m2, m1, m2, -1.0, da2.p, ldi, db2.p, m2, dc2.p, ldi, (int64_t)a2.size(), s);  // -Li22 (..)
      HC_CUDA(cudaStreamSynchronize(s));  // the pointer lists go out of scope
      i = j;
    }
  }
}

void trtri_lower(int64_t n, const double* L, int64_t ldl, double* Li, int64_t ldi, cudaStream_t s) {
  if (n <= 0) return;
  if (n >= 16 * NB0 && !getenv("HCAMG_TRTRI_RECURSIVE")) {
    trtri_lower_levels(n, L, ldl, Li, ldi, s);
    return;
  }
  if (n <= NB0) {
    if (t_leaf && n == NB0) {
      auto it = t_leaf->map.find(L);
      if (it != t_leaf->map.end()) {
        copy2d(n, n, it->second, n, Li, ldi, s);
        return;
      }
    }
    leaf_init();
    k_trtri_leaf<<<1, NB0, LEAF_SMEM, s>>>((int)n, nullptr, L, ldl, nullptr, Li, ldi, 0);
    HC_CHECK_LAUNCH();
    count_flops((double)n * n * n / 3.0);
    return;
  }
  // [L11 0; L21 L22]^{-1} = [Li11 0; -Li22 L21 Li11  Li22]
  const int64_t m1 = split_at(n), m2 = n - m1;
  trtri_lower(m1, L, ldl, Li, ldi, s);
  trtri_lower(m2, L + m1 + m1 * ldl, ldl, Li + m1 + m1 * ldi, ldi, s);
  DBuf<double> Tm(m2 * m1, s);
  gemm(N, N, m2, m1, m1, 1.0, L + m1, ldl, Li, ldi, 0.0, Tm.p, m2, s);                    // L21 Li11
  gemm(N, N, m2, m1, m2, -1.0, Li + m1 + m1 * ldi, ldi, Tm.p, m2, 0.0, Li + m1, ldi, s);  // -Li22 (L21 Li11)
  if (m1 > 0) HC_CUDA(cudaMemset2DAsync(Li + m1 * ldi, sizeof(double) * ldi, 0, sizeof(double) * m1, m2, s));
}

void trtri_lower_batched(int64_t nb, const double* const* L, int64_t ldl, double* const* Li, int64_t ldi, int64_t batch,
                         cudaStream_t s) {
  if (batch <= 0) return;
  if (nb <= NB0) {
    leaf_init();
    k_trtri_leaf<<<(unsigned)batch, NB0, LEAF_SMEM, s>>>((int)nb, L, nullptr, ldl, Li, nullptr, ldi, 0);
    HC_CHECK_LAUNCH();
    count_flops((double)nb * nb * nb / 3.0 * batch);
    return;
  }
  std::vector<const double*> hl((size_t)batch);
  std::vector<double*> hi((size_t)batch);
  HC_CUDA(cudaMemcpyAsync(hl.data(), L, sizeof(void*) * batch, cudaMemcpyDeviceToHost, s));
  HC_CUDA(cudaMemcpyAsync(hi.data(), Li, sizeof(void*) * batch, cudaMemcpyDeviceToHost, s));
  HC_CUDA(cudaStreamSynchronize(s));
  for (int64_t b = 0; b < batch; ++b) trtri_lower(nb, hl[(size_t)b], ldl, hi[(size_t)b], ldi, s);
}

namespace {
__global__ void k_zero_upper(double* const* P, int64_t n, int64_t ld) {
  double* A = P[blockIdx.y];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % n, j = t / n;
    if (i < j) A[i + j * ld] = 0.0;
  }
}
}  // namespace

// Inverses of many lower-triangular n x n matrices at once (host pointer
// lists).  For n = NB0 * 2^k the recursion of trtri_lower is run level by
// level over ALL matrices: one launch inverts every 64 x 64 diagonal block of
// every matrix, then each doubling of the block size is two batched GEMMs
// (L21 Li11, then -Li22 (L21 Li11)) over every node of every matrix -- 2 k + 2
// launches in all, where the per-matrix recursion issues ~100 small ones each.
// Same arithmetic per matrix as trtri_lower.
void trtri_lower_many(int64_t n, const std::vector<const double*>& L, int64_t ldl, const std::vector<double*>& Li,
                      int64_t ldi, cudaStream_t s) {
  const int64_t batch = (int64_t)L.size();
  if (batch == 0 || n <= 0) return;
  bool pow2 = n % NB0 == 0;
  for (int64_t q = n / NB0; pow2 && q > 1; q /= 2) pow2 = q % 2 == 0;
  if (!pow2 || batch == 1) {
    for (int64_t b = 0; b < batch; ++b) trtri_lower(n, L[(size_t)b], ldl, Li[(size_t)b], ldi, s);
    return;
  }
  auto up = [&](const std::vector<const double*>& h, DBuf<const double*>& d) {
    d.upload(h.data(), (int64_t)h.size(), s);
    return d.p;
  };
  {
    DBuf<double*> dli;
    dli.upload(Li.data(), batch, s);
    k_zero_upper<<<dim3(kSMs / 2, (unsigned)batch), 256, 0, s>>>(dli.p, n, ldi);
    HC_CHECK_LAUNCH();
    const int64_t nl = n / NB0;
    std::vector<const double*> hl;
    std::vector<double*> hi;
    for (int64_t b = 0; b < batch; ++b)
      for (int64_t t = 0; t < nl; ++t) {
        hl.push_back(L[(size_t)b] + t * NB0 * (ldl + 1));
        hi.push_back(Li[(size_t)b] + t * NB0 * (ldi + 1));
      }
    DBuf<const double*> dl;
    DBuf<double*> di;
    dl.upload(hl.data(), (int64_t)hl.size(), s);
    di.upload(hi.data(), (int64_t)hi.size(), s);
    leaf_init();
    for (int64_t b0 = 0; b0 < (int64_t)hl.size(); b0 += 65535) {
      const int64_t nb = std::min<int64_t>(65535, (int64_t)hl.size() - b0);
      k_trtri_leaf<<<(unsigned)nb, NB0, LEAF_SMEM, s>>>((int)NB0, dl.p + b0, nullptr, ldl, di.p + b0, nullptr, ldi, 0);
      HC_CHECK_LAUNCH();
    }
    count_flops((double)NB0 * NB0 * NB0 / 3.0 * (double)hl.size());
    HC_CUDA(cudaStreamSynchronize(s));  // the host pointer lists above are staged
  }
  for (int64_t h = NB0; h < n; h *= 2) {
    const int64_t nodes = n / (2 * h);
    DBuf<double> Tm(batch * nodes * h * h, s);
    std::vector<const double*> a1, b1, a2, b2;
    std::vector<double*> c1, c2;
    for (int64_t b = 0; b < batch; ++b)
      for (int64_t q = 0; q < nodes; ++q) {
        const int64_t o = q * 2 * h;
        double* tm = Tm.p + (b * nodes + q) * h * h;
        a1.push_back(L[(size_t)b] + (o + h) + o * ldl);          // L21
        b1.push_back(Li[(size_t)b] + o * (ldi + 1));            // Li11
        c1.push_back(tm);
        a2.push_back(Li[(size_t)b] + (o + h) * (ldi + 1));      // Li22
        b2.push_back(tm);
        c2.push_back(Li[(size_t)b] + (o + h) + o * ldi);        // Li21
      }
    DBuf<const double*> da1, db1, da2, db2;
    DBuf<double*> dc1, dc2;
    dc1.upload(c1.data(), (int64_t)c1.size(), s);
    dc2.upload(c2.data(), (int64_t)c2.size(), s);
    gemm_batched_tri(1, h, h, h, 1.0, up(a1, da1), ldl, up(b1, db1), ldi, dc1.p, h, (int64_t)a1.size(), s);
    gemm_batched_tri(2, h, h, h, -1.0, up(a2, da2), ldi, up(b2, db2), h, dc2.p, ldi, (int64_t)a2.size(), s);
    HC_CUDA(cudaStreamSynchronize(s));  // Tm and the pointer lists go out of scope
  }
}

void trsm(Side side, Op op, int64_t m, int64_t n, const double* L, int64_t ldl, double* B, int64_t ldb,
          cudaStream_t s) {
  const int64_t d = side == Left ? m : n;  // dimension of L
  if (m <= 0 || n <= 0) return;
  if (d <= NB0) {
    // leaf: X = op(Li) B (left) or B op(Li) (right) through a temporary
    DBuf<double> Lt, X(m * n, s);
    const double* Li = leaf_inverse(d, L, ldl, Lt, s);
    if (side == Left) gemm(op, N, m, n, d, 1.0, Li, d, B, ldb, 0.0, X.p, m, s);
    else gemm(N, op, m, n, d, 1.0, B, ldb, Li, d, 0.0, X.p, m, s);
    copy2d(m, n, X.p, m, B, ldb, s);
    return;
  }
  const int64_t d1 = split_at(d), d2 = d - d1;
  const double* L11 = L;
  const double* L21 = L + d1;
  const double* L22 = L + d1 + d1 * ldl;
  if (side == Left && op == N) {        // L X = B
    trsm(side, op, d1, n, L11, ldl, B, ldb, s);
    gemm(N, N, d2, n, d1, -1.0, L21, ldl, B, ldb, 1.0, B + d1, ldb, s);
    trsm(side, op, d2, n, L22, ldl, B + d1, ldb, s);
  } else if (side == Left) {           // L^T X = B
    trsm(side, op, d2, n, L22, ldl, B + d1, ldb, s);
    gemm(T, N, d1, n, d2, -1.0, L21, ldl, B + d1, ldb, 1.0, B, ldb, s);
    trsm(side, op, d1, n, L11, ldl, B, ldb, s);
  } else if (op == T) {                // X L^T = B
    trsm(side, op, m, d1, L11, ldl, B, ldb, s);
    gemm(N, T, m, d2, d1, -1.0, B, ldb, L21, ldl, 1.0, B + d1 * ldb, ldb, s);
    trsm(side, op, m, d2, L22, ldl, B + d1 * ldb, ldb, s);
  } else {                             // X L = B
    trsm(side, op, m, d2, L22, ldl, B + d1 * ldb, ldb, s);
    gemm(N, N, m, d1, d2, -1.0, B + d1 * ldb, ldb, L21, ldl, 1.0, B, ldb, s);
    trsm(side, op, m, d1, L11, ldl, B, ldb, s);
  }
}

void copy_block(int64_t rows, int64_t cols, const double* src, int64_t lds, double* dst, int64_t ldd, cudaStream_t s) {
  copy2d(rows, cols, src, lds, dst, ldd, s);
}

// B_b := B_b Li^T for every tile of the batch, Li = L^{-1} (nb x nb, ld nb) given
void apply_rinv_t_batched(int64_t m, int64_t nb, const double* Li, const std::vector<double*>& hb, int64_t ldb,
                          cudaStream_t s) {
  const int64_t batch = (int64_t)hb.size();
  if (batch <= 0) return;
  DBuf<double> X(batch * m * nb, s);
  std::vector<const double*> pa((size_t)batch), pb((size_t)batch, Li);
  std::vector<double*> pc((size_t)batch);
  for (int64_t b = 0; b < batch; ++b) {
    pa[(size_t)b] = hb[(size_t)b];
    pc[(size_t)b] = X.p + b * m * nb;
  }
  DBuf<const double*> da, db;
  DBuf<double*> dc;
  da.upload(pa.data(), batch, s);
  db.upload(pb.data(), batch, s);
  dc.upload(pc.data(), batch, s);
  {
    GemmArgs g{m, nb, nb, ldb, nb, m, 1.0, 0.0, nullptr, nullptr, nullptr, da.p, db.p, dc.p, 0, 0, 0, 0, 1};
    launch(g, N, T, batch, s);  // (batch <= the tiles of one block column)
    count_flops(1.0 * m * nb * nb * batch);
  }
  for (int64_t b = 0; b < batch; ++b) copy2d(m, nb, X.p + b * m * nb, m, hb[(size_t)b], ldb, s);
}

void trsm_rlt_batched(int64_t m, int64_t nb, const std::vector<const double*>& hl, int64_t ldl,
                      const std::vector<double*>& hb, int64_t ldb, cudaStream_t s) {
  const int64_t batch = (int64_t)hb.size();
  if (batch <= 0) return;
  std::vector<const double*> uniq;
  std::vector<int64_t> which((size_t)batch);
  for (int64_t b = 0; b < batch; ++b) {
    auto it = std::find(uniq.begin(), uniq.end(), hl[(size_t)b]);
    which[(size_t)b] = it - uniq.begin();
    if (it == uniq.end()) uniq.push_back(hl[(size_t)b]);
  }
  DBuf<double> Li((int64_t)uniq.size() * nb * nb, s), X(batch * m * nb, s);
  for (size_t u = 0; u < uniq.size(); ++u) trtri_lower(nb, uniq[u], ldl, Li.p + u * nb * nb, nb, s);
  std::vector<const double*> pa((size_t)batch), pb((size_t)batch);
  std::vector<double*> pc((size_t)batch);
  for (int64_t b = 0; b < batch; ++b) {
    pa[(size_t)b] = hb[(size_t)b];
    pb[(size_t)b] = Li.p + which[(size_t)b] * nb * nb;
    pc[(size_t)b] = X.p + b * m * nb;
  }
  DBuf<const double*> da, db;
  DBuf<double*> dc;
  da.upload(pa.data(), batch, s);
  db.upload(pb.data(), batch, s);
  dc.upload(pc.data(), batch, s);
  gemm_batched(N, T, m, nb, nb, 1.0, da.p, ldb, db.p, nb, 0.0, dc.p, m, batch, s);
  for (int64_t b = 0; b < batch; ++b) copy2d(m, nb, X.p + b * m * nb, m, hb[(size_t)b], ldb, s);
}

}  // namespace dblas
}  // namespace hcamg
