// Dense-interpolation regime (see giant.cuh).
//
// In 3D the interior block A_II of the reference's harmonic extension
// (transfer.py:77-122) is one connected component with ~80 % of the DoFs
// (SURVEY.md F3), so P has dense interior rows and the work is dense linear
// algebra:
//   * Cholesky of A_GG after a reverse Cuthill-McKee ordering -- the ordering
//     the reference's own cholesky() applies to components above its dense
//     cutoff (sparse.py:276-301) -- kept in NB = 1024 tiles inside the block
//     envelope only (config 2: 5.4 GB instead of 113 GB for all lower tiles,
//     ~1 s instead of ~50 s), right-looking: own POTRF on the diagonal tile,
//     batched cuBLAS DTRSM/DGEMM panels (FP64; cuBLAS only for these plain
//     level-3 calls);
//   * Z = A_GG^{-1} W' solved on the row-major RHS (= the column-major
//     transpose) in the factored order, envelope tiles only (~4 s);
//   * P = P_s - S_G Z applied as CSR + a dense row-major block streamed at
//     HBM bandwidth (prolongation: row batches per CTA; restriction: chunked
//     column sums reduced in a fixed two-level order);
//   * Galerkin A_c = P^T A P in Schur form with the solve residual
//     rho = W' - A_GG Z (exact in exact arithmetic, second order in the
//     component-solve error like the reference's P^T (A P)); Z^T rho on the
//     tensor cores in TF32 (see galerkin_hybrid).
#include <cub/cub.cuh>

#include <algorithm>
#include <unordered_map>
#include <vector>

#include "dblas.cuh"
#include "dense.cuh"
#include "giant.cuh"
#include "dist.cuh"
#include "sparse.cuh"

namespace hcamg {

namespace {

constexpr int64_t kNB = 1024;


// Lower Cholesky factor in NB x NB column-major tiles, stored only inside the
// block envelope: block row I keeps tiles J in [j0[I], I], where j0[I] is the
// tile of the first nonzero of any row of the block.  Cholesky fill never
// leaves the envelope (row i of L starts where row i of A starts), so this
// is exact; under a reverse Cuthill-McKee order the envelope of config 2's
// 167,784-row block is 5.4 GB instead of the 113 GB of all lower tiles.
struct Packed {
  int64_t n = 0, T = 0;
  std::vector<int64_t> j0, off;
  DBuf<double> buf;
  bool has(int64_t I, int64_t J) const { return J >= j0[(size_t)I] && J <= I; }
  double* tile(int64_t I, int64_t J) const { return buf.p + (off[(size_t)I] + J - j0[(size_t)I]) * kNB * kNB; }
};

__global__ void k_pack_env(const int64_t* __restrict__ ap, const int32_t* __restrict__ ai,
                           const double* __restrict__ av, int64_t n, int64_t T, const int64_t* __restrict__ j0,
                           const int64_t* __restrict__ off, double* __restrict__ buf) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < T * kNB;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t I = q / kNB, li = q % kNB;
    if (q >= n) {  // identity padding keeps the padded matrix SPD
      buf[(off[I] + I - j0[I]) * kNB * kNB + li + li * kNB] = 1.0;
      continue;
    }
    for (int64_t e = ap[q]; e < ap[q + 1]; ++e) {
      const int64_t j = ai[e];
      if (j > q) continue;  // columns need not be sorted (permuted input)
      const int64_t J = j / kNB, lj = j % kNB;
      buf[(off[I] + J - j0[I]) * kNB * kNB + li + lj * kNB] = av[e];
    }
  }
}

// out[i, k] = in[src[i], col[k]]  (kScatter: out[src[i], col[k]] = in[i, k]) for row-major n x m
template <bool kScatter>
__global__ void k_permute_rc(int64_t n, int64_t m, const int32_t* __restrict__ src, const int32_t* __restrict__ col,
                             const double* __restrict__ in, double* __restrict__ out) {
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const double* a = kScatter ? in + i * m : in + (int64_t)src[i] * m;
    double* b = kScatter ? out + (int64_t)src[i] * m : out + i * m;
    if (kScatter)
      for (int64_t k = threadIdx.x; k < m; k += blockDim.x) b[col[k]] = a[k];
    else
      for (int64_t k = threadIdx.x; k < m; k += blockDim.x) b[k] = a[col[k]];
  }
}

// Same, one row per CTA staged in shared memory (m * 8 bytes <= 227 KB):
// coalesced global traffic, the column permutation done in shared memory.
template <bool kScatter>
__global__ void __launch_bounds__(1024) k_permute_rc_smem(int64_t n, int64_t m, const int32_t* __restrict__ src,
                                                           const int32_t* __restrict__ col,
                                                           const double* __restrict__ in, double* __restrict__ out) {
  extern __shared__ double row[];
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const double* a = kScatter ? in + i * m : in + (int64_t)src[i] * m;
    double* b = kScatter ? out + (int64_t)src[i] * m : out + i * m;
    if (kScatter) {
      for (int64_t k = threadIdx.x; k < m; k += blockDim.x) row[col[k]] = a[k];
    } else {
      for (int64_t k = threadIdx.x; k < m; k += blockDim.x) row[k] = a[k];
    }
    __syncthreads();
    if (kScatter) {
      for (int64_t k = threadIdx.x; k < m; k += blockDim.x) b[k] = row[k];
    } else {
      for (int64_t k = threadIdx.x; k < m; k += blockDim.x) b[k] = row[col[k]];
    }
    __syncthreads();
  }
}

template <bool kScatter>
void permute_rc(int64_t n, int64_t m, const int32_t* src, const int32_t* col, const double* in, double* out,
                cudaStream_t s) {
  const size_t smem = sizeof(double) * (size_t)m;
  if (smem <= 227 * 1024) {
    HC_CUDA(cudaFuncSetAttribute(k_permute_rc_smem<kScatter>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_permute_rc_smem<kScatter><<<(unsigned)std::min<int64_t>(n, kSMs * 2), 1024, smem, s>>>(n, m, src, col, in, out);
  } else {
    k_permute_rc<kScatter><<<(unsigned)std::min<int64_t>(n, kSMs * 16), 256, 0, s>>>(n, m, src, col, in, out);
  }
  HC_CHECK_LAUNCH();
}

// first[c] = min over rows r with B[r, c] != 0 of rank[r]  (first = n when the column is empty)
__global__ void k_first_row(int64_t n, int64_t m, const double* __restrict__ B, const int32_t* __restrict__ rank,
                            int* __restrict__ first) {
  for (int64_t r = blockIdx.x; r < n; r += gridDim.x)
    for (int64_t c = threadIdx.x; c < m; c += blockDim.x)
      if (B[r * m + c] != 0.0) atomicMin(first + c, rank[r]);
}

// the same from a CSR right-hand side (explicit zeros skipped, as the dense test does)
__global__ void k_first_row_csr(int64_t n, const int64_t* __restrict__ bp, const int32_t* __restrict__ bi,
                                const double* __restrict__ bv, const int32_t* __restrict__ rank,
                                int* __restrict__ first) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    for (int64_t e = bp[r]; e < bp[r + 1]; ++e)
      if (bv[e] != 0.0) atomicMin(first + bi[e], rank[r]);
}

// out[rank[r], colinv[c]] = B[r, c] for the entries of a CSR B (out zeroed before; row-major n x m)
__global__ void k_scatter_rc_csr(int64_t n, int64_t m, const int64_t* __restrict__ bp, const int32_t* __restrict__ bi,
                                 const double* __restrict__ bv, const int32_t* __restrict__ rank,
                                 const int32_t* __restrict__ colinv, double* __restrict__ out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    for (int64_t e = bp[r]; e < bp[r + 1]; ++e) out[(int64_t)rank[r] * m + colinv[bi[e]]] = bv[e];
}

__global__ void k_csr_diag_absmax(const int64_t* __restrict__ ap, const int32_t* __restrict__ ai,
                                  const double* __restrict__ av, int64_t n, unsigned long long* out) {
  double m = 0.0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    for (int64_t e = ap[q]; e < ap[q + 1]; ++e)
      if (ai[e] == q) m = fmax(m, fabs(av[e]));
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

template <class T>
const T** upload_ptrs(std::vector<const T*>& h, DBuf<const T*>& d, cudaStream_t s) {
  d.alloc((int64_t)h.size(), s);
  HC_CUDA(cudaMemcpyAsync(d.p, h.data(), sizeof(T*) * h.size(), cudaMemcpyHostToDevice, s));
  return d.p;
}

// ---- hybrid P kernels

// Prolongation, dense part, rows [q0, q1): one warp per PAIR of rows (the
// e loads are shared by both rows, halving their L1/L2 traffic), e staged in
// shared memory when it fits (n_c <= 25k), 8 independent 16-byte Z loads in
// flight per lane.  kMode 0: x[rows[q]] -= Z[q,:].e; 1: x[q] = M[q,:].e;
// 2: the row results go to every rank's exchange area at q (distributed
// solve), then the last CTA signals.  Every row is summed in the same order
// (4 lane-strided accumulators, then a butterfly) whatever rows share its
// warp, so a row-partitioned product is bit-identical.
__device__ __forceinline__ double2 ld_z2(const double* p, bool aligned) {
  if (aligned) return __ldcs(reinterpret_cast<const double2*>(p));
  return make_double2(__ldcs(p), __ldcs(p + 1));
}

__device__ __forceinline__ double2 ld_e2(const double* p) {
  return *reinterpret_cast<const double2*>(p);  // c even, e 16-byte aligned
}

template <bool kSmemE, int kMode>
__global__ void __launch_bounds__(512) k_z_rows(const int* stop, int64_t q0, int64_t q1, int64_t nc,
                                                const double* __restrict__ Z, const int32_t* __restrict__ rows,
                                                const double* __restrict__ e, double* __restrict__ x, Xchg xc) {
  if (*stop) return;
  extern __shared__ double2 es2[];
  const double* ev = e;
  if (kSmemE) {
    double* es = reinterpret_cast<double*>(es2);
    for (int64_t c = threadIdx.x; c < nc; c += blockDim.x) es[c] = e[c];
    __syncthreads();
    ev = es;
  }
  unsigned long long ep = 0;
  if (kMode == 2) ep = xepoch(xc);
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = q0 + 2 * (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); q < q1; q += 2 * nw) {
    const bool two = q + 1 < q1;
    const double* za = Z + q * nc;
    const double* zb = two ? za + nc : za;
    const bool ala = ((q * nc) & 1) == 0, alb = (((q + (two ? 1 : 0)) * nc) & 1) == 0;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, b0 = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0;
    int64_t c = 2 * lane;
    for (; c + 192 + 1 < nc; c += 256) {
      const double2 u0 = ld_z2(za + c, ala), u1 = ld_z2(za + c + 64, ala);
      const double2 u2 = ld_z2(za + c + 128, ala), u3 = ld_z2(za + c + 192, ala);
      const double2 w0 = ld_z2(zb + c, alb), w1 = ld_z2(zb + c + 64, alb);
      const double2 w2 = ld_z2(zb + c + 128, alb), w3 = ld_z2(zb + c + 192, alb);
      const double2 e0 = ld_e2(ev + c), e1 = ld_e2(ev + c + 64);
      const double2 e2 = ld_e2(ev + c + 128), e3 = ld_e2(ev + c + 192);
      a0 = fma(u0.x, e0.x, fma(u0.y, e0.y, a0));
      a1 = fma(u1.x, e1.x, fma(u1.y, e1.y, a1));
      a2 = fma(u2.x, e2.x, fma(u2.y, e2.y, a2));
      a3 = fma(u3.x, e3.x, fma(u3.y, e3.y, a3));
      b0 = fma(w0.x, e0.x, fma(w0.y, e0.y, b0));
      b1 = fma(w1.x, e1.x, fma(w1.y, e1.y, b1));
      b2 = fma(w2.x, e2.x, fma(w2.y, e2.y, b2));
      b3 = fma(w3.x, e3.x, fma(w3.y, e3.y, b3));
    }
    for (; c + 1 < nc; c += 64) {
      const double2 u0 = ld_z2(za + c, ala), w0 = ld_z2(zb + c, alb), e0 = ld_e2(ev + c);
      a0 = fma(u0.x, e0.x, fma(u0.y, e0.y, a0));
      b0 = fma(w0.x, e0.x, fma(w0.y, e0.y, b0));
    }
    if (c < nc) {
      a0 = fma(za[c], ev[c], a0);
      b0 = fma(zb[c], ev[c], b0);
    }
    double acc = (a0 + a1) + (a2 + a3), bcc = (b0 + b1) + (b2 + b3);
    for (int o = 16; o; o >>= 1) {
      acc += __shfl_xor_sync(0xffffffffu, acc, o);
      bcc += __shfl_xor_sync(0xffffffffu, bcc, o);
    }
    if (kMode == 2) {
      if (lane < xc.nranks) {
        double* y = xarea(xc, lane, ep + 1);
        y[q] = acc;
        if (two) y[q + 1] = bcc;
      }
    } else if (lane == 0) {
      if (kMode == 1) {
        x[q] = acc;
        if (two) x[q + 1] = bcc;
      } else {
        x[rows[q]] -= acc;
        if (two) x[rows[q + 1]] -= bcc;
      }
    }
  }
  if (kMode == 2) xsignal(xc, ep);
}

// Same product for wide rows (n_c >= 4096): a 256-thread CTA sweeps a batch
// of 16 consecutive rows together, 512 columns (4 KB of each row) per step,
// thread t owning columns 2t + 512k of all 16 rows -- 16 independent 16-byte
// loads in flight per thread and a few long sequential streams per CTA
// instead of many short ones (config 2: 5.0 ms for 35.2 GB = 7.0 TB/s vs
// 5.7 ms with a warp per row).  Per row: thread partials, butterfly within
// each warp, then the 8 warp sums in warp order (fixed for every row,
// independent of the batch it falls in).
template <int kMode, int kZrB, int kThr>
__global__ void __launch_bounds__(kThr) k_z_rows_cta(const int* stop, int64_t q0, int64_t q1, int64_t nc,
                                                     const double* __restrict__ Z, const int32_t* __restrict__ rows,
                                                     const double* __restrict__ e, double* __restrict__ x, Xchg xc) {
  if (*stop) return;
  constexpr int kW = kThr / 32;
  __shared__ double red[kW][kZrB];
  unsigned long long ep = 0;
  if (kMode == 2) ep = xepoch(xc);
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t nb = (q1 - q0 + kZrB - 1) / kZrB;
  for (int64_t bt = blockIdx.x; bt < nb; bt += gridDim.x) {
    const int64_t qb = q0 + bt * kZrB;
    const int nr = (int)min((int64_t)kZrB, q1 - qb);
    double acc[kZrB];
#pragma unroll
    for (int r = 0; r < kZrB; ++r) acc[r] = 0.0;
    for (int64_t c = 2 * t; c + 1 < nc; c += 2 * kThr) {
      const double2 ev = *reinterpret_cast<const double2*>(e + c);
      double2 z[kZrB];
#pragma unroll
      for (int r = 0; r < kZrB; ++r) {
        const int64_t off = (qb + r) * nc + c;
        z[r] = r < nr ? ld_z2(Z + off, (off & 1) == 0) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int r = 0; r < kZrB; ++r) acc[r] = fma(z[r].x, ev.x, fma(z[r].y, ev.y, acc[r]));
    }
    if ((nc & 1) && t == ((nc - 1) % (2 * kThr)) / 2) {
      const int64_t c = nc - 1;
#pragma unroll
      for (int r = 0; r < kZrB; ++r)
        if (r < nr) acc[r] = fma(Z[(qb + r) * nc + c], e[c], acc[r]);
    }
#pragma unroll
    for (int r = 0; r < kZrB; ++r) {
      double v = acc[r];
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[w][r] = v;
    }
    __syncthreads();
    if (t < nr) {
      double v = 0.0;
      for (int k = 0; k < kW; ++k) v += red[k][t];
      const int64_t q = qb + t;
      if (kMode == 2) {
        for (int r = 0; r < xc.nranks; ++r) xarea(xc, r, ep + 1)[q] = v;
      } else if (kMode == 1) {
        x[q] = v;
      } else {
        x[rows[q]] -= v;
      }
    }
    __syncthreads();
  }
  if (kMode == 2) xsignal(xc, ep);
}

// Restriction, dense part: partial[ch][c] = sum_{q in chunk ch} Z[q, c] r[rows[q]]
// for chunks [ch0, ch0 + gridDim.y).  CTA = (256 * kCpt-column tile, row
// chunk); kCpt contiguous columns per thread (kCpt/2 16-byte loads per row),
// kRif rows in flight.  Every column's fma chain runs over the chunk's rows
// in ascending order whatever kCpt / kRif are, so the variants agree bit for
// bit.  kZtCols is the tile width the chunk plan assumes (dist.py mirrors it).
constexpr int kZtCols = 1024;

template <int kCpt, int kRif>
__global__ void __launch_bounds__(256) k_zt_partial(const int* stop, int64_t nG, int64_t nc, int64_t chunk,
                                                    int64_t ch0, const double* __restrict__ Z,
                                                    const int32_t* __restrict__ rows, const double* __restrict__ r,
                                                    double* __restrict__ partial) {
  if (*stop) return;
  extern __shared__ double rv[];
  const int64_t ch = ch0 + blockIdx.y;
  const int64_t q0 = ch * chunk, q1 = min(nG, q0 + chunk);
  for (int64_t q = q0 + threadIdx.x; q < q1; q += blockDim.x) rv[q - q0] = r[rows[q]];
  __syncthreads();
  const int64_t c = (int64_t)blockIdx.x * (256 * kCpt) + kCpt * threadIdx.x;
  if (c >= nc) return;
  double a[kCpt];
#pragma unroll
  for (int j = 0; j < kCpt; ++j) a[j] = 0.0;
  if (c + kCpt - 1 < nc && (nc & 1) == 0) {
    int64_t q = q0;
    for (; q + kRif - 1 < q1; q += kRif) {
      double2 u[kRif][kCpt / 2];
#pragma unroll
      for (int k = 0; k < kRif; ++k)
#pragma unroll
        for (int j = 0; j < kCpt / 2; ++j) u[k][j] = __ldcs(reinterpret_cast<const double2*>(Z + (q + k) * nc + c + 2 * j));
#pragma unroll
      for (int k = 0; k < kRif; ++k) {
        const double sk = rv[q + k - q0];
#pragma unroll
        for (int j = 0; j < kCpt / 2; ++j) {
          a[2 * j] = fma(u[k][j].x, sk, a[2 * j]);
          a[2 * j + 1] = fma(u[k][j].y, sk, a[2 * j + 1]);
        }
      }
    }
    for (; q < q1; ++q) {
      const double s0 = rv[q - q0];
#pragma unroll
      for (int j = 0; j < kCpt; ++j) a[j] = fma(Z[q * nc + c + j], s0, a[j]);
    }
    double* o = partial + ch * nc + c;
#pragma unroll
    for (int j = 0; j < kCpt; ++j) o[j] = a[j];
  } else {
    for (int t = 0; t < kCpt && c + t < nc; ++t) {
      double acc = 0.0;
      for (int64_t q = q0; q < q1; ++q) acc = fma(Z[q * nc + c + t], rv[q - q0], acc);
      partial[ch * nc + c + t] = acc;
    }
  }
}

// launch the partials of chunks [c0, c1)
static void launch_zt_partial(const int* stop, const HybridP& hp, int64_t c0, int64_t c1, const double* r,
                              cudaStream_t s) {
  if (c1 <= c0) return;
  // 4 columns x 4 rows in flight per thread; measured on config 2 against
  // 2/8/16 columns and 2/8 rows: wider tiles are slower, the rest equal
  constexpr int kCpt = 4;
  const unsigned tiles = (unsigned)((hp.nc + 256 * kCpt - 1) / (256 * kCpt));
  k_zt_partial<kCpt, 4><<<dim3(tiles, (unsigned)(c1 - c0)), 256, sizeof(double) * hp.chunk, s>>>(
      stop, hp.nG, hp.nc, hp.chunk, c0, hp.Z.p, hp.rows.p, r, hp.partial.p);
  HC_CHECK_LAUNCH();
}

struct GrpBounds {
  int64_t b[kGroups + 1];
};

// bc[c] -= sum_g (sum_{ch in group g} partial[ch][c])  -- the same two-level
// order as the distributed group sums (dist.cu), hence bit-identical to them.
// CTA = 32 columns x kGroups warps: warp g sums group g, warp 0 folds.
__global__ void __launch_bounds__(32 * kGroups) k_zt_reduce(const int* stop, int64_t nc,
                                                            const double* __restrict__ partial, GrpBounds grp,
                                                            double* __restrict__ bc) {
  if (*stop) return;
  __shared__ double gs[kGroups][32];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t c = (int64_t)blockIdx.x * 32 + lane;
  double acc = 0.0;
  if (c < nc)
    for (int64_t ch = grp.b[g]; ch < grp.b[g + 1]; ++ch) acc += partial[ch * nc + c];
  gs[g][lane] = acc;
  __syncthreads();
  if (g == 0 && c < nc) {
    double t = 0.0;
    for (int k = 0; k < kGroups; ++k) t += gs[k][lane];
    bc[c] -= t;
  }
}

// ---- Galerkin helpers

// Y = A_GG Z (row-major), one CTA per output row, threads over columns
__global__ void __launch_bounds__(256) k_spmm_rows(const int64_t* __restrict__ ap, const int32_t* __restrict__ ai,
                                                   const double* __restrict__ av, int64_t n, int64_t nc,
                                                   const double* __restrict__ Z, double* __restrict__ Y) {
  for (int64_t q = blockIdx.x; q < n; q += gridDim.x) {
    for (int64_t c = threadIdx.x; c < nc; c += blockDim.x) {
      double acc = 0.0;
      for (int64_t e = ap[q]; e < ap[q + 1]; ++e) acc = fma(av[e], Z[(int64_t)ai[e] * nc + c], acc);
      Y[q * nc + c] = -acc;  // rho = W' - A_GG Z: start from -A_GG Z
    }
  }
}

__global__ void k_add_csr_dense(const int64_t* __restrict__ wp, const int32_t* __restrict__ wi,
                                const double* __restrict__ wv, int64_t n, int64_t nc, double* __restrict__ Y) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    for (int64_t e = wp[q]; e < wp[q + 1]; ++e) Y[q * nc + wi[e]] += wv[e];
}

// D1[:, c] = sum_q W'[q, c] Z[q, :]  (column-major nc x nc; W'^T given as CSR rows c)
__global__ void __launch_bounds__(256) k_zt_w(const int64_t* __restrict__ tp, const int32_t* __restrict__ ti,
                                              const double* __restrict__ tv, int64_t nc, const double* __restrict__ Z,
                                              double* __restrict__ D1) {
  for (int64_t c = blockIdx.x; c < nc; c += gridDim.x) {
    for (int64_t a = threadIdx.x; a < nc; a += blockDim.x) {
      double acc = 0.0;
      for (int64_t e = tp[c]; e < tp[c + 1]; ++e) acc = fma(tv[e], Z[(int64_t)ti[e] * nc + a], acc);
      D1[a + c * nc] = acc;
    }
  }
}

// Ac = -0.5 (D1 + D1^T) - 0.5 (E + E^T)  (exactly symmetric by construction)
__global__ void k_combine(int64_t nc, const double* __restrict__ D1, const double* __restrict__ E,
                          double* __restrict__ Ac) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nc * nc; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = t % nc, c = t / nc;
    const double d = D1[a + c * nc] + D1[c + a * nc];
    const double e = E[a + c * nc] + E[c + a * nc];
    Ac[t] = -0.5 * d - 0.5 * e;
  }
}

__global__ void k_add_sym_csr(const int64_t* __restrict__ sp, const int32_t* __restrict__ si,
                              const double* __restrict__ sv, int64_t nc, double* __restrict__ Ac) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < nc; a += (int64_t)gridDim.x * blockDim.x)
    for (int64_t e = sp[a]; e < sp[a + 1]; ++e) Ac[a + (int64_t)si[e] * nc] += sv[e];
}

template <bool kWrite>
__global__ void k_dense_to_csr(int64_t nc, const double* __restrict__ D, int64_t* __restrict__ cnt,
                               const int64_t* __restrict__ op, int32_t* __restrict__ oi, double* __restrict__ ov) {
  // row a of a column-major symmetric matrix = column a
  for (int64_t a = blockIdx.x; a < nc; a += gridDim.x) {
    __shared__ int64_t base;
    if (threadIdx.x == 0) base = 0;
    __syncthreads();
    int64_t out0 = kWrite ? op[a] : 0;
    for (int64_t c0 = 0; c0 < nc; c0 += blockDim.x) {
      const int64_t c = c0 + threadIdx.x;
      const double v = c < nc ? D[c + a * nc] : 0.0;
      const bool nz = c < nc && v != 0.0;
      // block-wide ordered compaction
      __shared__ int wsum[32];
      const unsigned m = __ballot_sync(0xffffffffu, nz);
      const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
      if (lane == 0) wsum[w] = __popc(m);
      __syncthreads();
      int before = 0;
      for (int k = 0; k < w; ++k) before += wsum[k];
      int total = 0;
      for (int k = 0; k < (int)(blockDim.x >> 5); ++k) total += wsum[k];
      if (kWrite && nz) {
        const int64_t pos = out0 + base + before + __popc(m & ((1u << lane) - 1u));
        oi[pos] = (int32_t)c;
        ov[pos] = v;
      }
      __syncthreads();
      if (threadIdx.x == 0) base += total;
      __syncthreads();
    }
    if (!kWrite && threadIdx.x == 0) cnt[a] = base;
    __syncthreads();
  }
}

template <bool kWrite>
__global__ void k_hybrid_csr(int64_t n, const int64_t* __restrict__ pp, const int32_t* __restrict__ pi,
                             const double* __restrict__ pv, const int32_t* __restrict__ rowmap, int64_t nc,
                             const double* __restrict__ Z, int64_t* __restrict__ cnt, const int64_t* __restrict__ op,
                             int32_t* __restrict__ oi, double* __restrict__ ov) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
    int64_t c_ = 0, o = kWrite ? op[u] : 0;
    for (int64_t e = pp[u]; e < pp[u + 1]; ++e) {
      if (kWrite) { oi[o + c_] = pi[e]; ov[o + c_] = pv[e]; }
      ++c_;
    }
    const int32_t q = rowmap[u];
    if (q >= 0) {
      for (int64_t c = 0; c < nc; ++c) {
        const double z = Z[(int64_t)q * nc + c];
        if (z != 0.0) {
          if (kWrite) { oi[o + c_] = (int32_t)c; ov[o + c_] = -z; }
          ++c_;
        }
      }
    }
    if (!kWrite) cnt[u] = c_;
  }
}

__global__ void k_rowmap(const int32_t* __restrict__ rows, int64_t nG, int32_t* __restrict__ map) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nG; q += (int64_t)gridDim.x * blockDim.x)
    map[rows[q]] = (int32_t)q;
}

__global__ void k_fill_m1(int32_t* v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) v[i] = -1;
}

constexpr int64_t kSB = kTriSB;  // sweep block (half a factor tile)

// dst[z] (SB x SB, ld SB) = src[z]^T, src[z] an SB x SB column-major block with
// leading dimension lds (32 x 32 sub-blocks through shared memory)
__global__ void __launch_bounds__(256) k_blocks_transpose(const double* const* __restrict__ src, int64_t lds,
                                                          double* const* __restrict__ dst) {
  __shared__ double sm[32][33];
  const double* S = src[blockIdx.z];
  double* D = dst[blockIdx.z];
  const int64_t bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += 8) sm[j][threadIdx.x] = S[(bx + threadIdx.x) + (by + j) * lds];
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += 8) D[(by + threadIdx.x) + (bx + j) * kSB] = sm[threadIdx.x][j];
}


// Per row of each source block (SB rows of SB doubles at p + r ld): the
// 64-column chunk range [j0, j1) holding its nonzeros (0, 0 when empty).
__global__ void __launch_bounds__(1024) k_block_ranges(const TriSrc* __restrict__ blocks, uint8_t* __restrict__ out) {
  const TriSrc B = blocks[blockIdx.x];
  const int lane = threadIdx.x & 31;
  for (int r = threadIdx.x >> 5; r < kSB; r += 32) {
    const double* row = B.p + (int64_t)r * B.ld;
    unsigned m = 0;
    for (int j = 0; j < kSB / 64; ++j) {
      const double2 v = *reinterpret_cast<const double2*>(row + 64 * j + 2 * lane);
      if (__any_sync(0xffffffffu, v.x != 0.0 || v.y != 0.0)) m |= 1u << j;
    }
    if (lane == 0) {
      uint8_t* o = out + ((int64_t)blockIdx.x * kSB + r) * 2;
      o[0] = m ? (uint8_t)(__ffs(m) - 1) : 0;
      o[1] = m ? (uint8_t)(32 - __clz(m)) : 0;
    }
  }
}

// dst[z] (an NB x NB quadrant of an SB-wide column-major block) = src[z] (an NB x NB tile)
__global__ void __launch_bounds__(256) k_tile_into_block(const double* const* __restrict__ src,
                                                         double* const* __restrict__ dst) {
  const double* S = src[blockIdx.z];
  double* D = dst[blockIdx.z];
  const int64_t bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += 8) D[(bx + threadIdx.x) + (by + j) * kSB] = S[(bx + threadIdx.x) + (by + j) * kNB];
}

// identity NB x NB quadrant of an SB-wide column-major block (padding past the last tile)
__global__ void k_tile_eye_in_block(double* const* __restrict__ dst) {
  double* D = dst[blockIdx.y];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < kNB; t += (int64_t)gridDim.x * blockDim.x)
    D[t + t * kSB] = 1.0;
}

void blocks_transpose(std::vector<const double*>& src, int64_t lds, std::vector<double*>& dst, cudaStream_t s) {
  for (size_t z0 = 0; z0 < src.size(); z0 += 32768) {
    const size_t nz = std::min<size_t>(32768, src.size() - z0);
    DBuf<const double*> ds;
    DBuf<double*> dd;
    ds.upload(src.data() + z0, (int64_t)nz, s);
    dd.upload(dst.data() + z0, (int64_t)nz, s);
    k_blocks_transpose<<<dim3(kSB / 32, kSB / 32, (unsigned)nz), dim3(32, 8), 0, s>>>(ds.p, lds, dd.p);
    HC_CHECK_LAUNCH();
    HC_CUDA(cudaStreamSynchronize(s));
  }
}

// Operators of the blocked sweeps (trisolve.cuh) from the envelope factor, on
// sweep blocks of SB rows (SB = NB, or NB / 2 for twice the steps with half
// the rows each -- measured slower: the per-step synchronisation dominates).
// Sub-block (I, J) of L is rows (I%SP) SB.., cols (J%SP) SB.. of tile
// (I/SP, J/SP) (column-major, ld NB); above-diagonal sub-blocks of a diagonal
// tile are not part of L.  Linv_II = L_II^{-1} (TRSM on identity blocks), M_I = Linv_II
// L_{I,I-1}, N_I = Linv_II^T L_{I+1,I}^T, forward folds L_{i,I-1} copied
// row-major; the backward folds are columns of L, read in place.
void build_factor_ops(const Packed& L, FactorP& f, cudaStream_t s) {
  StageTimer stf(s);
  // SP sweep blocks per factor tile (SB <= NB) or Q factor tiles per sweep block (SB = Q NB)
  constexpr int64_t SP = kSB <= kNB ? kNB / kSB : 1, Q = kSB > kNB ? kSB / kNB : 1;
  static_assert(SP * kSB == kNB || Q * kNB == kSB, "sweep block and factor tile must nest");
  const int64_t T = L.T, TS = Q > 1 ? (T + Q - 1) / Q : SP * T, SS = kSB * kSB;
  auto tile_ok = [&](int64_t I, int64_t J) { return I < T && J < T && J <= I && L.has(I, J); };
  auto valid = [&](int64_t I, int64_t J) {
    if (J > I) return false;
    if (Q > 1) {
      for (int64_t a = 0; a < Q; ++a)
        for (int64_t b = 0; b < Q; ++b)
          if (Q * J + b <= Q * I + a && tile_ok(Q * I + a, Q * J + b)) return true;
      return I == J;  // (a virtual identity diagonal block past the last tile)
    }
    const int64_t K = I / SP, Jt = J / SP;
    return L.has(K, Jt) && !(K == Jt && (I % SP) < (J % SP));
  };
  // SB = Q NB: the sweep blocks of L are assembled into dense column-major
  // SB x SB slots (missing tiles zero, blocks above the diagonal dropped, an
  // identity past the last tile); SB <= NB: they are views into the tiles
  std::vector<int64_t> lslot((size_t)(TS * TS), -1);
  int64_t nL = 0;
  if (Q > 1)
    for (int64_t I = 0; I < TS; ++I)
      for (int64_t J = 0; J <= I; ++J)
        if (valid(I, J)) lslot[(size_t)(I * TS + J)] = nL++;
  DBuf<double> Lsb(std::max<int64_t>(nL, 1) * SS, s);
  if (Q > 1) {
    Lsb.zero();
    std::vector<const double*> src;
    std::vector<double*> dst;
    std::vector<double*> eye;
    for (int64_t I = 0; I < TS; ++I)
      for (int64_t J = 0; J <= I; ++J) {
        const int64_t sl = lslot[(size_t)(I * TS + J)];
        if (sl < 0) continue;
        for (int64_t a = 0; a < Q; ++a)
          for (int64_t b = 0; b < Q; ++b) {
            double* d = Lsb.p + sl * SS + (b * kNB) * kSB + a * kNB;
            if (Q * J + b <= Q * I + a && tile_ok(Q * I + a, Q * J + b)) {
              src.push_back(L.tile(Q * I + a, Q * J + b));
              dst.push_back(d);
            } else if (I == J && a == b && Q * I + a >= T) {
              eye.push_back(d);
            }
          }
      }
    for (size_t z0 = 0; z0 < src.size(); z0 += 32768) {  // NB x NB tile copies into the SB-wide slots
      const size_t nz = std::min<size_t>(32768, src.size() - z0);
      DBuf<const double*> ds;
      DBuf<double*> dd;
      ds.upload(src.data() + z0, (int64_t)nz, s);
      dd.upload(dst.data() + z0, (int64_t)nz, s);
      k_tile_into_block<<<dim3(kNB / 32, kNB / 32, (unsigned)nz), dim3(32, 8), 0, s>>>(ds.p, dd.p);
      HC_CHECK_LAUNCH();
      HC_CUDA(cudaStreamSynchronize(s));
    }
    if (!eye.empty()) {
      DBuf<double*> de;
      de.upload(eye.data(), (int64_t)eye.size(), s);
      k_tile_eye_in_block<<<dim3(64, (unsigned)eye.size()), 256, 0, s>>>(de.p);
      HC_CHECK_LAUNCH();
      HC_CUDA(cudaStreamSynchronize(s));
    }
  }
  stf.mark("    ops: blocks of L");
  const int64_t LDS = Q > 1 ? kSB : kNB;  // leading dimension of the blocks of L
  auto sub = [&](int64_t I, int64_t J) -> double* {  // column-major, ld LDS
    if (Q > 1) return Lsb.p + lslot[(size_t)(I * TS + J)] * SS;
    return L.tile(I / SP, J / SP) + (J % SP) * kSB * kNB + (I % SP) * kSB;
  };
  std::vector<int64_t> mslot((size_t)TS, -1), nslot((size_t)TS, -1);
  int64_t nM = 0, nN = 0;
  for (int64_t I = 1; I < TS; ++I)
    if (valid(I, I - 1)) mslot[(size_t)I] = nM++;
  for (int64_t I = 0; I + 1 < TS; ++I)
    if (valid(I + 1, I)) nslot[(size_t)I] = nN++;
  std::vector<std::vector<int64_t>> ffold((size_t)TS);
  int64_t nF = 0;
  for (int64_t I = 1; I < TS; ++I)
    for (int64_t i = I + 1; i < TS; ++i)
      if (valid(i, I - 1)) {
        ffold[(size_t)I].push_back(i);
        ++nF;
      }
  // fpool: Linv_II row-major (TS), M_I (nM), forward folds (nF); bpool:
  // Linv_II column-major = Linv^T row-major (TS), N_I (nN)
  DBuf<double> fpool((TS + nM + nF) * SS, s), bpool((TS + nN) * SS, s);
  auto fp = [&](int64_t slot) { return fpool.p + slot * SS; };
  auto bp = [&](int64_t slot) { return bpool.p + slot * SS; };
  {
    {  // Linv_II of every block in one level-synchronous batch
      std::vector<const double*> hl;
      std::vector<double*> hi;
      for (int64_t I = 0; I < TS; ++I) {
        hl.push_back(sub(I, I));
        hi.push_back(bp(I));
      }
      dblas::trtri_lower_many(kSB, hl, LDS, hi, kSB, s);
    }
    HC_CUDA(cudaStreamSynchronize(s));
    std::vector<const double*> src;
    std::vector<double*> dst;
    for (int64_t I = 0; I < TS; ++I) {
      src.push_back(bp(I));
      dst.push_back(fp(I));
    }
    blocks_transpose(src, kSB, dst, s);
  }
  stf.mark("    ops: Linv_II");
  auto batched_gemm = [&](dblas::Op ta, std::vector<const double*>& ha, std::vector<const double*>& hb,
                          std::vector<double*>& hc) {
    if (ha.empty()) return;
    DBuf<const double*> da, db;
    DBuf<double*> dc;
    da.upload(ha.data(), (int64_t)ha.size(), s);
    db.upload(hb.data(), (int64_t)hb.size(), s);
    dc.upload(hc.data(), (int64_t)hc.size(), s);
    dblas::gemm_batched(ta, ta, kSB, kSB, kSB, 1.0, da.p, LDS, db.p, kSB, 0.0, dc.p, kSB, (int64_t)ha.size(), s);
    HC_CUDA(cudaStreamSynchronize(s));
  };
  {  // row-major M_I = column-major (L_{I,I-1}^T Linv_II^T)
    std::vector<const double*> ha, hb;
    std::vector<double*> hc;
    for (int64_t I = 1; I < TS; ++I)
      if (mslot[(size_t)I] >= 0) {
        ha.push_back(sub(I, I - 1));
        hb.push_back(bp(I));
        hc.push_back(fp(TS + mslot[(size_t)I]));
      }
    batched_gemm(dblas::T, ha, hb, hc);
  }
  {  // row-major N_I = column-major (L_{I+1,I} Linv_II)
    std::vector<const double*> ha, hb;
    std::vector<double*> hc;
    for (int64_t I = 0; I + 1 < TS; ++I)
      if (nslot[(size_t)I] >= 0) {
        ha.push_back(sub(I + 1, I));
        hb.push_back(bp(I));
        hc.push_back(bp(TS + nslot[(size_t)I]));
      }
    batched_gemm(dblas::N, ha, hb, hc);
  }
  std::vector<TriSrcStep> fs, bs;
  {
    std::vector<const double*> src;
    std::vector<double*> dst;
    int64_t slot = TS + nM;
    for (int64_t I = 0; I < TS; ++I) {
      TriSrcStep S;
      S.k = (int32_t)I;
      S.c = I >= 1 ? (int32_t)(I - 1) : -1;
      S.a.p = fp(I);
      S.a.ld = kSB;
      if (mslot[(size_t)I] >= 0) {
        S.b.p = fp(TS + mslot[(size_t)I]);
        S.b.ld = kSB;
      }
      for (int64_t i : ffold[(size_t)I]) {
        src.push_back(sub(i, I - 1));
        dst.push_back(fp(slot));
        TriSrc fo;
        fo.p = fp(slot);
        fo.ld = kSB;
        S.folds.emplace_back(fo, i);
        ++slot;
      }
      fs.push_back(std::move(S));
    }
    if (!src.empty()) blocks_transpose(src, LDS, dst, s);
  }
  for (int64_t I = TS - 1; I >= 0; --I) {
    TriSrcStep S;
    S.k = (int32_t)I;
    S.c = I + 1 < TS ? (int32_t)(I + 1) : -1;
    S.a.p = bp(I);
    S.a.ld = kSB;
    if (nslot[(size_t)I] >= 0) {
      S.b.p = bp(TS + nslot[(size_t)I]);
      S.b.ld = kSB;
    }
    if (I + 1 < TS)  // rows of L_{I+1,j}^T = columns of the column-major block (stride LDS)
      for (int64_t j = 0; j < I; ++j)
        if (valid(I + 1, j)) {
          TriSrc fo;
          fo.p = sub(I + 1, j);
          fo.ld = LDS;
          S.folds.emplace_back(fo, j);
        }
    bs.push_back(std::move(S));
  }
  // row ranges of every source block (data final), host copies for the compaction
  std::vector<TriSrc> blocks;
  std::unordered_map<const double*, size_t> index;
  auto add = [&](const TriSrc& b) {
    if (b.p && index.emplace(b.p, blocks.size()).second) blocks.push_back(b);
  };
  for (int d = 0; d < 2; ++d)
    for (const TriSrcStep& S : d == 0 ? fs : bs) {
      add(S.a);
      add(S.b);
      for (const auto& fo : S.folds) add(fo.first);
    }
  DBuf<TriSrc> dblocks;
  dblocks.upload(blocks.data(), (int64_t)blocks.size(), s);
  DBuf<uint8_t> rng((int64_t)blocks.size() * kSB * 2, s);
  for (size_t z0 = 0; z0 < blocks.size(); z0 += 65535) {
    const size_t nz = std::min<size_t>(65535, blocks.size() - z0);
    k_block_ranges<<<(unsigned)nz, 1024, 0, s>>>(dblocks.p + z0, rng.p + z0 * kSB * 2);
    HC_CHECK_LAUNCH();
  }
  const std::vector<uint8_t> hr = rng.download();
  auto ranges = [&](const double* p) -> const uint8_t* { return hr.data() + index.at(p) * kSB * 2; };
  stf.mark("    ops: M, N, folds, ranges");
  tri_compact(fs, ranges, f.fw, s, 0);
  tri_compact(bs, ranges, f.bw, s, 1);
  stf.mark("    ops: compact + partition");
  if (getenv("HCAMG_SETUP_TIMING"))
    fprintf(stderr, "[hcamg setup]   sweeps: %lld blocks of %lld rows, fwd %.3f GB, bwd %.3f GB\n", (long long)TS,
            (long long)kSB, f.fw.bytes / 1e9, f.bw.bytes / 1e9);
}

}  // namespace

// Reverse Cuthill-McKee order of a symmetric pattern: scipy's algorithm
// (csgraph reverse_cuthill_mckee, the ordering the reference's cholesky()
// applies before factoring, sparse.py:297): degree = row length (+1 when the
// diagonal is stored); seeds by increasing degree; BFS by levels, each node's
// unvisited neighbours appended in column order and insertion-sorted by
// degree; the final order reversed.  Seed ties are taken by lowest index
// (scipy's argsort is not stable, so its tie choice is platform dependent).
std::vector<int32_t> rcm_order(int64_t n, const std::vector<int64_t>& ptr, const std::vector<int32_t>& idx) {
  std::vector<int64_t> deg((size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    deg[(size_t)i] = ptr[(size_t)i + 1] - ptr[(size_t)i];
    for (int64_t e = ptr[(size_t)i]; e < ptr[(size_t)i + 1]; ++e)
      if (idx[(size_t)e] == i) {
        ++deg[(size_t)i];
        break;
      }
  }
  std::vector<int32_t> seeds((size_t)n);
  for (int64_t i = 0; i < n; ++i) seeds[(size_t)i] = (int32_t)i;
  std::stable_sort(seeds.begin(), seeds.end(), [&](int32_t a, int32_t b) { return deg[(size_t)a] < deg[(size_t)b]; });
  std::vector<char> seen((size_t)n, 0);
  std::vector<int32_t> order;
  order.reserve((size_t)n);
  for (int64_t zz = 0; zz < n && (int64_t)order.size() < n; ++zz) {
    const int32_t seed = seeds[(size_t)zz];
    if (seen[(size_t)seed]) continue;
    seen[(size_t)seed] = 1;
    order.push_back(seed);
    size_t lo = order.size() - 1, hi = order.size();
    while (lo < hi) {
      for (size_t ii = lo; ii < hi; ++ii) {
        const int32_t i = order[ii];
        const size_t n_old = order.size();
        for (int64_t e = ptr[(size_t)i]; e < ptr[(size_t)i + 1]; ++e) {
          const int32_t j = idx[(size_t)e];
          if (!seen[(size_t)j]) {
            seen[(size_t)j] = 1;
            order.push_back(j);
          }
        }
        for (size_t k = n_old + 1; k < order.size(); ++k) {  // stable insertion sort by degree
          const int32_t v = order[k];
          size_t l = k;
          while (l > n_old && deg[(size_t)v] < deg[(size_t)order[l - 1]]) {
            order[l] = order[l - 1];
            --l;
          }
          order[l] = v;
        }
      }
      lo = hi;
      hi = order.size();
    }
  }
  std::reverse(order.begin(), order.end());
  return order;
}

namespace {
// D[colperm[i], colperm[j]] = lower(Dp)[max(i,j), min(i,j)]  (column-major m x m)
__global__ void k_unperm_sym(int64_t m, const int32_t* __restrict__ colperm, const double* __restrict__ Dp,
                             double* __restrict__ D) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m * m; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % m, j = t / m;
    const double v = i >= j ? Dp[i + j * m] : Dp[j + i * m];
    D[(int64_t)colperm[i] + (int64_t)colperm[j] * m] = v;
  }
}
}  // namespace

void giant_factor_solve(const DCsr& Agg, double* B, int64_t m, cudaStream_t s, FactorP* fac, double* D,
                        bool want_z, const DCsr* Bs) {
  const int64_t n = Agg.nrows;
  const bool sparse_rhs = Bs != nullptr && !want_z;
  require(sparse_rhs || B != nullptr, "giant_factor_solve: no right-hand side");
  if (sparse_rhs) require(Bs->nrows == n && Bs->ncols == m, "giant_factor_solve: sparse right-hand side shape");
  StageTimer st(s);
  // ordering: reverse Cuthill-McKee (default) or the natural component order
  std::vector<int64_t> hptr = Agg.ptr.download();
  std::vector<int32_t> hidx = Agg.idx.download();
  std::vector<int32_t> perm;
  const char* ord = getenv("HCAMG_GIANT_ORDER");
  if (ord && std::string(ord) == "natural") {
    perm.resize((size_t)n);
    for (int64_t i = 0; i < n; ++i) perm[(size_t)i] = (int32_t)i;
  } else {
    perm = rcm_order(n, hptr, hidx);
  }
  std::vector<int32_t> inv((size_t)n);
  for (int64_t i = 0; i < n; ++i) inv[(size_t)perm[(size_t)i]] = (int32_t)i;
  DBuf<int32_t> dperm, dinv;
  dperm.upload(perm.data(), n);
  dinv.upload(inv.data(), n);
  DCsr Ap;
  csr_extract(Agg, dperm.p, n, dinv.p, n, Ap, s);
  // block envelope
  Packed L;
  L.n = n;
  L.T = (n + kNB - 1) / kNB;
  const int64_t T = L.T;
  L.j0.assign((size_t)T, 0);
  for (int64_t I = 0; I < T; ++I) L.j0[(size_t)I] = I;
  for (int64_t i = 0; i < n; ++i) {
    int64_t f = i;
    const int32_t r = perm[(size_t)i];
    for (int64_t e = hptr[(size_t)r]; e < hptr[(size_t)r + 1]; ++e) f = std::min<int64_t>(f, inv[(size_t)hidx[(size_t)e]]);
    int64_t& j0 = L.j0[(size_t)(i / kNB)];
    j0 = std::min(j0, f / kNB);
  }
  L.off.assign((size_t)T + 1, 0);
  for (int64_t I = 0; I < T; ++I) L.off[(size_t)I + 1] = L.off[(size_t)I] + (I - L.j0[(size_t)I] + 1);
  const int64_t ntiles = L.off[(size_t)T];
  st.mark("  giant: order + envelope");
  L.buf.alloc(ntiles * kNB * kNB, s);
  L.buf.zero();
  {
    DBuf<int64_t> dj0, doff;
    dj0.upload(L.j0.data(), T);
    doff.upload(L.off.data(), T + 1);
    k_pack_env<<<grid_for(T * kNB, 256), 256, 0, s>>>(Ap.ptr.p, Ap.idx.p, Ap.val.p, n, T, dj0.p, doff.p, L.buf.p);
    HC_CHECK_LAUNCH();
    HC_CUDA(cudaStreamSynchronize(s));
  }
  DBuf<unsigned long long> mx(1, s);
  mx.zero();
  k_csr_diag_absmax<<<grid_for(n, 256), 256, 0, s>>>(Agg.ptr.p, Agg.idx.p, Agg.val.p, n, mx.p);
  HC_CHECK_LAUNCH();
  unsigned long long hm = read_scalar(mx.p, s);
  double scale;
  memcpy(&scale, &hm, 8);
  DBuf<double> piv(T * kNB, s);
  DBuf<const double*> dA, dB;
  DBuf<const double*> dC;
  DBuf<long long> badf(1, s);
  badf.fill_bytes(0xff);
  // the inverse of every diagonal tile is kept: the forward solve of the
  // right-hand sides below applies it as one product per block column (the
  // recursive triangular solve inverted its 64 x 64 leaves again for each,
  // 2,600 single-CTA launches of 77 us)
  DBuf<double> LinvAll(T * kNB * kNB, s);
  LinvAll.zero();
  // HCAMG_SETUP_TIMING: per-phase totals of the factorisation loop (synchronises after every phase)
  double tphase[3] = {0, 0, 0};
  auto phase = [&](int which, std::chrono::steady_clock::time_point& t0) {
    if (!st.on) return;
    cudaStreamSynchronize(s);
    const auto t1 = std::chrono::steady_clock::now();
    tphase[which] += std::chrono::duration<double>(t1 - t0).count();
    t0 = t1;
  };
  for (int64_t K = 0; K < T; ++K) {  // right-looking, inside the envelope; no host sync until the end
    auto t0 = std::chrono::steady_clock::now();
    double* LinvKK = LinvAll.p + K * kNB * kNB;
    dense_cholesky_inv_async(L.tile(K, K), kNB, kNB, LinvKK, kNB, piv.p + K * kNB, badf.p, K * kNB, s);
    phase(0, t0);
    std::vector<int64_t> below;  // block rows I > K whose envelope reaches column K
    for (int64_t I = K + 1; I < T; ++I)
      if (L.has(I, K)) below.push_back(I);
    if (below.empty()) continue;
    {  // L_IK = A_IK L_KK^{-T} with the inverse the diagonal factorisation produced
      std::vector<double*> hb;
      for (int64_t I : below) hb.push_back(L.tile(I, K));
      dblas::apply_rinv_t_batched(kNB, kNB, LinvKK, hb, kNB, s);
    }
    phase(1, t0);
    {
      std::vector<const double*> ha, hb, hc;
      for (size_t a = 0; a < below.size(); ++a)
        for (size_t b = 0; b <= a; ++b) {  // (I, J) = (below[a], below[b]), J <= I, both reach K
          ha.push_back(L.tile(below[a], K));
          hb.push_back(L.tile(below[b], K));
          hc.push_back(L.tile(below[a], below[b]));
        }
      const double** pa = upload_ptrs(ha, dA, s);
      const double** pb = upload_ptrs(hb, dB, s);
      const double** pc = upload_ptrs(hc, dC, s);
      dblas::gemm_batched(dblas::N, dblas::T, kNB, kNB, kNB, -1.0, pa, kNB, pb, kNB, 1.0, (double* const*)pc, kNB,
                          (int64_t)ha.size(), s);
      // (pageable-host uploads are staged before cudaMemcpyAsync returns: no sync needed)
    }
    phase(2, t0);
  }
  if (st.on)
    fprintf(stderr, "[hcamg setup]   envelope Cholesky phases: potrf %.3f s, trsm %.3f s, gemm %.3f s (%lld block columns)\n",
            tphase[0], tphase[1], tphase[2], (long long)T);
  const long long badv = read_scalar(badf.p, s);
  const int64_t fail = badv >= 0 ? (int64_t)badv : -1;
  {
    // pivot indices are reported in the factored (permuted) order, as the
    // reference's cholesky() does for its RCM-permuted matrix
    std::vector<double> hp = piv.download();
    const int64_t j0 = fail >= 0 ? fail : n;
    const int64_t bad = pivot_verdict(hp, n, std::min(j0, n), scale);
    if (bad >= 0) throw Error(ENOTSPD_, "matrix is not positive definite (pivot " + std::to_string(bad) + ")", bad);
    if (fail >= 0) throw Error(ENOTSPD_, "matrix is not positive definite (pivot " + std::to_string(fail) + ")", fail);
  }
  st.mark("  giant: envelope Cholesky");
  if (fac) {
    build_factor_ops(L, *fac, s);
    fac->nG = n;
    fac->T = T;
    st.mark("  giant: sweep operators");
  }
  // Rows of B into the factored order; columns sorted by the first (factored)
  // row of their right-hand side, so that in the forward sweep block J only
  // involves the prefix of columns whose right-hand side starts at or above
  // block J -- the rest of the block is still zero (RCM keeps every coarse
  // DoF's coupling rows together, so this skips about half the forward work).
  std::vector<int32_t> colperm((size_t)m);
  std::vector<int64_t> active((size_t)T, m);
  {
    DBuf<int> first(m, s);
    HC_CUDA(cudaMemsetAsync(first.p, 0x7f, sizeof(int) * (size_t)m, s));
    if (sparse_rhs)
      k_first_row_csr<<<grid_for(n, 256), 256, 0, s>>>(n, Bs->ptr.p, Bs->idx.p, Bs->val.p, dinv.p, first.p);
    else
      k_first_row<<<(unsigned)std::min<int64_t>(n, kSMs * 16), 256, 0, s>>>(n, m, B, dinv.p, first.p);
    HC_CHECK_LAUNCH();
    st.mark("  giant: column order");
    std::vector<int> hf = first.download();
    for (int64_t c = 0; c < m; ++c) colperm[(size_t)c] = (int32_t)c;
    std::stable_sort(colperm.begin(), colperm.end(), [&](int32_t a, int32_t b) { return hf[(size_t)a] < hf[(size_t)b]; });
    int64_t k = 0;
    for (int64_t J = 0; J < T; ++J) {
      while (k < m && hf[(size_t)colperm[(size_t)k]] < (J + 1) * kNB) ++k;
      active[(size_t)J] = k;
    }
  }
  DBuf<int32_t> dcol;
  dcol.upload(colperm.data(), m);
  DBuf<double> Bp(n * m, s);
  if (sparse_rhs) {
    std::vector<int32_t> colinv((size_t)m);
    for (int64_t k = 0; k < m; ++k) colinv[(size_t)colperm[(size_t)k]] = (int32_t)k;
    DBuf<int32_t> dcinv;
    dcinv.upload(colinv.data(), m, s);
    Bp.zero();
    k_scatter_rc_csr<<<grid_for(n, 256), 256, 0, s>>>(n, m, Bs->ptr.p, Bs->idx.p, Bs->val.p, dinv.p, dcinv.p, Bp.p);
    HC_CHECK_LAUNCH();
    HC_CUDA(cudaStreamSynchronize(s));  // dcinv is a host-ordered upload: keep it alive until the kernel has run
  } else {
    permute_rc<false>(n, m, dperm.p, dcol.p, B, Bp.p, s);
  }
  st.mark("  giant: permute in");
  // Solve (A Z = B with B row-major n x m)  <=>  Z^T L L^T = B^T on the column-major m x n view.
  auto nbk = [&](int64_t K) { return std::min(kNB, n - K * kNB); };
  auto blk = [&](int64_t K) { return Bp.p + K * kNB * m; };
  DBuf<double> Xs(m * kNB, s);
  for (int64_t J = 0; J < T; ++J) {  // U^T = B^T L^{-T}; columns >= active[J] of blocks <= J are zero
    const int ma = (int)active[(size_t)J];
    if (ma == 0) continue;
    {  // blk(J) := blk(J) L_JJ^{-T} with the stored inverse (its leading nbk(J) block for a partial last tile)
      dblas::gemm_rinv_t(ma, nbk(J), blk(J), m, LinvAll.p + J * kNB * kNB, kNB, Xs.p, ma, s);
      dblas::copy_block(ma, nbk(J), Xs.p, ma, blk(J), m, s);
    }
    for (int64_t I = J + 1; I < T; ++I)
      if (L.has(I, J)) {
        dblas::gemm(dblas::N, dblas::T, ma, nbk(I), nbk(J), -1.0, blk(J), m, L.tile(I, J), kNB, 1.0, blk(I), m, s);
      }
  }
  st.mark("  giant: forward solve");
  if (D) {  // D = Y^T Y over the staircase: row block J of Y is zero beyond column active[J]
    DBuf<double> Dp(m * m, s);
    Dp.zero();
    for (int64_t J = 0; J < T; ++J) {
      const int ma = (int)active[(size_t)J];
      if (ma == 0) continue;
      dblas::syrk_ln(ma, nbk(J), 1.0, blk(J), m, 1.0, Dp.p, m, s);
    }
    k_unperm_sym<<<grid_for(m * m, 256, kSMs * 32), 256, 0, s>>>(m, dcol.p, Dp.p, D);
    HC_CHECK_LAUNCH();
    st.mark("  giant: Y^T Y");
  }
  if (!want_z) {
    L.buf.release();
    HC_CUDA(cudaStreamSynchronize(s));
    if (fac) fac->perm = std::move(dperm);
    return;
  }
  for (int64_t K = T - 1; K >= 0; --K) {  // Z^T = U^T L^{-1}
    dblas::trsm(dblas::Right, dblas::N, m, nbk(K), L.tile(K, K), kNB, blk(K), m, s);
    for (int64_t I = L.j0[(size_t)K]; I < K; ++I) {
      dblas::gemm(dblas::N, dblas::N, m, kNB, nbk(K), -1.0, blk(K), m, L.tile(K, I), kNB, 1.0, blk(I), m, s);
    }
  }
  st.mark("  giant: triangular solves");
  L.buf.release();
  permute_rc<true>(n, m, dperm.p, dcol.p, Bp.p, B, s);
  HC_CUDA(cudaStreamSynchronize(s));
  if (fac) fac->perm = std::move(dperm);
  st.mark("  giant: permute out");
}

template <int kMode>
static void launch_rows(const int* stop, int64_t q0, int64_t q1, int64_t nc, const double* Z, const int32_t* rows,
                        const double* e, double* x, const Xchg& xc, cudaStream_t s) {
  const bool smem = nc * 8 <= 200 * 1024;
  const int64_t nrows = std::max<int64_t>(q1 - q0, 0);
  static bool init = false;
  if (!init) {
    HC_CUDA(cudaFuncSetAttribute(k_z_rows<true, kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    init = true;
  }
  const char* zr = getenv("HCAMG_ZROWS");
  const int variant = zr ? atoi(zr) : 1;  // HCAMG_ZROWS=0: warp-per-row kernel (comparison)
  if (nc >= 4096 && variant > 0) {
    auto go = [&](auto kern, int rb, int thr) {
      int per_sm = 0;
      HC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, thr, 0));
      const int64_t nb = (nrows + rb - 1) / rb;
      const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nb, (int64_t)kSMs * std::max(per_sm, 1)));
      kern<<<g, thr, 0, s>>>(stop, q0, q1, nc, Z, rows, e, x, xc);
    };
    go(k_z_rows_cta<kMode, 16, 256>, 16, 256);  // measured best of 4..16 rows x 128..1024 threads
    HC_CHECK_LAUNCH();
    return;
  }
  // 16 warps per CTA, two rows per warp
  const int64_t ctas = std::max<int64_t>(1, (nrows + 31) / 32);
  if (smem) {
    // e staged once per CTA; as many 512-thread CTAs per SM as shared memory allows (<= 4)
    const int64_t per_sm = std::max<int64_t>(1, std::min<int64_t>(4, (220 * 1024) / std::max<int64_t>(8 * nc, 1)));
    const unsigned g = (unsigned)std::min<int64_t>(ctas, kSMs * per_sm);
    k_z_rows<true, kMode><<<g, 512, sizeof(double) * nc, s>>>(stop, q0, q1, nc, Z, rows, e, x, xc);
  } else {
    const unsigned g = (unsigned)std::min<int64_t>(ctas, kSMs * 4);
    k_z_rows<false, kMode><<<g, 512, 0, s>>>(stop, q0, q1, nc, Z, rows, e, x, xc);
  }
  HC_CHECK_LAUNCH();
}

static bool dist_on(const Dist* d) { return d && d->on; }

// rows [q0, q1) of Z owned by this rank: the rows of its chunk groups
static void rank_rows(const HybridP& hp, const Dist& d, int64_t& q0, int64_t& q1) {
  int g0, g1;
  rank_groups(d.rank, d.nranks, g0, g1);
  q0 = std::min(hp.nG, hp.grp[g0] * hp.chunk);
  q1 = std::min(hp.nG, hp.grp[g1] * hp.chunk);
}

void hybrid_prolong(const int* stop, const HybridP& hp, const double* e, double* x, cudaStream_t s, const Dist* d,
                    size_t off, int part) {
  if (!dist_on(d)) {
    if (part != 2) launch_rows<0>(stop, 0, hp.nG, hp.nc, hp.Z.p, hp.rows.p, e, x, Xchg{}, s);
    return;
  }
  const Xchg xc = d->site(off);
  if (part != 2) {
    int64_t q0, q1;
    rank_rows(hp, *d, q0, q1);
    launch_rows<2>(stop, q0, q1, hp.nc, hp.Z.p, hp.rows.p, e, nullptr, xc, s);
  }
  if (part != 1) xchg_scatter(stop, xc, hp.nG, hp.rows.p, x, s);
}

void dense_gemv_rows(const int* stop, int64_t n, int64_t m, const double* M, const double* e, double* x,
                     cudaStream_t s, const Dist* d, size_t off, int part) {
  if (!dist_on(d)) {
    if (part != 2) launch_rows<1>(stop, 0, n, m, M, nullptr, e, x, Xchg{}, s);
    return;
  }
  const Xchg xc = d->site(off);
  if (part != 2) {
    int64_t r0, r1;
    even_rows(n, d->rank, d->nranks, r0, r1);
    launch_rows<2>(stop, r0, r1, m, M, nullptr, e, nullptr, xc, s);
  }
  if (part != 1) xchg_scatter(stop, xc, n, nullptr, x, s);
}

namespace {
__global__ void k_rows_dense(const int64_t* __restrict__ wp, const int32_t* __restrict__ wi,
                             const double* __restrict__ wv, int64_t n, int64_t m, double* __restrict__ B) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    for (int64_t e = wp[t]; e < wp[t + 1]; ++e) B[t * m + wi[e]] = wv[e];
}
}  // namespace

void hybrid_ensure_z(HybridP& hp, cudaStream_t s) {
  if (!hp.on || hp.Z.p) return;
  require(hp.Agg.nrows == hp.nG && hp.Wg.nrows == hp.nG, "dense block data missing");
  hp.Z.alloc(hp.nG * hp.nc, s);
  hp.Z.zero();
  k_rows_dense<<<grid_for(hp.nG, 128), 128, 0, s>>>(hp.Wg.ptr.p, hp.Wg.idx.p, hp.Wg.val.p, hp.nG, hp.nc, hp.Z.p);
  HC_CHECK_LAUNCH();
  giant_factor_solve(hp.Agg, hp.Z.p, hp.nc, s, nullptr, nullptr, true);
  hybrid_prepare(hp, s);
}

void hybrid_prepare(HybridP& hp, cudaStream_t s) {
  // Row chunks, grouped into kGroups groups of whole chunks.  Enough chunks per
  // group that one group alone (one rank of eight) fills the GPU: ~4 CTAs
  // per SM over the column tiles.
  const int64_t ct = (hp.nc + kZtCols - 1) / kZtCols;
  const int64_t per_group = std::max<int64_t>(1, (4 * kSMs + ct - 1) / std::max<int64_t>(ct, 1));
  const int64_t want = kGroups * per_group;
  hp.chunk = std::max<int64_t>(16, std::min<int64_t>(4096, (hp.nG + want - 1) / want));
  hp.nchunk = (hp.nG + hp.chunk - 1) / hp.chunk;
  for (int g = 0; g <= kGroups; ++g) hp.grp[g] = hp.nchunk * g / kGroups;
  hp.partial.alloc(std::max<int64_t>(hp.nchunk * hp.nc, 1), s);
}

void hybrid_restrict(const int* stop, HybridP& hp, const double* r, double* bc, cudaStream_t s, const Dist* d,
                     size_t off, int part) {
  require(hp.nchunk > 0, "hybrid_restrict: plan not prepared");
  if (!dist_on(d)) {
    if (part == 2) return;
    launch_zt_partial(stop, hp, 0, hp.nchunk, r, s);
    GrpBounds g{};
    for (int t = 0; t <= kGroups; ++t) g.b[t] = hp.grp[t];
    k_zt_reduce<<<(unsigned)((hp.nc + 31) / 32), 32 * kGroups, 0, s>>>(stop, hp.nc, hp.partial.p, g, bc);
    HC_CHECK_LAUNCH();
    return;
  }
  const Xchg xc = d->site(off);
  if (part != 2) {
    int g0, g1;
    rank_groups(d->rank, d->nranks, g0, g1);
    launch_zt_partial(stop, hp, hp.grp[g0], hp.grp[g1], r, s);
    xchg_group_sums(stop, xc, hp.nc, hp.partial.p, hp.grp, g0, g1, s);
  }
  if (part != 1) xchg_group_final(stop, xc, hp.nc, bc, s);
}

namespace {
__global__ void k_neg_copy(int64_t n, const double* __restrict__ a, double* __restrict__ b) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    b[t] = -a[t];
}
// dense (column-major, symmetric) -> canonical CSR, exact zeros dropped
void dense_to_csr(int64_t nc, const DBuf<double>& Ad, DCsr& Ac, cudaStream_t s) {
  Ac.nrows = Ac.ncols = nc;
  Ac.ptr.alloc(nc + 1, s);
  DBuf<int64_t> cnt(nc, s);
  const unsigned g = (unsigned)std::min<int64_t>(nc, kSMs * 8);
  k_dense_to_csr<false><<<g, 256, 0, s>>>(nc, Ad.p, cnt.p, nullptr, nullptr, nullptr);
  HC_CHECK_LAUNCH();
  Ac.nnz = exclusive_scan(cnt.p, Ac.ptr.p, nc, s);
  Ac.idx.alloc(Ac.nnz, s);
  Ac.val.alloc(Ac.nnz, s);
  k_dense_to_csr<true><<<g, 256, 0, s>>>(nc, Ad.p, nullptr, Ac.ptr.p, Ac.idx.p, Ac.val.p);
  HC_CHECK_LAUNCH();
}
}  // namespace

void galerkin_hybrid(const DCsr& A, const DCsr& Ps, const DCsr& Pst, const HybridP& hp, DCsr& Ac, cudaStream_t s) {
  const int64_t nG = hp.nG, nc = hp.nc, n = A.nrows;
  // W' = A[G, :] P_s ; A_GG
  DBuf<int32_t> gmap(n, s);
  k_fill_m1<<<grid_for(n, 256), 256, 0, s>>>(gmap.p, n);
  k_rowmap<<<grid_for(nG, 256), 256, 0, s>>>(hp.rows.p, nG, gmap.p);
  HC_CHECK_LAUNCH();
  DBuf<double> Ad(nc * nc, s);
  DCsr APs, Ms, Ss;
  if (hp.D.p) {  // A_c = sym(P_s^T A P_s) - Y^T Y
    spgemm(A, Ps, APs, s);
    spgemm(Pst, APs, Ms, s);
    APs = DCsr();
    symmetrize(Ms, Ss, s);
    k_neg_copy<<<grid_for(nc * nc, 256, kSMs * 32), 256, 0, s>>>(nc * nc, hp.D.p, Ad.p);
    k_add_sym_csr<<<grid_for(nc, 256), 256, 0, s>>>(Ss.ptr.p, Ss.idx.p, Ss.val.p, nc, Ad.p);
    HC_CHECK_LAUNCH();
    dense_to_csr(nc, Ad, Ac, s);
    return;
  }
  DCsr AG, Wp0, Wp, Agg, WpT;
  csr_extract(A, hp.rows.p, nG, nullptr, n, AG, s);
  spgemm(AG, Ps, Wp0, s);
  drop_zeros(Wp0, Wp, s);
  Wp0 = DCsr();
  csr_extract(A, hp.rows.p, nG, gmap.p, nG, Agg, s);
  AG = DCsr();
  csr_transpose(Wp, WpT, s);
  // E = Z^T rho (column-major nc x nc), rho = W' - A_GG Z (row-major nG x nc).
  // rho is the residual of the component solve: O(eps |A_GG| |Z|), the same
  // order as the rounding already in the other Galerkin terms (and computed
  // in fp64 it is itself only accurate to O(1) relative).  Its product with Z
  // therefore needs no more than a few correct digits: it runs on the tensor
  // cores in TF32 (rho formed in fp64 block by block, then rounded to fp32),
  // 2.3e14 flops in well under a second instead of ~7 s of DGEMM.
  // HCAMG_GALERKIN_E=fp64 keeps the fp64 product (validation).
  DBuf<double> E(nc * nc, s);
  {
    // rho in row blocks of at most 512 MB, E += Z_blk^T rho_blk (own FP64 GEMM)
    const int64_t rb = std::max<int64_t>(1, std::min<int64_t>(nG, (int64_t)(512ll << 20) / (8 * std::max<int64_t>(nc, 1))));
    DBuf<double> blk(rb * nc, s);
    for (int64_t q0 = 0; q0 < nG; q0 += rb) {
      const int64_t nr = std::min(rb, nG - q0);
      k_spmm_rows<<<(unsigned)std::min<int64_t>(nr, kSMs * 16), 256, 0, s>>>(Agg.ptr.p + q0, Agg.idx.p, Agg.val.p, nr,
                                                                             nc, hp.Z.p, blk.p);
      k_add_csr_dense<<<grid_for(nr, 256), 256, 0, s>>>(Wp.ptr.p + q0, Wp.idx.p, Wp.val.p, nr, nc, blk.p);
      HC_CHECK_LAUNCH();
      // column-major nc x nc: E = sum over rows q of Z[q, :]^T rho[q, :]; the row-major
      // nr x nc blocks are column-major nc x nr views
      dblas::gemm(dblas::N, dblas::T, nc, nc, nr, 1.0, hp.Z.p + q0 * nc, nc, blk.p, nc, q0 == 0 ? 0.0 : 1.0, E.p, nc,
                  s);
    }
  }
  // D1 = Z^T W'
  DBuf<double> D1(nc * nc, s);
  k_zt_w<<<(unsigned)std::min<int64_t>(nc, kSMs * 16), 256, 0, s>>>(WpT.ptr.p, WpT.idx.p, WpT.val.p, nc, hp.Z.p, D1.p);
  HC_CHECK_LAUNCH();
  // sym(P_s^T A P_s)
  spgemm(A, Ps, APs, s);
  spgemm(Pst, APs, Ms, s);
  APs = DCsr();
  symmetrize(Ms, Ss, s);
  k_combine<<<grid_for(nc * nc, 256), 256, 0, s>>>(nc, D1.p, E.p, Ad.p);
  k_add_sym_csr<<<grid_for(nc, 256), 256, 0, s>>>(Ss.ptr.p, Ss.idx.p, Ss.val.p, nc, Ad.p);
  HC_CHECK_LAUNCH();
  D1.release();
  E.release();
  dense_to_csr(nc, Ad, Ac, s);
}

namespace {
__global__ void k_count_nz(const double* __restrict__ v, int64_t n, unsigned long long* out) {
  unsigned long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    c += v[i] != 0.0;
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, c);
}
}  // namespace

int64_t hybrid_nnz(const DCsr& Ps, const HybridP& hp, cudaStream_t s) {
  if (!hp.Z.p) return Ps.nnz + hp.nG * hp.nc;  // Z not formed: its entries are generically all nonzero
  DBuf<unsigned long long> c(1, s);
  c.zero();
  if (hp.nG * hp.nc) k_count_nz<<<grid_for(hp.nG * hp.nc, 256, kSMs * 8), 256, 0, s>>>(hp.Z.p, hp.nG * hp.nc, c.p);
  HC_CHECK_LAUNCH();
  return Ps.nnz + (int64_t)read_scalar(c.p, s);
}

void hybrid_to_csr(const DCsr& Ps, const HybridP& hp, DCsr& P, cudaStream_t s) {
  const int64_t n = Ps.nrows;
  DBuf<int32_t> map(n, s);
  k_fill_m1<<<grid_for(n, 256), 256, 0, s>>>(map.p, n);
  k_rowmap<<<grid_for(hp.nG, 256), 256, 0, s>>>(hp.rows.p, hp.nG, map.p);
  HC_CHECK_LAUNCH();
  P.nrows = n;
  P.ncols = Ps.ncols;
  P.ptr.alloc(n + 1, s);
  DBuf<int64_t> cnt(n, s);
  k_hybrid_csr<false><<<grid_for(n, 128), 128, 0, s>>>(n, Ps.ptr.p, Ps.idx.p, Ps.val.p, map.p, hp.nc, hp.Z.p, cnt.p,
                                                       nullptr, nullptr, nullptr);
  HC_CHECK_LAUNCH();
  P.nnz = exclusive_scan(cnt.p, P.ptr.p, n, s);
  require(P.nnz < (int64_t(1) << 31), "P too large to materialise as CSR");
  P.idx.alloc(P.nnz, s);
  P.val.alloc(P.nnz, s);
  k_hybrid_csr<true><<<grid_for(n, 128), 128, 0, s>>>(n, Ps.ptr.p, Ps.idx.p, Ps.val.p, map.p, hp.nc, hp.Z.p, nullptr,
                                                      P.ptr.p, P.idx.p, P.val.p);
  HC_CHECK_LAUNCH();
}

}  // namespace hcamg
