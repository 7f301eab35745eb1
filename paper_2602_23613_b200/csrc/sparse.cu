// Setup-phase sparse kernels (see sparse.cuh).
#include <cub/cub.cuh>

#include "sparse.cuh"

namespace hcamg {

namespace {

__global__ void k_copy_counts(const int64_t* __restrict__ c, int64_t* __restrict__ o, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; i <= n; i += st) o[i] = i < n ? c[i] : 0;
}

}  // namespace

int64_t exclusive_scan(const int64_t* counts, int64_t* out, int64_t n, cudaStream_t s) {
  DBuf<int64_t> tmp(n + 1, s);
  k_copy_counts<<<grid_for(n + 1, 256), 256, 0, s>>>(counts, tmp.p, n);
  HC_CHECK_LAUNCH();
  size_t bytes = 0;
  HC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, tmp.p, out, n + 1, s));
  DBuf<unsigned char> ws((int64_t)bytes + 1, s);
  HC_CUDA(cub::DeviceScan::ExclusiveSum(ws.p, bytes, tmp.p, out, n + 1, s));
  return read_scalar(out + n, s);
}

// ----------------------------------------------------------------------------- transpose

namespace {

__global__ void k_row_ids(const int64_t* __restrict__ ptr, int64_t nrows, int32_t* __restrict__ rowid) {
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < nrows; r += nw)
    for (int64_t e = ptr[r] + lane; e < ptr[r + 1]; e += 32) rowid[e] = (int32_t)r;
}

__global__ void k_iota(int32_t* __restrict__ v, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) v[i] = (int32_t)i;
}

__global__ void k_col_hist(const int32_t* __restrict__ idx, int64_t nnz, int64_t* __restrict__ cnt) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; i < nnz; i += st) atomicAdd((unsigned long long*)&cnt[idx[i]], 1ull);
}

__global__ void k_gather_t(const int32_t* __restrict__ perm, const int32_t* __restrict__ rowid,
                           const double* __restrict__ val, int32_t* __restrict__ oidx,
                           double* __restrict__ oval, int64_t nnz) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; i < nnz; i += st) {
    int32_t p = perm[i];
    oidx[i] = rowid[p];
    oval[i] = val[p];
  }
}

int bits_for(int64_t v) {
  int b = 1;
  while ((int64_t(1) << b) <= v) ++b;
  return b;
}

}  // namespace

void csr_transpose(const DCsr& A, DCsr& At, cudaStream_t s) {
  require(A.nnz < (int64_t(1) << 31), "transpose: nnz exceeds int32 positions");
  At.alloc(A.ncols, A.nrows, A.nnz, s);
  DBuf<int64_t> cnt(A.ncols, s);
  cnt.zero();
  if (A.nnz) {
    DBuf<int32_t> rowid(A.nnz, s), perm_in(A.nnz, s), perm(A.nnz, s), keys(A.nnz, s);
    k_row_ids<<<grid_for(A.nrows * 32, 256), 256, 0, s>>>(A.ptr.p, A.nrows, rowid.p);
    k_iota<<<grid_for(A.nnz, 256), 256, 0, s>>>(perm_in.p, A.nnz);
    k_col_hist<<<grid_for(A.nnz, 256), 256, 0, s>>>(A.idx.p, A.nnz, cnt.p);
    HC_CHECK_LAUNCH();
    size_t bytes = 0;
    int eb = bits_for(A.ncols);
    HC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, A.idx.p, keys.p, perm_in.p, perm.p,
                                            A.nnz, 0, eb, s));
    DBuf<unsigned char> ws((int64_t)bytes + 1, s);
    HC_CUDA(cub::DeviceRadixSort::SortPairs(ws.p, bytes, A.idx.p, keys.p, perm_in.p, perm.p,
                                            A.nnz, 0, eb, s));
    k_gather_t<<<grid_for(A.nnz, 256), 256, 0, s>>>(perm.p, rowid.p, A.val.p, At.idx.p, At.val.p,
                                                    A.nnz);
    HC_CHECK_LAUNCH();
  }
  exclusive_scan(cnt.p, At.ptr.p, A.ncols, s);
}

// ----------------------------------------------------------------------------- spgemm

namespace {

constexpr int kWarpsPerBlock = 4;

__device__ __forceinline__ void warp_bufs(unsigned char* smem, bool in_smem, double* gacc,
                                          unsigned char* gflag, int64_t ncols, double*& acc,
                                          unsigned char*& flag) {
  int wib = threadIdx.x >> 5;
  if (in_smem) {
    acc = reinterpret_cast<double*>(smem) + (int64_t)wib * ncols;
    flag = smem + (int64_t)kWarpsPerBlock * ncols * 8 + (int64_t)wib * ncols;
  } else {
    int64_t gw = (int64_t)blockIdx.x * kWarpsPerBlock + wib;
    acc = gacc + gw * ncols;
    flag = gflag + gw * ncols;
  }
}

__global__ void k_spgemm_count(const int64_t* __restrict__ ap, const int32_t* __restrict__ ai,
                               const int64_t* __restrict__ bp, const int32_t* __restrict__ bi,
                               int64_t nrows, int64_t ncols, bool in_smem, double* gacc,
                               unsigned char* gflag, int64_t* __restrict__ rownnz) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* acc;
  unsigned char* flag;
  warp_bufs(smem, in_smem, gacc, gflag, ncols, acc, flag);
  int lane = threadIdx.x & 31;
  if (in_smem) {
    for (int64_t t = threadIdx.x; t < (int64_t)kWarpsPerBlock * ncols; t += blockDim.x)
      smem[(int64_t)kWarpsPerBlock * ncols * 8 + t] = 0;
    __syncthreads();
  }
  int64_t gw = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  int64_t nw = (int64_t)gridDim.x * kWarpsPerBlock;
  for (int64_t i = gw; i < nrows; i += nw) {
    int cnt = 0;
    for (int64_t e = ap[i]; e < ap[i + 1]; ++e) {
      int32_t j = ai[e];
      for (int64_t t = bp[j] + lane; t < bp[j + 1]; t += 32) {
        int32_t k = bi[t];
        if (!flag[k]) { flag[k] = 1; ++cnt; }
      }
      __syncwarp();
    }
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) rownnz[i] = cnt;
    for (int64_t e = ap[i]; e < ap[i + 1]; ++e) {
      int32_t j = ai[e];
      for (int64_t t = bp[j] + lane; t < bp[j + 1]; t += 32) flag[bi[t]] = 0;
    }
    __syncwarp();
  }
}

__global__ void k_spgemm_fill(const int64_t* __restrict__ ap, const int32_t* __restrict__ ai,
                              const double* __restrict__ av, const int64_t* __restrict__ bp,
                              const int32_t* __restrict__ bi, const double* __restrict__ bv,
                              int64_t nrows, int64_t ncols, bool in_smem, double* gacc,
                              unsigned char* gflag, const int64_t* __restrict__ cp,
                              int32_t* __restrict__ ci, double* __restrict__ cv) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* acc;
  unsigned char* flag;
  warp_bufs(smem, in_smem, gacc, gflag, ncols, acc, flag);
  int lane = threadIdx.x & 31;
  unsigned lt = (1u << lane) - 1u;
  if (in_smem) {
    for (int64_t t = threadIdx.x; t < (int64_t)kWarpsPerBlock * ncols; t += blockDim.x)
      smem[(int64_t)kWarpsPerBlock * ncols * 8 + t] = 0;
    __syncthreads();
  }
  int64_t gw = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  int64_t nw = (int64_t)gridDim.x * kWarpsPerBlock;
  for (int64_t i = gw; i < nrows; i += nw) {
    int64_t base = cp[i];
    int64_t cnt = 0;
    for (int64_t e = ap[i]; e < ap[i + 1]; ++e) {
      int32_t j = ai[e];
      double a = av[e];
      int64_t b0 = bp[j], b1 = bp[j + 1];
      for (int64_t t0 = b0; t0 < b1; t0 += 32) {
        int64_t t = t0 + lane;
        bool active = t < b1;
        bool first = false;
        int32_t k = 0;
        if (active) {
          k = bi[t];
          double prod = __dmul_rn(a, bv[t]);
          first = !flag[k];
          if (first) {
            flag[k] = 1;
            acc[k] = __dadd_rn(0.0, prod);
          } else {
            acc[k] = __dadd_rn(acc[k], prod);
          }
        }
        unsigned m = __ballot_sync(0xffffffffu, first);
        if (first) ci[base + cnt + __popc(m & lt)] = k;
        cnt += __popc(m);
      }
      __syncwarp();
    }
    __syncwarp();
    for (int64_t t = lane; t < cnt; t += 32) {
      int32_t k = ci[base + t];
      cv[base + t] = acc[k];
      flag[k] = 0;
    }
    __syncwarp();
  }
}

}  // namespace

static void segmented_sort(DCsr& C, cudaStream_t s) {
  if (C.nnz == 0 || C.nrows == 0) return;
  DBuf<int32_t> ko(C.nnz, s);
  DBuf<double> vo(C.nnz, s);
  size_t bytes = 0;
  HC_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, bytes, C.idx.p, ko.p, C.val.p, vo.p, C.nnz,
                                              C.nrows, C.ptr.p, C.ptr.p + 1, s));
  DBuf<unsigned char> ws((int64_t)bytes + 1, s);
  HC_CUDA(cub::DeviceSegmentedSort::SortPairs(ws.p, bytes, C.idx.p, ko.p, C.val.p, vo.p, C.nnz,
                                              C.nrows, C.ptr.p, C.ptr.p + 1, s));
  C.idx = std::move(ko);
  C.val = std::move(vo);
}

// ---- left factor stored as a fully dense canonical CSR (the dense-regime
// coarse operator, config 2: 26,236^2 entries): the row kernels above walk
// the 26 k entries of a row one after the other, two lanes busy on a
// gradient's two entries (0.32 s for A_1 G~).  With every A[i, k] stored, the
// pattern of C is the same for every row (the non-empty columns of B) and
// C[i, v] = sum over the rows k of B's column v, ascending, of A[i, k] B[k, v]
// -- scipy's csr_matmat order (k ascending, product rounded, then added), one
// thread per output entry.
namespace {
__global__ void k_dense_canonical(const int64_t* __restrict__ ap, const int32_t* __restrict__ ai, int64_t nrows,
                                  int64_t ncols, int* __restrict__ bad) {
  const int64_t total = nrows * ncols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x)
    if (ai[e] != (int32_t)(e % ncols) || (e % ncols == 0 && ap[e / ncols] != e)) *bad = 1;
}
__global__ void k_col_nonempty(const int64_t* __restrict__ tp, int64_t m, int64_t* __restrict__ f) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < m; v += (int64_t)gridDim.x * blockDim.x)
    f[v] = tp[v + 1] > tp[v];
}
__global__ void k_dense_left_fill(const double* __restrict__ av, int64_t nrows, int64_t ka,
                                  const int64_t* __restrict__ tp, const int32_t* __restrict__ ti,
                                  const double* __restrict__ tv, int64_t m, const int64_t* __restrict__ cpos,
                                  int64_t nc, int64_t* __restrict__ cp, int32_t* __restrict__ ci,
                                  double* __restrict__ cv) {
  const int64_t i = blockIdx.y + (int64_t)gridDim.y * blockIdx.z;
  if (i >= nrows) return;
  const double* arow = av + i * ka;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < m; v += (int64_t)gridDim.x * blockDim.x) {
    if (tp[v + 1] == tp[v]) continue;
    double acc = 0.0;
    for (int64_t t = tp[v]; t < tp[v + 1]; ++t) acc = __dadd_rn(acc, __dmul_rn(arow[ti[t]], tv[t]));
    ci[i * nc + cpos[v]] = (int32_t)v;
    cv[i * nc + cpos[v]] = acc;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    cp[i] = i * nc;
    if (i == nrows - 1) cp[nrows] = nrows * nc;
  }
}
}  // namespace

bool csr_is_dense_canonical(const DCsr& A, cudaStream_t s) {
  if (A.nrows <= 0 || A.ncols <= 0 || A.nnz != A.nrows * A.ncols) return false;
  DBuf<int> bad(1, s);
  bad.zero();
  k_dense_canonical<<<kSMs * 8, 256, 0, s>>>(A.ptr.p, A.idx.p, A.nrows, A.ncols, bad.p);
  HC_CHECK_LAUNCH();
  return read_scalar(bad.p, s) == 0;
}

static bool spgemm_dense_left(const DCsr& A, const DCsr& B, DCsr& C, cudaStream_t s) {
  const int64_t nrows = A.nrows, ka = A.ncols, m = B.ncols;
  if (nrows < 32 || ka < 32 || nrows >= 65535LL * 65535LL || !csr_is_dense_canonical(A, s)) return false;
  DCsr Bt;
  csr_transpose(B, Bt, s);
  DBuf<int64_t> f(m, s), cpos(m + 1, s);  // the scan writes m + 1 offsets
  k_col_nonempty<<<grid_for(m, 256), 256, 0, s>>>(Bt.ptr.p, m, f.p);
  HC_CHECK_LAUNCH();
  const int64_t nc = exclusive_scan(f.p, cpos.p, m, s);
  C.nrows = nrows;
  C.ncols = m;
  C.nnz = nrows * nc;
  C.ptr.alloc(nrows + 1, s);
  C.idx.alloc(C.nnz, s);
  C.val.alloc(C.nnz, s);
  const unsigned gy = (unsigned)std::min<int64_t>(nrows, 65535), gz = (unsigned)((nrows + gy - 1) / gy);
  const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256, 64));
  k_dense_left_fill<<<dim3(gx, gy, gz), 256, 0, s>>>(A.val.p, nrows, ka, Bt.ptr.p, Bt.idx.p, Bt.val.p, m, cpos.p, nc,
                                                    C.ptr.p, C.idx.p, C.val.p);
  HC_CHECK_LAUNCH();
  return true;
}

void spgemm(const DCsr& A, const DCsr& B, DCsr& C, cudaStream_t s) {
  require(A.ncols == B.nrows, "spgemm: dimension mismatch");
  if (spgemm_dense_left(A, B, C, s)) return;
  const int64_t nrows = A.nrows, ncols = B.ncols;
  C.nrows = nrows;
  C.ncols = ncols;
  C.ptr.alloc(nrows + 1, s);
  DBuf<int64_t> rownnz(nrows, s);
  int64_t smem_bytes = (int64_t)kWarpsPerBlock * ncols * 9;
  bool in_smem = smem_bytes <= 200 * 1024;
  int blocks = kSMs * 4;
  if (nrows < (int64_t)blocks * kWarpsPerBlock) blocks = (int)((nrows + kWarpsPerBlock - 1) / kWarpsPerBlock);
  if (blocks < 1) blocks = 1;
  DBuf<double> gacc;
  DBuf<unsigned char> gflag;
  size_t dyn = 0;
  if (in_smem) {
    dyn = (size_t)smem_bytes;
    HC_CUDA(cudaFuncSetAttribute(k_spgemm_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    HC_CUDA(cudaFuncSetAttribute(k_spgemm_fill, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
  } else {
    gacc.alloc((int64_t)blocks * kWarpsPerBlock * ncols, s);
    gflag.alloc((int64_t)blocks * kWarpsPerBlock * ncols, s);
    gflag.zero();
  }
  if (nrows > 0) {
    k_spgemm_count<<<blocks, 32 * kWarpsPerBlock, dyn, s>>>(A.ptr.p, A.idx.p, B.ptr.p, B.idx.p, nrows,
                                                            ncols, in_smem, gacc.p, gflag.p, rownnz.p);
    HC_CHECK_LAUNCH();
  }
  C.nnz = exclusive_scan(rownnz.p, C.ptr.p, nrows, s);
  C.idx.alloc(C.nnz, s);
  C.val.alloc(C.nnz, s);
  if (nrows > 0 && C.nnz > 0) {
    k_spgemm_fill<<<blocks, 32 * kWarpsPerBlock, dyn, s>>>(A.ptr.p, A.idx.p, A.val.p, B.ptr.p, B.idx.p,
                                                           B.val.p, nrows, ncols, in_smem, gacc.p,
                                                           gflag.p, C.ptr.p, C.idx.p, C.val.p);
    HC_CHECK_LAUNCH();
  }
  segmented_sort(C, s);
}

// ----------------------------------------------------------------------------- symmetrize

namespace {

template <bool kWrite>
__global__ void k_sym(const int64_t* __restrict__ mp, const int32_t* __restrict__ mi,
                      const double* __restrict__ mv, const int64_t* __restrict__ tp,
                      const int32_t* __restrict__ ti, const double* __restrict__ tv, int64_t n,
                      int64_t* __restrict__ cnt, const int64_t* __restrict__ op,
                      int32_t* __restrict__ oi, double* __restrict__ ov) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; r < n; r += st) {
    int64_t a = mp[r], ae = mp[r + 1], b = tp[r], be = tp[r + 1];
    int64_t c = 0, o = kWrite ? op[r] : 0;
    while (a < ae || b < be) {
      int32_t ca = a < ae ? mi[a] : INT32_MAX;
      int32_t cb = b < be ? ti[b] : INT32_MAX;
      double v;
      int32_t col;
      if (ca == cb) { v = __dadd_rn(mv[a], tv[b]); col = ca; ++a; ++b; }
      else if (ca < cb) { v = __dadd_rn(mv[a], 0.0); col = ca; ++a; }
      else { v = __dadd_rn(0.0, tv[b]); col = cb; ++b; }
      double h = __dmul_rn(0.5, v);
      if (h != 0.0) {
        if (kWrite) { oi[o + c] = col; ov[o + c] = h; }
        ++c;
      }
    }
    if (!kWrite) cnt[r] = c;
  }
}

template <bool kWrite>
__global__ void k_dropz(const int64_t* __restrict__ mp, const int32_t* __restrict__ mi,
                        const double* __restrict__ mv, int64_t n, int64_t* __restrict__ cnt,
                        const int64_t* __restrict__ op, int32_t* __restrict__ oi,
                        double* __restrict__ ov) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; r < n; r += st) {
    int64_t c = 0, o = kWrite ? op[r] : 0;
    for (int64_t e = mp[r]; e < mp[r + 1]; ++e) {
      if (mv[e] != 0.0) {
        if (kWrite) { oi[o + c] = mi[e]; ov[o + c] = mv[e]; }
        ++c;
      }
    }
    if (!kWrite) cnt[r] = c;
  }
}

template <bool kWrite>
__global__ void k_extract(const int64_t* __restrict__ mp, const int32_t* __restrict__ mi,
                          const double* __restrict__ mv, const int32_t* __restrict__ rows,
                          int64_t nr, const int32_t* __restrict__ colmap, int64_t* __restrict__ cnt,
                          const int64_t* __restrict__ op, int32_t* __restrict__ oi,
                          double* __restrict__ ov) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; r < nr; r += st) {
    int64_t src = rows ? rows[r] : r;
    int64_t c = 0, o = kWrite ? op[r] : 0;
    for (int64_t e = mp[src]; e < mp[src + 1]; ++e) {
      int32_t col = colmap ? colmap[mi[e]] : mi[e];
      if (col >= 0) {
        if (kWrite) { oi[o + c] = col; ov[o + c] = mv[e]; }
        ++c;
      }
    }
    if (!kWrite) cnt[r] = c;
  }
}

}  // namespace

void symmetrize(const DCsr& M, DCsr& S, cudaStream_t s) {
  require(M.nrows == M.ncols, "symmetrize: matrix must be square");
  DCsr Mt;
  csr_transpose(M, Mt, s);
  int64_t n = M.nrows;
  S.nrows = S.ncols = n;
  S.ptr.alloc(n + 1, s);
  DBuf<int64_t> cnt(n, s);
  unsigned g = grid_for(n, 128);
  if (n) k_sym<false><<<g, 128, 0, s>>>(M.ptr.p, M.idx.p, M.val.p, Mt.ptr.p, Mt.idx.p, Mt.val.p, n,
                                        cnt.p, nullptr, nullptr, nullptr);
  HC_CHECK_LAUNCH();
  S.nnz = exclusive_scan(cnt.p, S.ptr.p, n, s);
  S.idx.alloc(S.nnz, s);
  S.val.alloc(S.nnz, s);
  if (n) k_sym<true><<<g, 128, 0, s>>>(M.ptr.p, M.idx.p, M.val.p, Mt.ptr.p, Mt.idx.p, Mt.val.p, n,
                                       nullptr, S.ptr.p, S.idx.p, S.val.p);
  HC_CHECK_LAUNCH();
}

void drop_zeros(const DCsr& M, DCsr& out, cudaStream_t s) {
  int64_t n = M.nrows;
  out.nrows = n;
  out.ncols = M.ncols;
  out.ptr.alloc(n + 1, s);
  DBuf<int64_t> cnt(n, s);
  unsigned g = grid_for(n, 128);
  if (n) k_dropz<false><<<g, 128, 0, s>>>(M.ptr.p, M.idx.p, M.val.p, n, cnt.p, nullptr, nullptr, nullptr);
  HC_CHECK_LAUNCH();
  out.nnz = exclusive_scan(cnt.p, out.ptr.p, n, s);
  out.idx.alloc(out.nnz, s);
  out.val.alloc(out.nnz, s);
  if (n) k_dropz<true><<<g, 128, 0, s>>>(M.ptr.p, M.idx.p, M.val.p, n, nullptr, out.ptr.p, out.idx.p,
                                         out.val.p);
  HC_CHECK_LAUNCH();
}

void csr_extract(const DCsr& M, const int32_t* rows, int64_t nr, const int32_t* colmap,
                 int64_t ncols_out, DCsr& out, cudaStream_t s) {
  out.nrows = nr;
  out.ncols = ncols_out;
  out.ptr.alloc(nr + 1, s);
  DBuf<int64_t> cnt(nr, s);
  unsigned g = grid_for(nr, 128);
  if (nr) k_extract<false><<<g, 128, 0, s>>>(M.ptr.p, M.idx.p, M.val.p, rows, nr, colmap, cnt.p,
                                             nullptr, nullptr, nullptr);
  HC_CHECK_LAUNCH();
  out.nnz = exclusive_scan(cnt.p, out.ptr.p, nr, s);
  out.idx.alloc(out.nnz, s);
  out.val.alloc(out.nnz, s);
  if (nr) k_extract<true><<<g, 128, 0, s>>>(M.ptr.p, M.idx.p, M.val.p, rows, nr, colmap, nullptr,
                                            out.ptr.p, out.idx.p, out.val.p);
  HC_CHECK_LAUNCH();
}

void csr_copy(const DCsr& M, DCsr& out, cudaStream_t s) {
  out.alloc(M.nrows, M.ncols, M.nnz, s);
  HC_CUDA(cudaMemcpyAsync(out.ptr.p, M.ptr.p, 8 * (M.nrows + 1), cudaMemcpyDeviceToDevice, s));
  if (M.nnz) {
    HC_CUDA(cudaMemcpyAsync(out.idx.p, M.idx.p, 4 * M.nnz, cudaMemcpyDeviceToDevice, s));
    HC_CUDA(cudaMemcpyAsync(out.val.p, M.val.p, 8 * M.nnz, cudaMemcpyDeviceToDevice, s));
  }
}

void csr_upload(const int64_t* indptr, const int32_t* indices, const double* data, int64_t nrows,
                int64_t ncols, DCsr& out, cudaStream_t s) {
  int64_t nnz = indptr[nrows];
  out.alloc(nrows, ncols, nnz, s);
  HC_CUDA(cudaMemcpyAsync(out.ptr.p, indptr, 8 * (nrows + 1), cudaMemcpyHostToDevice, s));
  if (nnz) {
    HC_CUDA(cudaMemcpyAsync(out.idx.p, indices, 4 * nnz, cudaMemcpyHostToDevice, s));
    HC_CUDA(cudaMemcpyAsync(out.val.p, data, 8 * nnz, cudaMemcpyHostToDevice, s));
  }
}

namespace {
__global__ void k_spmv_plain(const int64_t* __restrict__ p, const int32_t* __restrict__ i,
                             const double* __restrict__ v, const double* __restrict__ x,
                             double* __restrict__ y, int64_t n) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; r < n; r += st) {
    double acc = 0.0;
    for (int64_t e = p[r]; e < p[r + 1]; ++e) acc = __dadd_rn(acc, __dmul_rn(v[e], x[i[e]]));
    y[r] = acc;
  }
}

__global__ void k_maxabs(const double* __restrict__ v, int64_t n, unsigned long long* out) {
  double m = 0.0;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) m = fmax(m, fabs(v[i]));
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}
}  // namespace

void spmv(const DCsr& A, const double* x, double* y, cudaStream_t s) {
  if (A.nrows) k_spmv_plain<<<grid_for(A.nrows, 128), 128, 0, s>>>(A.ptr.p, A.idx.p, A.val.p, x, y, A.nrows);
  HC_CHECK_LAUNCH();
}

double max_abs(const DCsr& A, cudaStream_t s) {
  DBuf<unsigned long long> m(1, s);
  m.zero();
  if (A.nnz) k_maxabs<<<grid_for(A.nnz, 256), 256, 0, s>>>(A.val.p, A.nnz, m.p);
  HC_CHECK_LAUNCH();
  unsigned long long h = read_scalar(m.p, s);
  double d;
  memcpy(&d, &h, 8);
  return d;
}

}  // namespace hcamg
