// Sparse approximate ideal interpolation on the GPU (hcurl_amg/transfer.py:77-122):
//   P = R^T - S_I A_II^{-1} S_I^T A R^T,
// one dense SPD solve per connected component of the interior graph
// (transfer.py:49-52, 94-110): batched warp-level Cholesky for small
// components, a blocked tensor-free FP64 Cholesky (cuBLAS level-3 panels) for
// large ones.  Coarse gradient R G I_C: transfer.py:55-74, multilevel.py:71-75.
#include <cub/cub.cuh>

#include <algorithm>

#include "dense.cuh"
#include "interp.cuh"

namespace hcamg {

namespace {

constexpr double kInvSqrt2 = 0x1.6a09e667f3bccp-1;  // 1.0 / np.sqrt(2.0) (splitting.py:47)

__global__ void k_build_R(const int64_t* __restrict__ pairs, int64_t np_, int64_t* __restrict__ rp,
                          int32_t* __restrict__ ri, double* __restrict__ rv) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; p <= np_; p += st) {
    rp[p] = 2 * p;
    if (p == np_) continue;
    const int64_t* q = pairs + 7 * p;
    int64_t d1 = q[0], d2 = q[1];
    double v1 = (double)q[2] * kInvSqrt2, v2 = (double)q[3] * kInvSqrt2;
    if (d1 < d2) { ri[2 * p] = (int32_t)d1; rv[2 * p] = v1; ri[2 * p + 1] = (int32_t)d2; rv[2 * p + 1] = v2; }
    else { ri[2 * p] = (int32_t)d2; rv[2 * p] = v2; ri[2 * p + 1] = (int32_t)d1; rv[2 * p + 1] = v1; }
  }
}

// ---- union-find (hook larger root under smaller: the root is the component minimum)
__device__ __forceinline__ int uf_rep(int* par, int x) {
  int cur = par[x];
  if (cur != x) {
    int next, prev = x;
    while (cur > (next = par[cur])) {
      par[prev] = next;
      prev = cur;
      cur = next;
    }
  }
  return cur;
}

__global__ void k_uf_init(int* par, int64_t n) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    par[v] = (int)v;
}

__global__ void k_uf_hook(const int64_t* __restrict__ mp, const int32_t* __restrict__ mi, int64_t n, int* par) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
    for (int64_t e = mp[u]; e < mp[u + 1]; ++e) {
      int v = mi[e];
      if (v == u) continue;
      int ru = uf_rep(par, (int)u), rv = uf_rep(par, v);
      while (ru != rv) {
        if (ru < rv) { int t = ru; ru = rv; rv = t; }
        int old = atomicCAS(&par[ru], ru, rv);
        if (old == ru) break;
        ru = uf_rep(par, old);
        rv = uf_rep(par, rv);
      }
    }
  }
}

__global__ void k_uf_flatten(int* par, int64_t n, int64_t* __restrict__ is_root) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    int r = v;
    while (par[r] != r) r = par[r];
    par[v] = r;
    is_root[v] = r == v;
  }
}

__global__ void k_uf_label(const int* __restrict__ par, const int64_t* __restrict__ rank, int64_t n,
                           int32_t* __restrict__ label) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    label[v] = (int32_t)rank[par[v]];
}

__global__ void k_iota32(int32_t* v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (int32_t)i;
}

__global__ void k_hist32(const int32_t* __restrict__ key, int64_t n, int64_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd((unsigned long long*)&cnt[key[i]], 1ull);
}

__global__ void k_pos_in_comp(const int32_t* __restrict__ sorted_lab, const int32_t* __restrict__ members,
                              const int64_t* __restrict__ cptr, int64_t n, int32_t* __restrict__ pos) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    pos[members[t]] = (int32_t)(t - cptr[sorted_lab[t]]);
}

__global__ void k_keep_keys(const int64_t* __restrict__ wp, const int32_t* __restrict__ wi, int64_t nrows,
                            const int32_t* __restrict__ label, unsigned long long* __restrict__ keys) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nrows; q += (int64_t)gridDim.x * blockDim.x)
    for (int64_t e = wp[q]; e < wp[q + 1]; ++e)
      keys[e] = ((unsigned long long)(uint32_t)label[q] << 32) | (uint32_t)wi[e];
}

__global__ void k_keep_split(const unsigned long long* __restrict__ keys, int64_t n, int64_t* __restrict__ cnt,
                             int32_t* __restrict__ cols) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    atomicAdd((unsigned long long*)&cnt[keys[t] >> 32], 1ull);
    cols[t] = (int32_t)(keys[t] & 0xffffffffull);
  }
}

__device__ __forceinline__ int64_t lower_bound32(const int32_t* a, int64_t lo, int64_t hi, int32_t v) {
  while (lo < hi) {
    int64_t m = (lo + hi) >> 1;
    if (a[m] < v) lo = m + 1; else hi = m;
  }
  return lo;
}

__global__ void k_fill_dense(const int64_t* __restrict__ aip, const int32_t* __restrict__ aii,
                             const double* __restrict__ aiv, const int64_t* __restrict__ wp,
                             const int32_t* __restrict__ wi, const double* __restrict__ wv, int64_t ni,
                             const int32_t* __restrict__ label, const int32_t* __restrict__ pos,
                             const int64_t* __restrict__ cptr, const int64_t* __restrict__ kptr,
                             const int32_t* __restrict__ kcols, const int64_t* __restrict__ a_off,
                             const int64_t* __restrict__ b_off, double* __restrict__ Ad, double* __restrict__ Bd,
                             int giant) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < ni; q += (int64_t)gridDim.x * blockDim.x) {
    const int c = label[q];
    if (c == giant) continue;               // dense-regime component: handled separately
    if (kptr[c + 1] == kptr[c]) continue;  // component without coarse columns: skipped
    const int64_t k = cptr[c + 1] - cptr[c];
    const int64_t a = pos[q];
    double* Ac = Ad + a_off[c];
    double* Bc = Bd + b_off[c];
    for (int64_t e = aip[q]; e < aip[q + 1]; ++e) Ac[a + (int64_t)pos[aii[e]] * k] = aiv[e];
    for (int64_t e = wp[q]; e < wp[q + 1]; ++e) {
      int64_t kk = lower_bound32(kcols, kptr[c], kptr[c + 1], wi[e]) - kptr[c];
      Bc[a + kk * k] = wv[e];
    }
  }
}

// P rows: exterior dof -> one R^T entry; interior dof -> -Z row (exact zeros dropped).
template <bool kWrite>
__global__ void k_assemble_P(int64_t n, const int32_t* __restrict__ ext_p, const double* __restrict__ ext_v,
                             const int32_t* __restrict__ int_pos, const int32_t* __restrict__ label,
                             const int32_t* __restrict__ pos, const int64_t* __restrict__ cptr,
                             const int64_t* __restrict__ kptr, const int32_t* __restrict__ kcols,
                             const int64_t* __restrict__ b_off, const double* __restrict__ Bd, int giant,
                             int64_t* __restrict__ cnt, const int64_t* __restrict__ pp, int32_t* __restrict__ pi,
                             double* __restrict__ pv) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < n; d += (int64_t)gridDim.x * blockDim.x) {
    int64_t c_ = 0, o = kWrite ? pp[d] : 0;
    if (ext_p[d] >= 0) {
      if (kWrite) { pi[o] = ext_p[d]; pv[o] = ext_v[d]; }
      c_ = 1;
    } else if (label != nullptr && int_pos[d] >= 0) {
      const int64_t q = int_pos[d];
      const int c = label[q];
      if (c == giant) { if (!kWrite) cnt[d] = 0; continue; }
      const int64_t k = cptr[c + 1] - cptr[c];
      const int64_t nk = kptr[c + 1] - kptr[c];
      const double* Z = Bd + b_off[c] + pos[q];
      for (int64_t kk = 0; kk < nk; ++kk) {
        double z = Z[kk * k];
        if (z != 0.0) {
          if (kWrite) { pi[o + c_] = kcols[kptr[c] + kk]; pv[o + c_] = -z; }
          ++c_;
        }
      }
    }
    if (!kWrite) cnt[d] = c_;
  }
}

__global__ void k_ext_maps(const int64_t* __restrict__ pairs, int64_t np_, int32_t* __restrict__ ext_p,
                           double* __restrict__ ext_v) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < np_; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t* q = pairs + 7 * p;
    ext_p[q[0]] = (int32_t)p;
    ext_v[q[0]] = (double)q[2] * kInvSqrt2;
    ext_p[q[1]] = (int32_t)p;
    ext_v[q[1]] = (double)q[3] * kInvSqrt2;
  }
}

__global__ void k_int_maps(const int64_t* __restrict__ interior, int64_t ni, int32_t* __restrict__ int_pos,
                           int32_t* __restrict__ rows32) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < ni; q += (int64_t)gridDim.x * blockDim.x) {
    int_pos[interior[q]] = (int32_t)q;
    rows32[q] = (int32_t)interior[q];
  }
}

// positions of the giant component: gmap[q] = local index (or -1), mpos = member
// positions (ascending), rows = their DoFs
__global__ void k_giant_maps(const int32_t* __restrict__ label, const int32_t* __restrict__ pos, int64_t ni, int giant,
                             int32_t* __restrict__ gmap, const int32_t* __restrict__ members, int64_t nG,
                             const int64_t* __restrict__ interior, int32_t* __restrict__ mpos,
                             int32_t* __restrict__ rows) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ni || t < nG;
       t += (int64_t)gridDim.x * blockDim.x) {
    if (t < ni) gmap[t] = label[t] == giant ? pos[t] : -1;
    if (t < nG) {
      mpos[t] = members[t];
      rows[t] = (int32_t)interior[members[t]];
    }
  }
}

__global__ void k_giant_rhs(const int32_t* __restrict__ mpos, int64_t nG, const int64_t* __restrict__ wp,
                            const int32_t* __restrict__ wi, const double* __restrict__ wv, int64_t nc,
                            double* __restrict__ Z) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nG; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = mpos[t];
    for (int64_t e = wp[q]; e < wp[q + 1]; ++e) Z[t * nc + wi[e]] = wv[e];
  }
}

__global__ void k_fill_i32(int32_t* v, int64_t n, int32_t x) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) v[i] = x;
}

__global__ void k_col_count(const int32_t* __restrict__ idx, int64_t nnz, int64_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd((unsigned long long*)&cnt[idx[i]], 1ull);
}

__global__ void k_gc_keep(const int64_t* __restrict__ ccnt, int64_t m, const int64_t* __restrict__ cand,
                          int64_t ncand, int mode, int64_t* __restrict__ flag) {
  // mode 0 (refinement): every non-empty column; mode 1 (algebraic): listed c_G columns that are non-empty
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < m; v += (int64_t)gridDim.x * blockDim.x)
    flag[v] = mode == 0 ? (ccnt[v] > 0) : 0;
  if (mode == 1)
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ncand; t += (int64_t)gridDim.x * blockDim.x)
      if (ccnt[cand[t]] > 0) flag[cand[t]] = 1;
}

__global__ void k_colmap(const int64_t* __restrict__ flag, const int64_t* __restrict__ rank, int64_t m,
                         int32_t* __restrict__ cmap) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < m; v += (int64_t)gridDim.x * blockDim.x)
    cmap[v] = flag[v] ? (int32_t)rank[v] : -1;
}

__global__ void k_sign(double* v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (double)((v[i] > 0.0) - (v[i] < 0.0));
}

}  // namespace

int64_t connected_components(const DCsr& M, DBuf<int32_t>& label, cudaStream_t s) {
  const int64_t n = M.nrows;
  label.alloc(n, s);
  if (!n) return 0;
  DBuf<int> par(n, s);
  DBuf<int64_t> is_root(n, s), rank(n + 1, s);
  k_uf_init<<<grid_for(n, 256), 256, 0, s>>>(par.p, n);
  k_uf_hook<<<grid_for(n, 128), 128, 0, s>>>(M.ptr.p, M.idx.p, n, par.p);
  k_uf_flatten<<<grid_for(n, 256), 256, 0, s>>>(par.p, n, is_root.p);
  HC_CHECK_LAUNCH();
  int64_t nc = exclusive_scan(is_root.p, rank.p, n, s);
  k_uf_label<<<grid_for(n, 256), 256, 0, s>>>(par.p, rank.p, n, label.p);
  HC_CHECK_LAUNCH();
  return nc;
}

void build_interp(const DCsr& A, const DCsr& G, const SplitResult& sp, int mode, InterpResult& out, cudaStream_t s) {
  const int64_t n = A.nrows, npair = sp.n_pairs(), ni = (int64_t)sp.interior.size();
  StageTimer st(s);
  DBuf<int64_t> pairs(7 * std::max<int64_t>(npair, 1), s), interior(std::max<int64_t>(ni, 1), s);
  if (npair) pairs.upload(sp.pairs.data(), 7 * npair);
  if (ni) interior.upload(sp.interior.data(), ni);
  // R (np x n) and R^T
  DCsr& R = out.R;
  R.alloc(npair, n, 2 * npair, s);
  k_build_R<<<grid_for(npair + 1, 256), 256, 0, s>>>(pairs.p, npair, R.ptr.p, R.idx.p, R.val.p);
  HC_CHECK_LAUNCH();
  DCsr Rt;
  csr_transpose(R, Rt, s);

  DBuf<int32_t> ext_p(n, s), int_pos(n, s), rows32(std::max<int64_t>(ni, 1), s);
  DBuf<double> ext_v(n, s);
  k_fill_i32<<<grid_for(n, 256), 256, 0, s>>>(ext_p.p, n, -1);
  k_fill_i32<<<grid_for(n, 256), 256, 0, s>>>(int_pos.p, n, -1);
  if (npair) k_ext_maps<<<grid_for(npair, 256), 256, 0, s>>>(pairs.p, npair, ext_p.p, ext_v.p);
  if (ni) k_int_maps<<<grid_for(ni, 256), 256, 0, s>>>(interior.p, ni, int_pos.p, rows32.p);
  HC_CHECK_LAUNCH();

  st.mark("  interp: R, maps");
  // component data (empty when there is nothing to extend)
  DBuf<int32_t> label, pos, kcols;
  DBuf<int64_t> cptr, kptr, a_off_d, b_off_d;
  DBuf<double> Ad, Bd;
  out.ncomp = out.max_comp = out.ncomp_large = 0;
  const bool extend = ni > 0 && npair > 0;
  int giant = -1;
  if (extend) {
    DCsr Ai, W0, W, Aii;
    csr_extract(A, rows32.p, ni, nullptr, n, Ai, s);
    spgemm(Ai, Rt, W0, s);          // W = S_I^T A R^T in scipy order (transfer.py:96)
    drop_zeros(W0, W, s);
    W0 = DCsr();
    csr_extract(A, rows32.p, ni, int_pos.p, ni, Aii, s);  // A_II (transfer.py:97)
    Ai = DCsr();
    const int64_t ncomp = connected_components(Aii, label, s);
    out.ncomp = ncomp;
    // members sorted by (component, position)
    DBuf<int32_t> iota(ni, s), members(ni, s), slab(ni, s);
    k_iota32<<<grid_for(ni, 256), 256, 0, s>>>(iota.p, ni);
    HC_CHECK_LAUNCH();
    {
      size_t bytes = 0;
      HC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, label.p, slab.p, iota.p, members.p, ni, 0, 32, s));
      DBuf<unsigned char> ws((int64_t)bytes + 1, s);
      HC_CUDA(cub::DeviceRadixSort::SortPairs(ws.p, bytes, label.p, slab.p, iota.p, members.p, ni, 0, 32, s));
    }
    DBuf<int64_t> ccnt(ncomp, s);
    ccnt.zero();
    k_hist32<<<grid_for(ni, 256), 256, 0, s>>>(label.p, ni, ccnt.p);
    HC_CHECK_LAUNCH();
    cptr.alloc(ncomp + 1, s);
    exclusive_scan(ccnt.p, cptr.p, ncomp, s);
    pos.alloc(ni, s);
    k_pos_in_comp<<<grid_for(ni, 256), 256, 0, s>>>(slab.p, members.p, cptr.p, ni, pos.p);
    HC_CHECK_LAUNCH();
    // keep = nonzero W columns per component (transfer.py:101-102)
    DBuf<unsigned long long> keys(std::max<int64_t>(W.nnz, 1), s), skeys(std::max<int64_t>(W.nnz, 1), s),
        ukeys(std::max<int64_t>(W.nnz, 1), s);
    DBuf<int64_t> nuniq(1, s);
    nuniq.zero();
    if (W.nnz) {
      k_keep_keys<<<grid_for(ni, 256), 256, 0, s>>>(W.ptr.p, W.idx.p, ni, label.p, keys.p);
      HC_CHECK_LAUNCH();
      size_t bytes = 0;
      HC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, keys.p, skeys.p, W.nnz, 0, 64, s));
      DBuf<unsigned char> ws((int64_t)bytes + 1, s);
      HC_CUDA(cub::DeviceRadixSort::SortKeys(ws.p, bytes, keys.p, skeys.p, W.nnz, 0, 64, s));
      size_t b2 = 0;
      HC_CUDA(cub::DeviceSelect::Unique(nullptr, b2, skeys.p, ukeys.p, nuniq.p, W.nnz, s));
      DBuf<unsigned char> ws2((int64_t)b2 + 1, s);
      HC_CUDA(cub::DeviceSelect::Unique(ws2.p, b2, skeys.p, ukeys.p, nuniq.p, W.nnz, s));
    }
    const int64_t nkeep = read_scalar(nuniq.p, s);
    DBuf<int64_t> kcnt(ncomp, s);
    kcnt.zero();
    kcols.alloc(std::max<int64_t>(nkeep, 1), s);
    if (nkeep) k_keep_split<<<grid_for(nkeep, 256), 256, 0, s>>>(ukeys.p, nkeep, kcnt.p, kcols.p);
    HC_CHECK_LAUNCH();
    kptr.alloc(ncomp + 1, s);
    exclusive_scan(kcnt.p, kptr.p, ncomp, s);
    // dense block layout (host bookkeeping of offsets only)
    std::vector<int64_t> hc = cptr.download(), hk = kptr.download();
    std::vector<int64_t> a_off((size_t)ncomp), b_off((size_t)ncomp);
    std::vector<DenseJob> small;
    std::vector<int64_t> small_comp, large_comp;
    // the largest component above the dense-regime cutoff is kept as the
    // resident dense block (hybrid P); any other component, whatever its
    // size, is solved densely and lands in the CSR part of P, as in the
    // reference (transfer.py:100-116)
    for (int64_t c = 0; c < ncomp; ++c) {
      const int64_t k = hc[(size_t)c + 1] - hc[(size_t)c], nk = hk[(size_t)c + 1] - hk[(size_t)c];
      if (nk > 0 && k > opts().giant_min && (giant < 0 || k > hc[(size_t)giant + 1] - hc[(size_t)giant]))
        giant = (int)c;
    }
    int64_t at = 0, bt = 0, pt = 0;
    for (int64_t c = 0; c < ncomp; ++c) {
      const int64_t k = hc[(size_t)c + 1] - hc[(size_t)c], nk = hk[(size_t)c + 1] - hk[(size_t)c];
      out.max_comp = std::max(out.max_comp, k);
      a_off[(size_t)c] = at;
      b_off[(size_t)c] = bt;
      if (nk == 0 || c == giant) continue;
      if (k <= 32) {
        small.push_back(DenseJob{at, bt, pt, (int32_t)k, (int32_t)nk});
        small_comp.push_back(c);
      } else {
        large_comp.push_back(c);
      }
      at += k * k;
      bt += k * nk;
      pt += k;
    }
    out.ncomp_large = (int64_t)large_comp.size();
    a_off_d.upload(a_off.data(), ncomp, s);
    b_off_d.upload(b_off.data(), ncomp, s);
    Ad.alloc(std::max<int64_t>(at, 1), s);
    Bd.alloc(std::max<int64_t>(bt, 1), s);
    Ad.zero();
    Bd.zero();
    k_fill_dense<<<grid_for(ni, 128), 128, 0, s>>>(Aii.ptr.p, Aii.idx.p, Aii.val.p, W.ptr.p, W.idx.p, W.val.p, ni,
                                                   label.p, pos.p, cptr.p, kptr.p, kcols.p, a_off_d.p, b_off_d.p,
                                                   Ad.p, Bd.p, giant);
    HC_CHECK_LAUNCH();
    // solves; failures reported for the first component in component order
    int64_t fail_comp = INT64_MAX, fail_piv = -1;
    if (!small.empty()) {
      DBuf<DenseJob> jobs;
      jobs.upload(small.data(), (int64_t)small.size(), s);
      DBuf<double> piv(std::max<int64_t>(pt, 1), s);
      DBuf<int64_t> status((int64_t)small.size(), s);
      batched_small_spd_solve(jobs.p, (int64_t)small.size(), Ad.p, Bd.p, piv.p, status.p, s);
      std::vector<int64_t> hs = status.download();
      for (size_t t = 0; t < hs.size(); ++t)
        if (hs[t] >= 0 && small_comp[t] < fail_comp) { fail_comp = small_comp[t]; fail_piv = hs[t]; }
    }
    for (int64_t c : large_comp) {
      if (c > fail_comp) break;
      const int64_t k = hc[(size_t)c + 1] - hc[(size_t)c], nk = hk[(size_t)c + 1] - hk[(size_t)c];
      int64_t bad = dense_cholesky(Ad.p + a_off[(size_t)c], k, k, s);
      if (bad >= 0) {
        if (c < fail_comp) { fail_comp = c; fail_piv = bad; }
        break;
      }
      dense_cholesky_solve(Ad.p + a_off[(size_t)c], k, k, Bd.p + b_off[(size_t)c], nk, k, s);
    }
    if (giant >= 0 && giant < fail_comp) {
      // dense-regime component: packed tiled Cholesky, Z kept dense (row-major nG x n_c)
      const int64_t g0 = hc[(size_t)giant], nG = hc[(size_t)giant + 1] - g0;
      HybridP& hp = out.hp;
      hp.on = true;
      hp.nG = nG;
      hp.nc = npair;
      DBuf<int32_t> gmap(ni, s), mpos(nG, s);
      hp.rows.alloc(nG, s);
      k_giant_maps<<<grid_for(std::max<int64_t>(ni, nG), 256), 256, 0, s>>>(label.p, pos.p, ni, giant, gmap.p,
                                                                            members.p + g0, nG, interior.p, mpos.p,
                                                                            hp.rows.p);
      HC_CHECK_LAUNCH();
      csr_extract(Aii, mpos.p, nG, gmap.p, nG, hp.Agg, s);
      csr_extract(W, mpos.p, nG, nullptr, npair, hp.Wg, s);
      st.mark("  interp: components, small solves");
      // single-GPU default: the V-cycle applies A_GG^{-1} through the factor
      // and the Galerkin product needs only Y^T Y (Y = L^{-1} W'), so the
      // 35 GB explicit block Z is not formed (hybrid_ensure_z forms it
      // on demand) -- nor is its dense right-hand side: the solve scatters
      // the rows of W' straight into factored order; explicit-Z apply
      // (factor_apply = 0) or form_z keep it
      const bool fac = factorp_enabled();
      const bool want_z = !fac || opts().form_z;
      if (want_z) {
        hp.Z.alloc(nG * npair, s);
        hp.Z.zero();
        k_giant_rhs<<<grid_for(nG, 128), 128, 0, s>>>(mpos.p, nG, W.ptr.p, W.idx.p, W.val.p, npair, hp.Z.p);
        HC_CHECK_LAUNCH();
      }
      try {
        hp.D.alloc(npair * npair, s);
        giant_factor_solve(hp.Agg, hp.Z.p, npair, s, fac ? &hp.fac : nullptr, hp.D.p, want_z, &hp.Wg);
        if (hp.fac.T) factorp_attach(hp.fac, W, mpos.p, hp.rows.p, s);
      } catch (const Error& e) {
        if (e.code == ENOTSPD_ && giant < fail_comp) { fail_comp = giant; fail_piv = e.index; }
        else throw;
      }
    }
    if (fail_comp != INT64_MAX)
      throw Error(ENOTSPD_, "matrix is not positive definite (pivot " + std::to_string(fail_piv) + ")", fail_piv);
    Ad.release();
  }
  st.mark("  interp: components + solves");
  // assemble P = R^T + correction (transfer.py:111-116)
  DCsr& P = out.P;
  P.nrows = n;
  P.ncols = npair;
  P.ptr.alloc(n + 1, s);
  DBuf<int64_t> pc(n, s);
  int32_t* lab_p = extend ? label.p : nullptr;
  if (n)
    k_assemble_P<false><<<grid_for(n, 128), 128, 0, s>>>(n, ext_p.p, ext_v.p, int_pos.p, lab_p,
                                                         pos.p, cptr.p, kptr.p, kcols.p, b_off_d.p, Bd.p, giant, pc.p,
                                                         nullptr, nullptr, nullptr);
  HC_CHECK_LAUNCH();
  P.nnz = exclusive_scan(pc.p, P.ptr.p, n, s);
  P.idx.alloc(P.nnz, s);
  P.val.alloc(P.nnz, s);
  if (n)
    k_assemble_P<true><<<grid_for(n, 128), 128, 0, s>>>(n, ext_p.p, ext_v.p, int_pos.p, lab_p,
                                                        pos.p, cptr.p, kptr.p, kcols.p, b_off_d.p, Bd.p, giant, nullptr,
                                                        P.ptr.p, P.idx.p, P.val.p);
  HC_CHECK_LAUNCH();
  csr_transpose(P, out.Pt, s);

  st.mark("  interp: P assembly + P^T");
  // coarse gradient (transfer.py:55-74) + sign normalisation (multilevel.py:71-75)
  DCsr RG0, RG;
  spgemm(R, G, RG0, s);
  drop_zeros(RG0, RG, s);
  const int64_t m = G.ncols;
  DBuf<int64_t> ccnt(m, s), flag(m, s), rank(m + 1, s);
  ccnt.zero();
  if (RG.nnz) k_col_count<<<grid_for(RG.nnz, 256), 256, 0, s>>>(RG.idx.p, RG.nnz, ccnt.p);
  DBuf<int64_t> cand(std::max<int64_t>((int64_t)sp.coarse_nodes.size(), 1), s);
  if (!sp.coarse_nodes.empty()) cand.upload(sp.coarse_nodes.data(), (int64_t)sp.coarse_nodes.size(), s);
  if (m) {
    if (mode == 1) flag.zero();
    k_gc_keep<<<grid_for(std::max<int64_t>(m, 1), 256), 256, 0, s>>>(ccnt.p, m, cand.p,
                                                                     (int64_t)sp.coarse_nodes.size(), mode, flag.p);
    HC_CHECK_LAUNCH();
  }
  int64_t nkept = exclusive_scan(flag.p, rank.p, m, s);
  DBuf<int32_t> cmap(std::max<int64_t>(m, 1), s);
  if (m) k_colmap<<<grid_for(m, 256), 256, 0, s>>>(flag.p, rank.p, m, cmap.p);
  HC_CHECK_LAUNCH();
  csr_extract(RG, nullptr, npair, cmap.p, nkept, out.Gc, s);
  if (out.Gc.nnz) k_sign<<<grid_for(out.Gc.nnz, 256), 256, 0, s>>>(out.Gc.val.p, out.Gc.nnz);
  HC_CHECK_LAUNCH();
  DBuf<int64_t> kept;
  compact_flags(flag.p, m, kept, s);
  out.gc_cols = kept.download();
}

}  // namespace hcamg
