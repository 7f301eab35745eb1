// OSS-l1 smoother setup on the GPU (hcurl_amg/smoothers.py:50-95):
//   * vertex patches read off the level gradient (column v of G), singletons
//     for uncovered DoFs (smoothers.py:60-76);
//   * explicit inverses of the patch blocks A[patch, patch] (smoothers.py:78-89;
//     breakdown -> NotPositiveDefiniteError(pivot, "singular patch block id"));
//   * the wavefront schedule that reproduces the multiplicative sweep order
//     exactly: patch q waits for every earlier patch p with
//     patch_q ∩ upd_p ≠ ∅ or upd_q ∩ patch_p ≠ ∅ (smoothers.py:98-103);
//   * gather ("pull") lists for the lazily applied residual updates;
//   * the l1 diagonal d_i = sum_j |a_ij| (smoothers.py:50-52).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <thread>

#include "dense.cuh"
#include "smoother.cuh"

namespace hcamg {

namespace {

__global__ void k_nonempty(const int64_t* __restrict__ p, int64_t n, int64_t* __restrict__ f, int want_empty) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    bool ne = p[i + 1] > p[i];
    f[i] = want_empty ? !ne : ne;
  }
}

__global__ void k_patch_sizes(const int64_t* __restrict__ gtp, const int64_t* __restrict__ vcols, int64_t nv,
                              int64_t m, int64_t* __restrict__ sz) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x)
    sz[t] = t < nv ? gtp[vcols[t] + 1] - gtp[vcols[t]] : 1;
}

__global__ void k_patch_fill(const int64_t* __restrict__ gtp, const int32_t* __restrict__ gti,
                             const int64_t* __restrict__ vcols, int64_t nv, const int64_t* __restrict__ singles,
                             int64_t m, const int64_t* __restrict__ pp, int32_t* __restrict__ dofs) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = pp[t];
    if (t < nv) {
      int64_t c = vcols[t];
      for (int64_t e = gtp[c]; e < gtp[c + 1]; ++e) dofs[o++] = gti[e];
    } else {
      dofs[o] = (int32_t)singles[t - nv];
    }
  }
}

__global__ void k_patch_blocks(const int64_t* __restrict__ ap, const int32_t* __restrict__ ai,
                               const double* __restrict__ av, const int64_t* __restrict__ pp,
                               const int32_t* __restrict__ dofs, int64_t m, const int64_t* __restrict__ boff,
                               double* __restrict__ blk) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p0 = pp[t], k = pp[t + 1] - p0;
    double* B = blk + boff[t];
    for (int64_t a = 0; a < k; ++a) {
      const int32_t i = dofs[p0 + a];
      int64_t b = 0;
      for (int64_t e = ap[i]; e < ap[i + 1]; ++e) {
        const int32_t j = ai[e];
        while (b < k && dofs[p0 + b] < j) ++b;
        if (b == k) break;
        if (dofs[p0 + b] == j) B[a + b * k] = av[e];
      }
    }
  }
}

__global__ void k_jobs(const int64_t* __restrict__ pp, const int64_t* __restrict__ boff, int64_t m,
                       DenseJob* __restrict__ jobs) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
    int32_t k = (int32_t)(pp[t + 1] - pp[t]);
    jobs[t] = DenseJob{boff[t], boff[t], pp[t], k, k};
  }
}

__global__ void k_sq(const int64_t* __restrict__ pp, int64_t m, int64_t* __restrict__ o) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t k = pp[t + 1] - pp[t];
    o[t] = k * k;
  }
}

// Wavefront levels: level[q] = 1 + max level of the earlier patches q is
// A-coupled to (0 if none) -- the longest path of the sweep's dependency DAG.
// Computed as a monotone fixed point: every pass raises level[q] to what its
// earlier coupled patches currently imply (in place; values only grow and stop
// at the longest path), so it converges in at most as many passes as there are
// waves (7-10 in 2D, ~3n in 3D) where the sequential walk of round 1 took 6 us
// per patch on one warp (7 s at 10^6 patches).  A is structurally symmetric,
// so "coupled" is "contains a DoF of a row of A^T that a DoF of q indexes".
__global__ void k_entry_patch(const int64_t* __restrict__ pp, int64_t m, int32_t* __restrict__ pe) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x)
    for (int64_t e = pp[q]; e < pp[q + 1]; ++e) pe[e] = (int32_t)q;
}

__global__ void k_lower_bounds(const int32_t* __restrict__ keys, int64_t nk, int64_t n, int64_t* __restrict__ ptr) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j <= n; j += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = nk;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < j) lo = mid + 1; else hi = mid;
    }
    ptr[j] = lo;
  }
}

__global__ void k_wave_relax(const int64_t* __restrict__ pp, const int32_t* __restrict__ dofs, int64_t m,
                             const int64_t* __restrict__ atp, const int32_t* __restrict__ ati,
                             const int64_t* __restrict__ mem_ptr, const int32_t* __restrict__ mem_patch,
                             int32_t* level, int* changed) {
  const int lane = threadIdx.x & 31;
  for (int64_t q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; q < m;
       q += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    int lv = 0;
    for (int64_t e = pp[q]; e < pp[q + 1]; ++e) {
      const int32_t i = dofs[e];
      for (int64_t f = atp[i] + lane; f < atp[i + 1]; f += 32) {
        const int32_t j = ati[f];
        for (int64_t t = mem_ptr[j]; t < mem_ptr[j + 1]; ++t) {
          const int32_t p = mem_patch[t];
          if (p < q) lv = max(lv, ((volatile int32_t*)level)[p] + 1);
        }
      }
    }
    for (int o = 16; o; o >>= 1) lv = max(lv, __shfl_xor_sync(0xffffffffu, lv, o));
    if (lane == 0 && lv > level[q]) {
      level[q] = lv;
      *changed = 1;
    }
  }
}

__global__ void k_iota_i32(int32_t* v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) v[i] = (int32_t)i;
}

__global__ void k_reorder_sizes(const int32_t* __restrict__ order, const int64_t* __restrict__ pp, int64_t m,
                                int64_t* __restrict__ sz, int64_t* __restrict__ sq) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t k = pp[order[t] + 1] - pp[order[t]];
    sz[t] = k;
    sq[t] = k * k;
  }
}

__global__ void k_reorder_fill(const int32_t* __restrict__ order, const int64_t* __restrict__ pp,
                               const int32_t* __restrict__ dofs, const int64_t* __restrict__ boff,
                               const double* __restrict__ binv, int64_t m, const int64_t* __restrict__ npp,
                               const int64_t* __restrict__ nboff, int32_t* __restrict__ ndofs,
                               double* __restrict__ nbinv, const int32_t* __restrict__ level,
                               unsigned long long* __restrict__ mkeys, int32_t* __restrict__ mvals) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t q = order[t];
    const int64_t k = pp[q + 1] - pp[q];
    const unsigned long long w = (unsigned long long)(uint32_t)level[q];
    for (int64_t a = 0; a < k; ++a) {
      const int32_t dof = dofs[pp[q] + a];
      ndofs[npp[t] + a] = dof;
      mkeys[npp[t] + a] = (w << 32) | (uint32_t)dof;
      mvals[npp[t] + a] = (int32_t)(npp[t] + a);
    }
    for (int64_t e = 0; e < k * k; ++e) nbinv[nboff[t] + e] = binv[boff[q] + e];
  }
}

__global__ void k_entry_wave(const int64_t* __restrict__ npp, const int32_t* __restrict__ order,
                             const int32_t* __restrict__ level, int64_t m, int32_t* __restrict__ ewave) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x)
    for (int64_t e = npp[t]; e < npp[t + 1]; ++e) ewave[e] = level[order[t]];
}

__global__ void k_trip_count(const int32_t* __restrict__ ndofs, int64_t ne, const int64_t* __restrict__ atp,
                             int64_t* __restrict__ cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
    int32_t j = ndofs[e];
    cnt[e] = atp[j + 1] - atp[j];
  }
}

__global__ void k_trip_fill(const int32_t* __restrict__ ndofs, const int32_t* __restrict__ ewave, int64_t ne,
                            const int64_t* __restrict__ atp, const int32_t* __restrict__ ati,
                            const double* __restrict__ atv, const int64_t* __restrict__ toff,
                            unsigned long long* __restrict__ tkeys, int32_t* __restrict__ tcol,
                            double* __restrict__ tval, int32_t* __restrict__ tid) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t j = ndofs[e];
    const unsigned long long w = (unsigned long long)(uint32_t)ewave[e];
    int64_t o = toff[e];
    for (int64_t f = atp[j]; f < atp[j + 1]; ++f, ++o) {
      tkeys[o] = (w << 32) | (uint32_t)ati[f];  // row u = ati[f], value A[u, j] = atv[f]
      tcol[o] = j;
      tval[o] = atv[f];
      tid[o] = (int32_t)o;
    }
  }
}

__global__ void k_trip_gather(const int32_t* __restrict__ perm, const int32_t* __restrict__ tcol,
                              const double* __restrict__ tval, int64_t nt, int32_t* __restrict__ gcol,
                              double* __restrict__ gval) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nt; t += (int64_t)gridDim.x * blockDim.x) {
    gcol[t] = tcol[perm[t]];
    gval[t] = tval[perm[t]];
  }
}

__device__ __forceinline__ int64_t find_key(const unsigned long long* __restrict__ keys, int64_t n,
                                            unsigned long long k) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < k) lo = mid + 1; else hi = mid;
  }
  return (lo < n && keys[lo] == k) ? lo : -1;
}

// Classify gather rows (w, u) for both sweep directions.
__global__ void k_classify(const unsigned long long* __restrict__ gkeys, int64_t ng,
                           const unsigned long long* __restrict__ mkeys, const int32_t* __restrict__ mvals,
                           int64_t nm, int64_t nwave, int32_t* __restrict__ own_fw, int32_t* __restrict__ own_bw,
                           int64_t* __restrict__ gen_fw_flag, int64_t* __restrict__ gen_bw_flag,
                           int32_t* __restrict__ last_row, int32_t* __restrict__ grow_u) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < ng; r += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long key = gkeys[r];
    const int64_t w = (int64_t)(key >> 32);
    const uint32_t u = (uint32_t)(key & 0xffffffffull);
    grow_u[r] = (int32_t)u;
    gen_fw_flag[r] = 0;
    gen_bw_flag[r] = 0;
    if (w + 1 < nwave) {
      int64_t at = find_key(mkeys, nm, ((unsigned long long)(w + 1) << 32) | u);
      if (at >= 0) own_fw[mvals[at]] = (int32_t)r; else gen_fw_flag[r] = 1;
    } else {
      last_row[u] = (int32_t)r;
    }
    if (w >= 1) {
      int64_t at = find_key(mkeys, nm, ((unsigned long long)(w - 1) << 32) | u);
      if (at >= 0) own_bw[mvals[at]] = (int32_t)r; else gen_bw_flag[r] = 1;
    }
  }
}

__global__ void k_to_i32(const int64_t* __restrict__ a, int64_t n, int32_t* __restrict__ o) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    o[i] = (int32_t)a[i];
}

__global__ void k_wave_hist(const unsigned long long* __restrict__ gkeys, const int64_t* __restrict__ list,
                            int64_t n, int64_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd((unsigned long long*)&cnt[gkeys[list[i]] >> 32], 1ull);
}

__global__ void k_in_first(const unsigned long long* __restrict__ mkeys, int64_t nm, uint8_t* __restrict__ f) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nm; i += (int64_t)gridDim.x * blockDim.x)
    if ((mkeys[i] >> 32) == 0) f[mkeys[i] & 0xffffffffull] = 1;
}

__global__ void k_flat_gen(const int32_t* __restrict__ gen, int64_t n, const int32_t* __restrict__ grow_u,
                           const int64_t* __restrict__ gp, int32_t* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = gen[t];
    out[3 * t] = grow_u[r];
    out[3 * t + 1] = (int32_t)gp[r];
    out[3 * t + 2] = (int32_t)gp[r + 1];
  }
}

__global__ void k_flat_range(const int32_t* __restrict__ rho, int64_t n, const int64_t* __restrict__ gp,
                             int32_t* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = rho[t];
    out[2 * t] = r >= 0 ? (int32_t)gp[r] : -1;
    out[2 * t + 1] = r >= 0 ? (int32_t)gp[r + 1] : -1;
  }
}

__global__ void k_l1(const int64_t* __restrict__ ap, const double* __restrict__ av, int64_t n, double* __restrict__ d) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t e = ap[r]; e < ap[r + 1]; ++e) s = __dadd_rn(s, fabs(av[e]));
    d[r] = s;
  }
}

}  // namespace

void build_l1(const DCsr& A, DBuf<double>& l1, cudaStream_t s) {
  l1.alloc(A.nrows, s);
  if (A.nrows) k_l1<<<grid_for(A.nrows, 256), 256, 0, s>>>(A.ptr.p, A.val.p, A.nrows, l1.p);
  HC_CHECK_LAUNCH();
}

void build_smoother(const DCsr& A, const DCsr& G, Smoother& sm, cudaStream_t s) {
  const int64_t n = A.nrows;
  require(G.nrows == n, "smoother: gradient rows do not match the operator");
  DCsr GT, AT;
  csr_transpose(G, GT, s);
  csr_transpose(A, AT, s);
  // ---- patches in reference order
  DBuf<int64_t> fcol(std::max<int64_t>(G.ncols, 1), s), frow(std::max<int64_t>(n, 1), s);
  if (G.ncols) k_nonempty<<<grid_for(G.ncols, 256), 256, 0, s>>>(GT.ptr.p, G.ncols, fcol.p, 0);
  if (n) k_nonempty<<<grid_for(n, 256), 256, 0, s>>>(G.ptr.p, n, frow.p, 1);
  HC_CHECK_LAUNCH();
  DBuf<int64_t> vcols, singles;
  const int64_t nv = compact_flags(fcol.p, G.ncols, vcols, s);
  const int64_t nsg = compact_flags(frow.p, n, singles, s);
  const int64_t m = nv + nsg;
  sm.npatch = m;
  DBuf<int64_t> sz(std::max<int64_t>(m, 1), s), pp(m + 1, s);
  if (m) k_patch_sizes<<<grid_for(m, 256), 256, 0, s>>>(GT.ptr.p, vcols.p, nv, m, sz.p);
  HC_CHECK_LAUNCH();
  const int64_t ne = exclusive_scan(sz.p, pp.p, m, s);
  DBuf<int32_t> dofs(std::max<int64_t>(ne, 1), s);
  if (m) k_patch_fill<<<grid_for(m, 256), 256, 0, s>>>(GT.ptr.p, GT.idx.p, vcols.p, nv, singles.p, m, pp.p, dofs.p);
  HC_CHECK_LAUNCH();
  sm.h_patch_ptr = pp.download();
  {
    std::vector<int32_t> hd = dofs.download();
    sm.h_patch_dofs.assign(hd.begin(), hd.begin() + ne);
  }
  sm.kmax = 0;
  for (int64_t t = 0; t < m; ++t) sm.kmax = std::max(sm.kmax, sm.h_patch_ptr[(size_t)t + 1] - sm.h_patch_ptr[(size_t)t]);
  if (sm.kmax > 32) throw Error(EUNSUPPORTED_, "patch with more than 32 DoFs (" + std::to_string(sm.kmax) + ")");
  // ---- patch inverses (reference order)
  DBuf<int64_t> sq(std::max<int64_t>(m, 1), s), boff(m + 1, s);
  if (m) k_sq<<<grid_for(m, 256), 256, 0, s>>>(pp.p, m, sq.p);
  HC_CHECK_LAUNCH();
  const int64_t nb = exclusive_scan(sq.p, boff.p, m, s);
  DBuf<double> blk(std::max<int64_t>(nb, 1), s), binv(std::max<int64_t>(nb, 1), s), piv(std::max<int64_t>(ne, 1), s);
  blk.zero();
  DBuf<DenseJob> jobs(std::max<int64_t>(m, 1), s);
  DBuf<int64_t> status(std::max<int64_t>(m, 1), s);
  if (m) {
    k_patch_blocks<<<grid_for(m, 128), 128, 0, s>>>(A.ptr.p, A.idx.p, A.val.p, pp.p, dofs.p, m, boff.p, blk.p);
    k_jobs<<<grid_for(m, 256), 256, 0, s>>>(pp.p, boff.p, m, jobs.p);
    HC_CHECK_LAUNCH();
    batched_small_spd_inverse(jobs.p, m, blk.p, binv.p, piv.p, status.p, s);
    std::vector<int64_t> hs = status.download();
    for (int64_t t = 0; t < m; ++t)
      if (hs[(size_t)t] >= 0)
        throw Error(ENOTSPD_, "singular patch block " + std::to_string(t), hs[(size_t)t]);
  }
  blk.release();
  // ---- wavefront levels
  DBuf<int32_t> level(std::max<int64_t>(m, 1), s);
  level.zero();
  if (m) {
    // DoF -> patches containing it
    DBuf<int32_t> pe(std::max<int64_t>(ne, 1), s), skey(std::max<int64_t>(ne, 1), s), mem_patch(std::max<int64_t>(ne, 1), s);
    DBuf<int64_t> mem_ptr(n + 1, s);
    k_entry_patch<<<grid_for(m, 256), 256, 0, s>>>(pp.p, m, pe.p);
    HC_CHECK_LAUNCH();
    {
      size_t bytes = 0;
      HC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, dofs.p, skey.p, pe.p, mem_patch.p, ne, 0, 32, s));
      DBuf<unsigned char> ws((int64_t)bytes + 1, s);
      HC_CUDA(cub::DeviceRadixSort::SortPairs(ws.p, bytes, dofs.p, skey.p, pe.p, mem_patch.p, ne, 0, 32, s));
    }
    k_lower_bounds<<<grid_for(n + 1, 256), 256, 0, s>>>(skey.p, ne, n, mem_ptr.p);
    HC_CHECK_LAUNCH();
    DBuf<int> changed(1, s);
    for (int64_t pass = 0; pass <= m; ++pass) {
      changed.zero();
      k_wave_relax<<<grid_for(m * 32, 256), 256, 0, s>>>(pp.p, dofs.p, m, AT.ptr.p, AT.idx.p, mem_ptr.p,
                                                         mem_patch.p, level.p, changed.p);
      HC_CHECK_LAUNCH();
      if (!read_scalar(changed.p, s)) break;
    }
  }
  // ---- reorder wave-major (stable in reference order)
  DBuf<int32_t> iota(std::max<int64_t>(m, 1), s), order(std::max<int64_t>(m, 1), s), slev(std::max<int64_t>(m, 1), s);
  if (m) {
    k_iota_i32<<<grid_for(m, 256), 256, 0, s>>>(iota.p, m);
    HC_CHECK_LAUNCH();
    size_t bytes = 0;
    HC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, level.p, slev.p, iota.p, order.p, m, 0, 32, s));
    DBuf<unsigned char> ws((int64_t)bytes + 1, s);
    HC_CUDA(cub::DeviceRadixSort::SortPairs(ws.p, bytes, level.p, slev.p, iota.p, order.p, m, 0, 32, s));
  }
  std::vector<int32_t> hslev = slev.download();
  std::vector<int32_t> horder = order.download();
  sm.nwave = m ? (int64_t)hslev[(size_t)m - 1] + 1 : 0;
  sm.wave_ptr.assign((size_t)sm.nwave + 1, 0);
  for (int64_t t = 0; t < m; ++t) sm.wave_ptr[(size_t)hslev[(size_t)t] + 1]++;
  for (int64_t w = 0; w < sm.nwave; ++w) sm.wave_ptr[(size_t)w + 1] += sm.wave_ptr[(size_t)w];
  sm.orig_of.assign(horder.begin(), horder.begin() + m);
  DBuf<int64_t> nsz(std::max<int64_t>(m, 1), s), nsq(std::max<int64_t>(m, 1), s);
  sm.patch_ptr.alloc(m + 1, s);
  sm.binv_off.alloc(m + 1, s);
  if (m) k_reorder_sizes<<<grid_for(m, 256), 256, 0, s>>>(order.p, pp.p, m, nsz.p, nsq.p);
  HC_CHECK_LAUNCH();
  exclusive_scan(nsz.p, sm.patch_ptr.p, m, s);
  exclusive_scan(nsq.p, sm.binv_off.p, m, s);
  sm.patch_dofs.alloc(std::max<int64_t>(ne, 1), s);
  sm.binv.alloc(std::max<int64_t>(nb, 1), s);
  DBuf<unsigned long long> mkeys_in(std::max<int64_t>(ne, 1), s), mkeys(std::max<int64_t>(ne, 1), s);
  DBuf<int32_t> mvals_in(std::max<int64_t>(ne, 1), s), mvals(std::max<int64_t>(ne, 1), s);
  if (m)
    k_reorder_fill<<<grid_for(m, 128), 128, 0, s>>>(order.p, pp.p, dofs.p, boff.p, binv.p, m, sm.patch_ptr.p,
                                                    sm.binv_off.p, sm.patch_dofs.p, sm.binv.p, level.p, mkeys_in.p,
                                                    mvals_in.p);
  HC_CHECK_LAUNCH();
  binv.release();
  // membership (wave, dof) -> entry, sorted
  if (ne) {
    size_t bytes = 0;
    HC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, mkeys_in.p, mkeys.p, mvals_in.p, mvals.p, ne, 0, 64, s));
    DBuf<unsigned char> ws((int64_t)bytes + 1, s);
    HC_CUDA(cub::DeviceRadixSort::SortPairs(ws.p, bytes, mkeys_in.p, mkeys.p, mvals_in.p, mvals.p, ne, 0, 64, s));
  }
  // ---- gather triples (w, u, j, A[u, j]) over every patch entry
  DBuf<int32_t> ewave(std::max<int64_t>(ne, 1), s);
  if (m) k_entry_wave<<<grid_for(m, 256), 256, 0, s>>>(sm.patch_ptr.p, order.p, level.p, m, ewave.p);
  DBuf<int64_t> tcnt(std::max<int64_t>(ne, 1), s), toff(ne + 1, s);
  if (ne) k_trip_count<<<grid_for(ne, 256), 256, 0, s>>>(sm.patch_dofs.p, ne, AT.ptr.p, tcnt.p);
  HC_CHECK_LAUNCH();
  const int64_t nt = exclusive_scan(tcnt.p, toff.p, ne, s);
  require(nt < (int64_t(1) << 31), "smoother gather lists exceed int32 indexing");
  DBuf<unsigned long long> tkeys(std::max<int64_t>(nt, 1), s), skeys(std::max<int64_t>(nt, 1), s);
  DBuf<int32_t> tcol(std::max<int64_t>(nt, 1), s), tid(std::max<int64_t>(nt, 1), s), perm(std::max<int64_t>(nt, 1), s);
  DBuf<double> tval(std::max<int64_t>(nt, 1), s);
  if (ne) k_trip_fill<<<grid_for(ne, 128), 128, 0, s>>>(sm.patch_dofs.p, ewave.p, ne, AT.ptr.p, AT.idx.p, AT.val.p,
                                                       toff.p, tkeys.p, tcol.p, tval.p, tid.p);
  HC_CHECK_LAUNCH();
  if (nt) {
    size_t bytes = 0;
    HC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, tkeys.p, skeys.p, tid.p, perm.p, nt, 0, 64, s));
    DBuf<unsigned char> ws((int64_t)bytes + 1, s);
    HC_CUDA(cub::DeviceRadixSort::SortPairs(ws.p, bytes, tkeys.p, skeys.p, tid.p, perm.p, nt, 0, 64, s));
  }
  sm.gcol.alloc(std::max<int64_t>(nt, 1), s);
  sm.gval.alloc(std::max<int64_t>(nt, 1), s);
  if (nt) k_trip_gather<<<grid_for(nt, 256), 256, 0, s>>>(perm.p, tcol.p, tval.p, nt, sm.gcol.p, sm.gval.p);
  HC_CHECK_LAUNCH();
  // run-length encode the sorted keys -> gather rows
  DBuf<unsigned long long> gkeys(std::max<int64_t>(nt, 1), s);
  DBuf<int64_t> gcnt(std::max<int64_t>(nt, 1), s), ngr(1, s);
  ngr.zero();
  if (nt) {
    size_t bytes = 0;
    HC_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, bytes, skeys.p, gkeys.p, gcnt.p, ngr.p, nt, s));
    DBuf<unsigned char> ws((int64_t)bytes + 1, s);
    HC_CUDA(cub::DeviceRunLengthEncode::Encode(ws.p, bytes, skeys.p, gkeys.p, gcnt.p, ngr.p, nt, s));
  }
  const int64_t ng = read_scalar(ngr.p, s);
  sm.grow_ptr.alloc(ng + 1, s);
  exclusive_scan(gcnt.p, sm.grow_ptr.p, ng, s);
  sm.grow_u.alloc(std::max<int64_t>(ng, 1), s);
  sm.own_fw.alloc(std::max<int64_t>(ne, 1), s);
  sm.own_bw.alloc(std::max<int64_t>(ne, 1), s);
  sm.last_row.alloc(std::max<int64_t>(n, 1), s);
  sm.own_fw.fill_bytes(0xff);
  sm.own_bw.fill_bytes(0xff);
  sm.last_row.fill_bytes(0xff);
  DBuf<int64_t> gff(std::max<int64_t>(ng, 1), s), gbf(std::max<int64_t>(ng, 1), s);
  if (ng)
    k_classify<<<grid_for(ng, 256), 256, 0, s>>>(gkeys.p, ng, mkeys.p, mvals.p, ne, sm.nwave, sm.own_fw.p,
                                                 sm.own_bw.p, gff.p, gbf.p, sm.last_row.p, sm.grow_u.p);
  HC_CHECK_LAUNCH();
  for (int dir = 0; dir < 2; ++dir) {
    DBuf<int64_t> lst;
    const int64_t cnt = compact_flags(dir == 0 ? gff.p : gbf.p, ng, lst, s);
    DBuf<int64_t> wh(std::max<int64_t>(sm.nwave, 1), s), wp(sm.nwave + 1, s);
    wh.zero();
    if (cnt) k_wave_hist<<<grid_for(cnt, 256), 256, 0, s>>>(gkeys.p, lst.p, cnt, wh.p);
    HC_CHECK_LAUNCH();
    exclusive_scan(wh.p, wp.p, sm.nwave, s);
    DBuf<int32_t>& out = dir == 0 ? sm.gen_fw : sm.gen_bw;
    out.alloc(std::max<int64_t>(cnt, 1), s);
    if (cnt) k_to_i32<<<grid_for(cnt, 256), 256, 0, s>>>(lst.p, cnt, out.p);
    HC_CHECK_LAUNCH();
    (dir == 0 ? sm.gen_fw_ptr : sm.gen_bw_ptr) = wp.download();
  }
  sm.in_first.alloc(std::max<int64_t>(n, 1), s);
  sm.in_first.zero();
  if (ne) k_in_first<<<grid_for(ne, 256), 256, 0, s>>>(mkeys.p, ne, sm.in_first.p);
  HC_CHECK_LAUNCH();
  // flattened layout for the cluster sweep
  for (int dir = 0; dir < 2; ++dir) {
    const std::vector<int64_t>& gp = dir == 0 ? sm.gen_fw_ptr : sm.gen_bw_ptr;
    const int64_t cnt = gp.back();
    DBuf<int32_t>& out = dir == 0 ? sm.genrow_fw : sm.genrow_bw;
    out.alloc(3 * std::max<int64_t>(cnt, 1), s);
    if (cnt) k_flat_gen<<<grid_for(cnt, 256), 256, 0, s>>>(dir == 0 ? sm.gen_fw.p : sm.gen_bw.p, cnt, sm.grow_u.p,
                                                          sm.grow_ptr.p, out.p);
    DBuf<int32_t>& ow = dir == 0 ? sm.ownr_fw : sm.ownr_bw;
    ow.alloc(2 * std::max<int64_t>(ne, 1), s);
    if (ne) k_flat_range<<<grid_for(ne, 256), 256, 0, s>>>(dir == 0 ? sm.own_fw.p : sm.own_bw.p, ne, sm.grow_ptr.p,
                                                          ow.p);
    HC_CHECK_LAUNCH();
  }
  sm.lastr.alloc(2 * std::max<int64_t>(n, 1), s);
  if (n) k_flat_range<<<grid_for(n, 256), 256, 0, s>>>(sm.last_row.p, n, sm.grow_ptr.p, sm.lastr.p);
  HC_CHECK_LAUNCH();
  sm.d_wave_ptr.upload(sm.wave_ptr.data(), (int64_t)sm.wave_ptr.size(), s);
  sm.d_gen_fw_ptr.upload(sm.gen_fw_ptr.data(), (int64_t)sm.gen_fw_ptr.size(), s);
  sm.d_gen_bw_ptr.upload(sm.gen_bw_ptr.data(), (int64_t)sm.gen_bw_ptr.size(), s);
  build_program(sm, sm.pg, s);
  sm.max_wave_patches = sm.max_gen_rows = 0;
  for (int64_t w = 0; w < sm.nwave; ++w) {
    sm.max_wave_patches = std::max(sm.max_wave_patches, sm.wave_ptr[(size_t)w + 1] - sm.wave_ptr[(size_t)w]);
    sm.max_gen_rows = std::max(sm.max_gen_rows, sm.gen_fw_ptr[(size_t)w + 1] - sm.gen_fw_ptr[(size_t)w]);
    sm.max_gen_rows = std::max(sm.max_gen_rows, sm.gen_bw_ptr[(size_t)w + 1] - sm.gen_bw_ptr[(size_t)w]);
  }
  if (smoother_flow_auto(sm) || smoother_wave_auto(sm) || opts().sweep == SWEEP_FLOW || opts().sweep == SWEEP_FWAVE)
    build_flow(A, sm, s);
  HC_CUDA(cudaStreamSynchronize(s));
}

bool smoother_wide(const Smoother& sm) { return sm.max_wave_patches > 256 || sm.max_gen_rows > 8192; }

// The dataflow leg pays off on deep, narrow DAGs (3D Kuhn: ~3n waves, ~13
// patches per warp on config 2); on shallow, wide ones (2D: 7 waves, 100+
// patches per warp at L = 9) a warp's serial walk over its patches dominates
// and the grid leg's 7 barriers are cheaper.
// Shallow, very wide schedules (2D: 7-10 waves of up to tens of thousands of
// patches): one full-GPU launch per wavefront, several patches per warp.  The
// cooperative grid leg gives each warp one fast patch per wave and walks the
// rest serially; it is the right shape only while a wave fits its warps.
bool smoother_wave_auto(const Smoother& sm) {
  return sm.nwave > 0 && sm.max_wave_patches > (int64_t)kSMs * 16 && sm.npatch / sm.nwave > (int64_t)kSMs * 8;
}

bool smoother_flow_auto(const Smoother& sm) {
  return smoother_wide(sm) && sm.npatch <= 16 * (int64_t)kSMs * 16 && sm.nwave >= 16;
}

// Pulled terms of the dataflow leg (flow.cu).  Entry e = (patch q, DoF u) of
// the wave-major patch list pulls, for every j coupled to u and every entry
// e' = (patch p, DoF j) of a patch p != q that runs before q in the sweep
// direction, the term (e', A[u, j]): the reference's residual update
// r[upd_p] -= A[upd_p, patch_p] d_p (smoothers.py:101-103) restricted to the
// rows q reads, in the order q sees them.  Conflicting patches lie in
// different waves, and for them "runs before" is "lower wave" (forward) /
// "higher wave" (backward).  Host C++, once per level.
void build_flow(const DCsr& A, Smoother& sm, cudaStream_t s) {
  FlowProgram& f = sm.fl;
  if (f.built) return;
  const int64_t n = A.nrows, m = sm.npatch;
  if (m == 0) return;
  const std::vector<int64_t> pp = sm.patch_ptr.download();
  const int64_t ne = pp[(size_t)m];
  const std::vector<int32_t> dofs = sm.patch_dofs.download();
  const std::vector<int64_t> ap = A.ptr.download();
  const std::vector<int32_t> ai = A.idx.download();
  const std::vector<double> av = A.val.download();
  std::vector<int32_t> lev((size_t)m), pe((size_t)ne);
  for (int64_t w = 0; w < sm.nwave; ++w)
    for (int64_t t = sm.wave_ptr[(size_t)w]; t < sm.wave_ptr[(size_t)w + 1]; ++t) lev[(size_t)t] = (int32_t)w;
  for (int64_t t = 0; t < m; ++t)
    for (int64_t e = pp[(size_t)t]; e < pp[(size_t)t + 1]; ++e) pe[(size_t)e] = (int32_t)t;
  std::vector<int2> ent((size_t)n, make_int2(-1, -1));
  for (int64_t e = 0; e < ne; ++e) {
    int2& en = ent[(size_t)dofs[(size_t)e]];
    if (en.x < 0) en.x = (int32_t)e;
    else if (en.y < 0) en.y = (int32_t)e;
    else return;  // a DoF in more than two patches: the flow leg does not apply (grid leg instead)
  }
  const std::vector<int64_t> boff = sm.binv_off.download();
  const std::vector<double> binv = sm.binv.download();
  std::vector<std::vector<unsigned char>> recs(2);
  std::vector<std::vector<int64_t>> offs(2);
  int64_t rmax[2] = {0, 0};
  bool okdir[2] = {true, true};
  // the two directions are independent: built on two host threads
  auto build_dir = [&](int dir) {
    // execution order: waves ascending (forward) / descending (backward), patches ascending within a wave
    std::vector<int64_t> order;
    order.reserve((size_t)m);
    for (int64_t s0 = 0; s0 < sm.nwave; ++s0) {
      const int64_t w = dir == 0 ? s0 : sm.nwave - 1 - s0;
      for (int64_t t = sm.wave_ptr[(size_t)w]; t < sm.wave_ptr[(size_t)w + 1]; ++t) order.push_back(t);
    }
    std::vector<unsigned char>& R = recs[(size_t)dir];
    std::vector<int64_t>& off = offs[(size_t)dir];
    off.assign(1, 0);
    std::vector<int32_t> ts, tstart, xpart;
    std::vector<double> tv;
    for (int64_t q : order) {
      const int64_t e0 = pp[(size_t)q], k = pp[(size_t)q + 1] - e0;
      const int32_t lq = lev[(size_t)q];
      ts.clear();
      tv.clear();
      tstart.assign(1, 0);
      xpart.clear();
      int32_t glev = dir == 0 ? -1 : INT32_MAX;
      std::vector<std::pair<int32_t, int32_t>> gates;  // (predecessor patch, one of its slots) of the latest wave
      for (int64_t a = 0; a < k; ++a) {
        const int32_t u = dofs[(size_t)(e0 + a)];
        for (int64_t kk = ap[(size_t)u]; kk < ap[(size_t)u + 1]; ++kk) {
          const int2 en = ent[(size_t)ai[(size_t)kk]];
          for (int32_t e2 : {en.x, en.y}) {
            if (e2 < 0) continue;
            const int32_t p = pe[(size_t)e2];
            if (p == (int32_t)q) continue;
            if (dir == 0 ? lev[(size_t)p] < lq : lev[(size_t)p] > lq) {
              ts.push_back(e2);
              tv.push_back(av[(size_t)kk]);
              if (dir == 0 ? lev[(size_t)p] > glev : lev[(size_t)p] < glev) {
                glev = lev[(size_t)p];
                gates.clear();
              }
              if (lev[(size_t)p] == glev) {
                bool have = false;
                for (auto& g : gates) have |= g.first == p;
                if (!have) gates.emplace_back(p, e2);
              }
            }
          }
        }
        // the DoF's other patch entry: if it ran earlier, its term (A[u, u] d) is in this
        // entry's list and this patch writes x[u]
        const int2 eu = ent[(size_t)u];
        const int32_t other = eu.x == (int32_t)(e0 + a) ? eu.y : eu.x;
        int32_t xp = -2;
        if (other >= 0) {
          xp = -1;
          for (size_t t = (size_t)tstart.back(); t < ts.size(); ++t)
            if (ts[t] == other) {
              xp = (int32_t)(t - (size_t)tstart.back());
              break;
            }
          if (xp > 31) {  // beyond the unrolled term window of the kernel: flow leg not applicable
            okdir[dir] = false;
            return;
          }
        }
        xpart.push_back(xp);
        tstart.push_back((int32_t)ts.size());
      }
      const int64_t nt = (int64_t)ts.size();
      const int64_t k4 = (k + 3) & ~3, kp4 = (k + 1 + 3) & ~3, nt4 = (nt + 3) & ~3;
      const int64_t o_dof = 16 + 4 * 8, o_ts = o_dof + 4 * k4, o_xp = o_ts + 4 * kp4, o_binv = o_xp + 4 * k4,
                    o_slot = o_binv + 8 * k * k,
                    o_val = o_slot + 4 * nt4, bytes = (o_val + 8 * nt + 15) & ~(int64_t)15;
      const size_t base = R.size();
      R.resize(base + (size_t)bytes, 0);
      unsigned char* r = R.data() + base;
      const int32_t ng = (int32_t)std::min<size_t>(gates.size(), 8);
      const int32_t hd[4] = {(int32_t)k, (int32_t)e0, (int32_t)nt, ng};
      memcpy(r, hd, 16);
      for (int32_t g = 0; g < ng; ++g) memcpy(r + 16 + 4 * g, &gates[(size_t)g].second, 4);
      for (int64_t a = 0; a < k; ++a) {
        const int32_t u = dofs[(size_t)(e0 + a)];
        memcpy(r + o_dof + 4 * a, &u, 4);
      }
      memcpy(r + o_ts, tstart.data(), 4 * tstart.size());
      memcpy(r + o_xp, xpart.data(), 4 * xpart.size());
      for (int64_t a = 0; a < k; ++a)          // row-major: binv_rm[a k + c] = B^{-1}[a, c] (stored column-major)
        for (int64_t c = 0; c < k; ++c) {
          const double v = binv[(size_t)(boff[(size_t)q] + c * k + a)];
          memcpy(r + o_binv + 8 * (a * k + c), &v, 8);
        }
      if (nt) {
        memcpy(r + o_slot, ts.data(), 4 * (size_t)nt);
        memcpy(r + o_val, tv.data(), 8 * (size_t)nt);
      }
      rmax[dir] = std::max(rmax[dir], bytes);
      off.push_back((int64_t)R.size());
    }
  };
  std::thread th(build_dir, 1);
  build_dir(0);
  th.join();
  if (!okdir[0] || !okdir[1]) return;
  const int64_t recmax = std::max(rmax[0], rmax[1]);
  if (flow_smem_bytes(recmax) > 200 * 1024) return;  // a patch record too large to double-buffer per warp
  for (int dir = 0; dir < 2; ++dir) {
    f.recs[dir].upload(recs[(size_t)dir].data(), (int64_t)recs[(size_t)dir].size(), s);
    f.rec_off[dir].upload(offs[(size_t)dir].data(), (int64_t)offs[(size_t)dir].size(), s);
    f.d[dir].alloc(ne + 1, s);  // slot ne: a spare that always holds 0.0 (the target of unused term positions)
    flow_reset_slots(f.d[dir].p, ne, s);
    HC_CUDA(cudaMemsetAsync(f.d[dir].p + ne, 0, sizeof(double), s));
  }
  f.dw.alloc(std::max<int64_t>(ne, 1), s);
  f.dw.zero();
  f.recmax = recmax;
  f.bar.alloc(2, s);  // grid-barrier word, patch ticket
  f.bar.zero();
  f.ne = ne;
  HC_CUDA(cudaStreamSynchronize(s));
  f.built = true;
}

}  // namespace hcamg
