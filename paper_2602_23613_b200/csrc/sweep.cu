// Cluster-resident OSS-l1 smoothing legs of the V-cycle.
//
// One thread-block cluster (8-16 CTAs on neighbouring SMs) runs a whole
// smoothing leg in ONE launch: every wavefront of the multiplicative patch
// sweep is one phase, separated by a cluster barrier (barrier.cluster
// arrive.release / wait.acquire: global-memory writes of the previous phase
// are visible cluster-wide), instead of one kernel launch per wavefront.
//
//   down leg (smoothers.py:112-137 "forward", multilevel.py:181-183):
//     r = b, x = 0; waves 0..W-1; pull the last wave; d = r / l1; x += d;
//     r -= A d; [b_c = P^T r]
//   up leg (multilevel.py:183-184, smoothers.py "backward"):
//     [x += P x_c]; r = b - A x; d = r / l1; r -= A d; x += d; waves W-1..0
//
// The bracketed transfers are fused when P is small enough that one cluster
// streams it faster than a separate full-grid launch would start.
#include <cooperative_groups.h>

#include <algorithm>
#include <vector>

#include "sweep.cuh"

namespace cg = cooperative_groups;

namespace hcamg {

namespace {

constexpr int kSweepThreads = 512;
constexpr int64_t kSmemMaxN = (227 * 1024) / 32;

__device__ __forceinline__ double pull_range(int32_t s, int32_t e, const int32_t* __restrict__ gc,
                                             const double* __restrict__ gv, const double* d) {
  double acc = 0.0;
  for (int32_t k0 = s; k0 < e; k0 += 8) {
    int32_t c[8];
    double v[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const bool ok = k0 + t < e;
      c[t] = ok ? __ldg(gc + k0 + t) : 0;
      v[t] = ok ? __ldg(gv + k0 + t) : 0.0;
    }
    double dv[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) dv[t] = k0 + t < e ? d[c[t]] : 0.0;
#pragma unroll
    for (int t = 0; t < 8; ++t) acc = fma(v[t], dv[t], acc);
  }
  return acc;
}

template <bool kInit>
__device__ __forceinline__ void patch_solve(const SweepArgs& a, int64_t p, const int32_t* own, const double* dsrc,
                                            double* ddst, int lane) {
  const int64_t e0 = a.patch_ptr[p];
  const int k = (int)(a.patch_ptr[p + 1] - e0);
  const double* Bi = a.binv + a.binv_off[p];
  double bcol[16];  // this lane's row of B_p^{-1}, loaded before the pulls (memory-level parallelism)
#pragma unroll
  for (int c = 0; c < 16; ++c) bcol[c] = (c < k && lane < k) ? __ldg(Bi + (int64_t)c * k + lane) : 0.0;
  int32_t i = 0;
  double v = 0.0;
  if (lane < k) {
    i = a.dofs[e0 + lane];
    if (kInit) {
      v = a.b[i];
    } else {
      v = a.r[i];
      if (own) {
        const int32_t s = own[2 * (e0 + lane)], e = own[2 * (e0 + lane) + 1];
        if (s >= 0) {
          v -= pull_range(s, e, a.gcol, a.gval, dsrc);
          a.r[i] = v;
        }
      }
    }
  }
  double d = 0.0;
#pragma unroll
  for (int c = 0; c < 16; ++c) d = fma(bcol[c], __shfl_sync(0xffffffffu, v, c), d);
  for (int c = 16; c < k; ++c) {
    const double vc = __shfl_sync(0xffffffffu, v, c);
    if (lane < k) d = fma(Bi[(int64_t)c * k + lane], vc, d);
  }
  if (lane < k) {
    a.x[i] = kInit ? d : a.x[i] + d;
    ddst[i] = d;
  }
}

// rows handled by 8-lane groups: y = M[row,:] . v
template <class F>
__device__ __forceinline__ void rows8(const int64_t* __restrict__ mp, const int32_t* __restrict__ mi,
                                      const double* __restrict__ mv, int64_t nrows, const double* __restrict__ v,
                                      int64_t gtid, int64_t nth, F&& epi) {
  const int lg = (int)(gtid & 7);
  const int64_t g0 = gtid >> 3, ng = nth >> 3;
  const int64_t iters = (nrows + ng - 1) / ng;
  for (int64_t it = 0; it < iters; ++it) {
    const int64_t row = g0 + it * ng;
    double s = 0.0;
    if (row < nrows) {
      const int64_t e1 = mp[row + 1];
      for (int64_t e0 = mp[row] + lg; e0 < e1; e0 += 32) {
        int32_t c[4];
        double w[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const bool ok = e0 + 8 * t < e1;
          c[t] = ok ? __ldg(mi + e0 + 8 * t) : 0;
          w[t] = ok ? __ldg(mv + e0 + 8 * t) : 0.0;
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) s = fma(w[t], e0 + 8 * t < e1 ? v[c[t]] : 0.0, s);
      }
    }
    s += __shfl_xor_sync(0xffffffffu, s, 4, 8);
    s += __shfl_xor_sync(0xffffffffu, s, 2, 8);
    s += __shfl_xor_sync(0xffffffffu, s, 1, 8);
    if (lg == 0 && row < nrows) epi(row, s);
  }
}

__global__ void __launch_bounds__(kSweepThreads) k_down(SweepArgs a) {
  if (*a.stop) return;
  cg::cluster_group cl = cg::this_cluster();
  const int64_t nth = (int64_t)cl.num_blocks() * blockDim.x;
  const int64_t gtid = (int64_t)cl.block_rank() * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int64_t wg = gtid >> 5, nw = nth >> 5;
  const int64_t W = a.nwave, n = a.n;
  double* dbuf[2] = {a.d0, a.d1};
  if (W > 0) {
    for (int64_t u = gtid; u < n; u += nth) {
      a.r[u] = a.b[u];
      if (!a.in_first[u]) a.x[u] = 0.0;
    }
    for (int64_t p = a.wave_ptr[0] + wg; p < a.wave_ptr[1]; p += nw) patch_solve<true>(a, p, nullptr, nullptr, dbuf[0], lane);
    cl.sync();
    for (int64_t w = 1; w < W; ++w) {
      const double* dsrc = dbuf[(w - 1) & 1];
      double* ddst = dbuf[w & 1];
      for (int64_t t = a.gen_ptr[w - 1] + gtid; t < a.gen_ptr[w]; t += nth) {
        const int32_t* g = a.genrow + 3 * t;
        a.r[g[0]] -= pull_range(g[1], g[2], a.gcol, a.gval, dsrc);
      }
      for (int64_t p = a.wave_ptr[w] + wg; p < a.wave_ptr[w + 1]; p += nw) patch_solve<false>(a, p, a.ownr, dsrc, ddst, lane);
      cl.sync();
    }
  } else {
    for (int64_t u = gtid; u < n; u += nth) {
      a.r[u] = a.b[u];
      a.x[u] = 0.0;
    }
    cl.sync();
  }
  // pull the last wave, l1-Jacobi part 1 (smoothers.py:106-108)
  const double* dlast = W > 0 ? dbuf[(W - 1) & 1] : nullptr;
  for (int64_t u = gtid; u < n; u += nth) {
    double v = a.r[u];
    if (W > 0) {
      const int32_t s = a.lastr[2 * u], e = a.lastr[2 * u + 1];
      if (s >= 0) v -= pull_range(s, e, a.gcol, a.gval, dlast);
    }
    const double d = v / a.l1[u];
    a.x[u] += d;
    a.r[u] = v;
    a.dj[u] = d;
  }
  cl.sync();
  // r -= A d (smoothers.py:109)
  rows8(a.ap, a.ai, a.av, n, a.dj, gtid, nth, [&](int64_t row, double s) { a.r[row] -= s; });
  if (a.tp) {
    cl.sync();
    rows8(a.tp, a.ti, a.tv, a.tn, a.r, gtid, nth, [&](int64_t row, double s) { a.tout[row] = s; });
  }
}

__global__ void __launch_bounds__(kSweepThreads) k_up(SweepArgs a) {
  if (*a.stop) return;
  cg::cluster_group cl = cg::this_cluster();
  const int64_t nth = (int64_t)cl.num_blocks() * blockDim.x;
  const int64_t gtid = (int64_t)cl.block_rank() * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int64_t wg = gtid >> 5, nw = nth >> 5;
  const int64_t W = a.nwave, n = a.n;
  double* dbuf[2] = {a.d0, a.d1};
  if (a.tp) {
    rows8(a.tp, a.ti, a.tv, n, a.tin, gtid, nth, [&](int64_t row, double s) { a.x[row] += s; });
    cl.sync();
  }
  // r = b - A x ; d = r / l1
  rows8(a.ap, a.ai, a.av, n, a.x, gtid, nth, [&](int64_t row, double s) {
    const double r = a.b[row] - s;
    a.r[row] = r;
    a.dj[row] = r / a.l1[row];
  });
  cl.sync();
  // r -= A d ; x += d
  rows8(a.ap, a.ai, a.av, n, a.dj, gtid, nth, [&](int64_t row, double s) {
    a.r[row] -= s;
    a.x[row] += a.dj[row];
  });
  cl.sync();
  for (int64_t w = W - 1; w >= 0; --w) {
    double* ddst = dbuf[w & 1];
    if (w == W - 1) {
      for (int64_t p = a.wave_ptr[w] + wg; p < a.wave_ptr[w + 1]; p += nw) patch_solve<false>(a, p, nullptr, nullptr, ddst, lane);
    } else {
      const double* dsrc = dbuf[(w + 1) & 1];
      for (int64_t t = a.gen_ptr[w + 1] + gtid; t < a.gen_ptr[w + 2]; t += nth) {
        const int32_t* g = a.genrow + 3 * t;
        a.r[g[0]] -= pull_range(g[1], g[2], a.gcol, a.gval, dsrc);
      }
      for (int64_t p = a.wave_ptr[w] + wg; p < a.wave_ptr[w + 1]; p += nw) patch_solve<false>(a, p, a.ownr, dsrc, ddst, lane);
    }
    if (w > 0) cl.sync();
  }
}


// ----------------------------------------------------------------------------- single-CTA, shared-memory legs
//
// For levels with n <= kSmemMaxN the four working vectors (r, x and the two
// wave-parity correction buffers) live in shared memory of ONE CTA, so a
// wavefront phase costs a __syncthreads (tens of ns) instead of a kernel
// launch or a cluster barrier; only structure (gather entries, patch
// inverses, A) streams from L2.

constexpr int kSmemThreads = 512;

__device__ __forceinline__ double pull_smem(int32_t s, int32_t e, const int32_t* __restrict__ gc,
                                            const double* __restrict__ gv, const double* d) {
  double acc = 0.0;
  for (int32_t k0 = s; k0 < e; k0 += 8) {
    int32_t c[8];
    double v[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const bool ok = k0 + t < e;
      c[t] = ok ? __ldg(gc + k0 + t) : 0;
      v[t] = ok ? __ldg(gv + k0 + t) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) acc = fma(v[t], d[c[t]], acc);
  }
  return acc;
}

__device__ __forceinline__ void patch_smem(const SweepArgs& a, int64_t p, const int32_t* own, const double* dsrc,
                                           double* ddst, double* r, double* x, int lane) {
  const int64_t e0 = a.patch_ptr[p];
  const int k = (int)(a.patch_ptr[p + 1] - e0);
  const double* Bi = a.binv + a.binv_off[p];
  double bcol[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) bcol[c] = (c < k && lane < k) ? __ldg(Bi + (int64_t)c * k + lane) : 0.0;
  int32_t i = 0;
  double v = 0.0;
  if (lane < k) {
    i = a.dofs[e0 + lane];
    v = r[i];
    if (own) {
      const int32_t s = own[2 * (e0 + lane)], e = own[2 * (e0 + lane) + 1];
      if (s >= 0) {
        v -= pull_smem(s, e, a.gcol, a.gval, dsrc);
        r[i] = v;
      }
    }
  }
  double d = 0.0;
#pragma unroll
  for (int c = 0; c < 16; ++c) d = fma(bcol[c], __shfl_sync(0xffffffffu, v, c), d);
  for (int c = 16; c < k; ++c) {
    const double vc = __shfl_sync(0xffffffffu, v, c);
    if (lane < k) d = fma(Bi[(int64_t)c * k + lane], vc, d);
  }
  if (lane < k) {
    x[i] += d;
    ddst[i] = d;
  }
}

__device__ __forceinline__ double row_dot(const SweepArgs& a, int64_t row, const double* v) {
  return pull_smem((int32_t)a.ap[row], (int32_t)a.ap[row + 1], a.ai, a.av, v);
}

__global__ void __launch_bounds__(kSmemThreads, 1) k_down_smem(SweepArgs a) {
  if (*a.stop) return;
  extern __shared__ double smv[];
  const int64_t n = a.n, W = a.nwave;
  double* r = smv;
  double* x = smv + n;
  double* D[2] = {smv + 2 * n, smv + 3 * n};
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nth >> 5;
  for (int64_t u = tid; u < n; u += nth) {
    r[u] = a.b[u];
    x[u] = 0.0;
  }
  __syncthreads();
  for (int64_t w = 0; w < W; ++w) {
    const double* dsrc = w > 0 ? D[(w - 1) & 1] : nullptr;
    double* ddst = D[w & 1];
    if (w > 0)
      for (int64_t t = a.gen_ptr[w - 1] + tid; t < a.gen_ptr[w]; t += nth) {
        const int32_t* g = a.genrow + 3 * t;
        r[g[0]] -= pull_smem(g[1], g[2], a.gcol, a.gval, dsrc);
      }
    for (int64_t p = a.wave_ptr[w] + wid; p < a.wave_ptr[w + 1]; p += nw)
      patch_smem(a, p, w > 0 ? a.ownr : nullptr, dsrc, ddst, r, x, lane);
    __syncthreads();
  }
  double* dj = D[W & 1];
  const double* dl = W > 0 ? D[(W - 1) & 1] : nullptr;
  for (int64_t u = tid; u < n; u += nth) {
    double v = r[u];
    if (W > 0) {
      const int32_t s = a.lastr[2 * u], e = a.lastr[2 * u + 1];
      if (s >= 0) v -= pull_smem(s, e, a.gcol, a.gval, dl);
    }
    const double d = v / a.l1[u];
    x[u] += d;
    r[u] = v;
    dj[u] = d;
  }
  __syncthreads();
  for (int64_t u = tid; u < n; u += nth) {
    const double rv = r[u] - row_dot(a, u, dj);
    a.r[u] = rv;
    a.x[u] = x[u];
  }
}

__global__ void __launch_bounds__(kSmemThreads, 1) k_up_smem(SweepArgs a) {
  if (*a.stop) return;
  extern __shared__ double smv[];
  const int64_t n = a.n, W = a.nwave;
  double* r = smv;
  double* x = smv + n;
  double* D[2] = {smv + 2 * n, smv + 3 * n};
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nth >> 5;
  for (int64_t u = tid; u < n; u += nth) x[u] = a.x[u];
  __syncthreads();
  double* dj = D[0];
  for (int64_t u = tid; u < n; u += nth) {
    const double rv = a.b[u] - row_dot(a, u, x);
    r[u] = rv;
    dj[u] = rv / a.l1[u];
  }
  __syncthreads();
  for (int64_t u = tid; u < n; u += nth) {
    r[u] -= row_dot(a, u, dj);
    x[u] += dj[u];
  }
  __syncthreads();
  for (int64_t w = W - 1; w >= 0; --w) {
    const double* dsrc = w < W - 1 ? D[(w + 1) & 1] : nullptr;
    double* ddst = D[w & 1];
    if (w < W - 1)
      for (int64_t t = a.gen_ptr[w + 1] + tid; t < a.gen_ptr[w + 2]; t += nth) {
        const int32_t* g = a.genrow + 3 * t;
        r[g[0]] -= pull_smem(g[1], g[2], a.gcol, a.gval, dsrc);
      }
    for (int64_t p = a.wave_ptr[w] + wid; p < a.wave_ptr[w + 1]; p += nw)
      patch_smem(a, p, w < W - 1 ? a.ownr : nullptr, dsrc, ddst, r, x, lane);
    __syncthreads();
  }
  for (int64_t u = tid; u < n; u += nth) a.x[u] = x[u];
}

// ----------------------------------------------------------------------------- segmented transpose products

constexpr int kSeg = 256;

__global__ void __launch_bounds__(256) k_seg_partial(const int* stop, const int64_t* __restrict__ tp,
                                                     const int32_t* __restrict__ ti, const double* __restrict__ tv,
                                                     const int32_t* __restrict__ seg_row,
                                                     const int64_t* __restrict__ segoff, int64_t nseg,
                                                     const double* __restrict__ v, double* __restrict__ partial) {
  if (*stop) return;
  const int lane = threadIdx.x & 31;
  for (int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < nseg;
       g += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int32_t p = seg_row[g];
    const int64_t s = g - segoff[p];
    const int64_t e0 = tp[p] + s * kSeg, e1 = min(tp[p + 1], e0 + kSeg);
    double acc = 0.0;
    for (int64_t e = e0 + lane; e < e1; e += 32) acc = fma(tv[e], v[ti[e]], acc);
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) partial[g] = acc;
  }
}

__global__ void k_seg_reduce(const int* stop, const int64_t* __restrict__ segoff, int64_t nrows,
                             const double* __restrict__ partial, double* __restrict__ y) {
  if (*stop) return;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nrows; p += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int64_t g = segoff[p]; g < segoff[p + 1]; ++g) acc += partial[g];
    y[p] = acc;
  }
}

int g_cluster = 0;

int cluster_size() {
  if (g_cluster) return g_cluster;
  int best = 8;
  for (auto fn : {(const void*)k_down, (const void*)k_up}) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(16);
  cfg.blockDim = dim3(kSweepThreads);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 16;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, (const void*)k_down, &cfg) == cudaSuccess && nclusters > 0) best = 16;
  cudaGetLastError();
  const char* env = getenv("HCAMG_CLUSTER");
  if (env) best = atoi(env);
  g_cluster = best;
  return best;
}

}  // namespace

int sweep_cluster_size() { return cluster_size(); }

int64_t sweep_smem_max_n() { return kSmemMaxN; }

void launch_sweep_smem(bool down, const SweepArgs& args, cudaStream_t s) {
  const size_t smem = sizeof(double) * 4 * (size_t)args.n;
  static bool init = false;
  if (!init) {
    HC_CUDA(cudaFuncSetAttribute(k_down_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kSmemMaxN * 32)));
    HC_CUDA(cudaFuncSetAttribute(k_up_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kSmemMaxN * 32)));
    init = true;
  }
  if (down) k_down_smem<<<1, kSmemThreads, smem, s>>>(args);
  else k_up_smem<<<1, kSmemThreads, smem, s>>>(args);
  HC_CHECK_LAUNCH();
}

void build_segments(const DCsr& T, SegPlan& plan, cudaStream_t s) {
  std::vector<int64_t> ptr = T.ptr.download();
  std::vector<int64_t> off((size_t)T.nrows + 1, 0);
  for (int64_t p = 0; p < T.nrows; ++p) {
    const int64_t len = ptr[(size_t)p + 1] - ptr[(size_t)p];
    off[(size_t)p + 1] = off[(size_t)p] + std::max<int64_t>(1, (len + kSeg - 1) / kSeg);
  }
  std::vector<int32_t> row((size_t)off.back());
  for (int64_t p = 0; p < T.nrows; ++p)
    for (int64_t g = off[(size_t)p]; g < off[(size_t)p + 1]; ++g) row[(size_t)g] = (int32_t)p;
  plan.nseg = off.back();
  plan.segoff.upload(off.data(), (int64_t)off.size(), s);
  plan.seg_row.upload(row.data(), std::max<int64_t>(plan.nseg, 1), s);
  plan.partial.alloc(std::max<int64_t>(plan.nseg, 1), s);
}

void launch_segmented(const int* stop, const DCsr& T, const SegPlan& plan, const double* v, double* y,
                      cudaStream_t s) {
  const unsigned g1 = (unsigned)std::max<int64_t>(1, std::min<int64_t>((plan.nseg * 32 + 255) / 256, kSMs * 16));
  k_seg_partial<<<g1, 256, 0, s>>>(stop, T.ptr.p, T.idx.p, T.val.p, plan.seg_row.p, plan.segoff.p, plan.nseg, v,
                                   plan.partial.p);
  const unsigned g2 = (unsigned)std::max<int64_t>(1, std::min<int64_t>((T.nrows + 255) / 256, kSMs * 4));
  k_seg_reduce<<<g2, 256, 0, s>>>(stop, plan.segoff.p, T.nrows, plan.partial.p, y);
  HC_CHECK_LAUNCH();
}

void launch_sweep(bool down, const SweepArgs& args, cudaStream_t s) {
  const int C = cluster_size();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kSweepThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (down) HC_CUDA(cudaLaunchKernelEx(&cfg, k_down, args));
  else HC_CUDA(cudaLaunchKernelEx(&cfg, k_up, args));
}

}  // namespace hcamg
