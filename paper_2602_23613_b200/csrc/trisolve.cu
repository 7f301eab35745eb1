// Blocked triangular sweeps over the envelope Cholesky factor of A_GG, and
// the factored interpolation block built on them (see trisolve.cuh).
#include <algorithm>
#include <cstdlib>
#include <string>

#include "sparse.cuh"
#include "trisolve.cuh"

namespace hcamg {

namespace {

constexpr int kNB = (int)kTriNB;

struct TriArgs {
  const int* stop;
  int64_t nstep;
  const TriStepD* steps;
  const TriTask* tasks;
  const double* pool;
  double* u;  // right-hand side, folded in place
  double* y;  // solution
  unsigned* bar;
  int64_t pf;  // prefetch distance in steps
  int pfmode;  // 0: no prefetch, 1: at the start of a step (pf ahead), 2: between barrier arrive and wait (1 ahead)
  int dbg;     // measurement only: 1 = skip the grid barrier, 2 = skip the row work
};

// Sum over chunks [j0, j1) of row[64 j + 2 lane .. +1] * x[...] (x in shared
// memory), 8 chunks in flight per lane, butterfly-reduced: every lane returns
// the row's dot product, summed in the same order whichever warp computes it.
template <int kB>
__device__ __forceinline__ double warp_dot(const double* __restrict__ row, const double* x, int j0, int j1, int lane) {
  double acc0 = 0.0, acc1 = 0.0;
  const double2* rp = reinterpret_cast<const double2*>(row + 2 * lane);
  const double2* xp = reinterpret_cast<const double2*>(x + 2 * lane);
  for (int j = j0; j < j1; j += kB) {
    double2 v[kB];
#pragma unroll
    for (int q = 0; q < kB; ++q)
      if (j + q < j1) v[q] = __ldg(rp + 32 * (j + q));
#pragma unroll
    for (int q = 0; q < kB; ++q)
      if (j + q < j1) {
        const double2 xv = xp[32 * (j + q)];
        acc0 = fma(v[q].x, xv.x, acc0);
        acc1 = fma(v[q].y, xv.y, acc1);
      }
  }
  double acc = acc0 + acc1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// This warp's equal slice of a contiguous byte range [b0, b1) of base into L2.
__device__ __forceinline__ void prefetch_slice(const char* base, int64_t b0, int64_t b1, int64_t gw, int64_t W) {
  b0 &= ~int64_t(15);  // bulk prefetch: 16-byte aligned address and size
  const int64_t len = b1 - b0;
  if (len <= 0) return;
  const int64_t sl = ((len + W - 1) / W + 15) & ~int64_t(15);
  const int64_t p0 = b0 + gw * sl;
  if (p0 >= b1) return;
  prefetch_l2(base + p0, (unsigned)(std::min(sl, b1 - p0) & ~int64_t(15)));
}

__device__ __forceinline__ void prefetch_step(const TriArgs& a, const TriStepD& S, int64_t gw, int64_t W, int lane) {
  if (lane != 0) return;
  prefetch_slice(reinterpret_cast<const char*>(a.pool), S.pf0, S.pf1, gw, W);
  prefetch_slice(reinterpret_cast<const char*>(a.tasks), S.t0 * (int64_t)sizeof(TriTask),
                 S.t1 * (int64_t)sizeof(TriTask), gw, W);
}

// One blocked triangular sweep.  Cooperative launch (all CTAs co-resident);
// steps are separated by a sense-reversing grid barrier split into arrive /
// wait.  The word is shared by all sweeps of a handle and returns to its
// low bits after each barrier, so no reset is needed between launches.
template <int kThr, int kB>
__global__ void __launch_bounds__(kThr, 1) k_tri_sweep(TriArgs a) {
  if (*a.stop) return;
  __shared__ __align__(16) double su[kNB];
  __shared__ __align__(16) double sy[kNB];
  const int lane = threadIdx.x & 31;
  const int64_t W = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  unsigned old = 0;
  const int64_t pf = a.pfmode == 1 ? a.pf : (a.pfmode == 2 ? 1 : 0);
  for (int64_t q = 0; q < pf && q < a.nstep; ++q) prefetch_step(a, a.steps[q], gw, W, lane);
  for (int64_t st = 0; st < a.nstep; ++st) {
    const TriStepD S = a.steps[st];
    if (a.pfmode == 1 && st + pf < a.nstep) prefetch_step(a, a.steps[st + pf], gw, W, lane);
    for (int t = threadIdx.x; t < kNB; t += blockDim.x) {
      su[t] = __ldcg(a.u + (int64_t)S.k * kNB + t);
      sy[t] = S.c >= 0 ? __ldcg(a.y + (int64_t)S.c * kNB + t) : 0.0;
    }
    __syncthreads();
    const int64_t tend = a.dbg == 2 ? S.t0 : S.t1;
    for (int64_t t = S.t0 + gw; t < tend; t += W) {
      const TriTask T = a.tasks[t];
      if (T.b == -1) {  // fold (row bases are multiples of 64, never -1)
        const double d = warp_dot<kB>(a.pool + T.a, sy, T.ja0, T.ja1, lane);
        if (lane == 0) a.u[T.out] = __ldcg(a.u + T.out) - d;
      } else {
        const double da = warp_dot<kB>(a.pool + T.a, su, T.ja0, T.ja1, lane);
        const double db = warp_dot<kB>(a.pool + T.b, sy, T.jb0, T.jb1, lane);
        if (lane == 0) a.y[T.out] = da - db;
      }
    }
    if (st + 1 == a.nstep) break;
    if (a.dbg == 1) continue;
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
      asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(a.bar), "r"(inc) : "memory");
    }
    if (a.pfmode == 2) prefetch_step(a, a.steps[st + 1], gw, W, lane);
    if (threadIdx.x == 0) {
      unsigned cur;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(a.bar) : "memory");
      } while (((cur ^ old) & 0x80000000u) == 0);
    }
    __syncthreads();
  }
}

struct CopyJob {
  const double* src;
  int64_t dst;   // offset in the pool (doubles)
  int32_t n;     // doubles
  int32_t pad;
};

// warp per job: pool[dst .. dst + n) = src[0 .. n)
__global__ void k_compact_copy(const CopyJob* __restrict__ jobs, int64_t njobs, double* __restrict__ pool) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = w0; j < njobs; j += nw) {
    const CopyJob J = jobs[j];
    const double2* sp = reinterpret_cast<const double2*>(J.src);
    double2* dp = reinterpret_cast<double2*>(pool + J.dst);
    for (int q = lane; q < J.n / 2; q += 32) dp[q] = sp[q];
  }
}

// v[i] = r[dof[i]] (i < nG), 0 on the padding
__global__ void k_fp_gather(const int* stop, int64_t nG, int64_t npad, const int32_t* __restrict__ dof,
                            const double* __restrict__ r, double* __restrict__ v) {
  if (*stop) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npad; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = i < nG ? r[dof[i]] : 0.0;
}

// x[dof[i]] -= t[i]
__global__ void k_fp_scatter_sub(const int* stop, int64_t nG, const int32_t* __restrict__ dof,
                                 const double* __restrict__ t, double* __restrict__ x) {
  if (*stop) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nG; i += (int64_t)gridDim.x * blockDim.x)
    x[dof[i]] -= t[i];
}

// kSub = false: y[i] = M[i,:] x (rows >= nrows up to npad get 0);
// kSub = true:  y[i] -= M[i,:] x.   Warp per row, fixed order.
template <bool kSub>
__global__ void k_fp_spmv(const int* stop, int64_t nrows, int64_t npad, const int64_t* __restrict__ mp,
                          const int32_t* __restrict__ mi, const double* __restrict__ mv, const double* __restrict__ x,
                          double* __restrict__ y) {
  if (*stop) return;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w0; i < npad; i += nw) {
    double acc = 0.0;
    if (i < nrows)
      for (int64_t e = mp[i] + lane; e < mp[i + 1]; e += 32) acc = fma(mv[e], x[mi[e]], acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      if (kSub) y[i] -= acc;
      else y[i] = acc;
    }
  }
}

__global__ void k_fp_rowsel(int64_t nG, const int32_t* __restrict__ perm, const int32_t* __restrict__ mpos,
                            const int32_t* __restrict__ rows, int32_t* __restrict__ sel, int32_t* __restrict__ dof) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nG; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t q = perm[i];
    sel[i] = mpos[q];
    dof[i] = rows[q];
  }
}

template <int kThr, int kB>
void launch_sweep_t(const TriArgs& a, cudaStream_t s) {
  static int blocks = 0;
  if (!blocks) {
    int per_sm = 0, dev = 0, sms = kSMs;
    HC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tri_sweep<kThr, kB>, kThr, 0));
    HC_CUDA(cudaGetDevice(&dev));
    HC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    blocks = sms * std::max(1, per_sm);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(kThr);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  HC_CUDA(cudaLaunchKernelEx(&cfg, k_tri_sweep<kThr, kB>, a));
}

void launch_sweep_kernel(const int* stop, const TriSweep& sw, double* u, double* y, unsigned* bar, cudaStream_t s) {
  auto env = [](const char* k, int d) {
    const char* v = getenv(k);
    return v ? atoi(v) : d;
  };
  // measurement knobs: HCAMG_TRI_PFMODE / HCAMG_TRI_PF (L2 prefetch placement), HCAMG_TRI_DBG
  TriArgs a{stop, sw.nstep, sw.steps.p, sw.tasks.p, sw.pool.p, u, y, bar, std::max(1, env("HCAMG_TRI_PF", 1)),
            env("HCAMG_TRI_PFMODE", 2), env("HCAMG_TRI_DBG", 0)};
  launch_sweep_t<512, 8>(a, s);
}

}  // namespace

void tri_compact(const std::vector<TriSrcStep>& src, const std::function<const uint8_t*(const double*)>& ranges,
                 TriSweep& out, cudaStream_t s) {
  std::vector<TriStepD> steps;
  std::vector<TriTask> tasks;
  std::vector<CopyJob> jobs;
  int64_t off = 0;  // pool offset (doubles)
  auto place = [&](const double* tile, int r, uint8_t& j0, uint8_t& j1) -> int64_t {
    const uint8_t* rg = ranges(tile) + 2 * r;
    j0 = rg[0];
    j1 = rg[1];
    if (j0 >= j1) {
      j0 = j1 = 0;
      return 0;
    }
    const int32_t n = 64 * (j1 - j0);
    jobs.push_back(CopyJob{tile + (int64_t)r * kNB + 64 * j0, off, n, 0});
    const int64_t base = off - 64 * (int64_t)j0;
    off += n;
    return base;
  };
  for (const TriSrcStep& S : src) {
    TriStepD d{};
    d.k = S.k;
    d.c = S.c;
    d.t0 = (int64_t)tasks.size();
    d.pf0 = 8 * off;
    for (int r = 0; r < kNB; ++r) {
      TriTask t{};
      t.out = (int32_t)((int64_t)S.k * kNB + r);
      t.a = place(S.a, r, t.ja0, t.ja1);
      t.b = S.b ? place(S.b, r, t.jb0, t.jb1) : 0;
      tasks.push_back(t);
    }
    for (const auto& fo : S.folds)
      for (int r = 0; r < kNB; ++r) {
        TriTask t{};
        t.a = place(fo.first, r, t.ja0, t.ja1);
        if (t.ja0 >= t.ja1) continue;  // an all-zero fold row changes nothing
        t.b = -1;
        t.out = (int32_t)(fo.second * kNB + r);
        tasks.push_back(t);
      }
    d.t1 = (int64_t)tasks.size();
    d.pf1 = 8 * off;
    steps.push_back(d);
  }
  out.nstep = (int64_t)steps.size();
  out.bytes = 8 * off;
  out.pool.alloc(std::max<int64_t>(off, 2), s);
  out.steps.upload(steps.data(), out.nstep, s);
  out.tasks.upload(tasks.data(), (int64_t)tasks.size(), s);
  DBuf<CopyJob> dj;
  dj.upload(jobs.data(), (int64_t)jobs.size(), s);
  if (!jobs.empty()) k_compact_copy<<<grid_for((int64_t)jobs.size() * 32, 256), 256, 0, s>>>(dj.p, (int64_t)jobs.size(), out.pool.p);
  HC_CHECK_LAUNCH();
  HC_CUDA(cudaStreamSynchronize(s));
}

bool factorp_enabled() {
  const char* e = getenv("HCAMG_PAPPLY");
  return !(e && std::string(e) == "z");
}

void factorp_attach(FactorP& f, const DCsr& W, const int32_t* mpos, const int32_t* rows, cudaStream_t s) {
  const int64_t nG = f.nG;
  f.nc = W.ncols;
  DBuf<int32_t> sel(nG, s);
  f.dof.alloc(nG, s);
  k_fp_rowsel<<<grid_for(nG, 256), 256, 0, s>>>(nG, f.perm.p, mpos, rows, sel.p, f.dof.p);
  HC_CHECK_LAUNCH();
  csr_extract(W, sel.p, nG, nullptr, W.ncols, f.Wp, s);
  csr_transpose(f.Wp, f.Wpt, s);
  const int64_t npad = f.T * kTriNB;
  f.v0.alloc(npad, s);
  f.v1.alloc(npad, s);
  f.v2.alloc(npad, s);
  f.v0.zero();
  f.v1.zero();
  f.v2.zero();
  f.bar.alloc(1, s);
  f.bar.zero();
  f.on = true;
}

void factorp_solve(const int* stop, FactorP& f, double* v, double* y, cudaStream_t s) {
  launch_sweep_kernel(stop, f.fw, v, f.v1.p, f.bar.p, s);
  launch_sweep_kernel(stop, f.bw, f.v1.p, y, f.bar.p, s);
}

void factorp_restrict(const int* stop, FactorP& f, const double* r, double* bc, cudaStream_t s) {
  const int64_t npad = f.T * kTriNB;
  k_fp_gather<<<grid_for(npad, 256), 256, 0, s>>>(stop, f.nG, npad, f.dof.p, r, f.v0.p);
  HC_CHECK_LAUNCH();
  factorp_solve(stop, f, f.v0.p, f.v2.p, s);
  k_fp_spmv<true><<<grid_for(f.nc * 32, 256), 256, 0, s>>>(stop, f.nc, f.nc, f.Wpt.ptr.p, f.Wpt.idx.p, f.Wpt.val.p,
                                                           f.v2.p, bc);
  HC_CHECK_LAUNCH();
}

void factorp_prolong(const int* stop, FactorP& f, const double* e, double* x, cudaStream_t s) {
  const int64_t npad = f.T * kTriNB;
  k_fp_spmv<false><<<grid_for(npad * 32, 256), 256, 0, s>>>(stop, f.nG, npad, f.Wp.ptr.p, f.Wp.idx.p, f.Wp.val.p, e,
                                                            f.v0.p);
  HC_CHECK_LAUNCH();
  factorp_solve(stop, f, f.v0.p, f.v2.p, s);
  k_fp_scatter_sub<<<grid_for(f.nG, 256), 256, 0, s>>>(stop, f.nG, f.dof.p, f.v2.p, x);
  HC_CHECK_LAUNCH();
}

}  // namespace hcamg
