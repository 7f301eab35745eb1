// Blocked triangular sweeps over the envelope Cholesky factor of A_GG, and
// the factored interpolation block built on them (see trisolve.cuh).
#include <algorithm>
#include <cstdlib>
#include <string>

#include "sparse.cuh"
#include "trisolve.cuh"

namespace hcamg {

namespace {

constexpr int kTriThreads = 512;
constexpr int kNB = (int)kTriNB;
constexpr int kChunks = kNB / 64;  // a warp covers 64 columns (32 lanes x double2) per load

struct TriArgs {
  const int* stop;
  int64_t nstep;
  const TriStep* steps;
  const TriTile* tiles;
  double* u;  // right-hand side, folded in place
  double* y;  // solution
  unsigned* bar;
};

// Sum over chunks [j0, j1) of row[64 j + 2 lane .. +1] * x[...] (x in shared
// memory), butterfly-reduced: every lane returns the row's dot product, summed
// in the same order whichever warp computes it.
__device__ __forceinline__ double warp_dot(const double* __restrict__ row, const double* x, int j0, int j1, int lane) {
  double acc0 = 0.0, acc1 = 0.0;
  double2 v[kChunks];
#pragma unroll
  for (int j = 0; j < kChunks; ++j)
    if (j >= j0 && j < j1) v[j] = __ldg(reinterpret_cast<const double2*>(row + 64 * j + 2 * lane));
#pragma unroll
  for (int j = 0; j < kChunks; ++j)
    if (j >= j0 && j < j1) {
      const double2 xv = *reinterpret_cast<const double2*>(x + 64 * j + 2 * lane);
      acc0 = fma(v[j].x, xv.x, acc0);
      acc1 = fma(v[j].y, xv.y, acc1);
    }
  double acc = acc0 + acc1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// column range [c0, c1) (in 64-column chunks) of a critical row
__device__ __forceinline__ void crit_chunks(int tri, int r, int& j0, int& j1) {
  if (tri == 0) {
    j0 = 0;
    j1 = r / 64 + 1;
  } else {
    j0 = r / 64;
    j1 = kChunks;
  }
}

__device__ __forceinline__ int64_t step_tasks(const TriStep& S) { return (int64_t)kNB * (1 + (S.t1 - S.t0)); }

// L2 prefetch of the matrix rows this warp reads in step S (lane 0 issues).
__device__ __forceinline__ void prefetch_step(const TriArgs& a, const TriStep& S, int64_t gw, int64_t W, int lane) {
  if (lane != 0) return;
  const int64_t nt = step_tasks(S);
  for (int64_t t = gw; t < nt; t += W) {
    if (t < kNB) {
      const int r = (int)t;
      int j0, j1;
      crit_chunks(S.tri, r, j0, j1);
      prefetch_l2(S.a + (int64_t)r * kNB + 64 * j0, (unsigned)(512 * (j1 - j0)));
      if (S.b) prefetch_l2(S.b + (int64_t)r * kNB, kNB * 8);
    } else {
      const TriTile tt = a.tiles[S.t0 + (t - kNB) / kNB];
      prefetch_l2(tt.a + ((t - kNB) % kNB) * kNB, kNB * 8);
    }
  }
}

// One blocked triangular sweep.  Cooperative launch (all CTAs co-resident);
// steps are separated by a sense-reversing grid barrier split into arrive /
// wait so the next step's L2 prefetch overlaps the barrier.
__global__ void __launch_bounds__(kTriThreads, 1) k_tri_sweep(TriArgs a) {
  if (*a.stop) return;
  __shared__ __align__(16) double su[kNB];
  __shared__ __align__(16) double sy[kNB];
  const int lane = threadIdx.x & 31;
  const int64_t W = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  unsigned old = 0;
  if (a.nstep > 0) prefetch_step(a, a.steps[0], gw, W, lane);
  for (int64_t st = 0; st < a.nstep; ++st) {
    const TriStep S = a.steps[st];
    for (int t = threadIdx.x; t < kNB; t += blockDim.x) {
      su[t] = __ldcg(a.u + (int64_t)S.k * kNB + t);
      sy[t] = S.c >= 0 ? __ldcg(a.y + (int64_t)S.c * kNB + t) : 0.0;
    }
    __syncthreads();
    const int64_t nt = step_tasks(S);
    for (int64_t t = gw; t < nt; t += W) {
      if (t < kNB) {
        const int r = (int)t;
        int j0, j1;
        crit_chunks(S.tri, r, j0, j1);
        const double da = warp_dot(S.a + (int64_t)r * kNB, su, j0, j1, lane);
        const double db = S.b ? warp_dot(S.b + (int64_t)r * kNB, sy, 0, kChunks, lane) : 0.0;
        if (lane == 0) a.y[(int64_t)S.k * kNB + r] = da - db;
      } else {
        const TriTile tt = a.tiles[S.t0 + (t - kNB) / kNB];
        const int r = (int)((t - kNB) % kNB);
        const double d = warp_dot(tt.a + (int64_t)r * kNB, sy, 0, kChunks, lane);
        if (lane == 0) {
          double* o = a.u + tt.blk * kNB + r;
          *o = __ldcg(o) - d;
        }
      }
    }
    if (st + 1 == a.nstep) break;
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
      asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(a.bar), "r"(inc) : "memory");
    }
    prefetch_step(a, a.steps[st + 1], gw, W, lane);
    if (threadIdx.x == 0) {
      unsigned cur;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(a.bar) : "memory");
      } while (((cur ^ old) & 0x80000000u) == 0);
    }
    __syncthreads();
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

void launch_sweep_kernel(const int* stop, const TriSweep& sw, double* u, double* y, unsigned* bar, cudaStream_t s) {
  static int blocks = 0;
  if (!blocks) {
    int per_sm = 0, dev = 0, sms = kSMs;
    HC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tri_sweep, kTriThreads, 0));
    HC_CUDA(cudaGetDevice(&dev));
    HC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    blocks = sms * std::max(1, per_sm);
  }
  TriArgs a{stop, sw.nstep, sw.steps.p, sw.tiles.p, u, y, bar};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(kTriThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  HC_CUDA(cudaLaunchKernelEx(&cfg, k_tri_sweep, a));
}

}  // namespace

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
