// Solve-phase kernels and their recording into CUDA graphs.
//
// V(1,1) cycle (multilevel.py:177-196) per non-coarsest level:
//   forward OSS-l1 (smoothers.py:112-137, x = 0): one k_wave launch per
//     wavefront of the multiplicative patch sweep, then the l1-Jacobi step as
//     k_fw_final (applies the last wave's pending update, d = r / l1, x += d)
//     and an SpMV-update r -= A d;
//   restriction b_c = P^T r (maintained residual; the reference recomputes
//     b - A x, the same vector up to roundoff);
//   recursion, prolongation x += P x_c;
//   backward OSS-l1: r = b - A x fused with d = r / l1, then r -= A d and
//     x += d, then the sweep in reverse wave order;
// coarsest level: x = A^{-1} b with the explicit dense inverse.
// PCG (multilevel.py:238-281) and the AMG iteration (204-235) keep every
// scalar on the device; reductions are deterministic (per-block partials
// summed in block order by the last block to finish).
#include <cuda_runtime.h>

#include <algorithm>

#include "rows_dev.cuh"
#include "solve.cuh"
#include "sweep.cuh"
#include <cstdlib>

namespace hcamg {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* sh) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  return t;  // valid in thread 0
}

// Publish this block's partial(s); returns true in the last block to finish,
// which then sees every partial.  Deterministic: the caller sums in order.
__device__ __forceinline__ bool publish(double v, double v2, double* part, double* part2, unsigned* ticket) {
  __shared__ double sh[32];
  __shared__ bool last;
  double s = block_sum(v, sh);
  double s2 = part2 ? block_sum(v2, sh) : 0.0;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s;
    if (part2) part2[blockIdx.x] = s2;
    __threadfence();
    unsigned t = atomicAdd(ticket, 1u);
    last = t == gridDim.x - 1;
  }
  __syncthreads();
  return last;
}

__device__ __forceinline__ double ordered_sum(const double* part, int n) {
  // fixed order: thread-strided partial sums, then a fixed tree
  __shared__ double sh[32];
  double v = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v += ((volatile const double*)part)[i];
  return block_sum(v, sh);
}

__device__ __forceinline__ void set_cond(unsigned long long cond, unsigned v) {
  if (cond) cudaGraphSetConditional((cudaGraphConditionalHandle)cond, v);
}

// ----------------------------------------------------------------------------- smoother kernels

struct WaveArgs {
  const int* stop;
  int64_t n;
  // generic pulled rows: (u, start, end) triples of the source wave, or -- row
  // partition -- this rank's subset of them through `gen` (indices into the triples)
  const int32_t* genrow;
  const int32_t* gen;
  int64_t ngen;
  const int32_t* gcol;
  const double* gval;
  const double* dsrc;
  // patches of the destination wave: [p0, p0 + np), or plist[0..np)
  int64_t p0, np;
  const int32_t* plist;
  const int64_t* patch_ptr;
  const int32_t* dofs;
  const int64_t* binv_off;
  const double* binv;
  const int32_t* ownr;        // per patch entry: (start, end) of the gather row pulled before the solve, or (-1, -1)
  double* r;
  double* x;
  double* ddst;
  const double* b;            // init step only
  const uint8_t* in_first;    // init step only
  const int32_t* rows;        // init step only: the rows this rank initialises (null: all n)
  int64_t nrows;
  int gen_blocks;
};

// sum_k gval[k] d[gcol[k]] over [s, e), sequential fma order
__device__ __forceinline__ double pull(int32_t s, int32_t e, const int32_t* __restrict__ gc,
                                       const double* __restrict__ gv, const double* __restrict__ d) {
  double acc = 0.0;
  for (int32_t k0 = s; k0 < e; k0 += 4) {
    int32_t c[4];
    double v[4], dv[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const bool ok = k0 + t < e;
      c[t] = ok ? __ldg(gc + k0 + t) : 0;
      v[t] = ok ? __ldg(gv + k0 + t) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) dv[t] = k0 + t < e ? d[c[t]] : 0.0;
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (k0 + t < e) acc = fma(v[t], dv[t], acc);
  }
  return acc;
}

// One wavefront of the multiplicative sweep.  KG lanes per patch (the level's
// largest patch rounded up to 8 / 16 / 32), so a warp solves 32 / KG patches:
// on the wide 2D waves (tens of thousands of 6-DoF patches) the kernel is
// bound by loads in flight, not by lanes.
template <int KG, bool kInit>
__global__ void __launch_bounds__(kThreads) k_wave(WaveArgs a) {
  if (*a.stop) return;
  if ((int)blockIdx.x < a.gen_blocks) {
    const int64_t t = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (kInit) {
      for (int64_t q = t; q < a.nrows; q += (int64_t)a.gen_blocks * kThreads) {
        const int64_t u = a.rows ? a.rows[q] : q;
        a.r[u] = a.b[u];
        if (!a.in_first[u]) a.x[u] = 0.0;
      }
    } else if (t < a.ngen) {
      const int32_t* g = a.genrow + 3 * (int64_t)(a.gen ? a.gen[t] : t);
      const int32_t u = g[0];
      a.r[u] -= pull(g[1], g[2], a.gcol, a.gval, a.dsrc);
    }
    return;
  }
  constexpr int kB = KG < 16 ? KG : 16;  // inverse columns held in registers
  const int sub = threadIdx.x & (KG - 1);
  const int64_t t = ((int64_t)(blockIdx.x - a.gen_blocks) * kThreads + threadIdx.x) / KG;
  const bool have = t < a.np;
  const int64_t p = have ? (a.plist ? (int64_t)a.plist[t] : a.p0 + t) : 0;
  const int64_t e0 = have ? a.patch_ptr[p] : 0;
  const int k = have ? (int)(a.patch_ptr[p + 1] - e0) : 0;
  const bool act = sub < k;
  const double* Bi = a.binv + (have ? a.binv_off[p] : 0);
  double bcol[kB];
#pragma unroll
  for (int c = 0; c < kB; ++c) bcol[c] = (c < k && act) ? __ldg(Bi + (int64_t)c * k + sub) : 0.0;
  int32_t i = 0;
  double v = 0.0;
  if (act) {
    i = a.dofs[e0 + sub];
    if (kInit) {
      v = a.b[i];
    } else {
      v = a.r[i];
      if (a.ownr) {
        const int32_t s = a.ownr[2 * (e0 + sub)], e = a.ownr[2 * (e0 + sub) + 1];
        if (s >= 0) {
          v -= pull(s, e, a.gcol, a.gval, a.dsrc);
          a.r[i] = v;
        }
      }
    }
  }
  // d = B_p^{-1} r[patch]  (column-major inverse: coalesced over the lanes)
  double d = 0.0;
#pragma unroll
  for (int c = 0; c < kB; ++c) d = fma(bcol[c], __shfl_sync(0xffffffffu, v, c, KG), d);
  if (KG > kB) {
    int kmax = k;
    for (int o = 16; o; o >>= 1) kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    for (int c = kB; c < kmax; ++c) {
      const double vc = __shfl_sync(0xffffffffu, v, c, KG);
      if (act && c < k) d = fma(Bi[(int64_t)c * k + sub], vc, d);
    }
  }
  if (act) {
    a.x[i] = kInit ? d : a.x[i] + d;
    a.ddst[i] = d;
  }
}

struct FinalArgs {
  const int* stop;
  int64_t n;                  // rows handled: all of the level, or rows[0..n)
  const int32_t* rows;
  const int32_t* lastr;       // per DoF: (start, end) of the last wave's gather row, or (-1, -1)
  const int32_t* gcol;
  const double* gval;
  const double* dsrc;
  const double* l1;
  double* r;
  double* x;
  double* dj;
};

__global__ void __launch_bounds__(kThreads) k_fw_final(FinalArgs a) {
  if (*a.stop) return;
  for (int64_t q = (int64_t)blockIdx.x * kThreads + threadIdx.x; q < a.n; q += (int64_t)gridDim.x * kThreads) {
    const int64_t u = a.rows ? a.rows[q] : q;
    double v = a.r[u];
    if (a.lastr) {
      const int32_t s = a.lastr[2 * u], e = a.lastr[2 * u + 1];
      if (s >= 0) v -= pull(s, e, a.gcol, a.gval, a.dsrc);
    }
    const double d = v / a.l1[u];
    a.x[u] += d;
    a.r[u] = v;
    a.dj[u] = d;
  }
}

__global__ void k_init_rb(const int* stop, int64_t n, const double* __restrict__ b, double* __restrict__ r,
                          double* __restrict__ x, const int32_t* __restrict__ rows) {
  if (*stop) return;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = rows ? (int64_t)rows[q] : q;
    r[u] = b[u];
    x[u] = 0.0;
  }
}

// ----------------------------------------------------------------------------- SpMV with epilogues

enum Epi : int {
  EPI_SET = 0,       // y = s
  EPI_ADD,           // y += s
  EPI_JAC_FW,        // r -= s
  EPI_RES_JAC,       // r = b - s; dj = r / l1
  EPI_JAC_BW,        // r -= s; x += dj
  EPI_AP,            // y = s; partial p.y -> pAp, alpha
  EPI_PCG_INIT,      // r = b - s; partials r.r, b.b
  EPI_AMG_INIT,      // r = b - s; partials r.r, b.b
  EPI_AMG_RES,       // r = b - s; partial r.r -> rel, history, divergence guard
  EPI_RES_PLAIN,     // r = b - s; partials r.r, b.b (generic PCG init)
};

struct SpmvArgs {
  const int* stop;
  int64_t nrows;
  const int64_t* ptr;
  const int32_t* idx;
  const double* val;
  const double* xin;   // vector multiplied
  double* y;           // EPI_SET/ADD/AP output; r for residual kinds
  const double* b;
  const double* l1;
  double* dj;
  double* x;           // EPI_JAC_BW
  Ctl* ctl;
  double* part;
  double* part2;
  double* hist;
  unsigned long long cond;
  const DSell* sell;    // row partition: sliced-ELLPACK copy of exactly the listed rows (host-side pointer)
  const int32_t* rows;  // row partition: this rank's rows (nrows of them); null: rows [0, nrows)
  double* red;          // row partition: the rank's partial sum(s) go here, k_finish completes the reduction
};

// ---- scalar logic behind the reductions (run by the last block of the
// reducing kernel, or by k_finish after the cross-rank sum)

__device__ __forceinline__ void fin_ap(Ctl* c, double S, unsigned long long cond) {
  c->pAp = S;
  if (!(S > 0.0)) { c->error = kErrPAp; c->stop = 1; set_cond(cond, 0); }
  else c->alpha = c->rz / S;
}

__device__ __forceinline__ void fin_init(Ctl* c, double S, double S2, unsigned long long cond) {
  c->bnorm = sqrt(S2);
  c->it = 0;
  c->error = kErrNone;
  c->growth = 0;
  c->converged = 0;
  c->zero_b = 0;
  c->stop = 0;
  if (c->bnorm == 0.0) {
    c->zero_b = 1; c->converged = 1; c->stop = 1;
  } else {
    c->rel = sqrt(S) / c->bnorm;
    c->prev_rel = c->rel;
    if (c->rel <= c->tol) { c->converged = 1; c->stop = 1; }
    else if (c->maxit <= 0) c->stop = 1;
  }
  set_cond(cond, c->stop ? 0u : 1u);
}

__device__ __forceinline__ void fin_update(Ctl* c, double S, double* hist, unsigned long long cond) {
  const double rel = sqrt(S) / c->bnorm;
  c->rel = rel;
  hist[c->it] = rel;
  c->it += 1;
  if (rel <= c->tol) { c->converged = 1; c->stop = 1; }
  else if (c->it >= c->maxit) c->stop = 1;
  set_cond(cond, c->stop ? 0u : 1u);
}

__device__ __forceinline__ void fin_amg_res(Ctl* c, double S, double* hist, unsigned long long cond) {
  const double prev = c->rel;
  const double rel = sqrt(S) / c->bnorm;
  c->rel = rel;
  hist[c->it] = rel;
  c->it += 1;
  if (rel <= c->tol) { c->converged = 1; c->stop = 1; }
  else {
    c->growth = rel > prev ? c->growth + 1 : 0;
    if (c->growth >= 5) { c->error = 3; c->stop = 1; }
    else if (c->it >= c->maxit) c->stop = 1;
  }
  set_cond(cond, c->stop ? 0u : 1u);
}

template <bool kFirst>
__device__ __forceinline__ void fin_rz(Ctl* c, double S, unsigned long long cond) {
  if (kFirst) { c->rz = S; return; }
  if (!(S > 0.0)) { c->error = kErrRz; c->stop = 1; set_cond(cond, 0); return; }
  c->beta = S / c->rz;
  c->rz = S;
}

// what a row does with its product s = (M xin)[row]
template <int E>
__device__ __forceinline__ void spmv_epi(const SpmvArgs& a, int64_t r_, double s, double& part, double& part2) {
  if (E == EPI_SET) a.y[r_] = s;
  else if (E == EPI_ADD) a.y[r_] += s;
  else if (E == EPI_JAC_FW) a.y[r_] -= s;
  else if (E == EPI_RES_JAC) { const double r = a.b[r_] - s; a.y[r_] = r; a.dj[r_] = r / a.l1[r_]; }
  else if (E == EPI_JAC_BW) { a.y[r_] -= s; a.x[r_] += a.dj[r_]; }
  else if (E == EPI_AP) { a.y[r_] = s; part = fma(a.xin[r_], s, part); }
  else if (E == EPI_PCG_INIT || E == EPI_AMG_INIT || E == EPI_RES_PLAIN) {
    const double bb = a.b[r_], r = bb - s;
    a.y[r_] = r;
    part = fma(r, r, part);
    part2 = fma(bb, bb, part2);
  } else if (E == EPI_AMG_RES) { const double r = a.b[r_] - s; a.y[r_] = r; part = fma(r, r, part); }
}

// the reduction tail of the reducing epilogues (every thread of every block calls it)
template <int E>
__device__ __forceinline__ void spmv_reduce(const SpmvArgs& a, double part, double part2) {
  const bool two = E == EPI_PCG_INIT || E == EPI_AMG_INIT || E == EPI_RES_PLAIN;
  Ctl* c = a.ctl;
  if (!publish(part, part2, a.part, two ? a.part2 : nullptr, &c->ticket[E - EPI_AP])) return;
  const double S = ordered_sum(a.part, gridDim.x);
  const double S2 = two ? ordered_sum(a.part2, gridDim.x) : 0.0;
  if (threadIdx.x != 0) return;
  c->ticket[E - EPI_AP] = 0u;
  if (a.red) {  // row partition: publish the rank's partials, k_finish sums over the ranks
    a.red[0] = S;
    a.red[1] = S2;
    return;
  }
  if (E == EPI_AP) {
    fin_ap(c, S, a.cond);
  } else if (E == EPI_PCG_INIT || E == EPI_AMG_INIT || E == EPI_RES_PLAIN) {
    fin_init(c, S, S2, a.cond);
  } else if (E == EPI_AMG_RES) {
    fin_amg_res(c, S, a.hist, a.cond);
  }
}

// Thread per row over the sliced-ELLPACK copy: every load of a warp is one
// coalesced 128 / 256-byte line, a row's entries are independent loads (no row
// pointers, no shuffles), and the row sum reproduces the CSR kernel's order --
// entry j into partial j mod G, partials folded as the xor butterfly does -- so
// the two kernels are bit-identical and interchangeable (the row partition
// runs the CSR kernel on row lists).
template <int G, int E>
__global__ void __launch_bounds__(kThreads) k_spmv_sell(SpmvArgs a, const int64_t* __restrict__ soff,
                                                        const int32_t* __restrict__ sidx,
                                                        const double* __restrict__ sval) {
  if (E != EPI_PCG_INIT && E != EPI_AMG_INIT && E != EPI_RES_PLAIN && *a.stop) {
    if (E == EPI_AP && blockIdx.x == 0 && threadIdx.x == 0) set_cond(a.cond, 0);
    return;
  }
  const int lane = threadIdx.x & 31;
  const int64_t nsl = (a.nrows + 31) >> 5;
  double part = 0.0, part2 = 0.0;
  for (int64_t sl = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5; sl < nsl;
       sl += ((int64_t)gridDim.x * kThreads) >> 5) {
    const int64_t base = soff[sl];
    const int width = (int)((soff[sl + 1] - base) >> 5);
    const int64_t q = sl * 32 + lane;
    const int64_t row = a.rows ? (q < a.nrows ? (int64_t)a.rows[q] : 0) : q;
    const int32_t* ip = sidx + base + lane;
    const double* vp = sval + base + lane;
    double acc[G];
#pragma unroll
    for (int g = 0; g < G; ++g) acc[g] = 0.0;
    for (int j0 = 0; j0 < width; j0 += G) {
      int32_t c[G];
      double v[G], xv[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const bool ok = j0 + g < width;
        c[g] = ok ? __ldg(ip + (int64_t)(j0 + g) * 32) : -1;
        v[g] = ok ? __ldg(vp + (int64_t)(j0 + g) * 32) : 0.0;
      }
#pragma unroll
      for (int g = 0; g < G; ++g) xv[g] = c[g] >= 0 ? a.xin[c[g]] : 0.0;
#pragma unroll
      for (int g = 0; g < G; ++g)
        if (c[g] >= 0) acc[g] = fma(v[g], xv[g], acc[g]);
    }
#pragma unroll
    for (int o = G / 2; o; o >>= 1)
#pragma unroll
      for (int g = 0; g < o; ++g) acc[g] += acc[g + o];
    if (q < a.nrows) spmv_epi<E>(a, row, acc[0], part, part2);
  }
  if (E < EPI_AP) return;
  spmv_reduce<E>(a, part, part2);
}

template <int G, int E>
__global__ void __launch_bounds__(kThreads) k_spmv(SpmvArgs a) {
  if (E != EPI_PCG_INIT && E != EPI_AMG_INIT && E != EPI_RES_PLAIN && *a.stop) {
    if (E == EPI_AP && blockIdx.x == 0 && threadIdx.x == 0) set_cond(a.cond, 0);
    return;
  }
  const int lg = threadIdx.x & (G - 1);
  const int64_t grp = ((int64_t)blockIdx.x * kThreads + threadIdx.x) / G;
  const int64_t ngrp = (int64_t)gridDim.x * kThreads / G;
  double part = 0.0, part2 = 0.0;
  // kU rows per thread group and pass, their loads issued together: the rows
  // of the sparse-regime operators hold 3-6 entries, so a pass is one
  // dependent chain (row pointers -> entries -> x) and the kernel is bound by
  // chains in flight, not by lanes
  constexpr int kU = 4;
  const int64_t span = ngrp * kU;
  const int64_t rows_iter = ((a.nrows + span - 1) / span) * span;
  for (int64_t q0 = grp; q0 < rows_iter; q0 += span) {
    int64_t row[kU], e0[kU], e1[kU];
    bool live[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t q = q0 + u * ngrp;
      live[u] = q < a.nrows;
      row[u] = live[u] ? (a.rows ? (int64_t)a.rows[q] : q) : 0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      e0[u] = live[u] ? a.ptr[row[u]] + lg : 0;
      e1[u] = live[u] ? a.ptr[row[u] + 1] : 0;
    }
    double v[kU], xv[kU], sum[kU];
    int32_t c[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const bool ok = e0[u] < e1[u];
      v[u] = ok ? a.val[e0[u]] : 0.0;
      c[u] = ok ? a.idx[e0[u]] : -1;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) xv[u] = c[u] >= 0 ? a.xin[c[u]] : 0.0;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      sum[u] = c[u] >= 0 ? fma(v[u], xv[u], 0.0) : 0.0;
      for (int64_t e = e0[u] + G; e < e1[u]; e += G) sum[u] = fma(a.val[e], a.xin[a.idx[e]], sum[u]);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      double s = sum[u];
      for (int o = G / 2; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, G);
      if (lg != 0 || !live[u]) continue;
      spmv_epi<E>(a, row[u], s, part, part2);
    }
  }
  if (E < EPI_AP) return;
  spmv_reduce<E>(a, part, part2);
}

// ----------------------------------------------------------------------------- PCG vector kernels

__global__ void __launch_bounds__(kThreads) k_pcg_update(const int* stop, int64_t n, double* __restrict__ x,
                                                         double* __restrict__ r, const double* __restrict__ p,
                                                         const double* __restrict__ Ap, Ctl* c, double* part,
                                                         double* hist, unsigned long long cond,
                                                         const int32_t* __restrict__ rows, double* red) {
  if (*stop) return;
  const double alpha = c->alpha;
  double acc = 0.0;
  for (int64_t q = (int64_t)blockIdx.x * kThreads + threadIdx.x; q < n; q += (int64_t)gridDim.x * kThreads) {
    const int64_t u = rows ? (int64_t)rows[q] : q;
    x[u] = fma(alpha, p[u], x[u]);
    const double rv = fma(-alpha, Ap[u], r[u]);
    r[u] = rv;
    acc = fma(rv, rv, acc);
  }
  if (!publish(acc, 0.0, part, nullptr, &c->ticket[6])) return;
  const double S = ordered_sum(part, gridDim.x);
  if (threadIdx.x != 0) return;
  c->ticket[6] = 0u;
  if (red) { red[0] = S; red[1] = 0.0; return; }
  fin_update(c, S, hist, cond);
}

template <bool kFirst>
__global__ void __launch_bounds__(kThreads) k_dot_rz(const int* stop, int64_t n, const double* __restrict__ r,
                                                     const double* __restrict__ z, double* __restrict__ p, Ctl* c,
                                                     double* part, unsigned long long cond,
                                                     const int32_t* __restrict__ rows, double* red) {
  if (*stop) return;
  double acc = 0.0;
  for (int64_t q = (int64_t)blockIdx.x * kThreads + threadIdx.x; q < n; q += (int64_t)gridDim.x * kThreads) {
    const int64_t u = rows ? (int64_t)rows[q] : q;
    const double zv = z[u];
    acc = fma(r[u], zv, acc);
    if (kFirst) p[u] = zv;
  }
  if (!publish(acc, 0.0, part, nullptr, &c->ticket[7])) return;
  const double S = ordered_sum(part, gridDim.x);
  if (threadIdx.x != 0) return;
  c->ticket[7] = 0u;
  if (red) { red[0] = S; red[1] = 0.0; return; }
  fin_rz<kFirst>(c, S, cond);
}

__global__ void __launch_bounds__(kThreads) k_p_update(const int* stop, int64_t n, const double* __restrict__ z,
                                                       double* __restrict__ p, const Ctl* c,
                                                       const int32_t* __restrict__ rows) {
  if (*stop) return;
  const double beta = c->beta;
  for (int64_t q = (int64_t)blockIdx.x * kThreads + threadIdx.x; q < n; q += (int64_t)gridDim.x * kThreads) {
    const int64_t u = rows ? (int64_t)rows[q] : q;
    p[u] = fma(beta, p[u], z[u]);
  }
}

// Row partition: complete a reduction.  red holds (S, S2) per rank; every rank
// sums them in rank order, so all ranks take identical decisions.
// site: 0 PCG / AMG init, 1 pAp, 2 residual update, 3 r.z (first), 4 r.z, 5 AMG residual
__global__ void k_finish(const int* stop, int site, Ctl* c, const double* red, int nranks, double* hist,
                         unsigned long long cond) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (site != 0 && *stop) {
    if (site == 1) set_cond(cond, 0);
    return;
  }
  double S = 0.0, S2 = 0.0;
  for (int r = 0; r < nranks; ++r) {
    S += red[2 * r];
    S2 += red[2 * r + 1];
  }
  if (site == 0) fin_init(c, S, S2, cond);
  else if (site == 1) fin_ap(c, S, cond);
  else if (site == 2) fin_update(c, S, hist, cond);
  else if (site == 3) fin_rz<true>(c, S, cond);
  else if (site == 4) fin_rz<false>(c, S, cond);
  else fin_amg_res(c, S, hist, cond);
}

__global__ void k_loop_guard(const int* stop, unsigned long long cond) {
  if (*stop && threadIdx.x == 0) set_cond(cond, 0);
}

__global__ void __launch_bounds__(kThreads) k_axpy1(const int* stop, int64_t n, const double* __restrict__ e,
                                                    double* __restrict__ x, const int32_t* __restrict__ rows) {
  if (*stop) return;
  for (int64_t q = (int64_t)blockIdx.x * kThreads + threadIdx.x; q < n; q += (int64_t)gridDim.x * kThreads) {
    const int64_t u = rows ? (int64_t)rows[q] : q;
    x[u] += e[u];
  }
}

// coarsest: x = Ainv b (row-major, one warp per row)
__global__ void __launch_bounds__(kThreads) k_gemv_dense(const int* stop, int64_t n, const double* __restrict__ M,
                                                         const double* __restrict__ b, double* __restrict__ x) {
  if (*stop) return;
  const int lane = threadIdx.x & 31;
  for (int64_t row = ((int64_t)blockIdx.x * kThreads + threadIdx.x) / 32; row < n;
       row += (int64_t)gridDim.x * kThreads / 32) {
    const double* m = M + row * n;
    double s = 0.0;
    for (int64_t c = lane; c < n; c += 32) s = fma(m[c], b[c], s);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) x[row] = s;
  }
}

// ----------------------------------------------------------------------------- launch helpers

int group_for(const DCsr& M) {
  const double avg = M.nrows ? (double)M.nnz / (double)M.nrows : 0.0;
  if (avg <= 6) return 4;
  if (avg <= 20) return 8;
  if (avg <= 64) return 16;
  return 32;
}

unsigned spmv_grid(int64_t nrows, int G) {
  const int64_t rows_per_block = kThreads / G;
  int64_t g = (nrows + rows_per_block - 1) / rows_per_block;
  g = std::max<int64_t>(1, std::min<int64_t>(g, kSMs * 8));
  return (unsigned)g;
}

template <int E>
void launch_spmv_g(int G, unsigned grid, SpmvArgs& a, cudaStream_t s) {
  switch (G) {
    case 4: k_spmv<4, E><<<grid, kThreads, 0, s>>>(a); break;
    case 8: k_spmv<8, E><<<grid, kThreads, 0, s>>>(a); break;
    case 16: k_spmv<16, E><<<grid, kThreads, 0, s>>>(a); break;
    default: k_spmv<32, E><<<grid, kThreads, 0, s>>>(a); break;
  }
  HC_CHECK_LAUNCH();
}

template <int E>
unsigned spmv(const DCsr& M, SpmvArgs a, cudaStream_t s) {
  if (!a.rows) a.nrows = M.nrows;  // a row list carries its own count
  a.ptr = M.ptr.p;
  a.idx = M.idx.p;
  a.val = M.val.p;
  const int G = group_for(M);
  const DSell* sell = a.rows ? a.sell : M.sell.get();
  if (sell && (G == 4 || G == 8)) {
    const DSell& S = *sell;
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((S.nslice + 7) / 8, kSMs * 8));
    if (G == 4) k_spmv_sell<4, E><<<grid, kThreads, 0, s>>>(a, S.soff.p, S.idx.p, S.val.p);
    else k_spmv_sell<8, E><<<grid, kThreads, 0, s>>>(a, S.soff.p, S.idx.p, S.val.p);
    HC_CHECK_LAUNCH();
    return grid;
  }
  const unsigned grid = spmv_grid(a.nrows, G);
  launch_spmv_g<E>(G, grid, a, s);
  return grid;
}

unsigned vec_grid(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + kThreads - 1) / kThreads, kSMs * 4)); }

}  // namespace

namespace {
__global__ void k_sell_width(const int64_t* __restrict__ ptr, const int32_t* __restrict__ rows, int64_t nrows,
                             int64_t nsl, int64_t* __restrict__ w) {
  for (int64_t sl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sl < nsl; sl += (int64_t)gridDim.x * blockDim.x) {
    int64_t m = 0;
    for (int64_t q = sl * 32; q < min(nrows, sl * 32 + 32); ++q) {
      const int64_t r = rows ? (int64_t)rows[q] : q;
      m = max(m, ptr[r + 1] - ptr[r]);
    }
    w[sl] = 32 * m;
  }
}
__global__ void k_sell_fill(const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                            const double* __restrict__ val, const int32_t* __restrict__ rows, int64_t nrows,
                            int64_t nsl,
                            const int64_t* __restrict__ soff, int32_t* __restrict__ sidx, double* __restrict__ sval) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nsl * 32; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t sl = t >> 5, base = soff[sl];
    const int lane = (int)(t & 31), width = (int)((soff[sl + 1] - base) >> 5);
    const int64_t r = t < nrows ? (rows ? (int64_t)rows[t] : t) : 0;
    const int64_t e0 = t < nrows ? ptr[r] : 0, e1 = t < nrows ? ptr[r + 1] : 0;
    for (int j = 0; j < width; ++j) {
      const bool ok = e0 + j < e1;
      sidx[base + (int64_t)j * 32 + lane] = ok ? idx[e0 + j] : -1;
      sval[base + (int64_t)j * 32 + lane] = ok ? val[e0 + j] : 0.0;
    }
  }
}
}  // namespace

// Sliced-ELLPACK copy of M's rows (all of them, or the listed ones in list
// order), when they are short (the 4- and 8-lane classes of group_for) and
// the padding stays below 50 %.
std::unique_ptr<DSell> build_sell_rows(const DCsr& M, const int32_t* rows, int64_t nrows, cudaStream_t s) {
  const int G = group_for(M);
  if (nrows < 1 || (G != 4 && G != 8)) return nullptr;
  const int64_t nsl = (nrows + 31) / 32;
  DBuf<int64_t> w(nsl, s);
  k_sell_width<<<grid_for(nsl, 256), 256, 0, s>>>(M.ptr.p, rows, nrows, nsl, w.p);
  HC_CHECK_LAUNCH();
  std::unique_ptr<DSell> S(new DSell());
  S->nslice = nsl;
  S->soff.alloc(nsl + 1, s);
  S->padded = exclusive_scan(w.p, S->soff.p, nsl, s);
  const int64_t share = rows ? (int64_t)((double)M.nnz * (double)nrows / (double)std::max<int64_t>(M.nrows, 1)) : M.nnz;
  if (S->padded > 2 * share + 32 * 16) return nullptr;
  S->idx.alloc(std::max<int64_t>(S->padded, 1), s);
  S->val.alloc(std::max<int64_t>(S->padded, 1), s);
  k_sell_fill<<<grid_for(nsl * 32, 256), 256, 0, s>>>(M.ptr.p, M.idx.p, M.val.p, rows, nrows, nsl, S->soff.p,
                                                      S->idx.p, S->val.p);
  HC_CHECK_LAUNCH();
  return S;
}

void build_sell(DCsr& M, cudaStream_t s) {
  M.sell.reset();
  if (M.nrows < 4096) return;
  M.sell = build_sell_rows(M, nullptr, M.nrows, s);
}

void Workspace::ensure(int64_t n_, int64_t maxit, cudaStream_t s) {
  if (!ctl.p) {
    ctl.alloc(1, s);
    ctl.zero();
    part.alloc(kSMs * 8 + 64, s);
    part2.alloc(kSMs * 8 + 64, s);
    zero_flag.alloc(1, s);
    zero_flag.zero();
  }
  if (n_ != n) {
    n = n_;
    for (DBuf<double>* v : {&x, &r, &z, &p, &Ap, &b}) v->alloc(std::max<int64_t>(n, 1), s);
  }
  if (hist.n < maxit + 1) hist.alloc(maxit + 1, s);
}

// ----------------------------------------------------------------------------- V-cycle

long long* g_leg_trace = nullptr;  // debug: set by hcamg_debug_trace

// ---- one wavefront launch (shared by the per-wave leg and the row partition)

// The ranges of a wave step this process computes: everything (single GPU,
// agglomerated levels) or one rank's share of a row-partitioned level.
struct WaveShare {
  const int32_t* plist = nullptr;  // this rank's patches of the destination wave (null: the whole wave)
  int64_t np = -1;
  const int32_t* gen = nullptr;    // this rank's generic rows of the source wave (indices into the wave's triples)
  int64_t ngen = -1;
  const int32_t* rows = nullptr;   // init step: this rank's rows
  int64_t nrows = -1;
};

template <bool kInit>
static void launch_wave_kg(int kg, unsigned grid, const WaveArgs& a, cudaStream_t s) {
  if (kg == 8) k_wave<8, kInit><<<grid, kThreads, 0, s>>>(a);
  else if (kg == 16) k_wave<16, kInit><<<grid, kThreads, 0, s>>>(a);
  else k_wave<32, kInit><<<grid, kThreads, 0, s>>>(a);
  HC_CHECK_LAUNCH();
}

// destination wave `dst`, pulling the corrections of wave `src` (-1: none);
// dir 0 forward / 1 backward; init: the first forward wave (r = b, x = 0)
static void launch_wave(DevLevel& L, const double* b, double* x, const int* stop, bool init, int64_t dst, int64_t src,
                        int dir, const WaveShare& sh, cudaStream_t s) {
  Smoother& sm = L.sm;
  const int64_t n = L.n;
  double* dbuf[2] = {L.d0.p, L.d1.p};
  WaveArgs a{};
  a.stop = stop;
  a.n = n;
  a.gcol = sm.gcol.p;
  a.gval = sm.gval.p;
  a.p0 = sm.wave_ptr[(size_t)dst];
  a.np = sh.np >= 0 ? sh.np : sm.wave_ptr[(size_t)dst + 1] - a.p0;
  a.plist = sh.plist;
  a.patch_ptr = sm.patch_ptr.p;
  a.dofs = sm.patch_dofs.p;
  a.binv_off = sm.binv_off.p;
  a.binv = sm.binv.p;
  a.r = L.r.p;
  a.x = x;
  a.ddst = dbuf[dst & 1];
  if (init) {
    a.b = b;
    a.in_first = sm.in_first.p;
    a.rows = sh.rows;
    a.nrows = sh.nrows >= 0 ? sh.nrows : n;
    a.gen_blocks = (int)std::max<int64_t>(1, std::min<int64_t>((a.nrows + kThreads - 1) / kThreads, kSMs * 4));
  } else if (src >= 0) {
    const std::vector<int64_t>& gp = dir == 0 ? sm.gen_fw_ptr : sm.gen_bw_ptr;
    const int64_t g0 = gp[(size_t)src], g1 = gp[(size_t)src + 1];
    a.genrow = (dir == 0 ? sm.genrow_fw.p : sm.genrow_bw.p) + 3 * g0;
    a.gen = sh.gen;
    a.ngen = sh.ngen >= 0 ? sh.ngen : g1 - g0;
    a.dsrc = dbuf[src & 1];
    a.ownr = dir == 0 ? sm.ownr_fw.p : sm.ownr_bw.p;
    a.gen_blocks = (int)((a.ngen + kThreads - 1) / kThreads);
  }
  const int kg = sm.kmax <= 8 ? 8 : sm.kmax <= 16 ? 16 : 32;
  const int64_t per_block = kThreads / kg;
  const int64_t pb = (a.np + per_block - 1) / per_block;
  const unsigned grid = (unsigned)std::max<int64_t>(1, a.gen_blocks + pb);
  if (init) launch_wave_kg<true>(kg, grid, a, s);
  else launch_wave_kg<false>(kg, grid, a, s);
}

static void launch_fw_final(DevLevel& L, double* x, const int* stop, const int32_t* rows, int64_t nrows,
                            cudaStream_t s) {
  Smoother& sm = L.sm;
  const int64_t W = sm.nwave;
  double* dbuf[2] = {L.d0.p, L.d1.p};
  const int64_t cnt = rows ? nrows : L.n;
  FinalArgs f{stop, cnt, rows, W > 0 ? sm.lastr.p : nullptr, sm.gcol.p, sm.gval.p,
              W > 0 ? dbuf[(W - 1) & 1] : nullptr, L.l1.p, L.r.p, x, L.dj.p};
  k_fw_final<<<vec_grid(std::max<int64_t>(cnt, 1)), kThreads, 0, s>>>(f);
  HC_CHECK_LAUNCH();
}

// per-wave kernel sequence of one smoothing leg (one launch per wavefront)
static int64_t record_leg_waves(DevLevel& L, const double* b, double* x, const int* stop, bool down, cudaStream_t s) {
  Smoother& sm = L.sm;
  const int64_t n = L.n, W = sm.nwave;
  int64_t launches = 0;
  const WaveShare all{};
  if (down) {
    if (W > 0) {
      launch_wave(L, b, x, stop, true, 0, -1, 0, all, s);
      for (int64_t d = 1; d < W; ++d) launch_wave(L, b, x, stop, false, d, d - 1, 0, all, s);
      launches += W;
    } else {
      k_init_rb<<<vec_grid(n), kThreads, 0, s>>>(stop, n, b, L.r.p, x, nullptr);
      HC_CHECK_LAUNCH();
      ++launches;
    }
    launch_fw_final(L, x, stop, nullptr, 0, s);
    SpmvArgs a{};
    a.stop = stop;
    a.xin = L.dj.p;
    a.y = L.r.p;
    spmv<EPI_JAC_FW>(L.A, a, s);
    return launches + 2;
  }
  SpmvArgs rj{};
  rj.stop = stop;
  rj.xin = x;
  rj.y = L.r.p;
  rj.b = b;
  rj.l1 = L.l1.p;
  rj.dj = L.dj.p;
  spmv<EPI_RES_JAC>(L.A, rj, s);
  SpmvArgs jb{};
  jb.stop = stop;
  jb.xin = L.dj.p;
  jb.y = L.r.p;
  jb.dj = L.dj.p;
  jb.x = x;
  spmv<EPI_JAC_BW>(L.A, jb, s);
  launches += 2;
  for (int64_t d = W - 1; d >= 0; --d) launch_wave(L, b, x, stop, false, d, d == W - 1 ? -1 : d + 1, 1, all, s);
  return launches + W;
}

// Coarsest levels of at least this size apply their inverse with the
// HBM-streaming row GEMV (row-partitioned in the distributed solve); smaller
// ones with the latency-oriented k_gemv_dense.  Option "coarse_gemv_min"
// (tests lower it to exercise the streaming paths on small cases).
int64_t coarse_gemv_min() { return opts().coarse_gemv_min; }

// Which leg kernels run on a level under the handle's options: the record-
// streaming wavefront launches on very wide schedules, the dataflow leg on
// deep narrow ones, else AUTO (cluster / grid leg by width) or the forced mode.
int leg_mode(const DevLevel& L) {
  int m = opts().sweep;
  if (m == SWEEP_AUTO && smoother_wave_auto(L.sm)) m = SWEEP_FWAVE;
  if (m == SWEEP_FWAVE && !(L.sm.fl.built && flow_wave_ok(L.sm.kmax, L.sm.fl.recmax))) m = SWEEP_WAVE;
  if (m == SWEEP_AUTO && smoother_flow_auto(L.sm) && L.sm.fl.built) m = SWEEP_FLOW;
  if (m == SWEEP_FLOW && !L.sm.fl.built) m = SWEEP_GRID;  // a DoF in > 2 patches (or not prepared)
  return m;
}

// One piece of a level's V-cycle work (separately launchable for profiling).
int64_t record_piece(int pc, DevLevel& L, DevLevel* C, const double* b, double* x, const int* stop, cudaStream_t s,
                     int part) {
  const int64_t n = L.n;
  // this piece exchanges when the handle is distributed and dist_prepare gave
  // it a site (pieces whose split would move more bytes than the single-GPU
  // form stay replicated: "representation per N", capi.cu)
  const bool dist_on = L.dist && L.dist->on;
  const bool xd = dist_on && ((pc == PC_COARSE && L.xoff_c != DevLevel::kNoSite) ||
                              ((pc == PC_RESTRICT || pc == PC_PROLONG) && L.xoff_g != DevLevel::kNoSite));
  if (part == 2 && !xd) return 0;
  if (pc == PC_COARSE) {
    if (!n) return 0;
    if (n >= coarse_gemv_min() && !xd && L.Asym.on) {  // lower triangle read once (symv.cu)
      symv_apply(stop, L.Asym, b, x, s);
      return 2;
    }
    if (n >= coarse_gemv_min()) {
      dense_gemv_rows(stop, n, n, L.Ainv.p, b, x, s, xd ? L.dist : nullptr, L.xoff_c, part);
      return xd ? (part == 0 ? 2 : 1) : 1;
    } else {
      k_gemv_dense<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 7) / 8, kSMs * 8)), kThreads, 0, s>>>(
          stop, n, L.Ainv.p, b, x);
      HC_CHECK_LAUNCH();
    }
    return 1;
  }
  if (pc == PC_RESTRICT) {
    if (L.hp.on) {  // b_c = P_s^T r - Z^T r_G
      if (part != 2) {
        SpmvArgs rs{};
        rs.stop = stop;
        rs.xin = L.r.p;
        rs.y = C->b.p;
        spmv<EPI_SET>(L.Pt, rs, s);
      }
      if (!xd && L.hp.fac.on) {  // bc -= W'^T A_GG^{-1} r_G through the factor
        factorp_restrict(stop, L.hp.fac, L.r.p, C->b.p, s);
        return 5;
      }
      hybrid_restrict(stop, L.hp, L.r.p, C->b.p, s, xd ? L.dist : nullptr, L.xoff_g, part);
      if (!xd) return 3;
      return part == 0 ? 4 : (part == 1 ? 3 : 1);
    }
    if (L.pt_seg.nseg) {
      launch_segmented(stop, L.Pt, L.pt_seg, L.r.p, C->b.p, s);
      return 2;
    }
    SpmvArgs rs{};
    rs.stop = stop;
    rs.xin = L.r.p;
    rs.y = C->b.p;
    spmv<EPI_SET>(L.Pt, rs, s);
    return 1;
  }
  if (pc == PC_PROLONG) {
    if (part != 2) {
      SpmvArgs pr{};
      pr.stop = stop;
      pr.xin = C->x.p;
      pr.y = x;
      spmv<EPI_ADD>(L.P, pr, s);
    }
    if (L.hp.on && !xd && L.hp.fac.on) {  // x[G] -= A_GG^{-1} W' x_c through the factor
      factorp_prolong(stop, L.hp.fac, C->x.p, x, s);
      return 5;
    }
    if (L.hp.on) {  // x[G] -= Z x_c
      hybrid_prolong(stop, L.hp, C->x.p, x, s, xd ? L.dist : nullptr, L.xoff_y, part);
      if (!xd) return 2;
      return part == 0 ? 3 : (part == 1 ? 2 : 1);
    }
    return 1;
  }
  const bool down = pc == PC_DOWN;
  const bool wide = smoother_wide(L.sm);
  int m = leg_mode(L);
  if (m == SWEEP_FWAVE) {
    Smoother& sm = L.sm;
    FlowProgram& fl = sm.fl;
    const int dir = down ? 0 : 1;
    FlowArgs fa{};
    fa.stop = stop;
    fa.n = n;
    fa.nwave = sm.nwave;
    fa.ne = fl.ne;
    fa.npatch = sm.npatch;
    fa.recmax = fl.recmax;
    fa.recs = fl.recs[dir].p;
    fa.rec_off = fl.rec_off[dir].p;
    fa.d = fl.dw.p;
    fa.x = x;
    SpmvArgs rj{};  // r = b - A x ; dj = r / l1
    rj.stop = stop;
    rj.xin = x;
    rj.y = L.r.p;
    rj.b = b;
    rj.l1 = L.l1.p;
    rj.dj = L.dj.p;
    SpmvArgs jb{};  // r -= A dj ; x += dj
    jb.stop = stop;
    jb.xin = L.dj.p;
    jb.y = L.r.p;
    jb.dj = L.dj.p;
    jb.x = x;
    const int64_t W = sm.nwave;
    if (down) {
      fa.r0 = b;
      for (int64_t w = 0; w < W; ++w)
        launch_flow_wave(true, fa, sm.wave_ptr[(size_t)w], sm.wave_ptr[(size_t)w + 1] - sm.wave_ptr[(size_t)w], s);
      spmv<EPI_RES_JAC>(L.A, rj, s);
      spmv<EPI_JAC_BW>(L.A, jb, s);
    } else {
      spmv<EPI_RES_JAC>(L.A, rj, s);
      spmv<EPI_JAC_BW>(L.A, jb, s);
      fa.r0 = L.r.p;
      int64_t pos = 0;  // the backward records run the waves in descending order
      for (int64_t w = W - 1; w >= 0; --w) {
        const int64_t c = sm.wave_ptr[(size_t)w + 1] - sm.wave_ptr[(size_t)w];
        launch_flow_wave(false, fa, pos, c, s);
        pos += c;
      }
    }
    return W + 2;
  }
  if (m == SWEEP_FLOW) {
    Smoother& sm = L.sm;
    FlowProgram& fl = sm.fl;
    const int dir = down ? 0 : 1;
    FlowArgs fa{};
    fa.stop = stop;
    fa.n = n;
    fa.nwave = sm.nwave;
    fa.ne = fl.ne;
    fa.npatch = sm.npatch;
    fa.recmax = fl.recmax;
    fa.recs = fl.recs[dir].p;
    fa.rec_off = fl.rec_off[dir].p;
    fa.d = fl.d[dir].p;
    fa.x = x;
    fa.bar = fl.bar.p;
    fa.trace = g_leg_trace;
    SpmvArgs rj{};  // r = b - A x ; dj = r / l1
    rj.stop = stop;
    rj.xin = x;
    rj.y = L.r.p;
    rj.b = b;
    rj.l1 = L.l1.p;
    rj.dj = L.dj.p;
    SpmvArgs jb{};  // r -= A dj ; x += dj
    jb.stop = stop;
    jb.xin = L.dj.p;
    jb.y = L.r.p;
    jb.dj = L.dj.p;
    jb.x = x;
    if (down) {
      fa.r0 = b;
      launch_flow_leg(true, fa, s);
      spmv<EPI_RES_JAC>(L.A, rj, s);
      spmv<EPI_JAC_BW>(L.A, jb, s);
    } else {
      spmv<EPI_RES_JAC>(L.A, rj, s);
      spmv<EPI_JAC_BW>(L.A, jb, s);
      fa.r0 = L.r.p;
      launch_flow_leg(false, fa, s);
    }
    return 3;
  }
  if (m == SWEEP_AUTO || m == SWEEP_LEG || m == SWEEP_GRID) {
    Smoother& sm = L.sm;
    SweepProgram& pg = sm.pg;
    LegArgs la{};
    la.stop = stop;
    la.n = n;
    la.nwave = sm.nwave;
    la.m = pg.m;
    la.wave_ptr = sm.d_wave_ptr.p;
    la.gen_fw_ptr = sm.d_gen_fw_ptr.p;
    la.gen_bw_ptr = sm.d_gen_bw_ptr.p;
    la.pk = pg.pk.p;
    la.pdof = pg.pdof.p;
    la.pbinv = pg.pbinv.p;
    la.ocnt = pg.ocnt.p;
    la.ogc = pg.ogc.p;
    la.ogv = pg.ogv.p;
    for (int d = 0; d < 2; ++d) {
      la.ng[d] = pg.ng[d];
      la.gu[d] = pg.gu[d].p;
      la.gcnt[d] = pg.gcnt[d].p;
      la.ggc[d] = pg.ggc[d].p;
      la.ggv[d] = pg.ggv[d].p;
    }
    la.genrow_fw = sm.genrow_fw.p;
    la.genrow_bw = sm.genrow_bw.p;
    la.ownr_fw = sm.ownr_fw.p;
    la.ownr_bw = sm.ownr_bw.p;
    la.lastr = sm.lastr.p;
    la.in_first = sm.in_first.p;
    la.patch_ptr = sm.patch_ptr.p;
    la.dofs = sm.patch_dofs.p;
    la.binv_off = sm.binv_off.p;
    la.binv = sm.binv.p;
    la.gcol = sm.gcol.p;
    la.gval = sm.gval.p;
    la.ap = L.A.ptr.p;
    la.ai = L.A.idx.p;
    la.av = L.A.val.p;
    la.l1 = L.l1.p;
    la.b = b;
    la.x = x;
    la.r = L.r.p;
    la.d0 = L.d0.p;
    la.d1 = L.d1.p;
    la.dj = L.dj.p;
    la.trace = g_leg_trace;
    la.gbar = pg.gbar.p;
    if ((m == SWEEP_AUTO && wide) || m == SWEEP_GRID) launch_leg_grid(down, la, s);
    else launch_leg(down, la, s);
    return 1;
  }
  return record_leg_waves(L, b, x, stop, down, s);
}

static int64_t record_level(std::vector<DevLevel*>& lv, size_t ell, const double* b, double* x, const int* stop,
                            cudaStream_t s) {
  DevLevel& L = *lv[ell];
  if (L.coarsest) return record_piece(PC_COARSE, L, nullptr, b, x, stop, s);
  DevLevel& C = *lv[ell + 1];
  int64_t launches = record_piece(PC_DOWN, L, &C, b, x, stop, s);
  launches += record_piece(PC_RESTRICT, L, &C, b, x, stop, s);
  launches += record_level(lv, ell + 1, C.b.p, C.x.p, stop, s);
  launches += record_piece(PC_PROLONG, L, &C, b, x, stop, s);
  launches += record_piece(PC_UP, L, &C, b, x, stop, s);
  return launches;
}

int64_t record_vcycle(std::vector<DevLevel*>& lv, const double* b0, double* x0, const int* stop, cudaStream_t s) {
  return record_level(lv, 0, b0, x0, stop, s);
}

// ----------------------------------------------------------------------------- PCG / AMG recording

int64_t record_pcg_init(DevLevel& L0, Workspace& w, const double* b, const double* x0, cudaStream_t s,
                        unsigned long long cond) {
  (void)x0;
  SpmvArgs a{};
  a.stop = &w.ctl.p->stop;
  a.xin = w.x.p;
  a.y = w.r.p;
  a.b = b;
  a.ctl = w.ctl.p;
  a.part = w.part.p;
  a.part2 = w.part2.p;
  a.cond = cond;
  spmv<EPI_PCG_INIT>(L0.A, a, s);
  return 1;
}

int64_t record_pcg_first(std::vector<DevLevel*>& lv, Workspace& w, cudaStream_t s) {
  const int* stop = &w.ctl.p->stop;
  int64_t l = record_vcycle(lv, w.r.p, w.z.p, stop, s);
  k_dot_rz<true><<<vec_grid(w.n), kThreads, 0, s>>>(stop, w.n, w.r.p, w.z.p, w.p.p, w.ctl.p, w.part.p, 0, nullptr, nullptr);
  HC_CHECK_LAUNCH();
  return l + 1;
}

int64_t record_pcg_body(std::vector<DevLevel*>& lv, Workspace& w, cudaStream_t s, unsigned long long cond) {
  const int* stop = &w.ctl.p->stop;
  DevLevel& L0 = *lv[0];
  SpmvArgs a{};
  a.stop = stop;
  a.xin = w.p.p;
  a.y = w.Ap.p;
  a.ctl = w.ctl.p;
  a.part = w.part.p;
  a.cond = cond;
  spmv<EPI_AP>(L0.A, a, s);
  k_pcg_update<<<vec_grid(w.n), kThreads, 0, s>>>(stop, w.n, w.x.p, w.r.p, w.p.p, w.Ap.p, w.ctl.p, w.part.p,
                                                  w.hist.p, cond, nullptr, nullptr);
  HC_CHECK_LAUNCH();
  int64_t l = 2 + record_vcycle(lv, w.r.p, w.z.p, stop, s);
  k_dot_rz<false><<<vec_grid(w.n), kThreads, 0, s>>>(stop, w.n, w.r.p, w.z.p, w.p.p, w.ctl.p, w.part.p, cond, nullptr, nullptr);
  k_p_update<<<vec_grid(w.n), kThreads, 0, s>>>(stop, w.n, w.z.p, w.p.p, w.ctl.p, nullptr);
  HC_CHECK_LAUNCH();
  return l + 2;
}

int64_t record_amg_init(DevLevel& L0, Workspace& w, const double* b, const double* x0, cudaStream_t s,
                        unsigned long long cond) {
  (void)x0;
  SpmvArgs a{};
  a.stop = &w.ctl.p->stop;
  a.xin = w.x.p;
  a.y = w.r.p;
  a.b = b;
  a.ctl = w.ctl.p;
  a.part = w.part.p;
  a.part2 = w.part2.p;
  a.cond = cond;
  spmv<EPI_AMG_INIT>(L0.A, a, s);
  return 1;
}

int64_t record_amg_body(std::vector<DevLevel*>& lv, Workspace& w, cudaStream_t s, unsigned long long cond) {
  const int* stop = &w.ctl.p->stop;
  k_loop_guard<<<1, 32, 0, s>>>(stop, cond);
  HC_CHECK_LAUNCH();
  int64_t l = 1 + record_vcycle(lv, w.r.p, w.z.p, stop, s);
  k_axpy1<<<vec_grid(w.n), kThreads, 0, s>>>(stop, w.n, w.z.p, w.x.p, nullptr);
  HC_CHECK_LAUNCH();
  SpmvArgs a{};
  a.stop = stop;
  a.xin = w.x.p;
  a.y = w.r.p;
  a.b = w.b.p;
  a.ctl = w.ctl.p;
  a.part = w.part.p;
  a.hist = w.hist.p;
  a.cond = cond;
  spmv<EPI_AMG_RES>(lv[0]->A, a, s);
  return l + 2;
}

// ----------------------------------------------------------------------------- subdomain row partition (rows.cuh)

static_assert((int)RE_SET == (int)EPI_SET && (int)RE_ADD == (int)EPI_ADD && (int)RE_JAC_FW == (int)EPI_JAC_FW &&
                  (int)RE_RES_JAC == (int)EPI_RES_JAC && (int)RE_JAC_BW == (int)EPI_JAC_BW &&
                  (int)RE_AP == (int)EPI_AP && (int)RE_PCG_INIT == (int)EPI_PCG_INIT &&
                  (int)RE_AMG_INIT == (int)EPI_AMG_INIT && (int)RE_AMG_RES == (int)EPI_AMG_RES,
              "rows.cuh REpi mirrors Epi");

// One step of the partitioned program on this rank: the single-GPU kernel on
// the rank's row list / patch list (or on everything, for agglomerated levels).
int64_t rows_launch_step(const RStep& st, RowsCtx& rc, std::vector<DevLevel*>& lv, Workspace& w, const int* stop,
                         unsigned long long cond, cudaStream_t s) {
  const int depth = rc.depth, N = rc.nranks;
  double* red_base = rc.vec(rows_vec_red(depth));
  auto red = [&](int site) { return red_base + (int64_t)site * 2 * N + 2 * rc.rank; };
  const RowsLevelDev& D0 = rc.lev[0];
  switch (st.kind) {
    case RK_GATHER:
      return 0;
    case RK_FINISH:
      k_finish<<<1, 32, 0, s>>>(stop, st.site, w.ctl.p, red_base + (int64_t)st.site * 2 * N, N, w.hist.p, cond);
      HC_CHECK_LAUNCH();
      return 1;
    case RK_PCG_UPDATE: {
      const int64_t cnt = D0.split ? D0.nrows : w.n;
      k_pcg_update<<<vec_grid(cnt), kThreads, 0, s>>>(stop, cnt, w.x.p, w.r.p, w.p.p, w.Ap.p, w.ctl.p, w.part.p,
                                                      w.hist.p, cond, D0.split ? D0.rows.p : nullptr, red(st.site));
      HC_CHECK_LAUNCH();
      return 1;
    }
    case RK_DOT_RZ: {
      const int64_t cnt = D0.split ? D0.nrows : w.n;
      const int32_t* rows = D0.split ? D0.rows.p : nullptr;
      if (st.site == RS_RZ_FIRST)
        k_dot_rz<true><<<vec_grid(cnt), kThreads, 0, s>>>(stop, cnt, w.r.p, w.z.p, w.p.p, w.ctl.p, w.part.p, cond,
                                                          rows, red(st.site));
      else
        k_dot_rz<false><<<vec_grid(cnt), kThreads, 0, s>>>(stop, cnt, w.r.p, w.z.p, w.p.p, w.ctl.p, w.part.p, cond,
                                                           rows, red(st.site));
      HC_CHECK_LAUNCH();
      return 1;
    }
    case RK_GUARD:
      k_loop_guard<<<1, 32, 0, s>>>(stop, cond);
      HC_CHECK_LAUNCH();
      return 1;
    case RK_AXPY1: {
      const int64_t cnt = D0.split ? D0.nrows : w.n;
      k_axpy1<<<vec_grid(cnt), kThreads, 0, s>>>(stop, cnt, w.z.p, w.x.p, D0.split ? D0.rows.p : nullptr);
      HC_CHECK_LAUNCH();
      return 1;
    }
    case RK_P_UPDATE: {
      const int64_t cnt = D0.split ? D0.nrows : w.n;
      k_p_update<<<vec_grid(cnt), kThreads, 0, s>>>(stop, cnt, w.z.p, w.p.p, w.ctl.p, D0.split ? D0.rows.p : nullptr);
      HC_CHECK_LAUNCH();
      return 1;
    }
    default:
      break;
  }
  DevLevel& L = *lv[(size_t)st.level];
  const RowsLevelDev& D = rc.lev[(size_t)st.level];
  const double* b = st.level == 0 ? w.r.p : L.b.p;
  double* x = st.level == 0 ? w.z.p : L.x.p;
  switch (st.kind) {
    case RK_COARSE:
      return record_piece(PC_COARSE, L, nullptr, b, x, stop, s);
    case RK_LEG:
      return record_piece(st.down ? PC_DOWN : PC_UP, L, nullptr, b, x, stop, s);
    case RK_FWAVE: {
      Smoother& sm = L.sm;
      FlowArgs fa{};
      fa.stop = stop;
      fa.n = L.n;
      fa.nwave = sm.nwave;
      fa.ne = sm.fl.ne;
      fa.npatch = sm.npatch;
      fa.recmax = sm.fl.recmax;
      fa.recs = D.frecs[st.dir].p;          // this rank's records, compacted
      fa.rec_off = D.frec_off[st.dir].p;
      fa.d = sm.fl.dw.p;
      fa.x = x;
      fa.r0 = st.dir == 0 ? b : L.r.p;
      const int64_t i0 = D.foff[st.dir][(size_t)st.dst], i1 = D.foff[st.dir][(size_t)st.dst + 1];
      launch_flow_wave(st.dir == 0, fa, i0, i1 - i0, s);
      return i1 > i0 ? 1 : 0;
    }
    case RK_INIT_RB: {
      const int64_t cnt = D.split ? D.nrows : L.n;
      k_init_rb<<<vec_grid(cnt), kThreads, 0, s>>>(stop, cnt, b, L.r.p, x, D.split ? D.rows.p : nullptr);
      HC_CHECK_LAUNCH();
      return 1;
    }
    case RK_FW_FINAL:
      launch_fw_final(L, x, stop, D.split ? D.rows.p : nullptr, D.nrows, s);
      return 1;
    case RK_WAVE: {
      WaveShare sh{};
      if (D.split) {
        const int64_t p0 = D.poff[(size_t)st.dst], p1 = D.poff[(size_t)st.dst + 1];
        sh.plist = D.plist.p + p0;
        sh.np = p1 - p0;
        if (st.init) {
          sh.rows = D.rows.p;
          sh.nrows = D.nrows;
        } else if (st.src >= 0) {
          const int64_t g0 = D.goff[st.dir][(size_t)st.src], g1 = D.goff[st.dir][(size_t)st.src + 1];
          sh.gen = D.gen[st.dir].p + g0;
          sh.ngen = g1 - g0;
        }
      }
      launch_wave(L, b, x, stop, st.init, st.dst, st.src, st.dir, sh, s);
      return 1;
    }
    case RK_SPMV: {
      SpmvArgs a{};
      a.stop = stop;
      if (st.epi == RE_AP || st.epi == RE_PCG_INIT || st.epi == RE_AMG_INIT || st.epi == RE_AMG_RES) {
        DevLevel& L0 = *lv[0];
        a.ctl = w.ctl.p;
        a.part = w.part.p;
        a.part2 = w.part2.p;
        a.red = red(st.site);
        if (D0.split) {
          a.rows = D0.rows.p;
          a.nrows = D0.nrows;
          a.sell = D0.sA.get();
        }
        if (st.epi == RE_AP) {
          a.xin = w.p.p;
          a.y = w.Ap.p;
          a.cond = cond;
          spmv<EPI_AP>(L0.A, a, s);
        } else {
          a.xin = w.x.p;
          a.y = w.r.p;
          a.b = w.b.p;
          a.hist = w.hist.p;
          a.cond = cond;
          if (st.epi == RE_PCG_INIT) spmv<EPI_PCG_INIT>(L0.A, a, s);
          else if (st.epi == RE_AMG_INIT) spmv<EPI_AMG_INIT>(L0.A, a, s);
          else spmv<EPI_AMG_RES>(L0.A, a, s);
        }
        return 1;
      }
      if (st.mat == 2) {  // b_c = P^T r: rows of the coarser level
        DevLevel& C = *lv[(size_t)st.level + 1];
        const RowsLevelDev& DC = rc.lev[(size_t)st.level + 1];
        if (D.split) {
          a.rows = DC.rows.p;
          a.nrows = DC.nrows;
          a.sell = D.sPt.get();
        }
        a.xin = L.r.p;
        a.y = C.b.p;
        if (!D.split && L.pt_seg.nseg) {
          launch_segmented(stop, L.Pt, L.pt_seg, L.r.p, C.b.p, s);
          return 2;
        }
        spmv<EPI_SET>(L.Pt, a, s);
        return 1;
      }
      if (D.split) {
        a.rows = D.rows.p;
        a.nrows = D.nrows;
        a.sell = st.mat == 1 ? D.sP.get() : D.sA.get();
      }
      if (st.mat == 1) {  // x += P x_c
        DevLevel& C = *lv[(size_t)st.level + 1];
        a.xin = C.x.p;
        a.y = x;
        spmv<EPI_ADD>(L.P, a, s);
        return 1;
      }
      if (st.epi == RE_JAC_FW) {
        a.xin = L.dj.p;
        a.y = L.r.p;
        spmv<EPI_JAC_FW>(L.A, a, s);
      } else if (st.epi == RE_RES_JAC) {
        a.xin = x;
        a.y = L.r.p;
        a.b = b;
        a.l1 = L.l1.p;
        a.dj = L.dj.p;
        spmv<EPI_RES_JAC>(L.A, a, s);
      } else {
        a.xin = L.dj.p;
        a.y = L.r.p;
        a.dj = L.dj.p;
        a.x = x;
        spmv<EPI_JAC_BW>(L.A, a, s);
      }
      return 1;
    }
    default:
      return 0;
  }
}

// ----------------------------------------------------------------------------- generic PCG helpers

void apply_operator(const DCsr& A, const double* x, double* y, cudaStream_t s) {
  DBuf<int> z(1, s);
  z.zero();
  SpmvArgs a{};
  a.stop = z.p;
  a.xin = x;
  a.y = y;
  spmv<EPI_SET>(A, a, s);
}

void generic_init(const DCsr& A, Workspace& w, cudaStream_t s) {
  SpmvArgs a{};
  a.stop = &w.ctl.p->stop;
  a.xin = w.x.p;
  a.y = w.r.p;
  a.b = w.b.p;
  a.ctl = w.ctl.p;
  a.part = w.part.p;
  a.part2 = w.part2.p;
  spmv<EPI_RES_PLAIN>(A, a, s);
}

void generic_pap(const DCsr& A, Workspace& w, cudaStream_t s) {
  SpmvArgs a{};
  a.stop = w.zero_flag.p;
  a.xin = w.p.p;
  a.y = w.Ap.p;
  a.ctl = w.ctl.p;
  a.part = w.part.p;
  spmv<EPI_AP>(A, a, s);
}

void generic_update(Workspace& w, cudaStream_t s) {
  k_pcg_update<<<vec_grid(w.n), kThreads, 0, s>>>(w.zero_flag.p, w.n, w.x.p, w.r.p, w.p.p, w.Ap.p, w.ctl.p,
                                                  w.part.p, w.hist.p, 0, nullptr, nullptr);
  HC_CHECK_LAUNCH();
}

void generic_rz(Workspace& w, bool first, cudaStream_t s) {
  if (first) k_dot_rz<true><<<vec_grid(w.n), kThreads, 0, s>>>(w.zero_flag.p, w.n, w.r.p, w.z.p, w.p.p, w.ctl.p, w.part.p, 0, nullptr, nullptr);
  else k_dot_rz<false><<<vec_grid(w.n), kThreads, 0, s>>>(w.zero_flag.p, w.n, w.r.p, w.z.p, w.p.p, w.ctl.p, w.part.p, 0, nullptr, nullptr);
  HC_CHECK_LAUNCH();
}

namespace {
__global__ void k_vec_add(int64_t n, const double* __restrict__ a, const double* __restrict__ b, double* out) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
    out[u] = a[u] + b[u];
}
}  // namespace

namespace {
// r = b - A x with scipy's csr_matvec rounding (per row: sequential sum in
// ascending column order from +0.0, separate multiply / add roundings), then
// numpy's b - y: the residual the reference's smooth() forms (smoothers.py:122)
__global__ void k_residual_seq(int64_t n, const int64_t* __restrict__ ap, const int32_t* __restrict__ ai,
                               const double* __restrict__ av, const double* __restrict__ x,
                               const double* __restrict__ b, double* __restrict__ r) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int64_t e = ap[u]; e < ap[u + 1]; ++e) acc = __dadd_rn(acc, __dmul_rn(av[e], x[ai[e]]));
    r[u] = __dsub_rn(b[u], acc);
  }
}
__global__ void k_axpby(int64_t n, double a, const double* __restrict__ x, double b, const double* y, double* out) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
    out[u] = a * x[u] + b * y[u];
}
__global__ void k_zero_if_zero_rhs(const Ctl* __restrict__ c, int64_t n, double* __restrict__ x) {
  if (!c->zero_b) return;
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
    x[u] = 0.0;
}
}  // namespace

void residual_scipy_order(const DCsr& A, const double* x, const double* b, double* r, cudaStream_t s) {
  if (A.nrows) k_residual_seq<<<vec_grid(A.nrows), kThreads, 0, s>>>(A.nrows, A.ptr.p, A.idx.p, A.val.p, x, b, r);
  HC_CHECK_LAUNCH();
}

void vec_axpby(int64_t n, double a, const double* x, double b, const double* y, double* out, cudaStream_t s) {
  if (n) k_axpby<<<vec_grid(n), kThreads, 0, s>>>(n, a, x, b, y, out);
  HC_CHECK_LAUNCH();
}

void zero_x_if_zero_rhs(Workspace& w, cudaStream_t s) {
  if (w.n) k_zero_if_zero_rhs<<<vec_grid(w.n), kThreads, 0, s>>>(w.ctl.p, w.n, w.x.p);
  HC_CHECK_LAUNCH();
}

void vec_add(int64_t n, const double* a, const double* b, double* out, cudaStream_t s) {
  if (n) k_vec_add<<<vec_grid(n), kThreads, 0, s>>>(n, a, b, out);
  HC_CHECK_LAUNCH();
}

void generic_p(Workspace& w, cudaStream_t s) {
  k_p_update<<<vec_grid(w.n), kThreads, 0, s>>>(w.zero_flag.p, w.n, w.z.p, w.p.p, w.ctl.p, nullptr);
  HC_CHECK_LAUNCH();
}

}  // namespace hcamg
