// Software-pipelined cluster sweep (default for levels above the single-CTA
// shared-memory size).
//
// A wavefront phase has a fixed, static structure (which patch each warp
// solves, which rows each thread pulls, the patch inverses, the gather
// coefficients) and a small dynamic part (r, x and the previous wave's
// corrections).  Every warp loads the static part of its NEXT phase before it
// waits at the cluster barrier, so after the barrier only the dynamic loads
// remain on the critical path (one dependent L2 round trip instead of five).
// Static data is padded to fixed strides (16 lanes per patch, 8 inline gather
// slots per row) so that every address is computable from the patch / row id.
#include <cooperative_groups.h>

#include <algorithm>
#include <vector>

#include "sweep.cuh"
#include "level.cuh"

namespace cg = cooperative_groups;

namespace hcamg {

namespace {

constexpr int kLegThreads = 512;
constexpr int kSlots = 12;

// ---- program construction

__global__ void k_prog_patch(int64_t m, const int64_t* __restrict__ pp, const int32_t* __restrict__ dofs,
                             const int64_t* __restrict__ boff, const double* __restrict__ binv,
                             const int32_t* __restrict__ own_fw, const int32_t* __restrict__ own_bw,
                             const int32_t* __restrict__ gcol, const double* __restrict__ gval, int8_t* __restrict__ pk,
                             int32_t* __restrict__ pdof, double* __restrict__ pbinv, int32_t* __restrict__ ocnt,
                             int32_t* __restrict__ ogc, double* __restrict__ ogv) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m * 16; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = t >> 4;
    const int l = (int)(t & 15);
    const int64_t e0 = pp[p];
    const int k = (int)(pp[p + 1] - e0);
    if (l == 0) pk[p] = k <= 16 ? (int8_t)k : 0;
    const bool live = k <= 16 && l < k;
    pdof[t] = live ? dofs[e0 + l] : -1;
    for (int c = 0; c < 16; ++c) pbinv[p * 256 + c * 16 + l] = (live && c < k) ? binv[boff[p] + (int64_t)c * k + l] : 0.0;
    for (int dir = 0; dir < 2; ++dir) {
      const int32_t* own = dir == 0 ? own_fw : own_bw;
      int32_t s = -1, e = -1;
      if (live) { s = own[2 * (e0 + l)]; e = own[2 * (e0 + l) + 1]; }
      const int32_t cnt = s >= 0 ? e - s : -1;
      ocnt[(int64_t)dir * m * 16 + t] = cnt;
      for (int j = 0; j < kSlots; ++j) {
        const int64_t o = (((int64_t)dir * m + p) * kSlots + j) * 16 + l;
        const bool ok = cnt > j;
        ogc[o] = ok ? gcol[s + j] : 0;
        ogv[o] = ok ? gval[s + j] : 0.0;
      }
    }
  }
}

__global__ void k_prog_gen(int64_t ng, const int32_t* __restrict__ genrow, const int32_t* __restrict__ gcol,
                           const double* __restrict__ gval, int32_t* __restrict__ gu, int32_t* __restrict__ gcnt,
                           int32_t* __restrict__ ggc, double* __restrict__ ggv) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ng; t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = genrow[3 * t], s = genrow[3 * t + 1], e = genrow[3 * t + 2];
    gu[t] = u;
    gcnt[t] = e - s;
    for (int j = 0; j < kSlots; ++j) {
      const bool ok = e - s > j;
      ggc[(int64_t)j * ng + t] = ok ? gcol[s + j] : 0;
      ggv[(int64_t)j * ng + t] = ok ? gval[s + j] : 0.0;
    }
  }
}

// ---- the leg kernel

struct PatchPre {
  int64_t p;
  int k;
  int32_t i;
  int32_t cnt;
  int32_t gc[kSlots];
};

struct RowPre {
  int64_t t;
  int32_t u;
  int32_t cnt;
  int32_t gc[kSlots];
};

// Only the index structure is prefetched (it gates the dependent loads); the
// coefficients (inverse column, gather weights) are loaded after the barrier
// in parallel with the dynamic loads, keeping the register budget spill-free.
__device__ __forceinline__ void load_patch(const LegArgs& a, int dir, int64_t p, int lane, bool own, PatchPre& q) {
  q.p = p;
  q.k = a.pk[p];
  q.i = a.pdof[p * 16 + (lane & 15)];
  q.cnt = own ? a.ocnt[(int64_t)dir * a.m * 16 + p * 16 + (lane & 15)] : -1;
#pragma unroll
  for (int j = 0; j < kSlots; ++j) {
    const int64_t o = (((int64_t)dir * a.m + p) * kSlots + j) * 16 + (lane & 15);
    q.gc[j] = own ? __ldg(a.ogc + o) : 0;
  }
}

__device__ __forceinline__ void load_row(const LegArgs& a, int dir, int64_t t, RowPre& q) {
  const int64_t ng = a.ng[dir];
  q.t = t;
  q.u = a.gu[dir][t];
  q.cnt = a.gcnt[dir][t];
#pragma unroll
  for (int j = 0; j < kSlots; ++j) q.gc[j] = __ldg(a.ggc[dir] + (int64_t)j * ng + t);
}

// sum_j gv[j] d[gc[j]] with the weights streamed from `gv` (stride `gs`)
__device__ __forceinline__ double slots_dot(const int32_t* gc, const double* __restrict__ gv, int64_t gs, int cnt,
                                            const double* d) {
  double dv[kSlots], w[kSlots];
#pragma unroll
  for (int j = 0; j < kSlots; ++j) {
    w[j] = j < cnt ? __ldg(gv + j * gs) : 0.0;
    dv[j] = j < cnt ? d[gc[j]] : 0.0;
  }
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < kSlots; ++j) acc = fma(w[j], dv[j], acc);
  return acc;
}

__device__ __forceinline__ double overflow_dot(const int32_t* rng, const int32_t* __restrict__ gcol,
                                               const double* __restrict__ gval, const double* d) {
  double acc = 0.0;
  for (int32_t k = rng[0] + kSlots; k < rng[1]; ++k) acc = fma(gval[k], d[gcol[k]], acc);
  return acc;
}

__device__ __forceinline__ void pf_l2(const void* p) {
  asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
}

// L2 prefetch of everything static that phase `dst` (a patch of this warp, the
// pulled row of this thread) will load: on the wide levels the leg's static
// data (~230 MB on config 2) does not survive the dense sweeps in L2, so
// without it every phase's coefficient loads are HBM misses after the barrier.
__device__ __forceinline__ void l2_prefetch_phase(const LegArgs& a, int dir, int64_t p, bool own, int64_t t,
                                                  int lane) {
  if (p >= 0) {
    pf_l2(a.pbinv + p * 256 + (lane & 15) * 16);  // 2 KB inverse: 16 lines
    if (own) {
      if (lane < kSlots) pf_l2(a.ogv + (((int64_t)dir * a.m + p) * kSlots + lane) * 16);
      else if (lane < kSlots + (kSlots + 1) / 2)
        pf_l2(a.ogc + (((int64_t)dir * a.m + p) * kSlots + 2 * (lane - kSlots)) * 16);
      else if (lane == 31) pf_l2(a.ocnt + (int64_t)dir * a.m * 16 + p * 16);
    }
    if (lane == 30) pf_l2(a.pdof + p * 16);
  }
  if (t >= 0) {
    const int64_t ng = a.ng[dir];
    pf_l2(a.gu[dir] + t);
    pf_l2(a.gcnt[dir] + t);
#pragma unroll
    for (int j = 0; j < kSlots; ++j) {
      pf_l2(a.ggc[dir] + (int64_t)j * ng + t);
      pf_l2(a.ggv[dir] + (int64_t)j * ng + t);
    }
  }
}

// one patch solve from prefetched structure
__device__ __forceinline__ void solve_patch(const LegArgs& a, int dir, const PatchPre& q, int lane, bool init_x,
                                            const double* vin, const double* dsrc, double* ddst) {
  const bool act = lane < q.k;
  const int l = lane & 15;
  double bcol[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) bcol[c] = __ldg(a.pbinv + q.p * 256 + c * 16 + l);
  double v = 0.0, xo = 0.0;
  if (act) {
    if (!init_x) xo = a.x[q.i];
    v = vin[q.i];
    if (q.cnt >= 0) {
      const double* gv = a.ogv + (((int64_t)dir * a.m + q.p) * kSlots) * 16 + l;
      v -= slots_dot(q.gc, gv, 16, q.cnt, dsrc);
      if (q.cnt > kSlots) {
        const int64_t e = a.patch_ptr[q.p] + lane;
        v -= overflow_dot((dir == 0 ? a.ownr_fw : a.ownr_bw) + 2 * e, a.gcol, a.gval, dsrc);
      }
      a.r[q.i] = v;
    }
  }
  double d = 0.0;
#pragma unroll
  for (int c = 0; c < 16; ++c) d = fma(bcol[c], __shfl_sync(0xffffffffu, v, c), d);
  if (act) {
    a.x[q.i] = xo + d;
    ddst[q.i] = d;
  }
}

// generic patch path (k > 16 or more patches than warps): no prefetch
__device__ void solve_patch_slow(const LegArgs& a, int dir, int64_t p, int lane, bool own, bool init_x,
                                 const double* vin, const double* dsrc, double* ddst) {
  const int64_t e0 = a.patch_ptr[p];
  const int k = (int)(a.patch_ptr[p + 1] - e0);
  const double* Bi = a.binv + a.binv_off[p];
  const int32_t* ownr = dir == 0 ? a.ownr_fw : a.ownr_bw;
  double vals[1] = {0.0};
  (void)vals;
  for (int base = 0; base < k; base += 32) {
    // k <= 32 guaranteed by setup
    int32_t i = 0;
    double v = 0.0;
    const int l = base + lane;
    if (l < k) {
      i = a.dofs[e0 + l];
      v = vin[i];
      if (own) {
        const int32_t s = ownr[2 * (e0 + l)], e = ownr[2 * (e0 + l) + 1];
        if (s >= 0) {
          for (int32_t t = s; t < e; ++t) v -= a.gval[t] * dsrc[a.gcol[t]];
          a.r[i] = v;
        }
      }
    }
    double d = 0.0;
    for (int c = 0; c < k; ++c) {
      const double vc = __shfl_sync(0xffffffffu, v, c);
      if (l < k) d = fma(Bi[(int64_t)c * k + l], vc, d);
    }
    if (l < k) {
      a.x[i] = init_x ? d : a.x[i] + d;
      ddst[i] = d;
    }
  }
}

// kGrid = false: one 16-CTA cluster (split barrier.cluster); kGrid = true: the
// whole GPU as one cooperative grid (grid.sync), for levels whose waves are
// wider than a cluster.
template <bool kDown, bool kGrid = false>
__global__ void __launch_bounds__(kLegThreads, 1) k_leg(LegArgs a) {
  if (*a.stop) return;
  // Grid barrier in two halves (arrive / wait) so the next phase's index
  // prefetch overlaps the barrier latency, as the cluster barrier does.  The
  // word is sense-reversing: block 0 adds 0x80000000 - (blocks - 1), the
  // others add 1, so each barrier flips bit 31 and leaves the low bits as
  // they were (no reset between launches).
  struct Sync {
    cg::cluster_group cl;
    unsigned* bar;
    unsigned old;
    __device__ void arrive() {
      if (kGrid) {
        __syncthreads();
        if (threadIdx.x == 0) {
          const unsigned inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
          asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(bar), "r"(inc) : "memory");
        }
      } else {
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      }
    }
    __device__ void wait() {
      if (kGrid) {
        if (threadIdx.x == 0) {
          unsigned cur;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
          } while (((cur ^ old) & 0x80000000u) == 0);
        }
        __syncthreads();
      } else {
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
      }
    }
    __device__ void sync() {
      arrive();
      wait();
    }
    __device__ unsigned rank() const { return kGrid ? blockIdx.x : cl.block_rank(); }
    __device__ unsigned blocks() const { return kGrid ? gridDim.x : cl.num_blocks(); }
  } cl{cg::this_cluster(), a.gbar, 0u};
  extern __shared__ int64_t sh_ptrs[];  // wave_ptr (W+1) then gen_ptr (W+1)
  const int64_t W = a.nwave, n = a.n;
  int64_t* wp = sh_ptrs;
  int64_t* gp = sh_ptrs + W + 1;
  const int dir = kDown ? 0 : 1;
  for (int64_t t = threadIdx.x; t <= W; t += blockDim.x) {
    wp[t] = a.wave_ptr[t];
    gp[t] = kDown ? a.gen_fw_ptr[t] : a.gen_bw_ptr[t];
  }
  const int64_t nth = (int64_t)cl.blocks() * blockDim.x;
  const int64_t gtid = (int64_t)cl.rank() * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int64_t wg = gtid >> 5, nw = nth >> 5;
  double* dbuf0 = a.d0;
  double* dbuf1 = a.d1;
  __syncthreads();

  if (!kDown) {
    // x += P x_c happened in the previous launch.  r = b - A x ; d = r / l1
    for (int64_t u = gtid; u < n; u += nth) {
      double s = 0.0;
      for (int64_t e = a.ap[u]; e < a.ap[u + 1]; ++e) s = fma(a.av[e], a.x[a.ai[e]], s);
      const double r = a.b[u] - s;
      a.r[u] = r;
      a.dj[u] = r / a.l1[u];
    }
    cl.sync();
    for (int64_t u = gtid; u < n; u += nth) {
      double s = 0.0;
      for (int64_t e = a.ap[u]; e < a.ap[u + 1]; ++e) s = fma(a.av[e], a.dj[a.ai[e]], s);
      a.r[u] -= s;
      a.x[u] += a.dj[u];
    }
    cl.sync();
  }

  // steps: down dst = s (src s-1); up dst = W-1-s (src dst+1)
  PatchPre pq;
  RowPre rq;
  auto prefetch = [&](int64_t s) {
    const int64_t dst = kDown ? s : W - 1 - s;
    const int64_t p = wp[dst] + wg;
    pq.p = -1;
    if (p < wp[dst + 1]) load_patch(a, dir, p, lane, s > 0, pq);
    rq.t = -1;
    if (s > 0) {
      const int64_t src = kDown ? s - 1 : dst + 1;
      const int64_t g0 = kDown ? gp[src] : gp[src], g1 = kDown ? gp[src + 1] : gp[src + 1];
      // rows go to the highest-numbered threads, patches to the lowest warps:
      // a warp never serialises a row pull and a patch solve in one phase
      const int64_t t = g0 + (nth - 1 - gtid);
      if (t < g1) load_row(a, dir, t, rq);
    }
  };
  auto l2pf = [&](int64_t s) {
    if (!kGrid || s >= W) return;
    const int64_t dst = kDown ? s : W - 1 - s;
    int64_t p = wp[dst] + wg, t = -1;
    if (p >= wp[dst + 1]) p = -1;
    if (s > 0) {
      const int64_t src = kDown ? s - 1 : dst + 1;
      t = gp[src] + (nth - 1 - gtid);
      if (t >= gp[src + 1]) t = -1;
    }
    l2_prefetch_phase(a, dir, p, s > 0, t, lane);
  };
  for (int64_t s = 1; s <= a.l2pf; ++s) l2pf(s);
  if (W > 0) prefetch(0);
  if (kDown) {
    for (int64_t u = gtid; u < n; u += nth) {
      a.r[u] = a.b[u];
      if (!a.in_first[u]) a.x[u] = 0.0;
    }
  }
  auto stamp = [&](int64_t s, int which) {
    if (a.trace && lane == 0) {
      long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.trace[(s * nw + wg) * 2 + which] = t;
    }
  };
  for (int64_t s = 0; s < W; ++s) {
    stamp(s, 0);
    if (a.l2pf > 0 && s > 0) l2pf(s + a.l2pf);
    const int64_t dst = kDown ? s : W - 1 - s;
    const int64_t src = kDown ? s - 1 : dst + 1;
    const double* dsrc = s > 0 ? ((src & 1) ? dbuf1 : dbuf0) : nullptr;
    double* ddst = (dst & 1) ? dbuf1 : dbuf0;
    const bool init = kDown && s == 0;
    const double* vin = init ? a.b : a.r;
    // generic pulled rows of the previous wave
    if (s > 0) {
      if (rq.t >= 0) {
        const double r0 = a.r[rq.u];
        double acc = slots_dot(rq.gc, a.ggv[dir] + rq.t, a.ng[dir], rq.cnt, dsrc);
        if (rq.cnt > kSlots) acc += overflow_dot((kDown ? a.genrow_fw : a.genrow_bw) + 3 * rq.t + 1, a.gcol, a.gval, dsrc);
        a.r[rq.u] = r0 - acc;
      }
      const int64_t g0 = gp[src], g1 = gp[src + 1];
      for (int64_t t = g0 + (nth - 1 - gtid) + nth; t < g1; t += nth) {
        const int32_t* g = (kDown ? a.genrow_fw : a.genrow_bw) + 3 * t;
        double acc = 0.0;
        for (int32_t k = g[1]; k < g[2]; ++k) acc = fma(a.gval[k], dsrc[a.gcol[k]], acc);
        a.r[g[0]] -= acc;
      }
    }
    // patches of this wave
    if (pq.p >= 0) {
      if (pq.k > 0) solve_patch(a, dir, pq, lane, init, vin, dsrc, ddst);
      else solve_patch_slow(a, dir, pq.p, lane, s > 0, init, vin, dsrc, ddst);
    }
    for (int64_t p = wp[dst] + wg + nw; p < wp[dst + 1]; p += nw)
      solve_patch_slow(a, dir, p, lane, s > 0, init, vin, dsrc, ddst);
    if (kDown || s + 1 < W) {
      // split cluster barrier: release this phase's stores, then prefetch the
      // next phase's static structure while waiting (the loads are issued
      // after the arrive, so the release does not wait for them)
      stamp(s, 1);
      cl.arrive();
      if (s + 1 < W) prefetch(s + 1);
      cl.wait();
    }
  }
  if (!kDown) return;
  if (W == 0) {
    for (int64_t u = gtid; u < n; u += nth) {
      a.r[u] = a.b[u];
      a.x[u] = 0.0;
    }
    cl.sync();
  }
  // pull the last wave, l1-Jacobi (smoothers.py:106-109)
  const double* dl = W > 0 ? (((W - 1) & 1) ? dbuf1 : dbuf0) : nullptr;
  for (int64_t u = gtid; u < n; u += nth) {
    double v = a.r[u];
    if (W > 0) {
      const int32_t s0 = a.lastr[2 * u], e0 = a.lastr[2 * u + 1];
      for (int32_t k = s0; k < e0 && s0 >= 0; ++k) v -= a.gval[k] * dl[a.gcol[k]];
    }
    const double d = v / a.l1[u];
    a.x[u] += d;
    a.r[u] = v;
    a.dj[u] = d;
  }
  cl.sync();
  for (int64_t u = gtid; u < n; u += nth) {
    double s = 0.0;
    for (int64_t e = a.ap[u]; e < a.ap[u + 1]; ++e) s = fma(a.av[e], a.dj[a.ai[e]], s);
    a.r[u] -= s;
  }
}


}  // namespace

void build_program(Smoother& sm, SweepProgram& pg, cudaStream_t s) {
  const int64_t m = sm.npatch;
  pg.m = m;
  pg.gbar.alloc(1, s);
  pg.gbar.zero();
  pg.pk.alloc(std::max<int64_t>(m, 1), s);
  pg.pdof.alloc(std::max<int64_t>(m * 16, 1), s);
  pg.pbinv.alloc(std::max<int64_t>(m * 256, 1), s);
  pg.ocnt.alloc(std::max<int64_t>(2 * m * 16, 1), s);
  pg.ogc.alloc(std::max<int64_t>(2 * m * kSlots * 16, 1), s);
  pg.ogv.alloc(std::max<int64_t>(2 * m * kSlots * 16, 1), s);
  if (m)
    k_prog_patch<<<grid_for(m * 16, 256), 256, 0, s>>>(m, sm.patch_ptr.p, sm.patch_dofs.p, sm.binv_off.p, sm.binv.p,
                                                        sm.ownr_fw.p, sm.ownr_bw.p, sm.gcol.p, sm.gval.p, pg.pk.p,
                                                        pg.pdof.p, pg.pbinv.p, pg.ocnt.p, pg.ogc.p, pg.ogv.p);
  HC_CHECK_LAUNCH();
  for (int dir = 0; dir < 2; ++dir) {
    const int64_t ng = (dir == 0 ? sm.gen_fw_ptr : sm.gen_bw_ptr).back();
    pg.ng[dir] = ng;
    pg.gu[dir].alloc(std::max<int64_t>(ng, 1), s);
    pg.gcnt[dir].alloc(std::max<int64_t>(ng, 1), s);
    pg.ggc[dir].alloc(std::max<int64_t>(ng * kSlots, 1), s);
    pg.ggv[dir].alloc(std::max<int64_t>(ng * kSlots, 1), s);
    if (ng)
      k_prog_gen<<<grid_for(ng, 256), 256, 0, s>>>(ng, dir == 0 ? sm.genrow_fw.p : sm.genrow_bw.p, sm.gcol.p,
                                                   sm.gval.p, pg.gu[dir].p, pg.gcnt[dir].p, pg.ggc[dir].p,
                                                   pg.ggv[dir].p);
    HC_CHECK_LAUNCH();
  }
}

void launch_leg_grid(bool down, const LegArgs& args, cudaStream_t s) {
  const size_t smem = sizeof(int64_t) * 2 * (size_t)(args.nwave + 1);
  static int per_sm = 0;
  if (!per_sm) {
    int a = 0, b = 0;
    HC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_leg<true, true>, kLegThreads, 16 * 1024));
    HC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_leg<false, true>, kLegThreads, 16 * 1024));
    per_sm = std::max(1, std::min(a, b));
  }
  require(smem <= 16 * 1024, "too many wavefronts for the grid leg");
  int dev = 0, sms = kSMs;
  HC_CUDA(cudaGetDevice(&dev));
  HC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  cudaLaunchConfig_t cfg = {};
  int blocks = sms * per_sm;
  if (const char* e = getenv("HCAMG_GRID_BLOCKS")) blocks = std::min(blocks, std::max(1, atoi(e)));
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(kLegThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  // HCAMG_LEG_L2PF: L2 prefetch distance in waves (0: off)
  static const int l2pf = getenv("HCAMG_LEG_L2PF") ? std::max(0, atoi(getenv("HCAMG_LEG_L2PF"))) : 1;
  LegArgs ga = args;
  ga.l2pf = l2pf;
  if (down) HC_CUDA(cudaLaunchKernelEx(&cfg, k_leg<true, true>, ga));
  else HC_CUDA(cudaLaunchKernelEx(&cfg, k_leg<false, true>, ga));
}

// Largest cluster the leg can use on this device: 16 (non-portable) when
// the occupancy query admits it, else the portable 8.
int sweep_cluster_size() {
  static int c = 0;
  if (c) return c;
  int best = 8;
  cudaFuncSetAttribute(k_leg<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_leg<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(16);
  cfg.blockDim = dim3(kLegThreads);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 16;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, (const void*)k_leg<true>, &cfg) == cudaSuccess && nclusters > 0)
    best = 16;
  cudaGetLastError();
  c = best;
  return c;
}

void launch_leg(bool down, const LegArgs& args, cudaStream_t s) {
  const int C = sweep_cluster_size();
  static bool init = false;
  if (!init) {
    HC_CUDA(cudaFuncSetAttribute(k_leg<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    HC_CUDA(cudaFuncSetAttribute(k_leg<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    init = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(kLegThreads);
  cfg.dynamicSmemBytes = sizeof(int64_t) * 2 * (size_t)(args.nwave + 1);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (down) HC_CUDA(cudaLaunchKernelEx(&cfg, k_leg<true>, args));
  else HC_CUDA(cudaLaunchKernelEx(&cfg, k_leg<false>, args));
}

}  // namespace hcamg
