// Dataflow OSS-l1 smoothing leg (option sweep = 4, "flow"; the default for
// levels whose waves are wider than one cluster).
//
// The reference's multiplicative Schwarz sweep (smoothers.py:98-103) visits
// the patches in order; patch q must see the corrections of every earlier
// patch p that is A-coupled to it.  Round 1 ran the sweep wave by wave with a
// grid barrier between waves (k_leg<., true>): 94 waves on config 2's level 0
// at ~4 us each.  Here there is no barrier inside the sweep:
//
//   * every patch entry (patch q, DoF u) owns a correction slot d[e];
//   * the residual patch q needs is r0[u] - sum over the earlier coupled
//     patches p of A[u, j] d_p[j] -- a fixed list of (slot, A[u, j]) terms per
//     entry built at setup (smoother.cu, build_flow), identical whatever the
//     timing, so the result is deterministic run to run;
//   * slots start as a sentinel NaN and are written exactly once per leg; a
//     consumer spins (ld.relaxed.gpu) on the slots it reads until they hold a
//     value, so a patch starts as soon as its own predecessors are done and
//     the critical path is the dependency chain (one L2 round trip per link)
//     instead of waves x (barrier + latency);
//   * warps take the patches of every wave round-robin in wave order, so the
//     globally first unfinished patch is always runnable (no deadlock in a
//     co-resident cooperative grid).
//
// Around the sweep the leg does the l1-Jacobi step and the bookkeeping in
// grid-wide phases separated by a sense-reversing barrier:
//   down: sweep from r0 = b (x0 = 0) | x = delta, r1 = b - A delta, dj = r1 / l1,
//         x += dj | r = r1 - A dj, slots reset
//   up:   r = b - A x, dj = r / l1 | r0 = r - A dj, x += dj | sweep (reverse
//         wave order) | x += delta, slots reset
// where delta[u] is the sum of u's entry slots (a DoF sits in <= 2 vertex
// patches).
#include <cooperative_groups.h>

#include <algorithm>

#include "level.cuh"
#include "sweep.cuh"

namespace hcamg {

namespace {

constexpr int kFlowThreads = 256;
constexpr unsigned long long kSentinel = 0x7ff4dead5eed0001ull;  // a NaN no arithmetic produces

__device__ __forceinline__ double ld_slot(const double* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return __longlong_as_double((long long)v);
}
__device__ __forceinline__ void st_slot(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"((unsigned long long)__double_as_longlong(v))
               : "memory");
}
__device__ __forceinline__ bool is_sentinel(double v) {
  return (unsigned long long)__double_as_longlong(v) == kSentinel;
}

struct GridBar {
  unsigned* bar;
  __device__ void sync() {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
      unsigned old, cur;
      asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(bar), "r"(inc) : "memory");
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
      } while (((cur ^ old) & 0x80000000u) == 0);
    }
    __syncthreads();
  }
};

// sum of the pulled terms of one entry: spins on every slot still holding the sentinel
__device__ __forceinline__ double pull_terms(const FlowArgs& a, int32_t t0, int32_t t1) {
  double acc = 0.0;
  for (int32_t t = t0; t < t1; t += 8) {
    int32_t sl[8];
    double w[8], v[8];
    const int cnt = min(8, t1 - t);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      sl[i] = i < cnt ? __ldg(a.tslot + t + i) : -1;
      w[i] = i < cnt ? __ldg(a.tval + t + i) : 0.0;
    }
    unsigned pending = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      v[i] = 0.0;
      if (sl[i] >= 0) {
        v[i] = ld_slot(a.d + sl[i]);
        if (is_sentinel(v[i])) pending |= 1u << i;
      }
    }
    while (pending) {
      __nanosleep(32);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (pending & (1u << i)) {
          v[i] = ld_slot(a.d + sl[i]);
          if (!is_sentinel(v[i])) pending &= ~(1u << i);
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) acc = fma(w[i], v[i], acc);
  }
  return acc;
}

__device__ __forceinline__ void flow_patch(const FlowArgs& a, int64_t p, int lane, const double* r0) {
  const int64_t e0 = a.patch_ptr[p];
  const int k = (int)(a.patch_ptr[p + 1] - e0);
  const bool act = lane < k;
  const int64_t e = e0 + lane;
  int32_t u = 0;
  int32_t t0 = 0, t1 = 0;
  double v = 0.0;
  if (act) {
    u = a.dofs[e];
    t0 = a.tp[e];
    t1 = a.tp[e + 1];
    v = r0[u];
  }
  // row `lane` of the k x k inverse (column-major), loaded before the spin
  const double* Bi = a.binv + a.binv_off[p];
  double d = 0.0;
  if (k <= 16) {
    double brow[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) brow[c] = (act && c < k) ? __ldg(Bi + (int64_t)c * k + lane) : 0.0;
    if (act) v -= pull_terms(a, t0, t1);
#pragma unroll
    for (int c = 0; c < 16; ++c) d = fma(brow[c], __shfl_sync(0xffffffffu, v, c), d);
  } else {
    double brow[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) brow[c] = (act && c < k) ? __ldg(Bi + (int64_t)c * k + lane) : 0.0;
    if (act) v -= pull_terms(a, t0, t1);
#pragma unroll
    for (int c = 0; c < 32; ++c) d = fma(brow[c], __shfl_sync(0xffffffffu, v, c), d);
  }
  if (act) st_slot(a.d + e, d);
}

template <bool kDown>
__global__ void __launch_bounds__(kFlowThreads, 1) k_flow_leg(FlowArgs a) {
  if (*a.stop) return;
  GridBar gb{a.bar};
  const int64_t n = a.n, W = a.nwave;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int64_t wg = gtid >> 5, nw = nth >> 5;
  if (!kDown) {
    // r = b - A x ; dj = r / l1   (smoothers.py:106-109, before the reverse sweep)
    for (int64_t u = gtid; u < n; u += nth) {
      double s = 0.0;
      for (int64_t e = a.ap[u]; e < a.ap[u + 1]; ++e) s = fma(a.av[e], a.x[a.ai[e]], s);
      const double r = a.b[u] - s;
      a.r[u] = r;
      a.dj[u] = r / a.l1[u];
    }
    gb.sync();
    for (int64_t u = gtid; u < n; u += nth) {
      double s = 0.0;
      for (int64_t e = a.ap[u]; e < a.ap[u + 1]; ++e) s = fma(a.av[e], a.dj[a.ai[e]], s);
      a.r1[u] = a.r[u] - s;
      a.x[u] += a.dj[u];
    }
    gb.sync();
  }
  const double* r0 = kDown ? a.b : a.r1;
  for (int64_t s = 0; s < W; ++s) {
    const int64_t w = kDown ? s : W - 1 - s;
    const int64_t p0 = a.wave_ptr[w], p1 = a.wave_ptr[w + 1];
    for (int64_t p = p0 + wg; p < p1; p += nw) flow_patch(a, p, lane, r0);
  }
  gb.sync();
  if (kDown) {
    // x = delta ; r1 = b - A delta ; dj = r1 / l1 ; x += dj
    for (int64_t u = gtid; u < n; u += nth) {
      double s = 0.0;
      for (int64_t e = a.ap[u]; e < a.ap[u + 1]; ++e) {
        const int2 en = a.ent[a.ai[e]];
        double dl = 0.0;
        if (en.x >= 0) dl = ld_slot(a.d + en.x);
        if (en.y >= 0) dl += ld_slot(a.d + en.y);
        s = fma(a.av[e], dl, s);
      }
      const int2 me = a.ent[u];
      double xu = 0.0;
      if (me.x >= 0) xu = ld_slot(a.d + me.x);
      if (me.y >= 0) xu += ld_slot(a.d + me.y);
      const double r1 = a.b[u] - s;
      const double dj = r1 / a.l1[u];
      a.r1[u] = r1;
      a.dj[u] = dj;
      a.x[u] = xu + dj;
    }
    gb.sync();
    for (int64_t u = gtid; u < n; u += nth) {
      double s = 0.0;
      for (int64_t e = a.ap[u]; e < a.ap[u + 1]; ++e) s = fma(a.av[e], a.dj[a.ai[e]], s);
      a.r[u] = a.r1[u] - s;
    }
  } else {
    for (int64_t u = gtid; u < n; u += nth) {
      const int2 me = a.ent[u];
      double dl = 0.0;
      if (me.x >= 0) dl = ld_slot(a.d + me.x);
      if (me.y >= 0) dl += ld_slot(a.d + me.y);
      a.x[u] += dl;
    }
    gb.sync();  // the slot reads above must finish before the reset
  }
  // every slot was read above; hand them back to the sentinel for the next leg
  const double sent = __longlong_as_double((long long)kSentinel);
  for (int64_t e = gtid; e < a.ne; e += nth) a.d[e] = sent;
}

__global__ void k_fill_sentinel(double* d, int64_t n) {
  const double sent = __longlong_as_double((long long)kSentinel);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    d[e] = sent;
}

}  // namespace

void flow_reset_slots(double* d, int64_t ne, cudaStream_t s) {
  if (ne) k_fill_sentinel<<<grid_for(ne, 256), 256, 0, s>>>(d, ne);
  HC_CHECK_LAUNCH();
}

void launch_flow_leg(bool down, const FlowArgs& args, cudaStream_t s) {
  static int per_sm = 0;
  if (!per_sm) {
    int a = 0, b = 0;
    HC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_flow_leg<true>, kFlowThreads, 0));
    HC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_flow_leg<false>, kFlowThreads, 0));
    per_sm = std::max(1, std::min(a, b));
  }
  int dev = 0, sms = kSMs;
  HC_CUDA(cudaGetDevice(&dev));
  HC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int blocks = sms * std::min(per_sm, 2);
  if (const char* e = getenv("HCAMG_FLOW_BLOCKS")) blocks = std::min(blocks, std::max(1, atoi(e)));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(kFlowThreads);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (down) HC_CUDA(cudaLaunchKernelEx(&cfg, k_flow_leg<true>, args));
  else HC_CUDA(cudaLaunchKernelEx(&cfg, k_flow_leg<false>, args));
}

}  // namespace hcamg
