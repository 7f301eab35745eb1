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
// The kernel is the sweep alone (the last of a DoF's <= 2 patches writes x);
// the l1-Jacobi step around it runs on the fused SpMV kernels (solve.cu:
// r = b - A x, dj = r / l1, then r -= A dj, x += dj) -- after the sweep in
// the down leg, before it in the up leg.
#include <cooperative_groups.h>

#include <algorithm>

#include "level.cuh"
#include "sweep.cuh"

namespace hcamg {

namespace {

constexpr int kFlowThreads = 256;
constexpr int kFlowGates = 8;  // gate slots per record (one per predecessor patch of the latest wave)
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
      // back-off: CTAs that finish their patches early would otherwise poll
      // one L2 line for the rest of the sweep and stall the slot traffic
      unsigned ns = 64;
      while (true) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
        if ((cur ^ old) & 0x80000000u) break;
        __nanosleep(ns);
        ns = min(ns * 2, 1024u);
      }
    }
    __syncthreads();
  }
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// every lane observes the phase (acquire of the bulk copy), and the loop ends
// for the whole warp at once so the warp stays converged
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!__all_sync(0xffffffffu, done != 0))
    if (!done)
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(bar), "r"(parity)
          : "memory");
}

// Patch record (built by build_flow; 16-byte aligned):
//   int32 {k, e0, nt, ngate} | int32 gate[8] (a slot of each latest-wave predecessor) | int32 dof[k4]
//   | int32 tstart[kp4] | int32 xpart[k4] (term index of the DoF's other patch entry when that patch ran
//   earlier: this patch then writes x[u]; -1: the other patch runs later; -2: no other patch) | int32 tstart[kp4] | double binv[k*k] (row-major)
//   | int32 tslot[nt4] | double tval[nt] | pad to 16
__device__ __forceinline__ void rec_layout(int k, int nt, int& o_dof, int& o_ts, int& o_binv, int& o_slot,
                                           int& o_val) {
  const int k4 = (k + 3) & ~3, kp4 = (k + 1 + 3) & ~3, nt4 = (nt + 3) & ~3;
  o_dof = 16 + 4 * kFlowGates;
  o_ts = o_dof + 4 * k4;
  o_binv = o_ts + 4 * kp4 + 4 * k4;  // tstart, then xpart[k4]
  o_slot = o_binv + 8 * k * k;
  o_val = o_slot + 4 * nt4;
}

// one patch from its staged record: v = r0[u] - sum of the pulled terms
// (spinning on slots that still hold the sentinel), d = B_p^{-1} v
__device__ __forceinline__ long long gclock() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
  return t;
}

__device__ __forceinline__ void flow_patch(const FlowArgs& a, const unsigned char* rec, int lane, const double* r0,
                                           const double* x0, long long* tr) {
  const int4 hd = *reinterpret_cast<const int4*>(rec);
  const int k = hd.x, e0 = hd.y, nt = hd.z, ngate = a.gates ? hd.w : 0;
  int o_dof, o_ts, o_binv, o_slot, o_val;
  rec_layout(k, nt, o_dof, o_ts, o_binv, o_slot, o_val);
  const int32_t* dof = reinterpret_cast<const int32_t*>(rec + o_dof);
  const int32_t* ts = reinterpret_cast<const int32_t*>(rec + o_ts);
  const int32_t* xpart = reinterpret_cast<const int32_t*>(rec + o_ts + 4 * ((k + 1 + 3) & ~3));
  const double* binv = reinterpret_cast<const double*>(rec + o_binv);
  const int32_t* tslot = reinterpret_cast<const int32_t*>(rec + o_slot);
  const double* tval = reinterpret_cast<const double*>(rec + o_val);
  const bool act = lane < k;
  double v = 0.0;
  // r0 and the patch's row of B^{-1} are independent of the predecessors:
  // in flight / in registers before the wait.  All control flow below is
  // warp-uniform (spins end on __all_sync / __any_sync): a warp left
  // diverged by per-lane spin loops runs the B^{-1} shuffles on the slow
  // collective path (measured 4 us per patch instead of 0.5)
  const int32_t u = act ? dof[lane] : 0;
  const int32_t xp = act ? xpart[lane] : -1;
  const double rv = act ? r0[u] : 0.0;
  const double xv = (act && xp != -1 && x0) ? x0[u] : 0.0;
  double brow16[16];
  if (k <= 16) {
#pragma unroll
    for (int c = 0; c < 16; ++c) brow16[c] = (act && c < k) ? binv[lane * k + c] : 0.0;
  }
  if (tr) {
    double t_;
    asm volatile("mov.b64 %0, %1;" : "=d"(t_) : "d"(rv) : "memory");  // (trace: wait for it here)
    __syncwarp();
    if (lane == 0) tr[4] = gclock() + (t_ == 1.2345e300);
  }
  // lanes 0..ngate-1 wait on one slot of each predecessor patch of the
  // latest wave (few polling lanes: polls from every term of every lane
  // flood the L2 and delay the very stores being waited for)
  if (ngate > 0) {
    const int32_t g = lane < ngate ? reinterpret_cast<const int32_t*>(rec + 16)[lane] : 0;
    bool ok = lane >= ngate;
    while (!__all_sync(0xffffffffu, ok)) {
      if (!ok) ok = !is_sentinel(ld_slot(a.d + g));
      if (a.spin_ns && !__all_sync(0xffffffffu, ok)) __nanosleep(a.spin_ns);
    }
  }
  // every pulled slot of the entry loaded at once (one L2 round trip); slots
  // of earlier-wave predecessors that are still pending are polled again
  // Branch- and predicate-free: a lane's unused positions load the spare slot
  // d[ne] (always 0.0), so all 32 loads are issued before the first result is
  // tested.  With a load-and-test per term under `i < cnt` the compiler runs
  // out of predicate registers and waits for the loads in groups of 2-5
  // (SASS: ISETP on the first result between the LDGs): 3-4 L2 round trips
  // per patch instead of one.
  const int t0 = act ? ts[lane] : 0, t1 = act ? ts[lane + 1] : 0;
  const int cnt = min(32, t1 - t0);
  const int tl = max(nt - 1, 0);
  const int32_t spare = (int32_t)a.ne;
  double x[32];
  unsigned pend = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int32_t sl = tslot[min(t0 + i, tl)];
    x[i] = ld_slot(a.d + (i < cnt ? sl : spare));
  }
  // (scheduling fence: every load above is issued before any result below is tested)
  asm volatile("" : "+d"(x[0]), "+d"(x[1]), "+d"(x[2]), "+d"(x[3]), "+d"(x[4]), "+d"(x[5]), "+d"(x[6]), "+d"(x[7]),
                    "+d"(x[8]), "+d"(x[9]), "+d"(x[10]), "+d"(x[11]), "+d"(x[12]), "+d"(x[13]), "+d"(x[14]), "+d"(x[15]));
  asm volatile("" : "+d"(x[16]), "+d"(x[17]), "+d"(x[18]), "+d"(x[19]), "+d"(x[20]), "+d"(x[21]), "+d"(x[22]),
                    "+d"(x[23]), "+d"(x[24]), "+d"(x[25]), "+d"(x[26]), "+d"(x[27]), "+d"(x[28]), "+d"(x[29]),
                    "+d"(x[30]), "+d"(x[31]));
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (is_sentinel(x[i])) pend |= 1u << i;  // (the spare slot never holds the sentinel)
  while (__any_sync(0xffffffffu, pend != 0)) {
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (pend & (1u << i)) {
        x[i] = ld_slot(a.d + tslot[t0 + i]);
        if (!is_sentinel(x[i])) pend &= ~(1u << i);
      }
  }
  double acc = 0.0, dpart = 0.0;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    if (i < cnt) acc = fma(tval[t0 + i], x[i], acc);
    if (i == xp) dpart = x[i];
  }
  for (int t = t0 + 32; __any_sync(0xffffffffu, t < t1); ++t) {  // entries with more than 32 terms (rare)
    bool done = t >= t1;
    double y = 0.0;
    while (!__all_sync(0xffffffffu, done))
      if (!done) {
        y = ld_slot(a.d + tslot[t]);
        done = !is_sentinel(y);
      }
    if (t < t1) acc = fma(tval[t], y, acc);
  }
  v = act ? rv - acc : 0.0;
  if (tr) {
    double t_;
    asm volatile("mov.b64 %0, %1;" : "=d"(t_) : "d"(v) : "memory");
    __syncwarp();
    if (lane == 0) tr[1] = gclock() + (t_ == 1.2345e300);
  }
  double d = 0.0;
  if (k <= 16) {
#pragma unroll
    for (int c = 0; c < 16; ++c) d = fma(brow16[c], __shfl_sync(0xffffffffu, v, c), d);
  } else {
    const double* brow = binv + (act ? lane * k : 0);
    for (int c = 0; c < k; ++c) d = fma(act ? brow[c] : 0.0, __shfl_sync(0xffffffffu, v, c), d);
  }
  if (tr) {
    double t_;
    asm volatile("mov.b64 %0, %1;" : "=d"(t_) : "d"(d) : "memory");
    __syncwarp();
    if (lane == 0) tr[5] = gclock() + (t_ == 1.2345e300);
  }
  if (act) {
    st_slot(a.d + e0 + lane, d);
    // the last of the DoF's (<= 2) patches writes x: (x0 + d_earlier) + d,
    // the reference's x[patch] += d order (smoothers.py:102)
    if (xp >= 0) a.x[u] = x0 ? (xv + dpart) + d : dpart + d;
    else if (xp == -2) a.x[u] = x0 ? xv + d : d;
  }
  if (tr) {
    __syncwarp();
    if (lane == 0) tr[2] = gclock();
  }
}

template <bool kDown>
__global__ void __launch_bounds__(kFlowThreads, 1) k_flow_leg(FlowArgs a) {
  if (*a.stop) return;
  GridBar gb{a.bar};
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int64_t wg = gtid >> 5, nw = nth >> 5;
  const double* r0 = a.r0;
  {
    // each warp walks its patches (exec positions wg, wg + nw, ...) with the
    // next record streamed into the other half of its double buffer by one
    // cp.async.bulk while the current one waits on its predecessors
    extern __shared__ __align__(16) unsigned char flow_smem[];
    __shared__ __align__(8) unsigned long long bars[kFlowThreads / 32][2];
    const int wl = threadIdx.x >> 5;
    unsigned char* buf0 = flow_smem + (size_t)wl * 2 * a.recmax;
    const uint32_t bar0 = smem_u32(&bars[wl][0]), bar1 = smem_u32(&bars[wl][1]);
    if (lane == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar1));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const unsigned char* recs = a.recs;
    auto issue = [&](int64_t i, int b) {
      const int64_t o = a.rec_off[i];
      const uint32_t bytes = (uint32_t)(a.rec_off[i + 1] - o);
      const uint32_t bar = b ? bar1 : bar0;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(buf0 + (size_t)b * a.recmax)),
                   "l"(recs + o), "r"(bytes), "r"(bar)
                   : "memory");
    };
    const int64_t m = a.npatch;
    if (a.dynamic) {
      // Patches claimed in execution order from a ticket (a.bar[1]) when the
      // warp has finished its previous one.  With the static round-robin a warp
      // whose patch i is late (its predecessors straggle) cannot attend patch
      // i + nw, seven waves on, although that patch's own predecessors are
      // done: head-of-line blocking put 5-15 us links on the critical chain
      // (tools/trace_flow.py: median link 1.5 us, mean 3).  A claimed patch
      // always has its own waiting warp; the claim frontier runs nw patches
      // ahead of the completion frontier, so the claim (ticket, offsets,
      // record copy: ~2.5 us) is off the critical path.  The first unfinished
      // patch is always held by a running warp: no deadlock.
      unsigned* ticket = a.bar + 1;
      int64_t i = wg;
      for (uint32_t j = 0; i < m; ++j) {
        if (lane == 0) issue(i, 0);
        __syncwarp();
        mbar_wait(bar0, j & 1u);
        long long* tr = a.trace ? a.trace + 6 * i : nullptr;
        if (tr && lane == 0) {
          tr[0] = gclock();
          tr[3] = wg;
        }
        flow_patch(a, buf0, lane, r0, kDown ? nullptr : a.x, tr);
        __syncwarp();
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(ticket, 1u);
        i = nw + (int64_t)__shfl_sync(0xffffffffu, t, 0);
      }
    } else {
      if (lane == 0 && wg < m) issue(wg, 0);
      int64_t j = 0;
      for (int64_t i = wg; i < m; i += nw, ++j) {
        const int b = (int)(j & 1);
        if (lane == 0 && i + nw < m) issue(i + nw, b ^ 1);
        __syncwarp();
        mbar_wait(b ? bar1 : bar0, (uint32_t)((j >> 1) & 1));
        long long* tr = a.trace ? a.trace + 6 * i : nullptr;
        if (tr && lane == 0) {
          tr[0] = gclock();
          tr[3] = wg;
        }
        flow_patch(a, buf0 + (size_t)b * a.recmax, lane, r0, kDown ? nullptr : a.x, tr);
        __syncwarp();
      }
    }
  }
  gb.sync();  // every slot has been read: hand them back to the sentinel for the next leg
  const double sent = __longlong_as_double((long long)kSentinel);
  for (int64_t e = gtid; e < a.ne; e += nth) a.d[e] = sent;
  if (gtid == 0) a.bar[1] = 0u;  // the ticket of the next leg
}

// ---- wave-parallel sweep over the same records (mode "fwave": the default for
// shallow, very wide schedules -- 2D: 7-10 waves of tens of thousands of 6-DoF
// patches).  One launch per wavefront, so no slot is ever pending and there are
// no gates or sentinels; what the records buy here is traffic: a patch needs
// its record (streamed once, contiguous per wave), r0 at its DoFs and the slots
// of its terms -- no read-modify-write of a full-length residual and of two
// full-length correction vectors per wave, which on these schedules touch one
// DoF in seven per wave and so move every 32-byte sector of r, x, d0, d1 seven
// times per leg (measured: 314 MB per level-0 wave at 3.1 M DoFs, 2x the
// algorithmic bytes).  A CTA copies the records of its kPer consecutive patches
// into shared memory with 16-byte loads (a contiguous range: full-rate,
// independent loads), then kG lanes per patch parse them there; the only
// dependent global loads are r0[u] and the term slots.
constexpr int kFwThreads = 256;
#ifndef FW_TERM_BATCH
#define FW_TERM_BATCH 8
#endif

template <int kG, bool kDown>
__global__ void __launch_bounds__(kFwThreads) k_flow_wave(FlowArgs a, int64_t i0, int64_t cnt) {
  if (*a.stop) return;
  extern __shared__ __align__(16) unsigned char fw_smem[];
  constexpr int kPer = kFwThreads / kG;
  __shared__ int64_t off_sh[kPer + 1];
  const int64_t tb = (int64_t)blockIdx.x * kPer;
  const int np = (int)(cnt - tb < (int64_t)kPer ? cnt - tb : (int64_t)kPer);
  for (int j = threadIdx.x; j <= np; j += kFwThreads) off_sh[j] = a.rec_off[i0 + tb + j];
  __syncthreads();
  const int64_t base = off_sh[0];
  const int bytes = (int)(off_sh[np] - base);
  {
    const int4* src = reinterpret_cast<const int4*>(a.recs + base);
    int4* dst = reinterpret_cast<int4*>(fw_smem);
    for (int q = threadIdx.x; q < bytes / 16; q += kFwThreads) dst[q] = __ldg(src + q);
  }
  __syncthreads();
  const int sub = threadIdx.x & (kG - 1), pl = threadIdx.x / kG;
  const bool have = pl < np;
  const unsigned char* rec = fw_smem + (have ? (off_sh[pl] - base) : 0);
  const int4 hd = have ? *reinterpret_cast<const int4*>(rec) : make_int4(0, 0, 0, 0);
  const int k = hd.x, e0 = hd.y, nt = hd.z;
  int o_dof, o_ts, o_binv, o_slot, o_val;
  rec_layout(k, nt, o_dof, o_ts, o_binv, o_slot, o_val);
  const int32_t* dof = reinterpret_cast<const int32_t*>(rec + o_dof);
  const int32_t* ts = reinterpret_cast<const int32_t*>(rec + o_ts);
  const int32_t* xpart = reinterpret_cast<const int32_t*>(rec + o_ts + 4 * ((k + 1 + 3) & ~3));
  const double* binv = reinterpret_cast<const double*>(rec + o_binv);
  const int32_t* tslot = reinterpret_cast<const int32_t*>(rec + o_slot);
  const double* tval = reinterpret_cast<const double*>(rec + o_val);
  const bool act = have && sub < k;
  const int32_t u = act ? dof[sub] : 0;
  const int32_t xp = act ? xpart[sub] : -1;
  const double rv = act ? a.r0[u] : 0.0;
  const double xv = (!kDown && act && xp != -1) ? a.x[u] : 0.0;
  const int t0 = act ? ts[sub] : 0, t1 = act ? ts[sub + 1] : 0;
  double acc = 0.0, dpart = 0.0;
  constexpr int kTB = FW_TERM_BATCH;  // term loads in flight per lane
  for (int tt = t0; tt < t1; tt += kTB) {
    double xs[kTB];
#pragma unroll
    for (int j = 0; j < kTB; ++j) xs[j] = tt + j < t1 ? __ldcg(a.d + tslot[tt + j]) : 0.0;
#pragma unroll
    for (int j = 0; j < kTB; ++j)
      if (tt + j < t1) {
        acc = fma(tval[tt + j], xs[j], acc);
        if (tt + j - t0 == xp) dpart = xs[j];
      }
  }
  const double v = act ? rv - acc : 0.0;
  double d = 0.0;
#pragma unroll
  for (int c = 0; c < kG; ++c) {
    const double vc = __shfl_sync(0xffffffffu, v, c, kG);
    if (act && c < k) d = fma(binv[sub * k + c], vc, d);
  }
  if (act) {
    a.d[e0 + sub] = d;
    // the last of the DoF's (<= 2) patches writes x: (x0 + d_earlier) + d (smoothers.py:102)
    if (xp >= 0) a.x[u] = kDown ? dpart + d : (xv + dpart) + d;
    else if (xp == -2) a.x[u] = kDown ? d : xv + d;
  }
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

int64_t flow_smem_bytes(int64_t recmax) { return (kFlowThreads / 32) * 2 * recmax; }

bool flow_wave_ok(int64_t kmax, int64_t recmax) { return kmax <= 8 && (kFwThreads / 8) * recmax <= 96 * 1024; }

// patches [i0, i0 + cnt) of the direction's execution order: one wavefront
void launch_flow_wave(bool down, const FlowArgs& args, int64_t i0, int64_t cnt, cudaStream_t s) {
  if (cnt <= 0) return;
  constexpr int kG = 8, kPer = kFwThreads / kG;
  const size_t smem = (size_t)kPer * (size_t)args.recmax;
  static size_t attr = 0;
  if (smem > attr) {
    HC_CUDA(cudaFuncSetAttribute(k_flow_wave<kG, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    HC_CUDA(cudaFuncSetAttribute(k_flow_wave<kG, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  const unsigned grid = (unsigned)((cnt + kPer - 1) / kPer);
  if (down) k_flow_wave<kG, true><<<grid, kFwThreads, smem, s>>>(args, i0, cnt);
  else k_flow_wave<kG, false><<<grid, kFwThreads, smem, s>>>(args, i0, cnt);
  HC_CHECK_LAUNCH();
}

void launch_flow_leg(bool down, const FlowArgs& args, cudaStream_t s) {
  const size_t smem = (size_t)flow_smem_bytes(args.recmax);
  static size_t attr = 0;
  if (smem > attr) {
    HC_CUDA(cudaFuncSetAttribute(k_flow_leg<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    HC_CUDA(cudaFuncSetAttribute(k_flow_leg<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  int a = 0, b = 0;
  HC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_flow_leg<true>, kFlowThreads, smem));
  HC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_flow_leg<false>, kFlowThreads, smem));
  const int per_sm = std::max(1, std::min(a, b));
  int dev = 0, sms = kSMs;
  HC_CUDA(cudaGetDevice(&dev));
  HC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int blocks = sms * std::min(per_sm, 2);
  if (const char* e = getenv("HCAMG_FLOW_BLOCKS")) blocks = std::min(blocks, std::max(1, atoi(e)));
  FlowArgs fa = args;
  fa.spin_ns = getenv("HCAMG_FLOW_NS") ? (unsigned)atoi(getenv("HCAMG_FLOW_NS")) : 0u;  // measurement knobs
  fa.gates = getenv("HCAMG_FLOW_GATE") ? atoi(getenv("HCAMG_FLOW_GATE")) : 1;
  fa.dynamic = getenv("HCAMG_FLOW_DYN") ? atoi(getenv("HCAMG_FLOW_DYN")) : 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(kFlowThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (down) HC_CUDA(cudaLaunchKernelEx(&cfg, k_flow_leg<true>, fa));
  else HC_CUDA(cudaLaunchKernelEx(&cfg, k_flow_leg<false>, fa));
}

}  // namespace hcamg
