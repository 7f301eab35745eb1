// Blocked triangular sweeps over the envelope Cholesky factor of A_GG, and
// the factored interpolation block built on them (see trisolve.cuh).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include "sparse.cuh"
#include "trisolve.cuh"

namespace hcamg {

namespace {

constexpr int kNB = (int)kTriSB;  // rows per sweep step

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
      if (T.b < 0) {  // fold
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

// ---- dataflow sweep (default) ----------------------------------------------
//
// No grid barriers: every task (one operator row) waits only for what it
// reads.  Tasks keep the step order of the sweep and are dealt to warps
// round-robin (warp w: tasks w, w + W, ...); every dependency points to an
// earlier task, so with all warps resident the sweep cannot deadlock.
//   crit task of step s (block k): y_k[r] = Linv_k[r].u_k - M_k[r].y_c, after
//     ydone[s-1] = NB (all of y_c) and ufull[k] = nfold[k] (every fold into u_k);
//   fold task of step s: u[out] -= L[r].y_c, after ydone[s-1] = NB and after
//     the previous fold into the same row (rowseq[out] = its sequence number),
//     so the folds into a row happen in step order: bit-identical to the
//     barrier kernel and deterministic.
// While it waits, a warp holds its row's operator chunks in registers (the
// rows do not depend on the vectors) and has the next task's rows prefetched
// into L2, so the dependency chain costs only vector reads and the dot.

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void spin_until(const unsigned* p, unsigned want) {
  while (ld_acq(p) < want) __nanosleep(40);
}

struct FlowArgs {
  TriArgs t;
  int64_t ntask;
  const int32_t* nfold;
  unsigned* ydone;   // per step: crit rows done
  unsigned* ufull;   // per block: fold rows done
  unsigned* rowseq;  // per row: folds applied so far
};

__global__ void __launch_bounds__(512, 1) k_tri_flow(FlowArgs F) {
  const TriArgs& a = F.t;
  if (*a.stop) return;
  const int lane = threadIdx.x & 31;
  const int64_t W = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int64_t st = 0;
  TriStepD S = a.steps[0];
  for (int64_t t = gw; t < F.ntask; t += W) {
    while (t >= S.t1) S = a.steps[++st];
    const TriTask T = a.tasks[t];
    if (lane == 0 && t + W < F.ntask) {  // the next task's rows into L2
      const TriTask Tn = a.tasks[t + W];
      prefetch_l2(a.pool + Tn.a + 64 * Tn.ja0, 512u * (Tn.ja1 - Tn.ja0));
      if (Tn.b >= 0 && Tn.jb1 > Tn.jb0) prefetch_l2(a.pool + Tn.b + 64 * Tn.jb0, 512u * (Tn.jb1 - Tn.jb0));
    }
    // this row's operator chunks (A part) into registers while the dependencies resolve
    double2 v[16];
    const double2* rp = reinterpret_cast<const double2*>(a.pool + T.a + 2 * lane);
#pragma unroll
    for (int q = 0; q < 16; ++q)
      if (q >= T.ja0 && q < T.ja1) v[q] = __ldg(rp + 32 * q);
    const bool fold = T.b < 0;
    const int blk = T.out / kNB;
    if (lane == 0 && a.dbg != 1) {
      if (st > 0) spin_until(F.ydone + st - 1, (unsigned)kNB);
      if (fold) spin_until(F.rowseq + T.out, (unsigned)(-1 - T.b));
      else spin_until(F.ufull + blk, (unsigned)F.nfold[blk]);
    }
    __syncwarp();
    const double* xa = fold ? a.y + (int64_t)S.c * kNB : a.u + (int64_t)blk * kNB;
    double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
    for (int q = 0; q < 16; ++q)
      if (q >= T.ja0 && q < T.ja1) {
        const double2 xv = __ldcg(reinterpret_cast<const double2*>(xa + 64 * q + 2 * lane));
        acc0 = fma(v[q].x, xv.x, acc0);
        acc1 = fma(v[q].y, xv.y, acc1);
      }
    for (int q = 16; q < T.ja1; ++q)  // rows longer than 16 chunks (sweep blocks above 1024 rows)
      if (q >= T.ja0) {
        const double2 w = __ldg(rp + 32 * q);
        const double2 xv = __ldcg(reinterpret_cast<const double2*>(xa + 64 * q + 2 * lane));
        acc0 = fma(w.x, xv.x, acc0);
        acc1 = fma(w.y, xv.y, acc1);
      }
    double da = acc0 + acc1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) da += __shfl_xor_sync(0xffffffffu, da, o);
    if (fold) {
      if (lane == 0) {
        double* o = a.u + T.out;
        *o = __ldcg(o) - da;
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(F.rowseq + T.out), "r"((unsigned)(-T.b)) : "memory");
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(F.ufull + blk) : "memory");
      }
    } else {
      double db = 0.0;
      if (S.c >= 0) {  // M_k row . y_c, same chunk order as warp_dot
        const double2* bp = reinterpret_cast<const double2*>(a.pool + T.b + 2 * lane);
        const double2* yp = reinterpret_cast<const double2*>(a.y + (int64_t)S.c * kNB + 2 * lane);
        double b0 = 0.0, b1 = 0.0;
        for (int j = T.jb0; j < T.jb1; j += 8) {
          double2 w[8];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (j + q < T.jb1) w[q] = __ldg(bp + 32 * (j + q));
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (j + q < T.jb1) {
              const double2 yv = __ldcg(yp + 32 * (j + q));
              b0 = fma(w[q].x, yv.x, b0);
              b1 = fma(w[q].y, yv.y, b1);
            }
        }
        db = b0 + b1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) db += __shfl_xor_sync(0xffffffffu, db, o);
      }
      if (lane == 0) {
        a.y[T.out] = da - db;
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(F.ydone + st) : "memory");
      }
    }
  }
}

// ---- TMA-streamed sweep (default) -----------------------------------------
//
// One CTA per SM; the tasks of a step are split across CTAs contiguously by
// bytes, so the operator rows a CTA needs in a step are one contiguous pool
// region, cut into batches of whole tasks (<= one ring slot).  Warp 0 (one lane)
// streams the batches, step after step, into a ring of 3 x 61 KB shared
// buffers with cp.async.bulk (completion on the buffer's "full" mbarrier),
// running ahead of the grid barriers as far as the ring allows: HBM keeps
// streaming while the consumers synchronise.  Warps 1..kCons (16) consume: per
// step they load the CTA's task descriptors (before the grid barrier: they do
// not depend on it), then after the barrier stage u_k / y_c and the fold
// targets' current values in one round trip, compute every row dot from
// shared memory (same order as the other kernels: bit-identical), and write
// all outputs at the end of the step.

constexpr int kRingB = (kNB == 512 ? 192 : kNB == 1024 ? 184 : 168) * 1024, kMaxCtaTasks = 352,
              kMaxCtaBatches = 64;
constexpr size_t kTmaSmem = 2 * kNB * 8 + (size_t)kRingB + (size_t)kMaxCtaTasks * (2 * sizeof(TriTask) + 8) +
                            (2 * 8 + 4) * 8;

struct TmaArgs {
  TriArgs t;
  unsigned long long* trace;  // HCAMG_TRI_DBG=3: per CTA accumulated phase times (ns)
  const int64_t* ctask;
  const int64_t* bptr;
  const TriBatch* batches;
  const int64_t* cptr;   // the same batches per CTA in stream order
  const TriBatch* cbat;
  int G, pfd, barmode;
  int tmem;  // stage the next step's first rows in tensor memory across the barrier
  unsigned long long* tl;  // HCAMG_TRI_DBG=4: per step and CTA, tasks done / barrier passed (globaltimer)
  long long* tlb;          // HCAMG_TRI_DBG=4: batches of later steps already issued to the ring, at done / at pass
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// tensor memory (TMEM) as a second staging level: a warp's 32 lanes x 4
// columns of 32 bits hold one 64-column chunk of a row (lane l: doubles 2l, 2l+1)
__device__ __forceinline__ void tmem_st4(uint32_t taddr, double2 v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr),
               "r"((uint32_t)__double2loint(v.x)), "r"((uint32_t)__double2hiint(v.x)),
               "r"((uint32_t)__double2loint(v.y)), "r"((uint32_t)__double2hiint(v.y))
               : "memory");
}
__device__ __forceinline__ double2 tmem_ld4(uint32_t taddr) {
  uint32_t r0, r1, r2, r3;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(taddr)
               : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  return make_double2(__hiloint2double((int)r1, (int)r0), __hiloint2double((int)r3, (int)r2));
}
// dot of n chunks held in TMEM (chunk q at column col + 4 q) with x, in smem_dot's order
__device__ __forceinline__ double tmem_dot(uint32_t taddr, const double* x, int n, int lane) {
  double acc0 = 0.0, acc1 = 0.0;
  const double2* xp = reinterpret_cast<const double2*>(x + 2 * lane);
  for (int q = 0; q < n; ++q) {
    const double2 v = tmem_ld4(taddr + 4 * q), xv = xp[32 * q];
    acc0 = fma(v.x, xv.x, acc0);
    acc1 = fma(v.y, xv.y, acc1);
  }
  double acc = acc0 + acc1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

template <int kCons>
__device__ __forceinline__ void cons_sync() { asm volatile("bar.sync 1, %0;" ::"r"(32 * kCons) : "memory"); }

// dot of chunks [0, n) of a row in shared memory (chunk q at row + 64 q) with x (chunk q at x + 64 q)
__device__ __forceinline__ double smem_dot(const double* row, const double* x, int n, int lane) {
  double acc0 = 0.0, acc1 = 0.0;
  const double2* rp = reinterpret_cast<const double2*>(row + 2 * lane);
  const double2* xp = reinterpret_cast<const double2*>(x + 2 * lane);
#pragma unroll 4
  for (int q = 0; q < n; ++q) {
    const double2 v = rp[32 * q], xv = xp[32 * q];
    acc0 = fma(v.x, xv.x, acc0);
    acc1 = fma(v.y, xv.y, acc1);
  }
  double acc = acc0 + acc1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

template <int kCons, int kNBuf>
__global__ void __launch_bounds__(32 * (2 + kCons), 1) k_tri_tma(TmaArgs A) {
  constexpr int kBufB = (kRingB / kNBuf) & ~511;  // slot stride (= the host batch cap)
  const TriArgs& a = A.t;
  if (*a.stop) return;
  extern __shared__ __align__(128) unsigned char smem[];
  double* su = reinterpret_cast<double*>(smem);
  double* sy = su + kNB;
  unsigned char* buf = smem + 2 * kNB * 8;
  TriTask* sdesc = reinterpret_cast<TriTask*>(buf + (size_t)kRingB);
  double* sold = reinterpret_cast<double*>(sdesc + 2 * kMaxCtaTasks);  // fold targets' values
  uint64_t* bars = reinterpret_cast<uint64_t*>(sold + kMaxCtaTasks);  // full[kNBuf], empty[kNBuf], dfull[2], dempty[2]
  uint64_t* dfull = bars + 2 * kNBuf;
  uint64_t* dempty = dfull + 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x, G = A.G;
  if (threadIdx.x == 0) {
    for (int q = 0; q < 2 * kNBuf + 4; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + q)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // per step (double-buffered, loaded one step ahead -- none of it depends on
  // the barrier): task and batch descriptors, the batch of each task, the step record
  __shared__ TriBatch sbat[2][kMaxCtaBatches];
  __shared__ unsigned sdone[2][kMaxCtaBatches];  // tasks of each batch finished
  __shared__ uint8_t sbidx[2][kMaxCtaTasks];     // batch of each task
  __shared__ TriStepD sstep[2];
  __shared__ int64_t sinfo[2][2];  // task count, batch count
  // batches released so far per ring slot: a warp may wait on batch g (slot
  // g % kNBuf, round g / kNBuf) only once every earlier round of that slot was
  // released -- the parity wait cannot tell round r from round r - 2
  __shared__ unsigned sgen[kNBuf];
  if (threadIdx.x < kNBuf) sgen[threadIdx.x] = 0;
  auto load_desc = [&](int64_t st, int ct, int nthr) {
    const int d = (int)(st & 1);
    const int64_t t0 = A.ctask[st * (G + 1) + c], t1 = A.ctask[st * (G + 1) + c + 1];
    const int64_t b0 = A.bptr[st * G + c], b1 = A.bptr[st * G + c + 1];
    for (int64_t i = ct; i < t1 - t0; i += nthr) sdesc[d * kMaxCtaTasks + i] = a.tasks[t0 + i];
    for (int64_t i = ct; i < b1 - b0; i += nthr) {
      const TriBatch B = A.batches[b0 + i];
      sbat[d][i] = B;
      sdone[d][i] = 0;
      for (int64_t t = B.t0; t < B.t1; ++t) sbidx[d][t - t0] = (uint8_t)i;
    }
    if (ct == 0) {
      sstep[d] = a.steps[st];
      sinfo[d][0] = t1 - t0;
      sinfo[d][1] = b1 - b0;
    }
  };
  __shared__ uint32_t s_tmem;
  __shared__ long long s_issued;  // (HCAMG_TRI_DBG=4) batches the producer has issued
  if (threadIdx.x == 0) s_issued = 0;
  const bool use_tmem = A.tmem && kCons == 16;
  if (use_tmem && warp == 1) {  // 512 columns = one 2048-column row per consumer warp (4 per lane quadrant)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0) {  // producer: the warp loads 32 batch descriptors at a time, lane 0 issues
    // the CTA's batches in order are cbat[cptr[c] .. cptr[c+1]); batch i + pfd is
    // prefetched into L2 when batch i enters the ring (a second lookahead level
    // behind the 168 KB ring, across steps and barriers)
    int64_t nb = 0;
    const char* pool = reinterpret_cast<const char*>(a.pool);
    const int64_t i0 = A.cptr[c], i1 = A.cptr[c + 1];
    const int pfd = A.pfd;
    for (int64_t qb = i0; qb < i1; qb += 32) {
      TriBatch Bl{}, Bp{};
      if (qb + lane < i1) Bl = A.cbat[qb + lane];
      if (pfd > 0 && qb + lane + pfd < i1) Bp = A.cbat[qb + lane + pfd];
      const int nl = (int)std::min<int64_t>(32, i1 - qb);
      for (int l = 0; l < nl; ++l, ++nb) {
        const int64_t off = __shfl_sync(0xffffffffu, Bl.off, l), bytes = __shfl_sync(0xffffffffu, Bl.bytes, l);
        const int64_t poff = __shfl_sync(0xffffffffu, Bp.off, l), pbytes = __shfl_sync(0xffffffffu, Bp.bytes, l);
        if (lane == 0) {
          if (pbytes > 0) prefetch_l2(pool + poff, (unsigned)pbytes);
          const int s = (int)(nb % kNBuf);
          const uint32_t r = (uint32_t)(nb / kNBuf);
          const unsigned long long w0 = A.trace ? gtime() : 0;
          mbar_wait(smem_u32(bars + kNBuf + s), (r & 1) ^ 1);
          if (A.trace) A.trace[c * 8 + 5] += gtime() - w0;
          const uint32_t full = smem_u32(bars + s);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full), "r"((uint32_t)bytes)
                       : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           smem_u32(buf + (size_t)s * kBufB)),
                       "l"(pool + off), "r"((uint32_t)bytes), "r"(full)
                       : "memory");
          if (A.tlb) *reinterpret_cast<volatile long long*>(&s_issued) = nb + 1;
        }
        __syncwarp();
      }
    }
    return;
  }
  if (warp == 1 + kCons) {  // descriptor loader: step st into buffer st & 1, one step ahead of the consumers
    for (int64_t st = 0; st < a.nstep; ++st) {
      const int d = (int)(st & 1);
      const uint32_t r = (uint32_t)(st >> 1);
      mbar_wait(smem_u32(dempty + d), (r & 1) ^ 1);
      load_desc(st, lane, 32);
      __syncwarp();

      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(dfull + d)) : "memory");
    }
    return;
  }
  const int cw = warp - 1, ct = threadIdx.x - 32;
  unsigned old = 0;
  int64_t nb = 0;
  // this warp's TMEM columns: lane quadrant warp % 4, 128 columns (32 chunks) each
  const uint32_t tb = use_tmem ? s_tmem + ((uint32_t)(32 * (warp % 4)) << 16) + 128u * (uint32_t)(cw / 4) : 0u;
  bool staged = false;  // the warp's first row of this step is already in TMEM (and counted for its batch)
  // per step: task descriptors, batch descriptors and the step record in shared memory,
  // loaded before the grid barrier (none of them depends on it)
  unsigned long long tp = A.trace ? gtime() : 0;
  auto mark = [&](int k) {
    if (A.trace && ct == 0) {
      const unsigned long long n = gtime();
      A.trace[c * 8 + k] += n - tp;
      tp = n;
    }
  };
  for (int64_t st = 0; st < a.nstep; ++st) {
    const int d = (int)(st & 1);
    mbar_wait(smem_u32(dfull + d), (uint32_t)((st >> 1) & 1));  // this step's descriptors in place
    mark(0);
    const TriStepD S = sstep[d];
    const int64_t nt = sinfo[d][0], nbat = sinfo[d][1];
    const TriTask* desc = sdesc + d * kMaxCtaTasks;
    {  // u_k, y_c and the fold targets' values: every load issued before any is used (one L2 round trip)
      constexpr int kPer = (kNB + 32 * kCons - 1) / (32 * kCons);
      const bool hv = ct < nt && desc[ct].b < 0;
      const double ov = hv ? __ldcg(a.u + desc[ct].out) : 0.0;
      double uu[kPer], yy[kPer];
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int t = ct + q * 32 * kCons;
        uu[q] = t < kNB ? __ldcg(a.u + (int64_t)S.k * kNB + t) : 0.0;
        yy[q] = t < kNB && S.c >= 0 ? __ldcg(a.y + (int64_t)S.c * kNB + t) : 0.0;
      }
      if (hv) sold[ct] = ov;
      for (int64_t i = ct + 32 * kCons; i < nt; i += 32 * kCons)
        if (desc[i].b < 0) sold[i] = __ldcg(a.u + desc[i].out);
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int t = ct + q * 32 * kCons;
        if (t < kNB) {
          su[t] = uu[q];
          sy[t] = yy[q];
        }
      }
    }
    cons_sync<kCons>();
    mark(1);
    // each warp takes the step's tasks round-robin and waits only for the batch
    // holding its task; the last task finished in a batch frees its buffer
    for (int64_t i = cw; i < nt; i += kCons) {
      if (staged && i == cw) {  // staged across the barrier: operator row from TMEM
        const TriTask& T = desc[i];
        const int na = T.ja1 - T.ja0;
        double r;
        if (T.b < 0) r = tmem_dot(tb, sy + 64 * T.ja0, na, lane);
        else r = tmem_dot(tb, su + 64 * T.ja0, na, lane) - tmem_dot(tb + 4 * na, sy + 64 * T.jb0, T.jb1 - T.jb0, lane);
        __syncwarp();
        if (lane == 0) {
          if (T.b < 0) a.u[T.out] = sold[i] - r;
          else a.y[T.out] = r;
        }
        continue;
      }
      const int q = sbidx[d][i];
      const int64_t g = nb + q;  // global batch number of this CTA
      const int s = (int)(g % kNBuf);
      const unsigned rnd = (unsigned)(g / kNBuf);
      while (*reinterpret_cast<volatile unsigned*>(&sgen[s]) < rnd) __nanosleep(20);
      mbar_wait(smem_u32(bars + s), rnd & 1);
      const TriBatch& B = sbat[d][q];
      const unsigned char* bb = buf + (size_t)s * kBufB - B.off;  // pool byte offset -> buffer address
      const TriTask& T = desc[i];
      const double* ra = reinterpret_cast<const double*>(bb + 8 * (T.a + 64 * T.ja0));
      double r;
      if (T.b < 0) {
        r = a.dbg == 2 ? 0.0 : smem_dot(ra, sy + 64 * T.ja0, T.ja1 - T.ja0, lane);
      } else {
        const double* rb = reinterpret_cast<const double*>(bb + 8 * (T.b + 64 * T.jb0));
        r = smem_dot(ra, su + 64 * T.ja0, T.ja1 - T.ja0, lane) - smem_dot(rb, sy + 64 * T.jb0, T.jb1 - T.jb0, lane);
      }
      __syncwarp();
      if (lane == 0) {
        if (T.b < 0) a.u[T.out] = sold[i] - r;
        else a.y[T.out] = r;
        if (atomicAdd(&sdone[d][q], 1u) + 1 == (unsigned)(B.t1 - B.t0)) {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bars + kNBuf + s)) : "memory");
          atomicAdd(&sgen[s], 1u);
        }
      }
    }
    nb += nbat;
    mark(2);
    if (st + 1 == a.nstep) {
      if (A.tl) {
        cons_sync<kCons>();
        if (ct == 0) A.tl[(st * G + c) * 2] = gtime();
      }
      break;
    }
    cons_sync<kCons>();  // every row of the step written, its descriptors no longer read
    if (A.tl && ct == 0) A.tl[(st * G + c) * 2] = gtime();  // the CTA's step done
    if (A.tlb && ct == 0) A.tlb[(st * G + c) * 2] = *reinterpret_cast<volatile long long*>(&s_issued) - nb;
    if (ct == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(dempty + d)) : "memory");
    mark(3);
    if (ct == 0 && a.dbg != 1) {
      const unsigned inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
      asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(a.bar), "r"(inc) : "memory");
    }
    // between arrive and wait: copy this warp's first row of the next step from
    // the ring into TMEM when its batch is one of the first kNBuf (those arrive
    // without any release) -- fully staged batches free their slots, so the
    // producer streams further into the next step across the barrier
    staged = false;
    if (use_tmem) {
      const int64_t st1 = st + 1;
      const int d1 = (int)(st1 & 1);
      mbar_wait(smem_u32(dfull + d1), (uint32_t)((st1 >> 1) & 1));
      if (cw < sinfo[d1][0]) {
        const int q = sbidx[d1][cw];
        const TriTask& T = sdesc[d1 * kMaxCtaTasks + cw];
        const int na = T.ja1 - T.ja0, nbb = T.b < 0 ? 0 : T.jb1 - T.jb0;
        if (q < kNBuf && na + nbb <= 32) {
          const int64_t g = nb + q;
          const int sl = (int)(g % kNBuf);
          const unsigned rnd = (unsigned)(g / kNBuf);
          while (*reinterpret_cast<volatile unsigned*>(&sgen[sl]) < rnd) __nanosleep(20);
          mbar_wait(smem_u32(bars + sl), rnd & 1);
          const TriBatch& B = sbat[d1][q];
          const unsigned char* bb = buf + (size_t)sl * kBufB - B.off;
          const double2* ra = reinterpret_cast<const double2*>(bb + 8 * (T.a + 64 * T.ja0)) + lane;
          for (int k = 0; k < na; ++k) tmem_st4(tb + 4 * k, ra[32 * k]);
          if (nbb) {
            const double2* rb = reinterpret_cast<const double2*>(bb + 8 * (T.b + 64 * T.jb0)) + lane;
            for (int k = 0; k < nbb; ++k) tmem_st4(tb + 4 * (na + k), rb[32 * k]);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          __syncwarp();
          if (lane == 0 && atomicAdd(&sdone[d1][q], 1u) + 1 == (unsigned)(B.t1 - B.t0)) {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bars + kNBuf + sl)) : "memory");
            atomicAdd(&sgen[sl], 1u);
          }
          staged = true;
        }
      }
    }
    if (ct == 0 && a.dbg != 1) {
      unsigned cur;
      if (A.barmode == 1) {  // relaxed polling, one acquire fence after
        do {
          asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(a.bar) : "memory");
        } while (((cur ^ old) & 0x80000000u) == 0);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      } else if (A.barmode == 2) {  // acquire polling with a short back-off
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(a.bar) : "memory");
          if (((cur ^ old) & 0x80000000u) == 0) __nanosleep(32);
        } while (((cur ^ old) & 0x80000000u) == 0);
      } else {
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(a.bar) : "memory");
        } while (((cur ^ old) & 0x80000000u) == 0);
      }
    }
    cons_sync<kCons>();  // every consumer past the grid barrier
    mark(4);
    if (A.tl && ct == 0) A.tl[(st * G + c) * 2 + 1] = gtime();
    if (A.tlb && ct == 0) A.tlb[(st * G + c) * 2 + 1] = *reinterpret_cast<volatile long long*>(&s_issued) - nb;
  }
  if (use_tmem) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cons_sync<kCons>();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem));
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
// kSub = true:  y[i] -= M[i,:] x.   kL lanes per row (32 / kL rows per warp:
// W' has a handful of entries per row), fixed order.
template <bool kSub, int kL = 32>
__global__ void k_fp_spmv(const int* stop, int64_t nrows, int64_t npad, const int64_t* __restrict__ mp,
                          const int32_t* __restrict__ mi, const double* __restrict__ mv, const double* __restrict__ x,
                          double* __restrict__ y) {
  if (*stop) return;
  const int lane = threadIdx.x & (kL - 1);
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / kL;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) / kL;
  for (int64_t i = w0; i < npad; i += nw) {
    double acc = 0.0;
    if (i < nrows)
      for (int64_t e = mp[i] + lane; e < mp[i + 1]; e += kL) acc = fma(mv[e], x[mi[e]], acc);
#pragma unroll
    for (int o = kL / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, kL);
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

void launch_sweep_kernel(const int* stop, const TriSweep& sw, double* u, double* y, unsigned* bar, cudaStream_t s,
                         unsigned long long* tl_out = nullptr) {
  auto env = [](const char* k, int d) {
    const char* v = getenv(k);
    return v ? atoi(v) : d;
  };
  // measurement knobs: HCAMG_TRI_KERNEL (1 dataflow, 0 grid-barrier steps),
  // HCAMG_TRI_PFMODE / HCAMG_TRI_PF (L2 prefetch placement), HCAMG_TRI_DBG
  TriArgs a{stop, sw.nstep, sw.steps.p, sw.tasks.p, sw.pool.p, u, y, bar, std::max(1, env("HCAMG_TRI_PF", 1)),
            env("HCAMG_TRI_PFMODE", 2), env("HCAMG_TRI_DBG", 0)};
  const int kern = env("HCAMG_TRI_KERNEL", 2);
  if (kern == 2 && !(sw.max_cta_tasks <= kMaxCtaTasks && sw.max_cta_batches <= kMaxCtaBatches)) {
    static bool warned = false;
    if (!warned)
      fprintf(stderr, "[hcamg] sweep partition exceeds the TMA kernel's per-CTA limits (%d tasks, %d batches); "
                      "using the grid-barrier sweep kernel\n", sw.max_cta_tasks, sw.max_cta_batches);
    warned = true;
  }
  if (kern == 2 && sw.G > 0 && sw.max_cta_tasks <= kMaxCtaTasks && sw.max_cta_batches <= kMaxCtaBatches &&
      (env("HCAMG_TRI_CONS", 16) != 12 || sw.nbuf == 4)) {
    const int cons = env("HCAMG_TRI_CONS", 16);
    static bool init = false;
    if (!init) {
      const int sm = (int)kTmaSmem;
      HC_CUDA(cudaFuncSetAttribute(k_tri_tma<12, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      HC_CUDA(cudaFuncSetAttribute(k_tri_tma<16, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      HC_CUDA(cudaFuncSetAttribute(k_tri_tma<16, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      HC_CUDA(cudaFuncSetAttribute(k_tri_tma<16, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      HC_CUDA(cudaFuncSetAttribute(k_tri_tma<16, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      HC_CUDA(cudaFuncSetAttribute(k_tri_tma<16, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      init = true;
    }
    static unsigned long long* trace = nullptr;
    if (a.dbg == 3 && !trace) {
      HC_CUDA(cudaMalloc(&trace, 8 * 8 * (size_t)sw.G));
      HC_CUDA(cudaMemset(trace, 0, 8 * 8 * (size_t)sw.G));
    }
    if (a.dbg != 3 && trace) {  // print and drop the accumulated phase times
      std::vector<unsigned long long> h((size_t)8 * sw.G);
      HC_CUDA(cudaMemcpy(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost));
      double m[6] = {0, 0, 0, 0, 0, 0}, mx[6] = {0, 0, 0, 0, 0, 0}, mn[6] = {1e30, 1e30, 1e30, 1e30, 1e30, 1e30};
      int amx = 0, amn = 0;
      for (int c = 0; c < sw.G; ++c)
        for (int k = 0; k < 6; ++k) {
          const double v = (double)h[(size_t)c * 8 + k];
          m[k] += v / sw.G;
          if (k == 2 && v > mx[k]) amx = c;
          if (k == 2 && v < mn[k]) amn = c;
          mx[k] = std::max(mx[k], v);
          mn[k] = std::min(mn[k], v);
        }
      fprintf(stderr, "[tri trace] tasks phase min %.3f (cta %d) max %.3f (cta %d); stage min %.3f max %.3f; out max %.3f\n",
              mn[2] / 1e6, amn, mx[2] / 1e6, amx, mn[1] / 1e6, mx[1] / 1e6, mx[3] / 1e6);
      fprintf(stderr, "[tri trace] tasks+out per CTA (ms):");
      for (int c = 0; c < sw.G; ++c) fprintf(stderr, " %.2f", (h[(size_t)c * 8 + 2] + h[(size_t)c * 8 + 3]) / 1e6);
      fprintf(stderr, "\n");
      fprintf(stderr, "[tri trace] per CTA (ms): top-wait %.3f stage %.3f tasks %.3f out %.3f barrier %.3f | producer empty-wait %.3f\n",
              m[0] / 1e6, m[1] / 1e6, m[2] / 1e6, m[3] / 1e6, m[4] / 1e6, m[5] / 1e6);
      cudaFree(trace);
      trace = nullptr;
    }
    TmaArgs A{a, a.dbg == 3 ? trace : nullptr, sw.ctask.p, sw.bptr.p, sw.batches.p, sw.cptr.p, sw.cbat.p, sw.G,
              env("HCAMG_TRI_L2PF", 1), env("HCAMG_TRI_BAR", 0), env("HCAMG_TRI_TMEM", 1), nullptr, nullptr};
    DBuf<unsigned long long> tl;
    DBuf<long long> tlb;
    if (tl_out) {
      A.tl = tl_out;
    } else if (a.dbg == 4) {  // timeline dump (not graph-capturable): HCAMG_TRI_DUMP.<n>.bin
      tl.alloc(2 * sw.nstep * sw.G, s);
      tl.zero();
      A.tl = tl.p;
      tlb.alloc(2 * sw.nstep * sw.G, s);
      tlb.zero();
      A.tlb = tlb.p;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)sw.G);
    cfg.blockDim = dim3(32 * (2 + (cons == 12 ? 12 : 16)));
    cfg.dynamicSmemBytes = kTmaSmem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cons == 12) HC_CUDA(cudaLaunchKernelEx(&cfg, k_tri_tma<12, 4>, A));
    else if (sw.nbuf == 6) HC_CUDA(cudaLaunchKernelEx(&cfg, k_tri_tma<16, 6>, A));
    else if (sw.nbuf == 8) HC_CUDA(cudaLaunchKernelEx(&cfg, k_tri_tma<16, 8>, A));
    else if (sw.nbuf == 2) HC_CUDA(cudaLaunchKernelEx(&cfg, k_tri_tma<16, 2>, A));
    else if (sw.nbuf == 3) HC_CUDA(cudaLaunchKernelEx(&cfg, k_tri_tma<16, 3>, A));
    else HC_CUDA(cudaLaunchKernelEx(&cfg, k_tri_tma<16, 4>, A));
    if (A.tl && !tl_out) {
      static int seq = 0;
      HC_CUDA(cudaStreamSynchronize(s));
      std::vector<unsigned long long> ht((size_t)tl.n);
      std::vector<int64_t> ct((size_t)sw.ctask.n), bp((size_t)sw.bptr.n);
      std::vector<TriBatch> bt((size_t)sw.batches.n);
      HC_CUDA(cudaMemcpy(ht.data(), tl.p, 8 * ht.size(), cudaMemcpyDeviceToHost));
      HC_CUDA(cudaMemcpy(ct.data(), sw.ctask.p, 8 * ct.size(), cudaMemcpyDeviceToHost));
      HC_CUDA(cudaMemcpy(bp.data(), sw.bptr.p, 8 * bp.size(), cudaMemcpyDeviceToHost));
      HC_CUDA(cudaMemcpy(bt.data(), sw.batches.p, sizeof(TriBatch) * bt.size(), cudaMemcpyDeviceToHost));
      const char* base = getenv("HCAMG_TRI_DUMP");
      const std::string fn = std::string(base ? base : "tri_timeline") + "." + std::to_string(seq++) + ".bin";
      std::vector<long long> hb((size_t)tlb.n);
      HC_CUDA(cudaMemcpy(hb.data(), tlb.p, 8 * hb.size(), cudaMemcpyDeviceToHost));
      if (FILE* fb = fopen((fn + ".bank").c_str(), "wb")) {  // per (step, cta): batches issued ahead at done, at pass
        fwrite(hb.data(), 8, hb.size(), fb);
        fclose(fb);
      }
      if (FILE* f = fopen(fn.c_str(), "wb")) {  // nstep, G, then per (step, cta): t_done, t_pass, tasks, bytes
        const int64_t hdr[2] = {sw.nstep, sw.G};
        fwrite(hdr, 8, 2, f);
        for (int64_t st = 0; st < sw.nstep; ++st)
          for (int c = 0; c < sw.G; ++c) {
            int64_t by = 0;
            for (int64_t q = bp[(size_t)(st * sw.G + c)]; q < bp[(size_t)(st * sw.G + c + 1)]; ++q) by += bt[(size_t)q].bytes;
            const int64_t rec[4] = {(int64_t)ht[(size_t)(st * sw.G + c) * 2], (int64_t)ht[(size_t)(st * sw.G + c) * 2 + 1],
                                    ct[(size_t)(st * (sw.G + 1) + c + 1)] - ct[(size_t)(st * (sw.G + 1) + c)], by};
            fwrite(rec, 8, 4, f);
          }
        fclose(f);
      }
    }
    return;
  }
  if (kern == 1) {
    HC_CUDA(cudaMemsetAsync(sw.flags.p, 0, sizeof(unsigned) * (size_t)sw.flags.n, s));
    FlowArgs F{a, sw.ntask, sw.nfold.p, sw.flags.p, sw.flags.p + sw.nstep, sw.flags.p + sw.nstep + sw.T};
    static int blocks = 0;
    if (!blocks) {
      int per_sm = 0, dev = 0, sms = kSMs;
      HC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tri_flow, 512, 0));
      HC_CUDA(cudaGetDevice(&dev));
      HC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      blocks = sms * std::max(1, per_sm);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(512);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;  // co-residency: every warp must run to guarantee progress
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    HC_CUDA(cudaLaunchKernelEx(&cfg, k_tri_flow, F));
    return;
  }
  launch_sweep_t<512, 8>(a, s);
}

}  // namespace

// Contiguous CTA partition of every step's tasks and their batches (<= one
// ring slot) for the TMA kernel.  A task weighs its bytes (critical rows
// scaled by critpct %) + taskw; CTA c's share of a step's weight is 1/G, or
// share[k G + c] after calibration (tri_calibrate).  A step whose cut exceeds
// the kernel's per-CTA limits (the last CTA takes the remainder) is re-cut with
// a heavier per-row weight, which spreads the many short fold rows.
void tri_partition(TriSweep& out, cudaStream_t s) {
  const std::vector<TriTask>& tasks = out.htasks;
  const int G = out.G;
  const int64_t slotb = (kRingB / out.nbuf) & ~int64_t(511);
  auto tbytes = [&](int64_t t) {
    const TriTask& x = tasks[(size_t)t];
    return 512 * (int64_t)(x.ja1 - x.ja0 + (x.b < 0 ? 0 : x.jb1 - x.jb0));
  };
  int64_t taskw = out.taskw;
  auto tcost = [&](int64_t t) {
    const int64_t b = tbytes(t);
    return (tasks[(size_t)t].b < 0 ? b : b * out.critpct / 100) + taskw;
  };
  auto tstart = [&](int64_t t) { return 8 * (tasks[(size_t)t].a + 64 * tasks[(size_t)t].ja0); };
  std::vector<int64_t> ct, bptr(1, 0);
  std::vector<TriBatch> batches;
  out.hcost.assign(out.hsteps.size() * (size_t)G, 0.0);
  int maxt = 0, maxb = 0;
  for (size_t k = 0; k < out.hsteps.size(); ++k) {
    const TriStepD& d = out.hsteps[k];
    const bool calib = !out.share.empty();
    std::vector<int64_t> sct, sbn;
    std::vector<TriBatch> sbat;
    std::vector<double> scost;
    for (int attempt = 0;; ++attempt) {
      sct.clear();
      sbat.clear();
      sbn.clear();
      scost.clear();
      int st_maxt = 0, st_maxb = 0;
      int64_t total = 0;
      for (int64_t t = d.t0; t < d.t1; ++t) total += tcost(t);
      int64_t acc = 0, t = d.t0;
      double cum = 0.0;
      for (int c = 0; c < G; ++c) {
        sct.push_back(t);
        cum += calib ? out.share[k * G + c] : 1.0 / G;
        const int64_t target = c + 1 == G ? INT64_MAX : (int64_t)((double)total * std::min(1.0, cum));
        const int64_t c0 = t, a0 = acc;
        while (t < d.t1 && (c + 1 == G || (t - c0 < kMaxCtaTasks && acc + tcost(t) / 2 <= target))) acc += tcost(t++);
        scost.push_back((double)(acc - a0));
        st_maxt = std::max<int>(st_maxt, (int)(t - c0));
        const size_t nb0 = sbat.size();
        for (int64_t b0 = c0; b0 < t;) {
          int64_t b1 = b0, bytes = 0;
          while (b1 < t && bytes + tbytes(b1) <= slotb) bytes += tbytes(b1++);
          // a single row larger than a ring slot can never be staged
          require(b1 > b0, "sweep ring slot (" + std::to_string(slotb) + " B) smaller than one factor row (" +
                               std::to_string(tbytes(b0)) + " B): use fewer ring slots");
          sbat.push_back(TriBatch{b0, b1, tstart(b0), bytes});
          b0 = b1;
        }
        st_maxb = std::max<int>(st_maxb, (int)(sbat.size() - nb0));
        sbn.push_back((int64_t)sbat.size());
      }
      const bool fits = st_maxt <= kMaxCtaTasks && st_maxb <= kMaxCtaBatches;
      if (fits || attempt == 40) {
        maxt = std::max(maxt, st_maxt);
        maxb = std::max(maxb, st_maxb);
        break;
      }
      taskw = taskw * 5 / 4 + 256;
    }
    // each CTA's weight under the base model (what the calibration rescales)
    taskw = out.taskw;
    for (int c = 0; c < G; ++c) {
      const int64_t e = c + 1 < G ? sct[(size_t)c + 1] : d.t1;
      double w = 0.0;
      for (int64_t t = sct[(size_t)c]; t < e; ++t) w += (double)tcost(t);
      out.hcost[k * G + c] = w;
    }
    const int64_t nb0 = (int64_t)batches.size();
    for (int64_t x : sct) ct.push_back(x);
    ct.push_back(d.t1);
    for (const TriBatch& b : sbat) batches.push_back(b);
    for (int64_t x : sbn) bptr.push_back(nb0 + x);
  }
  std::vector<int64_t> cptr(1, 0);
  std::vector<TriBatch> cbat;
  for (int c = 0; c < G; ++c) {
    for (size_t k = 0; k < out.hsteps.size(); ++k)
      for (int64_t q = bptr[k * G + c]; q < bptr[k * G + c + 1]; ++q) cbat.push_back(batches[(size_t)q]);
    cptr.push_back((int64_t)cbat.size());
  }
  out.cptr.upload(cptr.data(), (int64_t)cptr.size(), s);
  if (cbat.empty()) cbat.push_back(TriBatch{});
  out.cbat.upload(cbat.data(), (int64_t)cbat.size(), s);
  out.max_cta_tasks = maxt;
  out.max_cta_batches = maxb;
  out.ctask.upload(ct.data(), (int64_t)ct.size(), s);
  out.bptr.upload(bptr.data(), (int64_t)bptr.size(), s);
  if (batches.empty()) batches.push_back(TriBatch{});
  out.batches.upload(batches.data(), (int64_t)batches.size(), s);
}

void tri_compact(const std::vector<TriSrcStep>& src, const std::function<const uint8_t*(const double*)>& ranges,
                 TriSweep& out, cudaStream_t s, int dir) {
  std::vector<TriStepD> steps;
  std::vector<TriTask> tasks;
  std::vector<CopyJob> jobs;
  int64_t T = 0;
  for (const TriSrcStep& S : src) {
    T = std::max<int64_t>(T, S.k + 1);
    for (const auto& fo : S.folds) T = std::max<int64_t>(T, fo.second + 1);
  }
  std::vector<int32_t> fseq((size_t)(T * kNB), 0);  // folds so far into each row
  int64_t off = 64 * 16;  // pool offset (doubles); the 8 KB pad keeps every row base (off - 64 j0) >= 0
  // rgt: the block's range table (looked up once per block, not per row)
  auto place = [&](const TriSrc& src, const uint8_t* rgt, int r, uint8_t& j0, uint8_t& j1) -> int64_t {
    const uint8_t* rg = rgt + 2 * r;
    j0 = rg[0];
    j1 = rg[1];
    if (j0 >= j1) {
      j0 = j1 = 0;
      return 0;
    }
    const int32_t n = 64 * (j1 - j0);
    jobs.push_back(CopyJob{src.p + (int64_t)r * src.ld + 64 * j0, off, n, 0});
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
    const uint8_t* rga = ranges(S.a.p);
    const uint8_t* rgb = S.b.p ? ranges(S.b.p) : nullptr;
    for (int r = 0; r < kNB; ++r) {
      TriTask t{};
      t.out = (int32_t)((int64_t)S.k * kNB + r);
      t.a = place(S.a, rga, r, t.ja0, t.ja1);
      t.b = S.b.p ? place(S.b, rgb, r, t.jb0, t.jb1) : 0;
      tasks.push_back(t);
    }
    for (const auto& fo : S.folds) {
      const uint8_t* rgf = ranges(fo.first.p);
      for (int r = 0; r < kNB; ++r) {
        TriTask t{};
        t.a = place(fo.first, rgf, r, t.ja0, t.ja1);
        if (t.ja0 >= t.ja1) continue;  // an all-zero fold row changes nothing
        t.b = -1 - fseq[(size_t)(fo.second * kNB + r)]++;
        t.out = (int32_t)(fo.second * kNB + r);
        tasks.push_back(t);
      }
    }
    d.t1 = (int64_t)tasks.size();
    d.pf1 = 8 * off;
    steps.push_back(d);
  }
  {  // dataflow counters
    std::vector<int32_t> nf((size_t)T, 0);
    for (const TriTask& t : tasks)
      if (t.b < 0) ++nf[(size_t)(t.out / kNB)];
    out.nfold.upload(nf.data(), T, s);
    out.flags.alloc((int64_t)steps.size() + T + T * kNB, s);
  }
  {  // CTA partition and batches for the TMA kernel (tri_partition)
    // (HCAMG_TRI_TASKW / HCAMG_TRI_CRITW, and *_BW for the backward sweep: measurement knobs)
    auto knob = [&](const char* k, int64_t d) {
      const std::string kb = std::string(k) + "_BW";
      const char* v = dir == 1 && getenv(kb.c_str()) ? getenv(kb.c_str()) : getenv(k);
      return v ? atoll(v) : d;
    };
    out.taskw = knob("HCAMG_TRI_TASKW", 3072);
    out.critpct = knob("HCAMG_TRI_CRITW", 140);
    // ring slots (measured on config 2: 1024-row steps best with 3, 2048-row steps with 2)
    const int nbuf = getenv("HCAMG_TRI_SLOTS") ? atoi(getenv("HCAMG_TRI_SLOTS")) : (kNB >= 2048 ? 2 : 3);
    require(nbuf >= 2 && nbuf <= 8 && nbuf != 5 && nbuf != 7, "HCAMG_TRI_SLOTS must be 2, 3, 4, 6 or 8");
    out.nbuf = nbuf;
    int dev = 0, sms = kSMs;
    HC_CUDA(cudaGetDevice(&dev));
    HC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    out.G = sms;
    out.htasks = tasks;
    out.hsteps = steps;
    out.share.clear();
    tri_partition(out, s);
    if (getenv("HCAMG_SETUP_TIMING"))
      fprintf(stderr, "[hcamg setup]   sweep: %zu steps, %zu tasks, max %d tasks / %d batches per CTA step\n",
              steps.size(), tasks.size(), out.max_cta_tasks, out.max_cta_batches);
  }
  out.T = T;
  out.ntask = (int64_t)tasks.size();
  out.nstep = (int64_t)steps.size();
  out.bytes = 8 * (off - 64 * 16);
  out.pool.alloc(std::max<int64_t>(off, 2), s);
  out.steps.upload(steps.data(), out.nstep, s);
  out.tasks.upload(tasks.data(), (int64_t)tasks.size(), s);
  DBuf<CopyJob> dj;
  dj.upload(jobs.data(), (int64_t)jobs.size(), s);
  if (!jobs.empty()) k_compact_copy<<<grid_for((int64_t)jobs.size() * 32, 256), 256, 0, s>>>(dj.p, (int64_t)jobs.size(), out.pool.p);
  HC_CHECK_LAUNCH();
  HC_CUDA(cudaStreamSynchronize(s));
}

// Calibrate the TMA sweep's CTA partition on the device.  A step ends when its
// slowest CTA arrives at the grid barrier, and which CTA that is depends less on
// its bytes than on how much it could stream ahead during the previous barrier
// -- a pattern that repeats run to run (per-(step, CTA) work correlates 0.99
// between runs).  Each round times every (step, CTA) (one launch with the
// timeline stamps) and moves weight from the slow CTAs of a step to the fast
// ones (share *= (mean / own work)^0.8, damped); the best of the rounds is
// kept.  Only the assignment of rows to CTAs changes, never a row's dot
// order, so results are bit-identical whatever the partition.
// HCAMG_TRI_CALIB = rounds (0: off).
void tri_calibrate(TriSweep& sw, double* u, double* y, unsigned* bar, int rounds, cudaStream_t s) {
  if (rounds <= 0 || sw.nstep < 3 || !tri_tma_fits(sw) || sw.htasks.empty()) return;
  const char* ke = getenv("HCAMG_TRI_KERNEL");
  if (ke && atoi(ke) != 2) return;
  const int G = sw.G;
  const int64_t K = sw.nstep;
  DBuf<int> stop(1, s);
  stop.zero();
  DBuf<unsigned long long> tl(2 * K * G, s);
  std::vector<unsigned long long> h((size_t)(2 * K * G));
  std::vector<double> best_share = sw.share;
  double best = 1e300;
  const double alpha = getenv("HCAMG_TRI_CALIB_ALPHA") ? atof(getenv("HCAMG_TRI_CALIB_ALPHA")) : 0.8;
  for (int r = 0; r <= rounds; ++r) {
    if (!tri_tma_fits(sw)) break;
    for (int rep = 0; rep < 2; ++rep) {
      tl.zero();
      launch_sweep_kernel(stop.p, sw, u, y, bar, s, tl.p);
    }
    HC_CUDA(cudaStreamSynchronize(s));
    HC_CUDA(cudaMemcpy(h.data(), tl.p, 8 * h.size(), cudaMemcpyDeviceToHost));
    auto done = [&](int64_t k, int c) { return (double)h[(size_t)(k * G + c) * 2]; };
    auto pass = [&](int64_t k, int c) { return (double)h[(size_t)(k * G + c) * 2 + 1]; };
    double t0 = 1e300, t1 = 0;
    for (int c = 0; c < G; ++c) {
      t0 = std::min(t0, pass(0, c));
      t1 = std::max(t1, done(K - 1, c));
    }
    const double span = t1 - t0;
    if (getenv("HCAMG_SETUP_TIMING"))
      fprintf(stderr, "[hcamg setup]   sweep calibration round %d: %.1f us for steps 1..%lld\n", r, span / 1e3,
              (long long)(K - 1));
    if (span < best) {
      best = span;
      best_share = sw.share;
    }
    if (r == rounds) break;
    std::vector<double> ns((size_t)(K * G));
    for (int64_t k = 0; k < K; ++k) {
      double tot = 0.0;
      for (int c = 0; c < G; ++c) tot += sw.hcost[(size_t)(k * G + c)];
      std::vector<double> w((size_t)G);
      double wbar = 0.0;
      for (int c = 0; c < G; ++c) {
        w[(size_t)c] = k == 0 ? 1.0 : std::max(1.0, done(k, c) - pass(k - 1, c));
        wbar += w[(size_t)c] / G;
      }
      double sum = 0.0;
      for (int c = 0; c < G; ++c) {
        const double base = std::max(sw.hcost[(size_t)(k * G + c)] / std::max(tot, 1.0), 1e-4 / G);
        ns[(size_t)(k * G + c)] = base * std::pow(wbar / w[(size_t)c], alpha);
        sum += ns[(size_t)(k * G + c)];
      }
      for (int c = 0; c < G; ++c) ns[(size_t)(k * G + c)] /= sum;
    }
    sw.share = ns;
    tri_partition(sw, s);
  }
  if (best_share != sw.share) {
    sw.share = best_share;
    tri_partition(sw, s);
  }
  HC_CUDA(cudaStreamSynchronize(s));
}

bool tri_tma_fits(const TriSweep& sw) {
  return sw.G > 0 && sw.max_cta_tasks <= kMaxCtaTasks && sw.max_cta_batches <= kMaxCtaBatches;
}

int64_t factorp_npad(const FactorP& f) { return (f.T * kTriNB + kTriSB - 1) / kTriSB * kTriSB; }

bool factorp_enabled() { return opts().factor_apply != 0; }

void factorp_attach(FactorP& f, const DCsr& W, const int32_t* mpos, const int32_t* rows, cudaStream_t s) {
  const int64_t nG = f.nG;
  f.nc = W.ncols;
  DBuf<int32_t> sel(nG, s);
  f.dof.alloc(nG, s);
  k_fp_rowsel<<<grid_for(nG, 256), 256, 0, s>>>(nG, f.perm.p, mpos, rows, sel.p, f.dof.p);
  HC_CHECK_LAUNCH();
  csr_extract(W, sel.p, nG, nullptr, W.ncols, f.Wp, s);
  csr_transpose(f.Wp, f.Wpt, s);
  const int64_t npad = factorp_npad(f);
  f.v0.alloc(npad, s);
  f.v1.alloc(npad, s);
  f.v2.alloc(npad, s);
  f.v0.zero();
  f.v1.zero();
  f.v2.zero();
  f.bar.alloc(1, s);
  f.bar.zero();
  const int rounds = opts().tri_calib;
  tri_calibrate(f.fw, f.v0.p, f.v1.p, f.bar.p, rounds, s);
  tri_calibrate(f.bw, f.v1.p, f.v2.p, f.bar.p, rounds, s);
  f.v0.zero();
  f.v1.zero();
  f.v2.zero();
  f.on = true;
}

void factorp_solve(const int* stop, FactorP& f, double* v, double* y, cudaStream_t s) {
  launch_sweep_kernel(stop, f.fw, v, f.v1.p, f.bar.p, s);
  launch_sweep_kernel(stop, f.bw, f.v1.p, y, f.bar.p, s);
}

void factorp_restrict(const int* stop, FactorP& f, const double* r, double* bc, cudaStream_t s) {
  const int64_t npad = factorp_npad(f);
  k_fp_gather<<<grid_for(npad, 256), 256, 0, s>>>(stop, f.nG, npad, f.dof.p, r, f.v0.p);
  HC_CHECK_LAUNCH();
  factorp_solve(stop, f, f.v0.p, f.v2.p, s);
  k_fp_spmv<true><<<grid_for(f.nc * 32, 256), 256, 0, s>>>(stop, f.nc, f.nc, f.Wpt.ptr.p, f.Wpt.idx.p, f.Wpt.val.p,
                                                           f.v2.p, bc);
  HC_CHECK_LAUNCH();
}

void factorp_prolong(const int* stop, FactorP& f, const double* e, double* x, cudaStream_t s) {
  const int64_t npad = factorp_npad(f);
  k_fp_spmv<false, 8><<<grid_for(npad * 8, 256), 256, 0, s>>>(stop, f.nG, npad, f.Wp.ptr.p, f.Wp.idx.p, f.Wp.val.p, e,
                                                            f.v0.p);
  HC_CHECK_LAUNCH();
  factorp_solve(stop, f, f.v0.p, f.v2.p, s);
  k_fp_scatter_sub<<<grid_for(f.nG, 256), 256, 0, s>>>(stop, f.nG, f.dof.p, f.v2.p, x);
  HC_CHECK_LAUNCH();
}

}  // namespace hcamg
