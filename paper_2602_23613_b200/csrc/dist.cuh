// Row-partitioned solve across GPUs (one process per GPU, NVLink peer memory).
//
// The setup is replicated on every rank (the greedy splittings are global
// sequential greedies).  In the solve, every rank streams only
// its share of the bytes that dominate a V-cycle -- the rows of the dense
// interpolation block Z of each dense-regime level and the rows of the
// coarsest inverse -- and the results are exchanged through a symmetric
// buffer that every rank maps (CUDA IPC): the producing kernel stores its
// slice straight into every peer's buffer and its last CTA raises a flag
// there; the consuming kernel waits for all flags.  Everything else (smoother,
// sparse transfer parts, PCG vectors) is computed redundantly and bit-
// identically on every rank, so no other exchange is needed.
//
// The restriction sums the row-chunk partials of Z^T r in kGroups fixed groups
// (groups own whole chunks; ranks own whole groups), so the result is
// bit-identical for every rank count and to the single-GPU path.
#pragma once
#include <cstdint>

#include "common.cuh"

namespace hcamg {

constexpr int kMaxRanks = 8;
constexpr int kGroups = 8;
constexpr size_t kFlagBytes = 256;  // flags[kMaxRanks] (u64) at the start of every symmetric buffer

// Everything a producing / consuming kernel needs, passed by value.
struct Xchg {
  char* base[kMaxRanks];       // each rank's symmetric buffer, as mapped in this process
  int rank, nranks;
  size_t area_bytes;           // one parity area (double-buffered by epoch parity)
  size_t off;                  // byte offset of this exchange site inside an area
  unsigned long long* ep;      // this rank's exchange epoch (device)
  unsigned* cta;               // last-CTA counter (device)
  int* err;                    // set when a wait times out
};

struct Dist {
  int rank = 0, nranks = 1;
  bool on = false;
  char* sym = nullptr;         // cudaMalloc'd (IPC-exportable)
  size_t sym_bytes = 0, area_bytes = 0;
  char* base[kMaxRanks] = {};
  bool opened[kMaxRanks] = {};
  DBuf<unsigned long long> ep;
  DBuf<unsigned> cta;
  DBuf<int> err;
  Xchg site(size_t off) const;
  void release();
  ~Dist() { release(); }
};

// rows [r0, r1) of an n-row block owned by `rank` of `nranks` (contiguous, balanced)
inline void even_rows(int64_t n, int rank, int nranks, int64_t& r0, int64_t& r1) {
  r0 = n * rank / nranks;
  r1 = n * (rank + 1) / nranks;
}
// groups [g0, g1) owned by `rank`
inline void rank_groups(int rank, int nranks, int& g0, int& g1) {
  g0 = kGroups * rank / nranks;
  g1 = kGroups * (rank + 1) / nranks;
}

// ---- device side of the protocol
//
// Epochs: the producer's CTAs read e = *ep at start and store into parity
// area (e+1)&1; its last CTA publishes *ep = e+1 and raises flag[rank] = e+1
// in every rank's buffer.  The consumer (next kernel on the stream) reads
// *ep (= e+1) and waits until every flag reaches it.  A peer can only reuse
// a parity area after passing the next exchange, which needs this rank's
// signal, which comes after this rank's consumer -- so two areas suffice.

__device__ __forceinline__ double* xarea(const Xchg& x, int r, unsigned long long e) {
  return reinterpret_cast<double*>(x.base[r] + kFlagBytes + (e & 1ull) * x.area_bytes + x.off);
}

__device__ __forceinline__ unsigned long long xepoch(const Xchg& x) {
  return *reinterpret_cast<volatile unsigned long long*>(x.ep);
}

// called by every thread of every CTA of the producing kernel, at its end
__device__ __forceinline__ void xsignal(const Xchg& x, unsigned long long e) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned total = gridDim.x * gridDim.y * gridDim.z;
    if (atomicAdd(x.cta, 1u) == total - 1) {
      __threadfence_system();
      *x.cta = 0u;
      *x.ep = e + 1;
      for (int r = 0; r < x.nranks; ++r) {
        unsigned long long* f = reinterpret_cast<unsigned long long*>(x.base[r]) + x.rank;
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(e + 1) : "memory");
      }
    }
  }
}

// called by every thread of every CTA of the consuming kernel, at its start;
// returns the epoch to read.  Waits at most ~60 s, then flags *err (the solve
// continues on stale data and the host reports the error).
__device__ __forceinline__ unsigned long long xwait(const Xchg& x) {
  __shared__ unsigned long long e_sh;
  if (threadIdx.x == 0) {
    const unsigned long long e = xepoch(x);
    if (*reinterpret_cast<volatile int*>(x.err) == 0) {
      unsigned long long t0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      const unsigned long long* flags = reinterpret_cast<const unsigned long long*>(x.base[x.rank]);
      for (int r = 0; r < x.nranks; ++r) {
        for (unsigned it = 0;; ++it) {
          unsigned long long v;
          asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + r) : "memory");
          if (v >= e) break;
          if ((it & 1023u) == 1023u) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > 60ull * 1000000000ull) {
              atomicExch(x.err, 1);
              r = x.nranks;
              break;
            }
          }
        }
      }
    }
    e_sh = e;
  }
  __syncthreads();
  return e_sh;
}

// ---- kernels (dist.cu)

// partial[ch] (chunks of the rank's groups) -> group sums, stored into every
// rank's area at site x (kGroups x nc doubles), then signal.
void xchg_group_sums(const int* stop, const Xchg& x, int64_t nc, const double* partial, const int64_t* grp_host,
                     int g0, int g1, cudaStream_t s);
// wait; bc[c] -= sum_g gsum[g][c]
void xchg_group_final(const int* stop, const Xchg& x, int64_t nc, double* bc, cudaStream_t s);
// wait; x[rows[q]] -= y[q]   (rows == nullptr: x[q] = y[q])
void xchg_scatter(const int* stop, const Xchg& x, int64_t n, const int32_t* rows, double* out, cudaStream_t s);
// same-stream signal from a kernel that stored its slice already (used by the
// row GEMV producer, which signals from its own last CTA)

}  // namespace hcamg
