// Coarsest solve x = A_c^{-1} b with the explicit inverse stored once: the
// lower triangle of the symmetric inverse, read ONCE per application (config
// 2: 2.76 GB instead of the 5.5 GB of the full matrix; the coarsest solve is
// a pure HBM stream, so the bytes are the time).
//
// Layout: 32 x 32 sub-tiles (row-major, 8 KB, one coalesced 256-byte row per
// warp load), grouped into items of 4 x 4 sub-tiles (128 rows x 128 columns)
// over the lower triangle, items back to back in row-major order; a diagonal
// item holds only its 10 lower sub-tiles, and a diagonal sub-tile is stored
// full (both halves of the symmetric 32 x 32 block).
//
// One warp per item (static round-robin).  Lane l owns column l of every
// sub-tile: for sub-tile (i, j) it loads rows k = 0..31 of column l and
//   * accumulates p[k] += v[k] b_j[l]        (row sums, across the item's columns)
//   * accumulates c[j] += v[k] b_i[k]        (transposed product, j < i only)
// and after each sub-tile row reduces p with a 31-shuffle transpose-reduce so
// lane l holds row l's sum.  Items write 128 row and 128 column partials to
// fixed slots; a second kernel sums, for every row, its item row's row
// partials and its item column's column partials in fixed order: the result
// is bit-identical run to run.
#include <algorithm>
#include <vector>

#include "symv.cuh"

namespace hcamg {

namespace {

constexpr int kT = SymPacked::kTile, kB = SymPacked::kBlk, kR = SymPacked::kRows;
constexpr int kSymThreads = 256;

__device__ __forceinline__ int item_of(int bi, int bj) { return bi * (bi + 1) / 2 + bj; }

__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

__global__ void __launch_bounds__(kSymThreads) k_symv_items(const int* stop, int64_t n, int nb, int items,
                                                            const double* __restrict__ val,
                                                            const int64_t* __restrict__ ioff,
                                                            const double* __restrict__ b,
                                                            double* __restrict__ rowpart,
                                                            double* __restrict__ colpart) {
  if (*stop) return;
  const int lane = threadIdx.x & 31;
  const int nwarps = gridDim.x * (kSymThreads / 32);
  for (int q = blockIdx.x * (kSymThreads / 32) + (threadIdx.x >> 5); q < items; q += nwarps) {
    // item (bi, bj) from its row-major lower index
    int bi = (int)((sqrt(8.0 * q + 1.0) - 1.0) * 0.5);
    while (item_of(bi + 1, 0) <= q) ++bi;
    while (item_of(bi, 0) > q) --bi;
    const int bj = q - item_of(bi, 0);
    const bool diag = bi == bj;
    const double* tile = val + ioff[q];
    double bjl[kB], cacc[kB];
#pragma unroll
    for (int c = 0; c < kB; ++c) {
      const int64_t j = (int64_t)bj * kR + c * kT + lane;
      bjl[c] = j < n ? b[j] : 0.0;
      cacc[c] = 0.0;
    }
#pragma unroll
    for (int r = 0; r < kB; ++r) {
      const int64_t i = (int64_t)bi * kR + r * kT + lane;
      const double bil = i < n ? b[i] : 0.0;
      double p[kT];
#pragma unroll
      for (int k = 0; k < kT; ++k) p[k] = 0.0;
#pragma unroll
      for (int c = 0; c < kB; ++c) {
        if (diag && c > r) break;
        double v[kT];
#pragma unroll
        for (int k = 0; k < kT; ++k) v[k] = ld_stream(tile + k * kT + lane);
        tile += kT * kT;
#pragma unroll
        for (int k = 0; k < kT; ++k) p[k] = fma(v[k], bjl[c], p[k]);
        if (!(diag && c == r)) {
#pragma unroll
          for (int k = 0; k < kT; ++k) cacc[c] = fma(v[k], __shfl_sync(0xffffffffu, bil, k), cacc[c]);
        }
      }
      // transpose-reduce: lane l ends with sum over lanes of p[l]
#pragma unroll
      for (int o = kT / 2; o > 0; o >>= 1) {
        const bool up = lane & o;
#pragma unroll
        for (int k = 0; k < o; ++k) {
          const double send = up ? p[k] : p[k + o];
          const double keep = up ? p[k + o] : p[k];
          p[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      rowpart[(int64_t)q * kR + r * kT + lane] = p[0];
    }
#pragma unroll
    for (int c = 0; c < kB; ++c) colpart[(int64_t)q * kR + c * kT + lane] = cacc[c];
  }
}

// x[j] = sum over bj <= bi of rowpart(bi, bj)[o] + sum over bi' >= bi of colpart(bi', bi)[o]
// The nb + 1 terms of a row are split into kParts contiguous runs, one thread
// each (32 consecutive rows per warp: coalesced, and one bi per warp since
// 32 | kR), each run summed in order, then the runs in order: a fixed order,
// so results are bit-identical run to run.  One thread per row was
// latency-bound (~26 dependent L2 round trips).
constexpr int kParts = 8;
__global__ void __launch_bounds__(32 * kParts) k_symv_reduce(const int* stop, int64_t n, int nb,
                                                             const double* __restrict__ rowpart,
                                                             const double* __restrict__ colpart,
                                                             double* __restrict__ x) {
  if (*stop) return;
  __shared__ double part[kParts][32];
  const int lane = threadIdx.x & 31, p = threadIdx.x >> 5;
  const int64_t j = blockIdx.x * 32LL + lane;
  const int bi = (int)((blockIdx.x * 32LL) / kR), o = (int)(j % kR);
  const int T = nb + 1;  // bi + 1 row terms, then nb - bi column terms
  const int t0 = (int)((int64_t)T * p / kParts), t1 = (int)((int64_t)T * (p + 1) / kParts);
  double s = 0.0;
  if (j < n) {
    const double* rp = rowpart + (int64_t)item_of(bi, 0) * kR + o;  // items (bi, 0..bi) are consecutive
#pragma unroll 8
    for (int t = t0; t < t1; ++t) {
      const double v = t <= bi ? __ldcs(rp + (int64_t)t * kR) : __ldcs(colpart + (int64_t)item_of(t - 1, bi) * kR + o);
      s += v;
    }
  }
  part[p][lane] = s;
  __syncthreads();
  if (p == 0 && j < n) {
    double r = part[0][lane];
#pragma unroll
    for (int q = 1; q < kParts; ++q) r += part[q][lane];
    x[j] = r;
  }
}

// one CTA per item: copy its sub-tiles out of the full row-major matrix (zeros past n)
__global__ void k_pack_items(int64_t n, const double* __restrict__ full, const int64_t* __restrict__ ioff,
                             double* __restrict__ val) {
  const int q = blockIdx.x;
  int bi = 0;
  while ((bi + 1) * (bi + 2) / 2 <= q) ++bi;
  const int bj = q - bi * (bi + 1) / 2;
  double* out = val + ioff[q];
  int t = 0;
  for (int r = 0; r < kB; ++r)
    for (int c = 0; c < kB; ++c) {
      if (bi == bj && c > r) break;
      for (int e = threadIdx.x; e < kT * kT; e += blockDim.x) {
        const int64_t i = (int64_t)bi * kR + r * kT + e / kT, j = (int64_t)bj * kR + c * kT + e % kT;
        out[(int64_t)t * kT * kT + e] = (i < n && j < n) ? full[i * n + j] : 0.0;
      }
      ++t;
    }
}

}  // namespace

void symv_build(const double* full, int64_t n, SymPacked& sp, cudaStream_t s) {
  sp.on = false;
  if (n <= 0) return;
  sp.n = n;
  sp.nb = (int)((n + kR - 1) / kR);
  sp.items = sp.nb * (sp.nb + 1) / 2;
  std::vector<int64_t> ioff((size_t)sp.items + 1, 0);
  for (int bi = 0, q = 0; bi < sp.nb; ++bi)
    for (int bj = 0; bj <= bi; ++bj, ++q)
      ioff[(size_t)q + 1] = ioff[(size_t)q] + (int64_t)(bi == bj ? kB * (kB + 1) / 2 : kB * kB) * kT * kT;
  sp.ioff.upload(ioff.data(), sp.items + 1, s);
  sp.val.alloc(ioff[(size_t)sp.items], s);
  sp.rowpart.alloc((int64_t)sp.items * kR, s);
  sp.colpart.alloc((int64_t)sp.items * kR, s);
  k_pack_items<<<(unsigned)sp.items, 256, 0, s>>>(n, full, sp.ioff.p, sp.val.p);
  HC_CHECK_LAUNCH();
  int per_sm = 0;
  HC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_symv_items, kSymThreads, 0));
  sp.grid = std::max(1, std::min(kSMs * std::max(per_sm, 1), (sp.items + kSymThreads / 32 - 1) / (kSymThreads / 32)));
  sp.on = true;
}

void symv_apply(const int* stop, const SymPacked& sp, const double* b, double* x, cudaStream_t s) {
  k_symv_items<<<(unsigned)sp.grid, kSymThreads, 0, s>>>(stop, sp.n, sp.nb, sp.items, sp.val.p, sp.ioff.p, b,
                                                         sp.rowpart.p, sp.colpart.p);
  HC_CHECK_LAUNCH();
  k_symv_reduce<<<(unsigned)((sp.n + 31) / 32), 32 * kParts, 0, s>>>(stop, sp.n, sp.nb, sp.rowpart.p, sp.colpart.p, x);
  HC_CHECK_LAUNCH();
}

}  // namespace hcamg
