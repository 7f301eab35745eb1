// Restriction with long CSR P^T rows (dense interior rows of a hybrid P below
// the dense-regime cutoff): every row is cut into fixed 256-entry segments,
// one warp per segment, and the segment partials of a row are summed in
// segment order by a second kernel -- deterministic, and no row waits on a
// single warp streaming thousands of entries.
#include <algorithm>
#include <vector>

#include "sweep.cuh"

namespace hcamg {

namespace {

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

}  // namespace

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

}  // namespace hcamg
