// Exchange kernels of the row-partitioned solve (see dist.cuh).
#include "dist.cuh"

namespace hcamg {

namespace {

struct Grp {
  int64_t b[kGroups + 1];  // chunk boundaries of the groups
};

__global__ void __launch_bounds__(256) k_group_sums(const int* stop, Xchg x, int64_t nc,
                                                    const double* __restrict__ partial, Grp grp, int g0, int g1) {
  if (*stop) return;
  const unsigned long long e = xepoch(x);
  // one thread per (group, column)
  const int64_t total = (int64_t)(g1 - g0) * nc;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int g = g0 + (int)(t / nc);
    const int64_t c = t % nc;
    double gs = 0.0;
    for (int64_t ch = grp.b[g]; ch < grp.b[g + 1]; ++ch) gs += partial[ch * nc + c];
    for (int r = 0; r < x.nranks; ++r) xarea(x, r, e + 1)[g * nc + c] = gs;
  }
  xsignal(x, e);
}

__global__ void __launch_bounds__(256) k_group_final(const int* stop, Xchg x, int64_t nc, double* __restrict__ bc) {
  if (*stop) return;
  const unsigned long long e = xwait(x);
  const double* gsum = xarea(x, x.rank, e);
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int g = 0; g < kGroups; ++g) acc += __ldcg(gsum + g * nc + c);
    bc[c] -= acc;
  }
}

__global__ void __launch_bounds__(256) k_scatter(const int* stop, Xchg x, int64_t n, const int32_t* __restrict__ rows,
                                                 double* __restrict__ out) {
  if (*stop) return;
  const unsigned long long e = xwait(x);
  const double* y = xarea(x, x.rank, e);
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    if (rows) out[rows[q]] -= __ldcg(y + q);
    else out[q] = __ldcg(y + q);
  }
}

}  // namespace

Xchg Dist::site(size_t off) const {
  Xchg x{};
  for (int r = 0; r < kMaxRanks; ++r) x.base[r] = base[r];
  x.rank = rank;
  x.nranks = nranks;
  x.area_bytes = area_bytes;
  x.off = off;
  x.ep = ep.p;
  x.cta = cta.p;
  x.err = err.p;
  return x;
}

void Dist::release() {
  for (int r = 0; r < kMaxRanks; ++r) {
    if (opened[r] && base[r]) cudaIpcCloseMemHandle(base[r]);
    opened[r] = false;
    base[r] = nullptr;
  }
  if (sym) cudaFree(sym);
  sym = nullptr;
  sym_bytes = area_bytes = 0;
  on = false;
}

void xchg_group_sums(const int* stop, const Xchg& x, int64_t nc, const double* partial, const int64_t* grp_host,
                     int g0, int g1, cudaStream_t s) {
  Grp g{};
  for (int t = 0; t <= kGroups; ++t) g.b[t] = grp_host[t];
  k_group_sums<<<grid_for(std::max<int64_t>((int64_t)(g1 - g0) * nc, 1), 256), 256, 0, s>>>(stop, x, nc, partial, g,
                                                                                           g0, g1);
  HC_CHECK_LAUNCH();
}

void xchg_group_final(const int* stop, const Xchg& x, int64_t nc, double* bc, cudaStream_t s) {
  k_group_final<<<grid_for(std::max<int64_t>(nc, 1), 256), 256, 0, s>>>(stop, x, nc, bc);
  HC_CHECK_LAUNCH();
}

void xchg_scatter(const int* stop, const Xchg& x, int64_t n, const int32_t* rows, double* out, cudaStream_t s) {
  k_scatter<<<grid_for(std::max<int64_t>(n, 1), 256), 256, 0, s>>>(stop, x, n, rows, out);
  HC_CHECK_LAUNCH();
}

}  // namespace hcamg
