// Shared device infrastructure for libhcamg: error plumbing, stream-ordered
// device buffers, device CSR, and small launch helpers.  sm_100a only.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <stdexcept>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <utility>
#include <vector>

namespace hcamg {

// Status codes mirrored in include/hcamg.h.
enum Status : int {
  OK = 0,
  EINVAL_ = -1,      // bad argument / shape -> ValueError
  ENOTSPD_ = -2,     // Cholesky breakdown -> NotPositiveDefiniteError(pivot)
  EBREAKDOWN_ = -3,  // PCG breakdown -> RuntimeError
  ENOMEM_ = -4,
  ECUDA_ = -5,
  ENOTSYM_ = -6,     // coarsest symmetry check -> ValueError
  EUNSUPPORTED_ = -7,
};

struct Error : std::runtime_error {
  int code;
  int64_t index;
  Error(int c, const std::string& m, int64_t idx = -1) : std::runtime_error(m), code(c), index(idx) {}
};

#define HC_CUDA(x)                                                                          \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess)                                                                  \
      throw ::hcamg::Error(e_ == cudaErrorMemoryAllocation ? ::hcamg::ENOMEM_ : ::hcamg::ECUDA_, \
                           std::string(#x) + ": " + cudaGetErrorString(e_) + " @" __FILE__ ":" + \
                               std::to_string(__LINE__));                                   \
  } while (0)

#define HC_CHECK_LAUNCH() HC_CUDA(cudaGetLastError())

inline void require(bool ok, const std::string& msg) {
  if (!ok) throw Error(EINVAL_, msg);
}

cudaMemPool_t current_pool();

// Stream-ordered device buffer (the handle's private pool when one is in
// scope, else the device's default cudaMallocAsync pool).
template <class T>
struct DBuf {
  T* p = nullptr;
  int64_t n = 0;
  cudaStream_t s = 0;
  bool view = false;  // points into memory owned elsewhere (the row partition's symmetric buffer)
  DBuf() = default;
  DBuf(int64_t count, cudaStream_t st) { alloc(count, st); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s), view(o.view) { o.p = nullptr; o.n = 0; o.view = false; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; s = o.s; view = o.view; o.p = nullptr; o.n = 0; o.view = false; }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(int64_t count, cudaStream_t st) {
    release();
    s = st;
    n = count;
    if (count > 0) {
      cudaMemPool_t pool = current_pool();
      if (pool) HC_CUDA(cudaMallocFromPoolAsync((void**)&p, sizeof(T) * (size_t)count, pool, st));
      else HC_CUDA(cudaMallocAsync((void**)&p, sizeof(T) * (size_t)count, st));
    }
  }
  void release() {
    if (p && !view) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
    view = false;
  }
  void alias(T* ptr, int64_t count, cudaStream_t st) {
    release();
    p = ptr;
    n = count;
    s = st;
    view = true;
  }
  void zero() { if (n) HC_CUDA(cudaMemsetAsync(p, 0, sizeof(T) * (size_t)n, s)); }
  void fill_bytes(int v) { if (n) HC_CUDA(cudaMemsetAsync(p, v, sizeof(T) * (size_t)n, s)); }
  void upload(const T* host, int64_t count) {
    alloc(count, s);
    if (count) HC_CUDA(cudaMemcpyAsync(p, host, sizeof(T) * (size_t)count, cudaMemcpyHostToDevice, s));
  }
  void upload(const T* host, int64_t count, cudaStream_t st) { s = st; upload(host, count); }
  std::vector<T> download() const {
    std::vector<T> h((size_t)n);
    if (n) {
      HC_CUDA(cudaMemcpyAsync(h.data(), p, sizeof(T) * (size_t)n, cudaMemcpyDeviceToHost, s));
      HC_CUDA(cudaStreamSynchronize(s));
    }
    return h;
  }
  T* get() const { return p; }
};

template <class T>
inline T read_scalar(const T* dev, cudaStream_t s) {
  T h;
  HC_CUDA(cudaMemcpyAsync(&h, dev, sizeof(T), cudaMemcpyDeviceToHost, s));
  HC_CUDA(cudaStreamSynchronize(s));
  return h;
}

// Sliced-ELLPACK copy of a short-row CSR (solve.cu build_sell): 32 rows per
// slice, entries of a slice column-major (entry j of the slice's row l at
// soff[slice] + 32 j + l), padded to the slice's longest row with column -1.
struct DSell {
  int64_t nslice = 0, padded = 0;
  DBuf<int64_t> soff;
  DBuf<int32_t> idx;
  DBuf<double> val;
};

// Device CSR: int64 row pointers, int32 column indices, fp64 values.
struct DCsr {
  int64_t nrows = 0, ncols = 0, nnz = 0;
  DBuf<int64_t> ptr;
  DBuf<int32_t> idx;
  DBuf<double> val;
  std::unique_ptr<DSell> sell;  // optional SpMV layout of the solve phase
  void alloc(int64_t r, int64_t c, int64_t z, cudaStream_t s) {
    nrows = r; ncols = c; nnz = z;
    ptr.alloc(r + 1, s);
    idx.alloc(z, s);
    val.alloc(z, s);
  }
};

// HCAMG_SETUP_TIMING=1: print the wall time of setup stages to stderr
// (synchronises the stream at every mark; off by default).
struct StageTimer {
  cudaStream_t s;
  bool on;
  std::chrono::steady_clock::time_point t;
  double f0 = 0.0;  // dense FP64 flops counted when the stage began (count_flops)
  explicit StageTimer(cudaStream_t st) : s(st), on(getenv("HCAMG_SETUP_TIMING") != nullptr), t(std::chrono::steady_clock::now()) {
    if (on) f0 = peek_flops();
  }
  static double peek_flops();
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    const double dt = std::chrono::duration<double>(now - t).count(), f = peek_flops();
    if (f - f0 > 1e9) fprintf(stderr, "[hcamg setup] %-28s %9.3f s  %6.1f TF/s\n", what, dt, (f - f0) / dt / 1e12);
    else fprintf(stderr, "[hcamg setup] %-28s %9.3f s\n", what, dt);
    t = now;
    f0 = f;
  }
};

inline unsigned grid_for(int64_t work, int threads, int64_t cap = 148 * 32) {
  int64_t g = (work + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

constexpr int kSMs = 148;

// Per-handle options (hcamg_set_option).  They replace the process-wide
// HCAMG_* environment switches of round 1: the environment only seeds the
// defaults when a handle is created, and every entry point runs with its
// handle's options installed (OptionsScope), so tests can force a code path
// per hierarchy.
enum SweepMode : int {
  SWEEP_AUTO = 0,     // cluster leg when a wave fits 16 CTAs, else the grid leg
  SWEEP_LEG = 1,      // cluster leg (one 16-CTA cluster, prefetching)
  SWEEP_GRID = 2,     // cooperative grid leg
  SWEEP_WAVE = 3,     // one launch per wavefront
  SWEEP_FLOW = 4,     // dataflow leg: per-patch ready counters, no wave barriers
  SWEEP_FWAVE = 5,    // one launch per wavefront over the dataflow records (wide 2D schedules)
};
struct Options {
  int sweep = SWEEP_AUTO;
  int64_t giant_min = 4096;        // dense-regime cutoff (= reference _DENSE_COMPONENT_CUTOFF, transfer.py:35)
  int64_t coarse_gemv_min = 8192;  // coarsest solve: HBM row GEMV from this size on
  int coarse_symv = 1;             // single GPU: packed lower triangle of the inverse
  int factor_apply = 1;            // dense block applied through the envelope factor (0: explicit Z)
  int form_z = 0;                  // keep the explicit Z block resident even when the factor applies P
  int tri_calib = 4;               // calibration rounds of the TMA sweep partition
};
Options options_from_env();
const Options& opts();
struct OptionsScope {
  const Options* prev;
  explicit OptionsScope(const Options* o);
  ~OptionsScope();
};
// Allocation pool of the handle in scope (nullptr: the device default pool).
struct PoolScope {
  cudaMemPool_t prev;
  explicit PoolScope(cudaMemPool_t p);
  ~PoolScope();
};
cudaMemPool_t current_pool();

// FP64 flops of the dense setup work issued while a handle's setup runs
// (counted at each level-3 call from its dimensions; hcamg_info.setup_flops).
void count_flops(double f);
double take_flops();

}  // namespace hcamg
