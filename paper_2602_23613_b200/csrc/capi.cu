// C-ABI of libhcamg (include/hcamg.h): handle lifetime, the build_hierarchy
// driver (hcurl_amg/multilevel.py:78-164) and the solve entry points
// (multilevel.py:187-281) with their CUDA-graph executables.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/hcamg.h"
#include "dblas.cuh"
#include "dense.cuh"
#include "dist.cuh"
#include "rows_dev.cuh"
#include "giant.cuh"
#include "kuhn.cuh"
#include "interp.cuh"
#include "smoother.cuh"
#include "solve.cuh"

using namespace hcamg;

namespace {

constexpr int kSmootherOnly = 3;  // hcamg_info.method of a hcamg_smoother_setup handle

struct Graph {
  cudaGraphExec_t exec = nullptr;
  cudaGraphExec_t pre = nullptr, body = nullptr;  // host-driven fallback
  bool conditional = false;
  int64_t launches_pre = 0, launches_body = 0;
  void reset() {
    if (exec) cudaGraphExecDestroy(exec);
    if (pre) cudaGraphExecDestroy(pre);
    if (body) cudaGraphExecDestroy(body);
    exec = pre = body = nullptr;
    launches_pre = launches_body = 0;
  }
};

}  // namespace

struct hcamg_handle {
  int device = 0;
  cudaStream_t stream = nullptr, aux = nullptr;
  bool own_stream = false;
  std::vector<std::unique_ptr<DevLevel>> levels;
  std::vector<DevLevel*> lv;
  bool stalled = false;
  int method = 1;
  std::vector<std::string> notes;
  double setup_seconds = 0.0, setup_flops = 0.0;
  Workspace ws;
  Graph g_vc, g_pcg, g_amg;
  DBuf<double> vc_b, vc_x;
  int64_t graph_maxit = -1;
  std::string err;
  int64_t err_index = -1;
  // user-assembled hierarchy under construction
  std::vector<std::unique_ptr<DevLevel>> pending;
  // result of the last hcamg_split_alg (level-0 splitting only)
  SplitResult last_split;
  // row-partitioned solve across processes (dist.cuh)
  Dist dist;
  // subdomain row partition of the sparse regime (rows.cuh)
  std::unique_ptr<RowsCtx> rows;
  // last hcamg_kuhn_assemble result (kuhn.cuh)
  DCsr kuhn_A, kuhn_G;
  std::vector<int64_t> kuhn_fe, kuhn_fv;
  // per-handle options (hcamg_set_option) and private allocation pool
  Options opts;
  cudaMemPool_t pool = nullptr;
};

namespace {

void upload_csr(const hcamg_csr* M, DCsr& out, cudaStream_t s) {
  require(M != nullptr, "missing matrix");
  require(M->nrows >= 0 && M->ncols >= 0, "negative matrix shape");
  csr_upload(M->indptr, M->indices, M->data, M->nrows, M->ncols, out, s);
}

void invalidate(hcamg_handle* h) {
  h->g_vc.reset();
  h->g_pcg.reset();
  h->g_amg.reset();
  h->graph_maxit = -1;
}

bool rows_on(const hcamg_handle* h) { return h->rows && h->rows->on; }

void drop_rows(hcamg_handle* h) {
  if (!h->rows) return;
  // the level / workspace vectors point into the partition's symmetric buffer
  std::vector<DevLevel*> lv;
  for (auto& l : h->levels) lv.push_back(l.get());
  rows_detach(*h->rows, lv, h->ws, h->stream);
  h->rows.reset();
}

void refresh_views(hcamg_handle* h) {
  h->dist.release();  // a new hierarchy needs a new exchange layout
  if (h->rows) {      // the old levels are gone: nothing to re-point
    for (DBuf<double>* v : {&h->ws.x, &h->ws.r, &h->ws.z, &h->ws.p, &h->ws.Ap, &h->ws.b})
      if (v->view) { v->release(); h->ws.n = -1; }
    h->rows.reset();
  }
  h->lv.clear();
  for (auto& l : h->levels) h->lv.push_back(l.get());
}

void alloc_level_vectors(DevLevel& L, cudaStream_t s) {
  const int64_t n = std::max<int64_t>(L.n, 1);
  for (DBuf<double>* v : {&L.b, &L.x, &L.r, &L.d0, &L.d1, &L.dj}) {
    v->alloc(n, s);
    v->zero();
  }
}

// ---- Galerkin product P^T (A P), symmetrised (sparse.py:113-122)
void galerkin(const DCsr& P, const DCsr& Pt, const DCsr& A, DCsr& out, cudaStream_t s) {
  DCsr AP, M;
  spgemm(A, P, AP, s);
  spgemm(Pt, AP, M, s);
  AP = DCsr();
  symmetrize(M, out, s);
}

__global__ void k_asym(const int64_t* __restrict__ p, const int32_t* __restrict__ ix, const double* __restrict__ v,
                       int64_t n, unsigned long long* out) {
  double m = 0.0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    for (int64_t e = p[r]; e < p[r + 1]; ++e) {
      const int32_t c = ix[e];
      int64_t lo = p[c], hi = p[c + 1];
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (ix[mid] < r) lo = mid + 1; else hi = mid;
      }
      const double t = (lo < p[c + 1] && ix[lo] == r) ? v[lo] : 0.0;
      m = fmax(m, fabs(v[e] - t));
    }
  }
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// the same for a fully dense canonical CSR (val[i n + j] = M[i, j]): 32 x 32 tiles
// against their mirror tiles through shared memory (config 2's 26,236^2 coarse
// operator: the row-walk with a binary search per entry took 144 ms)
__global__ void k_asym_dense(const double* __restrict__ v, int64_t n, unsigned long long* out) {
  __shared__ double t[32][33];
  const int64_t nt = (n + 31) / 32;
  double m = 0.0;
  for (int64_t b = blockIdx.x; b < nt * nt; b += gridDim.x) {
    const int64_t bi = b / nt, bj = b % nt;
    if (bj > bi) continue;
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
      const int64_t i = bj * 32 + r, j = bi * 32 + threadIdx.x;  // the mirror tile, read by rows
      t[r][threadIdx.x] = (i < n && j < n) ? v[i * n + j] : 0.0;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
      const int64_t i = bi * 32 + r, j = bj * 32 + threadIdx.x;
      if (i < n && j < n) m = fmax(m, fabs(v[i * n + j] - t[threadIdx.x][r]));
    }
  }
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (threadIdx.x == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

__global__ void k_densify(const int64_t* __restrict__ p, const int32_t* __restrict__ ix, const double* __restrict__ v,
                          int64_t n, double* __restrict__ D) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    for (int64_t e = p[r]; e < p[r + 1]; ++e) D[r + (int64_t)ix[e] * n] = v[e];  // column-major
}


// Coarsest level: cholesky(A) (sparse.py:276-301) -> explicit inverse.
void factor_coarsest(hcamg_handle* h, DevLevel& L, const DCsr& M) {
  cudaStream_t s = h->stream;
  const int64_t n = M.nrows;
  require(M.nrows == M.ncols, "matrix must be square");
  {
    DBuf<unsigned long long> a(1, s);
    a.zero();
    if (n >= 64 && csr_is_dense_canonical(M, s)) k_asym_dense<<<kSMs * 8, dim3(32, 8), 0, s>>>(M.val.p, n, a.p);
    else if (n) k_asym<<<grid_for(n, 128), 128, 0, s>>>(M.ptr.p, M.idx.p, M.val.p, n, a.p);
    HC_CHECK_LAUNCH();
    unsigned long long ha = read_scalar(a.p, s);
    double asym;
    memcpy(&asym, &ha, 8);
    const double scale = max_abs(M, s);
    if (scale > 0 && asym > 1e-12 * scale) {
      char buf[128];
      snprintf(buf, sizeof buf, "matrix not symmetric: asymmetry %.3e", asym);
      throw Error(ENOTSYM_, buf);
    }
  }
  L.coarsest = true;
  if (n == 0) return;
  DBuf<double> D(n * n, s);
  D.zero();
  k_densify<<<grid_for(n, 128), 128, 0, s>>>(M.ptr.p, M.idx.p, M.val.p, n, D.p);
  HC_CHECK_LAUNCH();
  StageTimer st(s);
  dblas::LeafCacheScope leaves;  // the factor's 64 x 64 diagonal leaves are inverted once for both steps
  int64_t bad = dense_cholesky(D.p, n, n, s);
  st.mark("  coarsest: cholesky");
  if (bad >= 0) throw Error(ENOTSPD_, "matrix is not positive definite (pivot " + std::to_string(bad) + ")", bad);
  L.Ainv.alloc(n * n, s);
  dense_spd_inverse(D.p, n, L.Ainv.p, s);
  st.mark("  coarsest: inverse");
  if (n >= coarse_gemv_min() && opts().coarse_symv) symv_build(L.Ainv.p, n, L.Asym, s);
}

void finish_level(hcamg_handle* h, DevLevel& L) {
  cudaStream_t s = h->stream;
  L.n = L.A.nrows;
  alloc_level_vectors(L, s);
  if (L.has_P) {
    build_l1(L.A, L.l1, s);
    build_smoother(L.A, L.G, L.sm, s);
    build_sell(L.A, s);
    build_sell(L.P, s);
    build_sell(L.Pt, s);
    // restriction with long P^T rows (dense interior blocks): segmented plan
    std::vector<int64_t> tp = L.Pt.ptr.download();
    L.pt_maxrow = 0;
    for (int64_t p = 0; p < L.Pt.nrows; ++p) L.pt_maxrow = std::max(L.pt_maxrow, tp[(size_t)p + 1] - tp[(size_t)p]);
    if (L.pt_maxrow > 512) build_segments(L.Pt, L.pt_seg, s);
  }
}

struct RefChain {
  int32_t nm = 0;
  const int64_t* ne = nullptr;
  const int64_t* const* edges = nullptr;
  const int64_t* const* children = nullptr;
  const int64_t* free_edges = nullptr;
};

void build_hierarchy(hcamg_handle* h, const hcamg_csr* Ah, const hcamg_csr* Gh, int method, int32_t max_levels,
                     int64_t min_coarse, double theta, const RefChain* chain) {
  cudaStream_t s = h->stream;
  invalidate(h);
  h->levels.clear();
  h->lv.clear();
  h->notes.clear();
  h->stalled = false;
  h->method = method;
  require(Ah->nrows == Ah->ncols, "A must be square");
  require(Gh->nrows == Ah->nrows, "G rows must match A");
  HC_CUDA(cudaStreamSynchronize(s));
  auto t0 = std::chrono::steady_clock::now();
  take_flops();
  StageTimer st(s);
  auto cur = std::make_unique<DevLevel>();
  upload_csr(Ah, cur->A, s);
  upload_csr(Gh, cur->G, s);
  st.mark("upload");
  int32_t pos = method == 0 ? chain->nm - 1 : 0;
  std::vector<int64_t> e2d;
  if (method == 0) e2d.assign(chain->free_edges, chain->free_edges + chain->ne[chain->nm - 1]);
  while (true) {
    const int64_t n = cur->A.nrows;
    if (n <= min_coarse || (int64_t)h->levels.size() + 1 >= max_levels) break;
    SplitResult sp;
    int mode;
    if (method == 0) {
      if (pos == 0) {
        if (n > min_coarse) {
          h->stalled = true;
          h->notes.push_back("mesh chain exhausted at " + std::to_string(n) + " DoFs");
        }
        break;
      }
      refinement_splitting(chain->edges[pos - 1], chain->ne[pos - 1], chain->edges[pos], chain->ne[pos],
                           chain->children[pos - 1], e2d.data(), n, sp, s);
      if (sp.n_pairs() == 0) {
        h->stalled = true;
        h->notes.push_back("refinement splitting produced no pairs");
        break;
      }
      mode = 0;
    } else {
      algebraic_splitting(cur->A, cur->G, theta, sp, s);
      st.mark("splitting");
      if (sp.n_pairs() == 0 || sp.n_pairs() >= n) {
        if (sp.n_pairs() == 0) {
          h->stalled = true;
          h->notes.push_back("algebraic coarsening found no pairs");
        }
        break;
      }
      mode = 1;
    }
    InterpResult ip;
    build_interp(cur->A, cur->G, sp, mode, ip, s);
    st.mark("interpolation");
    if (ip.P.ncols == 0 || ip.P.ncols >= n) {
      h->stalled = true;
      h->notes.push_back("no size reduction (" + std::to_string(n) + " -> " + std::to_string(ip.P.ncols) + ")");
      break;
    }
    auto next = std::make_unique<DevLevel>();
    if (ip.hp.on) {
      galerkin_hybrid(cur->A, ip.P, ip.Pt, ip.hp, next->A, s);
      ip.hp.D.release();
    } else {
      galerkin(ip.P, ip.Pt, cur->A, next->A, s);
    }
    st.mark("galerkin");
    cur->hp = std::move(ip.hp);
    if (cur->hp.on) hybrid_prepare(cur->hp, s);
    next->G = std::move(ip.Gc);
    cur->has_P = true;
    cur->P = std::move(ip.P);
    cur->Pt = std::move(ip.Pt);
    cur->gc_cols = ip.gc_cols;
    if (method == 0) {
      std::vector<int64_t> nx((size_t)chain->ne[pos - 1], -1);
      for (size_t t = 0; t < sp.pair_mesh_edges.size(); ++t) nx[(size_t)sp.pair_mesh_edges[t]] = (int64_t)t;
      e2d.swap(nx);
      --pos;
    }
    cur->split = std::move(sp);
    finish_level(h, *cur);
    st.mark("smoother + level data");
    h->levels.push_back(std::move(cur));
    cur = std::move(next);
  }
  factor_coarsest(h, *cur, cur->A);
  st.mark("coarsest factor");
  finish_level(h, *cur);
  st.mark("coarsest level data");
  h->levels.push_back(std::move(cur));
  refresh_views(h);
  HC_CUDA(cudaStreamSynchronize(s));
  h->setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  h->setup_flops = take_flops();
  // hand the setup's transient buffers (tens of GB on config 2) back to the
  // device: the private pool keeps freed memory only while a build runs
  if (h->pool) HC_CUDA(cudaMemPoolTrimTo(h->pool, 0));
}

void fill_info(hcamg_handle* h, hcamg_info* info) {
  if (!info) return;
  info->depth = (int32_t)h->levels.size();
  info->stalled = h->stalled;
  info->method = h->method;
  double tot = 0;
  for (auto& l : h->levels) tot += (double)l->A.nnz;
  info->operator_complexity = h->levels.empty() || h->levels[0]->A.nnz == 0 ? 0.0 : tot / (double)h->levels[0]->A.nnz;
  info->setup_seconds = h->setup_seconds;
  info->setup_flops = h->setup_flops;
}

// ---- graphs

void ensure_ws(hcamg_handle* h, int64_t maxit) {
  const int64_t n = h->levels.empty() ? 0 : h->levels[0]->n;
  const void* old[] = {h->ws.x.p, h->ws.hist.p, h->ws.ctl.p};
  h->ws.ensure(n, std::max<int64_t>(maxit, 1), h->stream);
  const void* now[] = {h->ws.x.p, h->ws.hist.p, h->ws.ctl.p};
  if (memcmp(old, now, sizeof old) != 0) invalidate(h);
}

void build_loop_graph(hcamg_handle* h, Graph& G, bool pcg) {
  cudaStream_t s = h->stream, s2 = h->aux;
  Workspace& w = h->ws;
  const double* b = w.b.p;
  G.reset();
  // try a single graph with a device-side WHILE loop
  cudaGraph_t g = nullptr;
  HC_CUDA(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle cond;
  // HCAMG_HOST_LOOP=1 forces the host-driven loop (same kernels; lets ncu profile graph nodes,
  // which it cannot do inside graphs that contain conditional nodes)
  const char* hl = getenv("HCAMG_HOST_LOOP");
  cudaError_t ce = (hl && hl[0] == '1') ? cudaErrorNotSupported
                                        : cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault);
  if (ce == cudaSuccess) {
    HC_CUDA(cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    int64_t lp = rows_on(h) && !pcg ? rows_record(*h->rows, SEG_AMG_INIT, h->lv, w, &w.ctl.p->stop, 0, s)
                 : rows_on(h) ? rows_record(*h->rows, SEG_INIT, h->lv, w, &w.ctl.p->stop, 0, s) +
                                  rows_record(*h->rows, SEG_FIRST, h->lv, w, &w.ctl.p->stop, 0, s)
                 : pcg ? record_pcg_init(*h->lv[0], w, b, nullptr, s, 0) + record_pcg_first(h->lv, w, s)
                       : record_amg_init(*h->lv[0], w, b, nullptr, s, 0);
    cudaStreamCaptureStatus st;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    cudaGraph_t cg = nullptr;
    HC_CUDA(cudaStreamGetCaptureInfo(s, &st, nullptr, &cg, &deps, &nd));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cn;
    HC_CUDA(cudaGraphAddNode(&cn, cg, deps, nd, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    HC_CUDA(cudaStreamUpdateCaptureDependencies(s, &cn, 1, cudaStreamSetCaptureDependencies));
    HC_CUDA(cudaStreamBeginCaptureToGraph(s2, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    const unsigned long long hc = (unsigned long long)cond;
    int64_t lb = rows_on(h) ? rows_record(*h->rows, pcg ? SEG_BODY : SEG_AMG_BODY, h->lv, w, &w.ctl.p->stop, hc, s2)
                 : pcg ? record_pcg_body(h->lv, w, s2, hc) : record_amg_body(h->lv, w, s2, hc);
    HC_CUDA(cudaStreamEndCapture(s2, &body));
    cudaGraph_t gout = nullptr;
    HC_CUDA(cudaStreamEndCapture(s, &gout));
    ce = cudaGraphInstantiate(&G.exec, g, 0);
    cudaGraphDestroy(g);
    if (ce == cudaSuccess) {
      G.conditional = true;
      G.launches_pre = lp;
      G.launches_body = lb;
      return;
    }
    cudaGetLastError();
    G.exec = nullptr;
  } else {
    cudaGetLastError();
    cudaGraphDestroy(g);
  }
  // fallback: host-driven loop over a body graph
  cudaGraph_t gp = nullptr, gb = nullptr;
  HC_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  G.launches_pre = rows_on(h) && !pcg ? rows_record(*h->rows, SEG_AMG_INIT, h->lv, w, &w.ctl.p->stop, 0, s)
                   : rows_on(h) ? rows_record(*h->rows, SEG_INIT, h->lv, w, &w.ctl.p->stop, 0, s) +
                                    rows_record(*h->rows, SEG_FIRST, h->lv, w, &w.ctl.p->stop, 0, s)
                   : pcg ? record_pcg_init(*h->lv[0], w, b, nullptr, s, 0) + record_pcg_first(h->lv, w, s)
                         : record_amg_init(*h->lv[0], w, b, nullptr, s, 0);
  HC_CUDA(cudaStreamEndCapture(s, &gp));
  HC_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  G.launches_body = rows_on(h) ? rows_record(*h->rows, pcg ? SEG_BODY : SEG_AMG_BODY, h->lv, w, &w.ctl.p->stop, 0, s)
                    : pcg ? record_pcg_body(h->lv, w, s, 0) : record_amg_body(h->lv, w, s, 0);
  HC_CUDA(cudaStreamEndCapture(s, &gb));
  HC_CUDA(cudaGraphInstantiate(&G.pre, gp, 0));
  HC_CUDA(cudaGraphInstantiate(&G.body, gb, 0));
  cudaGraphDestroy(gp);
  cudaGraphDestroy(gb);
  G.conditional = false;
}

void run_loop_graph(hcamg_handle* h, Graph& G) {
  cudaStream_t s = h->stream;
  if (G.conditional) {
    HC_CUDA(cudaGraphLaunch(G.exec, s));
    return;
  }
  HC_CUDA(cudaGraphLaunch(G.pre, s));
  while (true) {
    int stop = read_scalar(&h->ws.ctl.p->stop, s);
    if (stop) break;
    HC_CUDA(cudaGraphLaunch(G.body, s));
  }
}

void set_ctl(hcamg_handle* h, double tol, int64_t maxit) {
  Ctl c{};
  c.tol = tol;
  c.maxit = maxit;
  HC_CUDA(cudaMemcpyAsync(h->ws.ctl.p, &c, sizeof(Ctl), cudaMemcpyHostToDevice, h->stream));
}

void require_hierarchy(hcamg_handle* h) {
  require(!h->levels.empty(), "no hierarchy: call hcamg_setup_* first");
  require(h->method != kSmootherOnly, "the handle holds a smoother only (hcamg_smoother_setup)");
}

void prepare_loop(hcamg_handle* h, Graph& G, bool pcg, int64_t maxit) {
  ensure_ws(h, maxit);
  if (!(G.exec || G.pre)) build_loop_graph(h, G, pcg);
}

void read_report(hcamg_handle* h, hcamg_report* rep, int* error) {
  Ctl c = read_scalar(h->ws.ctl.p, h->stream);
  if (rep) {
    rep->iterations = c.it;
    rep->converged = c.converged;
    rep->zero_rhs = c.zero_b;
    rep->diverged = c.error == 3;
    rep->final_relres = c.rel;
  }
  *error = c.error;
}

template <class F>
int guarded(hcamg_handle* h, F&& f) {
  if (!h) return HCAMG_EINVAL;
  h->err.clear();
  h->err_index = -1;
  try {
    HC_CUDA(cudaSetDevice(h->device));
    OptionsScope os(&h->opts);
    PoolScope ps(h->pool);
    f();
    return HCAMG_OK;
  } catch (const Error& e) {
    h->err = e.what();
    h->err_index = e.index;
    cudaGetLastError();
    return e.code;
  } catch (const std::exception& e) {
    h->err = e.what();
    return HCAMG_ECUDA;
  }
}

// Distributed solve: a consumer that waited ~60 s for a peer flags the
// handle (the solve then finishes on stale data); report it as an error.
void check_dist(hcamg_handle* h) {
  if (rows_on(h)) {
    int e = 0;
    HC_CUDA(cudaMemcpyAsync(&e, h->rows->err.p, sizeof e, cudaMemcpyDeviceToHost, h->stream));
    HC_CUDA(cudaStreamSynchronize(h->stream));
    if (e) {
      h->rows->err.zero();
      throw Error(ECUDA_, e == 2 ? "row partition: a peer rank had not reached the boundary (lockstep emulation)"
                                 : "row partition: timed out waiting for a peer rank at a boundary");
    }
  }
  if (!h->dist.on) return;
  int e = 0;
  HC_CUDA(cudaMemcpyAsync(&e, h->dist.err.p, sizeof e, cudaMemcpyDeviceToHost, h->stream));
  HC_CUDA(cudaStreamSynchronize(h->stream));
  if (e) {
    h->dist.err.zero();
    throw Error(ECUDA_, "distributed solve: timed out waiting for a peer rank's exchange");
  }
}

int pcg_breakdown(hcamg_handle* h, int error) {
  if (error == kErrPAp) {
    Ctl c = read_scalar(h->ws.ctl.p, h->stream);
    char buf[160];
    snprintf(buf, sizeof buf, "PCG breakdown: p^T A p = %.3e (non-SPD operator)", c.pAp);
    throw Error(EBREAKDOWN_, buf);
  }
  if (error == kErrRz) throw Error(EBREAKDOWN_, "PCG breakdown: preconditioner is not SPD");
  return 0;
}

}  // namespace

// ============================================================================ C-ABI

extern "C" {

int hcamg_version(void) { return 1; }

int hcamg_create(hcamg_handle** out, int device, void* cuda_stream) {
  if (!out) return HCAMG_EINVAL;
  auto* h = new hcamg_handle();
  h->device = device;
  try {
    HC_CUDA(cudaSetDevice(device));
    if (cuda_stream) {
      h->stream = (cudaStream_t)cuda_stream;
    } else {
      HC_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
      h->own_stream = true;
    }
    HC_CUDA(cudaStreamCreateWithFlags(&h->aux, cudaStreamNonBlocking));
    h->opts = options_from_env();
    {
      // private stream-ordered pool: freed setup transients are reused within
      // a build without re-mapping (release threshold: never at sync) and
      // trimmed when the build ends; the device's default pool, which torch
      // and other libraries in the process use, is left untouched
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = device;
      HC_CUDA(cudaMemPoolCreate(&h->pool, &props));
      uint64_t thr = UINT64_MAX;
      HC_CUDA(cudaMemPoolSetAttribute(h->pool, cudaMemPoolAttrReleaseThreshold, &thr));
    }
  } catch (const Error& e) {
    fprintf(stderr, "hcamg_create: %s\n", e.what());
    delete h;
    *out = nullptr;
    return e.code;
  }
  *out = h;
  return HCAMG_OK;
}

void hcamg_destroy(hcamg_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->stream);
  invalidate(h);
  h->levels.clear();
  h->pending.clear();
  h->ws = Workspace();
  h->vc_b.release();
  h->vc_x.release();
  if (h->rows) drop_rows(h);
  h->dist.release();
  h->dist.ep.release();
  h->dist.cta.release();
  h->dist.err.release();
  cudaStreamSynchronize(h->stream);
  if (h->aux) cudaStreamDestroy(h->aux);
  if (h->own_stream) cudaStreamDestroy(h->stream);
  if (h->pool) {
    cudaMemPoolTrimTo(h->pool, 0);
    cudaMemPoolDestroy(h->pool);  // outstanding blocks (none expected) release it later
  }
  delete h;
}

const char* hcamg_last_error(const hcamg_handle* h) { return h ? h->err.c_str() : "null handle"; }

namespace {
struct OptKey {
  const char* name;
  double Options::*d;
  int Options::*i;
  int64_t Options::*l;
};
const OptKey kOptKeys[] = {
    {"sweep", nullptr, &Options::sweep, nullptr},
    {"giant_min", nullptr, nullptr, &Options::giant_min},
    {"coarse_gemv_min", nullptr, nullptr, &Options::coarse_gemv_min},
    {"coarse_symv", nullptr, &Options::coarse_symv, nullptr},
    {"factor_apply", nullptr, &Options::factor_apply, nullptr},
    {"form_z", nullptr, &Options::form_z, nullptr},
    {"tri_calib", nullptr, &Options::tri_calib, nullptr},
};
const OptKey* find_opt(const char* key) {
  if (!key) return nullptr;
  for (const OptKey& k : kOptKeys)
    if (!strcmp(k.name, key)) return &k;
  return nullptr;
}
}  // namespace

int hcamg_set_option(hcamg_handle* h, const char* key, double value) {
  return guarded(h, [&] {
    const OptKey* k = find_opt(key);
    require(k != nullptr, std::string("unknown option ") + (key ? key : "(null)"));
    require(!h->rows, "options cannot change while a row partition is attached (hcamg_rows_disconnect first)");
    if (k->i) {
      require(value == (double)(int)value, std::string("option ") + key + " takes an integer");
      if (k->i == &Options::sweep) {
        require(value >= SWEEP_AUTO && value <= SWEEP_FWAVE, "sweep mode out of range");
        if (value == SWEEP_FLOW || value == SWEEP_FWAVE)  // the dataflow terms are built on first request
          for (auto& l : h->levels)
            if (!l->coarsest && l->l1.p) build_flow(l->A, l->sm, h->stream);
      }
      h->opts.*(k->i) = (int)value;
    } else {
      require(value == (double)(int64_t)value, std::string("option ") + key + " takes an integer");
      h->opts.*(k->l) = (int64_t)value;
    }
    invalidate(h);  // recorded graphs embed the previous choices
  });
}

int hcamg_get_option(hcamg_handle* h, const char* key, double* value) {
  return guarded(h, [&] {
    const OptKey* k = find_opt(key);
    require(k != nullptr && value, std::string("unknown option ") + (key ? key : "(null)"));
    *value = k->i ? (double)(h->opts.*(k->i)) : (double)(h->opts.*(k->l));
  });
}
int64_t hcamg_error_index(const hcamg_handle* h) { return h ? h->err_index : -1; }
void* hcamg_stream(hcamg_handle* h) { return h ? (void*)h->stream : nullptr; }

int hcamg_setup_alg(hcamg_handle* h, const hcamg_csr* A, const hcamg_csr* G, int32_t max_levels, int64_t min_coarse,
                    double theta, hcamg_info* info) {
  return guarded(h, [&] {
    require(A && G, "A and G are required");
    build_hierarchy(h, A, G, 1, max_levels, min_coarse, theta, nullptr);
    fill_info(h, info);
  });
}

int hcamg_setup_ref(hcamg_handle* h, const hcamg_csr* A, const hcamg_csr* G, int32_t n_meshes, const int64_t* ne,
                    const int64_t* const* edges, const int64_t* const* children, const int64_t* free_edges,
                    int32_t max_levels, int64_t min_coarse, hcamg_info* info) {
  return guarded(h, [&] {
    require(A && G, "A and G are required");
    require(n_meshes >= 1 && ne && edges && free_edges && (n_meshes == 1 || children),
            "method 'ref' requires the nested mesh chain");
    RefChain c{n_meshes, ne, edges, children, free_edges};
    build_hierarchy(h, A, G, 0, max_levels, min_coarse, 0.25, &c);
    fill_info(h, info);
  });
}

int hcamg_hier_begin(hcamg_handle* h) {
  return guarded(h, [&] { h->pending.clear(); });
}

int hcamg_hier_push(hcamg_handle* h, const hcamg_csr* A, const hcamg_csr* G, const hcamg_csr* P) {
  return guarded(h, [&] {
    cudaStream_t s = h->stream;
    auto L = std::make_unique<DevLevel>();
    upload_csr(A, L->A, s);
    require(L->A.nrows == L->A.ncols, "A must be square");
    if (G) upload_csr(G, L->G, s);
    else { L->G.alloc(L->A.nrows, 0, 0, s); L->G.ptr.zero(); }
    if (P) {
      require(P->nrows == A->nrows, "P rows must match A");
      upload_csr(P, L->P, s);
      csr_transpose(L->P, L->Pt, s);
      L->has_P = true;
    }
    h->pending.push_back(std::move(L));
  });
}

// Coarsest level of a user-assembled hierarchy: coarse_matrix (if given) is
// the matrix whose Cholesky factor the user attached (Level.coarse_factor).
int hcamg_hier_end_with(hcamg_handle* h, const hcamg_csr* coarse_matrix, hcamg_info* info) {
  return guarded(h, [&] {
    require(!h->pending.empty(), "empty hierarchy");
    invalidate(h);
    h->levels = std::move(h->pending);
    h->pending.clear();
    h->notes.clear();
    h->stalled = false;
    h->method = 2;
    for (size_t i = 0; i + 1 < h->levels.size(); ++i)
      require(h->levels[i]->has_P, "only the last level may lack P");
    DevLevel& last = *h->levels.back();
    last.has_P = false;
    if (coarse_matrix) {
      upload_csr(coarse_matrix, last.cmat, h->stream);
      factor_coarsest(h, last, last.cmat);
    } else {
      factor_coarsest(h, last, last.A);
    }
    for (auto& l : h->levels) finish_level(h, *l);
    refresh_views(h);
    HC_CUDA(cudaStreamSynchronize(h->stream));
    fill_info(h, info);
  });
}

int hcamg_hier_end(hcamg_handle* h, hcamg_info* info) { return hcamg_hier_end_with(h, nullptr, info); }

int hcamg_split_alg(hcamg_handle* h, const hcamg_csr* A, const hcamg_csr* G, double theta, int64_t* sizes) {
  return guarded(h, [&] {
    require(A && G && sizes, "A, G and sizes are required");
    DCsr dA, dG;
    upload_csr(A, dA, h->stream);
    upload_csr(G, dG, h->stream);
    h->last_split = SplitResult();
    algebraic_splitting(dA, dG, theta, h->last_split, h->stream);
    sizes[0] = h->last_split.n_pairs();
    sizes[1] = (int64_t)h->last_split.interior.size();
    sizes[2] = (int64_t)h->last_split.coarse_nodes.size();
    sizes[3] = h->last_split.n_triples;
  });
}

int hcamg_split_export(hcamg_handle* h, int64_t* pairs, int64_t* interior, int64_t* coarse_nodes) {
  return guarded(h, [&] {
    const SplitResult& sp = h->last_split;
    if (pairs && !sp.pairs.empty()) memcpy(pairs, sp.pairs.data(), 8 * sp.pairs.size());
    if (interior && !sp.interior.empty()) memcpy(interior, sp.interior.data(), 8 * sp.interior.size());
    if (coarse_nodes && !sp.coarse_nodes.empty())
      memcpy(coarse_nodes, sp.coarse_nodes.data(), 8 * sp.coarse_nodes.size());
  });
}

int hcamg_info_get(hcamg_handle* h, hcamg_info* info) {
  return guarded(h, [&] { fill_info(h, info); });
}

int hcamg_notes(hcamg_handle* h, char* buf, int64_t cap) {
  return guarded(h, [&] {
    std::string all;
    for (size_t i = 0; i < h->notes.size(); ++i) all += (i ? "\n" : "") + h->notes[i];
    if (buf && cap > 0) {
      int64_t n = std::min<int64_t>(cap - 1, (int64_t)all.size());
      memcpy(buf, all.data(), (size_t)n);
      buf[n] = 0;
    }
  });
}

int hcamg_level(hcamg_handle* h, int32_t level, hcamg_level_info* o) {
  return guarded(h, [&] {
    require(level >= 0 && level < (int32_t)h->levels.size() && o, "level out of range");
    DevLevel& L = *h->levels[(size_t)level];
    memset(o, 0, sizeof *o);
    o->n = L.n;
    o->nnz_A = L.A.nnz;
    o->ncols_G = L.G.ncols;
    o->nnz_G = L.G.nnz;
    o->nnz_P = L.has_P ? (L.hp.on ? hybrid_nnz(L.P, L.hp, h->stream) : L.P.nnz) : 0;
    o->n_components = L.hp.on ? 1 : 0;
    o->max_component = L.hp.on ? L.hp.nG : 0;
    o->factor_bytes = L.hp.on && L.hp.fac.on ? L.hp.fac.fw.bytes + L.hp.fac.bw.bytes : 0;
    o->factor_steps = L.hp.on && L.hp.fac.on ? L.hp.fac.T : 0;
    o->factor_tma = L.hp.on && L.hp.fac.on && tri_tma_fits(L.hp.fac.fw) && tri_tma_fits(L.hp.fac.bw);
    o->pad = L.hp.on ? L.P.nnz : 0;  // nnz of the sparse part of a hybrid P
    o->n_pairs = L.split.n_pairs();
    o->n_interior = (int64_t)L.split.interior.size();
    o->n_coarse_nodes = (int64_t)(h->method == 0 ? L.split.pair_mesh_edges.size() : L.split.coarse_nodes.size());
    o->n_patches = L.sm.npatch;
    o->n_patch_entries = L.sm.h_patch_dofs.size();
    o->n_waves = L.sm.nwave;
    o->n_gc_cols = (int64_t)L.gc_cols.size();
    o->coarsest = L.coarsest;
  });
}

int hcamg_export_csr(hcamg_handle* h, int32_t level, int32_t which, int64_t* indptr, int32_t* indices, double* data) {
  return guarded(h, [&] {
    require(level >= 0 && level < (int32_t)h->levels.size(), "level out of range");
    DevLevel& L = *h->levels[(size_t)level];
    const DCsr* M = which == 0 ? &L.A : (which == 1 || which == 3) ? (L.has_P ? &L.P : nullptr) : &L.G;
    require(M != nullptr, "level has no P");
    if (which == 3) {  // sparse part of a hybrid P (the whole P otherwise)
      require(L.has_P, "level has no P");
      M = &L.P;
    }
    DCsr full;
    if (which == 1 && L.hp.on) {
      hybrid_ensure_z(L.hp, h->stream);
      hybrid_to_csr(L.P, L.hp, full, h->stream);
      M = &full;
    }
    cudaStream_t s = h->stream;
    if (indptr) HC_CUDA(cudaMemcpyAsync(indptr, M->ptr.p, 8 * (M->nrows + 1), cudaMemcpyDeviceToHost, s));
    if (M->nnz && indices) HC_CUDA(cudaMemcpyAsync(indices, M->idx.p, 4 * M->nnz, cudaMemcpyDeviceToHost, s));
    if (M->nnz && data) HC_CUDA(cudaMemcpyAsync(data, M->val.p, 8 * M->nnz, cudaMemcpyDeviceToHost, s));
    HC_CUDA(cudaStreamSynchronize(s));
  });
}

int hcamg_export_splitting(hcamg_handle* h, int32_t level, int64_t* pairs, int64_t* interior, int64_t* coarse_nodes) {
  return guarded(h, [&] {
    require(level >= 0 && level < (int32_t)h->levels.size(), "level out of range");
    const SplitResult& sp = h->levels[(size_t)level]->split;
    if (pairs && !sp.pairs.empty()) memcpy(pairs, sp.pairs.data(), 8 * sp.pairs.size());
    if (interior && !sp.interior.empty()) memcpy(interior, sp.interior.data(), 8 * sp.interior.size());
    const std::vector<int64_t>& cn = h->method == 0 ? sp.pair_mesh_edges : sp.coarse_nodes;
    if (coarse_nodes && !cn.empty()) memcpy(coarse_nodes, cn.data(), 8 * cn.size());
  });
}

int hcamg_export_dense(hcamg_handle* h, int32_t level, int32_t which, void* out) {
  return guarded(h, [&] {
    require(level >= 0 && level < (int32_t)h->levels.size(), "level out of range");
    DevLevel& L = *h->levels[(size_t)level];
    cudaStream_t s = h->stream;
    if (which == 0) {
      require(L.hp.on, "level has no dense interpolation block");
      hybrid_ensure_z(L.hp, s);
      HC_CUDA(cudaMemcpyAsync(out, L.hp.Z.p, 8 * L.hp.nG * L.hp.nc, cudaMemcpyDeviceToHost, s));
    } else if (which == 1) {
      require(L.hp.on, "level has no dense interpolation block");
      std::vector<int32_t> r((size_t)L.hp.nG);
      HC_CUDA(cudaMemcpyAsync(r.data(), L.hp.rows.p, 4 * L.hp.nG, cudaMemcpyDeviceToHost, s));
      HC_CUDA(cudaStreamSynchronize(s));
      for (int64_t q = 0; q < L.hp.nG; ++q) static_cast<int64_t*>(out)[q] = r[(size_t)q];
    } else if (which == 2) {
      require(L.coarsest && L.Ainv.p, "not the coarsest level");
      HC_CUDA(cudaMemcpyAsync(out, L.Ainv.p, 8 * L.n * L.n, cudaMemcpyDeviceToHost, s));
    } else {
      require(false, "unknown dense export");
    }
    HC_CUDA(cudaStreamSynchronize(s));
  });
}

int hcamg_component_solve(hcamg_handle* h, int32_t level, const double* v, double* out) {
  return guarded(h, [&] {
    require(level >= 0 && level < (int32_t)h->levels.size(), "level out of range");
    DevLevel& L = *h->levels[(size_t)level];
    require(L.hp.on && L.hp.fac.on, "level has no factored interpolation block");
    FactorP& f = L.hp.fac;
    cudaStream_t s = h->stream;
    std::vector<int32_t> perm = f.perm.download();
    std::vector<double> hv((size_t)factorp_npad(f), 0.0);
    for (int64_t i = 0; i < f.nG; ++i) hv[(size_t)i] = v[perm[(size_t)i]];
    HC_CUDA(cudaMemcpyAsync(f.v0.p, hv.data(), 8 * hv.size(), cudaMemcpyHostToDevice, s));
    DBuf<int> stop(1, s);
    stop.zero();
    factorp_solve(stop.p, f, f.v0.p, f.v2.p, s);
    HC_CUDA(cudaMemcpyAsync(hv.data(), f.v2.p, 8 * hv.size(), cudaMemcpyDeviceToHost, s));
    HC_CUDA(cudaStreamSynchronize(s));
    for (int64_t i = 0; i < f.nG; ++i) out[perm[(size_t)i]] = hv[(size_t)i];
  });
}

int hcamg_kuhn_assemble(hcamg_handle* h, int64_t n, const double* muinv, double beta, const double* S6,
                        const double* M6, int64_t* sizes) {
  return guarded(h, [&] {
    require(muinv && S6 && M6 && sizes, "null argument");
    require(beta >= 0, "shift must be nonnegative");
    kuhn_assemble(n, muinv, beta, S6, M6, h->kuhn_A, h->kuhn_G, h->kuhn_fe, h->kuhn_fv, h->stream);
    sizes[0] = h->kuhn_A.nrows;
    sizes[1] = h->kuhn_A.nnz;
    sizes[2] = h->kuhn_G.ncols;
    sizes[3] = h->kuhn_G.nnz;
    sizes[4] = (int64_t)h->kuhn_fe.size();
    sizes[5] = (int64_t)h->kuhn_fv.size();
  });
}

int hcamg_kuhn_export(hcamg_handle* h, int64_t* a_ptr, int32_t* a_idx, double* a_val, int64_t* g_ptr, int32_t* g_idx,
                      double* g_val, int64_t* free_edges, int64_t* free_nodes) {
  return guarded(h, [&] {
    require(h->kuhn_A.nrows > 0, "no assembled system (call hcamg_kuhn_assemble first)");
    cudaStream_t s = h->stream;
    const DCsr& A = h->kuhn_A;
    const DCsr& G = h->kuhn_G;
    HC_CUDA(cudaMemcpyAsync(a_ptr, A.ptr.p, 8 * (A.nrows + 1), cudaMemcpyDeviceToHost, s));
    if (A.nnz) HC_CUDA(cudaMemcpyAsync(a_idx, A.idx.p, 4 * A.nnz, cudaMemcpyDeviceToHost, s));
    if (A.nnz) HC_CUDA(cudaMemcpyAsync(a_val, A.val.p, 8 * A.nnz, cudaMemcpyDeviceToHost, s));
    HC_CUDA(cudaMemcpyAsync(g_ptr, G.ptr.p, 8 * (G.nrows + 1), cudaMemcpyDeviceToHost, s));
    if (G.nnz) HC_CUDA(cudaMemcpyAsync(g_idx, G.idx.p, 4 * G.nnz, cudaMemcpyDeviceToHost, s));
    if (G.nnz) HC_CUDA(cudaMemcpyAsync(g_val, G.val.p, 8 * G.nnz, cudaMemcpyDeviceToHost, s));
    HC_CUDA(cudaStreamSynchronize(s));
    if (free_edges) memcpy(free_edges, h->kuhn_fe.data(), 8 * h->kuhn_fe.size());
    if (free_nodes) memcpy(free_nodes, h->kuhn_fv.data(), 8 * h->kuhn_fv.size());
    h->kuhn_A = DCsr();
    h->kuhn_G = DCsr();
  });
}

int hcamg_export_l1(hcamg_handle* h, int32_t level, double* d) {
  return guarded(h, [&] {
    require(level >= 0 && level < (int32_t)h->levels.size(), "level out of range");
    DevLevel& L = *h->levels[(size_t)level];
    require(L.has_P, "coarsest level has no smoother");
    HC_CUDA(cudaMemcpyAsync(d, L.l1.p, 8 * L.n, cudaMemcpyDeviceToHost, h->stream));
    HC_CUDA(cudaStreamSynchronize(h->stream));
  });
}

int hcamg_export_patches(hcamg_handle* h, int32_t level, int64_t* ptr, int64_t* dofs, int64_t* wave) {
  return guarded(h, [&] {
    require(level >= 0 && level < (int32_t)h->levels.size(), "level out of range");
    const Smoother& sm = h->levels[(size_t)level]->sm;
    if (ptr) memcpy(ptr, sm.h_patch_ptr.data(), 8 * sm.h_patch_ptr.size());
    if (dofs && !sm.h_patch_dofs.empty()) memcpy(dofs, sm.h_patch_dofs.data(), 8 * sm.h_patch_dofs.size());
    if (wave) {
      for (int64_t w = 0; w < sm.nwave; ++w)
        for (int64_t t = sm.wave_ptr[(size_t)w]; t < sm.wave_ptr[(size_t)w + 1]; ++t) wave[sm.orig_of[(size_t)t]] = w;
    }
  });
}

int hcamg_export_coarse_cols(hcamg_handle* h, int32_t level, int64_t* cols) {
  return guarded(h, [&] {
    require(level >= 0 && level < (int32_t)h->levels.size(), "level out of range");
    const auto& c = h->levels[(size_t)level]->gc_cols;
    if (cols && !c.empty()) memcpy(cols, c.data(), 8 * c.size());
  });
}

int hcamg_coarse_solve(hcamg_handle* h, int32_t level, const double* b, double* x) {
  return guarded(h, [&] {
    require(level >= 0 && level < (int32_t)h->levels.size(), "level out of range");
    DevLevel& L = *h->levels[(size_t)level];
    require(L.coarsest, "level has no coarse factor");
    cudaStream_t s = h->stream;
    const int64_t n = L.n;
    if (!n) return;
    DBuf<double> db(n, s), dx(n, s);
    DBuf<int> stop(1, s);
    stop.zero();
    HC_CUDA(cudaMemcpyAsync(db.p, b, 8 * n, cudaMemcpyHostToDevice, s));
    dense_gemv_rows(stop.p, n, n, L.Ainv.p, db.p, dx.p, s);
    HC_CUDA(cudaMemcpyAsync(x, dx.p, 8 * n, cudaMemcpyDeviceToHost, s));
    HC_CUDA(cudaStreamSynchronize(s));
  });
}

int hcamg_cholesky_factor(hcamg_handle* h, int32_t level, int64_t* ordering, double* factor) {
  return guarded(h, [&] {
    require(level >= 0 && level < (int32_t)h->levels.size(), "level out of range");
    DevLevel& L = *h->levels[(size_t)level];
    require(L.coarsest, "level has no coarse factor");
    cudaStream_t s = h->stream;
    const DCsr& M = L.cmat.nrows ? L.cmat : L.A;
    const int64_t n = M.nrows;
    if (!n) return;
    std::vector<int64_t> hp = M.ptr.download();
    std::vector<int32_t> hi = M.idx.download();
    std::vector<int32_t> perm = rcm_order(n, hp, hi), inv((size_t)n);
    for (int64_t i = 0; i < n; ++i) inv[(size_t)perm[(size_t)i]] = (int32_t)i;
    DBuf<int32_t> dperm, dinv;
    dperm.upload(perm.data(), n, s);
    dinv.upload(inv.data(), n, s);
    DCsr Mp;
    csr_extract(M, dperm.p, n, dinv.p, n, Mp, s);
    DBuf<double> D(n * n, s);
    D.zero();
    k_densify<<<grid_for(n, 128), 128, 0, s>>>(Mp.ptr.p, Mp.idx.p, Mp.val.p, n, D.p);
    HC_CHECK_LAUNCH();
    const int64_t bad = dense_cholesky(D.p, n, n, s);
    if (bad >= 0) throw Error(ENOTSPD_, "matrix is not positive definite (pivot " + std::to_string(bad) + ")", bad);
    std::vector<double> hL = D.download();  // column-major, lower triangle valid
    for (int64_t i = 0; i < n; ++i) {
      if (ordering) ordering[i] = perm[(size_t)i];
      if (factor)
        for (int64_t j = 0; j < n; ++j) factor[i * n + j] = j <= i ? hL[(size_t)(i + j * n)] : 0.0;
    }
  });
}

int hcamg_smoother_setup(hcamg_handle* h, const hcamg_csr* A, const hcamg_csr* G) {
  return guarded(h, [&] {
    require(A && G, "A and G are required");
    cudaStream_t s = h->stream;
    invalidate(h);
    h->levels.clear();
    h->notes.clear();
    h->stalled = false;
    h->method = kSmootherOnly;
    auto L = std::make_unique<DevLevel>();
    upload_csr(A, L->A, s);
    upload_csr(G, L->G, s);
    require(L->A.nrows == L->A.ncols, "A must be square");
    require(L->G.nrows == L->A.nrows, "G rows must match A");
    L->n = L->A.nrows;
    alloc_level_vectors(*L, s);
    build_l1(L->A, L->l1, s);
    build_smoother(L->A, L->G, L->sm, s);
    h->levels.push_back(std::move(L));
    refresh_views(h);
    HC_CUDA(cudaStreamSynchronize(s));
  });
}

int hcamg_smooth(hcamg_handle* h, int32_t level, int32_t direction, const double* x_or_null, const double* b,
                 double* out) {
  return guarded(h, [&] {
    require(level >= 0 && level < (int32_t)h->levels.size(), "level out of range");
    require(direction >= 0 && direction <= 2, "unknown direction");
    DevLevel& L = *h->levels[(size_t)level];
    require(!L.coarsest && L.sm.npatch >= 0 && L.l1.p, "level has no smoother");
    cudaStream_t s = h->stream;
    const int64_t n = L.n;
    ensure_ws(h, 1);
    const int* stop = h->ws.zero_flag.p;
    DBuf<double> db(std::max<int64_t>(n, 1), s), dx(std::max<int64_t>(n, 1), s), rb(std::max<int64_t>(n, 1), s),
        dd(std::max<int64_t>(n, 1), s);
    if (n) HC_CUDA(cudaMemcpyAsync(db.p, b, 8 * n, cudaMemcpyHostToDevice, s));
    if (x_or_null && n) HC_CUDA(cudaMemcpyAsync(dx.p, x_or_null, 8 * n, cudaMemcpyHostToDevice, s));
    else dx.zero();
    // smooth(x, b) = x + S(0, b - A x) for either direction (the legs start
    // from x = 0; the residual is formed in scipy's rounding order, so a
    // fixed point x* with b = A x* (scipy) stays exactly fixed, as in the
    // reference's smoothers.py:122)
    for (int dir : {0, 1}) {
      if ((dir == 0 && direction == 1) || (dir == 1 && direction == 0)) continue;
      residual_scipy_order(L.A, dx.p, db.p, rb.p, s);
      if (dir == 0) {
        record_piece(PC_DOWN, L, nullptr, rb.p, dd.p, stop, s);
      } else {
        dd.zero();
        record_piece(PC_UP, L, nullptr, rb.p, dd.p, stop, s);
      }
      vec_add(n, dx.p, dd.p, dx.p, s);
    }
    if (n) HC_CUDA(cudaMemcpyAsync(out, dx.p, 8 * n, cudaMemcpyDeviceToHost, s));
    HC_CUDA(cudaStreamSynchronize(s));
  });
}

int hcamg_vcycle(hcamg_handle* h, const double* b, const double* x_or_null, double* out) {
  return guarded(h, [&] {
    require_hierarchy(h);
    cudaStream_t s = h->stream;
    const int64_t n = h->levels[0]->n;
    ensure_ws(h, 1);
    if (!h->g_vc.exec) {
      cudaGraph_t g;
      HC_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      h->g_vc.launches_pre = rows_on(h) ? rows_record(*h->rows, SEG_VCYCLE, h->lv, h->ws, h->ws.zero_flag.p, 0, s)
                                        : record_vcycle(h->lv, h->ws.r.p, h->ws.z.p, h->ws.zero_flag.p, s);
      HC_CUDA(cudaStreamEndCapture(s, &g));
      HC_CUDA(cudaGraphInstantiate(&h->g_vc.exec, g, 0));
      cudaGraphDestroy(g);
    }
    HC_CUDA(cudaMemcpyAsync(h->ws.b.p, b, 8 * n, cudaMemcpyHostToDevice, s));
    if (x_or_null) {
      // out = x + V(b - A x)  (multilevel.py:196)
      HC_CUDA(cudaMemcpyAsync(h->ws.x.p, x_or_null, 8 * n, cudaMemcpyHostToDevice, s));
      set_ctl(h, 1.0, 1);
      generic_init(h->levels[0]->A, h->ws, s);  // ws.r = b - A x
    } else {
      HC_CUDA(cudaMemcpyAsync(h->ws.r.p, h->ws.b.p, 8 * n, cudaMemcpyDeviceToDevice, s));
    }
    HC_CUDA(cudaGraphLaunch(h->g_vc.exec, s));
    if (x_or_null) vec_add(n, h->ws.x.p, h->ws.z.p, h->ws.z.p, s);
    HC_CUDA(cudaMemcpyAsync(out, h->ws.z.p, 8 * n, cudaMemcpyDeviceToHost, s));
    HC_CUDA(cudaStreamSynchronize(s));
    check_dist(h);
  });
}

static int pcg_impl(hcamg_handle* h, const double* b, bool b_dev, const double* x0, bool x0_dev, double tol,
                    int64_t maxit, double* x, bool x_dev, double* history, hcamg_report* report, bool sync) {
  return guarded(h, [&] {
    require_hierarchy(h);
    require(tol > 0, "tolerance must be positive");
    cudaStream_t s = h->stream;
    const int64_t n = h->levels[0]->n;
    prepare_loop(h, h->g_pcg, true, maxit);
    HC_CUDA(cudaMemcpyAsync(h->ws.b.p, b, 8 * n, b_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    if (x0) HC_CUDA(cudaMemcpyAsync(h->ws.x.p, x0, 8 * n, x0_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    else h->ws.x.zero();
    set_ctl(h, tol, maxit);
    run_loop_graph(h, h->g_pcg);
    zero_x_if_zero_rhs(h->ws, s);
    if (rows_on(h)) rows_record(*h->rows, SEG_GATHER, h->lv, h->ws, h->ws.zero_flag.p, 0, s);  // every rank gets all of x
    HC_CUDA(cudaMemcpyAsync(x, h->ws.x.p, 8 * n, x_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
    if (!sync && !report && !history) return;  // errors deferred: hcamg_solve_status
    int error = 0;
    hcamg_report rep{};
    read_report(h, &rep, &error);
    pcg_breakdown(h, error);
    if (history && rep.iterations)
      HC_CUDA(cudaMemcpyAsync(history, h->ws.hist.p, 8 * rep.iterations, cudaMemcpyDeviceToHost, s));
    HC_CUDA(cudaStreamSynchronize(s));
    check_dist(h);
    if (report) *report = rep;
  });
}

int hcamg_pcg(hcamg_handle* h, const double* b, const double* x0, double tol, int64_t maxit, double* x,
              double* history, hcamg_report* report) {
  return pcg_impl(h, b, false, x0, false, tol, maxit, x, false, history, report, true);
}

int hcamg_pcg_device(hcamg_handle* h, const double* d_b, const double* d_x0, double tol, int64_t maxit, double* d_x,
                     hcamg_report* report) {
  return pcg_impl(h, d_b, true, d_x0, true, tol, maxit, d_x, true, nullptr, report, report != nullptr);
}

int hcamg_amg_solve(hcamg_handle* h, const double* b, const double* x0, double tol, int64_t maxit, double* x,
                    double* history, hcamg_report* report) {
  return guarded(h, [&] {
    require_hierarchy(h);
    require(tol > 0, "tolerance must be positive");
    cudaStream_t s = h->stream;
    const int64_t n = h->levels[0]->n;
    prepare_loop(h, h->g_amg, false, maxit);
    HC_CUDA(cudaMemcpyAsync(h->ws.b.p, b, 8 * n, cudaMemcpyHostToDevice, s));
    if (x0) HC_CUDA(cudaMemcpyAsync(h->ws.x.p, x0, 8 * n, cudaMemcpyHostToDevice, s));
    else h->ws.x.zero();
    set_ctl(h, tol, maxit);
    run_loop_graph(h, h->g_amg);
    zero_x_if_zero_rhs(h->ws, s);
    if (rows_on(h)) rows_record(*h->rows, SEG_GATHER, h->lv, h->ws, h->ws.zero_flag.p, 0, s);
    HC_CUDA(cudaMemcpyAsync(x, h->ws.x.p, 8 * n, cudaMemcpyDeviceToHost, s));
    int error = 0;
    hcamg_report rep{};
    read_report(h, &rep, &error);
    if (history && rep.iterations)
      HC_CUDA(cudaMemcpyAsync(history, h->ws.hist.p, 8 * rep.iterations, cudaMemcpyDeviceToHost, s));
    HC_CUDA(cudaStreamSynchronize(s));
    check_dist(h);
    if (report) *report = rep;
  });
}

int hcamg_solve_status(hcamg_handle* h, hcamg_report* report) {
  return guarded(h, [&] {
    require_hierarchy(h);
    require(h->ws.ctl.p != nullptr, "no solve has run on this handle");
    int error = 0;
    hcamg_report rep{};
    read_report(h, &rep, &error);
    if (report) *report = rep;
    pcg_breakdown(h, error);
    check_dist(h);
  });
}

int64_t hcamg_graph_launches(hcamg_handle* h, int32_t which) {
  if (!h) return -1;
  if (which == 0) return h->g_vc.launches_pre;
  if (which == 1) return h->g_pcg.launches_pre;
  if (which == 2) return h->g_pcg.launches_body;
  if (which == 3) return h->g_amg.launches_pre;
  if (which == 4) return h->g_amg.launches_body;
  return -1;
}

int hcamg_profile_vcycle(hcamg_handle* h, int32_t reps, int32_t cap, int32_t* kind, int32_t* level, double* us,
                         int64_t* launches, int32_t* count) {
  return guarded(h, [&] {
    require_hierarchy(h);
    require(reps > 0, "reps must be positive");
    cudaStream_t s = h->stream;
    ensure_ws(h, 1);
    cudaEvent_t e0, e1;
    HC_CUDA(cudaEventCreate(&e0));
    HC_CUDA(cudaEventCreate(&e1));
    int32_t k = 0;
    const int* stop = h->ws.zero_flag.p;
    for (size_t ell = 0; ell < h->lv.size(); ++ell) {
      DevLevel& L = *h->lv[ell];
      DevLevel* C = ell + 1 < h->lv.size() ? h->lv[ell + 1] : nullptr;
      const double* b = ell == 0 ? h->ws.r.p : L.b.p;
      double* x = ell == 0 ? h->ws.z.p : L.x.p;
      const int pcs_fine[] = {PC_DOWN, PC_RESTRICT, PC_PROLONG, PC_UP};
      const int pcs_coarse[] = {PC_COARSE};
      const int* pcs = L.coarsest ? pcs_coarse : pcs_fine;
      const int npc = L.coarsest ? 1 : 4;
      for (int t = 0; t < npc && k < cap; ++t) {
        int64_t nl = 0;
        for (int wv = 0; wv < 2; ++wv) nl = record_piece(pcs[t], L, C, b, x, stop, s);
        HC_CUDA(cudaEventRecord(e0, s));
        for (int r = 0; r < reps; ++r) record_piece(pcs[t], L, C, b, x, stop, s);
        HC_CUDA(cudaEventRecord(e1, s));
        HC_CUDA(cudaEventSynchronize(e1));
        float ms = 0;
        HC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        kind[k] = pcs[t];
        level[k] = (int32_t)ell;
        us[k] = 1e3 * ms / reps;
        launches[k] = nl;
        ++k;
      }
    }
    *count = k;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

// Debug (not in the public header): record per-phase timestamps of one
// level-0 down leg into host buffer `out` (phases x warps x 2 int64).
int hcamg_debug_trace_leg(hcamg_handle* h, int down, long long* out, int64_t cap) {
  return guarded(h, [&] {
    require_hierarchy(h);
    cudaStream_t s = h->stream;
    ensure_ws(h, 1);
    DBuf<long long> tr(cap, s);
    tr.zero();
    hcamg::g_leg_trace = tr.p;
    DevLevel& L = *h->lv[0];
    DevLevel* C = h->lv.size() > 1 ? h->lv[1] : nullptr;
    for (int r = 0; r < 3; ++r) record_piece(down ? PC_DOWN : PC_UP, L, C, h->ws.r.p, h->ws.z.p, h->ws.zero_flag.p, s);
    hcamg::g_leg_trace = nullptr;
    HC_CUDA(cudaMemcpyAsync(out, tr.p, sizeof(long long) * cap, cudaMemcpyDeviceToHost, s));
    HC_CUDA(cudaStreamSynchronize(s));
  });
}

int hcamg_spmv(hcamg_handle* h, const hcamg_csr* A, const double* x, double* y) {
  return guarded(h, [&] {
    cudaStream_t s = h->stream;
    DCsr M;
    upload_csr(A, M, s);
    DBuf<double> dx(std::max<int64_t>(M.ncols, 1), s), dy(std::max<int64_t>(M.nrows, 1), s);
    if (M.ncols) HC_CUDA(cudaMemcpyAsync(dx.p, x, 8 * M.ncols, cudaMemcpyHostToDevice, s));
    dy.zero();
    if (M.nrows) apply_operator(M, dx.p, dy.p, s);
    if (M.nrows) HC_CUDA(cudaMemcpyAsync(y, dy.p, 8 * M.nrows, cudaMemcpyDeviceToHost, s));
    HC_CUDA(cudaStreamSynchronize(s));
  });
}

// Debug (not in the public header): C = A B with the library's SpGEMM (scipy
// csr_matmat order, canonical output).  *nnz receives nnz(C); when indptr is
// non-null and cap >= nnz(C) the product is copied out.  Tests use it to hold
// every SpGEMM path (row kernels, dense-left) against scipy bit for bit.
int hcamg_debug_spgemm(hcamg_handle* h, const hcamg_csr* A, const hcamg_csr* B, int64_t* nnz, int64_t* indptr,
                       int32_t* indices, double* data, int64_t cap) {
  return guarded(h, [&] {
    cudaStream_t s = h->stream;
    DCsr Ma, Mb, Mc;
    upload_csr(A, Ma, s);
    upload_csr(B, Mb, s);
    spgemm(Ma, Mb, Mc, s);
    require(nnz != nullptr, "nnz output missing");
    *nnz = Mc.nnz;
    if (indptr && cap >= Mc.nnz) {
      HC_CUDA(cudaMemcpyAsync(indptr, Mc.ptr.p, 8 * (Mc.nrows + 1), cudaMemcpyDeviceToHost, s));
      if (Mc.nnz) {
        HC_CUDA(cudaMemcpyAsync(indices, Mc.idx.p, 4 * Mc.nnz, cudaMemcpyDeviceToHost, s));
        HC_CUDA(cudaMemcpyAsync(data, Mc.val.p, 8 * Mc.nnz, cudaMemcpyDeviceToHost, s));
      }
    }
    HC_CUDA(cudaStreamSynchronize(s));
  });
}

int hcamg_pcg_generic(hcamg_handle* h, const hcamg_csr* A, const double* b, const double* x0, double tol,
                      int64_t maxit, hcamg_precond_fn precond, void* ctx, double* x, double* history,
                      hcamg_report* report) {
  return guarded(h, [&] {
    require(tol > 0, "tolerance must be positive");
    require(A && A->nrows == A->ncols, "A must be square");
    cudaStream_t s = h->stream;
    DCsr M;
    upload_csr(A, M, s);
    const int64_t n = M.nrows;
    Workspace& w = h->ws;
    invalidate(h);
    w.ensure(n, std::max<int64_t>(maxit, 1), s);
    HC_CUDA(cudaMemcpyAsync(w.b.p, b, 8 * n, cudaMemcpyHostToDevice, s));
    if (x0) HC_CUDA(cudaMemcpyAsync(w.x.p, x0, 8 * n, cudaMemcpyHostToDevice, s));
    else w.x.zero();
    set_ctl(h, tol, maxit);
    generic_init(M, w, s);
    Ctl c = read_scalar(w.ctl.p, s);
    hcamg_report rep{};
    std::vector<double> hr((size_t)n), hz((size_t)n);
    auto call_precond = [&]() {
      HC_CUDA(cudaMemcpyAsync(hr.data(), w.r.p, 8 * n, cudaMemcpyDeviceToHost, s));
      HC_CUDA(cudaStreamSynchronize(s));
      if (precond(hr.data(), hz.data(), n, ctx) != 0) throw Error(EINVAL_, "preconditioner callback failed");
      HC_CUDA(cudaMemcpyAsync(w.z.p, hz.data(), 8 * n, cudaMemcpyHostToDevice, s));
    };
    if (!c.stop) {
      call_precond();
      generic_rz(w, true, s);
      for (;;) {
        generic_pap(M, w, s);
        c = read_scalar(w.ctl.p, s);
        if (c.error) break;
        generic_update(w, s);
        c = read_scalar(w.ctl.p, s);
        if (c.stop) break;
        call_precond();
        generic_rz(w, false, s);
        c = read_scalar(w.ctl.p, s);
        if (c.error) break;
        generic_p(w, s);
      }
    }
    rep.iterations = c.it;
    rep.converged = c.converged;
    rep.zero_rhs = c.zero_b;
    rep.final_relres = c.rel;
    pcg_breakdown(h, c.error);
    HC_CUDA(cudaMemcpyAsync(x, w.x.p, 8 * n, cudaMemcpyDeviceToHost, s));
    if (history && c.it) HC_CUDA(cudaMemcpyAsync(history, w.hist.p, 8 * c.it, cudaMemcpyDeviceToHost, s));
    HC_CUDA(cudaStreamSynchronize(s));
    if (rep.zero_rhs) memset(x, 0, 8 * n);
    if (report) *report = rep;
  });
}

// ---- row-partitioned solve across processes (dist.cuh)

static void dist_attach(hcamg_handle* h) {
  for (DevLevel* L : h->lv) L->dist = &h->dist;
  h->dist.on = true;
  invalidate(h);
}

int hcamg_dist_prepare(hcamg_handle* h, int32_t rank, int32_t nranks, void* ipc_handle, void** dev_ptr) {
  return guarded(h, [&] {
    require_hierarchy(h);
    require(nranks >= 1 && nranks <= kMaxRanks, "nranks must be in 1..8");
    require(rank >= 0 && rank < nranks, "rank out of range");
    cudaStream_t s = h->stream;
    HC_CUDA(cudaStreamSynchronize(s));
    Dist& d = h->dist;
    d.release();
    for (DevLevel* L : h->lv) L->dist = nullptr;
    invalidate(h);
    d.rank = rank;
    d.nranks = nranks;
    // exchange sites of every level, 256-byte aligned, identical on all ranks
    size_t off = 0;
    auto take = [&](int64_t nd) {
      const size_t o = off;
      off += ((size_t)std::max<int64_t>(nd, 1) * 8 + 255) / 256 * 256;
      return o;
    };
    // Representation per N: a piece is split across the
    // ranks only when its per-rank bytes beat the single-GPU representation --
    // the dense block: 2 x 8 nG nc / N (row blocks of Z, restriction + prolongation)
    // against 2 x the envelope-factor sweeps; the coarsest solve: 8 n^2 / N (rows
    // of the inverse) against the packed lower triangle (8 n^2 / 2).  Pieces that
    // are not split run replicated on every rank with the single-GPU kernels.
    for (DevLevel* L : h->lv) {
      L->xoff_g = L->xoff_y = L->xoff_c = DevLevel::kNoSite;
      if (L->hp.on) {
        const double z_rank = 2.0 * 8.0 * (double)L->hp.nG * (double)L->hp.nc / nranks;
        const double fac = L->hp.fac.on ? 2.0 * (double)(L->hp.fac.fw.bytes + L->hp.fac.bw.bytes) : 1e300;
        if (z_rank < fac) {
          hybrid_ensure_z(L->hp, s);  // ranks stream row blocks of the explicit Z
          L->xoff_g = take(kGroups * L->hp.nc);
          L->xoff_y = take(L->hp.nG);
        }
      }
      if (L->coarsest && L->n >= coarse_gemv_min()) {
        const double rows = 8.0 * (double)L->n * (double)L->n / nranks;
        const double packed = L->Asym.on ? 4.0 * (double)L->n * (double)L->n : 1e300;
        if (rows < packed) L->xoff_c = take(L->n);
      }
    }
    d.area_bytes = std::max<size_t>(off, 256);
    d.sym_bytes = kFlagBytes + 2 * d.area_bytes;
    HC_CUDA(cudaMalloc(&d.sym, d.sym_bytes));  // not pool memory: exported through CUDA IPC
    HC_CUDA(cudaMemset(d.sym, 0, d.sym_bytes));
    if (!d.ep.p) {
      d.ep.alloc(1, s);
      d.cta.alloc(1, s);
      d.err.alloc(1, s);
    }
    d.ep.zero();
    d.cta.zero();
    d.err.zero();
    HC_CUDA(cudaStreamSynchronize(s));
    if (ipc_handle) {
      cudaIpcMemHandle_t mh;
      HC_CUDA(cudaIpcGetMemHandle(&mh, d.sym));
      memcpy(ipc_handle, &mh, sizeof mh);
    }
    if (dev_ptr) *dev_ptr = d.sym;
  });
}

int hcamg_dist_connect(hcamg_handle* h, const void* ipc_handles) {
  return guarded(h, [&] {
    Dist& d = h->dist;
    require(d.sym != nullptr, "hcamg_dist_prepare must be called first");
    require(ipc_handles != nullptr, "missing peer handles");
    for (int r = 0; r < d.nranks; ++r) {
      if (r == d.rank) {
        d.base[r] = d.sym;
        continue;
      }
      cudaIpcMemHandle_t mh;
      memcpy(&mh, static_cast<const char*>(ipc_handles) + (size_t)r * sizeof mh, sizeof mh);
      void* p = nullptr;
      HC_CUDA(cudaIpcOpenMemHandle(&p, mh, cudaIpcMemLazyEnablePeerAccess));
      d.base[r] = static_cast<char*>(p);
      d.opened[r] = true;
    }
    dist_attach(h);
  });
}

int hcamg_dist_connect_ptrs(hcamg_handle* h, void* const* bufs) {
  return guarded(h, [&] {
    Dist& d = h->dist;
    require(d.sym != nullptr, "hcamg_dist_prepare must be called first");
    require(bufs != nullptr, "missing peer buffers");
    for (int r = 0; r < d.nranks; ++r) {
      require(bufs[r] != nullptr, "null peer buffer");
      d.base[r] = static_cast<char*>(bufs[r]);
    }
    require(d.base[d.rank] == d.sym, "bufs[rank] must be this handle's own buffer");
    dist_attach(h);
  });
}

int hcamg_dist_disconnect(hcamg_handle* h) {
  return guarded(h, [&] {
    HC_CUDA(cudaStreamSynchronize(h->stream));
    h->dist.release();
    for (DevLevel* L : h->lv) L->dist = nullptr;
    invalidate(h);
  });
}

int hcamg_dist_info(hcamg_handle* h, int32_t* rank, int32_t* nranks, int32_t* connected, int64_t* buffer_bytes) {
  return guarded(h, [&] {
    if (rank) *rank = h->dist.rank;
    if (nranks) *nranks = h->dist.nranks;
    if (connected) *connected = h->dist.on ? 1 : 0;
    if (buffer_bytes) *buffer_bytes = (int64_t)h->dist.sym_bytes;
  });
}

// Debug (not in the public header): run one piece (or one half of a piece,
// `part` 1 = up to its exchange signal, 2 = from its wait on) of the V-cycle
// of level `level` on the V-cycle buffers; b (host, level-0 input) is loaded
// first when given, x (host) receives the level-0 result when given.  Lets a
// test emulate several ranks on one GPU: every rank's part 1, then every
// rank's part 2, so no kernel ever waits on a kernel that has not run.
int hcamg_debug_dist_piece(hcamg_handle* h, int32_t level, int32_t piece, int32_t part, const double* b, double* x) {
  return guarded(h, [&] {
    require_hierarchy(h);
    require(level >= 0 && level < (int32_t)h->lv.size(), "level out of range");
    require(part >= 0 && part <= 2, "part must be 0, 1 or 2");
    cudaStream_t s = h->stream;
    ensure_ws(h, 1);
    const int64_t n = h->levels[0]->n;
    if (b) HC_CUDA(cudaMemcpyAsync(h->ws.r.p, b, 8 * n, cudaMemcpyHostToDevice, s));
    DevLevel& L = *h->lv[(size_t)level];
    DevLevel* C = (size_t)level + 1 < h->lv.size() ? h->lv[(size_t)level + 1] : nullptr;
    const double* bb = level == 0 ? h->ws.r.p : L.b.p;
    double* xx = level == 0 ? h->ws.z.p : L.x.p;
    if (piece >= 0) record_piece(piece, L, C, bb, xx, h->ws.zero_flag.p, s, part);
    if (x) HC_CUDA(cudaMemcpyAsync(x, h->ws.z.p, 8 * n, cudaMemcpyDeviceToHost, s));
    HC_CUDA(cudaStreamSynchronize(s));
    check_dist(h);
  });
}

// Debug (not in the public header): the interpolation of level `level` as the
// V-cycle applies it (record_piece): kind 0: out = P in (in: n_c, out: n);
// kind 1: out = P^T in (in: n, out: n_c).  Host buffers.
int hcamg_debug_apply_p(hcamg_handle* h, int32_t level, int32_t kind, const double* in, double* out) {
  return guarded(h, [&] {
    require_hierarchy(h);
    require(level >= 0 && level + 1 < (int32_t)h->lv.size(), "level has no interpolation");
    cudaStream_t s = h->stream;
    ensure_ws(h, 1);
    DevLevel& L = *h->lv[(size_t)level];
    DevLevel* C = h->lv[(size_t)level + 1];
    if (kind == 0) {
      DBuf<double> x(L.n, s);
      x.zero();
      HC_CUDA(cudaMemcpyAsync(C->x.p, in, 8 * C->n, cudaMemcpyHostToDevice, s));
      record_piece(PC_PROLONG, L, C, nullptr, x.p, h->ws.zero_flag.p, s, 0);
      HC_CUDA(cudaMemcpyAsync(out, x.p, 8 * L.n, cudaMemcpyDeviceToHost, s));
    } else {
      HC_CUDA(cudaMemcpyAsync(L.r.p, in, 8 * L.n, cudaMemcpyHostToDevice, s));
      record_piece(PC_RESTRICT, L, C, nullptr, nullptr, h->ws.zero_flag.p, s, 0);
      HC_CUDA(cudaMemcpyAsync(out, C->b.p, 8 * C->n, cudaMemcpyDeviceToHost, s));
    }
    HC_CUDA(cudaStreamSynchronize(s));
  });
}


// ---- subdomain row partition (rows.cuh)

int hcamg_rows_prepare(hcamg_handle* h, int32_t rank, int32_t nranks, int64_t min_rows, void* ipc_handle,
                       void** dev_ptr) {
  return guarded(h, [&] {
    require_hierarchy(h);
    cudaStream_t s = h->stream;
    HC_CUDA(cudaStreamSynchronize(s));
    if (h->rows) drop_rows(h);
    h->dist.release();
    for (DevLevel* L : h->lv) L->dist = nullptr;
    ensure_ws(h, 1);
    invalidate(h);
    h->rows.reset(new RowsCtx());
    try {
      rows_prepare(*h->rows, h->lv, h->ws, rank, nranks, min_rows, s);
    } catch (...) {
      drop_rows(h);
      throw;
    }
    if (ipc_handle) {
      cudaIpcMemHandle_t mh;
      HC_CUDA(cudaIpcGetMemHandle(&mh, h->rows->sym));
      memcpy(ipc_handle, &mh, sizeof mh);
    }
    if (dev_ptr) *dev_ptr = h->rows->sym;
  });
}

int hcamg_rows_connect(hcamg_handle* h, const void* ipc_handles) {
  return guarded(h, [&] {
    require(h->rows && h->rows->sym, "hcamg_rows_prepare must be called first");
    require(ipc_handles != nullptr, "missing peer handles");
    RowsCtx& rc = *h->rows;
    for (int r = 0; r < rc.nranks; ++r) {
      if (r == rc.rank) {
        rc.base[r] = rc.sym;
        continue;
      }
      cudaIpcMemHandle_t mh;
      memcpy(&mh, static_cast<const char*>(ipc_handles) + (size_t)r * sizeof mh, sizeof mh);
      void* p = nullptr;
      HC_CUDA(cudaIpcOpenMemHandle(&p, mh, cudaIpcMemLazyEnablePeerAccess));
      rc.base[r] = static_cast<char*>(p);
      rc.opened[r] = true;
    }
    rc.on = true;
    invalidate(h);
  });
}

int hcamg_rows_connect_ptrs(hcamg_handle* h, void* const* bufs) {
  return guarded(h, [&] {
    require(h->rows && h->rows->sym, "hcamg_rows_prepare must be called first");
    require(bufs != nullptr, "missing peer buffers");
    RowsCtx& rc = *h->rows;
    for (int r = 0; r < rc.nranks; ++r) {
      require(bufs[r] != nullptr, "null peer buffer");
      rc.base[r] = static_cast<char*>(bufs[r]);
    }
    require(rc.base[rc.rank] == rc.sym, "bufs[rank] must be this handle's own buffer");
    rc.on = true;
    invalidate(h);
  });
}

int hcamg_rows_disconnect(hcamg_handle* h) {
  return guarded(h, [&] {
    HC_CUDA(cudaStreamSynchronize(h->stream));
    if (h->rows) drop_rows(h);
    invalidate(h);
  });
}

// out[0..]: rank, nranks, connected, split levels, buffer bytes, owned rows of
// level 0, ghost columns of level 0, then per segment (V-cycle, init, first,
// body, gather): steps, barriers, entries this rank pushes, entries all ranks push
int hcamg_rows_info(hcamg_handle* h, int64_t* out, int32_t cap) {
  return guarded(h, [&] {
    require(h->rows != nullptr, "no row partition on this handle");
    const RowsCtx& rc = *h->rows;
    std::vector<int64_t> v = {rc.rank, rc.nranks, rc.on ? 1 : 0, rc.stats.split_levels, (int64_t)rc.sym_bytes,
                              rc.stats.own_rows0, rc.stats.ghost_rows0};
    for (int g = 0; g < SEG_COUNT; ++g) {
      v.push_back(rc.stats.boundaries[g]);
      v.push_back(rc.stats.barriers[g]);
      v.push_back(rc.stats.push_out[g]);
      v.push_back(rc.stats.push_all[g]);
    }
    for (int32_t i = 0; i < cap && i < (int32_t)v.size(); ++i) out[i] = v[(size_t)i];
  });
}

namespace {

struct HandleScope {  // what guarded() installs, for a loop over several handles
  OptionsScope os;
  PoolScope ps;
  explicit HandleScope(hcamg_handle* h) : os(&h->opts), ps(h->pool) {}
};

// every rank's boundary k (push + signal), then every rank's check + step k:
// no kernel ever waits for a kernel that has not run
void lockstep(hcamg_handle* const* hs, int n, int g, bool use_stop) {
  const size_t steps = hs[0]->rows->seg[g].size();
  for (size_t k = 0; k < steps; ++k) {
    for (int r = 0; r < n; ++r) {
      HandleScope sc(hs[r]);
      const int* stop = use_stop ? &hs[r]->ws.ctl.p->stop : hs[r]->ws.zero_flag.p;
      rows_boundary(*hs[r]->rows, g, k, stop, false, hs[r]->stream);
    }
    HC_CUDA(cudaDeviceSynchronize());
    for (int r = 0; r < n; ++r) {
      HandleScope sc(hs[r]);
      const int* stop = use_stop ? &hs[r]->ws.ctl.p->stop : hs[r]->ws.zero_flag.p;
      const int32_t b = hs[r]->rows->seg_boundary[g][k];
      if (hs[r]->rows->barrier[(size_t)b]) rows_wait(*hs[r]->rows, stop, hs[r]->stream);
      rows_launch_step(hs[r]->rows->seg[g][k], *hs[r]->rows, hs[r]->lv, hs[r]->ws, stop, 0, hs[r]->stream);
    }
    HC_CUDA(cudaDeviceSynchronize());
  }
}

}  // namespace

// Lockstep emulation of an n-rank partitioned solve on ONE GPU (tests): hs are
// n handles of this process holding the same hierarchy, prepared as ranks
// 0..n-1 and connected with each other's buffers (hcamg_rows_connect_ptrs).
// kind 0: V-cycle z = V(b); kind 1: PCG from x0 = 0.  b: n0 doubles (host);
// x: n x n0 doubles (host), row r = the full result as rank r holds it.
// `poison` != 0 fills every working vector with NaN first, so an entry that
// was neither computed nor received shows up in the result.
int hcamg_rows_emulate(hcamg_handle* const* hs, int32_t n, int32_t kind, const double* b, double* x, double tol,
                       int64_t maxit, int32_t poison, hcamg_report* report) {
  if (!hs || n < 1 || !hs[0]) return HCAMG_EINVAL;
  return guarded(hs[0], [&] {
    for (int r = 0; r < n; ++r) {
      require(hs[r] && rows_on(hs[r]), "every handle must hold a connected row partition");
      require(hs[r]->rows->nranks == n && hs[r]->rows->rank == r, "handles must be ranks 0..n-1 of an n-rank partition");
      require(hs[r]->device == hs[0]->device, "lockstep emulation runs on one GPU");
    }
    const int64_t n0 = hs[0]->levels[0]->n;
    for (int r = 0; r < n; ++r) {
      HandleScope sc(hs[r]);
      hcamg_handle* h = hs[r];
      ensure_ws(h, std::max<int64_t>(maxit, 1));
      cudaStream_t s = h->stream;
      if (poison) {
        RowsCtx& rc = *h->rows;
        HC_CUDA(cudaMemsetAsync(rc.sym + kRowsFlagBytes, 0xff, rc.sym_bytes - kRowsFlagBytes, s));
      }
      require(kind >= 0 && kind <= 2, "kind: 0 V-cycle, 1 PCG, 2 stand-alone AMG iteration");
      if (kind == 0) {
        HC_CUDA(cudaMemcpyAsync(h->ws.r.p, b, 8 * n0, cudaMemcpyHostToDevice, s));
      } else {
        HC_CUDA(cudaMemcpyAsync(h->ws.b.p, b, 8 * n0, cudaMemcpyHostToDevice, s));
        h->ws.x.zero();
        set_ctl(h, tol, maxit);
      }
    }
    HC_CUDA(cudaDeviceSynchronize());
    if (kind == 0) {
      lockstep(hs, n, SEG_VCYCLE, false);
      for (int r = 0; r < n; ++r)
        HC_CUDA(cudaMemcpy(x + (size_t)r * n0, hs[r]->ws.z.p, 8 * n0, cudaMemcpyDeviceToHost));
    } else {
      if (kind == 1) {
        lockstep(hs, n, SEG_INIT, true);
        lockstep(hs, n, SEG_FIRST, true);
      } else {
        lockstep(hs, n, SEG_AMG_INIT, true);
      }
      while (true) {
        int stop0 = read_scalar(&hs[0]->ws.ctl.p->stop, hs[0]->stream);
        for (int r = 1; r < n; ++r)
          require(read_scalar(&hs[r]->ws.ctl.p->stop, hs[r]->stream) == stop0, "ranks disagree on convergence");
        if (stop0) break;
        lockstep(hs, n, kind == 1 ? SEG_BODY : SEG_AMG_BODY, true);
      }
      for (int r = 0; r < n; ++r) {
        HandleScope sc(hs[r]);
        zero_x_if_zero_rhs(hs[r]->ws, hs[r]->stream);
      }
      HC_CUDA(cudaDeviceSynchronize());
      lockstep(hs, n, SEG_GATHER, false);
      for (int r = 0; r < n; ++r)
        HC_CUDA(cudaMemcpy(x + (size_t)r * n0, hs[r]->ws.x.p, 8 * n0, cudaMemcpyDeviceToHost));
      int error = 0;
      hcamg_report rep{};
      read_report(hs[0], &rep, &error);
      for (int r = 1; r < n; ++r) {
        int e2 = 0;
        hcamg_report r2{};
        read_report(hs[r], &r2, &e2);
        require(r2.iterations == rep.iterations && r2.final_relres == rep.final_relres,
                "ranks disagree on the iteration count / residual");
      }
      pcg_breakdown(hs[0], error);
      if (report) *report = rep;
    }
    for (int r = 0; r < n; ++r) check_dist(hs[r]);
  });
}


// ---- the partition's planner as a host-only API (no device call below)

struct hcamg_plan {
  PlanState st;
  PlanResult out;
  int32_t steps = 0;
};

int hcamg_rows_owner(int64_t n, const int64_t* indptr, const int32_t* indices, int32_t nranks, int8_t* owner) {
  if (n < 0 || !indptr || (!indices && n > 0 && indptr[n] > 0) || nranks < 1 || nranks > kRowsMaxRanks || !owner)
    return HCAMG_EINVAL;
  try {
    std::vector<int8_t> o;
    rows_bfs_owner(n, indptr, indices, nranks, o);
    memcpy(owner, o.data(), (size_t)n);
    return HCAMG_OK;
  } catch (...) {
    return HCAMG_ENOMEM;
  }
}

int hcamg_plan_create(hcamg_plan** out, int32_t nranks, int32_t nvec, const int64_t* vec_len) {
  if (!out || nranks < 1 || nranks > kRowsMaxRanks || nvec < 1 || !vec_len) return HCAMG_EINVAL;
  try {
    std::unique_ptr<hcamg_plan> p(new hcamg_plan());
    p->st.init(nranks, std::vector<int64_t>(vec_len, vec_len + nvec));
    *out = p.release();
    return HCAMG_OK;
  } catch (...) {
    return HCAMG_ENOMEM;
  }
}

int hcamg_plan_destroy(hcamg_plan* p) {
  delete p;
  return HCAMG_OK;
}

int hcamg_plan_set_vector(hcamg_plan* p, int32_t vec, int32_t holder_mask, const int8_t* owner) {
  if (!p || vec < 0 || vec + 1 >= (int32_t)p->st.vec_off.size()) return HCAMG_EINVAL;
  p->st.set_vector(vec, (uint8_t)holder_mask, owner);
  return HCAMG_OK;
}

int hcamg_plan_invalidate(hcamg_plan* p, int32_t vec) {
  if (!p || vec < 0 || vec + 1 >= (int32_t)p->st.vec_off.size()) return HCAMG_EINVAL;
  p->st.invalidate_vector(vec);
  return HCAMG_OK;
}

int hcamg_plan_step(hcamg_plan* p, const int64_t* nreads, const int32_t* rvec, const int32_t* ridx,
                    const int64_t* nwrites, const int32_t* wvec, const int32_t* widx) {
  if (!p || !nreads || !nwrites) return HCAMG_EINVAL;
  try {
    const int N = p->st.nranks;
    const int nvec = (int)p->st.vec_off.size() - 1;
    std::vector<PlanAccess> acc((size_t)N);
    int64_t ro = 0, wo = 0;
    for (int q = 0; q < N; ++q) {
      PlanAccess& a = acc[(size_t)q];
      for (int64_t k = 0; k < nreads[q]; ++k) {
        const int32_t v = rvec[ro + k], i = ridx[ro + k];
        if (v < 0 || v >= nvec || i < 0 || i >= p->st.vec_off[(size_t)v + 1] - p->st.vec_off[(size_t)v]) return HCAMG_EINVAL;
        a.rvec.push_back(v);
        a.ridx.push_back(i);
      }
      for (int64_t k = 0; k < nwrites[q]; ++k) {
        const int32_t v = wvec[wo + k], i = widx[wo + k];
        if (v < 0 || v >= nvec || i < 0 || i >= p->st.vec_off[(size_t)v + 1] - p->st.vec_off[(size_t)v]) return HCAMG_EINVAL;
        a.wvec.push_back(v);
        a.widx.push_back(i);
      }
      ro += nreads[q];
      wo += nwrites[q];
    }
    plan_step(p->st, p->steps, p->steps, acc, p->out);
    ++p->steps;
    return HCAMG_OK;
  } catch (...) {
    return HCAMG_ENOMEM;
  }
}

int hcamg_plan_counts(hcamg_plan* p, int64_t* counts) {
  if (!p || !counts) return HCAMG_EINVAL;
  counts[0] = (int64_t)p->out.segs.size();
  counts[1] = (int64_t)p->out.idx.size();
  counts[2] = p->out.unheld_reads;
  return HCAMG_OK;
}

int hcamg_plan_pushes(hcamg_plan* p, int32_t* seg, int32_t* idx) {
  if (!p || (!seg && !p->out.segs.empty()) || (!idx && !p->out.idx.empty())) return HCAMG_EINVAL;
  for (size_t k = 0; k < p->out.segs.size(); ++k) {
    const PushSeg& s = p->out.segs[k];
    seg[5 * k] = s.boundary;
    seg[5 * k + 1] = s.src;
    seg[5 * k + 2] = s.dst;
    seg[5 * k + 3] = s.vec;
    seg[5 * k + 4] = (int32_t)(s.end - s.begin);
  }
  if (!p->out.idx.empty()) memcpy(idx, p->out.idx.data(), p->out.idx.size() * sizeof(int32_t));
  return HCAMG_OK;
}

}  // extern "C"
