// Subdomain row partition: device context, boundary kernel, recording (rows.cuh).
#include <algorithm>
#include <cstring>

#include "rows_dev.cuh"

namespace hcamg {

namespace {

constexpr int kPushThreads = 256;

// Boundary: copy this rank's push entries into the peers' vectors, then the
// last block raises the rank's epoch flag in every peer's buffer and (wait != 0)
// spins until every peer has raised the same epoch here.  One launch = one
// barrier over the ranks; the next kernel on the stream starts after it.
__global__ void __launch_bounds__(kPushThreads) k_xpush(const int* stop, XPush x) {
  if (*stop) return;
  __shared__ int64_t cum[64];
  const int ns = x.nseg;
  for (int j = threadIdx.x; j <= ns && j < 64; j += blockDim.x) cum[j] = x.seg_cum[j];
  __syncthreads();
  const int64_t total = ns > 0 ? cum[ns] : 0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int j = 0;
    while (j + 1 < ns && cum[j + 1] <= t) ++j;
    const int32_t i = x.idx[x.seg_off[j] + (t - cum[j])];
    const int64_t vo = x.voff[x.seg_vec[j]];
    const double v = reinterpret_cast<const double*>(x.base[x.rank] + vo)[i];
    reinterpret_cast<double*>(x.base[x.seg_dst[j]] + vo)[i] = v;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  __threadfence_system();
  if (gridDim.x > 1) {  // the last block to finish signals (most boundaries are one block: no ticket)
    if (atomicAdd(x.cta, 1u) != gridDim.x - 1) return;
    __threadfence_system();
    *x.cta = 0u;
  }
  const unsigned long long e = *x.ep + 1;
  *x.ep = e;
  for (int r = 0; r < x.nranks; ++r) {
    unsigned long long* f = reinterpret_cast<unsigned long long*>(x.base[r]) + x.rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(e) : "memory");
  }
  if (!x.wait) return;
  if (*reinterpret_cast<volatile int*>(x.err)) return;
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
          return;
        }
      }
    }
  }
}

// second half of a boundary in the lockstep emulation: every peer must have
// signalled already (no spinning: a missing flag is an error at once)
__global__ void k_xcheck(const int* stop, XPush x) {
  if (*stop || threadIdx.x != 0 || blockIdx.x != 0) return;
  const unsigned long long e = *x.ep;
  const unsigned long long* flags = reinterpret_cast<const unsigned long long*>(x.base[x.rank]);
  for (int r = 0; r < x.nranks; ++r) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + r) : "memory");
    if (v < e) atomicExch(x.err, 2);
  }
}

template <class T>
void fetch(const DBuf<T>& d, int64_t count, std::vector<T>& out, cudaStream_t s) {
  out.resize((size_t)std::max<int64_t>(count, 0));
  if (count > 0) HC_CUDA(cudaMemcpyAsync(out.data(), d.p, sizeof(T) * (size_t)count, cudaMemcpyDeviceToHost, s));
}

void host_image(std::vector<DevLevel*>& lv, std::vector<RowsHostLevel>& out, cudaStream_t s) {
  out.assign(lv.size(), RowsHostLevel{});
  for (size_t l = 0; l < lv.size(); ++l) {
    DevLevel& L = *lv[l];
    RowsHostLevel& H = out[l];
    H.n = L.n;
    H.coarsest = L.coarsest;
    fetch(L.A.ptr, L.A.nrows + 1, H.a_ptr, s);
    fetch(L.A.idx, L.A.nnz, H.a_idx, s);
    if (L.has_P) {
      fetch(L.P.ptr, L.P.nrows + 1, H.p_ptr, s);
      fetch(L.P.idx, L.P.nnz, H.p_idx, s);
      fetch(L.Pt.ptr, L.Pt.nrows + 1, H.pt_ptr, s);
      fetch(L.Pt.idx, L.Pt.nnz, H.pt_idx, s);
      fetch(L.Pt.val, L.Pt.nnz, H.pt_val, s);
    }
    if (!L.coarsest) {
      Smoother& sm = L.sm;
      H.nwave = sm.nwave;
      H.wave_ptr = sm.wave_ptr;
      if (H.wave_ptr.empty()) H.wave_ptr.assign(1, 0);
      fetch(sm.patch_ptr, sm.npatch + 1, H.patch_ptr, s);
      HC_CUDA(cudaStreamSynchronize(s));
      const int64_t ne = sm.npatch ? H.patch_ptr[(size_t)sm.npatch] : 0;
      fetch(sm.patch_dofs, ne, H.patch_dofs, s);
      fetch(sm.ownr_fw, 2 * ne, H.ownr[0], s);
      fetch(sm.ownr_bw, 2 * ne, H.ownr[1], s);
      H.gen_ptr[0] = sm.gen_fw_ptr;
      H.gen_ptr[1] = sm.gen_bw_ptr;
      for (int d = 0; d < 2; ++d)
        if (H.gen_ptr[d].empty()) H.gen_ptr[d].assign((size_t)H.nwave + 1, 0);
      fetch(sm.genrow_fw, 3 * H.gen_ptr[0].back(), H.genrow[0], s);
      fetch(sm.genrow_bw, 3 * H.gen_ptr[1].back(), H.genrow[1], s);
      fetch(sm.lastr, 2 * L.n, H.lastr, s);
      fetch(sm.gcol, sm.gcol.n, H.gcol, s);
      fetch(sm.in_first, L.n, H.in_first, s);
      H.fw = leg_mode(L) == SWEEP_FWAVE;
      H.ne = sm.fl.built ? sm.fl.ne : 0;
      if (H.fw)
        for (int d = 0; d < 2; ++d) {
          fetch(sm.fl.rec_off[d], sm.npatch + 1, H.rec_off[d], s);
          fetch(sm.fl.recs[d], sm.fl.recs[d].n, H.recs[d], s);
        }
    }
    HC_CUDA(cudaStreamSynchronize(s));
  }
}

}  // namespace

void RowsCtx::release() {
  for (int r = 0; r < kRowsMaxRanks; ++r) {
    if (opened[r] && base[r]) cudaIpcCloseMemHandle(base[r]);
    opened[r] = false;
    base[r] = nullptr;
  }
  if (sym) cudaFree(sym);
  sym = nullptr;
  sym_bytes = 0;
  on = false;
}

void rows_prepare(RowsCtx& rc, std::vector<DevLevel*>& lv, Workspace& w, int rank, int nranks, int64_t min_rows,
                  cudaStream_t s) {
  require(nranks >= 1 && nranks <= kRowsMaxRanks, "nranks must be in 1..8");
  require(rank >= 0 && rank < nranks, "rank out of range");
  require(!lv.empty(), "no hierarchy");
  for (DevLevel* L : lv) {
    require(!L->hp.on, "the subdomain row partition covers the sparse regime (no dense interpolation block); "
                       "dense-regime hierarchies use hcamg_dist_prepare");
    require(L->coarsest || L->sm.kmax <= 32, "patch larger than a warp");
  }
  rc.release();
  rc.rank = rank;
  rc.nranks = nranks;
  rc.min_rows = min_rows;
  rc.depth = (int)lv.size();
  const int depth = rc.depth;
  // ---- host image, ownership, shares
  std::vector<RowsHostLevel> H;
  host_image(lv, H, s);
  rows_bfs_owner(H[0].n, H[0].a_ptr.data(), H[0].a_idx.data(), nranks, H[0].owner);
  for (int l = 1; l < depth; ++l)
    rows_coarse_owner(H[(size_t)l].n, H[(size_t)l - 1].pt_ptr.data(), H[(size_t)l - 1].pt_idx.data(),
                      H[(size_t)l - 1].pt_val.data(), H[(size_t)l - 1].owner, H[(size_t)l].owner);
  // a level is split when it and every finer level has at least min_rows rows
  // (a one-rank partition splits too: it exchanges with itself, which is how
  // the graph-captured boundary kernels are tested); the coarsest level never is
  bool finer = true;
  rc.stats = RowsStats{};
  for (int l = 0; l < depth; ++l) {
    // (a level whose P^T has long rows -- 3D levels below the dense-regime cutoff -- is split too:
    // its restriction runs the row-list SpMV instead of the segmented single-GPU plan)
    H[(size_t)l].split = finer && !H[(size_t)l].coarsest && H[(size_t)l].n >= std::max<int64_t>(min_rows, 1);
    finer = H[(size_t)l].split;
    rc.stats.split_levels += H[(size_t)l].split ? 1 : 0;
  }
  std::vector<std::vector<RowsShare>> sh((size_t)depth);
  for (int l = 0; l < depth; ++l) rows_shares(H[(size_t)l], nranks, sh[(size_t)l]);
  // ---- program and plan
  rows_program(H, rc.seg);
  RowsPlan plan;
  rows_plan_all(H, sh, nranks, rc.seg, plan);
  require(plan.push.unheld_reads == 0,
          "row partition: the planner met " + std::to_string(plan.push.unheld_reads) + " reads of undefined entries");
  for (int g = 0; g < SEG_COUNT; ++g) rc.seg_boundary[g] = plan.seg_boundary[g];
  rc.barrier = plan.barrier;
  // ---- this rank's lists on the device
  rc.lev.clear();
  rc.lev.resize((size_t)depth);
  for (int l = 0; l < depth; ++l) {
    RowsLevelDev& D = rc.lev[(size_t)l];
    const RowsShare& S = sh[(size_t)l][(size_t)rank];
    D.split = H[(size_t)l].split;
    D.nrows = (int64_t)S.rows.size();
    D.rows.s = s;
    D.rows.upload(S.rows.data(), (int64_t)S.rows.size());
    D.fw = D.split && H[(size_t)l].fw;
    if (D.fw) {
      const RowsHostLevel& HL = H[(size_t)l];
      for (int d = 0; d < 2; ++d) {
        std::vector<unsigned char> loc;
        std::vector<int64_t> off(1, 0);
        for (int64_t pos : S.fpos[d]) {
          const int64_t b0 = HL.rec_off[d][(size_t)pos], b1 = HL.rec_off[d][(size_t)pos + 1];
          loc.insert(loc.end(), HL.recs[d].begin() + b0, HL.recs[d].begin() + b1);
          off.push_back((int64_t)loc.size());
        }
        if (loc.empty()) loc.assign(16, 0);
        D.frecs[d].s = s;
        D.frecs[d].upload(loc.data(), (int64_t)loc.size());
        D.frec_off[d].s = s;
        D.frec_off[d].upload(off.data(), (int64_t)off.size());
        D.foff[d] = S.foff[d];
      }
    } else if (D.split) {
      D.plist.s = s;
      D.plist.upload(S.plist.data(), (int64_t)S.plist.size());
      D.poff = S.poff;
      for (int d = 0; d < 2; ++d) {
        D.gen[d].s = s;
        D.gen[d].upload(S.gen[d].data(), (int64_t)S.gen[d].size());
        D.goff[d] = S.goff[d];
      }
    }
    if (D.split) {  // this rank's rows of the level's operators in the SpMV layout
      DevLevel& L = *lv[(size_t)l];
      D.sA = build_sell_rows(L.A, D.rows.p, D.nrows, s);
      if (L.has_P) D.sP = build_sell_rows(L.P, D.rows.p, D.nrows, s);
    }
    if (l > 0 && H[(size_t)l - 1].split)  // rows of P^T of the finer level
      rc.lev[(size_t)l - 1].sPt = build_sell_rows(lv[(size_t)l - 1]->Pt, D.rows.p, D.nrows, s);
  }
  // ---- push tables of this rank as the source
  const int32_t nb = plan.nboundary;
  rc.bfirst.assign((size_t)nb + 1, 0);
  rc.bcount.assign((size_t)nb, 0);
  std::vector<int32_t> hidx, hdst, hvec;
  std::vector<int64_t> hcum, hoff;
  {
    size_t k = 0;
    const std::vector<PushSeg>& segs = plan.push.segs;  // generated boundary by boundary
    for (int32_t b = 0; b < nb; ++b) {
      rc.bfirst[(size_t)b] = (int64_t)hdst.size();
      int64_t cum = 0;
      for (; k < segs.size() && segs[k].boundary == b; ++k) {
        const PushSeg& sg = segs[k];
        require(plan.barrier[(size_t)b] != 0, "row partition: push at a boundary without a barrier");
        if (sg.src != rank) continue;
        hcum.push_back(cum);
        hoff.push_back((int64_t)hidx.size());
        hdst.push_back(sg.dst);
        hvec.push_back(sg.vec);
        hidx.insert(hidx.end(), plan.push.idx.begin() + sg.begin, plan.push.idx.begin() + sg.end);
        cum += sg.end - sg.begin;
      }
      hcum.push_back(cum);  // closing entry (each boundary owns nseg + 1 cum entries)
      rc.bcount[(size_t)b] = cum;
      require((int64_t)hdst.size() - rc.bfirst[(size_t)b] < 63, "row partition: too many push segments at one boundary");
    }
    rc.bfirst[(size_t)nb] = (int64_t)hdst.size();
  }
  auto up32 = [&](DBuf<int32_t>& d, std::vector<int32_t>& h) {
    if (h.empty()) h.push_back(0);
    d.s = s;
    d.upload(h.data(), (int64_t)h.size());
  };
  auto up64 = [&](DBuf<int64_t>& d, std::vector<int64_t>& h) {
    if (h.empty()) h.push_back(0);
    d.s = s;
    d.upload(h.data(), (int64_t)h.size());
  };
  up32(rc.xidx, hidx);
  up32(rc.seg_dst, hdst);
  up32(rc.seg_vec, hvec);
  up64(rc.seg_cum, hcum);
  up64(rc.seg_off, hoff);
  // ---- statistics
  for (int g = 0; g < SEG_COUNT; ++g) {
    rc.stats.boundaries[g] = (int64_t)rc.seg[g].size();
    for (int32_t b : rc.seg_boundary[g]) {
      rc.stats.barriers[g] += plan.barrier[(size_t)b] ? 1 : 0;
      rc.stats.push_out[g] += rc.bcount[(size_t)b];
    }
  }
  {
    std::vector<int> seg_of((size_t)nb, 0);
    for (int g = 0; g < SEG_COUNT; ++g)
      for (int32_t b : rc.seg_boundary[g]) seg_of[(size_t)b] = g;
    for (const PushSeg& sg : plan.push.segs) rc.stats.push_all[seg_of[(size_t)sg.boundary]] += sg.end - sg.begin;
    rc.stats.own_rows0 = (int64_t)sh[0][(size_t)rank].rows.size();
    std::vector<char> seen((size_t)H[0].n, 0);
    for (int32_t u : sh[0][(size_t)rank].rows)
      for (int64_t e = H[0].a_ptr[(size_t)u]; e < H[0].a_ptr[(size_t)u + 1]; ++e) {
        const int32_t c = H[0].a_idx[(size_t)e];
        if (H[0].owner[(size_t)c] != rank && !seen[(size_t)c]) {
          seen[(size_t)c] = 1;
          ++rc.stats.ghost_rows0;
        }
      }
  }
  // ---- symmetric buffer: flags, then every vector at the same offset on every rank
  const int nvec = rows_vec_count(depth);
  rc.voff.assign((size_t)nvec, 0);
  rc.vlen.assign((size_t)nvec, 0);
  size_t off = kRowsFlagBytes;
  auto take = [&](int id, int64_t len) {
    rc.voff[(size_t)id] = (int64_t)off;
    rc.vlen[(size_t)id] = len;
    off += ((size_t)std::max<int64_t>(len, 1) * 8 + 255) / 256 * 256;
  };
  for (int l = 0; l < depth; ++l)
    for (int k = 0; k < LV_COUNT; ++k)
      take(rows_vec_level(l, k), k == LV_DW ? std::max<int64_t>(H[(size_t)l].ne, 1) : lv[(size_t)l]->n);
  for (int k = 0; k < WS_COUNT; ++k) take(rows_vec_ws(depth, k), lv[0]->n);
  take(rows_vec_red(depth), (int64_t)RS_COUNT * 2 * nranks);
  rc.sym_bytes = off;
  HC_CUDA(cudaMalloc(&rc.sym, rc.sym_bytes));  // not pool memory: exported through CUDA IPC
  HC_CUDA(cudaMemset(rc.sym, 0, rc.sym_bytes));
  rc.d_voff.s = s;
  rc.d_voff.upload(rc.voff.data(), (int64_t)rc.voff.size());
  if (!rc.ep.p) {
    rc.ep.alloc(1, s);
    rc.cta.alloc(1, s);
    rc.err.alloc(1, s);
  }
  rc.ep.zero();
  rc.cta.zero();
  rc.err.zero();
  // ---- re-point the working vectors into the symmetric buffer
  for (int l = 0; l < depth; ++l) {
    DevLevel& L = *lv[(size_t)l];
    DBuf<double>* v[6] = {&L.b, &L.x, &L.r, &L.d0, &L.d1, &L.dj};
    for (int k = 0; k < 6; ++k) v[k]->alias(rc.vec(rows_vec_level(l, k)), std::max<int64_t>(L.n, 1), s);
    if (L.sm.fl.built) L.sm.fl.dw.alias(rc.vec(rows_vec_level(l, LV_DW)), std::max<int64_t>(L.sm.fl.ne, 1), s);
  }
  {
    DBuf<double>* v[WS_COUNT] = {&w.x, &w.r, &w.z, &w.p, &w.Ap, &w.b};
    for (int k = 0; k < WS_COUNT; ++k) v[k]->alias(rc.vec(rows_vec_ws(depth, k)), std::max<int64_t>(lv[0]->n, 1), s);
  }
  HC_CUDA(cudaStreamSynchronize(s));
}

void rows_detach(RowsCtx& rc, std::vector<DevLevel*>& lv, Workspace& w, cudaStream_t s) {
  for (DevLevel* L : lv) {
    for (DBuf<double>* v : {&L->b, &L->x, &L->r, &L->d0, &L->d1, &L->dj}) {
      if (!v->view) continue;
      v->alloc(std::max<int64_t>(L->n, 1), s);
      v->zero();
    }
    if (L->sm.fl.dw.view) {
      L->sm.fl.dw.alloc(std::max<int64_t>(L->sm.fl.ne, 1), s);
      L->sm.fl.dw.zero();
    }
  }
  for (DBuf<double>* v : {&w.x, &w.r, &w.z, &w.p, &w.Ap, &w.b}) {
    if (!v->view) continue;
    v->alloc(std::max<int64_t>(w.n, 1), s);
    v->zero();
  }
  HC_CUDA(cudaStreamSynchronize(s));
  rc.release();
}

static XPush make_push(RowsCtx& rc, int32_t b, bool wait) {
  XPush x{};
  for (int r = 0; r < kRowsMaxRanks; ++r) x.base[r] = rc.base[r];
  x.rank = rc.rank;
  x.nranks = rc.nranks;
  x.voff = rc.d_voff.p;
  x.idx = rc.xidx.p;
  const int64_t f = rc.bfirst[(size_t)b];
  x.nseg = (int)(rc.bfirst[(size_t)b + 1] - f);
  // boundary b owns cum entries [f + b, f + b + nseg] (one closing entry per boundary)
  x.seg_cum = rc.seg_cum.p + f + b;
  x.seg_off = rc.seg_off.p + f;
  x.seg_dst = rc.seg_dst.p + f;
  x.seg_vec = rc.seg_vec.p + f;
  x.ep = rc.ep.p;
  x.cta = rc.cta.p;
  x.err = rc.err.p;
  x.wait = wait ? 1 : 0;
  return x;
}

int64_t rows_boundary(RowsCtx& rc, int g, size_t k, const int* stop, bool wait, cudaStream_t s) {
  const int32_t b = rc.seg_boundary[g][k];
  if (!rc.barrier[(size_t)b]) return 0;
  const XPush x = make_push(rc, b, wait);
  const int64_t cnt = rc.bcount[(size_t)b];
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((cnt + kPushThreads - 1) / kPushThreads, kSMs));
  k_xpush<<<grid, kPushThreads, 0, s>>>(stop, x);
  HC_CHECK_LAUNCH();
  return 1;
}

void rows_wait(RowsCtx& rc, const int* stop, cudaStream_t s) {
  const XPush x = make_push(rc, 0, false);
  k_xcheck<<<1, 32, 0, s>>>(stop, x);
  HC_CHECK_LAUNCH();
}

int64_t rows_record(RowsCtx& rc, int g, std::vector<DevLevel*>& lv, Workspace& w, const int* stop,
                    unsigned long long cond, cudaStream_t s) {
  int64_t launches = 0;
  for (size_t k = 0; k < rc.seg[g].size(); ++k) {
    launches += rows_boundary(rc, g, k, stop, true, s);
    launches += rows_launch_step(rc.seg[g][k], rc, lv, w, stop, cond, s);
  }
  return launches;
}

}  // namespace hcamg
