// Coarse/fine edge variables on the GPU: boundary augmentation, nodal dual,
// strong adjacency, greedy C/F and distance-two path matching (algebraic
// route), and the refinement splitting (ref route).
//
// Reference semantics (file:line in hcurl_amg/splitting.py):
//   augment_gradient 100-125, nodal_dual 128-133, _strong_adjacency 136-155,
//   _graph_neighbors 158-165, classical_cf 171-211, nodal_cf 214-229,
//   _edge_lookup 232-243, build_algebraic_splitting 246-298,
//   build_refinement_splitting 301-330.
// The greedy C/F pick and the matching are order-dependent; both run with the
// reference's exact sequential semantics (single-CTA pick loop; parallel
// candidate enumeration followed by an in-order acceptance scan).
#include <cub/cub.cuh>

#include "split.cuh"

namespace hcamg {

// ----------------------------------------------------------------------------- augment

namespace {

__global__ void k_aug_check(const int64_t* __restrict__ gp, const double* __restrict__ gv,
                            int64_t n, int64_t nnz, int64_t* __restrict__ bad_row,
                            int* __restrict__ bad_val, int64_t* __restrict__ single) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = i; r < n; r += st) {
    int64_t c = gp[r + 1] - gp[r];
    if (c > 2) atomicMin((unsigned long long*)bad_row, (unsigned long long)r);
    single[r] = c == 1;
  }
  for (int64_t e = i; e < nnz; e += st)
    if (fabs(gv[e]) != 1.0) *bad_val = 1;
}

__global__ void k_aug_fill(const int64_t* __restrict__ gp, const int32_t* __restrict__ gi,
                           const double* __restrict__ gv, const int64_t* __restrict__ rank,
                           int64_t n, int64_t m, const int64_t* __restrict__ op,
                           int32_t* __restrict__ oi, double* __restrict__ ov) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; r < n; r += st) {
    int64_t o = op[r];
    int64_t c = gp[r + 1] - gp[r];
    for (int64_t e = gp[r]; e < gp[r + 1]; ++e) { oi[o] = gi[e]; ov[o] = gv[e]; ++o; }
    if (c == 1) { oi[o] = (int32_t)(m + rank[r]); ov[o] = -gv[gp[r]]; }
  }
}

__global__ void k_aug_counts(const int64_t* __restrict__ gp, int64_t n, int64_t* __restrict__ cnt) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; r < n; r += st) {
    int64_t c = gp[r + 1] - gp[r];
    cnt[r] = c == 1 ? 2 : c;
  }
}

}  // namespace

int64_t augment_gradient(const DCsr& G, DCsr& Gt, cudaStream_t s) {
  const int64_t n = G.nrows, m = G.ncols;
  DBuf<int64_t> bad_row(1, s), single(n, s), rank(n + 1, s);
  DBuf<int> bad_val(1, s);
  bad_row.fill_bytes(0x7f);
  bad_val.zero();
  if (n || G.nnz)
    k_aug_check<<<grid_for(std::max(n, G.nnz), 256), 256, 0, s>>>(G.ptr.p, G.val.p, n, G.nnz, bad_row.p,
                                                                 bad_val.p, single.p);
  HC_CHECK_LAUNCH();
  int64_t br = read_scalar(bad_row.p, s);
  if (br != INT64_C(0x7f7f7f7f7f7f7f7f))
    throw Error(EINVAL_, "row " + std::to_string(br) + " has more than 2 nonzeros");
  if (G.nnz && read_scalar(bad_val.p, s)) throw Error(EINVAL_, "gradient entries must be +-1");
  int64_t k = exclusive_scan(single.p, rank.p, n, s);
  Gt.nrows = n;
  Gt.ncols = m + k;
  Gt.ptr.alloc(n + 1, s);
  DBuf<int64_t> cnt(n, s);
  if (n) k_aug_counts<<<grid_for(n, 256), 256, 0, s>>>(G.ptr.p, n, cnt.p);
  HC_CHECK_LAUNCH();
  Gt.nnz = exclusive_scan(cnt.p, Gt.ptr.p, n, s);
  Gt.idx.alloc(Gt.nnz, s);
  Gt.val.alloc(Gt.nnz, s);
  if (n) k_aug_fill<<<grid_for(n, 256), 256, 0, s>>>(G.ptr.p, G.idx.p, G.val.p, rank.p, n, m, Gt.ptr.p,
                                                    Gt.idx.p, Gt.val.p);
  HC_CHECK_LAUNCH();
  return k;
}

// ----------------------------------------------------------------------------- nodal graph

namespace {

// offdiag pattern (neighbours) and strong pattern in one sweep; kWrite=false counts.
template <bool kWrite>
__global__ void k_graph(const int64_t* __restrict__ ap, const int32_t* __restrict__ ai,
                        const double* __restrict__ av, int64_t n, double theta,
                        int64_t* __restrict__ ncnt, int64_t* __restrict__ scnt,
                        const int64_t* __restrict__ np_, int32_t* __restrict__ ni,
                        const int64_t* __restrict__ sp_, int32_t* __restrict__ si) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; r < n; r += st) {
    double mx = -1.0;
    bool any = false;
    for (int64_t e = ap[r]; e < ap[r + 1]; ++e)
      if (ai[e] != r) { any = true; mx = fmax(mx, fabs(av[e])); }
    double thr = __dmul_rn(theta, mx);
    int64_t cn = 0, cs = 0;
    int64_t on = kWrite ? np_[r] : 0, os = kWrite ? sp_[r] : 0;
    for (int64_t e = ap[r]; e < ap[r + 1]; ++e) {
      int32_t c = ai[e];
      if (c == r) continue;
      if (kWrite) ni[on + cn] = c;
      ++cn;
      if (any && fabs(av[e]) >= thr) {
        if (kWrite) si[os + cs] = c;
        ++cs;
      }
    }
    if (!kWrite) { ncnt[r] = cn; scnt[r] = cs; }
  }
}

}  // namespace

void nodal_graph(const DCsr& An, double theta, DCsr& nbr, DCsr& strong, cudaStream_t s) {
  const int64_t n = An.nrows;
  DBuf<int64_t> nc(n, s), sc(n, s);
  nbr.nrows = nbr.ncols = strong.nrows = strong.ncols = n;
  nbr.ptr.alloc(n + 1, s);
  strong.ptr.alloc(n + 1, s);
  unsigned g = grid_for(n, 128);
  if (n) k_graph<false><<<g, 128, 0, s>>>(An.ptr.p, An.idx.p, An.val.p, n, theta, nc.p, sc.p, nullptr,
                                          nullptr, nullptr, nullptr);
  HC_CHECK_LAUNCH();
  nbr.nnz = exclusive_scan(nc.p, nbr.ptr.p, n, s);
  strong.nnz = exclusive_scan(sc.p, strong.ptr.p, n, s);
  nbr.idx.alloc(nbr.nnz, s);
  strong.idx.alloc(strong.nnz, s);
  nbr.val.alloc(nbr.nnz, s);
  strong.val.alloc(strong.nnz, s);
  nbr.val.zero();
  strong.val.zero();
  if (n) k_graph<true><<<g, 128, 0, s>>>(An.ptr.p, An.idx.p, An.val.p, n, theta, nullptr, nullptr,
                                         nbr.ptr.p, nbr.idx.p, strong.ptr.p, strong.idx.p);
  HC_CHECK_LAUNCH();
}

// ----------------------------------------------------------------------------- greedy C/F

namespace {

constexpr int8_t kU = 0, kC = 1, kF = 2;

__global__ void k_cf_init(const int64_t* __restrict__ bcols, int64_t nb, const int64_t* __restrict__ np_,
                          const int32_t* __restrict__ ni, int8_t* __restrict__ state) {
  // state pre-set: U everywhere, C on B.  Neighbours of B that are not B -> F.
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; t < nb; t += st) {
    int64_t b = bcols[t];
    for (int64_t e = np_[b]; e < np_[b + 1]; ++e) {
      int32_t j = ni[e];
      if (state[j] != kC) state[j] = kF;
    }
  }
}

__global__ void k_set_state(const int64_t* __restrict__ ids, int64_t cnt, int8_t v, int8_t* state) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; t < cnt; t += st) state[ids[t]] = v;
}

// Unassigned nodes by measure: one hierarchical bitmap per measure value
// (level 0: a bit per node, level l + 1: a bit per level-l word), so the
// reference's pick -- np.argmax over the masked measure, lowest index on ties
// (splitting.py:197-208) -- is "first set bit of the highest non-empty
// bucket": a handful of dependent loads per pick instead of a scan over all
// nodes (the scan made the setup quadratic: 500 s at 12.6 M DoFs).
constexpr int kBkLevels = 4;
struct Buckets {
  unsigned long long* w;
  int64_t off[kBkLevels], nw[kBkLevels], stride;
  int nb;
};

// set-only phase (any number of threads; readers come after a barrier)
__device__ __forceinline__ void bk_set(const Buckets& b, int m, int64_t i) {
  unsigned long long* base = b.w + (int64_t)m * b.stride;
  int64_t idx = i;
  for (int l = 0; l < kBkLevels; ++l) {
    const unsigned long long bit = 1ull << (idx & 63);
    const unsigned long long old = atomicOr(base + b.off[l] + (idx >> 6), bit);
    if (old != 0ull) break;  // the word was non-empty: its summaries are (being) set
    idx >>= 6;
  }
}

// clear-only phase: the thread that empties a word clears its summary bit
__device__ __forceinline__ void bk_clear(const Buckets& b, int m, int64_t i) {
  unsigned long long* base = b.w + (int64_t)m * b.stride;
  int64_t idx = i;
  for (int l = 0; l < kBkLevels; ++l) {
    const unsigned long long bit = 1ull << (idx & 63);
    const unsigned long long old = atomicAnd(base + b.off[l] + (idx >> 6), ~bit);
    if (!(old & bit) || (old & ~bit) != 0ull) break;
    idx >>= 6;
  }
}

// first node of bucket m, or -1 (one thread)
__device__ __forceinline__ int64_t bk_first(const Buckets& b, int m) {
  const unsigned long long* base = b.w + (int64_t)m * b.stride;
  int64_t idx = -1;
  for (int64_t t = 0; t < b.nw[kBkLevels - 1]; ++t) {
    const unsigned long long v = ((volatile const unsigned long long*)base)[b.off[kBkLevels - 1] + t];
    if (v) {
      idx = t * 64 + (__ffsll((long long)v) - 1);
      break;
    }
  }
  if (idx < 0) return -1;
  for (int l = kBkLevels - 2; l >= 0; --l) {
    const unsigned long long v = ((volatile const unsigned long long*)base)[b.off[l] + idx];
    idx = idx * 64 + (__ffsll((long long)v) - 1);
  }
  return idx;
}

__global__ void k_cf_measure(const int64_t* __restrict__ sp_, const int32_t* __restrict__ si,
                             const int8_t* __restrict__ state, int64_t n,
                             int32_t* __restrict__ measure, Buckets bk) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; r < n; r += st) {
    int32_t m = 0;
    for (int64_t e = sp_[r]; e < sp_[r + 1]; ++e) m += state[si[e]] == kF;
    measure[r] = m;
    if (state[r] == kU) bk_set(bk, m, r);
  }
}

// One CTA runs the whole pick loop (splitting.py:197-208).
constexpr int kCfThreads = 1024;

__global__ void __launch_bounds__(kCfThreads) k_cf_greedy(
    int64_t n, const int64_t* __restrict__ np_, const int32_t* __restrict__ ni,
    const int64_t* __restrict__ tp, const int32_t* __restrict__ ti, int8_t* state, int32_t* measure,
    Buckets bk, int32_t* scratch /* n */) {
  __shared__ int64_t pick;
  __shared__ int nnew, top;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) top = bk.nb - 1;
  __syncthreads();
  while (true) {
    if (tid == 0) {
      int64_t i = -1;
      int t = top;
      while (t >= 0 && (i = bk_first(bk, t)) < 0) --t;
      top = t < 0 ? 0 : t;
      pick = i;
      nnew = 0;
      if (i >= 0) {
        state[i] = kC;
        bk_clear(bk, measure[i], i);
      }
    }
    __syncthreads();
    const int64_t i = pick;
    if (i < 0) break;
    // all unassigned graph neighbours of i become fine
    for (int64_t e = np_[i] + tid; e < np_[i + 1]; e += kCfThreads) {
      int32_t j = ni[e];
      if (state[j] == kU) {
        state[j] = kF;
        scratch[atomicAdd(&nnew, 1)] = j;
      }
    }
    __syncthreads();
    const int cnt = nnew;
    // clear phase: the new fine nodes and every unassigned node whose measure is about to change
    for (int t = tid; t < cnt; t += kCfThreads) bk_clear(bk, measure[scratch[t]], scratch[t]);
    for (int t = wid; t < cnt; t += kCfThreads / 32) {
      int32_t j = scratch[t];
      for (int64_t e = tp[j] + lane; e < tp[j + 1]; e += 32) {
        int32_t k = ti[e];
        if (state[k] == kU) bk_clear(bk, measure[k], k);
      }
    }
    __syncthreads();
    // measure[k] += 1 for k in strong_to[j] (one warp per new fine node)
    for (int t = wid; t < cnt; t += kCfThreads / 32) {
      int32_t j = scratch[t];
      for (int64_t e = tp[j] + lane; e < tp[j + 1]; e += 32) atomicAdd(&measure[ti[e]], 1);
    }
    __syncthreads();
    // set phase: back into the bucket of the new measure
    for (int t = wid; t < cnt; t += kCfThreads / 32) {
      int32_t j = scratch[t];
      for (int64_t e = tp[j] + lane; e < tp[j + 1]; e += 32) {
        int32_t k = ti[e];
        if (state[k] == kU) {
          const int m = measure[k];
          bk_set(bk, m, k);
          if (m > top) atomicMax(&top, m);
        }
      }
    }
    __syncthreads();
  }
}

__global__ void k_row_len_max(const int64_t* __restrict__ ptr, int64_t n, int* __restrict__ out) {
  int m = 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    m = max(m, (int)(ptr[r + 1] - ptr[r]));
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

__global__ void k_flag_state(const int8_t* __restrict__ state, int8_t v, int64_t n, int64_t* __restrict__ f) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; r < n; r += st) f[r] = state[r] == v;
}

__global__ void k_compact(const int64_t* __restrict__ flag, const int64_t* __restrict__ pos, int64_t n,
                          int64_t* __restrict__ out) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; r < n; r += st)
    if (flag[r]) out[pos[r]] = r;
}

}  // namespace

int64_t compact_flags(const int64_t* flag, int64_t n, DBuf<int64_t>& out, cudaStream_t s) {
  DBuf<int64_t> pos(n + 1, s);
  int64_t cnt = exclusive_scan(flag, pos.p, n, s);
  out.alloc(cnt, s);
  if (n && cnt) k_compact<<<grid_for(n, 256), 256, 0, s>>>(flag, pos.p, n, out.p);
  HC_CHECK_LAUNCH();
  return cnt;
}

void nodal_cf(const DCsr& An, const DBuf<int64_t>& bcols, double theta, DCsr& nbr,
              DBuf<int8_t>& state, cudaStream_t s) {
  const int64_t n = An.nrows;
  DCsr strong, strongT;
  nodal_graph(An, theta, nbr, strong, s);
  csr_transpose(strong, strongT, s);
  state.alloc(n, s);
  state.zero();
  if (bcols.n) {
    k_set_state<<<grid_for(bcols.n, 256), 256, 0, s>>>(bcols.p, bcols.n, kC, state.p);
    k_cf_init<<<grid_for(bcols.n, 256), 256, 0, s>>>(bcols.p, bcols.n, nbr.ptr.p, nbr.idx.p, state.p);
    HC_CHECK_LAUNCH();
  }
  DBuf<int32_t> measure(n, s), scratch(n + 1, s);
  if (n) {
    // a node's measure never exceeds the length of its strong row (each strong
    // neighbour counts once: fine from the start, or one increment when it turns fine)
    DBuf<int> mx(1, s);
    mx.zero();
    k_row_len_max<<<grid_for(n, 256), 256, 0, s>>>(strong.ptr.p, n, mx.p);
    HC_CHECK_LAUNCH();
    Buckets bk{};
    bk.nb = read_scalar(mx.p, s) + 1;
    int64_t words = 0, cnt = n;
    for (int l = 0; l < kBkLevels; ++l) {
      cnt = (cnt + 63) / 64;
      bk.off[l] = words;
      bk.nw[l] = cnt;
      words += cnt;
    }
    require(bk.nw[kBkLevels - 1] <= 64, "nodal graph too large for the C/F bucket index");
    bk.stride = words;
    DBuf<unsigned long long> bits(words * bk.nb, s);
    bits.zero();
    bk.w = bits.p;
    k_cf_measure<<<grid_for(n, 256), 256, 0, s>>>(strong.ptr.p, strong.idx.p, state.p, n, measure.p, bk);
    k_cf_greedy<<<1, kCfThreads, 0, s>>>(n, nbr.ptr.p, nbr.idx.p, strongT.ptr.p, strongT.idx.p, state.p,
                                         measure.p, bk, scratch.p);
    HC_CHECK_LAUNCH();
    HC_CUDA(cudaStreamSynchronize(s));  // bits is released below
  }
}

// ----------------------------------------------------------------------------- matching

namespace {

// edge (u, v) -> last two-entry row of Gt whose columns are {u, v} (splitting.py:232-243);
// scans the rows incident to u (GtT row u, ascending).  Returns -1 if absent.
__device__ __forceinline__ int64_t edge_of(int64_t u, int64_t v, const int64_t* __restrict__ tp,
                                           const int32_t* __restrict__ ti, const int64_t* __restrict__ gp,
                                           const int32_t* __restrict__ gi, double* gu, double* gv_) {
  int64_t found = -1;
  for (int64_t e = tp[u]; e < tp[u + 1]; ++e) {
    int64_t r = ti[e];
    int64_t a = gp[r];
    if (gp[r + 1] - a != 2) continue;
    int32_t c0 = gi[a], c1 = gi[a + 1];
    if ((c0 == u && c1 == v) || (c0 == v && c1 == u)) found = r;
  }
  return found;
}

constexpr int kMatchWarps = 4;
constexpr int kMatchCap = 4096;  // (j, k) candidates per coarse node (global scratch per warp)

__device__ __forceinline__ bool adjacent(int64_t u, int64_t v, const int64_t* __restrict__ np_,
                                         const int32_t* __restrict__ ni) {
  int64_t lo = np_[u], hi = np_[u + 1];
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if (ni[m] < v) lo = m + 1; else hi = m;
  }
  return lo < np_[u + 1] && ni[lo] == v;
}

// Enumerate, for each coarse node i (ascending), the statically valid triples
// (i, j, k) in the reference's (j asc, k asc) order.  Only paths whose two
// edges exist in G~ can ever be accepted (splitting.py:283-286), so the
// candidates are generated from the edge graph (k an edge-neighbour of i, j an
// edge-neighbour of k) and filtered by the nodal adjacency k in N(i) & N(j):
// the same set as the reference's two-hop scan, at O(edge degree^2) per node
// even on dense coarse levels.  kWrite=false counts.
template <bool kWrite>
__global__ void __launch_bounds__(32 * kMatchWarps) k_match_enum(
    const int64_t* __restrict__ coarse, int64_t ncoarse, const int8_t* __restrict__ is_c,
    const int8_t* __restrict__ in_b, const int64_t* __restrict__ np_, const int32_t* __restrict__ ni,
    const int64_t* __restrict__ tp, const int32_t* __restrict__ ti, const int64_t* __restrict__ gp,
    const int32_t* __restrict__ gi, const double* __restrict__ gv, int64_t* __restrict__ cnt,
    const int64_t* __restrict__ off, int64_t* __restrict__ trip /* 7 per triple */, int* overflow,
    unsigned long long* __restrict__ scratch) {
  __shared__ int ncand[kMatchWarps];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * kMatchWarps + w;
  const int64_t nw = (int64_t)gridDim.x * kMatchWarps;
  unsigned long long* keys = scratch + gw * 2 * kMatchCap;
  unsigned long long* sorted = keys + kMatchCap;
  for (int64_t t = gw; t < ncoarse; t += nw) {
    const int64_t i = coarse[t];
    if (lane == 0) ncand[w] = 0;
    __syncwarp();
    // lanes over the rows incident to i
    for (int64_t e = tp[i] + lane; e < tp[i + 1]; e += 32) {
      const int64_t r = ti[e];
      if (gp[r + 1] - gp[r] != 2) continue;
      const int64_t k = gi[gp[r]] == i ? gi[gp[r] + 1] : gi[gp[r]];
      if (!adjacent(i, k, np_, ni)) continue;
      for (int64_t f = tp[k]; f < tp[k + 1]; ++f) {
        const int64_t r2 = ti[f];
        if (gp[r2 + 1] - gp[r2] != 2) continue;
        const int64_t j = gi[gp[r2]] == k ? gi[gp[r2] + 1] : gi[gp[r2]];
        if (j <= i || !is_c[j] || (in_b[i] && in_b[j])) continue;
        if (!adjacent(j, k, np_, ni)) continue;
        const int pos = atomicAdd(&ncand[w], 1);
        if (pos < kMatchCap) keys[pos] = ((unsigned long long)j << 32) | (unsigned long long)k;
      }
    }
    __syncwarp();
    int nc = ncand[w];
    if (nc > kMatchCap) {
      if (lane == 0) *overflow = 1;
      nc = kMatchCap;
    }
    // rank sort (stable on position), then emit unique keys in order
    for (int q = lane; q < nc; q += 32) {
      const unsigned long long kq = keys[q];
      int rank = 0;
      for (int o = 0; o < nc; ++o) {
        const unsigned long long ko = keys[o];
        rank += ko < kq || (ko == kq && o < q);
      }
      sorted[rank] = kq;
    }
    __syncwarp();
    int64_t emitted = 0;
    const int64_t base = kWrite ? off[t] : 0;
    if (lane == 0) {
      unsigned long long prev = ~0ull;
      for (int q = 0; q < nc; ++q) {
        const unsigned long long key = sorted[q];
        if (key == prev) continue;
        prev = key;
        const int64_t j = (int64_t)(key >> 32), k = (int64_t)(key & 0xffffffffull);
        if (kWrite) {
          double d0, d1;
          const int64_t e1 = edge_of(i < k ? i : k, i < k ? k : i, tp, ti, gp, gi, &d0, &d1);
          const int64_t e2 = edge_of(k < j ? k : j, k < j ? j : k, tp, ti, gp, gi, &d0, &d1);
          const double g1 = gi[gp[e1]] == k ? gv[gp[e1]] : gv[gp[e1] + 1];
          const double g2 = gi[gp[e2]] == k ? gv[gp[e2]] : gv[gp[e2] + 1];
          int64_t* o = trip + 7 * (base + emitted);
          o[0] = i; o[1] = j; o[2] = k; o[3] = e1; o[4] = e2;
          o[5] = (g1 > 0) - (g1 < 0);
          o[6] = -((g2 > 0) - (g2 < 0));
        }
        ++emitted;
      }
      if (!kWrite) cnt[t] = emitted;
    }
    __syncwarp();
  }
}

// e1 == e2 (parallel duplicate path) is rejected at acceptance like the reference.
// In-order acceptance scan (splitting.py:277-295): the first statically valid
// k of each (i, j) whose mid node is unused and whose two DoFs are still free.
__global__ void k_match_accept(const int64_t* __restrict__ trip, int64_t ntrip, uint8_t* used_mid,
                               uint8_t* avail, int64_t* __restrict__ pairs /* 7 per pair */,
                               int64_t* __restrict__ npairs) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int64_t cnt = 0;
  int64_t li = -1, lj = -1;
  for (int64_t t = 0; t < ntrip; ++t) {
    const int64_t* q = trip + 7 * t;
    int64_t i = q[0], j = q[1];
    if (i == li && j == lj) continue;
    int64_t k = q[2], e1 = q[3], e2 = q[4];
    if (e1 == e2 || used_mid[k] || !avail[e1] || !avail[e2]) continue;
    int64_t* o = pairs + 7 * cnt;
    o[0] = e1; o[1] = e2; o[2] = q[5]; o[3] = q[6]; o[4] = i; o[5] = k; o[6] = j;
    avail[e1] = 0;
    avail[e2] = 0;
    used_mid[k] = 1;
    li = i;
    lj = j;
    ++cnt;
  }
  *npairs = cnt;
}

__global__ void k_u8_to_flag(const uint8_t* __restrict__ a, int64_t n, int64_t* __restrict__ f) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; r < n; r += st) f[r] = a[r] != 0;
}

__global__ void k_b_flags(const int64_t* __restrict__ b, int64_t nb, int8_t* __restrict__ in_b) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; t < nb; t += st) in_b[b[t]] = 1;
}

__global__ void k_cg_flag(const int8_t* __restrict__ state, int64_t n, int64_t m, int64_t* __restrict__ f) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; r < n; r += st) f[r] = state[r] == kC && r < m;
}

__global__ void k_is_coarse(const int8_t* __restrict__ state, int64_t n, int8_t* __restrict__ is_c) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; r < n; r += st) is_c[r] = state[r] == kC;
}

}  // namespace

void algebraic_splitting(const DCsr& A, const DCsr& G, double theta, SplitResult& out, cudaStream_t s) {
  const int64_t n = A.nrows;
  require(G.nrows == n, "dimension mismatch: A and G");
  DCsr Gt;
  int64_t k = augment_gradient(G, Gt, s);
  const int64_t mt = Gt.ncols;
  DBuf<int64_t> bcols(k, s);
  {
    std::vector<int64_t> h((size_t)k);
    for (int64_t t = 0; t < k; ++t) h[(size_t)t] = G.ncols + t;
    bcols.upload(h.data(), k);
  }
  StageTimer stt(s);
  // nodal dual  G~^T (A G~), symmetrised
  DCsr X, GtT, M, An;
  spgemm(A, Gt, X, s);
  stt.mark("    split: A G~");
  csr_transpose(Gt, GtT, s);
  spgemm(GtT, X, M, s);
  stt.mark("    split: G~^T (A G~)");
  X = DCsr();
  symmetrize(M, An, s);
  M = DCsr();
  stt.mark("    split: symmetrise");
  require(An.nrows == mt, "nodal dual size mismatch");
  DCsr nbr;
  DBuf<int8_t> state;
  nodal_cf(An, bcols, theta, nbr, state, s);
  stt.mark("    split: graph + C/F");
  // c_G = C \ B ; coarse = C (B is prescribed coarse)
  DBuf<int8_t> in_b(mt, s), is_c(mt, s);
  in_b.zero();
  if (k) k_b_flags<<<grid_for(k, 256), 256, 0, s>>>(bcols.p, k, in_b.p);
  if (mt) k_is_coarse<<<grid_for(mt, 256), 256, 0, s>>>(state.p, mt, is_c.p);
  HC_CHECK_LAUNCH();
  DBuf<int64_t> cflag(mt, s);
  if (mt) k_flag_state<<<grid_for(mt, 256), 256, 0, s>>>(state.p, kC, mt, cflag.p);
  HC_CHECK_LAUNCH();
  DBuf<int64_t> coarse;
  int64_t ncoarse = compact_flags(cflag.p, mt, coarse, s);
  {
    // c_G = C \ B: coarse nodes below the original column count (B = m..m+k-1)
    DBuf<int64_t> gflag(mt, s), cg;
    if (mt) k_cg_flag<<<grid_for(mt, 256), 256, 0, s>>>(state.p, mt, G.ncols, gflag.p);
    HC_CHECK_LAUNCH();
    compact_flags(gflag.p, mt, cg, s);
    out.coarse_nodes = cg.download();
  }
  // candidate triples
  DBuf<int64_t> cnt(ncoarse, s), off(ncoarse + 1, s);
  DBuf<int> overflow(1, s);
  overflow.zero();
  int blocks = (int)std::min<int64_t>(std::max<int64_t>((ncoarse + kMatchWarps - 1) / kMatchWarps, 1), kSMs * 8);
  DBuf<unsigned long long> scratch((int64_t)blocks * kMatchWarps * 2 * kMatchCap, s);
  if (ncoarse)
    k_match_enum<false><<<blocks, 32 * kMatchWarps, 0, s>>>(
        coarse.p, ncoarse, is_c.p, in_b.p, nbr.ptr.p, nbr.idx.p, GtT.ptr.p, GtT.idx.p, Gt.ptr.p, Gt.idx.p,
        Gt.val.p, cnt.p, nullptr, nullptr, overflow.p, scratch.p);
  HC_CHECK_LAUNCH();
  int64_t ntrip = exclusive_scan(cnt.p, off.p, ncoarse, s);
  if (read_scalar(overflow.p, s)) throw Error(EUNSUPPORTED_, "matching: candidate list overflow");
  DBuf<int64_t> trip(7 * std::max<int64_t>(ntrip, 1), s);
  if (ncoarse && ntrip)
    k_match_enum<true><<<blocks, 32 * kMatchWarps, 0, s>>>(
        coarse.p, ncoarse, is_c.p, in_b.p, nbr.ptr.p, nbr.idx.p, GtT.ptr.p, GtT.idx.p, Gt.ptr.p, Gt.idx.p,
        Gt.val.p, nullptr, off.p, trip.p, overflow.p, scratch.p);
  HC_CHECK_LAUNCH();
  DBuf<uint8_t> used_mid(mt, s), avail(n, s);
  used_mid.zero();
  avail.fill_bytes(1);
  DBuf<int64_t> pairs(7 * std::max<int64_t>(std::min(ntrip, n), 1), s), npairs(1, s);
  k_match_accept<<<1, 32, 0, s>>>(trip.p, ntrip, used_mid.p, avail.p, pairs.p, npairs.p);
  HC_CHECK_LAUNCH();
  stt.mark("    split: matching");
  int64_t np_h = read_scalar(npairs.p, s);
  out.pairs.resize((size_t)(7 * np_h));
  if (np_h)
    HC_CUDA(cudaMemcpyAsync(out.pairs.data(), pairs.p, 8 * 7 * np_h, cudaMemcpyDeviceToHost, s));
  DBuf<int64_t> aflag(n, s);
  if (n) k_u8_to_flag<<<grid_for(n, 256), 256, 0, s>>>(avail.p, n, aflag.p);
  HC_CHECK_LAUNCH();
  DBuf<int64_t> interior;
  compact_flags(aflag.p, n, interior, s);
  out.interior = interior.download();
  out.n = n;
  out.n_triples = ntrip;
  HC_CUDA(cudaStreamSynchronize(s));
}

// ----------------------------------------------------------------------------- refinement route

namespace {

__global__ void k_ref_pairs(const int64_t* __restrict__ cedges, const int64_t* __restrict__ fedges,
                            const int64_t* __restrict__ children, const int64_t* __restrict__ e2d,
                            int64_t nec, int64_t* __restrict__ flag, int64_t* __restrict__ rec) {
  int64_t E = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; E < nec; E += st) {
    int64_t c1 = children[2 * E], c2 = children[2 * E + 1];
    int64_t d1 = e2d[c1], d2 = e2d[c2];
    flag[E] = d1 >= 0 && d2 >= 0;
    if (!flag[E]) continue;
    int64_t a0 = fedges[2 * c1], a1 = fedges[2 * c1 + 1], b0 = fedges[2 * c2], b1 = fedges[2 * c2 + 1];
    // smallest common vertex (np.intersect1d(...)[0])
    int64_t mid = INT64_MAX;
    if (a0 == b0 || a0 == b1) mid = min(mid, a0);
    if (a1 == b0 || a1 == b1) mid = min(mid, a1);
    int64_t* o = rec + 8 * E;
    o[0] = d1; o[1] = d2;
    o[2] = fedges[2 * c1 + 1] == mid ? 1 : -1;
    o[3] = fedges[2 * c2] == mid ? 1 : -1;
    o[4] = cedges[2 * E]; o[5] = mid; o[6] = cedges[2 * E + 1];
    o[7] = E;
  }
}

__global__ void k_ref_gather(const int64_t* __restrict__ sel, int64_t np_, const int64_t* __restrict__ rec,
                             int64_t* __restrict__ pairs, uint8_t* __restrict__ avail) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; t < np_; t += st) {
    const int64_t* q = rec + 8 * sel[t];
    for (int c = 0; c < 7; ++c) pairs[7 * t + c] = q[c];
    avail[q[0]] = 0;
    avail[q[1]] = 0;
  }
}

}  // namespace

void refinement_splitting(const int64_t* h_cedges, int64_t nec, const int64_t* h_fedges, int64_t nef,
                          const int64_t* h_children, const int64_t* h_e2d, int64_t n, SplitResult& out,
                          cudaStream_t s) {
  DBuf<int64_t> ce(2 * nec, s), fe(2 * nef, s), ch(2 * nec, s), e2d(nef, s), flag(nec, s), rec(8 * std::max<int64_t>(nec, 1), s);
  ce.upload(h_cedges, 2 * nec);
  fe.upload(h_fedges, 2 * nef);
  ch.upload(h_children, 2 * nec);
  e2d.upload(h_e2d, nef);
  if (nec) k_ref_pairs<<<grid_for(nec, 256), 256, 0, s>>>(ce.p, fe.p, ch.p, e2d.p, nec, flag.p, rec.p);
  HC_CHECK_LAUNCH();
  DBuf<int64_t> sel;
  int64_t npair = compact_flags(flag.p, nec, sel, s);
  DBuf<int64_t> pairs(7 * std::max<int64_t>(npair, 1), s), aflag(n, s);
  DBuf<uint8_t> avail(n, s);
  avail.fill_bytes(1);
  if (npair) {
    k_ref_gather<<<grid_for(npair, 256), 256, 0, s>>>(sel.p, npair, rec.p, pairs.p, avail.p);
    HC_CHECK_LAUNCH();
  }
  out.pairs.resize((size_t)(7 * npair));
  if (npair) HC_CUDA(cudaMemcpyAsync(out.pairs.data(), pairs.p, 8 * 7 * npair, cudaMemcpyDeviceToHost, s));
  out.pair_mesh_edges = sel.download();
  if (n) k_u8_to_flag<<<grid_for(n, 256), 256, 0, s>>>(avail.p, n, aflag.p);
  HC_CHECK_LAUNCH();
  DBuf<int64_t> interior;
  compact_flags(aflag.p, n, interior, s);
  out.interior = interior.download();
  for (int64_t t = 0; t < npair; ++t)
    require(out.pairs[(size_t)(7 * t + 5)] != INT64_MAX, "refinement children do not share a vertex");
  out.n = n;
  out.coarse_nodes.clear();
}

}  // namespace hcamg
