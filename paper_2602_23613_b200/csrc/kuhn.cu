// GPU assembly of the seeded 3D Kuhn-cube curl-curl systems (the input
// generator in front of the hot path).  Follows
// paper_2602_23613_b200/kuhn.py (assemble_kuhn, lexicographic vertex
// numbering), which restates the reference's 2D fem.py:111-195 in 3D:
//   * vertices of the (n+1)^3 grid, v = (k(n+1)+j)(n+1)+i;
//   * 6 Kuhn tets per hex, cube-major / permutation-minor, vertices
//     v0 -> v0+e_a -> v0+e_a+e_b -> v0+(1,1,1): every vertex sequence rises,
//     so every local edge is positively oriented (the sign outer product is 1);
//   * edge (v, v+d), d in {0,1}^3 \ 0, exists iff v+d is in the grid; edges
//     numbered by (tail, head), i.e. per tail by the offset of d;
//   * element matrices S, M of the 6 tet shapes come from the host (the same
//     numpy code as kuhn.py, so bit-identical); S is scaled by mu^{-1} per tet;
//   * duplicates are summed in tet order (a stable sort by (row, col) of the
//     contributions in tet order, then sequential segment sums);
//   * tangential Dirichlet elimination, the discrete gradient, then
//     As = canon(0.5 (As + As^T)), Am likewise, A = canon(As + beta Am),
//     A = canon(0.5 (A + A^T)) exactly as kuhn.py / fem.py:188-194.
// The only difference from the host generator is the order in which the
// duplicate contributions of one entry are summed (scipy's sum_duplicates
// follows an unstable std::sort), i.e. entries can differ in the last bit.
#include <cub/cub.cuh>

#include "kuhn.cuh"
#include "sparse.cuh"

namespace hcamg {

namespace {

// local edges (0,1),(0,2),(0,3),(1,2),(1,3),(2,3) (kuhn.py _LOCAL_EDGES)
__constant__ int c_le[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
// permutations (a, b) of itertools.permutations(range(3)), first two entries
__constant__ int c_perm[6][2] = {{0, 1}, {0, 2}, {1, 0}, {1, 2}, {2, 0}, {2, 1}};

struct Grid {
  int64_t n, N;
  __device__ int64_t vid(int64_t i, int64_t j, int64_t k) const { return (k * N + j) * N + i; }
};

// directions sorted by offset: x, y, xy, z, xz, yz, xyz
__device__ __forceinline__ void dir_of(int r, int& dx, int& dy, int& dz) {
  const int t[7][3] = {{1, 0, 0}, {0, 1, 0}, {1, 1, 0}, {0, 0, 1}, {1, 0, 1}, {0, 1, 1}, {1, 1, 1}};
  dx = t[r][0];
  dy = t[r][1];
  dz = t[r][2];
}

__global__ void k_edge_counts(Grid g, int64_t* __restrict__ cnt) {
  const int64_t nv = g.N * g.N * g.N;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = v % g.N, j = (v / g.N) % g.N, k = v / (g.N * g.N);
    cnt[v] = (1 + (i < g.n)) * (1 + (j < g.n)) * (1 + (k < g.n)) - 1;
  }
}

// global id of edge (v, v + d)
__device__ __forceinline__ int64_t edge_id(const Grid& g, const int64_t* __restrict__ eoff, int64_t v, int dx, int dy,
                                           int dz) {
  const int64_t i = v % g.N, j = (v / g.N) % g.N, k = v / (g.N * g.N);
  int rank = 0;
  for (int r = 0; r < 7; ++r) {
    int ex, ey, ez;
    dir_of(r, ex, ey, ez);
    if (ex == dx && ey == dy && ez == dz) break;
    if (i + ex <= g.n && j + ey <= g.n && k + ez <= g.n) ++rank;
  }
  return eoff[v] + rank;
}

// per edge: tail, head, boundary flag
__global__ void k_edges(Grid g, const int64_t* __restrict__ eoff, int64_t* __restrict__ tail, int64_t* __restrict__ head,
                        uint8_t* __restrict__ bnd) {
  const int64_t nv = g.N * g.N * g.N;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = v % g.N, j = (v / g.N) % g.N, k = v / (g.N * g.N);
    int64_t e = eoff[v];
    for (int r = 0; r < 7; ++r) {
      int dx, dy, dz;
      dir_of(r, dx, dy, dz);
      if (i + dx > g.n || j + dy > g.n || k + dz > g.n) continue;
      tail[e] = v;
      head[e] = g.vid(i + dx, j + dy, k + dz);
      // both endpoints on a common face: a coordinate that does not move and sits at 0 or n
      const bool fb = (dx == 0 && (i == 0 || i == g.n)) || (dy == 0 && (j == 0 || j == g.n)) ||
                      (dz == 0 && (k == 0 || k == g.n));
      bnd[e] = fb ? 1 : 0;
      ++e;
    }
  }
}

// 36 contributions per tet (row edge, col edge; key = row * ne + col), tet order
__global__ void k_contrib(Grid g, const int64_t* __restrict__ eoff, int64_t ne, const double* __restrict__ muinv,
                          const double* __restrict__ S6, const double* __restrict__ M6, uint64_t* __restrict__ key,
                          double* __restrict__ sv, double* __restrict__ mv) {
  const int64_t nt = 6 * g.n * g.n * g.n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nt; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t hx = t / 6;
    const int p = (int)(t % 6);
    const int64_t ci = hx % g.n, cj = (hx / g.n) % g.n, ck = hx / (g.n * g.n);
    int c[4][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {1, 1, 1}};
    c[1][c_perm[p][0]] = 1;
    c[2][c_perm[p][0]] = 1;
    c[2][c_perm[p][1]] = 1;
    int64_t ge[6];
    for (int a = 0; a < 6; ++a) {
      const int* u = c[c_le[a][0]];
      const int* w = c[c_le[a][1]];
      ge[a] = edge_id(g, eoff, g.vid(ci + u[0], cj + u[1], ck + u[2]), w[0] - u[0], w[1] - u[1], w[2] - u[2]);
    }
    const double mu = muinv[t];
    for (int a = 0; a < 6; ++a)
      for (int b = 0; b < 6; ++b) {
        const int64_t q = t * 36 + a * 6 + b;
        key[q] = (uint64_t)ge[a] * (uint64_t)ne + (uint64_t)ge[b];
        sv[q] = S6[p * 36 + a * 6 + b] * mu;
        mv[q] = M6[p * 36 + a * 6 + b];
      }
  }
}

__global__ void k_seg_heads(const uint64_t* __restrict__ k, int64_t m, int64_t* __restrict__ flag) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x)
    flag[q] = q == 0 || k[q] != k[q - 1];
}

// per segment (equal keys, contributions in tet order): sequential sums;
// entries restricted to free rows/cols (fmap >= 0) with the new numbering
__global__ void k_seg_sums(const uint64_t* __restrict__ k, const double* __restrict__ sv, const double* __restrict__ mv,
                           int64_t m, const int64_t* __restrict__ head_pos, int64_t nseg, int64_t ne,
                           const int64_t* __restrict__ fmap, int64_t* __restrict__ row, int32_t* __restrict__ col,
                           double* __restrict__ s_out, double* __restrict__ m_out) {
  for (int64_t sg = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sg < nseg; sg += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q0 = head_pos[sg], q1 = sg + 1 < nseg ? head_pos[sg + 1] : m;
    double a = 0.0, b = 0.0;
    for (int64_t q = q0; q < q1; ++q) {
      a = a + sv[q];
      b = b + mv[q];
    }
    const int64_t r = (int64_t)(k[q0] / (uint64_t)ne), c = (int64_t)(k[q0] % (uint64_t)ne);
    row[sg] = fmap[r] >= 0 && fmap[c] >= 0 ? fmap[r] : -1;
    col[sg] = fmap[c] >= 0 ? (int32_t)fmap[c] : -1;
    s_out[sg] = a;
    m_out[sg] = b;
  }
}

__global__ void k_scatter_pos(const int64_t* __restrict__ flag, int64_t m, const int64_t* __restrict__ pos,
                              int64_t* __restrict__ out) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x)
    if (flag[q]) out[pos[q]] = q;
}

// CSR of the free block from (row, col, value) triples already in (row, col) order; exact zeros dropped
template <bool kFill>
__global__ void k_free_csr(const int64_t* __restrict__ row, const int32_t* __restrict__ col,
                           const double* __restrict__ val, int64_t nseg, int64_t* __restrict__ cnt,
                           const int64_t* __restrict__ pos, int32_t* __restrict__ oi, double* __restrict__ ov) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nseg; q += (int64_t)gridDim.x * blockDim.x) {
    if (row[q] < 0 || val[q] == 0.0) continue;
    if (!kFill) {
      atomicAdd((unsigned long long*)&cnt[row[q]], 1ull);
    } else {
      // rank among the kept entries of the row preceding q (rows are contiguous, sorted)
      int64_t r = 0;
      for (int64_t p = q - 1; p >= 0 && (row[p] == row[q] || row[p] < 0); --p)
        if (row[p] == row[q] && val[p] != 0.0) ++r;
      oi[pos[row[q]] + r] = col[q];
      ov[pos[row[q]] + r] = val[q];
    }
  }
}

// C = A + s B (both canonical CSR, same shape); exact zeros dropped (csr_binop + canon)
template <bool kFill>
__global__ void k_axpby(int64_t n, const int64_t* __restrict__ ap, const int32_t* __restrict__ ai,
                        const double* __restrict__ av, const int64_t* __restrict__ bp, const int32_t* __restrict__ bi,
                        const double* __restrict__ bv, double sc, int64_t* __restrict__ cnt,
                        const int64_t* __restrict__ cp, int32_t* __restrict__ ci, double* __restrict__ cv) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = ap[r], q = bp[r], o = kFill ? cp[r] : 0, c = 0;
    while (p < ap[r + 1] || q < bp[r + 1]) {
      int32_t j;
      double v;
      if (q >= bp[r + 1] || (p < ap[r + 1] && ai[p] < bi[q])) {
        j = ai[p];
        v = av[p++];
      } else if (p >= ap[r + 1] || bi[q] < ai[p]) {
        j = bi[q];
        v = sc * bv[q++];
      } else {
        j = ai[p];
        v = av[p++] + sc * bv[q++];
      }
      if (v == 0.0) continue;
      if (kFill) {
        ci[o] = j;
        cv[o++] = v;
      } else {
        ++c;
      }
    }
    if (!kFill) cnt[r] = c;
  }
}

void csr_axpby(const DCsr& A, const DCsr& B, double sc, DCsr& C, cudaStream_t s) {
  const int64_t n = A.nrows;
  C.nrows = n;
  C.ncols = A.ncols;
  C.ptr.alloc(n + 1, s);
  DBuf<int64_t> cnt(n, s);
  if (n)
    k_axpby<false><<<grid_for(n, 128), 128, 0, s>>>(n, A.ptr.p, A.idx.p, A.val.p, B.ptr.p, B.idx.p, B.val.p, sc, cnt.p,
                                                    nullptr, nullptr, nullptr);
  HC_CHECK_LAUNCH();
  C.nnz = exclusive_scan(cnt.p, C.ptr.p, n, s);
  C.idx.alloc(C.nnz, s);
  C.val.alloc(C.nnz, s);
  if (n)
    k_axpby<true><<<grid_for(n, 128), 128, 0, s>>>(n, A.ptr.p, A.idx.p, A.val.p, B.ptr.p, B.idx.p, B.val.p, sc, nullptr,
                                                   C.ptr.p, C.idx.p, C.val.p);
  HC_CHECK_LAUNCH();
}

// map[q] = pos[q] where the flag (inverted when inv) is set, else -1
__global__ void k_free_maps(const uint8_t* __restrict__ flag, const int64_t* __restrict__ pos, int64_t n,
                            int64_t* __restrict__ map, int inv = 0) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    map[q] = (inv ? !flag[q] : flag[q]) ? pos[q] : -1;
}

__global__ void k_iota64(int64_t* __restrict__ v, int64_t n) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) v[q] = q;
}

__global__ void k_gather2(const int64_t* __restrict__ perm, int64_t m, const double* __restrict__ a,
                          const double* __restrict__ b, double* __restrict__ oa, double* __restrict__ ob) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x) {
    oa[q] = a[perm[q]];
    ob[q] = b[perm[q]];
  }
}

__global__ void k_vertex_free(Grid g, uint8_t* __restrict__ f, int64_t* __restrict__ cnt) {
  const int64_t nv = g.N * g.N * g.N;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = v % g.N, j = (v / g.N) % g.N, k = v / (g.N * g.N);
    f[v] = !(i == 0 || i == g.n || j == 0 || j == g.n || k == 0 || k == g.n);
    cnt[v] = f[v];
  }
}

__global__ void k_flag_count(const uint8_t* __restrict__ f, int64_t n, int64_t* __restrict__ cnt, int inv) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    cnt[q] = inv ? !f[q] : f[q];
}

// G rows of the free edges: -1 at a free tail, +1 at a free head (columns ascend: tail < head)
template <bool kFill>
__global__ void k_gradient(int64_t ne, const uint8_t* __restrict__ ebnd, const int64_t* __restrict__ emap,
                           const int64_t* __restrict__ tail, const int64_t* __restrict__ head,
                           const int64_t* __restrict__ vmap, int64_t* __restrict__ cnt, const int64_t* __restrict__ gp,
                           int32_t* __restrict__ gi, double* __restrict__ gv) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
    if (ebnd[e]) continue;
    const int64_t r = emap[e], t = vmap[tail[e]], h = vmap[head[e]];
    if (!kFill) {
      cnt[r] = (t >= 0) + (h >= 0);
    } else {
      int64_t o = gp[r];
      if (t >= 0) {
        gi[o] = (int32_t)t;
        gv[o++] = -1.0;
      }
      if (h >= 0) {
        gi[o] = (int32_t)h;
        gv[o] = 1.0;
      }
    }
  }
}

}  // namespace

void kuhn_assemble(int64_t n, const double* h_muinv, double beta, const double* h_S6, const double* h_M6, DCsr& A,
                   DCsr& G, std::vector<int64_t>& free_edges, std::vector<int64_t>& free_nodes, cudaStream_t s) {
  require(n >= 1, "n must be >= 1");
  Grid g{n, n + 1};
  const int64_t nv = g.N * g.N * g.N, nt = 6 * n * n * n;
  // edges
  DBuf<int64_t> ecnt(nv, s), eoff(nv + 1, s);
  k_edge_counts<<<grid_for(nv, 256), 256, 0, s>>>(g, ecnt.p);
  HC_CHECK_LAUNCH();
  const int64_t ne = exclusive_scan(ecnt.p, eoff.p, nv, s);
  DBuf<int64_t> tail(ne, s), head(ne, s);
  DBuf<uint8_t> ebnd(ne, s);
  k_edges<<<grid_for(nv, 256), 256, 0, s>>>(g, eoff.p, tail.p, head.p, ebnd.p);
  HC_CHECK_LAUNCH();
  // free numbering of edges and vertices
  DBuf<int64_t> fcnt(ne, s), fpos(ne + 1, s), emap(ne, s);
  k_flag_count<<<grid_for(ne, 256), 256, 0, s>>>(ebnd.p, ne, fcnt.p, 1);
  HC_CHECK_LAUNCH();
  const int64_t nfe = exclusive_scan(fcnt.p, fpos.p, ne, s);
  k_free_maps<<<grid_for(ne, 256), 256, 0, s>>>(ebnd.p, fpos.p, ne, emap.p, 1);
  HC_CHECK_LAUNCH();
  DBuf<uint8_t> vfree(nv, s);
  DBuf<int64_t> vcnt(nv, s), vpos(nv + 1, s), vmap(nv, s);
  k_vertex_free<<<grid_for(nv, 256), 256, 0, s>>>(g, vfree.p, vcnt.p);
  HC_CHECK_LAUNCH();
  const int64_t nfv = exclusive_scan(vcnt.p, vpos.p, nv, s);
  k_free_maps<<<grid_for(nv, 256), 256, 0, s>>>(vfree.p, vpos.p, nv, vmap.p);
  HC_CHECK_LAUNCH();
  // contributions, stably sorted by (row, col): duplicates in tet order
  DBuf<double> muinv, S6, M6;
  muinv.upload(h_muinv, nt, s);
  S6.upload(h_S6, 6 * 36, s);
  M6.upload(h_M6, 6 * 36, s);
  const int64_t m = 36 * nt;
  DBuf<uint64_t> key(m, s), key2(m, s);
  DBuf<double> sv(m, s), mv(m, s);
  k_contrib<<<grid_for(nt, 128), 128, 0, s>>>(g, eoff.p, ne, muinv.p, S6.p, M6.p, key.p, sv.p, mv.p);
  HC_CHECK_LAUNCH();
  DBuf<int64_t> perm_in(m, s), perm(m, s);
  k_iota64<<<grid_for(m, 256), 256, 0, s>>>(perm_in.p, m);
  HC_CHECK_LAUNCH();
  {
    int bits = 1;
    while (bits < 64 && ((uint64_t)1 << bits) <= (uint64_t)ne * (uint64_t)ne) ++bits;
    size_t bytes = 0;
    HC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key.p, key2.p, perm_in.p, perm.p, m, 0, bits, s));
    DBuf<unsigned char> ws((int64_t)bytes + 1, s);
    HC_CUDA(cub::DeviceRadixSort::SortPairs(ws.p, bytes, key.p, key2.p, perm_in.p, perm.p, m, 0, bits, s));
  }
  perm_in.release();
  // values into sorted order
  DBuf<double> sv2(m, s), mv2(m, s);
  k_gather2<<<grid_for(m, 256), 256, 0, s>>>(perm.p, m, sv.p, mv.p, sv2.p, mv2.p);
  HC_CHECK_LAUNCH();
  sv.release();
  mv.release();
  key.release();
  DBuf<int64_t> flag(m, s), spos(m + 1, s);
  k_seg_heads<<<grid_for(m, 256), 256, 0, s>>>(key2.p, m, flag.p);
  HC_CHECK_LAUNCH();
  const int64_t nseg = exclusive_scan(flag.p, spos.p, m, s);
  DBuf<int64_t> heads(nseg, s);
  k_scatter_pos<<<grid_for(m, 256), 256, 0, s>>>(flag.p, m, spos.p, heads.p);
  HC_CHECK_LAUNCH();
  DBuf<int64_t> srow(nseg, s);
  DBuf<int32_t> scol(nseg, s);
  DBuf<double> ssum(nseg, s), msum(nseg, s);
  k_seg_sums<<<grid_for(nseg, 256), 256, 0, s>>>(key2.p, sv2.p, mv2.p, m, heads.p, nseg, ne, emap.p, srow.p, scol.p,
                                                   ssum.p, msum.p);
  HC_CHECK_LAUNCH();
  // free-block CSR of As and Am (csr(As_full)[keep][:, keep] with exact zeros dropped)
  auto build = [&](const DBuf<double>& val, DCsr& out) {
    out.nrows = out.ncols = nfe;
    out.ptr.alloc(nfe + 1, s);
    DBuf<int64_t> cnt(nfe, s);
    cnt.zero();
    k_free_csr<false><<<grid_for(nseg, 256), 256, 0, s>>>(srow.p, scol.p, val.p, nseg, cnt.p, nullptr, nullptr,
                                                         nullptr);
    HC_CHECK_LAUNCH();
    out.nnz = exclusive_scan(cnt.p, out.ptr.p, nfe, s);
    out.idx.alloc(out.nnz, s);
    out.val.alloc(out.nnz, s);
    k_free_csr<true><<<grid_for(nseg, 256), 256, 0, s>>>(srow.p, scol.p, val.p, nseg, nullptr, out.ptr.p, out.idx.p,
                                                        out.val.p);
    HC_CHECK_LAUNCH();
  };
  DCsr As0, Am0, As, Am;
  build(ssum, As0);
  build(msum, Am0);
  symmetrize(As0, As, s);
  symmetrize(Am0, Am, s);
  As0 = DCsr();
  Am0 = DCsr();
  DCsr A0;
  if (beta > 0) csr_axpby(As, Am, beta, A0, s);
  else csr_copy(As, A0, s);
  symmetrize(A0, A, s);
  // gradient
  G.nrows = nfe;
  G.ncols = nfv;
  G.ptr.alloc(nfe + 1, s);
  DBuf<int64_t> gcnt(nfe, s);
  k_gradient<false><<<grid_for(ne, 256), 256, 0, s>>>(ne, ebnd.p, emap.p, tail.p, head.p, vmap.p, gcnt.p, nullptr,
                                                      nullptr, nullptr);
  HC_CHECK_LAUNCH();
  G.nnz = exclusive_scan(gcnt.p, G.ptr.p, nfe, s);
  G.idx.alloc(G.nnz, s);
  G.val.alloc(G.nnz, s);
  k_gradient<true><<<grid_for(ne, 256), 256, 0, s>>>(ne, ebnd.p, emap.p, tail.p, head.p, vmap.p, nullptr, G.ptr.p,
                                                     G.idx.p, G.val.p);
  HC_CHECK_LAUNCH();
  free_edges = emap.download();
  free_nodes = vmap.download();
  HC_CUDA(cudaStreamSynchronize(s));
}

}  // namespace hcamg
