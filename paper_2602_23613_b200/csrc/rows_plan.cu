// Dataflow planner of the subdomain row partition (rows.cuh): pure host code.
#include <algorithm>
#include <map>
#include <tuple>

#include "rows.cuh"

namespace hcamg {

void PlanState::init(int nranks_, const std::vector<int64_t>& vec_len) {
  nranks = nranks_;
  vec_off.assign(vec_len.size() + 1, 0);
  for (size_t v = 0; v < vec_len.size(); ++v) vec_off[v + 1] = vec_off[v] + vec_len[v];
  const size_t tot = (size_t)vec_off.back();
  holder.assign(tot, 0);
  prod.assign(tot, 0);
  stamp.assign(tot, -1);
}

void PlanState::set_vector(int vec, uint8_t mask, const int8_t* owner) {
  const int64_t o = vec_off[(size_t)vec], n = vec_off[(size_t)vec + 1] - o;
  for (int64_t i = 0; i < n; ++i) {
    if (owner) {
      holder[(size_t)(o + i)] = (uint8_t)(mask & (1u << owner[i]));
      prod[(size_t)(o + i)] = owner[i];
    } else {
      holder[(size_t)(o + i)] = mask;
      prod[(size_t)(o + i)] = 0;
    }
    stamp[(size_t)(o + i)] = -1;
  }
}

void PlanState::invalidate_vector(int vec) {
  const int64_t o = vec_off[(size_t)vec], n = vec_off[(size_t)vec + 1] - o;
  std::fill(holder.begin() + o, holder.begin() + o + n, (uint8_t)0);
  std::fill(stamp.begin() + o, stamp.begin() + o + n, -1);
}

void plan_step(PlanState& st, int32_t boundary, int32_t step_id, const std::vector<PlanAccess>& acc,
               PlanResult& out) {
  const int N = st.nranks;
  // reads first (every rank reads the values in front of the step), then writes
  std::map<std::tuple<int, int, int>, std::vector<int32_t>> lists;  // (src, dst, vec) -> entries
  for (int q = 0; q < N && q < (int)acc.size(); ++q) {
    const PlanAccess& a = acc[(size_t)q];
    const uint8_t bit = (uint8_t)(1u << q);
    for (size_t k = 0; k < a.ridx.size(); ++k) {
      const int v = a.rvec[k];
      const size_t at = (size_t)(st.vec_off[(size_t)v] + a.ridx[k]);
      const uint8_t hm = st.holder[at];
      if (hm & bit) continue;
      if (!hm) {
        ++out.unheld_reads;
        continue;
      }
      int src = st.prod[at];
      if (!(hm & (1u << src))) {  // the producer's copy was dropped by a canonicalisation: any holder serves
        src = 0;
        while (!(hm & (1u << src))) ++src;
      }
      lists[std::make_tuple(src, q, v)].push_back(a.ridx[k]);
      st.holder[at] = (uint8_t)(hm | bit);
    }
  }
  for (int q = 0; q < N && q < (int)acc.size(); ++q) {
    const PlanAccess& a = acc[(size_t)q];
    const uint8_t bit = (uint8_t)(1u << q);
    for (size_t k = 0; k < a.widx.size(); ++k) {
      const int v = a.wvec[k];
      const size_t at = (size_t)(st.vec_off[(size_t)v] + a.widx[k]);
      if (st.stamp[at] == step_id) {  // the same entry written by several ranks in one step: replicated work
        st.holder[at] |= bit;
      } else {
        st.stamp[at] = step_id;
        st.holder[at] = bit;
        st.prod[at] = (int8_t)q;
      }
    }
  }
  for (auto& kv : lists) {
    std::vector<int32_t>& l = kv.second;
    std::sort(l.begin(), l.end());
    PushSeg sg{};
    sg.boundary = boundary;
    sg.src = std::get<0>(kv.first);
    sg.dst = std::get<1>(kv.first);
    sg.vec = std::get<2>(kv.first);
    sg.begin = (int64_t)out.idx.size();
    out.idx.insert(out.idx.end(), l.begin(), l.end());
    sg.end = (int64_t)out.idx.size();
    out.segs.push_back(sg);
  }
}

}  // namespace hcamg

// ----------------------------------------------------------------------------- ownership

namespace hcamg {

namespace {

void bfs_levels(int64_t n, const int64_t* ptr, const int32_t* idx, int64_t start, std::vector<int32_t>& lev,
                std::vector<int32_t>& order) {
  lev.assign((size_t)n, -1);
  order.clear();
  order.reserve((size_t)n);
  int64_t next_seed = 0;
  int32_t base = 0;
  auto run = [&](int64_t src) {
    size_t head = order.size();
    lev[(size_t)src] = base;
    order.push_back((int32_t)src);
    while (head < order.size()) {
      const int32_t u = order[head++];
      const int32_t l = lev[(size_t)u];
      for (int64_t e = ptr[u]; e < ptr[u + 1]; ++e) {
        const int32_t v = idx[e];
        if (lev[(size_t)v] < 0) {
          lev[(size_t)v] = l + 1;
          order.push_back(v);
        }
      }
      base = std::max(base, l + 1);
    }
  };
  if (n) run(start);
  while ((int64_t)order.size() < n) {  // further components continue the level count
    while (lev[(size_t)next_seed] >= 0) ++next_seed;
    run(next_seed);
  }
}

}  // namespace

void rows_bfs_owner(int64_t n, const int64_t* ptr, const int32_t* idx, int nranks, std::vector<int8_t>& owner) {
  owner.assign((size_t)n, 0);
  if (n == 0 || nranks <= 1) return;
  std::vector<int32_t> lev, order;
  // pseudo-peripheral start: the far end of the far end of DoF 0
  int64_t start = 0;
  for (int sweep = 0; sweep < 2; ++sweep) {
    bfs_levels(n, ptr, idx, start, lev, order);
    // deepest level of the start's own component: the last DoF reached before another seed was needed
    int32_t best = order[0];
    for (int32_t u : order)
      if (lev[(size_t)u] >= lev[(size_t)best]) best = u;
    start = best;
  }
  bfs_levels(n, ptr, idx, start, lev, order);
  // BFS discovery order is level-major; within a level keep it (neighbours of
  // earlier DoFs first), which keeps the chunks compact along the level too
  const double total = (double)ptr[n];
  double acc = 0.0;
  for (int32_t u : order) {
    const double w = (double)(ptr[u + 1] - ptr[u]);
    int r = total > 0 ? (int)((acc + 0.5 * w) * nranks / total) : 0;
    owner[(size_t)u] = (int8_t)std::min(std::max(r, 0), nranks - 1);
    acc += w;
  }
}

void rows_coarse_owner(int64_t nc, const int64_t* pt_ptr, const int32_t* pt_idx, const double* pt_val,
                       const std::vector<int8_t>& fine_owner, std::vector<int8_t>& owner) {
  owner.assign((size_t)nc, 0);
  for (int64_t c = 0; c < nc; ++c) {
    double best = -1.0;
    int8_t o = 0;
    for (int64_t e = pt_ptr[c]; e < pt_ptr[c + 1]; ++e) {
      const double a = pt_val[e] < 0 ? -pt_val[e] : pt_val[e];
      if (a > best) {
        best = a;
        o = fine_owner[(size_t)pt_idx[e]];
      }
    }
    owner[(size_t)c] = o;
  }
}

FlowRecView flow_rec_view(const unsigned char* rec) {
  FlowRecView v{};
  const int32_t* hd = reinterpret_cast<const int32_t*>(rec);
  v.k = hd[0];
  v.e0 = hd[1];
  v.nt = hd[2];
  const int k4 = (v.k + 3) & ~3, kp4 = (v.k + 1 + 3) & ~3;
  const int o_dof = 16 + 4 * 8, o_ts = o_dof + 4 * k4, o_xp = o_ts + 4 * kp4, o_binv = o_xp + 4 * k4,
            o_slot = o_binv + 8 * v.k * v.k;
  v.dof = reinterpret_cast<const int32_t*>(rec + o_dof);
  v.ts = reinterpret_cast<const int32_t*>(rec + o_ts);
  v.xpart = reinterpret_cast<const int32_t*>(rec + o_xp);
  v.tslot = reinterpret_cast<const int32_t*>(rec + o_slot);
  return v;
}

void rows_shares(const RowsHostLevel& L, int nranks, std::vector<RowsShare>& out) {
  out.assign((size_t)nranks, RowsShare{});
  for (int64_t u = 0; u < L.n; ++u) out[(size_t)L.owner[(size_t)u]].rows.push_back((int32_t)u);
  if (!L.split) return;
  const int64_t W = L.nwave;
  if (L.fw) {
    // execution order of direction d: waves ascending (0) / descending (1), patches ascending inside
    for (int d = 0; d < 2; ++d) {
      for (int r = 0; r < nranks; ++r) out[(size_t)r].foff[d].assign((size_t)W + 1, 0);
      int64_t pos = 0;
      for (int64_t s0 = 0; s0 < W; ++s0) {
        const int64_t w = d == 0 ? s0 : W - 1 - s0;
        for (int64_t t = L.wave_ptr[(size_t)w]; t < L.wave_ptr[(size_t)w + 1]; ++t, ++pos) {
          const int32_t first = L.patch_dofs[(size_t)L.patch_ptr[(size_t)t]];
          out[(size_t)L.owner[(size_t)first]].fpos[d].push_back(pos);
        }
        for (int r = 0; r < nranks; ++r) out[(size_t)r].foff[d][(size_t)s0 + 1] = (int64_t)out[(size_t)r].fpos[d].size();
      }
    }
    return;
  }
  for (int r = 0; r < nranks; ++r) {
    out[(size_t)r].poff.assign((size_t)W + 1, 0);
    for (int d = 0; d < 2; ++d) out[(size_t)r].goff[d].assign((size_t)W + 1, 0);
  }
  for (int64_t w = 0; w < W; ++w) {
    for (int64_t p = L.wave_ptr[(size_t)w]; p < L.wave_ptr[(size_t)w + 1]; ++p) {
      const int32_t first = L.patch_dofs[(size_t)L.patch_ptr[(size_t)p]];
      out[(size_t)L.owner[(size_t)first]].plist.push_back((int32_t)p);
    }
    for (int r = 0; r < nranks; ++r) out[(size_t)r].poff[(size_t)w + 1] = (int64_t)out[(size_t)r].plist.size();
    for (int d = 0; d < 2; ++d) {
      const int64_t g0 = L.gen_ptr[d][(size_t)w], g1 = L.gen_ptr[d][(size_t)w + 1];
      for (int64_t t = g0; t < g1; ++t) {
        const int32_t u = L.genrow[d][(size_t)(3 * t)];
        out[(size_t)L.owner[(size_t)u]].gen[d].push_back((int32_t)(t - g0));
      }
      for (int r = 0; r < nranks; ++r) out[(size_t)r].goff[d][(size_t)w + 1] = (int64_t)out[(size_t)r].gen[d].size();
    }
  }
}

// ----------------------------------------------------------------------------- program

namespace {

void level_steps(const std::vector<RowsHostLevel>& lv, size_t ell, std::vector<RStep>& out) {
  const RowsHostLevel& L = lv[ell];
  RStep st{};
  st.level = (int)ell;
  if (L.coarsest) {
    st.kind = RK_COARSE;
    out.push_back(st);
    return;
  }
  const int64_t W = L.nwave;
  auto wave = [&](bool init, int64_t dst, int64_t src, int dir) {
    RStep w{};
    w.kind = RK_WAVE;
    w.level = (int)ell;
    w.init = init;
    w.dst = dst;
    w.src = src;
    w.dir = dir;
    out.push_back(w);
  };
  auto fwave = [&](int dir, int64_t s0) {
    RStep w{};
    w.kind = RK_FWAVE;
    w.level = (int)ell;
    w.dir = dir;
    w.dst = s0;
    out.push_back(w);
  };
  auto spmv = [&](int mat, int epi) {
    RStep m{};
    m.kind = RK_SPMV;
    m.level = (int)ell;
    m.mat = mat;
    m.epi = epi;
    out.push_back(m);
  };
  auto leg = [&](bool down) {
    RStep g{};
    g.kind = RK_LEG;
    g.level = (int)ell;
    g.down = down;
    out.push_back(g);
  };
  // down leg
  if (!L.split) {
    leg(true);  // agglomerated: one step, whatever kernels the single-GPU solve picks
  } else if (L.fw) {
    for (int64_t s0 = 0; s0 < W; ++s0) fwave(0, s0);
    spmv(0, RE_RES_JAC);
    spmv(0, RE_JAC_BW);
  } else {
    if (W > 0) {
      wave(true, 0, -1, 0);
      for (int64_t d = 1; d < W; ++d) wave(false, d, d - 1, 0);
    } else {
      st.kind = RK_INIT_RB;
      out.push_back(st);
    }
    st.kind = RK_FW_FINAL;
    out.push_back(st);
    spmv(0, RE_JAC_FW);
  }
  spmv(2, RE_SET);
  level_steps(lv, ell + 1, out);
  spmv(1, RE_ADD);
  // up leg
  if (!L.split) {
    leg(false);
  } else {
    spmv(0, RE_RES_JAC);
    spmv(0, RE_JAC_BW);
    if (L.fw) for (int64_t s0 = 0; s0 < W; ++s0) fwave(1, s0);
    else for (int64_t d = W - 1; d >= 0; --d) wave(false, d, d == W - 1 ? -1 : d + 1, 1);
  }
}

RStep simple(int kind, int site = 0, int vec = -1, int epi = 0) {
  RStep s{};
  s.kind = kind;
  s.site = site;
  s.vec = vec;
  s.epi = epi;
  return s;
}

}  // namespace

void rows_program(const std::vector<RowsHostLevel>& lv, std::vector<RStep> seg[SEG_COUNT]) {
  const int depth = (int)lv.size();
  for (int g = 0; g < SEG_COUNT; ++g) seg[g].clear();
  level_steps(lv, 0, seg[SEG_VCYCLE]);
  seg[SEG_VCYCLE].push_back(simple(RK_GATHER, 0, rows_vec_ws(depth, WS_Z)));
  seg[SEG_INIT].push_back(simple(RK_SPMV, RS_INIT, -1, RE_PCG_INIT));
  seg[SEG_INIT].push_back(simple(RK_FINISH, RS_INIT));
  level_steps(lv, 0, seg[SEG_FIRST]);
  seg[SEG_FIRST].push_back(simple(RK_DOT_RZ, RS_RZ_FIRST));
  seg[SEG_FIRST].push_back(simple(RK_FINISH, RS_RZ_FIRST));
  seg[SEG_BODY].push_back(simple(RK_SPMV, RS_AP, -1, RE_AP));
  seg[SEG_BODY].push_back(simple(RK_FINISH, RS_AP));
  seg[SEG_BODY].push_back(simple(RK_PCG_UPDATE, RS_UPD));
  seg[SEG_BODY].push_back(simple(RK_FINISH, RS_UPD));
  level_steps(lv, 0, seg[SEG_BODY]);
  seg[SEG_BODY].push_back(simple(RK_DOT_RZ, RS_RZ));
  seg[SEG_BODY].push_back(simple(RK_FINISH, RS_RZ));
  seg[SEG_BODY].push_back(simple(RK_P_UPDATE));
  seg[SEG_GATHER].push_back(simple(RK_GATHER, 0, rows_vec_ws(depth, WS_X)));
  // stand-alone AMG iteration (multilevel.py:204-235): r = b - A x; loop { x += V(r); r = b - A x }
  seg[SEG_AMG_INIT].push_back(simple(RK_SPMV, RS_INIT, -1, RE_AMG_INIT));
  seg[SEG_AMG_INIT].push_back(simple(RK_FINISH, RS_INIT));
  seg[SEG_AMG_BODY].push_back(simple(RK_GUARD));
  level_steps(lv, 0, seg[SEG_AMG_BODY]);
  seg[SEG_AMG_BODY].push_back(simple(RK_AXPY1));
  seg[SEG_AMG_BODY].push_back(simple(RK_SPMV, RS_AMG, -1, RE_AMG_RES));
  seg[SEG_AMG_BODY].push_back(simple(RK_FINISH, RS_AMG));
}

// ----------------------------------------------------------------------------- accesses

void rows_access(const RStep& st, const std::vector<RowsHostLevel>& lv, const std::vector<std::vector<RowsShare>>& sh,
                 int nranks, std::vector<PlanAccess>& acc) {
  const int depth = (int)lv.size();
  acc.resize((size_t)nranks);
  for (PlanAccess& a : acc) {
    a.rvec.clear();
    a.ridx.clear();
    a.wvec.clear();
    a.widx.clear();
  }
  const int ell = st.level;
  const RowsHostLevel& L = lv[(size_t)ell];
  const int vB = ell == 0 ? rows_vec_ws(depth, WS_R) : rows_vec_level(ell, LV_B);
  const int vX = ell == 0 ? rows_vec_ws(depth, WS_Z) : rows_vec_level(ell, LV_X);
  const int vR = rows_vec_level(ell, LV_R), vDJ = rows_vec_level(ell, LV_DJ);
  const int vD[2] = {rows_vec_level(ell, LV_D0), rows_vec_level(ell, LV_D1)};
  const int vDW = rows_vec_level(ell, LV_DW);
  const int vRed = rows_vec_red(depth);
  for (int q = 0; q < nranks; ++q) {
    PlanAccess& a = acc[(size_t)q];
    auto R = [&](int v, int64_t i) { a.rvec.push_back(v); a.ridx.push_back((int32_t)i); };
    auto Wr = [&](int v, int64_t i) { a.wvec.push_back(v); a.widx.push_back((int32_t)i); };
    auto red = [&](int site) {
      Wr(vRed, (int64_t)site * 2 * nranks + 2 * q);
      Wr(vRed, (int64_t)site * 2 * nranks + 2 * q + 1);
    };
    // rows of level `lvl` this rank handles when `split` governs the step
    auto for_rows = [&](int lvl, bool split, auto&& f) {
      if (split) for (int32_t u : sh[(size_t)lvl][(size_t)q].rows) f((int64_t)u);
      else for (int64_t u = 0; u < lv[(size_t)lvl].n; ++u) f(u);
    };
    switch (st.kind) {
      case RK_SPMV: {
        if (st.epi == RE_AP || st.epi == RE_PCG_INIT || st.epi == RE_AMG_INIT || st.epi == RE_AMG_RES) {
          const RowsHostLevel& L0 = lv[0];
          const int xin = rows_vec_ws(depth, st.epi == RE_AP ? WS_P : WS_X);
          const int y = rows_vec_ws(depth, st.epi == RE_AP ? WS_AP : WS_R);
          for_rows(0, L0.split, [&](int64_t row) {
            for (int64_t e = L0.a_ptr[(size_t)row]; e < L0.a_ptr[(size_t)row + 1]; ++e) R(xin, L0.a_idx[(size_t)e]);
            if (st.epi == RE_AP) R(xin, row);
            else R(rows_vec_ws(depth, WS_B), row);
            Wr(y, row);
          });
          red(st.site);
          break;
        }
        if (st.mat == 0) {
          const int xin = st.epi == RE_RES_JAC ? vX : vDJ;
          for_rows(ell, L.split, [&](int64_t row) {
            for (int64_t e = L.a_ptr[(size_t)row]; e < L.a_ptr[(size_t)row + 1]; ++e) R(xin, L.a_idx[(size_t)e]);
            if (st.epi == RE_JAC_FW) { R(vR, row); Wr(vR, row); }
            else if (st.epi == RE_RES_JAC) { R(vB, row); Wr(vR, row); Wr(vDJ, row); }
            else { R(vR, row); Wr(vR, row); R(vDJ, row); R(vX, row); Wr(vX, row); }
          });
        } else if (st.mat == 1) {  // x += P x_c
          const int xin = rows_vec_level(ell + 1, LV_X);
          for_rows(ell, L.split, [&](int64_t row) {
            for (int64_t e = L.p_ptr[(size_t)row]; e < L.p_ptr[(size_t)row + 1]; ++e) R(xin, L.p_idx[(size_t)e]);
            R(vX, row);
            Wr(vX, row);
          });
        } else {  // b_c = P^T r
          const int y = rows_vec_level(ell + 1, LV_B);
          for_rows(ell + 1, L.split, [&](int64_t row) {
            for (int64_t e = L.pt_ptr[(size_t)row]; e < L.pt_ptr[(size_t)row + 1]; ++e) R(vR, L.pt_idx[(size_t)e]);
            Wr(y, row);
          });
        }
        break;
      }
      case RK_WAVE: {
        const int dir = st.dir;
        const int dsrc = st.src >= 0 ? vD[st.src & 1] : -1, ddst = vD[st.dst & 1];
        if (st.init) {
          for_rows(ell, L.split, [&](int64_t u) {
            R(vB, u);
            Wr(vR, u);
            if (!L.in_first[(size_t)u]) Wr(vX, u);
          });
        } else if (st.src >= 0) {
          const int64_t g0 = L.gen_ptr[dir][(size_t)st.src], g1 = L.gen_ptr[dir][(size_t)st.src + 1];
          auto row = [&](int64_t t) {
            const int32_t* g = &L.genrow[dir][(size_t)(3 * (g0 + t))];
            R(vR, g[0]);
            for (int32_t k = g[1]; k < g[2]; ++k) R(dsrc, L.gcol[(size_t)k]);
            Wr(vR, g[0]);
          };
          if (L.split) {
            const RowsShare& s = sh[(size_t)ell][(size_t)q];
            for (int64_t k = s.goff[dir][(size_t)st.src]; k < s.goff[dir][(size_t)st.src + 1]; ++k)
              row(s.gen[dir][(size_t)k]);
          } else {
            for (int64_t t = 0; t < g1 - g0; ++t) row(t);
          }
        }
        auto patch = [&](int64_t p) {
          for (int64_t e = L.patch_ptr[(size_t)p]; e < L.patch_ptr[(size_t)p + 1]; ++e) {
            const int32_t i = L.patch_dofs[(size_t)e];
            if (st.init) {
              R(vB, i);
            } else {
              R(vR, i);
              if (st.src >= 0) {
                const int32_t s0 = L.ownr[dir][(size_t)(2 * e)], s1 = L.ownr[dir][(size_t)(2 * e + 1)];
                if (s0 >= 0) {
                  for (int32_t k = s0; k < s1; ++k) R(dsrc, L.gcol[(size_t)k]);
                  Wr(vR, i);
                }
              }
              R(vX, i);
            }
            Wr(vX, i);
            Wr(ddst, i);
          }
        };
        if (L.split) {
          const RowsShare& s = sh[(size_t)ell][(size_t)q];
          for (int64_t k = s.poff[(size_t)st.dst]; k < s.poff[(size_t)st.dst + 1]; ++k) patch(s.plist[(size_t)k]);
        } else {
          for (int64_t p = L.wave_ptr[(size_t)st.dst]; p < L.wave_ptr[(size_t)st.dst + 1]; ++p) patch(p);
        }
        break;
      }
      case RK_FWAVE: {
        const int d = st.dir;
        const int r0 = d == 0 ? vB : vR;
        const RowsShare& sq = sh[(size_t)ell][(size_t)q];
        for (int64_t t = sq.foff[d][(size_t)st.dst]; t < sq.foff[d][(size_t)st.dst + 1]; ++t) {
          const FlowRecView v = flow_rec_view(L.recs[d].data() + L.rec_off[d][(size_t)sq.fpos[d][(size_t)t]]);
          for (int a = 0; a < v.k; ++a) {
            const int32_t u = v.dof[a], xp = v.xpart[a];
            R(r0, u);
            if (d == 1 && xp != -1) R(vX, u);
            for (int32_t tt = v.ts[a]; tt < v.ts[a + 1]; ++tt) R(vDW, v.tslot[tt]);
            Wr(vDW, v.e0 + a);
            if (xp >= 0 || xp == -2) Wr(vX, u);
          }
        }
        break;
      }
      case RK_LEG: {
        // a whole leg of an agglomerated level on every rank: reads the level's right-hand side
        // (and iterate, going up), defines every working vector of the level
        for (int64_t u = 0; u < L.n; ++u) {
          R(vB, u);
          if (!st.down) R(vX, u);
        }
        for (int64_t u = 0; u < L.n; ++u) {
          Wr(vX, u);
          Wr(vR, u);
          Wr(vDJ, u);
          Wr(vD[0], u);
          Wr(vD[1], u);
        }
        break;
      }
      case RK_FW_FINAL: {
        const int64_t W = L.nwave;
        const int dsrc = W > 0 ? vD[(W - 1) & 1] : -1;
        for_rows(ell, L.split, [&](int64_t u) {
          R(vR, u);
          if (W > 0) {
            const int32_t s0 = L.lastr[(size_t)(2 * u)], s1 = L.lastr[(size_t)(2 * u + 1)];
            if (s0 >= 0)
              for (int32_t k = s0; k < s1; ++k) R(dsrc, L.gcol[(size_t)k]);
          }
          R(vX, u);
          Wr(vX, u);
          Wr(vR, u);
          Wr(vDJ, u);
        });
        break;
      }
      case RK_INIT_RB:
        for_rows(ell, L.split, [&](int64_t u) { R(vB, u); Wr(vR, u); Wr(vX, u); });
        break;
      case RK_COARSE:
        for (int64_t u = 0; u < L.n; ++u) R(vB, u);
        for (int64_t u = 0; u < L.n; ++u) Wr(vX, u);
        break;
      case RK_PCG_UPDATE:
        for_rows(0, lv[0].split, [&](int64_t u) {
          R(rows_vec_ws(depth, WS_X), u);
          R(rows_vec_ws(depth, WS_R), u);
          R(rows_vec_ws(depth, WS_P), u);
          R(rows_vec_ws(depth, WS_AP), u);
          Wr(rows_vec_ws(depth, WS_X), u);
          Wr(rows_vec_ws(depth, WS_R), u);
        });
        red(st.site);
        break;
      case RK_DOT_RZ:
        for_rows(0, lv[0].split, [&](int64_t u) {
          R(rows_vec_ws(depth, WS_R), u);
          R(rows_vec_ws(depth, WS_Z), u);
          if (st.site == RS_RZ_FIRST) Wr(rows_vec_ws(depth, WS_P), u);
        });
        red(st.site);
        break;
      case RK_AXPY1:
        for_rows(0, lv[0].split, [&](int64_t u) {
          R(rows_vec_ws(depth, WS_Z), u);
          R(rows_vec_ws(depth, WS_X), u);
          Wr(rows_vec_ws(depth, WS_X), u);
        });
        break;
      case RK_P_UPDATE:
        for_rows(0, lv[0].split, [&](int64_t u) {
          R(rows_vec_ws(depth, WS_Z), u);
          R(rows_vec_ws(depth, WS_P), u);
          Wr(rows_vec_ws(depth, WS_P), u);
        });
        break;
      case RK_FINISH:
        for (int r = 0; r < nranks; ++r) {
          R(vRed, (int64_t)st.site * 2 * nranks + 2 * r);
          R(vRed, (int64_t)st.site * 2 * nranks + 2 * r + 1);
        }
        break;
      case RK_GATHER: {
        const int64_t len = st.vec >= rows_vec_ws(depth, 0) ? lv[0].n : lv[(size_t)(st.vec / LV_COUNT)].n;
        for (int64_t u = 0; u < len; ++u) R(st.vec, u);
        break;
      }
      default:
        break;
    }
  }
}

// ----------------------------------------------------------------------------- plan of all segments

namespace {

bool step_partitioned(const RStep& st, const std::vector<RowsHostLevel>& lv) {
  switch (st.kind) {
    case RK_COARSE: return false;
    case RK_SPMV:
      if (st.epi == RE_AP || st.epi == RE_PCG_INIT || st.epi == RE_AMG_INIT || st.epi == RE_AMG_RES) return lv[0].split;
      return lv[(size_t)st.level].split;
    case RK_WAVE:
    case RK_FWAVE:
    case RK_LEG:
    case RK_FW_FINAL:
    case RK_INIT_RB: return lv[(size_t)st.level].split;
    default: return lv[0].split;
  }
}

}  // namespace

void rows_plan_all(const std::vector<RowsHostLevel>& lv, const std::vector<std::vector<RowsShare>>& sh, int nranks,
                   const std::vector<RStep> seg[SEG_COUNT], RowsPlan& plan) {
  const int depth = (int)lv.size();
  std::vector<int64_t> len((size_t)rows_vec_count(depth), 0);
  for (int l = 0; l < depth; ++l)
    for (int k = 0; k < LV_COUNT; ++k)
      len[(size_t)rows_vec_level(l, k)] = k == LV_DW ? std::max<int64_t>(lv[(size_t)l].ne, 1) : lv[(size_t)l].n;
  for (int k = 0; k < WS_COUNT; ++k) len[(size_t)rows_vec_ws(depth, k)] = lv[0].n;
  len[(size_t)rows_vec_red(depth)] = (int64_t)RS_COUNT * 2 * nranks;
  PlanState st;
  st.init(nranks, len);
  const uint8_t all = (uint8_t)((1u << nranks) - 1);
  const int8_t* own0 = lv[0].split ? lv[0].owner.data() : nullptr;
  plan = RowsPlan{};
  std::vector<PlanAccess> acc;
  int32_t boundary = 0, step_id = 0;
  for (int g = 0; g < SEG_COUNT; ++g) {
    // canonical state in front of the segment: the PCG vectors it inherits
    // live where their rows are owned (the kernels that wrote them ran on row
    // lists); everything else is undefined
    for (int v = 0; v < rows_vec_count(depth); ++v) st.invalidate_vector(v);
    auto owned = [&](int w) { st.set_vector(rows_vec_ws(depth, w), all, own0); };
    auto everywhere = [&](int w) { st.set_vector(rows_vec_ws(depth, w), all, nullptr); };
    if (g == SEG_VCYCLE) everywhere(WS_R);
    else if (g == SEG_INIT) { everywhere(WS_B); everywhere(WS_X); }
    else if (g == SEG_FIRST) { owned(WS_X); owned(WS_R); }
    else if (g == SEG_BODY) { owned(WS_X); owned(WS_R); owned(WS_P); }
    else if (g == SEG_AMG_INIT) { everywhere(WS_B); everywhere(WS_X); }
    else if (g == SEG_AMG_BODY) { everywhere(WS_B); owned(WS_X); owned(WS_R); }
    else owned(WS_X);
    plan.seg_boundary[g].clear();
    for (size_t k = 0; k < seg[g].size(); ++k) {
      const bool bar = step_partitioned(seg[g][k], lv) || (k > 0 ? step_partitioned(seg[g][k - 1], lv) : lv[0].split);
      rows_access(seg[g][k], lv, sh, nranks, acc);
      const size_t before = plan.push.segs.size();
      plan_step(st, boundary, step_id++, acc, plan.push);
      plan.seg_boundary[g].push_back(boundary);
      plan.barrier.push_back(bar || plan.push.segs.size() != before ? 1 : 0);
      ++boundary;
    }
  }
  plan.nboundary = boundary;
}

}  // namespace hcamg
