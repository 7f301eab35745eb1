// Device-resident hierarchy: one DevLevel per AMG level, laid out for the
// solve kernels.
#pragma once
#include <memory>
#include <string>
#include <vector>

#include "giant.cuh"
#include "symv.cuh"
#include "split.cuh"
#include "sweep.cuh"

namespace hcamg {

// Padded copy of the smoother structure for the prefetching cluster leg.
struct SweepProgram {
  int64_t m = 0;
  DBuf<int8_t> pk;
  DBuf<int32_t> pdof, ocnt, ogc;
  DBuf<double> pbinv, ogv;
  int64_t ng[2] = {0, 0};
  DBuf<int32_t> gu[2], gcnt[2], ggc[2];
  DBuf<double> ggv[2];
  DBuf<unsigned> gbar;  // grid-barrier word of the cooperative leg (sense-reversing, starts 0)
};

// Dataflow-leg program (flow.cu): per direction the pulled terms of every
// patch entry and its correction slots.
struct FlowProgram {
  bool built = false;
  int64_t ne = 0, recmax = 0;
  DBuf<unsigned char> recs[2];   // per direction: one record per patch, in execution order
  DBuf<int64_t> rec_off[2];
  DBuf<double> d[2];
  DBuf<double> dw;               // slots of the wave-parallel variant (no sentinel protocol)
  DBuf<unsigned> bar;
};

// OSS-l1 smoother data in wavefront order (smoothers.py:60-137).
//
// Patches are renumbered wave-major: wave w holds patches [wave_ptr[w],
// wave_ptr[w+1]) of the reordered list; within a wave they are pairwise
// non-conflicting (no DoF of one is A-coupled to a DoF of another), so a wave
// is one parallel step of the multiplicative sweep.  The residual update of a
// wave is applied lazily by the NEXT step as a gather ("pull"): a gather row
// (w, u) lists A[u, j] for the DoFs j of wave w; rows inside a patch of the
// next wave are pulled by that patch's warp, the others by generic threads.
struct Smoother {
  int64_t npatch = 0, nwave = 0, kmax = 0;
  int64_t max_wave_patches = 0, max_gen_rows = 0;  // cluster-leg eligibility
  std::vector<int64_t> wave_ptr;        // host copy (launch geometry)
  DBuf<int64_t> patch_ptr;              // reordered patches -> entries
  DBuf<int32_t> patch_dofs;             // entry -> DoF
  DBuf<int64_t> binv_off;               // reordered patch -> offset of its k x k inverse
  DBuf<double> binv;                    // column-major inverses
  std::vector<int64_t> orig_of;         // reordered patch -> reference patch id
  // gather rows
  DBuf<int64_t> grow_ptr;
  DBuf<int32_t> grow_u, gcol;
  DBuf<double> gval;
  DBuf<int32_t> own_fw, own_bw;         // per entry: gather row pulled before the patch solve (-1: none)
  DBuf<int32_t> gen_fw, gen_bw;         // generic gather rows, grouped by source wave
  std::vector<int64_t> gen_fw_ptr, gen_bw_ptr;  // per source wave offsets (host)
  DBuf<int32_t> last_row;               // per DoF: gather row of the last wave (-1: none)
  DBuf<uint8_t> in_first;               // per DoF: member of a wave-0 patch
  // flattened copies for the cluster sweep (one fewer dependent load per pull):
  // genrow_*: (u, start, end) per generic row; ownr_*: (start, end) per patch
  // entry or (-1, -1); lastr: (start, end) per DoF for the last forward wave
  DBuf<int32_t> genrow_fw, genrow_bw, ownr_fw, ownr_bw, lastr;
  DBuf<int64_t> d_wave_ptr, d_gen_fw_ptr, d_gen_bw_ptr;
  // host copies for export (reference PatchSet layout, original patch order)
  std::vector<int64_t> h_patch_ptr, h_patch_dofs;
  SweepProgram pg;
  FlowProgram fl;
};

// Build the dataflow-leg terms of a smoother (once; a no-op when a DoF lies
// in more than two patches -- the leg then falls back to the grid leg).
void build_flow(const DCsr& A, Smoother& sm, cudaStream_t s);
// Waves wider than one 16-CTA cluster (the auto mode runs such levels on the whole GPU).
bool smoother_wide(const Smoother& sm);
// Auto mode runs this level one launch per wavefront (shallow, very wide schedules).
bool smoother_wave_auto(const Smoother& sm);
// Auto mode runs the dataflow leg on this level.
bool smoother_flow_auto(const Smoother& sm);

void build_program(Smoother& sm, SweepProgram& pg, cudaStream_t s);

struct DevLevel {
  int64_t n = 0;
  DCsr A, G;
  bool has_P = false;
  DCsr P, Pt;
  DBuf<double> l1;
  Smoother sm;
  SplitResult split;     // diagnostics (pairs / interior / c_G)
  std::vector<int64_t> gc_cols;
  bool coarsest = false;
  DBuf<double> Ainv;     // coarsest: dense inverse (row-major n x n)
  DCsr cmat;             // coarsest of a user-assembled hierarchy: the matrix its coarse_factor inverts
  SymPacked Asym;        // coarsest: its lower triangle (single-GPU GEMV reading it once)
  SegPlan pt_seg;        // segmented restriction plan when P^T has long rows
  HybridP hp;            // dense-regime interpolation block (P/Pt then hold the sparse part)
  // distributed solve (dist.cuh): context and exchange-site offsets of this level
  const Dist* dist = nullptr;
  static constexpr size_t kNoSite = ~(size_t)0;
  size_t xoff_g = kNoSite, xoff_y = kNoSite, xoff_c = kNoSite;
  int64_t pt_maxrow = 0;
  // work vectors
  DBuf<double> b, x, r, d0, d1, dj;
};

}  // namespace hcamg
