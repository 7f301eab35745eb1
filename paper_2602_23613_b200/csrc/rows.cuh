// Subdomain row partition of the solve across GPUs (the
// north-star layout): every level of a sparse-regime hierarchy is split by
// rows into one subdomain per rank, each rank computes only its rows of every
// SpMV, its patches of every smoother wavefront, its rows of P / P^T and its
// share of the PCG reductions, and pushes the entries a neighbour needs next
// straight into that neighbour's vectors over NVLink peer memory.  Levels
// below a size threshold are agglomerated: every rank keeps the whole level
// and solves it redundantly (the same latency as gather-solve-broadcast with
// one exchange fewer).
//
// How the exchanges are found.  The solve is a fixed sequence of STEPS (one
// kernel each).  Every rank keeps full-length vectors indexed by global DoF
// number, of which only the entries it computes or receives are meaningful.
// At setup the host walks the step sequence symbolically (rows_plan): for
// each vector entry it tracks which rank produced the current value and which
// ranks hold it; a step that reads an entry its rank does not hold adds that
// entry to the push list (producer -> reader) of the boundary in front of the
// step.  The result is one push list per (boundary, destination, vector); the
// halo exchange of an SpMV, the per-wavefront exchange of the multiplicative
// sweep, the P / P^T halos, the all-gather at the agglomeration level and the
// all-reduce of the PCG partial sums all fall out of the same rule.  The
// planner is pure host code (no CUDA), so the CPU tests drive it directly.
//
// A boundary is one kernel (rows.cu k_xpush): every block copies list entries
// into the peers' vectors; the last block to finish raises this rank's epoch
// flag in every peer's buffer and then waits for every peer's flag, so each
// boundary is a barrier over all ranks (a rank is never more than one step
// ahead of a peer, which is what makes pushing into live vectors safe).
#pragma once
#include <cstdint>
#include <vector>

namespace hcamg {

constexpr int kRowsMaxRanks = 8;

// ---- generic dataflow planner (host only)

// One step as the planner sees it: for every rank the entries it reads and
// the entries it writes, as (vector id, index) pairs.
struct PlanAccess {
  std::vector<int32_t> rvec, wvec;   // vector id per access
  std::vector<int32_t> ridx, widx;   // entry index per access
};

struct PushSeg {   // entries [begin, end) of PlanResult::idx go from `src` to `dst` in vector `vec`
  int32_t boundary, src, dst, vec;
  int64_t begin, end;
};

struct PlanResult {
  std::vector<PushSeg> segs;        // sorted by (boundary, src, dst, vec)
  std::vector<int32_t> idx;
  int64_t unheld_reads = 0;         // reads of an entry nobody holds (a modelling error unless allowed)
};

// State of the symbolic walk.  `holder` is a bit mask of ranks per entry,
// `prod` the rank that wrote the current value.
struct PlanState {
  int nranks = 0;
  std::vector<int64_t> vec_off;     // entry offset of every vector in the flat state arrays (nvec + 1)
  std::vector<uint8_t> holder;
  std::vector<int8_t> prod;
  std::vector<int32_t> stamp;       // last step that wrote the entry (same-step multi-rank writes)
  void init(int nranks_, const std::vector<int64_t>& vec_len);
  // entries of `vec` become valid on `mask`, produced by prod_of(i) (owner[i] when given, else rank 0)
  void set_vector(int vec, uint8_t mask, const int8_t* owner);
  void invalidate_vector(int vec);
};

// One step of the walk: `acc[rank]` are the accesses of the step (all reads see
// the values in front of the step).  Pushes go to `boundary` (the boundary in
// front of the step); `step_id` must be unique per step of a walk.
void plan_step(PlanState& st, int32_t boundary, int32_t step_id, const std::vector<PlanAccess>& acc,
               PlanResult& out);


// ---- the partitioned solve as a step program

enum RKind : int {
  RK_SPMV = 0,     // rows of a level matrix (mat 0: A, 1: P, 2: P^T) with an epilogue
  RK_WAVE,         // one wavefront of the multiplicative sweep
  RK_FW_FINAL,     // last wave's pending update + l1-Jacobi correction
  RK_INIT_RB,      // r = b, x = 0 (levels without patches)
  RK_COARSE,       // coarsest solve (always agglomerated)
  RK_PCG_UPDATE,   // x += alpha p, r -= alpha Ap, partial r.r
  RK_DOT_RZ,       // partial r.z (first: p = z)
  RK_P_UPDATE,     // p = z + beta p
  RK_FINISH,       // sum a reduction over the ranks, scalar logic
  RK_GATHER,       // no kernel: every rank reads the whole vector (all-gather through the push lists)
  RK_FWAVE,        // one wavefront of the sweep over the dataflow records (flow.cu k_flow_wave)
  RK_LEG,          // a whole smoothing leg of an agglomerated level, as the single-GPU solve runs it
  RK_AXPY1,        // stand-alone AMG iteration: x += z
  RK_GUARD,        // stand-alone AMG iteration: leave the device loop when the solve has stopped
};

// SpMV epilogues a step can ask for (numerically equal to solve.cu's Epi)
enum REpi : int { RE_SET = 0, RE_ADD = 1, RE_JAC_FW = 2, RE_RES_JAC = 3, RE_JAC_BW = 4, RE_AP = 5, RE_PCG_INIT = 6,
                  RE_AMG_INIT = 7, RE_AMG_RES = 8 };

// reduction sites: (S, S2) per rank each
enum RSite : int { RS_INIT = 0, RS_AP = 1, RS_UPD = 2, RS_RZ_FIRST = 3, RS_RZ = 4, RS_AMG = 5, RS_COUNT = 6 };

// program segments; the planner canonicalises the state between them so the
// body's push lists hold for every iteration of the PCG loop
enum RSeg : int { SEG_VCYCLE = 0, SEG_INIT = 1, SEG_FIRST = 2, SEG_BODY = 3, SEG_GATHER = 4, SEG_AMG_INIT = 5,
                  SEG_AMG_BODY = 6, SEG_COUNT = 7 };

// vectors of a level / of the PCG workspace, as the planner numbers them
enum RVec : int { LV_B = 0, LV_X, LV_R, LV_D0, LV_D1, LV_DJ, LV_DW, LV_COUNT };  // LV_DW: correction slots, one per patch entry
enum RWs : int { WS_X = 0, WS_R, WS_Z, WS_P, WS_AP, WS_B, WS_COUNT };

struct RStep {
  int kind = 0, level = 0;
  int mat = 0, epi = 0;       // RK_SPMV
  int dir = 0;                // RK_WAVE / RK_FWAVE (RK_FWAVE: dst = position of the wave in the direction's order)
  int64_t dst = 0, src = -1;
  bool init = false;
  bool down = false;          // RK_LEG
  int site = 0;               // reductions
  int vec = -1;               // RK_GATHER: vector id
};

// Host image of one level (what the planner needs to enumerate accesses)
struct RowsHostLevel {
  int64_t n = 0;
  bool split = false, coarsest = false;
  std::vector<int64_t> a_ptr, p_ptr, pt_ptr;
  std::vector<int32_t> a_idx, p_idx, pt_idx;
  std::vector<double> pt_val;
  // smoother
  int64_t nwave = 0;
  std::vector<int64_t> wave_ptr, patch_ptr, gen_ptr[2];
  std::vector<int32_t> patch_dofs, ownr[2], genrow[2], lastr, gcol;
  std::vector<uint8_t> in_first;
  std::vector<int8_t> owner;  // row -> rank
  // dataflow records (levels swept by k_flow_wave): per direction the byte
  // offsets of the patch records in execution order, and the records
  bool fw = false;
  int64_t ne = 0;
  std::vector<int64_t> rec_off[2];
  std::vector<unsigned char> recs[2];
};

// one patch record as the host sees it (layout: flow.cu rec_layout)
struct FlowRecView {
  int32_t k, e0, nt;
  const int32_t *dof, *ts, *xpart, *tslot;
};
FlowRecView flow_rec_view(const unsigned char* rec);

// One rank's share of a level
struct RowsShare {
  std::vector<int32_t> rows;                 // owned rows, ascending
  std::vector<int32_t> plist;                // its patches, wave-major
  std::vector<int64_t> poff;                 // nwave + 1 offsets into plist
  std::vector<int32_t> gen[2];               // its generic rows per direction (indices relative to the wave's first triple)
  std::vector<int64_t> goff[2];              // nwave + 1 offsets into gen[dir]
  std::vector<int64_t> fpos[2];              // fw levels: its record positions per direction, in execution order
  std::vector<int64_t> foff[2];              // nwave + 1 offsets into fpos[dir] (by position of the wave in the order)
};

// slab ownership of a graph (BFS level sets from a pseudo-peripheral node,
// cut into nranks chunks of equal nonzero count)
void rows_bfs_owner(int64_t n, const int64_t* ptr, const int32_t* idx, int nranks, std::vector<int8_t>& owner);
// coarse rows follow the fine DoF that carries the largest |P| entry of their column
void rows_coarse_owner(int64_t nc, const int64_t* pt_ptr, const int32_t* pt_idx, const double* pt_val,
                       const std::vector<int8_t>& fine_owner, std::vector<int8_t>& owner);
// the shares of every rank on one level (split: by owner; else everything on every rank)
void rows_shares(const RowsHostLevel& L, int nranks, std::vector<RowsShare>& out);

// vector numbering of a hierarchy of `depth` levels
inline int rows_vec_level(int level, int which) { return level * LV_COUNT + which; }
inline int rows_vec_ws(int depth, int which) { return depth * LV_COUNT + which; }
inline int rows_vec_red(int depth) { return depth * LV_COUNT + WS_COUNT; }
inline int rows_vec_count(int depth) { return depth * LV_COUNT + WS_COUNT + 1; }

// the step sequence of every segment for a hierarchy with the given wave counts
void rows_program(const std::vector<RowsHostLevel>& lv, std::vector<RStep> seg[SEG_COUNT]);

// accesses of one step for every rank
void rows_access(const RStep& st, const std::vector<RowsHostLevel>& lv, const std::vector<std::vector<RowsShare>>& sh,
                 int nranks, std::vector<PlanAccess>& acc);

struct RowsPlan {
  PlanResult push;                                // boundary ids are global over the segments
  std::vector<int32_t> seg_boundary[SEG_COUNT];   // per segment: boundary id in front of each step
  std::vector<char> barrier;                      // per boundary: ranks synchronise here
  int32_t nboundary = 0;
};

// plan every segment (canonical state between segments, see rows.cu)
void rows_plan_all(const std::vector<RowsHostLevel>& lv, const std::vector<std::vector<RowsShare>>& sh, int nranks,
                   const std::vector<RStep> seg[SEG_COUNT], RowsPlan& plan);

}  // namespace hcamg
