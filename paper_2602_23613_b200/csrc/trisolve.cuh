// Factored interpolation block: P = P_s - S_G A_GG^{-1} W' applied through
// the envelope Cholesky factor of A_GG instead of the explicit dense block Z.
//
// The reference stores the harmonic extension explicitly (transfer.py:104-116:
// Z = cho_solve(A_cc, W[comp, keep]), P = R^T - Z scattered into P).  In the
// 3D dense regime Z is n_G x n_c dense (config 2: 35.2 GB) and every V-cycle
// streams it twice (P e and P^T r).  The same linear map is
//   P e   = P_s e   - S_G  A_GG^{-1} (W' e)
//   P^T r = P_s^T r - W'^T A_GG^{-1} (S_G^T r)
// and A_GG^{-1} v = perm^T L^{-T} L^{-1} perm v with L the RCM-envelope
// Cholesky factor (config 2: 5.7 GB of tiles).  Two triangular sweeps per
// application read ~2 x 5.7 GB instead of 35.2 GB.
//
// Each sweep is one cooperative kernel over the whole GPU, one step per
// NB-row block, one grid barrier per step.  Forward step k computes
//   y_k = Linv_kk u_k - M_k y_{k-1},  M_k = Linv_kk L_{k,k-1}
// (u_k already holds the contributions of y_0..y_{k-2}) and, in the same
// phase, folds y_{k-1} into the later blocks: u_i -= L_{i,k-1} y_{k-1}
// (i >= k+1).  The backward sweep is the same with Linv_kk^T, N_k =
// Linv_kk^T L_{k+1,k}^T and the transposed tiles.  Every output row is one
// warp's dot product in a fixed order, so a sweep is deterministic.
#pragma once
#include <functional>
#include <utility>
#include <vector>

#include "common.cuh"

namespace hcamg {

constexpr int64_t kTriNB = 1024;  // factor tile (giant.cu); work vectors are padded to T * kTriNB
// sweep block: one step solves kTriSB rows (kTriNB / 2, kTriNB or 2 kTriNB;
// measured on config 2 per restriction/prolongation: 512 -> 3.2-3.3 ms,
// 1024 -> 2.62 ms, 2048 -> 2.43 ms: fewer grid barriers for 7 % more bytes)
constexpr int64_t kTriSB = 2048;

// One step of a blocked sweep: rows of block k are the "critical" rows
// y_k = A u_k - B y_c (A row-major, lower (tri 0) or upper (tri 1)
// triangular; B row-major or null); tiles [t0, t1) fold y_c into other blocks.
// Source description of one sweep step (setup only): the critical rows of
// block k are y_k = A u_k - B y_c (A, B row-major NB x NB tiles; B may be
// null), and each fold (tile, blk) does u[blk] -= tile y_c.
// A kTriSB x kTriSB operator block as rows: row r = p[r * ld .. r * ld + kTriSB).
struct TriSrc {
  const double* p = nullptr;
  int64_t ld = 0;
};
struct TriSrcStep {
  int32_t k, c;  // sweep blocks (kTriSB rows each)
  TriSrc a, b;   // b.p == nullptr: no coupling block
  std::vector<std::pair<TriSrc, int64_t>> folds;
};

// Device form.  Every operator row is stored compactly (only its 64-column
// chunks [j0, j1) that hold nonzeros, so the envelope zeros and the zero half
// of the triangular Linv rows are never read), rows of one step contiguous
// and steps in execution order: a step's operator data is one contiguous
// region, which the kernel prefetches into L2 in equal slices per warp.
struct TriTask {
  int64_t a, b;   // row bases in the pool (chunk j at base + 64 j; bases >= 0);
                  // b < 0: fold task, the (-1 - b)-th fold into row `out` (step order)
  int32_t out;    // crit: y[out] = A.su - B.sy; fold: u[out] -= A.sy
  uint8_t ja0, ja1, jb0, jb1;
};
struct TriStepD {
  int32_t k, c;
  int64_t t0, t1;    // tasks
  int64_t pf0, pf1;  // byte range of the step's rows in the pool
};

struct TriBatch {
  int64_t t0, t1;      // tasks
  int64_t off, bytes;  // their rows: one contiguous pool byte range
};

struct TriSweep {
  int64_t nstep = 0, ntask = 0, T = 0;
  DBuf<TriStepD> steps;
  DBuf<TriTask> tasks;
  DBuf<double> pool;
  int64_t bytes = 0;  // operator bytes one sweep reads
  // dataflow kernel: nfold[k] = fold tasks into block k; flags = [ydone (nstep)
  // | ufull (T) | rowseq (T*NB)] counters, zeroed before every sweep
  DBuf<int32_t> nfold;
  DBuf<unsigned> flags;
  // TMA-streamed kernel: the tasks of step k for CTA c are contiguous,
  // [ctask[k (G+1) + c], ctask[k (G+1) + c + 1]) (split by bytes), and their
  // rows, one contiguous pool region, are cut into batches
  // [bptr[k G + c], bptr[k G + c + 1]) of whole tasks, <= one ring slot each
  int G = 0, max_cta_tasks = 0, max_cta_batches = 0, nbuf = 4;
  DBuf<int64_t> ctask, bptr, cptr;
  DBuf<TriBatch> batches, cbat;  // cbat: the batches again, per CTA in stream order ([cptr[c], cptr[c+1]))
  // host copies for re-partitioning (tri_partition / tri_calibrate): the tasks and
  // steps, the partition weights, per-(step, CTA) shares (empty: 1/G) and the
  // weight each CTA got
  std::vector<TriTask> htasks;
  std::vector<TriStepD> hsteps;
  int64_t taskw = 3072, critpct = 140;
  std::vector<double> share, hcost;
};

// Compact the source blocks into a sweep.  ranges(p) returns the host copy of
// the row-range table (kTriSB x {j0, j1}, 64-column chunks) of the block at p.
void tri_compact(const std::vector<TriSrcStep>& src, const std::function<const uint8_t*(const double*)>& ranges,
                 TriSweep& out, cudaStream_t s, int dir);  // dir: 0 forward, 1 backward sweep

struct FactorP {
  bool on = false;
  int64_t nG = 0, nc = 0, T = 0;
  DBuf<int32_t> perm;   // factored position -> position in the component (RCM order)
  TriSweep fw, bw;
  DBuf<int32_t> dof;    // factored position -> DoF of the level
  DCsr Wp, Wpt;         // W' with rows in factored order, and its transpose (n_c x n_G)
  DBuf<double> v0, v1, v2;  // T*NB work vectors
  DBuf<unsigned> bar;       // grid-barrier word (sense-reversing)
};

// Rows of W (in the component's member order given by mpos) and the level
// DoFs of the members (rows), both taken into factored order.
void factorp_attach(FactorP& f, const DCsr& W, const int32_t* mpos, const int32_t* rows, cudaStream_t s);

// bc -= W'^T A_GG^{-1} r[G]          (restriction, dense part)
void factorp_restrict(const int* stop, FactorP& f, const double* r, double* bc, cudaStream_t s);
// x[G] -= A_GG^{-1} W' e             (prolongation, dense part)
void factorp_prolong(const int* stop, FactorP& f, const double* e, double* x, cudaStream_t s);
// y = A_GG^{-1} v in factored order (v, y of length T*NB; v is overwritten)
void factorp_solve(const int* stop, FactorP& f, double* v, double* y, cudaStream_t s);

// the sweep fits the TMA-streamed kernel's per-CTA limits (else: grid-barrier kernel)
bool tri_tma_fits(const TriSweep& sw);
// (re)build the CTA partition and batches from the host copies (uses sw.share when set)
void tri_partition(TriSweep& sw, cudaStream_t s);
// time the sweep per (step, CTA) and re-partition to balance the CTAs (rounds; see trisolve.cu)
void tri_calibrate(TriSweep& sw, double* u, double* y, unsigned* bar, int rounds, cudaStream_t s);

// HCAMG_PAPPLY=z keeps the explicit-Z kernels (comparison); default: factor.
bool factorp_enabled();
// length of the padded work vectors (whole sweep blocks)
int64_t factorp_npad(const FactorP& f);

}  // namespace hcamg
