/*
 * libhcamg — C-ABI of the B200-native AMG-PCG hot path for lowest-order
 * Nédélec H(curl) systems (arXiv 2602.23613).
 *
 * The reference package exposes this path as Python functions in
 * hcurl_amg/multilevel.py; every entry point below replaces one of them and
 * is what a ctypes / cffi binding of that module binds (INTEGRATION.md shows
 * the binding).  Plain pointers and sizes only: matrices are canonical CSR
 * (int64 row pointers, int32 column indices, fp64 values, sorted, no stored
 * zeros — the normal form of hcurl_amg/sparse.py:58-65); vectors are fp64.
 *
 * Return codes: 0 on success, a negative HCAMG_E* code otherwise; the
 * message is available from hcamg_last_error() and, for HCAMG_ENOTSPD, the
 * failing pivot from hcamg_error_index().  Calls on one handle are not
 * thread-safe; distinct handles are independent.  One handle = one device
 * and one CUDA stream; every matrix of the hierarchy stays resident in HBM
 * between calls.
 */
#ifndef HCAMG_H_
#define HCAMG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HCAMG_OK 0
#define HCAMG_EINVAL (-1)      /* ValueError (shapes, method, malformed G)      */
#define HCAMG_ENOTSPD (-2)     /* NotPositiveDefiniteError(pivot)  sparse.py:50 */
#define HCAMG_EBREAKDOWN (-3)  /* RuntimeError("PCG breakdown…") multilevel.py:265,278 */
#define HCAMG_ENOMEM (-4)
#define HCAMG_ECUDA (-5)
#define HCAMG_ENOTSYM (-6)     /* ValueError("matrix not symmetric…") sparse.py:294 */
#define HCAMG_EUNSUPPORTED (-7)

typedef struct hcamg_handle hcamg_handle;

/* Host CSR view (read-only). */
typedef struct {
  int64_t nrows, ncols;
  const int64_t* indptr;   /* nrows + 1 */
  const int32_t* indices;  /* indptr[nrows] */
  const double* data;      /* indptr[nrows] */
} hcamg_csr;

/* Solve report (multilevel.py:62-68 SolveReport, minus the history array,
 * which is written to a caller buffer). */
typedef struct {
  int64_t iterations;
  int32_t converged;
  int32_t zero_rhs;        /* b == 0: x = 0, 0 iterations */
  int32_t diverged;        /* amg_solve divergence guard fired (multilevel.py:230-233) */
  int32_t pad;
  double final_relres;
} hcamg_report;

/* Hierarchy summary (multilevel.py:50-59 Hierarchy). */
typedef struct {
  int32_t depth;
  int32_t stalled;
  int32_t method;          /* 0 = "ref", 1 = "alg", 2 = user-assembled */
  int32_t pad;
  double operator_complexity;   /* multilevel.py:199-201 */
  double setup_seconds;         /* device-synchronised wall time of the setup */
  double setup_flops;           /* FP64 flops of the dense setup work (Cholesky, triangular solves, Y^T Y,
                                   coarsest factor and inverse), counted from the call dimensions */
} hcamg_info;

/* Per-level sizes for exports. */
typedef struct {
  int64_t n, nnz_A, ncols_G, nnz_G, nnz_P, n_pairs, n_interior, n_coarse_nodes;
  int64_t n_patches, n_patch_entries, n_waves, n_gc_cols, coarsest, n_components, max_component, pad;
  /* dense regime, single GPU: the V-cycle applies A_GG^{-1} through the
   * envelope Cholesky factor (two blocked sweeps of factor_steps steps);
   * factor_bytes = operator bytes one application reads (0: explicit Z);
   * factor_tma = 1 when both sweeps fit the TMA-streamed kernel's per-CTA
   * limits (otherwise they run on the grid-barrier kernel). */
  int64_t factor_bytes, factor_steps, factor_tma;
} hcamg_level_info;

/* ---- lifetime ---------------------------------------------------------- */
int hcamg_create(hcamg_handle** out, int device, void* cuda_stream /* NULL: own stream */);
void hcamg_destroy(hcamg_handle* h);
const char* hcamg_last_error(const hcamg_handle* h);
int64_t hcamg_error_index(const hcamg_handle* h);
int hcamg_version(void);

/* ---- per-handle options ------------------------------------------------
 * Select code paths per handle (they seed from the HCAMG_* environment at
 * hcamg_create).  Keys: "sweep" (smoothing leg: 0 auto, 1 cluster leg, 2 grid
 * leg, 3 one launch per wavefront, 4 dataflow leg, 5 one launch per wavefront
 * over the dataflow records), "giant_min" (dense-regime
 * cutoff, reference transfer.py:35 _DENSE_COMPONENT_CUTOFF = 4096),
 * "coarse_gemv_min" (coarsest solve streams its inverse from this size on),
 * "coarse_symv" (packed-triangle coarsest solve), "factor_apply" (apply the dense
 * interpolation block through the envelope factor, 0 = explicit Z),
 * "form_z" (keep the explicit Z block), "tri_calib" (sweep calibration rounds).
 * Setting an option drops the recorded solve graphs; setup options apply to
 * the next hcamg_setup_*.  Unknown keys: HCAMG_EINVAL. */
int hcamg_set_option(hcamg_handle* h, const char* key, double value);
int hcamg_get_option(hcamg_handle* h, const char* key, double* value);

/* ---- setup: build_hierarchy (multilevel.py:78-164) ---------------------- */
/* method "alg": splitting.py:246-298 + transfer.py:77-122 per level. */
int hcamg_setup_alg(hcamg_handle* h, const hcamg_csr* A, const hcamg_csr* G, int32_t max_levels,
                    int64_t min_coarse, double theta, hcamg_info* info);
/* method "ref": the nested mesh chain, coarsest first (multilevel.py:118-131,
 * splitting.py:301-330).  edges[i]: ne[i] x 2 (tail < head) of mesh i;
 * children[i]: ne[i] x 2 fine-edge ids of coarse edge E of mesh i in mesh i+1
 * (RefinementMap.coarse_edge_children); free_edges: finest mesh edge -> DoF
 * (-1 eliminated). */
int hcamg_setup_ref(hcamg_handle* h, const hcamg_csr* A, const hcamg_csr* G, int32_t n_meshes,
                    const int64_t* ne, const int64_t* const* edges, const int64_t* const* children,
                    const int64_t* free_edges, int32_t max_levels, int64_t min_coarse, hcamg_info* info);
/* user-assembled hierarchy (Hierarchy(levels=[Level(A, G, P)...]) built by
 * hand, as tests/test_multilevel.py:125-134 does): push levels finest first;
 * a level with P == NULL is the coarsest and is factored directly
 * (sparse.py:276-301). */
int hcamg_hier_begin(hcamg_handle* h);
int hcamg_hier_push(hcamg_handle* h, const hcamg_csr* A, const hcamg_csr* G /* may be NULL */,
                    const hcamg_csr* P /* NULL: coarsest */);
int hcamg_hier_end(hcamg_handle* h, hcamg_info* info);
/* as hcamg_hier_end, but the coarsest solve applies coarse_matrix^{-1}: the
 * matrix whose Cholesky factor the user attached as Level.coarse_factor. */
int hcamg_hier_end_with(hcamg_handle* h, const hcamg_csr* coarse_matrix, hcamg_info* info);

/* ---- level-0 splitting only: build_algebraic_splitting (splitting.py:246-298)
 * on (A, G) without the interpolation; sizes[4] = n_pairs, n_interior,
 * n_coarse_nodes, n_candidate_triples.  Lets the bit-exact integer parity be
 * checked at sizes whose full hierarchy is infeasible. */
int hcamg_split_alg(hcamg_handle* h, const hcamg_csr* A, const hcamg_csr* G, double theta, int64_t* sizes);
int hcamg_split_export(hcamg_handle* h, int64_t* pairs, int64_t* interior, int64_t* coarse_nodes);

/* ---- queries / exports (lazily materialised Level fields) -------------- */
int hcamg_info_get(hcamg_handle* h, hcamg_info* info);
int hcamg_notes(hcamg_handle* h, char* buf, int64_t cap);   /* '\n'-separated Hierarchy.notes */
int hcamg_level(hcamg_handle* h, int32_t level, hcamg_level_info* out);
/* which: 0 = A, 1 = P, 2 = G.  Buffers sized from hcamg_level. */
int hcamg_export_csr(hcamg_handle* h, int32_t level, int32_t which, int64_t* indptr, int32_t* indices,
                     double* data);
/* pairs: n_pairs x 7 (dof1, dof2, sign1, sign2, tail, mid, head); interior:
 * n_interior; coarse_nodes: n_coarse_nodes (algebraic c_G) or mesh edges
 * of the pairs (refinement route); any pointer may be NULL. */
int hcamg_export_splitting(hcamg_handle* h, int32_t level, int64_t* pairs, int64_t* interior,
                           int64_t* coarse_nodes);
int hcamg_export_l1(hcamg_handle* h, int32_t level, double* d);
/* Dense-regime data: which 0 = interpolation block Z (n_G x n_c row-major,
 * P[rows[q], c] = -Z[q, c]), 1 = its DoF rows (int64), 2 = the coarsest
 * level's dense inverse (n x n).  hcamg_export_csr which = 3 gives the sparse
 * part of a hybrid P; hcamg_level_info.max_component = n_G, .pad = its nnz. */
int hcamg_export_dense(hcamg_handle* h, int32_t level, int32_t which, void* out);
/* out = A_GG^{-1} v through the factored block (two blocked triangular sweeps,
 * csrc/trisolve.cu); v, out of length n_G in the member order of
 * hcamg_export_dense(which = 1).  Test/inspection entry (transfer.py:104). */
int hcamg_component_solve(hcamg_handle* h, int32_t level, const double* v, double* out);
/* ---- input generation: 3D Kuhn-cube curl-curl system on the GPU ---------
 * (the 3D analogue of fem.py:143-195 assemble(); lexicographic vertex numbering;
 * paper_2602_23613_b200/kuhn.py is the host restatement).  muinv: 6 n^3 per-tet
 * mu^{-1} (cube-major, permutation-minor); S6, M6: 6 x 36 element matrices of the
 * six tet shapes.  sizes[6] = {n_free_edges, nnz(A), n_free_nodes, nnz(G),
 * n_edges, n_vertices}; hcamg_kuhn_export then copies A, G (canonical CSR) and the
 * full -> free index maps (-1: eliminated) into caller buffers. */
int hcamg_kuhn_assemble(hcamg_handle* h, int64_t n, const double* muinv, double beta, const double* S6,
                        const double* M6, int64_t* sizes);
int hcamg_kuhn_export(hcamg_handle* h, int64_t* a_ptr, int32_t* a_idx, double* a_val, int64_t* g_ptr,
                      int32_t* g_idx, double* g_val, int64_t* free_edges, int64_t* free_nodes);
/* patches in reference order: ptr (n_patches + 1), dofs (n_patch_entries), wave of each patch */
int hcamg_export_patches(hcamg_handle* h, int32_t level, int64_t* ptr, int64_t* dofs, int64_t* wave);
int hcamg_export_coarse_cols(hcamg_handle* h, int32_t level, int64_t* cols);

/* coarsest level's solve (sparse.py:304-321 solve(factor, b)): x = A_c^{-1} b
 * for host vectors of the coarsest size; HCAMG_EINVAL on any other level. */
int hcamg_coarse_solve(hcamg_handle* h, int32_t level, const double* b, double* x);

/* The coarse level's Cholesky factor as the reference's CholeskyFactor holds
 * it (sparse.py:146-165, 276-301): ordering = reverse Cuthill-McKee
 * permutation (n), factor = dense lower L (n x n row-major) with
 * L L^T = A[ordering][:, ordering].  Either pointer may be NULL. */
int hcamg_cholesky_factor(hcamg_handle* h, int32_t level, int64_t* ordering, double* factor);

/* ---- OSS-l1 smoother (smoothers.py:60-137) ------------------------------
 * hcamg_smoother_setup: build_patches + build_l1_jacobi for one operator
 * (A, G_level) into the handle (replacing any hierarchy; the handle then only
 * smooths).  hcamg_smooth: smooth(A, patches, l1, x, b, direction) of level
 * `level` (0 on a smoother handle); direction 0 forward, 1 backward,
 * 2 symmetric; x NULL = zeros; out = the new iterate. */
int hcamg_smoother_setup(hcamg_handle* h, const hcamg_csr* A, const hcamg_csr* G);
int hcamg_smooth(hcamg_handle* h, int32_t level, int32_t direction, const double* x_or_null, const double* b,
                 double* out);

/* ---- solve ------------------------------------------------------------- */
/* vcycle(h, b, x=None) (multilevel.py:187-196): out = x + V(b - A x), or V(b). */
int hcamg_vcycle(hcamg_handle* h, const double* b, const double* x_or_null, double* out);
/* pcg(A, b, precond=lambda r: vcycle(h, r), x0, tol, maxit) (multilevel.py:238-281)
 * with A = the finest operator; history: maxit doubles (may be NULL). */
int hcamg_pcg(hcamg_handle* h, const double* b, const double* x0_or_null, double tol, int64_t maxit,
              double* x, double* history, hcamg_report* report);
/* amg_solve(h, b, x0, tol, maxit) (multilevel.py:204-235). */
int hcamg_amg_solve(hcamg_handle* h, const double* b, const double* x0_or_null, double tol, int64_t maxit,
                    double* x, double* history, hcamg_report* report);
/* Device-resident variant of hcamg_pcg: b, x0, x are device pointers on the
 * handle's device; no host synchronisation when report == NULL -- breakdown
 * and peer errors are then deferred to hcamg_solve_status. */
int hcamg_pcg_device(hcamg_handle* h, const double* d_b, const double* d_x0_or_null, double tol,
                     int64_t maxit, double* d_x, hcamg_report* report);
/* Report and status of the last PCG / AMG solve on the handle (synchronises):
 * HCAMG_EBREAKDOWN or HCAMG_ECUDA if it broke down or a peer timed out. */
int hcamg_solve_status(hcamg_handle* h, hcamg_report* report);
/* Kernel launches recorded in the last PCG / V-cycle graph (gpu_launches). */
int64_t hcamg_graph_launches(hcamg_handle* h, int32_t which /* 0 vcycle, 1 pcg init, 2 pcg body */);
/* Time each piece of the V-cycle alone (warm, CUDA events on the handle's
 * stream, reps launches each): kind 0 down leg, 1 restriction, 2 coarsest
 * solve, 3 prolongation, 4 up leg; writes up to cap records, *count set. */
int hcamg_profile_vcycle(hcamg_handle* h, int32_t reps, int32_t cap, int32_t* kind, int32_t* level, double* us,
                         int64_t* launches, int32_t* count);
/* Device stream of the handle (cudaStream_t) for event timing. */
void* hcamg_stream(hcamg_handle* h);

/* ---- generic PCG with a host preconditioner (any `precond` callable) ---- */
typedef int (*hcamg_precond_fn)(const double* r, double* z, int64_t n, void* ctx);
/* A: any square operator (uploaded); precond called with host vectors. */
int hcamg_pcg_generic(hcamg_handle* h, const hcamg_csr* A, const double* b, const double* x0_or_null,
                      double tol, int64_t maxit, hcamg_precond_fn precond, void* ctx, double* x,
                      double* history, hcamg_report* report);
/* y = A x on the device (A uploaded per call; used by the drop-in for A @ x). */
int hcamg_spmv(hcamg_handle* h, const hcamg_csr* A, const double* x, double* y);

/* ---- Row-partitioned solve across GPUs (one process per GPU, NVLink peer memory).
 * the reference is single-process; this replaces nothing in it
 * and is what a multi-GPU caller of pcg / vcycle / amg_solve (multilevel.py:238,
 * 187, 204) adds after build_hierarchy (multilevel.py:78).  Every rank builds the
 * same hierarchy (setup is replicated); in the solve each rank streams only its
 * rows of the dense interpolation blocks and of the coarsest inverse and
 * exchanges the results through a symmetric buffer mapped by every rank.  The
 * solution is bit-identical to the single-GPU solve for every rank count.
 * Protocol: every rank calls hcamg_dist_prepare (after setup), the callers
 * all-gather the 64-byte IPC handles in rank order, every rank calls
 * hcamg_dist_connect; from then on vcycle / pcg / amg_solve on the handle are
 * collective (all ranks must call them in the same order). */
/* Allocate this rank's exchange buffer; ipc_handle (64 bytes, may be NULL)
 * receives its CUDA IPC handle, dev_ptr (may be NULL) its device address. */
int hcamg_dist_prepare(hcamg_handle* h, int32_t rank, int32_t nranks, void* ipc_handle, void** dev_ptr);
/* Map the peers' buffers: ipc_handles = nranks x 64 bytes in rank order. */
int hcamg_dist_connect(hcamg_handle* h, const void* ipc_handles);
/* Same, for ranks living in one process on one device (bufs[r] = rank r's dev_ptr). */
int hcamg_dist_connect_ptrs(hcamg_handle* h, void* const* bufs);
/* Back to the single-GPU solve. */
int hcamg_dist_disconnect(hcamg_handle* h);
int hcamg_dist_info(hcamg_handle* h, int32_t* rank, int32_t* nranks, int32_t* connected, int64_t* buffer_bytes);

/* ---- Subdomain row partition of the sparse regime (the north-star
 * layout; csrc/rows.cuh).  Every level with at least `min_rows` rows is split by rows
 * into one subdomain per rank (BFS slabs of A's graph on level 0, coarse rows follow
 * the fine DoF carrying their largest |P| entry); each rank computes its rows of every
 * SpMV (multilevel.py:177-184), its patches of every smoother wavefront
 * (smoothers.py:98-109), its rows of P / P^T and its partial CG dot products
 * (multilevel.py:238-281), and pushes the entries a neighbour reads next into that
 * neighbour's vectors over NVLink peer memory; coarser levels are agglomerated (kept
 * whole and solved redundantly on every rank).  The V-cycle is bit-identical to the
 * single-GPU per-wavefront V-cycle; PCG differs by the grouping of its dot products.
 * Protocol as hcamg_dist_*: prepare on every rank, all-gather the 64-byte IPC handles,
 * connect; vcycle / pcg then are collective.  b, x0 are passed in full by every rank
 * and x is returned in full to every rank. */
int hcamg_rows_prepare(hcamg_handle* h, int32_t rank, int32_t nranks, int64_t min_rows, void* ipc_handle,
                       void** dev_ptr);
int hcamg_rows_connect(hcamg_handle* h, const void* ipc_handles);
int hcamg_rows_connect_ptrs(hcamg_handle* h, void* const* bufs);
int hcamg_rows_disconnect(hcamg_handle* h);
/* out[0..cap): rank, nranks, connected, split levels, buffer bytes, owned rows and ghost
 * columns of level 0, then per program segment (V-cycle, PCG init, first, body, gather):
 * steps, barriers, entries this rank pushes, entries all ranks push. */
int hcamg_rows_info(hcamg_handle* h, int64_t* out, int32_t cap);
/* Lockstep emulation of an n-rank partitioned solve on ONE GPU (tests): hs = n handles
 * of this process holding the same hierarchy, prepared as ranks 0..n-1 and connected with
 * hcamg_rows_connect_ptrs.  kind 0: z = V(b); kind 1: PCG from x0 = 0; kind 2: the
 * stand-alone AMG iteration from x0 = 0.  x: n x n0 doubles,
 * row r = the full result as rank r holds it.  poison != 0 fills the working vectors with
 * NaN first (an entry neither computed nor received then shows). */
int hcamg_rows_emulate(hcamg_handle* const* hs, int32_t n, int32_t kind, const double* b, double* x, double tol,
                       int64_t maxit, int32_t poison, hcamg_report* report);

/* The partition's planner, host only (no GPU needed; csrc/rows_plan.cu).  Ownership:
 * owner[u] = rank of row u (BFS slabs of the graph, equal nonzero counts).  Planner: a
 * symbolic walk over steps; each step lists, per rank, the (vector, entry) pairs it reads
 * and writes; a read of an entry the rank does not hold becomes a push (producer ->
 * reader) at the boundary in front of the step (= the step's index). */
typedef struct hcamg_plan hcamg_plan;
int hcamg_rows_owner(int64_t n, const int64_t* indptr, const int32_t* indices, int32_t nranks, int8_t* owner);
int hcamg_plan_create(hcamg_plan** out, int32_t nranks, int32_t nvec, const int64_t* vec_len);
int hcamg_plan_destroy(hcamg_plan* p);
/* entries of `vec` are held by the ranks in `holder_mask`; owner != NULL: only by owner[i] */
int hcamg_plan_set_vector(hcamg_plan* p, int32_t vec, int32_t holder_mask, const int8_t* owner);
int hcamg_plan_invalidate(hcamg_plan* p, int32_t vec);
/* nreads / nwrites: per rank counts; rvec / ridx, wvec / widx: the accesses, rank after rank */
int hcamg_plan_step(hcamg_plan* p, const int64_t* nreads, const int32_t* rvec, const int32_t* ridx,
                    const int64_t* nwrites, const int32_t* wvec, const int32_t* widx);
/* counts[0] = push segments, counts[1] = push entries, counts[2] = reads of undefined entries */
int hcamg_plan_counts(hcamg_plan* p, int64_t* counts);
/* seg: 5 ints per segment (boundary, src, dst, vec, count); idx: the entries, segment after segment */
int hcamg_plan_pushes(hcamg_plan* p, int32_t* seg, int32_t* idx);

#ifdef __cplusplus
}
#endif
#endif /* HCAMG_H_ */
