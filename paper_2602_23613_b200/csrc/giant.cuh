// Dense-interpolation regime (3D): one interior component with thousands of
// DoFs.  Its A_GG block is factored in packed lower-triangular tiles, the
// harmonic extension Z = A_GG^{-1} W' is kept as a dense row-major block, P
// is applied in hybrid form (sparse part + dense block) and the Galerkin
// product uses the Schur form with the solve residual (see giant.cu).
#pragma once

#include "common.cuh"
#include "dist.cuh"
#include "trisolve.cuh"

namespace hcamg {


// Factor the SPD matrix given as CSR (positions 0..n-1) into packed tiles and
// solve A Z = B for the row-major n x m right-hand side B (overwritten by Z).
// Throws Error(ENOTSPD_) with the reference's pivot semantics (scale =
// max |diag|, floor 1e-13 * scale).  With `fac`, the factor is kept and the
// blocked-sweep operators of trisolve.cuh are built from it (perm, Lc, pools,
// sweeps; the caller finishes with factorp_attach).
// With `D` (m x m, column-major, full symmetric): D = B^T A^{-1} B = Y^T Y,
// Y = L^{-1} B (the forward half of the solve, staircase-restricted: column c
// of Y is zero above the first row of its right-hand side), and, unless
// want_z, the backward solve is skipped and B is left as it was.
// With `Bs` (the right-hand side as CSR, n x m) and !want_z, B_rowmajor may be
// null: the permuted dense right-hand side is scattered straight from Bs, so
// the unpermuted dense copy (config 2: 35 GB, its allocation, fill and the
// 70 GB permutation pass) never exists.
void giant_factor_solve(const DCsr& Agg, double* B_rowmajor, int64_t m, cudaStream_t s, FactorP* fac = nullptr,
                        double* D = nullptr, bool want_z = true, const DCsr* Bs = nullptr);

// Reverse Cuthill-McKee order of a symmetric CSR pattern (scipy's
// csgraph.reverse_cuthill_mckee, which the reference's cholesky() applies,
// sparse.py:297); host C++.
std::vector<int32_t> rcm_order(int64_t n, const std::vector<int64_t>& ptr, const std::vector<int32_t>& idx);

// Hybrid interpolation data of one level.
struct HybridP {
  bool on = false;
  int64_t nG = 0, nc = 0;
  DBuf<int32_t> rows;   // DoF of each dense row (ascending)
  DBuf<double> Z;       // nG x nc row-major; P[rows[q], c] = -Z[q, c] (formed on demand: hybrid_ensure_z)
  DCsr Agg;             // the component block A_GG (component order) and its right-hand side W' (nG x nc):
  DCsr Wg;              // kept so Z = A_GG^{-1} W' can be formed when it is needed (export, explicit-Z apply)
  DBuf<double> D;       // setup only: W'^T A_GG^{-1} W' = Y^T Y (nc x nc) for the Galerkin product
  // restriction partials (deterministic chunked column reduction)
  int64_t chunk = 512, nchunk = 0;
  int64_t grp[kGroups + 1] = {};  // chunk boundaries of the kGroups reduction groups
  DBuf<double> partial;
  FactorP fac;          // A_GG^{-1} through its envelope factor (single-GPU solve)
};

// allocate the restriction partials (outside any graph capture)
void hybrid_prepare(HybridP& hp, cudaStream_t s);
// Form the explicit block Z = A_GG^{-1} W' if the setup did not keep it
// (one more factorisation and a full two-sided solve, ~4 s on config 2).
void hybrid_ensure_z(HybridP& hp, cudaStream_t s);
// The three products below take an optional distributed context `d` (rows
// split across ranks, results exchanged through exchange site `off`, see
// dist.cuh) and `part`: 0 = all, 1 = up to the exchange signal (producer),
// 2 = from the exchange wait on (consumer) -- the split lets tests emulate
// several ranks on one GPU without kernels that wait on each other.
// x[rows[q]] -= Z[q,:] . e   (prolongation, dense part)
void hybrid_prolong(const int* stop, const HybridP& hp, const double* e, double* x, cudaStream_t s,
                    const Dist* d = nullptr, size_t off = 0, int part = 0);
// x = M e for a dense row-major n x m matrix (HBM-streaming GEMV)
void dense_gemv_rows(const int* stop, int64_t n, int64_t m, const double* M, const double* e, double* x,
                     cudaStream_t s, const Dist* d = nullptr, size_t off = 0, int part = 0);
// bc -= Z^T r[rows]            (restriction, dense part; bc already holds P_s^T r)
void hybrid_restrict(const int* stop, HybridP& hp, const double* r, double* bc, cudaStream_t s,
                     const Dist* d = nullptr, size_t off = 0, int part = 0);

// A_c = P^T A P for P = P_s - S_G A_GG^{-1} W':
//   with hp.D (default): A_c = sym(P_s^T A P_s) - Y^T Y, Y = L^{-1} W' (L the
//     envelope Cholesky factor of A_GG; W'^T A_GG^{-1} W' = Y^T Y exactly);
//   with Z: A_c = sym(P_s^T A P_s) - sym(W'^T Z) - sym(Z^T rho), rho = W' - A_GG Z
//     (the residual term Z^T rho in fp64).
// Output canonical CSR (exact zeros dropped).
void galerkin_hybrid(const DCsr& A, const DCsr& Ps, const DCsr& Pst, const HybridP& hp, DCsr& Ac, cudaStream_t s);

// nnz of the materialised P (exact zeros of Z excluded)
int64_t hybrid_nnz(const DCsr& Ps, const HybridP& hp, cudaStream_t s);

// Materialise P = P_s - S_G Z as canonical CSR (exact zeros of Z dropped).
void hybrid_to_csr(const DCsr& Ps, const HybridP& hp, DCsr& P, cudaStream_t s);

}  // namespace hcamg
