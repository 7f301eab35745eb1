// Solve phase: V(1,1) cycle with the OSS-l1 smoother, PCG and stand-alone
// AMG iteration, recorded into CUDA graphs (see solve.cu).
#pragma once
#include <vector>

#include "level.cuh"

namespace hcamg {

// Device control block shared by the PCG / AMG kernels.
struct Ctl {
  double bnorm, rel, prev_rel, tol;
  double rz, pAp, alpha, beta;
  long long it, maxit;
  int stop, converged, error, growth, zero_b, pad;
  unsigned int ticket[8];
};

enum CtlError : int { kErrNone = 0, kErrPAp = 1, kErrRz = 2 };

struct Workspace {
  int64_t n = 0;
  DBuf<Ctl> ctl;
  DBuf<double> part, part2;   // per-block partial sums (deterministic reductions)
  DBuf<double> hist;          // residual history (maxit)
  DBuf<double> x, r, z, p, Ap, b;
  DBuf<int> zero_flag;        // always-0 stop flag for stand-alone cycles
  void ensure(int64_t n_, int64_t maxit, cudaStream_t s);
};

extern long long* g_leg_trace;

int64_t coarse_gemv_min();

enum Piece : int { PC_DOWN = 0, PC_RESTRICT = 1, PC_COARSE = 2, PC_PROLONG = 3, PC_UP = 4 };

// One piece of a level's V-cycle (down leg, restriction, coarsest solve,
// prolongation, up leg); C is the next-coarser level (null on the coarsest).
// `part` (distributed solve only): 0 = whole piece, 1 = up to its exchange
// signal, 2 = from its exchange wait on (pieces without an exchange run
// entirely in part 1).
int64_t record_piece(int pc, DevLevel& L, DevLevel* C, const double* b, double* x, const int* stop, cudaStream_t s,
                     int part = 0);

// Record one V-cycle on `stream`: x0 := V(b0) for the finest level, reading
// b0 and writing x0 (level-0 work buffers are used for everything else).
// Every kernel returns immediately when *stop != 0.
int64_t record_vcycle(std::vector<DevLevel*>& lv, const double* b0, double* x0, const int* stop,
                      cudaStream_t s);

// PCG (multilevel.py:238-281) pieces.  `cond` is the WHILE-node handle
// (0 when the loop is driven from the host).
int64_t record_pcg_init(DevLevel& L0, Workspace& w, const double* b, const double* x0, cudaStream_t s,
                        unsigned long long cond);
int64_t record_pcg_first(std::vector<DevLevel*>& lv, Workspace& w, cudaStream_t s);
int64_t record_pcg_body(std::vector<DevLevel*>& lv, Workspace& w, cudaStream_t s, unsigned long long cond);

// Stand-alone AMG iteration (multilevel.py:204-235).
int64_t record_amg_init(DevLevel& L0, Workspace& w, const double* b, const double* x0, cudaStream_t s,
                        unsigned long long cond);
int64_t record_amg_body(std::vector<DevLevel*>& lv, Workspace& w, cudaStream_t s, unsigned long long cond);

// Sliced-ELLPACK SpMV layout for short-row operators (no-op otherwise).
void build_sell(DCsr& M, cudaStream_t s);

// y = A x (device), for the generic PCG path.
void apply_operator(const DCsr& A, const double* x, double* y, cudaStream_t s);

// Generic PCG vector kernels (arbitrary preconditioner driven from the host).
void generic_init(const DCsr& A, Workspace& w, cudaStream_t s);    // r = b - A x, norms
void generic_pap(const DCsr& A, Workspace& w, cudaStream_t s);     // Ap, pAp, alpha
void generic_update(Workspace& w, cudaStream_t s);                 // x, r, rel, history
void generic_rz(Workspace& w, bool first, cudaStream_t s);         // rz (first: p = z) / beta
void generic_p(Workspace& w, cudaStream_t s);                      // p = z + beta p
// b == 0 (multilevel.py:252-253): x = 0 whatever x0 was (on device, no sync)
void zero_x_if_zero_rhs(Workspace& w, cudaStream_t s);
// r = b - A x in scipy's rounding order (sequential rows, no FMA)
void residual_scipy_order(const DCsr& A, const double* x, const double* b, double* r, cudaStream_t s);
void vec_axpby(int64_t n, double a, const double* x, double b, const double* y, double* out, cudaStream_t s);
void vec_add(int64_t n, const double* a, const double* b, double* out, cudaStream_t s);  // out = a + b

}  // namespace hcamg
