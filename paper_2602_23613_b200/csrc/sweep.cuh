// OSS-l1 smoothing legs (sweep2.cu) and the segmented restriction (sweep.cu).
#pragma once
#include "common.cuh"

namespace hcamg {

// Prefetching cluster leg (sweep2.cu): padded static structure per patch/row.
struct LegArgs {
  const int* stop;
  int64_t n, nwave, m;
  const int64_t* wave_ptr;
  const int64_t* gen_fw_ptr;
  const int64_t* gen_bw_ptr;
  const int8_t* pk;
  const int32_t* pdof;
  const double* pbinv;
  const int32_t* ocnt;
  const int32_t* ogc;
  const double* ogv;
  int64_t ng[2];
  const int32_t* gu[2];
  const int32_t* gcnt[2];
  const int32_t* ggc[2];
  const double* ggv[2];
  // fallbacks / overflow
  const int32_t* genrow_fw;
  const int32_t* genrow_bw;
  const int32_t* ownr_fw;
  const int32_t* ownr_bw;
  const int32_t* lastr;
  const uint8_t* in_first;
  const int64_t* patch_ptr;
  const int32_t* dofs;
  const int64_t* binv_off;
  const double* binv;
  const int32_t* gcol;
  const double* gval;
  const int64_t* ap;
  const int32_t* ai;
  const double* av;
  const double* l1;
  const double* b;
  double* x;
  double* r;
  double* d0;
  double* d1;
  double* dj;
  unsigned* gbar;     // grid-barrier word (cooperative leg only)
  long long* trace;   // optional: per (phase, warp) [start, arrive] globaltimer stamps
  int l2pf;           // grid leg: L2-prefetch the static data of the wave this many waves ahead (0: off)
};
void launch_leg(bool down, const LegArgs& args, cudaStream_t s);
// whole-GPU cooperative variant (grid.sync between wavefronts)
void launch_leg_grid(bool down, const LegArgs& args, cudaStream_t s);
int sweep_cluster_size();

// Dataflow leg (flow.cu): per-entry correction slots, no barrier inside the sweep.
struct FlowArgs {
  const int* stop;
  int64_t n, nwave, ne, npatch, recmax;
  const unsigned char* recs;  // patch records of this direction, in its execution order
  const int64_t* rec_off;     // npatch + 1 byte offsets
  double* d;                  // slots (sentinel between legs)
  const double* r0;           // the sweep's starting residual (down: b; up: r after the Jacobi step)
  double* x;
  unsigned* bar;              // [0] grid-barrier word, [1] patch ticket (both 0 between legs)
  unsigned spin_ns;           // back-off of the slot spin (0: pure spin)
  int gates;                  // wait on the latest-wave predecessors first (1) or poll every term (0)
  int dynamic;                // patches claimed from a ticket in execution order (1) or dealt round-robin (0)
  long long* trace;           // debug: per execution position {record ready, pulls done, stored, warp} (globaltimer)
};
void launch_flow_leg(bool down, const FlowArgs& args, cudaStream_t s);
// wave-parallel sweep over the same records (mode "fwave"): one launch per wavefront
void launch_flow_wave(bool down, const FlowArgs& args, int64_t i0, int64_t cnt, cudaStream_t s);
bool flow_wave_ok(int64_t kmax, int64_t recmax);
int64_t flow_smem_bytes(int64_t recmax);
void flow_reset_slots(double* d, int64_t ne, cudaStream_t s);

// y = T v for a CSR T with long rows: fixed 256-entry segments, one warp each,
// then an in-order reduction of the segment partials (deterministic).
struct SegPlan {
  int64_t nseg = 0;
  DBuf<int64_t> segoff;
  DBuf<int32_t> seg_row;
  DBuf<double> partial;
};
void build_segments(const DCsr& T, SegPlan& plan, cudaStream_t s);
void launch_segmented(const int* stop, const DCsr& T, const SegPlan& plan, const double* v, double* y,
                      cudaStream_t s);

}  // namespace hcamg
