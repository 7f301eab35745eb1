// Device side of the subdomain row partition (rows.cuh): one rank's lists,
// the symmetric vector buffer every peer maps, the push tables and the
// boundary kernel.
#pragma once
#include <memory>
#include <vector>

#include "level.cuh"
#include "rows.cuh"
#include "solve.cuh"

namespace hcamg {

struct RowsLevelDev {
  bool split = false;
  int64_t nrows = 0;
  DBuf<int32_t> rows;
  DBuf<int32_t> plist;
  std::vector<int64_t> poff;
  DBuf<int32_t> gen[2];
  std::vector<int64_t> goff[2];
  // levels swept over the dataflow records: this rank's records, compacted in
  // execution order, and their per-wave offsets
  bool fw = false;
  DBuf<unsigned char> frecs[2];
  DBuf<int64_t> frec_off[2];
  std::vector<int64_t> foff[2];
  // sliced-ELLPACK copies of this rank's rows of A, P (rows of the level) and P^T (rows of the next level)
  std::unique_ptr<DSell> sA, sP, sPt;
};

// what the boundary kernel needs, by value
struct XPush {
  char* base[kRowsMaxRanks];        // every rank's symmetric buffer as mapped here
  int rank, nranks;
  const int64_t* voff;              // byte offset of every vector inside a symmetric buffer
  const int32_t* idx;               // push entries
  const int64_t* seg_cum;           // per segment of this boundary: first thread (nseg + 1)
  const int64_t* seg_off;           // per segment: first entry in idx
  const int32_t* seg_dst;
  const int32_t* seg_vec;
  int nseg;
  unsigned long long* ep;           // this rank's boundary epoch
  unsigned* cta;
  int* err;
  int wait;                         // 0: signal only (lockstep emulation waits in a second launch)
};

constexpr size_t kRowsFlagBytes = 256;

struct RowsStats {
  int64_t boundaries[SEG_COUNT] = {}, barriers[SEG_COUNT] = {};
  int64_t push_out[SEG_COUNT] = {};   // entries this rank sends per execution of the segment
  int64_t push_all[SEG_COUNT] = {};   // entries all ranks send
  int64_t own_rows0 = 0, ghost_rows0 = 0;  // level 0: owned rows / distinct foreign columns of A's owned rows
  int32_t split_levels = 0;
};

struct RowsCtx {
  int rank = 0, nranks = 1;
  bool on = false;
  int64_t min_rows = 0;
  int depth = 0;
  std::vector<RowsLevelDev> lev;
  std::vector<RStep> seg[SEG_COUNT];
  std::vector<int32_t> seg_boundary[SEG_COUNT];
  std::vector<char> barrier;
  // this rank's push tables, per boundary [bfirst[b], bfirst[b + 1]) segments
  std::vector<int64_t> bfirst, bcount;
  DBuf<int32_t> xidx, seg_dst, seg_vec;
  DBuf<int64_t> seg_cum, seg_off, d_voff;
  // symmetric memory
  char* sym = nullptr;
  size_t sym_bytes = 0;
  char* base[kRowsMaxRanks] = {};
  bool opened[kRowsMaxRanks] = {};
  std::vector<int64_t> voff;        // bytes
  std::vector<int64_t> vlen;        // entries
  DBuf<unsigned long long> ep;
  DBuf<unsigned> cta;
  DBuf<int> err;
  RowsStats stats;
  double* vec(int id) const { return reinterpret_cast<double*>(sym + voff[(size_t)id]); }
  void release();
  ~RowsCtx() { release(); }
};

// solve.cu: launch one step's kernel for this rank (no-op for RK_GATHER); returns launches
int64_t rows_launch_step(const RStep& st, RowsCtx& rc, std::vector<DevLevel*>& lv, Workspace& w, const int* stop,
                         unsigned long long cond, cudaStream_t s);

// solve.cu: the leg kernels record_piece would run on this level with the handle's options
int leg_mode(const DevLevel& L);
// solve.cu: sliced-ELLPACK copy of the listed rows of M (null when the rows are not short)
std::unique_ptr<DSell> build_sell_rows(const DCsr& M, const int32_t* rows, int64_t nrows, cudaStream_t s);

// rows.cu
// Build the context of `rank` for the resident hierarchy: ownership, lists,
// program, plan, symmetric buffer (vectors of `lv` and `w` are re-pointed into it).
void rows_prepare(RowsCtx& rc, std::vector<DevLevel*>& lv, Workspace& w, int rank, int nranks, int64_t min_rows,
                  cudaStream_t s);
// Undo the re-pointing (fresh private vectors).
void rows_detach(RowsCtx& rc, std::vector<DevLevel*>& lv, Workspace& w, cudaStream_t s);
// boundary in front of step k of segment g: push + signal (+ wait when `wait`)
int64_t rows_boundary(RowsCtx& rc, int g, size_t k, const int* stop, bool wait, cudaStream_t s);
void rows_wait(RowsCtx& rc, const int* stop, cudaStream_t s);
// record a whole segment (boundaries + steps) on a stream
int64_t rows_record(RowsCtx& rc, int g, std::vector<DevLevel*>& lv, Workspace& w, const int* stop,
                    unsigned long long cond, cudaStream_t s);

}  // namespace hcamg
