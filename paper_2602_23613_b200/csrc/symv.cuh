// Coarsest solve with the lower triangle of the symmetric explicit inverse (symv.cu).
#pragma once
#include "common.cuh"

namespace hcamg {

struct SymPacked {
  static constexpr int kTile = 32;            // sub-tile: 32 x 32 doubles, row-major, 8 KB
  static constexpr int kBlk = 4;              // work item: 4 x 4 sub-tiles (128 rows x 128 columns)
  static constexpr int kRows = kTile * kBlk;  // rows / columns per item
  bool on = false;
  int64_t n = 0;
  int nb = 0;     // item rows (ceil(n / 128))
  int items = 0;  // nb (nb + 1) / 2 lower items, row-major order
  int grid = 0;
  DBuf<double> val;       // items back to back; diagonal items hold their 10 lower sub-tiles
  DBuf<int64_t> ioff;     // item offsets into val (items)
  DBuf<double> rowpart;   // per item: its 128 row sums
  DBuf<double> colpart;   // per item: its 128 transposed column sums
};

// From the full symmetric row-major n x n matrix.
void symv_build(const double* full, int64_t n, SymPacked& sp, cudaStream_t s);
// x = A b, reading the triangle once; deterministic order.
void symv_apply(const int* stop, const SymPacked& sp, const double* b, double* x, cudaStream_t s);

}  // namespace hcamg
