// Cooperative Householder sweep (see sweep.cu).
#pragma once
#include <algorithm>
#include <climits>

#include "common.cuh"

namespace rq {

// Scratch handed to the cooperative kernels: a flat device buffer plus a ring
// of zero-initialised grid-barrier counters (one fresh counter per launch).
struct SweepWork {
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  void* ll = nullptr;  // sketch CPQR: its slots + LL columns live here (sketch_ll_bytes(m)) instead of in scratch
  unsigned int* barriers = nullptr;  // ring, zeroed by the owner
  int nbarriers = 0;
  int next = 0;
  bool wrapped = false;
  unsigned int* next_barrier() {
    unsigned int* b = barriers + next;
    if (++next == nbarriers) {
      next = 0;
      wrapped = true;
    }
    return b;
  }
};

struct SweepCall {
  double* a;
  int64_t lda;
  int64_t m;
  int n;
  int n_acc = 0;
  int steps;
  int pivot;
  const int* init_pos = nullptr;
  double* v = nullptr;
  int64_t ldv = 0;
  int* col_at_pos = nullptr;
  double* r_out = nullptr;
  int64_t ldr = 0;
  int grid = 0;
};

size_t sweep_workspace_bytes(int64_t m, int total_cols, int grid);
size_t sketch_ll_column_bytes(int m);
size_t sketch_ll_bytes(int m);  // slots + LL columns of the register sketch CPQR
size_t sketch_workspace_bytes(int m, int n);  // register-resident sketch CPQR (LL exchange) of n columns
// Smallest grid a sketch CPQR launch is given (the overlapped schedule leaves 16 SMs to the b x b
// CPQR's cluster); workspace sizes cover it.
constexpr int kSkMinGrid = kSMs - 16;
bool sketch_cpqr_preserves_input(int m, int n, int gmax = 0);
int sweep_grid_size(int total_cols);
int sweep_debug_timing(int on, unsigned long long* host, int count);
int sweep_launch(const SweepCall& c, SweepWork& w, cudaStream_t st, int64_t* launches);

// Pivot selection only (sketch CPQR): chosen[0..steps) = columns in pivot order.
// y (m x n, ld) is overwritten.  m <= 1024.
int sketch_cpqr_launch(const double* y, int64_t ld, int m, int n, int steps, const int* init_pos, int* chosen,
                       SweepWork& w, unsigned long long* counter, unsigned long long& counter_base, cudaStream_t st,
                       int64_t* launches, int gmax = 0);


// Batched sketch CPQR (sketch_batch.cu): the same greedy pivots with one grid-wide exchange per
// batch of provable pivots.  y is only read.  ws: sketch_batch_workspace_bytes(), zero at
// allocation, private to the context.  Returns -1 when the shape does not fit.
size_t sketch_batch_workspace_bytes();
bool sketch_batch_fits(int m, int n, int steps, int gmax = 0);
int sketch_batch_launch(const double* y, int64_t ld, int m, int n, int steps, const int* init_pos, int* chosen,
                        void* ws, unsigned long long& stamp_base, cudaStream_t st, int64_t* launches, int gmax = 0);

}  // namespace rq
