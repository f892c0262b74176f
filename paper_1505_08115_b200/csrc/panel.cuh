// Cluster leaf QR (see panel.cu).
#pragma once
#include "common.cuh"

namespace rq {

struct LeafCall {
  double* a;     // leaf top-left (rows mm, cols w), overwritten with R (zeros below diag)
  int64_t lda;
  int64_t mm;
  int w;
  double* v;     // mm x w unit reflectors (zeros above the diagonal)
  int64_t ldv;
  double* tl;    // w x w upper-triangular T (may be null)
  int64_t ldt;
};

int leaf_width_for(int64_t mm);
int leaf_reg_width_for(int64_t mm);
int leaf_debug_timing(int on, unsigned long long* host, int count);
int leaf_qr(const LeafCall& c, cudaStream_t st, int64_t* launches);
bool wy_update_fits(int64_t mm, int nr, int w);
int wy_cluster(double* a, int64_t lda, int64_t mm, int nr, const double* v, int64_t ldv, const double* t,
               int64_t ldt, int w, cudaStream_t st, int64_t* launches);
int wy_update(double* a, int64_t lda, int64_t mm, int nr, const double* v, int64_t ldv, const double* t, int64_t ldt,
              int w, double* scratch, size_t scratch_bytes, unsigned int* bar, cudaStream_t st, int64_t* launches);

}  // namespace rq
