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
// A_rest = A[row0 : row0 + mm, col0 : col0 + nr] of the column-major buffer A (m_total x n_total, lda)
// and V = Vb[vrow0 : vrow0 + mm, vcol0 : vcol0 + w] of the buffer Vb (v_rows x v_cols, ldv); the two
// row origins must have the same parity (TMA boxes start at even rows)
int wy_cluster(double* A, int64_t lda, int64_t m_total, int64_t n_total, int64_t row0, int64_t col0, int64_t mm,
               int nr, const double* Vb, int64_t ldv, int64_t v_rows, int64_t v_cols, int64_t vrow0, int64_t vcol0,
               const double* t, int64_t ldt, int w, cudaStream_t st, int64_t* launches);
int wy_update(double* a, int64_t lda, int64_t mm, int nr, const double* v, int64_t ldv, const double* t, int64_t ldt,
              int w, double* scratch, size_t scratch_bytes, unsigned int* bar, cudaStream_t st, int64_t* launches);

}  // namespace rq
