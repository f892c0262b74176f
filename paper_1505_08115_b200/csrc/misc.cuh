// Helper kernels around the panel loop (see misc.cu).
#pragma once
#include "common.cuh"

namespace rq {

int trailing_frobenius(const double* R, int64_t n, int64_t ldr, double* e2, cudaStream_t st, int64_t* launches);
int normalize_col(double* x, int64_t n, double* norms, int it, cudaStream_t st, int64_t* launches);
int trinv_upper(const double* R, int64_t ldr, int k, double* X, int64_t ldx, cudaStream_t st, int64_t* launches);
int q_from_reflectors(const double* V, int64_t ldv, int k, int n, double* Q, int64_t ldq, cudaStream_t st,
                      int64_t* launches);
int tfactor_from_gram(const double* G, int64_t ldg, int k, double* T, int64_t ldt, cudaStream_t st,
                      int64_t* launches);

struct PlanCall {
  const int* chosen;
  int b;
  const int* lorder;
  int np;
  unsigned char* flag;  // np
  int* newloc;          // np
  int* src;             // 2b
  int* dst;             // 2b
  int* nmoves;          // 1
  int* lorder_next;     // np - b
  int* rank_next;       // np - b
};
int plan_moves(const PlanCall& c, cudaStream_t st, int64_t* launches);

struct MoveCall {
  double* A;
  int64_t lda;
  int64_t coff;  // column offset of local index 0
  int64_t r0, r1;
  const int* src;
  const int* dst;
  const int* count;  // device count (or null: maxn)
  int maxn;
  double* stage;
  int64_t lds;
  int64_t* orig;     // optional label array moved alongside
  int64_t* ostage;
  unsigned long long* bytes = nullptr;  // profiling: += HBM bytes moved (device counter)
};
int move_columns(const MoveCall& c, cudaStream_t st, int64_t* launches);

int iota(int* a, int n, int64_t* b, int64_t nb, cudaStream_t st, int64_t* launches);
int fill_eye(double* X, int64_t ldx, int64_t rows, int64_t cols, int64_t diag_off, cudaStream_t st,
             int64_t* launches);
int copy2d(const double* S, int64_t lds, double* D, int64_t ldd, int64_t rows, int64_t cols, int upper_only,
           cudaStream_t st, int64_t* launches);
int perm_to_dense(const int64_t* perm, int64_t n, double* P, int64_t ldp, cudaStream_t st, int64_t* launches);
int transpose(const double* S, int64_t lds, double* D, int64_t ldd, int64_t rows, int64_t cols, cudaStream_t st,
              int64_t* launches);
int jacobi_svd(const double* r, int64_t ldr, int w, double* wbuf, int64_t ldw, double* vbuf, int64_t ldv, double* d,
               double* u, int64_t ldu, double* vt, int64_t ldvt, int* status, cudaStream_t st, int64_t* launches);
int set_diag_block(double* A, int64_t lda, int64_t rows, int w, const double* d, cudaStream_t st, int64_t* launches);
int widen(const int* a, int n, int64_t off, int64_t* out, cudaStream_t st, int64_t* launches);

int gaussian_fill(double* out, int64_t rows, int64_t cols, int64_t ld, uint64_t seed, uint64_t counter,
                  cudaStream_t st, int64_t* launches);
int splitmix_words(uint64_t* out, uint64_t seed, uint64_t first, int64_t count, cudaStream_t st,
                   int64_t* launches);

}  // namespace rq
