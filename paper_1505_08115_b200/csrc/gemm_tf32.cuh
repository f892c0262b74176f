// FP32 GEMM on tcgen05 tensor cores (3xTF32 split products, TMEM accumulator, TMA staging);
// see gemm_tf32.cu.  Same conventions as gemm_f64.cuh with fp32 operands:
//   C[M x N] = alpha * op(A) * B + beta * C,  op(A) = A^T (A stored K x M) or A (A stored M x K),
//   B stored K x N; views at element origins (r0, c0) of whole buffers (ld % 4 == 0, 16 B bases).
#pragma once
#include "common.cuh"
#include "gemm_f64.cuh"

namespace rq {

struct GemmOperandF32 {
  const float* base;
  int64_t rows, cols, ld;
  int64_t r0, c0;
};

struct GemmProblemF32 {
  int64_t M, N, K;
  GemmOperandF32 A;
  bool a_mmajor;
  GemmOperandF32 B;
  float* C;
  int64_t ldc;
  double alpha, beta;
  int max_ctas = 0;  // > 0: cap the persistent grid (leave SMs to a concurrent kernel)
  float* work = nullptr;  // split-K slabs (deterministic reduction); null: no split-K
  size_t work_bytes = 0;
};

int gemm_tf32x3(const GemmProblemF32& p, cudaStream_t st, int64_t* launches);
// The same 3xTF32 tensor-core product on fp64 operands and C (fp32-level accuracy: the inputs are
// rounded to fp32 once, partial sums accumulate in fp32): the trailing update of the fp32-accuracy
// mode of the monolithic driver (RQ_FLAG_TF32_UPDATE).  Honours max_ctas, pdl, tile ranges and
// split-K slabs (work, as fp32) like gemm_f64.
int gemm_tf32x3_f64(const GemmProblem& p, cudaStream_t st, int64_t* launches);
int64_t gemm_tf32x3_tiles(int64_t M, int64_t N, bool a_mmajor, int64_t a_r0);

}  // namespace rq
