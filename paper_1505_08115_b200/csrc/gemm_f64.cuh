// FP64 tensor-core GEMM for sm_100a: TMA (cp.async.bulk.tensor) -> mbarrier
// pipeline -> mma.sync m16n8k4 f64 (SASS: DMMA.8x8x4).  FP64 has no tcgen05
// kind on Blackwell (ptxas rejects kind::f64), so DMMA is the FP64 tensor path;
// measured 36.9 TFLOP/s peak on B200 (profiles/probe_r01.jsonl).
//
//   C[M x N] = alpha * op(A) * B + beta * C        (all column-major)
//     op(A) = A^T, A stored K x M  (A_MMAJOR = false, "TN": K contiguous)
//     op(A) = A,   A stored M x K  (A_MMAJOR = true,  "NN": M contiguous)
//     B stored K x N (K contiguous)
//
// The operands are addressed through TMA tensor maps over whole buffers plus
// element-coordinate origins, so sub-matrix views need no pointer alignment.
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace rq {

struct GemmOperand {
  const double* base;  // buffer base (16 B aligned)
  int64_t rows;        // buffer extent along the contiguous dimension
  int64_t cols;        // buffer extent along the strided dimension
  int64_t ld;          // leading dimension (elements, even)
  int64_t r0, c0;      // origin of the view inside the buffer
};

struct GemmProblem {
  int64_t M, N, K;
  GemmOperand A;  // TN: rows index K, cols index M.   NN: rows index M, cols index K.
  bool a_mmajor;
  GemmOperand B;  // rows index K, cols index N
  double* C;      // view pointer (already offset), column-major
  int64_t ldc;
  double alpha, beta;
  int splitk;            // 0: choose automatically; >1: deterministic split-K through `work`
  double* work;          // splitk * (M+1) * N doubles (slab per split)
  size_t work_bytes;
  int max_ctas = 0;      // > 0: cap the persistent grid (leave SMs to a concurrent kernel)
  bool pdl = false;      // programmatic dependent launch: may start once the previous kernel in the
                         // stream triggered (the GEMM must not read that kernel's output)
  unsigned long long* sched = nullptr;       // device counter: dynamic unit scheduling (see gemm_f64.cu)
  unsigned long long* sched_base = nullptr;  // host mirror of its value; advanced by every launch
  int64_t tile_begin = 0, tile_end = 0;  // tile_end > 0: only output tiles [tile_begin, tile_end)
                                         // (column-major tile order; see gemm_f64_tiles)
  cudaEvent_t mid_event = nullptr;  // profiling: recorded between the GEMM and its split-K reduce
  int* splitk_used = nullptr;       // profiling: receives the split-K factor used (1 = none)
};

int gemm_f64(const GemmProblem& p, cudaStream_t stream, int64_t* launches);
int64_t gemm_f64_tiles(const GemmProblem& p);
// 2-D fp64 tensor map (rows contiguous, ld elements between columns), box box0 x box1,
// optionally 128B-swizzled (box0 = 16 then); for kernels outside the GEMM (wy_cluster).
int make_tensor_map_f64(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld, int box0,
                        int box1, bool swizzle);
size_t gemm_splitk_workspace(int64_t M, int64_t N, int splitk);

}  // namespace rq
