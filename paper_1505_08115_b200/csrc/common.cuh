// Shared device/host helpers for librandqr_b200 (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>

#include "../../include/randqr_b200.h"

#define RQ_DEV __device__ __forceinline__

// Column-major element access.
#define CM(p, ld, i, j) ((p)[(int64_t)(j) * (int64_t)(ld) + (int64_t)(i)])

namespace rq {

constexpr int kSMs = 148;  // B200: 2 dies x 74 SMs (queried at runtime; this is the default)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// ---------------------------------------------------------------------------
// Grid-wide barrier for cooperative launches: one atomic per CTA, monotonically
// increasing target (no reset needed inside a launch).  `bar` must be zero at
// launch; the launcher clears it with cudaMemsetAsync.
// ---------------------------------------------------------------------------
RQ_DEV void grid_barrier(unsigned int* bar, unsigned int& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    gen += 1;
    const unsigned int target = gen * gridDim.x;
    __threadfence();
    atomicAdd(bar, 1u);
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// Loads that bypass L1 (data written by other CTAs within the same launch).
RQ_DEV double ld_cg(const double* p) { return __ldcg(p); }

// Deterministic warp reduction (fixed butterfly order).
RQ_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Pivot key: larger norm wins; on equal norms the lower position wins
// (strict '>' scan of the reference, _kernels_numba.py:20-26).
struct PivKey {
  double val;
  int pos;
  int col;
};
RQ_DEV bool piv_better(double v1, int p1, double v2, int p2) {
  return (v1 > v2) || (v1 == v2 && p1 < p2);
}

}  // namespace rq

// Error plumbing (host side) -------------------------------------------------
#define RQ_CUDA_TRY(expr)                                                     \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess) {                                                  \
      rq::set_error(RQ_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr,      \
                    cudaGetErrorString(_e));                                  \
      return RQ_ECUDA;                                                        \
    }                                                                         \
  } while (0)

#define RQ_TRY(expr)             \
  do {                           \
    int _rc = (expr);            \
    if (_rc != RQ_OK) return _rc; \
  } while (0)

namespace rq {
int set_error(int code, const char* fmt, ...);
}
