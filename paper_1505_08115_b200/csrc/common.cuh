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
// ---- cluster exchange without a GPU-scope fence --------------------------------
// barrier.cluster.arrive.release compiles to MEMBAR.ALL.GPU (~900 cycles measured in the
// leaf kernel); pushes made with st.async complete transaction bytes on the receiver's
// mbarrier instead, so the receiver waits for exactly the data it needs.
RQ_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
RQ_DEV uint32_t cluster_map(uint32_t local, unsigned rank) {
  uint32_t r;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
RQ_DEV void mbar_init(unsigned long long* mbar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
}
RQ_DEV void mbar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
RQ_DEV void mbar_expect_tx(unsigned long long* mbar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes) : "memory");
}
RQ_DEV void mbar_wait_cluster(unsigned long long* mbar, unsigned parity) {
  const uint32_t a = smem_u32(mbar);
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
// 8-byte push into a peer's shared memory; completes 8 transaction bytes on its mbarrier
RQ_DEV void st_async_f64(uint32_t remote_addr, double v, uint32_t remote_mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(remote_addr),
               "l"(__double_as_longlong(v)), "r"(remote_mbar)
               : "memory");
}

RQ_DEV void st_async_u64(uint32_t remote_addr, unsigned long long v, uint32_t remote_mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(remote_addr), "l"(v),
               "r"(remote_mbar)
               : "memory");
}

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
