// Small bandwidth/latency kernels around the panel loop:
//   * T factor from the Gram matrix (K7),
//   * pivot bookkeeping and the column moves (K5),
//   * matrix fills / copies used by the driver and by Q formation (K12).
#include <algorithm>

#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "misc.cuh"

namespace rq {

// ---------------------------------------------------------------------------
// T = (I/2 + striu(V^T V))^{-1}: the compact-WY factor of U = H_0...H_{k-1}
// with H_j = I - 2 u_j u_j^T (same T as the wy_accumulate recurrence,
// householder.py:91-102).  One warp per column j, right-looking:
//   for kk = j..0:  t_kk = (kk == j) ? 2 : -2 acc_kk;  acc_i += G(i, kk) t_kk (i < kk)
// so each step is an axpy with the contiguous column G(:, kk); the loads do not
// depend on the recurrence and are issued one step ahead.  acc lives in
// registers (lane l owns rows l, l+32, ...).
// ---------------------------------------------------------------------------
// Columns of G are prefetched TR_DEPTH steps ahead through a register ring: a
// step is ~100 cycles of dependent work, an L2 load ~600.
template <int RPL>
struct TrDepth {
  static constexpr int value = RPL >= 16 ? 3 : 8;  // register budget
};

template <int RPL>
__global__ void __launch_bounds__(128) tinv_kernel(const double* __restrict__ G, int64_t ldg, int k,
                                                   double* __restrict__ T, int64_t ldt) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int TR_DEPTH = TrDepth<RPL>::value;
  const int j = blockIdx.x * (blockDim.x >> 5) + warp;
  if (j >= k) return;
  double acc[RPL], t[RPL];
#pragma unroll
  for (int r = 0; r < RPL; r++) {
    acc[r] = 0.0;
    t[r] = 0.0;
  }
  // ring[d] holds G(i, kk) (i < kk) for the column kk = kb - d of the current group
  double ring[TR_DEPTH][RPL];
#pragma unroll
  for (int d = 0; d < TR_DEPTH; d++)
#pragma unroll
    for (int r = 0; r < RPL; r++) {
      const int i = lane + 32 * r, kk = j - d;
      ring[d][r] = (kk >= 0 && i < kk) ? __ldg(G + (int64_t)kk * ldg + i) : 0.0;
    }
  for (int kb = j; kb >= 0; kb -= TR_DEPTH) {
#pragma unroll
    for (int d = 0; d < TR_DEPTH; d++) {
      const int kk = kb - d;
      if (kk < 0) break;
      // t_kk from acc_kk (held by lane kk % 32, slot kk / 32)
      double sel = 0.0;
      const int rk = kk >> 5;
#pragma unroll
      for (int r = 0; r < RPL; r++) sel = (r == rk) ? acc[r] : sel;
      const double a = __shfl_sync(0xffffffffu, sel, kk & 31);
      const double tk = (kk == j) ? 2.0 : -2.0 * a;
      const int kn = kk - TR_DEPTH;
#pragma unroll
      for (int r = 0; r < RPL; r++) {
        const int i = lane + 32 * r;
        if (i == kk) t[r] = tk;
        acc[r] = fma(ring[d][r], tk, acc[r]);  // zero for i >= kk
        ring[d][r] = (kn >= 0 && i < kn) ? __ldg(G + (int64_t)kn * ldg + i) : 0.0;
      }
    }
  }
#pragma unroll
  for (int r = 0; r < RPL; r++) {
    const int i = lane + 32 * r;
    if (i < k) T[(int64_t)j * ldt + i] = (i <= j) ? t[r] : 0.0;
  }
}

// Inverse of an upper-triangular k x k matrix R (column-major), one warp per
// column, right-looking back substitution (same structure as tinv_kernel).
// Exactly-zero pivots (exactly rank-deficient input) give zero rows/columns,
// i.e. a generalised inverse, so the downdated sketch stays finite.
template <int RPL>
__global__ void __launch_bounds__(128) trinv_upper_kernel(const double* __restrict__ R, int64_t ldr, int k,
                                                          double* __restrict__ X, int64_t ldx) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int TR_DEPTH = TrDepth<RPL>::value;
  // reciprocals of the diagonal once per block: the substitution's serial step is then a
  // multiply instead of an fp64 division (0 for an exactly-zero pivot)
  __shared__ double rdiag[32 * RPL];
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const double d = __ldg(R + (int64_t)i * ldr + i);
    rdiag[i] = d != 0.0 ? 1.0 / d : 0.0;
  }
  __syncthreads();
  const int j = blockIdx.x * (blockDim.x >> 5) + warp;
  if (j >= k) return;
  double acc[RPL], xv[RPL];
#pragma unroll
  for (int r = 0; r < RPL; r++) {
    acc[r] = 0.0;
    xv[r] = 0.0;
  }
  // x_kk = (delta_kj - acc_kk) / R_kk ;  acc_i += R(i, kk) x_kk  (i < kk)
  double ring[TR_DEPTH][RPL];  // R(i, kk), i <= kk
#pragma unroll
  for (int d = 0; d < TR_DEPTH; d++)
#pragma unroll
    for (int r = 0; r < RPL; r++) {
      const int i = lane + 32 * r, kk = j - d;
      ring[d][r] = (kk >= 0 && i <= kk) ? __ldg(R + (int64_t)kk * ldr + i) : 0.0;
    }
  for (int kb = j; kb >= 0; kb -= TR_DEPTH) {
#pragma unroll
    for (int d = 0; d < TR_DEPTH; d++) {
      const int kk = kb - d;
      if (kk < 0) break;
      double sa = 0.0;
      const int rk = kk >> 5;
#pragma unroll
      for (int r = 0; r < RPL; r++) sa = (r == rk) ? acc[r] : sa;
      const double a = __shfl_sync(0xffffffffu, sa, kk & 31);
      const double rhs = ((kk == j) ? 1.0 : 0.0) - a;
      const double xk = rhs * rdiag[kk];
      const int kn = kk - TR_DEPTH;
#pragma unroll
      for (int r = 0; r < RPL; r++) {
        const int i = lane + 32 * r;
        if (i == kk) xv[r] = xk;
        if (i < kk) acc[r] = fma(ring[d][r], xk, acc[r]);
        ring[d][r] = (kn >= 0 && i <= kn) ? __ldg(R + (int64_t)kn * ldr + i) : 0.0;
      }
    }
  }
#pragma unroll
  for (int r = 0; r < RPL; r++) {
    const int i = lane + 32 * r;
    if (i < k) X[(int64_t)j * ldx + i] = (i <= j) ? xv[r] : 0.0;
  }
}

int trinv_upper(const double* R, int64_t ldr, int k, double* X, int64_t ldx, cudaStream_t st, int64_t* launches) {
  if (k <= 0) return RQ_OK;
  const int wpb = 4;
  const unsigned blocks = (unsigned)ceil_div(k, wpb);
  if (k <= 64) trinv_upper_kernel<2><<<blocks, wpb * 32, 0, st>>>(R, ldr, k, X, ldx);
  else if (k <= 128) trinv_upper_kernel<4><<<blocks, wpb * 32, 0, st>>>(R, ldr, k, X, ldx);
  else if (k <= 256) trinv_upper_kernel<8><<<blocks, wpb * 32, 0, st>>>(R, ldr, k, X, ldx);
  else if (k <= 512) trinv_upper_kernel<16><<<blocks, wpb * 32, 0, st>>>(R, ldr, k, X, ldx);
  else return set_error(RQ_EUNSUPPORTED, "triangular inverse for more than 512 columns");
  RQ_CUDA_TRY(cudaGetLastError());
  if (launches) (*launches)++;
  return RQ_OK;
}

// ---------------------------------------------------------------------------
// Q = H_0 H_1 ... H_{k-1} (n x n, n <= 32 RPL), H_j = I - 2 v_j v_j^T with unit reflectors
// v_j = V(:, j) (zero above row j; a zero column is the identity, as the reference skips
// it, _kernels_numba.py:35-41).  One warp per column of Q, applied to e_c from the last
// reflector to the first, 16 columns per CTA, reflectors staged through shared memory in
// chunks of 16.  Replaces Q2 = I - V2 T2 V2^T (Gram GEMM, triangular inverse, three
// GEMMs) for the b x b CPQR: columns are independent, so no grid-wide synchronisation.
// ---------------------------------------------------------------------------
constexpr int QR_WARPS = 16;

template <int RPL>
__global__ void __launch_bounds__(QR_WARPS * 32) q_from_reflectors_kernel(const double* __restrict__ V, int64_t ldv,
                                                                          int k, int n, double* __restrict__ Q,
                                                                          int64_t ldq) {
  constexpr int QC = 16;  // reflectors per shared-memory chunk (32 KB at RPL = 8)
  __shared__ double vs[QC][32 * RPL];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * QR_WARPS + warp;
  double x[RPL];
#pragma unroll
  for (int r = 0; r < RPL; r++) x[r] = (lane + 32 * r == c) ? 1.0 : 0.0;
  const int nchunks = (k + QC - 1) / QC;
  for (int ch = nchunks - 1; ch >= 0; ch--) {
    const int j0 = ch * QC;
    const int kc = min(QC, k - j0);
    __syncthreads();
    for (int e = threadIdx.x; e < QC * 32 * RPL; e += QR_WARPS * 32) {
      const int jj = e / (32 * RPL), i = e - jj * (32 * RPL);
      vs[jj][i] = (jj < kc && i < n) ? V[(int64_t)(j0 + jj) * ldv + i] : 0.0;
    }
    __syncthreads();
    if (c < n) {
      for (int jj = kc - 1; jj >= 0; jj--) {
        double u[RPL];
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int r = 0; r < RPL; r++) {
          u[r] = vs[jj][lane + 32 * r];
          if (r & 1) d1 = fma(u[r], x[r], d1);
          else d0 = fma(u[r], x[r], d0);
        }
        double d = d0 + d1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        d *= 2.0;
#pragma unroll
        for (int r = 0; r < RPL; r++) x[r] = fma(-d, u[r], x[r]);
      }
    }
  }
  if (c < n)
#pragma unroll
    for (int r = 0; r < RPL; r++)
      if (lane + 32 * r < n) Q[(int64_t)c * ldq + lane + 32 * r] = x[r];
}

int q_from_reflectors(const double* V, int64_t ldv, int k, int n, double* Q, int64_t ldq, cudaStream_t st,
                      int64_t* launches) {
  if (n <= 0) return RQ_OK;
  const unsigned blocks = (unsigned)ceil_div(n, QR_WARPS);
  if (n <= 64) q_from_reflectors_kernel<2><<<blocks, QR_WARPS * 32, 0, st>>>(V, ldv, k, n, Q, ldq);
  else if (n <= 128) q_from_reflectors_kernel<4><<<blocks, QR_WARPS * 32, 0, st>>>(V, ldv, k, n, Q, ldq);
  else if (n <= 256) q_from_reflectors_kernel<8><<<blocks, QR_WARPS * 32, 0, st>>>(V, ldv, k, n, Q, ldq);
  else return set_error(RQ_EUNSUPPORTED, "q_from_reflectors: %d rows > 256", n);
  RQ_CUDA_TRY(cudaGetLastError());
  if (launches) (*launches)++;
  return RQ_OK;
}

int tfactor_from_gram(const double* G, int64_t ldg, int k, double* T, int64_t ldt, cudaStream_t st,
                      int64_t* launches) {
  if (k <= 0) return RQ_OK;
  const int wpb = 4;
  const unsigned blocks = (unsigned)ceil_div(k, wpb);
  if (k <= 64) tinv_kernel<2><<<blocks, wpb * 32, 0, st>>>(G, ldg, k, T, ldt);
  else if (k <= 128) tinv_kernel<4><<<blocks, wpb * 32, 0, st>>>(G, ldg, k, T, ldt);
  else if (k <= 256) tinv_kernel<8><<<blocks, wpb * 32, 0, st>>>(G, ldg, k, T, ldt);
  else if (k <= 512) tinv_kernel<16><<<blocks, wpb * 32, 0, st>>>(G, ldg, k, T, ldt);
  else return set_error(RQ_EUNSUPPORTED, "T factor for more than 512 reflectors");
  RQ_CUDA_TRY(cudaGetLastError());
  if (launches) (*launches)++;
  return RQ_OK;
}

// ---------------------------------------------------------------------------
// Pivot bookkeeping for one panel (single CTA).
//
// Local column indices are relative to the trailing block start s.  Inputs:
//   chosen[b]  local physical columns picked by the sketch CPQR, pivot order
//   lorder[n'] local physical column of each logical rank (reference order)
// Outputs:
//   moves (src, dst) realising "chosen[k] -> slot k" with the displaced panel
//   columns moved into the vacated slots (no full-height gather of the rest,
//   unlike PermutationPivot.apply_right, pivoting.py:60-61);
//   lorder_next / rank_next of the remaining n'-b columns (rebased by b):
//   the reference's order "chosen ++ rest in original order" (pivoting.py:125-128).
// ---------------------------------------------------------------------------
constexpr int PLAN_THREADS = 1024;

__global__ void __launch_bounds__(PLAN_THREADS) plan_moves_kernel(const int* __restrict__ chosen, int b,
                                                                  const int* __restrict__ lorder, int np,
                                                                  unsigned char* __restrict__ flag,
                                                                  int* __restrict__ newloc, int* __restrict__ src,
                                                                  int* __restrict__ dst, int* __restrict__ nmoves,
                                                                  int* __restrict__ lorder_next,
                                                                  int* __restrict__ rank_next) {
  using Scan = cub::BlockScan<int, PLAN_THREADS>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int base;
  __shared__ int nm;
  for (int i = threadIdx.x; i < np; i += PLAN_THREADS) {
    flag[i] = 0;
    newloc[i] = i;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < b; k += PLAN_THREADS) flag[chosen[k]] = 1;
  if (threadIdx.x == 0) {
    base = 0;
    nm = 0;
  }
  __syncthreads();
  // chosen[k] -> k for k with chosen[k] != k
  for (int k0 = 0; k0 < b; k0 += PLAN_THREADS) {
    const int k = k0 + threadIdx.x;
    const int mv = (k < b && chosen[k] != k) ? 1 : 0;
    int off, tot;
    Scan(tmp).ExclusiveSum(mv, off, tot);
    if (mv) {
      src[base + off] = chosen[k];
      dst[base + off] = k;
    }
    __syncthreads();
    if (threadIdx.x == 0) base += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) nm = base;
  __syncthreads();
  // displaced panel slots (not chosen), in slot order, pair with vacancies
  // (chosen columns outside the panel), in pivot order.
  int dbase = 0, vbase = 0;
  for (int k0 = 0; k0 < b; k0 += PLAN_THREADS) {
    const int k = k0 + threadIdx.x;
    const int isd = (k < b && !flag[k]) ? 1 : 0;
    int doff, dtot;
    Scan(tmp).ExclusiveSum(isd, doff, dtot);
    __syncthreads();
    if (isd) src[nm + dbase + doff] = k;  // displaced column (local k)
    dbase += dtot;
    __syncthreads();
  }
  for (int k0 = 0; k0 < b; k0 += PLAN_THREADS) {
    const int k = k0 + threadIdx.x;
    const int isv = (k < b && chosen[k] >= b) ? 1 : 0;
    int voff, vtot;
    Scan(tmp).ExclusiveSum(isv, voff, vtot);
    __syncthreads();
    if (isv) dst[nm + vbase + voff] = chosen[k];
    vbase += vtot;
    __syncthreads();
  }
  __syncthreads();
  for (int t = threadIdx.x; t < dbase; t += PLAN_THREADS) newloc[src[nm + t]] = dst[nm + t];
  if (threadIdx.x == 0) *nmoves = nm + dbase;
  __syncthreads();
  // stable compaction of the logical order, dropping the chosen columns
  int cbase = 0;
  for (int r0 = 0; r0 < np; r0 += PLAN_THREADS) {
    const int r = r0 + threadIdx.x;
    int c = -1, keep = 0;
    if (r < np) {
      c = lorder[r];
      keep = flag[c] ? 0 : 1;
    }
    int off, tot;
    Scan(tmp).ExclusiveSum(keep, off, tot);
    if (keep) {
      const int nl = newloc[c] - b;
      lorder_next[cbase + off] = nl;
      rank_next[nl] = cbase + off;
    }
    cbase += tot;
    __syncthreads();
  }
}

int plan_moves(const PlanCall& c, cudaStream_t st, int64_t* launches) {
  plan_moves_kernel<<<1, PLAN_THREADS, 0, st>>>(c.chosen, c.b, c.lorder, c.np, c.flag, c.newloc, c.src, c.dst,
                                                c.nmoves, c.lorder_next, c.rank_next);
  RQ_CUDA_TRY(cudaGetLastError());
  if (launches) (*launches)++;
  return RQ_OK;
}

// ---------------------------------------------------------------------------
// Column moves through a staging buffer: dst[t] <- src[t] for rows [r0, r1),
// plus the same move on the int64 `orig` label array.  Two launches (gather,
// scatter) because src and dst overlap as sets.  One warp per column,
// vectorised 16 B accesses when the column start is aligned.
// ---------------------------------------------------------------------------
// Full-height column moves, two passes (all sources staged before any target is
// written, so a slot can be both).  Grid (row chunks, columns): every chunk is
// 2048 rows, 8 independent loads in flight per thread -> HBM-bound.
constexpr int MV_THREADS = 256;
constexpr int MV_PER = 8;
constexpr int MV_CHUNK = MV_THREADS * MV_PER;

__global__ void __launch_bounds__(MV_THREADS) gather_cols_kernel(const double* __restrict__ A, int64_t lda,
                                                                 int64_t coff, int64_t r0, int64_t r1,
                                                                 const int* __restrict__ src,
                                                                 const int* __restrict__ count, int maxn,
                                                                 double* __restrict__ stage, int64_t lds,
                                                                 const int64_t* __restrict__ orig,
                                                                 int64_t* __restrict__ ostage,
                                                                 unsigned long long* bytes) {
  const int n = count ? *count : maxn;
  const int t = blockIdx.y;
  if (t >= n) return;
  if (bytes && blockIdx.x == 0 && threadIdx.x == 0)  // gather + scatter: 2 reads + 2 writes per element
    atomicAdd(bytes, (unsigned long long)(r1 > r0 ? r1 - r0 : 0) * 32ull);
  const double* s = A + (coff + src[t]) * lda;
  double* d = stage + (int64_t)t * lds;
  const int64_t i0 = r0 + (int64_t)blockIdx.x * MV_CHUNK + threadIdx.x;
  double v[MV_PER];
#pragma unroll
  for (int k = 0; k < MV_PER; k++) {
    const int64_t i = i0 + (int64_t)k * MV_THREADS;
    v[k] = i < r1 ? __ldcs(&s[i]) : 0.0;
  }
#pragma unroll
  for (int k = 0; k < MV_PER; k++) {
    const int64_t i = i0 + (int64_t)k * MV_THREADS;
    if (i < r1) d[i - r0] = v[k];
  }
  if (orig && blockIdx.x == 0 && threadIdx.x == 0) ostage[t] = orig[coff + src[t]];
}
__global__ void __launch_bounds__(MV_THREADS) scatter_cols_kernel(double* __restrict__ A, int64_t lda, int64_t coff,
                                                                  int64_t r0, int64_t r1,
                                                                  const int* __restrict__ dst,
                                                                  const int* __restrict__ count, int maxn,
                                                                  const double* __restrict__ stage, int64_t lds,
                                                                  int64_t* __restrict__ orig,
                                                                  const int64_t* __restrict__ ostage) {
  const int n = count ? *count : maxn;
  const int t = blockIdx.y;
  if (t >= n) return;
  double* d = A + (coff + dst[t]) * lda;
  const double* s = stage + (int64_t)t * lds;
  const int64_t i0 = r0 + (int64_t)blockIdx.x * MV_CHUNK + threadIdx.x;
  double v[MV_PER];
#pragma unroll
  for (int k = 0; k < MV_PER; k++) {
    const int64_t i = i0 + (int64_t)k * MV_THREADS;
    v[k] = i < r1 ? s[i - r0] : 0.0;
  }
#pragma unroll
  for (int k = 0; k < MV_PER; k++) {
    const int64_t i = i0 + (int64_t)k * MV_THREADS;
    if (i < r1) d[i] = v[k];
  }
  if (orig && blockIdx.x == 0 && threadIdx.x == 0) orig[coff + dst[t]] = ostage[t];
}

int move_columns(const MoveCall& c, cudaStream_t st, int64_t* launches) {
  if (c.r1 <= c.r0 && !c.orig) return RQ_OK;
  if (c.maxn <= 0) return RQ_OK;
  const int64_t rows = c.r1 > c.r0 ? c.r1 - c.r0 : 0;
  const dim3 grid((unsigned)std::max<int64_t>(1, ceil_div(rows, MV_CHUNK)), (unsigned)c.maxn);
  gather_cols_kernel<<<grid, MV_THREADS, 0, st>>>(c.A, c.lda, c.coff, c.r0, c.r1, c.src, c.count, c.maxn, c.stage,
                                                  c.lds, c.orig, c.ostage, c.bytes);
  RQ_CUDA_TRY(cudaGetLastError());
  scatter_cols_kernel<<<grid, MV_THREADS, 0, st>>>(c.A, c.lda, c.coff, c.r0, c.r1, c.dst, c.count, c.maxn, c.stage,
                                                   c.lds, c.orig, c.ostage);
  RQ_CUDA_TRY(cudaGetLastError());
  if (launches) (*launches) += 2;
  return RQ_OK;
}

// e2[k] = sum_{i >= k} sum_{j >= i} R(i, j)^2 for upper-triangular R: row sums of squares
// (thread per row: for a fixed column the warp's loads are contiguous), then a suffix
// scan in fixed order (one thread; n <= a few 1e4).
__global__ void row_sq_kernel(const double* __restrict__ R, int64_t n, int64_t ldr, double* __restrict__ rs) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int64_t j = i; j < n; j++) {
      const double v = R[j * ldr + i];
      acc = fma(v, v, acc);
    }
    rs[i] = acc;
  }
}
__global__ void suffix_sum_kernel(double* e, int64_t n) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double acc = 0.0;
    e[n] = 0.0;
    for (int64_t k = n - 1; k >= 0; k--) {
      acc += e[k];
      e[k] = acc;
    }
  }
}
int trailing_frobenius(const double* R, int64_t n, int64_t ldr, double* e2, cudaStream_t st, int64_t* launches) {
  if (n > 0) {
    const int blocks = (int)std::min<int64_t>(4 * kSMs, ceil_div(n, 256));
    row_sq_kernel<<<blocks, 256, 0, st>>>(R, n, ldr, e2);
    RQ_CUDA_TRY(cudaGetLastError());
  }
  suffix_sum_kernel<<<1, 32, 0, st>>>(e2, n);
  RQ_CUDA_TRY(cudaGetLastError());
  if (launches) (*launches) += 2;
  return RQ_OK;
}

// identity index arrays
__global__ void iota_kernel(int* a, int n, int64_t* b, int64_t nb) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)n || i < nb;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (a && i < n) a[i] = (int)i;
    if (b && i < nb) b[i] = i;
  }
}
int iota(int* a, int n, int64_t* b, int64_t nb, cudaStream_t st, int64_t* launches) {
  const int64_t mx = n > nb ? n : nb;
  if (mx <= 0) return RQ_OK;
  int blocks = (int)ceil_div(mx, 256);
  if (blocks > 4 * kSMs) blocks = 4 * kSMs;
  iota_kernel<<<blocks, 256, 0, st>>>(a, n, b, nb);
  RQ_CUDA_TRY(cudaGetLastError());
  if (launches) (*launches)++;
  return RQ_OK;
}

// X (rows x cols) = [upper part of S (rows x cols_s) | I] helpers
__global__ void fill_eye_kernel(double* X, int64_t ldx, int64_t rows, int64_t cols, int64_t diag_off) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = idx / rows, i = idx - j * rows;
    X[j * ldx + i] = (i == j + diag_off) ? 1.0 : 0.0;
  }
}
int fill_eye(double* X, int64_t ldx, int64_t rows, int64_t cols, int64_t diag_off, cudaStream_t st,
             int64_t* launches) {
  if (rows <= 0 || cols <= 0) return RQ_OK;
  int blocks = (int)ceil_div(rows * cols, 256);
  if (blocks > 8 * kSMs) blocks = 8 * kSMs;
  fill_eye_kernel<<<blocks, 256, 0, st>>>(X, ldx, rows, cols, diag_off);
  RQ_CUDA_TRY(cudaGetLastError());
  if (launches) (*launches)++;
  return RQ_OK;
}

// 2-D copy (column-major), optionally zeroing strictly-below-diagonal entries
__global__ void copy2d_kernel(const double* __restrict__ S, int64_t lds, double* __restrict__ D, int64_t ldd,
                              int64_t rows, int64_t cols, int upper_only) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = idx / rows, i = idx - j * rows;
    D[j * ldd + i] = (upper_only && i > j) ? 0.0 : S[j * lds + i];
  }
}
int copy2d(const double* S, int64_t lds, double* D, int64_t ldd, int64_t rows, int64_t cols, int upper_only,
           cudaStream_t st, int64_t* launches) {
  if (rows <= 0 || cols <= 0) return RQ_OK;
  int blocks = (int)ceil_div(rows * cols, 256);
  if (blocks > 8 * kSMs) blocks = 8 * kSMs;
  copy2d_kernel<<<blocks, 256, 0, st>>>(S, lds, D, ldd, rows, cols, upper_only);
  RQ_CUDA_TRY(cudaGetLastError());
  if (launches) (*launches)++;
  return RQ_OK;
}

// dense P from a permutation: P[perm[k], k] = 1
__global__ void perm_to_dense_kernel(const int64_t* perm, int64_t n, double* P, int64_t ldp) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    P[k * ldp + perm[k]] = 1.0;
}
int perm_to_dense(const int64_t* perm, int64_t n, double* P, int64_t ldp, cudaStream_t st, int64_t* launches) {
  RQ_TRY(fill_eye(P, ldp, n, n, INT64_MAX / 4, st, launches));  // zeros
  perm_to_dense_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(perm, n, P, ldp);
  RQ_CUDA_TRY(cudaGetLastError());
  if (launches) (*launches)++;
  return RQ_OK;
}

// Out-of-place transpose (column-major rows x cols -> cols x rows), 32x32 smem tiles.
__global__ void transpose_kernel(const double* __restrict__ S, int64_t lds, double* __restrict__ D, int64_t ldd,
                                 int64_t rows, int64_t cols) {
  __shared__ double tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + threadIdx.x, c = c0 + k;
    tile[k][threadIdx.x] = (r < rows && c < cols) ? S[c * lds + r] : 0.0;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t c = c0 + threadIdx.x, r = r0 + k;  // D(c, r) = S(r, c)
    if (r < rows && c < cols) D[r * ldd + c] = tile[threadIdx.x][k];
  }
}
int transpose(const double* S, int64_t lds, double* D, int64_t ldd, int64_t rows, int64_t cols, cudaStream_t st,
              int64_t* launches) {
  if (rows <= 0 || cols <= 0) return RQ_OK;
  dim3 grid((unsigned)ceil_div(rows, 32), (unsigned)ceil_div(cols, 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(S, lds, D, ldd, rows, cols);
  RQ_CUDA_TRY(cudaGetLastError());
  if (launches) (*launches)++;
  return RQ_OK;
}

// A (rows x w) = [diag(d); 0]  (block_rrqr's diagonal block, blocked.py:266-268)
__global__ void set_diag_block_kernel(double* A, int64_t lda, int64_t rows, int w, const double* d) {
  const int64_t total = rows * w;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = idx / rows, i = idx - j * rows;
    A[j * lda + i] = (i == j) ? d[j] : 0.0;
  }
}
int set_diag_block(double* A, int64_t lda, int64_t rows, int w, const double* d, cudaStream_t st, int64_t* launches) {
  if (rows <= 0 || w <= 0) return RQ_OK;
  int blocks = (int)ceil_div(rows * w, 256);
  if (blocks > 8 * kSMs) blocks = 8 * kSMs;
  set_diag_block_kernel<<<blocks, 256, 0, st>>>(A, lda, rows, w, d);
  RQ_CUDA_TRY(cudaGetLastError());
  if (launches) (*launches)++;
  return RQ_OK;
}

// int32 -> int64 widening with offset (perm outputs)
__global__ void widen_kernel(const int* a, int n, int64_t off, int64_t* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = a[i] + off;
}
int widen(const int* a, int n, int64_t off, int64_t* out, cudaStream_t st, int64_t* launches) {
  if (n <= 0) return RQ_OK;
  widen_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(a, n, off, out);
  RQ_CUDA_TRY(cudaGetLastError());
  if (launches) (*launches)++;
  return RQ_OK;
}

// Power-iteration step helper (trailing spectral norms): x <- x / ||x||, norms[it] = ||x||.
// One CTA, fixed reduction order (deterministic).
__global__ void __launch_bounds__(1024) normalize_col_kernel(double* __restrict__ x, int64_t n,
                                                             double* __restrict__ norms, int it) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc = fma(x[i], x[i], acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const double nrm = sqrt(red[0]);
  const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) x[i] *= inv;
  if (threadIdx.x == 0) norms[it] = nrm;
}

int normalize_col(double* x, int64_t n, double* norms, int it, cudaStream_t st, int64_t* launches) {
  normalize_col_kernel<<<1, 1024, 0, st>>>(x, n, norms, it);
  RQ_CUDA_TRY(cudaGetLastError());
  if (launches) (*launches)++;
  return RQ_OK;
}

}  // namespace rq
