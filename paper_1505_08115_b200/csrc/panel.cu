// K6/K7: unpivoted Householder QR of a tall-skinny leaf (mm x WL, WL <= 32)
// plus its compact-WY T factor, as one thread-block-cluster kernel.
//
// Restates householder_sweep(pivot=False) (_kernels_numba.py:35-61) and the
// compact-WY recurrence of wy_accumulate (householder.py:91-102) in T form:
//   H_j = I - 2 u_j u_j^T,  U = H_0 ... H_{w-1} = I - V T V^T,
//   T_jj = 2,  T(0:j, j) = -2 T(0:j, 0:j) (V(:, 0:j)^T u_j).
//
// B200 mapping: a cluster of CS CTAs (16, non-portable) splits the rows; each
// CTA keeps its rows of the leaf in shared memory.  Per column ONE cluster
// barrier (~0.22 us measured) exchanges the partial sums (trailing norm,
// column dots, row-j entries, Gram entries for T) through DSMEM; every CTA
// then sums the CS partials in rank order (deterministic) and derives the
// same reflector.  The driver calls it once per WL-column leaf and applies
// the leaf's WY to the rest of the panel with the DMMA GEMM.
#include <cooperative_groups.h>

#include "common.cuh"
#include "gemm_f64.cuh"
#include "panel.cuh"

namespace cg = cooperative_groups;

namespace rq {

constexpr int PL_THREADS = 512;
constexpr int PL_WARPS = PL_THREADS / 32;

template <int WL>
struct LeafLayout {
  static constexpr int PV = 3 * WL + 1;  // [tail | dots(WL) | rowj(WL) | gram(WL)]
};

// DSMEM load without a memory clobber so consecutive loads can be in flight
// together (ordering w.r.t. the producers comes from the cluster barrier).
RQ_DEV double dsmem_ld(const double* local_addr, unsigned rank) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(local_addr);
  uint32_t r;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(r));
  return v;
}

RQ_DEV void dsmem_st(double* local_addr, unsigned rank, double v) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(local_addr);
  uint32_t r;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(r), "d"(v) : "memory");
}

RQ_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int WL>
__global__ void __launch_bounds__(PL_THREADS) leaf_qr_kernel(double* __restrict__ a, int64_t lda, int64_t mm,
                                                             int w, double* __restrict__ v, int64_t ldv,
                                                             double* __restrict__ tl, int64_t ldt,
                                                             int rows_per) {
  constexpr int PV = LeafLayout<WL>::PV;
  extern __shared__ double sm[];
  const unsigned CS = gridDim.x;  // one cluster spans the grid
  const unsigned rank = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)rank * rows_per;
  const int64_t r1 = min(mm, r0 + rows_per);
  const int nr = (int)max((int64_t)0, r1 - r0);

  double* A = sm;                                     // nr x WL (ld = rows_per)
  double* Vs = A + (int64_t)rows_per * WL;            // nr x WL own rows of V
  double* part = Vs + (int64_t)rows_per * WL;         // PV own partials
  double* pin = part + PV;                            // 2 x 16 x PV partials pushed by every CTA
  double* tot = pin + 2 * 16 * PV;                    // PV totals
  double* s = tot + PV;                               // WL coefficients
  double* Ts = s + WL;                                // WL x WL T (CTA-local copy)
  double* scal = Ts + WL * WL;                        // [refl, beta, inv, h]

  for (int c = warp; c < WL; c += PL_WARPS)
    for (int i = lane; i < nr; i += 32) {
      A[c * rows_per + i] = c < w ? a[(int64_t)c * lda + r0 + i] : 0.0;
      Vs[c * rows_per + i] = 0.0;
    }
  for (int e = threadIdx.x; e < WL * WL; e += PL_THREADS) Ts[e] = 0.0;
  __syncthreads();
  cluster_sync_all();  // all CTAs initialised before anyone pushes into them

  bool refl_prev = false;
  for (int j = 0; j <= w; j++) {
    const bool final_round = (j == w);  // only the last T column remains
    // ---------------- phase A: pending update + partials ----------------
    if (j > 0 && refl_prev && !final_round) {
      // A[i][c] -= s[c] * u_i for own rows i >= j-1, columns c in [j, w)
      const int lo = (int)max((int64_t)0, (int64_t)(j - 1) - r0);
      const double* uj = Vs + (j - 1) * rows_per;
      // 2-D work split: warp-strided columns, lanes over rows (no integer division)
      for (int c = j + warp; c < w; c += PL_WARPS) {
        const double sc = s[c];
        double* col = A + c * rows_per;
        for (int i = lo + lane; i < nr; i += 32) col[i] -= sc * uj[i];
      }
      __syncthreads();
    }
    double* mypart = part;
    const int par = j & 1;
    // items: 0 -> tail of column j; 1..w-j-1 -> dots with columns j+1..; gram k < j-1
    const int ndots = final_round ? 0 : (w - j);          // tail + dots
    const int ngram = (j >= 2) ? (j - 1) : 0;             // Gram entries for T column j-1
    const int nitems = ndots + ngram;
    for (int it = warp; it < nitems; it += PL_WARPS) {
      double acc = 0.0;
      if (it < ndots) {
        const int c = j + it;  // it == 0 -> tail (c == j)
        const int64_t lo = max((int64_t)0, (int64_t)(j + 1) - r0);
        const double* cj = A + (int64_t)j * rows_per;
        const double* cc = A + (int64_t)c * rows_per;
        for (int64_t i = lo + lane; i < nr; i += 32) acc += cj[i] * cc[i];
      } else {
        const int k = it - ndots;  // Gram entry V_k . u_{j-1}
        const double* vk = Vs + (int64_t)k * rows_per;
        const double* vj = Vs + (int64_t)(j - 1) * rows_per;
        for (int64_t i = lane; i < nr; i += 32) acc += vk[i] * vj[i];
      }
      acc = warp_sum(acc);
      if (lane == 0) {
        if (it < ndots) mypart[it == 0 ? 0 : 1 + (j + it)] = acc;
        else mypart[1 + 2 * WL + (it - ndots)] = acc;
      }
    }
    // row-j entries (exactly one CTA owns row j; others contribute zeros)
    if (!final_round)
      for (int c = j + threadIdx.x; c < w; c += PL_THREADS)
        mypart[1 + WL + c] = (j >= r0 && j < r1) ? A[(int64_t)c * rows_per + (j - r0)] : 0.0;
    __syncthreads();
    // push the partial vector into every CTA (fire-and-forget DSMEM stores)
    for (int dst = warp; dst < (int)CS; dst += PL_WARPS)
      for (int e = lane; e < PV; e += 32) dsmem_st(pin + (par * 16 + rank) * PV + e, (unsigned)dst, mypart[e]);
    cluster_sync_all();

    // ---------------- phase B: identical totals in every CTA ----------------
    for (int e = threadIdx.x; e < PV; e += PL_THREADS) {
      bool used;
      if (e == 0) used = !final_round;
      else if (e <= WL) used = !final_round && (e - 1) > j && (e - 1) < w;
      else if (e <= 2 * WL) used = !final_round && (e - 1 - WL) >= j && (e - 1 - WL) < w;
      else used = (e - 1 - 2 * WL) < ngram;
      if (!used) continue;
      double t = 0.0;
      for (unsigned r = 0; r < CS; r++) t += pin[(par * 16 + r) * PV + e];  // rank order: deterministic
      tot[e] = t;
    }
    __syncthreads();
    // T column j-1 (needs Gram entries of u_{j-1}); T_{jj} = 2 regardless
    if (j >= 1 && warp == 0) {
      const int jc = j - 1;
      // T(0:jc, jc) = -2 T(0:jc, 0:jc) g,   g_k = tot_gram[k]
      for (int i = lane; i < jc; i += 32) {
        double acc = 0.0;
        for (int k = i; k < jc; k++) acc += Ts[k * WL + i] * tot[1 + 2 * WL + k];
        Ts[jc * WL + i] = -2.0 * acc;
      }
      if (lane == 0) Ts[jc * WL + jc] = 2.0;
    }
    if (final_round) break;
    if (threadIdx.x == 0) {
      const double tail = tot[0];
      const double xjj = tot[1 + WL + j];
      const double normsq = xjj * xjj + tail;
      const bool refl = (mm - j >= 2) && (normsq != 0.0);
      double beta = 0.0, inv = 0.0, h = 0.0;
      if (refl) {
        const double nrm = sqrt(normsq);
        beta = (xjj >= 0.0) ? -nrm : nrm;
        h = beta - xjj;
        inv = 1.0 / sqrt(h * h + tail);
      }
      scal[0] = refl ? 1.0 : 0.0;
      scal[1] = beta;
      scal[2] = inv;
      scal[3] = h;
    }
    __syncthreads();
    const bool refl = scal[0] != 0.0;
    if (refl) {
      const double beta = scal[1], inv = scal[2], h = scal[3];
      for (int c = j + 1 + threadIdx.x; c < w; c += PL_THREADS)
        s[c] = 2.0 * inv * (h * tot[1 + WL + c] - tot[1 + c]);
      // own rows of u_j; column j becomes beta e_j
      for (int64_t i = threadIdx.x; i < nr; i += PL_THREADS) {
        const int64_t gi = r0 + i;
        double ui = 0.0;
        if (gi == j) {
          ui = h * inv;
          A[(int64_t)j * rows_per + i] = beta;
        } else if (gi > j) {
          ui = -A[(int64_t)j * rows_per + i] * inv;
          A[(int64_t)j * rows_per + i] = 0.0;
        }
        Vs[(int64_t)j * rows_per + i] = ui;
      }
    }
    refl_prev = refl;
    __syncthreads();
  }
  __syncthreads();  // warp 0 wrote the last T column in the final round
  // write back R (own rows) and V
  for (int c = warp; c < w; c += PL_WARPS)
    for (int i = lane; i < nr; i += 32) {
      a[(int64_t)c * lda + r0 + i] = A[c * rows_per + i];
      v[(int64_t)c * ldv + r0 + i] = Vs[c * rows_per + i];
    }
  if (rank == 0 && tl)
    for (int e = threadIdx.x; e < w * w; e += PL_THREADS) tl[(int64_t)(e / w) * ldt + e % w] = Ts[(e / w) * WL + e % w];
  cluster_sync_all();  // keep DSMEM alive until every CTA finished reading
}

// ---------------------------------------------------------------------------
// Register-resident leaf: thread t of CTA r owns leaf rows r*rows_per + t + 256*q
// (q < RPT) for all WL (<= 16) columns in registers.  Per column j the CTA
// reduces 32 partial sums [tail, dots(c = j+o), gram(k < j-1)] (two 16-value
// warp reduce-scatters + one smem pass), pushes them into every cluster peer,
// and after ONE cluster barrier warp 0 derives the reflector coefficients from
// the 16 pushed vectors (summed in rank order: deterministic) into smem.
// ---------------------------------------------------------------------------
__device__ unsigned long long g_leaf_dbg[64 * 8];
__device__ int g_leaf_dbg_on;
// Compiled in only with -DRQ_STAMPS (tuning builds): reading the flag from global memory on
// every call put an L2 round trip after each cluster acquire (which invalidates L1) on the
// per-column critical path.
RQ_DEV void leaf_stamp(int j, int k) {
#ifdef RQ_STAMPS
  if (blockIdx.x == 0 && threadIdx.x == 0 && j < 64) {  // (stamps build: always on)
    unsigned long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
    g_leaf_dbg[j * 8 + k] = c;
  }
#else
  (void)j;
  (void)k;
#endif
}
int leaf_debug_timing(int on, unsigned long long* host, int count) {
  RQ_CUDA_TRY(cudaMemcpyToSymbol(g_leaf_dbg_on, &on, sizeof(int)));
  if (host) RQ_CUDA_TRY(cudaMemcpyFromSymbol(host, g_leaf_dbg, sizeof(unsigned long long) * (count < 512 ? count : 512)));
  return RQ_OK;
}

constexpr int LR_THREADS = 256;
constexpr int LR_WARPS = LR_THREADS / 32;

// 16 values per lane -> lane l holds the warp sum of value (l & 15).
RQ_DEV double warp_reduce_scatter16(double (&v)[16], int lane) {
#pragma unroll
  for (int half = 8; half >= 1; half >>= 1) {
    const bool upper = (lane & half) != 0;
#pragma unroll
    for (int k = 0; k < half; k++) {
      const double send = upper ? v[k] : v[k + half];
      const double recv = __shfl_xor_sync(0xffffffffu, send, half);
      v[k] = (upper ? v[k + half] : v[k]) + recv;
    }
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
}

template <int WL, int RPT>
__global__ void __launch_bounds__(LR_THREADS, 1) leaf_reg_kernel(double* __restrict__ a, int64_t lda, int64_t mm, int w,
                                                                 double* __restrict__ v, int64_t ldv,
                                                                 double* __restrict__ tl, int64_t ldt, int rows_per) {
  static_assert(WL <= 16, "leaf width");
  extern __shared__ double Vs[];                  // [WL][RPT*LR_THREADS] own rows of V (lane-contiguous)
  constexpr int VLD = RPT * LR_THREADS;
  __shared__ double wpart[LR_WARPS][32];
  __shared__ double pin[2][16][32];               // pushed CTA partials, by step parity
  __shared__ double rowj[16];                     // row j of this CTA (if it owns it), window order
  __shared__ double rowp[2][16];                  // row j pushed by its owner, by step parity
  __shared__ double sc[17];                       // reflector coefficients of step j-1 (o = c - j + 1), sc[16] = 0
  __shared__ double scal[4];                      // refl, beta, h*inv, inv
  __shared__ double Ts[16][17];
  __shared__ __align__(8) unsigned long long lmbar[2];  // pushes of step j complete on lmbar[j & 1]
  // T is formed once per leaf, after the column loop: every CTA's partial Gram V_own^T V_own
  // (the 120 pairs k < l) is pushed to rank 0, which sums them in rank order and runs the T
  // recurrence -- none of it on the per-column critical path any more
  __shared__ double gin[16][120];
  __shared__ __align__(8) unsigned long long gbar;
  constexpr unsigned CS = 16;  // launch_leaf_reg: one 16-CTA cluster
  // look-ahead (driver.cu): a chunk of the previous panel's trailing update launched after this
  // kernel with programmatic stream serialization starts once the cluster is resident, on the
  // other 132 SMs (it touches neither this leaf's columns nor its outputs)
  asm volatile("griddepcontrol.launch_dependents;");
  const unsigned rank = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)rank * rows_per;

  // register window: x[q][o] holds column j + o of own row q (active column at o = 0)
  double x[RPT][WL];
  int64_t grow[RPT];
#pragma unroll
  for (int q = 0; q < RPT; q++) {
    const int lr = threadIdx.x + LR_THREADS * q;
    grow[q] = (lr < rows_per) ? r0 + lr : mm;  // rows beyond mm are inert
#pragma unroll
    for (int c = 0; c < WL; c++) {
      x[q][c] = (grow[q] < mm && c < w) ? a[(int64_t)c * lda + grow[q]] : 0.0;
      Vs[c * VLD + lr] = 0.0;
    }
  }
  for (int e = threadIdx.x; e < 16 * 17; e += LR_THREADS) (&Ts[0][0])[e] = 0.0;
  if (threadIdx.x < 17) sc[threadIdx.x] = 0.0;
  double uprev[RPT];
#pragma unroll
  for (int q = 0; q < RPT; q++) uprev[q] = 0.0;
  bool refl_prev = false;
  if (threadIdx.x == 0) {
    mbar_init(&lmbar[0], 1);
    mbar_init(&lmbar[1], 1);
    mbar_init(&gbar, 1);
    mbar_init_fence();
  }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");

  for (int j = 0; j < w; j++) {
    const int par = j & 1;
    leaf_stamp(j, 0);
    // this step's pushes: 16 partial sums from every CTA, plus row j from its owner
    if (threadIdx.x == 0) mbar_expect_tx(&lmbar[par], CS * 16 * 8 + 16 * 8);
    // ---- apply the pending reflector j-1 to the window (columns j..) ----
    if (refl_prev) {
      double s[WL];
#pragma unroll
      for (int o = 0; o < WL; o++) s[o] = sc[o + 1];  // window shifted by one since step j-1
#pragma unroll
      for (int q = 0; q < RPT; q++)
#pragma unroll
        for (int o = 0; o < WL; o++) x[q][o] -= s[o] * uprev[q];
    }
    // ---- partials: dv[o] = sum x_j x_{j+o} (o = 0: tail) ----
    double dv[16];
#pragma unroll
    for (int e = 0; e < 16; e++) dv[e] = 0.0;
#pragma unroll
    for (int q = 0; q < RPT; q++) {
      if (grow[q] > j && grow[q] < mm) {
#pragma unroll
        for (int o = 0; o < WL; o++) dv[o] += x[q][0] * x[q][o];
      }
      if (grow[q] == j)
#pragma unroll
        for (int o = 0; o < WL; o++) rowj[o] = x[q][o];
    }
    leaf_stamp(j, 1);
    const double dsum = warp_reduce_scatter16(dv, lane);
    if (lane < 16) wpart[warp][lane] = dsum;
    leaf_stamp(j, 2);
    __syncthreads();
    leaf_stamp(j, 3);
    {
      // every warp forms the CTA sum of slot `lane` (same order: identical values) and
      // pushes it to destinations warp, warp + 8: the remote stores are spread over all threads
      double sum = 0.0;
#pragma unroll
      for (int ww = 0; ww < LR_WARPS; ww++) sum += wpart[ww][lane];
      const bool owner = (unsigned)(j / rows_per) == rank;  // this CTA holds row j
      const double rv = (owner && lane < 16) ? rowj[lane] : 0.0;
      const uint32_t pin_l = smem_u32(&pin[par][rank][lane]);
      const uint32_t row_l = smem_u32(&rowp[par][lane & 15]);
      const uint32_t mb_l = smem_u32(&lmbar[par]);
#pragma unroll
      for (unsigned dst = warp; dst < CS; dst += LR_WARPS) {
        const uint32_t mb = cluster_map(mb_l, dst);
        if (lane < 16) st_async_f64(cluster_map(pin_l, dst), sum, mb);
        if (owner && lane < 16) st_async_f64(cluster_map(row_l, dst), rv, mb);
      }
    }
    leaf_stamp(j, 4);
    // warp 0 consumes the pushed partials; the others meet it at the __syncthreads below
    if (warp == 0) mbar_wait_cluster(&lmbar[par], (unsigned)(j >> 1) & 1u);
    leaf_stamp(j, 5);
    if (warp == 0) {
      double t = 0.0;
      double pv[CS];
#pragma unroll
      for (unsigned r = 0; r < CS; r++) pv[r] = (lane < 16) ? pin[par][r][lane] : 0.0;
#pragma unroll
      for (unsigned r = 0; r < CS; r++) t += pv[r];  // rank order
      {
        // row j entries (window order), pushed by the CTA that owns row j
        const double rj = (lane < 16 && j + lane < w) ? rowp[par][lane] : 0.0;
        const double tail = __shfl_sync(0xffffffffu, t, 0);
        const double xjj = __shfl_sync(0xffffffffu, rj, 0);
        const double normsq = xjj * xjj + tail;
        const bool refl = (mm - j >= 2) && (normsq != 0.0);
        double beta = 0.0, inv = 0.0, h = 0.0;
        if (refl) {
          const double nrm = sqrt(normsq);
          beta = (xjj >= 0.0) ? -nrm : nrm;
          h = beta - xjj;
          inv = 1.0 / sqrt(h * h + tail);
        }
        // coefficient for window slot o = lane (column j + o), dot_o on lane o
        if (lane < 16)
          sc[lane] = (refl && lane > 0 && j + lane < w) ? 2.0 * inv * (h * rj - t) : 0.0;
        if (lane == 0) {
          scal[0] = refl ? 1.0 : 0.0;
          scal[1] = beta;
          scal[2] = h * inv;
          scal[3] = inv;
        }
      }
    }
    leaf_stamp(j, 6);
    __syncthreads();
    leaf_stamp(j, 7);
    const bool refl = scal[0] != 0.0;
    const double beta = scal[1], hinv = scal[2], inv = scal[3];
#pragma unroll
    for (int q = 0; q < RPT; q++) {
      const int lr = threadIdx.x + LR_THREADS * q;
      double ui = 0.0;
      if (refl && grow[q] < mm) ui = (grow[q] == j) ? hinv : (grow[q] > j ? -x[q][0] * inv : 0.0);
      uprev[q] = ui;
      Vs[j * VLD + lr] = ui;
      // column j is final: write it out and shift the window
      if (grow[q] < mm) {
        const double rjv = (refl && grow[q] >= j) ? ((grow[q] == j) ? beta : 0.0) : x[q][0];
        a[(int64_t)j * lda + grow[q]] = rjv;
      }
#pragma unroll
      for (int o = 0; o + 1 < WL; o++) x[q][o] = x[q][o + 1];
      x[q][WL - 1] = 0.0;
    }
    refl_prev = refl;
  }
  __syncthreads();
  // write back V (R columns were written as they left the window)
#pragma unroll
  for (int q = 0; q < RPT; q++) {
    const int lr = threadIdx.x + LR_THREADS * q;
    if (grow[q] < mm)
      for (int c = 0; c < w; c++) v[(int64_t)c * ldv + grow[q]] = Vs[c * VLD + lr];
  }
  // ---- T (w x w): T_jj = 2, T(0:j, j) = -2 T(0:j, 0:j) (V(:, 0:j)^T u_j), from the Gram ----
  if (tl) {
    if (rank == 0 && threadIdx.x == 0) mbar_expect_tx(&gbar, CS * 120 * 8);
    // pairs p <-> (k, l), k < l < 16, l-major; warp w sums pairs w, w + 8, ... over its CTA's rows
    const uint32_t gin_l = smem_u32(&gin[rank][0]);
    const uint32_t gb0 = cluster_map(smem_u32(&gbar), 0u);
    for (int p = warp; p < 120; p += LR_WARPS) {
      int l = 1;
      while (l * (l + 1) / 2 <= p) l++;
      const int k = p - l * (l - 1) / 2;
      double acc = 0.0;
      if (l < w)
        for (int i = lane; i < VLD; i += 32) acc = fma(Vs[k * VLD + i], Vs[l * VLD + i], acc);
      acc = warp_sum(acc);
      if (lane == 0) st_async_f64(cluster_map(gin_l + 8 * p, 0u), acc, gb0);
    }
    if (rank == 0) {
      // Gram entries g(k, l): the 16 partials summed in rank order, one pair per thread
      mbar_wait_cluster(&gbar, 0u);
      if (threadIdx.x < 120) {
        double g = 0.0;
#pragma unroll
        for (unsigned r = 0; r < CS; r++) g += gin[r][threadIdx.x];
        gin[0][threadIdx.x] = g;  // (own slot: every read of this pair is done)
      }
      __syncthreads();
      if (warp == 0) {
        // T column by column (lane = row): T(0:jc, jc) = -2 T(0:jc, 0:jc) g(0:jc, jc)
        for (int jc = 0; jc < w; jc++) {
          double tcol = 0.0;
          const int p0 = jc * (jc - 1) / 2;
          for (int kk = jc - 1; kk >= 0; kk--)
            if (lane <= kk) tcol += Ts[lane][kk] * gin[0][p0 + kk];
          if (lane < jc) Ts[lane][jc] = -2.0 * tcol;
          if (lane == jc) Ts[jc][jc] = 2.0;
          __syncwarp();
        }
      }
      __syncthreads();
      for (int e = threadIdx.x; e < w * w; e += LR_THREADS) tl[(int64_t)(e / w) * ldt + e % w] = Ts[e % w][e / w];
    }
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int WL, int RPT>
static int launch_leaf_reg(const LeafCall& c, cudaStream_t st, int64_t* launches) {
  const int CS = 16;
  const int rows_per = (int)ceil_div(c.mm, CS);
  auto kern = leaf_reg_kernel<WL, RPT>;
  const size_t dsm = (size_t)RPT * LR_THREADS * WL * sizeof(double);
  static bool attr = false;
  if (!attr) {
    RQ_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    RQ_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CS);
  cfg.blockDim = dim3(LR_THREADS);
  cfg.dynamicSmemBytes = dsm;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  RQ_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, c.a, c.lda, c.mm, c.w, c.v, c.ldv, c.tl, c.ldt, rows_per));
  if (launches) (*launches)++;
  return RQ_OK;
}

// ---------------------------------------------------------------------------
// Fused WY update between panel leaves (one cooperative launch instead of three
// GEMMs):  A_rest <- (I - V T V^T)^T A_rest = A_rest - V T^T (V^T A_rest)
//   phase 1: every CTA forms the partial V^T A_rest over its row block
//   phase 2: column slices of W = sum of partials (CTA order: deterministic),
//            W2 = T^T W
//   phase 3: every CTA updates its row block with V W2
// ---------------------------------------------------------------------------
constexpr int WU_THREADS = 256;

struct WyUpdateArgs {
  double* a;  // A_rest top-left (mm x nr), lda
  int64_t lda;
  int64_t mm;
  int nr;
  const double* v;  // mm x w, ldv
  int64_t ldv;
  const double* t;  // w x w, ldt
  int64_t ldt;
  int w;
  int rows_per;
  double* part;  // G x w x nr partials
  double* w2;    // w x nr
  unsigned int* bar;
};

RQ_DEV void cp_async8(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}

__global__ void __launch_bounds__(WU_THREADS) wy_update_kernel(const WyUpdateArgs p) {
  extern __shared__ double sm[];
  const int G = gridDim.x;
  const int w = p.w, nr = p.nr;
  const int64_t r0 = (int64_t)blockIdx.x * p.rows_per;
  const int64_t r1 = min(p.mm, r0 + p.rows_per);
  const int nrows = (int)max((int64_t)0, r1 - r0);
  const int lds = p.rows_per | 1;              // odd stride: conflict-free column access
  double* Vr = sm;                             // rows_per x 16, row-major (zero-padded beyond w)
  double* As = Vr + (int64_t)p.rows_per * 16;  // nr columns x lds (this CTA's rows of A_rest)
  double* red = As + (int64_t)nr * lds;        // row-group partials (phase 1)
  // ---- stage the row block: every copy in flight at once (cp.async), V row-major ----
  for (int e = threadIdx.x; e < nr * nrows; e += WU_THREADS) {
    const int j = e / nrows, i = e - j * nrows;
    cp_async8(As + j * lds + i, p.a + (int64_t)j * p.lda + r0 + i);
  }
  for (int e = threadIdx.x; e < nrows * 16; e += WU_THREADS) {
    const int i = e >> 4, k = e & 15;
    if (k < w) cp_async8(Vr + e, p.v + (int64_t)k * p.ldv + r0 + i);
    else Vr[e] = 0.0;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  // ---- phase 1: partial W(k, j) over this block; thread -> (column j, row group) ----
  const int ngrp = nr >= WU_THREADS ? 1 : WU_THREADS / nr;
  double* mypart = p.part + (int64_t)blockIdx.x * nr * 16;  // [j][16]
  for (int jb = 0; jb < nr; jb += WU_THREADS) {
    const int j = jb + (threadIdx.x % (nr < WU_THREADS ? nr : WU_THREADS));
    const int grp = threadIdx.x / (nr < WU_THREADS ? nr : WU_THREADS);
    const bool live = grp < ngrp && j < nr;
    double acc[16];
#pragma unroll
    for (int k = 0; k < 16; k++) acc[k] = 0.0;
    if (live) {
      const double* ac = As + j * lds;
      for (int i = grp; i < nrows; i += ngrp) {
        const double av = ac[i];
        const double2* vr = reinterpret_cast<const double2*>(Vr + i * 16);
#pragma unroll
        for (int k2 = 0; k2 < 8; k2++) {
          const double2 vv = vr[k2];
          acc[2 * k2] = fma(vv.x, av, acc[2 * k2]);
          acc[2 * k2 + 1] = fma(vv.y, av, acc[2 * k2 + 1]);
        }
      }
    }
    if (ngrp > 1) {
      // combine the row groups in group order (deterministic)
      if (live && grp > 0)
#pragma unroll
        for (int k = 0; k < 16; k++) red[((grp - 1) * nr + j) * 17 + k] = acc[k];
      __syncthreads();
      if (live && grp == 0) {
        for (int g2 = 1; g2 < ngrp; g2++)
#pragma unroll
          for (int k = 0; k < 16; k++) acc[k] += red[((g2 - 1) * nr + j) * 17 + k];
      }
      __syncthreads();
    }
    if (live && grp == 0) {
      double2* dst = reinterpret_cast<double2*>(mypart + (int64_t)j * 16);
#pragma unroll
      for (int k2 = 0; k2 < 8; k2++) __stcg(dst + k2, make_double2(acc[2 * k2], acc[2 * k2 + 1]));
    }
  }
  unsigned int gen = 0;
  grid_barrier(p.bar, gen);
  // ---- phase 2: CTA g owns columns j = g, g+G, ...: W(:, j) = sum over CTAs (fixed order), W2 = T^T W ----
  __shared__ double wcol[16];
  __shared__ double wchunk[16][17];
  for (int j = blockIdx.x; j < nr; j += G) {
    {
      // thread (k, chunk): 16 chunks of CTAs summed in parallel, then combined in chunk order
      const int k = threadIdx.x & 15, ch = threadIdx.x >> 4;
      const int per = (G + 15) / 16;
      const int g0 = ch * per, g1 = min(G, g0 + per);
      double acc = 0.0;
      double vals[10];
      int g = g0;
      for (; g + 10 <= g1; g += 10) {
#pragma unroll
        for (int u = 0; u < 10; u++) vals[u] = __ldcg(p.part + ((int64_t)(g + u) * nr + j) * 16 + k);
#pragma unroll
        for (int u = 0; u < 10; u++) acc += vals[u];
      }
      for (; g < g1; g++) acc += __ldcg(p.part + ((int64_t)g * nr + j) * 16 + k);
      wchunk[k][ch] = acc;
    }
    __syncthreads();
    if (threadIdx.x < w) {
      double acc = 0.0;
      for (int ch = 0; ch < 16; ch++) acc += wchunk[threadIdx.x][ch];
      wcol[threadIdx.x] = acc;
    }
    __syncthreads();
    if (threadIdx.x < 16) {
      // (T^T W)_k = sum_{l <= k} T(l, k) W_l   (T upper triangular); zero beyond w
      double acc = 0.0;
      if (threadIdx.x < w)
        for (int l = 0; l <= threadIdx.x; l++) acc += p.t[(int64_t)threadIdx.x * p.ldt + l] * wcol[l];
      p.w2[(int64_t)j * 16 + threadIdx.x] = acc;
    }
    __syncthreads();
  }
  grid_barrier(p.bar, gen);
  // ---- phase 3: A(i, j) -= V(i, :) W2(:, j); thread -> (column j, row group), result back into As ----
  for (int jb = 0; jb < nr; jb += WU_THREADS) {
    const int j = jb + (threadIdx.x % (nr < WU_THREADS ? nr : WU_THREADS));
    const int grp = threadIdx.x / (nr < WU_THREADS ? nr : WU_THREADS);
    if (grp < ngrp && j < nr) {
      double w2[16];
      const double2* src = reinterpret_cast<const double2*>(p.w2 + (int64_t)j * 16);
#pragma unroll
      for (int k2 = 0; k2 < 8; k2++) {
        const double2 t2 = __ldcg(src + k2);
        w2[2 * k2] = t2.x;
        w2[2 * k2 + 1] = t2.y;
      }
      double* ac = As + j * lds;
      for (int i = grp; i < nrows; i += ngrp) {
        const double2* vr = reinterpret_cast<const double2*>(Vr + i * 16);
        double acc = 0.0;
#pragma unroll
        for (int k2 = 0; k2 < 8; k2++) {
          const double2 vv = vr[k2];
          acc = fma(vv.x, w2[2 * k2], acc);
          acc = fma(vv.y, w2[2 * k2 + 1], acc);
        }
        ac[i] -= acc;
      }
    }
  }
  __syncthreads();
  // coalesced write-back
  for (int e = threadIdx.x; e < nr * nrows; e += WU_THREADS) {
    const int j = e / nrows, i = e - j * nrows;
    p.a[(int64_t)j * p.lda + r0 + i] = As[j * lds + i];
  }
}

static size_t wy_update_smem(int64_t mm, int nr, int* G_out, int* rows_out) {
  int G = (int)ceil_div(mm, 32);
  if (G > kSMs) G = kSMs;
  if (G < 1) G = 1;
  const int rows_per = (int)ceil_div(mm, G);
  const int ngrp = nr >= WU_THREADS ? 1 : WU_THREADS / nr;
  if (G_out) *G_out = G;
  if (rows_out) *rows_out = rows_per;
  return ((size_t)rows_per * 16 + (size_t)(rows_per | 1) * nr + (ngrp > 1 ? (size_t)(ngrp - 1) * nr * 17 : 0)) *
         sizeof(double);
}

bool wy_update_fits(int64_t mm, int nr, int w) {
  return w <= 16 && nr > 0 && mm > 0 && wy_update_smem(mm, nr, nullptr, nullptr) <= 200 * 1024;
}

int wy_update(double* a, int64_t lda, int64_t mm, int nr, const double* v, int64_t ldv, const double* t, int64_t ldt,
              int w, double* scratch, size_t scratch_bytes, unsigned int* bar, cudaStream_t st, int64_t* launches) {
  if (nr <= 0 || mm <= 0) return RQ_OK;
  if (w > 16) return set_error(RQ_EINTERNAL, "wy_update: width %d > 16", w);
  int G = 0, rows_per = 0;
  const size_t smem = wy_update_smem(mm, nr, &G, &rows_per);
  if (smem > 200 * 1024) return set_error(RQ_EINTERNAL, "wy_update: %lld rows too many", (long long)mm);
  const size_t need = ((size_t)G * 16 * nr + (size_t)16 * nr) * sizeof(double);
  if (need > scratch_bytes) return set_error(RQ_EINTERNAL, "wy_update: scratch too small");
  WyUpdateArgs p;
  p.a = a;
  p.lda = lda;
  p.mm = mm;
  p.nr = nr;
  p.v = v;
  p.ldv = ldv;
  p.t = t;
  p.ldt = ldt;
  p.w = w;
  p.rows_per = rows_per;
  p.part = scratch;
  p.w2 = scratch + (size_t)G * 16 * nr;
  p.bar = bar;
  static bool attr = false;
  if (!attr) {
    RQ_CUDA_TRY(cudaFuncSetAttribute(wy_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  void* args[] = {(void*)&p};
  RQ_CUDA_TRY(cudaLaunchCooperativeKernel((void*)wy_update_kernel, dim3(G), dim3(WU_THREADS), args, smem, st));
  if (launches) (*launches)++;
  return RQ_OK;
}

// ---------------------------------------------------------------------------
// WY update of the rest of the panel on ONE 16-CTA cluster (16 SMs), for the look-ahead's
// space-sliced schedule (driver.cu): the previous panel's trailing update runs on the other
// 132 SMs meanwhile.  Same result as wy_update (A_rest <- A_rest - V T^T (V^T A_rest)) with a
// different summation order:
//   phase 1: CTA r forms P_r = V_r^T A_r over its row block on the FP64 tensor cores
//            (mma.sync m16n8k4: M = the w <= 16 reflectors, N = rest columns, K = rows);
//   phase 2: CTA r owns the rest columns n = r (mod 16): W(:, n) = sum over CTAs (rank order,
//            DSMEM loads), W2(:, n) = T^T W(:, n), pushed into every CTA's W2 table;
//   phase 3: A_r -= V_r W2 on the tensor cores (M = rows, N = rest columns, K = w).
// A_rest and V are read straight from global memory (L2): no row block is staged, so any
// height fits.
// ---------------------------------------------------------------------------
constexpr int WC_THREADS = 512;
constexpr int WC_WARPS = WC_THREADS / 32;
constexpr int WC_CS = 16;

RQ_DEV void wc_dmma(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// Row chunks of A_r (16 rows x all rest columns, one TMA box, 128B-swizzled) stream through
// WC_STAGES shared-memory stages; thread 0 issues the boxes and mbarriers track them, so no
// thread spends issue slots on addresses (per-element cp.async / loads left the kernel at
// ~20 GB/s per SM).  V_r fragments come from global memory (L1).
constexpr int WC_RC = 16;      // rows per chunk = one 128B swizzle row per column
constexpr int WC_STAGES = 4;

RQ_DEV void wc_mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
}
RQ_DEV void wc_mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WCW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WCW_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}
RQ_DEV void wc_tma(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// element (row k of the chunk, column c) of a 128B-swizzled [column][16] chunk
RQ_DEV double wc_ld(const double* tile, int c, int k) {
  return *reinterpret_cast<const double*>(reinterpret_cast<const char*>(tile) + c * 128 +
                                          ((((k >> 1) ^ (c & 7))) << 4) + ((k & 1) << 3));
}

__global__ void __launch_bounds__(WC_THREADS, 1)
    wy_cluster_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmV,
                      double* __restrict__ a, int64_t lda, int64_t mm, int nr, int64_t grow0, int64_t gcol0,
                      int64_t vrow0, int64_t vcol0, const double* __restrict__ t, int64_t ldt, int w, int rp) {
  extern __shared__ unsigned char wc_raw[];
  // 1024-B aligned stages (the 128B swizzle pattern repeats every 1 KB)
  const uint32_t mis = (uint32_t)__cvta_generic_to_shared(wc_raw) & 1023u;
  unsigned char* base = wc_raw + ((1024u - mis) & 1023u);
  const int nrp = (nr + 7) & ~7;
  const uint32_t a_bytes = (uint32_t)nrp * 128u;
  const uint32_t stage_bytes = a_bytes + 16u * 128u;                        // A box + V box
  double* stA = reinterpret_cast<double*>(base);  // [WC_STAGES] x {A [nrp][16], V [16][16]} (swizzled)
  // P and W2 rows padded to ldq = nrp + 4 (= 4 mod 16 doubles): the fragment reads of lanes
  // (g, tq) at row tq, column g hit distinct bank pairs (nrp = 0 mod 16 gave 4-way conflicts)
  const int ldq = nrp + 4;
  double* P = reinterpret_cast<double*>(base + WC_STAGES * stage_bytes);    // [16][ldq]
  double* W2s = P + 16 * ldq;                                               // [16][ldq]
  double* Wc = W2s + 16 * ldq;                                              // [16][nrp / 16 + 1]
  __shared__ __align__(8) uint64_t full[WC_STAGES];
  const unsigned rank = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int64_t r0 = (int64_t)rank * rp;
  const int64_t r1 = min(mm, r0 + rp);
  const int nrow = (int)max((int64_t)0, r1 - r0);
  const int shift = (int)((grow0 + r0) & 1);  // chunk boxes start at an even global row
  const int64_t cbase = r0 - shift;           // relative row of chunk 0's first row
  const int nchunks = nrow > 0 ? (nrow + shift + WC_RC - 1) / WC_RC : 0;
  const int ngroups = nrp / 8;
  constexpr int QG = (32 + WC_WARPS - 1) / WC_WARPS;  // n8 groups per warp (<= 30 groups)
  if (threadIdx.x == 0) {
    for (int s2 = 0; s2 < WC_STAGES; s2++) wc_mbar_init(&full[s2]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // load number q (phase 1: q = c, phase 3: q = nchunks + c) of chunk c goes to stage q % WC_STAGES;
  // that stage's barrier completes for the (q / WC_STAGES)-th time
  auto issue = [&](int q, int c) {
    double* st = stA + (size_t)(q % WC_STAGES) * (stage_bytes / 8);
    uint64_t* bar = &full[q % WC_STAGES];
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(stage_bytes)
                 : "memory");
    const int rr = (int)(cbase + c * WC_RC);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(st)),
        "l"(&tmA), "r"(smem_u32(bar)), "r"((int)(grow0 + rr)), "r"((int)gcol0)
        : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(st + nrp * 16)),
        "l"(&tmV), "r"(smem_u32(bar)), "r"((int)(vrow0 + rr)), "r"((int)vcol0)
        : "memory");
  };

  // ---- phase 1: P = V_r^T A_r (each warp: n8 groups warp, warp + WC_WARPS, ...) ----
  {
    double acc[QG][4];
#pragma unroll
    for (int q = 0; q < QG; q++)
#pragma unroll
      for (int e = 0; e < 4; e++) acc[q][e] = 0.0;
    if (threadIdx.x == 0)
      for (int c = 0; c < WC_STAGES && c < nchunks; c++) issue(c, c);
    for (int c = 0; c < nchunks; c++) {
      wc_mbar_wait(&full[c % WC_STAGES], (c / WC_STAGES) & 1);
      const double* As = stA + (size_t)(c % WC_STAGES) * (stage_bytes / 8);
      const double* Vs = As + nrp * 16;  // [reflector column][16 rows]
#pragma unroll
      for (int kk = 0; kk < 4; kk++) {
        const int k = kk * 4 + tq;                       // chunk row
        const int64_t row = cbase + c * WC_RC + k;       // relative to A_rest row 0
        const bool rok = row >= r0 && row < r1;          // (the box also holds neighbours' rows)
        const double a0 = (rok && g < w) ? wc_ld(Vs, g, k) : 0.0;
        const double a1 = (rok && g + 8 < w) ? wc_ld(Vs, g + 8, k) : 0.0;
#pragma unroll
        for (int q = 0; q < QG; q++) {
          const int grp = warp + WC_WARPS * q;
          if (grp < ngroups) wc_dmma(acc[q], a0, a1, wc_ld(As, grp * 8 + g, k));
        }
      }
      __syncthreads();  // every warp is done with this stage
      if (threadIdx.x == 0 && c + WC_STAGES < nchunks) issue(c + WC_STAGES, c + WC_STAGES);
    }
#pragma unroll
    for (int q = 0; q < QG; q++) {
      const int grp = warp + WC_WARPS * q;
      if (grp < ngroups) {
        const int n0 = grp * 8 + 2 * tq;
        P[g * ldq + n0] = acc[q][0];
        P[g * ldq + n0 + 1] = acc[q][1];
        P[(g + 8) * ldq + n0] = acc[q][2];
        P[(g + 8) * ldq + n0 + 1] = acc[q][3];
      }
    }
  }
  // phase 3's first chunks load while the cluster exchanges W
  if (threadIdx.x == 0)
    for (int c = 0; c < WC_STAGES && c < nchunks; c++) issue(nchunks + c, c);
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");

  // ---- phase 2: owned columns n = rank + 16 c: W = sum of the 16 partials, W2 = T^T W ----
  const int nown = (nr > (int)rank) ? (nr - (int)rank + WC_CS - 1) / WC_CS : 0;
  const int ldwc = nrp / 16 + 1;
  for (int e = threadIdx.x; e < 16 * nown; e += WC_THREADS) {
    const int k = e % 16, c = e / 16;
    const int n = (int)rank + WC_CS * c;
    double vals[WC_CS];
#pragma unroll
    for (unsigned r = 0; r < WC_CS; r++) vals[r] = dsmem_ld(&P[k * ldq + n], r);
    double s = 0.0;
#pragma unroll
    for (unsigned r = 0; r < WC_CS; r++) s += vals[r];  // rank order: deterministic
    Wc[k * ldwc + c] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 16 * nown; e += WC_THREADS) {
    const int k = e % 16, c = e / 16;
    const int n = (int)rank + WC_CS * c;
    double s = 0.0;
    if (k < w)
      for (int l = 0; l <= k; l++) s += t[(int64_t)k * ldt + l] * Wc[l * ldwc + c];  // (T^T W)_k, T upper
#pragma unroll
    for (unsigned r = 0; r < WC_CS; r++) dsmem_st(&W2s[k * ldq + n], r, s);
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");

  // ---- phase 3: A_r -= V_r W2, chunk by chunk (each warp: its n8 groups of the 16-row chunk) ----
  for (int c = 0; c < nchunks; c++) {
    const int q = nchunks + c;
    const int64_t rowa = cbase + c * WC_RC + g, rowb = rowa + 8;  // relative to A_rest row 0
    const bool oka = rowa >= r0 && rowa < r1, okb = rowb >= r0 && rowb < r1;
    wc_mbar_wait(&full[q % WC_STAGES], (q / WC_STAGES) & 1);
    const double* As = stA + (size_t)(q % WC_STAGES) * (stage_bytes / 8);
    const double* Vs = As + nrp * 16;
    double va[4], vb[4];
#pragma unroll
    for (int kk = 0; kk < 4; kk++) {
      const int k = kk * 4 + tq;
      va[kk] = (k < w) ? wc_ld(Vs, k, g) : 0.0;
      vb[kk] = (k < w) ? wc_ld(Vs, k, g + 8) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < QG; q++) {
      const int grp = warp + WC_WARPS * q;
      if (grp >= ngroups) break;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int kk = 0; kk < 4; kk++) wc_dmma(acc, va[kk], vb[kk], W2s[(kk * 4 + tq) * ldq + grp * 8 + g]);
      const int n0 = grp * 8 + 2 * tq;
      double* ca = a + (int64_t)n0 * lda;
      if (oka) {
        if (n0 < nr) __stcg(ca + rowa, wc_ld(As, n0, g) - acc[0]);
        if (n0 + 1 < nr) __stcg(ca + lda + rowa, wc_ld(As, n0 + 1, g) - acc[1]);
      }
      if (okb) {
        if (n0 < nr) __stcg(ca + rowb, wc_ld(As, n0, g + 8) - acc[2]);
        if (n0 + 1 < nr) __stcg(ca + lda + rowb, wc_ld(As, n0 + 1, g + 8) - acc[3]);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && c + WC_STAGES < nchunks) issue(q + WC_STAGES, c + WC_STAGES);
  }
}

size_t wy_cluster_smem(int nr) {
  const int nrp = (nr + 7) & ~7;
  return 1024 + (size_t)WC_STAGES * (nrp * 128 + 2048) +
         ((size_t)32 * (nrp + 4) + (size_t)16 * (nrp / 16 + 1)) * sizeof(double);
}

int wy_cluster(double* A, int64_t lda, int64_t m_total, int64_t n_total, int64_t row0, int64_t col0, int64_t mm,
               int nr, const double* Vb, int64_t ldv, int64_t v_rows, int64_t v_cols, int64_t vrow0, int64_t vcol0,
               const double* t, int64_t ldt, int w, cudaStream_t st, int64_t* launches) {
  if (nr <= 0 || mm <= 0) return RQ_OK;
  if (w > 16) return set_error(RQ_EINTERNAL, "wy_cluster: width %d > 16", w);
  const int nrp = (nr + 7) & ~7;
  if (nrp > 256) return set_error(RQ_EINTERNAL, "wy_cluster: %d rest columns > 256", nr);
  // rows per CTA: even, so every CTA's first row has the parity of row0
  const int rp = (int)((ceil_div(mm, WC_CS) + 1) & ~int64_t(1));
  const size_t smem = wy_cluster_smem(nr);
  if (smem > 220 * 1024) return set_error(RQ_EINTERNAL, "wy_cluster: %d rest columns too many", nr);
  if (((row0 ^ vrow0) & 1) != 0) return set_error(RQ_EINTERNAL, "wy_cluster: A and V row origins differ in parity");
  CUtensorMap map, vmap;
  RQ_TRY(make_tensor_map_f64(&map, A, m_total, n_total, lda, 16, nrp, true));
  RQ_TRY(make_tensor_map_f64(&vmap, Vb, v_rows, v_cols, ldv, 16, 16, true));
  static bool attr = false;
  if (!attr) {
    RQ_CUDA_TRY(cudaFuncSetAttribute(wy_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    RQ_CUDA_TRY(cudaFuncSetAttribute(wy_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(WC_CS);
  cfg.blockDim = dim3(WC_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = WC_CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  double* a = A + row0 + col0 * lda;
  RQ_CUDA_TRY(
      cudaLaunchKernelEx(&cfg, wy_cluster_kernel, map, vmap, a, lda, mm, nr, row0, col0, vrow0, vcol0, t, ldt, w, rp));
  if (launches) (*launches)++;
  return RQ_OK;
}

template <int WL>
static int launch_leaf(const LeafCall& c, cudaStream_t st, int64_t* launches) {
  constexpr int PV = LeafLayout<WL>::PV;
  const int CS = 16;
  const int rows_per = (int)ceil_div(c.mm, CS);
  const size_t smem = ((size_t)2 * rows_per * WL + PV + 2 * 16 * PV + PV + WL + WL * WL + 8) * sizeof(double);
  if (smem > 227 * 1024) return set_error(RQ_EINTERNAL, "leaf_qr: %lld rows x %d too large for smem", (long long)c.mm, WL);
  auto kern = leaf_qr_kernel<WL>;
  static bool attr = false;
  if (!attr) {
    RQ_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    RQ_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CS);
  cfg.blockDim = dim3(PL_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  RQ_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, c.a, c.lda, c.mm, c.w, c.v, c.ldv, c.tl, c.ldt, rows_per));
  if (launches) (*launches)++;
  return RQ_OK;
}

static size_t leaf_smem(int64_t mm, int WL) {
  const int64_t rows_per = ceil_div(mm, 16);
  const int PV = 3 * WL + 1;
  return ((size_t)2 * rows_per * WL + 34 * PV + WL + WL * WL + 8) * sizeof(double);
}

int leaf_width_for(int64_t mm) {
  // own rows of A and V plus the pushed partials must fit one CTA's shared memory
  for (int wl : {32, 16, 8, 4})
    if (leaf_smem(mm, wl) <= 220 * 1024) return wl;
  return 0;
}

// Register-resident leaf width for mm rows (16 CTAs x 256 threads x RPT rows).
int leaf_reg_width_for(int64_t mm) {
  const int64_t rows_per = ceil_div(mm, 16);
  if (rows_per <= 4 * LR_THREADS) return 16;
  if (rows_per <= 8 * LR_THREADS) return 8;
  if (rows_per <= 16 * LR_THREADS) return 4;
  return 0;
}

int leaf_qr(const LeafCall& c, cudaStream_t st, int64_t* launches) {
  if (c.w <= 0) return RQ_OK;
  {
    const int64_t rows_per = ceil_div(c.mm, 16);
    if (rows_per <= 1 * LR_THREADS && c.w <= 16) return launch_leaf_reg<16, 1>(c, st, launches);
    if (rows_per <= 2 * LR_THREADS && c.w <= 16) return launch_leaf_reg<16, 2>(c, st, launches);
    if (rows_per <= 3 * LR_THREADS && c.w <= 16) return launch_leaf_reg<16, 3>(c, st, launches);
    if (rows_per <= 4 * LR_THREADS && c.w <= 16) return launch_leaf_reg<16, 4>(c, st, launches);
    if (rows_per <= 8 * LR_THREADS && c.w <= 8) return launch_leaf_reg<8, 8>(c, st, launches);
    if (rows_per <= 16 * LR_THREADS && c.w <= 4) return launch_leaf_reg<4, 16>(c, st, launches);
  }
  if (c.w <= 4 && leaf_width_for(c.mm) >= 4) return launch_leaf<4>(c, st, launches);
  if (c.w <= 8 && leaf_width_for(c.mm) >= 8) return launch_leaf<8>(c, st, launches);
  if (c.w <= 16 && leaf_width_for(c.mm) >= 16) return launch_leaf<16>(c, st, launches);
  if (c.w <= 32 && leaf_width_for(c.mm) >= 32) return launch_leaf<32>(c, st, launches);
  return set_error(RQ_EINTERNAL, "leaf_qr: width %d too wide for %lld rows", c.w, (long long)c.mm);
}

}  // namespace rq
