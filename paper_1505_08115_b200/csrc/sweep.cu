// Column-distributed Householder sweep with optional column pivoting.
//
// Restates the reference kernel householder_sweep (contract
// _kernels_numpy.py:11-22, loop structure _kernels_numba.py:13-61):
//   step j: [pivot] pick the column of largest trailing norm (rows j..m-1),
//           strict '>' -> lowest position wins ties; swap it into position j;
//           if m - j >= 2 and the column is nonzero: beta = -sign(x_j)||x||
//           (sign(0) = +1), u = (beta e_j - x)/||beta e_j - x||, apply
//           H = I - 2 u u^T to every later column, write beta and zeros.
//
// B200 mapping: one cooperative launch, CTAs own contiguous column ranges
// (cached in shared memory when they fit), ONE grid barrier per step.  Columns
// never move: positions are labels, so a "swap" is two integer updates and the
// R output is gathered once at the end.  Each step every CTA publishes its
// best candidate (key, tail norm, position) plus the candidate column; after
// the barrier all CTAs pick the same winner and build the same reflector.
//
// Extra "accumulate" columns [n, n + n_acc) receive every reflector but never
// pivot; the driver appends I_b there to obtain Q2^T of the b x b CPQR.
#include "common.cuh"
#include "sk_common.cuh"
#include "sweep.cuh"

namespace rq {

constexpr int SW_THREADS = 256;
constexpr int SW_WARPS = SW_THREADS / 32;

struct SweepSlot {
  double key;   // trailing norm^2 rows j..m-1 (-1: no candidate)
  double tail;  // trailing norm^2 rows j+1..m-1
  int pos;
  int col;
};

struct SweepArgs {
  double* a;
  int64_t lda;
  int64_t m;
  int n;       // pivot-eligible columns
  int n_acc;   // accumulate-only columns after them
  int steps;
  int pivot;
  const int* init_pos;  // n entries or null (identity)
  double* v;            // m x steps or null
  int64_t ldv;
  int* col_at_pos;      // n entries out (may be null)
  double* r_out;        // m x n, R gathered in position order (may be null)
  int64_t ldr;
  SweepSlot* slots;     // 2 * G
  double* slotdata;     // 2 * G * m
  double* ubuf_global;  // G * m when u does not fit in smem
  unsigned int* bar;
  int cache_cols;       // per-CTA columns cached in smem
  int u_in_smem;
};

// Smem layout: [u (m doubles, if u_in_smem)] [cached columns (cache_cols * m)]
//              [pos (cols_per_cta ints)] [active (cols_per_cta)] [reduce scratch]
__global__ void __launch_bounds__(SW_THREADS) sweep_kernel(const SweepArgs p) {
  // a kernel launched after this one with programmatic stream serialization (the
  // overlapped W = V^T A2 GEMM, driver.cu) may start once every CTA is resident
  asm volatile("griddepcontrol.launch_dependents;");
  extern __shared__ double sm[];
  const int G = gridDim.x;
  const int total_cols = p.n + p.n_acc;
  const int per = (total_cols + G - 1) / G;
  const int c0 = blockIdx.x * per;
  const int c1 = min(total_cols, c0 + per);
  const int ncols = max(0, c1 - c0);
  const int64_t m = p.m;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  double* u = p.u_in_smem ? sm : p.ubuf_global + (int64_t)blockIdx.x * m;
  double* cache = sm + (p.u_in_smem ? m : 0);
  const int ncache = min(ncols, p.cache_cols);
  int* pos = reinterpret_cast<int*>(cache + (int64_t)p.cache_cols * m);
  unsigned char* active = reinterpret_cast<unsigned char*>(pos + per);
  SweepSlot* red = reinterpret_cast<SweepSlot*>(
      (reinterpret_cast<uintptr_t>(active + per) + 15) & ~uintptr_t(15));

  auto colptr = [&](int lc) -> double* {
    return lc < ncache ? cache + (int64_t)lc * m : p.a + (int64_t)(c0 + lc) * p.lda;
  };

  // load cached columns, init positions
  for (int lc = warp; lc < ncache; lc += SW_WARPS) {
    const double* src = p.a + (int64_t)(c0 + lc) * p.lda;
    double* dst = cache + (int64_t)lc * m;
    for (int64_t i = lane; i < m; i += 32) dst[i] = src[i];
  }
  for (int lc = threadIdx.x; lc < ncols; lc += SW_THREADS) {
    const int c = c0 + lc;
    pos[lc] = (c < p.n) ? (p.init_pos ? p.init_pos[c] : c) : -1;
    active[lc] = 1;
  }
  __syncthreads();

  unsigned int gen = 0;
  bool have_refl = false;
  int rj = -1;  // row where the pending reflector starts
  double* slotdata_mine;

  for (int j = 0; j <= p.steps; j++) {
    const bool last = (j == p.steps);
    // ---------------- phase A: apply pending reflector, score candidates ----------------
    double best_key = -1.0, best_tail = 0.0;
    int best_pos = INT_MAX, best_lc = -1;
    for (int lc = warp; lc < ncols; lc += SW_WARPS) {
      if (!active[lc]) continue;
      double* col = colptr(lc);
      if (have_refl) {
        double d = 0.0;
        for (int64_t i = rj + lane; i < m; i += 32) d += u[i] * col[i];
        d = 2.0 * warp_sum(d);
        for (int64_t i = rj + lane; i < m; i += 32) col[i] -= d * u[i];
      }
      if (last) continue;
      const bool eligible = (c0 + lc < p.n) && (p.pivot ? true : pos[lc] == j);
      if (!eligible) continue;
      double t = 0.0;
      for (int64_t i = j + 1 + lane; i < m; i += 32) t += col[i] * col[i];
      t = warp_sum(t);
      const double xj = col[j];
      const double key = xj * xj + t;
      if (piv_better(key, pos[lc], best_key, best_pos)) {
        best_key = key;
        best_tail = t;
        best_pos = pos[lc];
        best_lc = lc;
      }
    }
    if (last) break;
    // block argmax over warps (lane 0 holds each warp's candidate)
    if (lane == 0) red[warp] = SweepSlot{best_key, best_tail, best_pos, best_lc};
    __syncthreads();
    if (threadIdx.x == 0) {
      SweepSlot b = red[0];
      for (int w = 1; w < SW_WARPS; w++)
        if (red[w].col >= 0 && (b.col < 0 || piv_better(red[w].key, red[w].pos, b.key, b.pos))) b = red[w];
      red[SW_WARPS] = b;
      SweepSlot out = b;
      if (b.col >= 0) out.col = c0 + b.col;
      else out.key = -1.0;
      p.slots[(j & 1) * G + blockIdx.x] = out;
    }
    __syncthreads();
    slotdata_mine = p.slotdata + ((int64_t)(j & 1) * G + blockIdx.x) * m;
    if (red[SW_WARPS].col >= 0) {
      const double* src = colptr(red[SW_WARPS].col);
      for (int64_t i = j + threadIdx.x; i < m; i += SW_THREADS) slotdata_mine[i] = src[i];
    }
    grid_barrier(p.bar, gen);

    // ---------------- phase B: every CTA picks the same winner ----------------
    if (warp == 0) {
      SweepSlot b{-1.0, 0.0, INT_MAX, -1};
      int bcta = -1;
      for (int c = lane; c < G; c += 32) {
        SweepSlot s;
        const SweepSlot* sp = &p.slots[(j & 1) * G + c];
        s.key = __ldcg(&sp->key);
        s.tail = __ldcg(&sp->tail);
        s.pos = __ldcg(&sp->pos);
        s.col = __ldcg(&sp->col);
        if (s.key >= 0.0 && (bcta < 0 || piv_better(s.key, s.pos, b.key, b.pos))) {
          b = s;
          bcta = c;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        double k2 = __shfl_xor_sync(0xffffffffu, b.key, o);
        double t2 = __shfl_xor_sync(0xffffffffu, b.tail, o);
        int p2 = __shfl_xor_sync(0xffffffffu, b.pos, o);
        int c2 = __shfl_xor_sync(0xffffffffu, b.col, o);
        int cta2 = __shfl_xor_sync(0xffffffffu, bcta, o);
        if (cta2 >= 0 && (bcta < 0 || piv_better(k2, p2, b.key, b.pos))) {
          b = SweepSlot{k2, t2, p2, c2};
          bcta = cta2;
        }
      }
      if (lane == 0) {
        red[SW_WARPS + 1] = b;
        reinterpret_cast<int*>(&red[SW_WARPS + 2])[0] = bcta;
      }
    }
    __syncthreads();
    const SweepSlot win = red[SW_WARPS + 1];
    const int wcta = reinterpret_cast<int*>(&red[SW_WARPS + 2])[0];
    const double* x = p.slotdata + ((int64_t)(j & 1) * G + wcta) * m;
    const double xj = __ldcg(&x[j]);
    const bool refl = (m - j >= 2) && (win.key != 0.0);
    double beta = 0.0, inv = 0.0;
    if (refl) {
      const double nrm = sqrt(win.key);
      beta = (xj >= 0.0) ? -nrm : nrm;
      const double h = beta - xj;
      inv = 1.0 / sqrt(h * h + win.tail);
      for (int64_t i = j + threadIdx.x; i < m; i += SW_THREADS)
        u[i] = (i == j) ? h * inv : -__ldcg(&x[i]) * inv;
    }
    // position bookkeeping: winner takes position j, the column at j takes win.pos
    for (int lc = threadIdx.x; lc < ncols; lc += SW_THREADS) {
      const int c = c0 + lc;
      if (c == win.col) {
        pos[lc] = j;
        active[lc] = 0;
      } else if (pos[lc] == j) {
        pos[lc] = win.pos;
      }
    }
    __syncthreads();
    // the winner's owner finalises the column: beta e_j (rows >= j)
    if (win.col >= c0 && win.col < c1 && refl) {
      double* col = colptr(win.col - c0);
      for (int64_t i = j + threadIdx.x; i < m; i += SW_THREADS) col[i] = (i == j) ? beta : 0.0;
    }
    if (blockIdx.x == 0) {
      if (p.v && refl)
        for (int64_t i = j + threadIdx.x; i < m; i += SW_THREADS) p.v[(int64_t)j * p.ldv + i] = u[i];
      if (p.col_at_pos && threadIdx.x == 0) p.col_at_pos[j] = win.col;
    }
    have_refl = refl;
    rj = j;
    __syncthreads();
  }

  // write back cached columns; publish final positions of the never-chosen columns
  for (int lc = warp; lc < ncache; lc += SW_WARPS) {
    double* dst = p.a + (int64_t)(c0 + lc) * p.lda;
    const double* src = cache + (int64_t)lc * m;
    for (int64_t i = lane; i < m; i += 32) dst[i] = src[i];
  }
  if (p.col_at_pos)
    for (int lc = threadIdx.x; lc < ncols; lc += SW_THREADS)
      if (c0 + lc < p.n && active[lc]) p.col_at_pos[pos[lc]] = c0 + lc;
  if (p.r_out) {
    grid_barrier(p.bar, gen);
    // gather R in position order: one warp per output column
    for (int k = blockIdx.x * SW_WARPS + warp; k < p.n; k += G * SW_WARPS) {
      const int c = __ldcg(&p.col_at_pos[k]);
      const double* src = p.a + (int64_t)c * p.lda;
      double* dst = p.r_out + (int64_t)k * p.ldr;
      for (int64_t i = lane; i < m; i += 32) dst[i] = __ldcg(&src[i]);
    }
  }
}

// ---------------------------------------------------------------------------
// Cluster variant: the whole matrix lives in the shared memory of one thread-
// block cluster (<= 16 CTAs).  Candidates and the winning column are exchanged
// through DSMEM and the per-step barrier is the hardware cluster barrier
// (0.22 us measured vs 1.2 us for a grid barrier).  Used for the b x b CPQR
// of R' (with Q2^T accumulation) and any sweep that fits.
// ---------------------------------------------------------------------------
constexpr int SC_THREADS = 512;
constexpr int SC_WARPS = SC_THREADS / 32;

RQ_DEV uint32_t dsmem_addr(const void* local, unsigned rank) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(local);
  uint32_t r;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
RQ_DEV double dsmem_f64(const double* local, unsigned rank) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(dsmem_addr(local, rank)));
  return v;
}
RQ_DEV int dsmem_i32(const int* local, unsigned rank) {
  int v;
  asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(dsmem_addr(local, rank)));
  return v;
}
RQ_DEV void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Optional phase timestamps (rank 0, thread 0, first 64 steps) for tuning.
__device__ unsigned long long g_sweep_dbg[64 * 8];
__device__ int g_sweep_dbg_on;
// Compiled in only with -DRQ_STAMPS (tuning builds; see leaf_stamp in panel.cu).
RQ_DEV void dbg_stamp(int j, int k) {
#ifdef RQ_STAMPS
  if (blockIdx.x == 0 && threadIdx.x == 0 && j < 64) {  // (stamps build: always on)
    unsigned long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
    g_sweep_dbg[j * 8 + k] = c;
  }
#else
  (void)j;
  (void)k;
#endif
}

RQ_DEV void dsmem_st_f64(double* local, unsigned rank, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(dsmem_addr(local, rank)), "d"(v) : "memory");
}
RQ_DEV void dsmem_st_i32(int* local, unsigned rank, int v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(dsmem_addr(local, rank)), "r"(v) : "memory");
}

// Push-based exchange: before each barrier a CTA *stores* what the others need
// into their shared memory (DSMEM stores are fire-and-forget); after the
// barrier every read is local.  Two cluster barriers per step: candidates,
// then the winning column.
__global__ void __launch_bounds__(SC_THREADS) sweep_cluster_kernel(const SweepArgs p) {
  // a kernel launched after this one with programmatic stream serialization (the
  // overlapped W = V^T A2 GEMM, driver.cu) may start once every CTA is resident
  asm volatile("griddepcontrol.launch_dependents;");
  extern __shared__ double sm[];
  const unsigned CS = gridDim.x;
  const unsigned rank = blockIdx.x;
  const int total_cols = p.n + p.n_acc;
  const int per = (total_cols + CS - 1) / CS;
  const int c0 = rank * per;
  const int c1 = min(total_cols, c0 + per);
  const int ncols = max(0, c1 - c0);
  const int64_t m = p.m;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  double* cols = sm;                                   // per x m
  double* u = cols + (int64_t)per * m;                 // m
  double* xin = u + m;                                 // 2 x m: winning column pushed by its owner
  SweepSlot* keys = reinterpret_cast<SweepSlot*>(xin + 2 * m);  // 2 x 16 pushed candidates
  SweepSlot* red = keys + 32;                          // SC_WARPS + 2 scratch
  int* pos = reinterpret_cast<int*>(red + SC_WARPS + 2);
  unsigned char* active = reinterpret_cast<unsigned char*>(pos + per);

  for (int lc = warp; lc < ncols; lc += SC_WARPS) {
    const double* src = p.a + (int64_t)(c0 + lc) * p.lda;
    double* dst = cols + (int64_t)lc * m;
    for (int64_t i = lane; i < m; i += 32) dst[i] = src[i];
  }
  for (int lc = threadIdx.x; lc < ncols; lc += SC_THREADS) {
    const int c = c0 + lc;
    pos[lc] = (c < p.n) ? (p.init_pos ? p.init_pos[c] : c) : -1;
    active[lc] = 1;
  }
  __syncthreads();
  cluster_barrier();  // every CTA initialised before anyone pushes into it

  bool have_refl = false;
  int rj = -1;
  for (int j = 0; j <= p.steps; j++) {
    const bool last = (j == p.steps);
    const int par = j & 1;
    dbg_stamp(j, 0);
    double best_key = -1.0, best_tail = 0.0;
    int best_pos = INT_MAX, best_lc = -1;
    for (int lc = warp; lc < ncols; lc += SC_WARPS) {
      if (!active[lc]) continue;
      double* col = cols + (int64_t)lc * m;
      if (have_refl) {
        double d0 = 0.0, d1 = 0.0;
        int64_t i = rj + lane;
        for (; i + 32 < m; i += 64) {
          d0 += u[i] * col[i];
          d1 += u[i + 32] * col[i + 32];
        }
        if (i < m) d0 += u[i] * col[i];
        const double d = 2.0 * warp_sum(d0 + d1);
        double t = 0.0;
        for (int64_t r = rj + lane; r < m; r += 32) {
          const double v = col[r] - d * u[r];
          col[r] = v;
          if (r > j) t += v * v;
        }
        if (last) continue;
        const bool eligible = (c0 + lc < p.n) && (p.pivot ? true : pos[lc] == j);
        if (!eligible) continue;
        t = warp_sum(t);
        const double xj = col[j];
        const double key = xj * xj + t;
        if (piv_better(key, pos[lc], best_key, best_pos)) {
          best_key = key;
          best_tail = t;
          best_pos = pos[lc];
          best_lc = lc;
        }
      } else {
        if (last) continue;
        const bool eligible = (c0 + lc < p.n) && (p.pivot ? true : pos[lc] == j);
        if (!eligible) continue;
        double t = 0.0;
        for (int64_t r = j + 1 + lane; r < m; r += 32) t += col[r] * col[r];
        t = warp_sum(t);
        const double xj = col[j];
        const double key = xj * xj + t;
        if (piv_better(key, pos[lc], best_key, best_pos)) {
          best_key = key;
          best_tail = t;
          best_pos = pos[lc];
          best_lc = lc;
        }
      }
    }
    if (last) break;
    // CTA-local argmax across warps (warp 0 reduces the per-warp candidates)
    if (lane == 0) red[warp] = SweepSlot{best_key, best_tail, best_pos, best_lc};
    __syncthreads();
    dbg_stamp(j, 1);
    if (warp == 0) {
      SweepSlot b = (lane < SC_WARPS) ? red[lane] : SweepSlot{-1.0, 0.0, INT_MAX, -1};
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double k2 = __shfl_xor_sync(0xffffffffu, b.key, o);
        const double t2 = __shfl_xor_sync(0xffffffffu, b.tail, o);
        const int p2 = __shfl_xor_sync(0xffffffffu, b.pos, o);
        const int c2 = __shfl_xor_sync(0xffffffffu, b.col, o);
        if (c2 >= 0 && (b.col < 0 || piv_better(k2, p2, b.key, b.pos))) b = SweepSlot{k2, t2, p2, c2};
      }
      // push the candidate (global column id) into every CTA's key table
      if (lane < (int)CS) {
        SweepSlot* dst = &keys[par * 16 + rank];
        dsmem_st_f64(&dst->key, lane, b.col >= 0 ? b.key : -1.0);
        dsmem_st_f64(&dst->tail, lane, b.tail);
        dsmem_st_i32(&dst->pos, lane, b.pos);
        dsmem_st_i32(&dst->col, lane, b.col >= 0 ? c0 + b.col : -1);
      }
      if (lane == 0) red[SC_WARPS] = b;
    }
    dbg_stamp(j, 2);
    cluster_barrier();
    dbg_stamp(j, 3);
    // every CTA picks the same winner from its local table (ranks in order)
    if (warp == 0) {
      SweepSlot b{-1.0, 0.0, INT_MAX, -1};
      int brank = -1;
      if (lane < (int)CS) {
        b = keys[par * 16 + lane];
        if (b.key >= 0.0) brank = lane;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double k2 = __shfl_xor_sync(0xffffffffu, b.key, o);
        const double t2 = __shfl_xor_sync(0xffffffffu, b.tail, o);
        const int p2 = __shfl_xor_sync(0xffffffffu, b.pos, o);
        const int c2 = __shfl_xor_sync(0xffffffffu, b.col, o);
        const int r2 = __shfl_xor_sync(0xffffffffu, brank, o);
        if (r2 >= 0 && (brank < 0 || piv_better(k2, p2, b.key, b.pos))) {
          b = SweepSlot{k2, t2, p2, c2};
          brank = r2;
        }
      }
      if (lane == 0) {
        red[SC_WARPS + 1] = b;
        reinterpret_cast<int*>(&red[SC_WARPS])[2] = brank;
      }
    }
    __syncthreads();
    dbg_stamp(j, 4);
    const SweepSlot win = red[SC_WARPS + 1];
    const unsigned wrank = (unsigned)reinterpret_cast<int*>(&red[SC_WARPS])[2];
    double* xs = xin + (int64_t)par * m;
    if (rank == wrank) {
      // the owner pushes the winning column (rows j..m-1) to every CTA
      const double* src = cols + (int64_t)(win.col - c0) * m;
      for (int dstr = warp; dstr < (int)CS; dstr += SC_WARPS)
        for (int64_t i = j + lane; i < m; i += 32) dsmem_st_f64(xs + i, (unsigned)dstr, src[i]);
    }
    dbg_stamp(j, 5);
    cluster_barrier();
    dbg_stamp(j, 6);
    const double xj = xs[j];
    const bool refl = (m - j >= 2) && (win.key != 0.0);
    double beta = 0.0;
    if (refl) {
      const double nrm = sqrt(win.key);
      beta = (xj >= 0.0) ? -nrm : nrm;
      const double h = beta - xj;
      const double inv = 1.0 / sqrt(h * h + win.tail);
      for (int64_t i = j + threadIdx.x; i < m; i += SC_THREADS) u[i] = (i == j) ? h * inv : -xs[i] * inv;
    }
    for (int lc = threadIdx.x; lc < ncols; lc += SC_THREADS) {
      const int c = c0 + lc;
      if (c == win.col) {
        pos[lc] = j;
        active[lc] = 0;
      } else if (pos[lc] == j) {
        pos[lc] = win.pos;
      }
    }
    __syncthreads();
    if (win.col >= c0 && win.col < c1 && refl) {
      double* col = cols + (int64_t)(win.col - c0) * m;
      for (int64_t i = j + threadIdx.x; i < m; i += SC_THREADS) col[i] = (i == j) ? beta : 0.0;
    }
    if (rank == 0) {
      if (p.v && refl)
        for (int64_t i = j + threadIdx.x; i < m; i += SC_THREADS) p.v[(int64_t)j * p.ldv + i] = u[i];
      if (p.col_at_pos && threadIdx.x == 0) p.col_at_pos[j] = win.col;
    }
    have_refl = refl;
    rj = j;
    __syncthreads();
    dbg_stamp(j, 7);
  }
  // outputs: accumulate columns in place, pivot columns scattered by final position
  for (int lc = warp; lc < ncols; lc += SC_WARPS) {
    const int c = c0 + lc;
    const double* src = cols + (int64_t)lc * m;
    double* dst;
    if (c >= p.n) dst = p.a + (int64_t)c * p.lda;
    else if (p.r_out) dst = p.r_out + (int64_t)pos[lc] * p.ldr;
    else dst = p.a + (int64_t)c * p.lda;
    for (int64_t i = lane; i < m; i += 32) dst[i] = src[i];
  }
  if (p.col_at_pos)
    for (int lc = threadIdx.x; lc < ncols; lc += SC_THREADS)
      if (c0 + lc < p.n && active[lc]) p.col_at_pos[pos[lc]] = c0 + lc;
  cluster_barrier();  // no CTA exits while others may still push into it
}

// ---------------------------------------------------------------------------
// Register-resident cluster sweep for m <= 32*RPL rows and <= 16 columns per
// CTA (the b x b CPQR of R' and small final blocks): warp w of CTA r owns
// column r*16 + w, lane l holds rows l, l+32, ... in registers.  Per step:
// apply the pending reflector and score (registers + one smem broadcast of u),
// CTA argmax with __reduce_*_sync, stage the candidate column in local smem,
// ONE cluster barrier, pull the 16 keys and then the winning column over DSMEM.
// ---------------------------------------------------------------------------
struct RegKey {
  unsigned hi, lo;  // bits of the non-negative key (monotone as integers)
  int pos;
  int col;          // global column id, -1 = none
  double tail;      // trailing norm^2 below row j
  double xj;        // the candidate's entry in row j
};

RQ_DEV void push_key(RegKey* local_slot, unsigned rank, const RegKey& k) {
  const uint32_t a = dsmem_addr(local_slot, rank);
  asm volatile("st.shared::cluster.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(k.hi), "r"(k.lo) : "memory");
  asm volatile("st.shared::cluster.v2.s32 [%0], {%1, %2};" ::"r"(a + 8), "r"(k.pos), "r"(k.col) : "memory");
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(a + 16), "d"(k.tail), "d"(k.xj) : "memory");
}

template <int RPL>
__global__ void __launch_bounds__(512) sweep_reg_kernel(const SweepArgs p) {
  // a kernel launched after this one with programmatic stream serialization (the
  // overlapped W = V^T A2 GEMM, driver.cu) may start once every CTA is resident
  asm volatile("griddepcontrol.launch_dependents;");
  __shared__ double u[32 * RPL];
  __shared__ double cand[2][32 * RPL];          // this CTA's candidate column, by step parity
  __shared__ __align__(16) RegKey keys[2][16];  // candidates pushed by every CTA, by parity
  __shared__ RegKey wk[16];
  __shared__ __align__(8) unsigned long long kmbar[2];  // key pushes of step j complete on kmbar[j & 1]
  const unsigned CS = gridDim.x;
  const unsigned rank = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = (int)p.m;
  const int c = (int)rank * 16 + warp;  // global column owned by this warp
  const bool own = c < p.n;
  double x[RPL];
#pragma unroll
  for (int k = 0; k < RPL; k++) {
    const int i = lane + 32 * k;
    x[k] = (own && i < m) ? p.a[(int64_t)c * p.lda + i] : 0.0;
  }
  int pos = own ? (p.init_pos ? p.init_pos[c] : c) : INT_MAX;
  bool active = own;
  bool have_refl = false;
  int rj = -1;
  if (threadIdx.x == 0) {
    mbar_init(&kmbar[0], 1);
    mbar_init(&kmbar[1], 1);
    mbar_init_fence();
  }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");

  for (int j = 0; j <= p.steps; j++) {
    const bool last = (j == p.steps);
    const int par = j & 1;
    if (!last && threadIdx.x == 0) mbar_expect_tx(&kmbar[par], CS * (unsigned)sizeof(RegKey));
    // ---- A: apply the pending reflector to this warp's column, score it ----
    dbg_stamp(j, 0);
    double tail = 0.0;
    if (active) {
      if (have_refl) {
        double uk[RPL], pr[RPL];
#pragma unroll
        for (int k = 0; k < RPL; k++) {
          const int i = lane + 32 * k;
          uk[k] = (i >= rj && i < m) ? u[i] : 0.0;
          pr[k] = uk[k] * x[k];
        }
#pragma unroll
        for (int w2 = 1; w2 < RPL; w2 <<= 1)  // pairwise tree: depth log2(RPL)
#pragma unroll
          for (int k = 0; k + w2 < RPL; k += 2 * w2) pr[k] += pr[k + w2];
        const double d = 2.0 * warp_sum(pr[0]);
#pragma unroll
        for (int k = 0; k < RPL; k++) x[k] -= d * uk[k];
      }
      if (!last) {
        double sq[RPL];
#pragma unroll
        for (int k = 0; k < RPL; k++) {
          const int i = lane + 32 * k;
          sq[k] = (i > j && i < m) ? x[k] * x[k] : 0.0;
        }
#pragma unroll
        for (int w2 = 1; w2 < RPL; w2 <<= 1)
#pragma unroll
          for (int k = 0; k + w2 < RPL; k += 2 * w2) sq[k] += sq[k + w2];
        tail = warp_sum(sq[0]);
      }
    }
    if (last) break;
    double sel = 0.0;
    const int kj = j >> 5;
#pragma unroll
    for (int k = 0; k < RPL; k++) sel = (k == kj) ? x[k] : sel;  // select chain keeps x[] in registers
    const double xj = __shfl_sync(0xffffffffu, sel, j & 31);
    const bool elig = active && (p.pivot ? true : pos == j);
    const double key = xj * xj + tail;
    // ---- B/C: CTA candidate, pushed into every CTA's key table ----
    if (lane == 0) {
      const unsigned long long kb = __double_as_longlong(key);
      wk[warp] = RegKey{(unsigned)(kb >> 32), (unsigned)kb, pos, elig ? c : -1, tail, xj};
    }
    dbg_stamp(j, 1);
    __syncthreads();
    dbg_stamp(j, 2);
    {
      // the CTA's best warp (same answer in every warp) stages its column for the cluster
      const RegKey r = lane < 16 ? wk[lane] : RegKey{0u, 0u, INT_MAX, -1, 0.0, 0.0};
      const int wl = warp_argmax(r.hi, r.lo, r.pos, r.col >= 0);
      if (wl == warp) {
#pragma unroll
        for (int k = 0; k < RPL; k++) {
          const int i = lane + 32 * k;
          if (i < m) cand[par][i] = x[k];
        }
      }
      __syncthreads();  // cand complete before the key push below releases it to the cluster
      dbg_stamp(j, 3);
      if (warp == 0 && lane < (int)CS) {
        // push this CTA's key into every CTA's table; st.async completes on the receiver's mbarrier
        // (release at cluster scope: the staged column is visible to whoever acquires that phase)
        const RegKey best = wl >= 0 ? wk[wl] : RegKey{0u, 0u, INT_MAX, -1, 0.0, 0.0};
        const uint32_t dst_key = cluster_map(smem_u32(&keys[par][rank]), (unsigned)lane);
        const uint32_t mb = cluster_map(smem_u32(&kmbar[par]), (unsigned)lane);
        st_async_u64(dst_key, ((unsigned long long)best.lo << 32) | best.hi, mb);
        st_async_u64(dst_key + 8, ((unsigned long long)(unsigned)best.col << 32) | (unsigned)best.pos, mb);
        st_async_u64(dst_key + 16, (unsigned long long)__double_as_longlong(best.tail), mb);
        st_async_u64(dst_key + 24, (unsigned long long)__double_as_longlong(best.xj), mb);
      }
    }
    dbg_stamp(j, 4);
    mbar_wait_cluster(&kmbar[par], (unsigned)(j >> 1) & 1u);
    dbg_stamp(j, 5);
    // ---- F: every warp resolves the cluster winner from the local table ----
    const RegKey r = lane < (int)CS ? keys[par][lane] : RegKey{0u, 0u, INT_MAX, -1, 0.0, 0.0};
    const int wl = warp_argmax(r.hi, r.lo, r.pos, r.col >= 0);
    const unsigned whi = __shfl_sync(0xffffffffu, r.hi, wl);
    const unsigned wlo = __shfl_sync(0xffffffffu, r.lo, wl);
    const int wpos = __shfl_sync(0xffffffffu, r.pos, wl);
    const int wcol = __shfl_sync(0xffffffffu, r.col, wl);
    const double wtail = __shfl_sync(0xffffffffu, r.tail, wl);
    const double wxj = __shfl_sync(0xffffffffu, r.xj, wl);
    const double wkey = __longlong_as_double(((long long)whi << 32) | (long long)wlo);
    // ---- G: pull the winning column while computing the reflector scalars ----
    const bool refl = (m - j >= 2) && (wkey != 0.0);
    double pulled[(32 * RPL + 511) / 512];
#pragma unroll
    for (int t = 0; t < (32 * RPL + 511) / 512; t++) {
      const int i = j + threadIdx.x + 512 * t;
      pulled[t] = (refl && i < m) ? dsmem_f64(&cand[par][i], (unsigned)wl) : 0.0;
    }
    double beta = 0.0, h = 0.0, inv = 0.0;
    if (refl) {
      const double nrm = sqrt(wkey);
      beta = (wxj >= 0.0) ? -nrm : nrm;
      h = beta - wxj;
      inv = 1.0 / sqrt(h * h + wtail);
    }
#pragma unroll
    for (int t = 0; t < (32 * RPL + 511) / 512; t++) {
      const int i = j + threadIdx.x + 512 * t;
      if (refl && i < m) u[i] = (i == j) ? h * inv : -pulled[t] * inv;
    }
    dbg_stamp(j, 6);
    // ---- H: positions (registers), winner column finalised ----
    if (c == wcol) {
      pos = j;
      active = false;
      if (refl) {
#pragma unroll
        for (int k = 0; k < RPL; k++) {
          const int i = lane + 32 * k;
          if (i >= j) x[k] = (i == j) ? beta : 0.0;
        }
      }
    } else if (own && pos == j) {
      pos = wpos;
    }
    if (rank == 0 && threadIdx.x == 0 && p.col_at_pos) p.col_at_pos[j] = wcol;
    __syncthreads();  // u complete
    dbg_stamp(j, 7);
    if (rank == 0 && p.v && refl)
      for (int i = j + threadIdx.x; i < m; i += 512) p.v[(int64_t)j * p.ldv + i] = u[i];
    have_refl = refl;
    rj = j;
  }
  // outputs: pivot columns scattered by final position (or in place)
  if (own) {
    double* dst = p.r_out ? p.r_out + (int64_t)pos * p.ldr : p.a + (int64_t)c * p.lda;
#pragma unroll
    for (int k = 0; k < RPL; k++) {
      const int i = lane + 32 * k;
      if (i < m) dst[i] = x[k];
    }
    if (p.col_at_pos && active && lane == 0) p.col_at_pos[pos] = c;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int RPL>
static int launch_reg(const SweepArgs& a, int CS, cudaStream_t st, int64_t* launches) {
  static bool attr = false;
  if (!attr) {
    RQ_CUDA_TRY(cudaFuncSetAttribute(sweep_reg_kernel<RPL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CS);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  RQ_CUDA_TRY(cudaLaunchKernelEx(&cfg, sweep_reg_kernel<RPL>, a));
  if (launches) (*launches)++;
  return RQ_OK;
}

static size_t cluster_smem(int64_t m, int per) {
  return ((size_t)per * m + 3 * (size_t)m) * sizeof(double) + (32 + SC_WARPS + 2) * sizeof(SweepSlot) +
         (size_t)per * (sizeof(int) + 1) + 64;
}

// ---------------------------------------------------------------------------
// Sketch CPQR (pivot selection only): b steps of the pivoted sweep on the
// (b+p) x n' sketch Y^T, returning the chosen columns (pivoting.py:114-129).
// Columns are retired once chosen, so no R or V is written.
//
// One cooperative launch of G CTAs x 1024 threads; each CTA keeps its column
// slice in shared memory; a column is processed by an 8-lane group (4 per
// warp).  Per step there is no separate grid barrier: every CTA publishes
// (key, tail, position, column) + its candidate column with a release store of
// a launch-unique stamp, and warp 0 of every CTA polls the G stamps with
// acquire loads (all-gather), then fetches the winning column from L2.
// ---------------------------------------------------------------------------
constexpr int SK_THREADS = 1024;
constexpr int SK_WARPS = SK_THREADS / 32;
constexpr int SK_GROUP = 8;
constexpr int SK_GROUPS = SK_THREADS / SK_GROUP;
constexpr int kSkMaxSpw = 24;  // register sketch CPQR: non-register columns per warp (n' <= 148 * 360)

struct alignas(16) SkSlot {
  double key;
  double tail;
  int pos;
  int col;
  unsigned long long stamp;
};

struct SketchArgs {
  const double* y;  // m x n (col-major, ld); destroyed
  double* ywork;    // same storage (writable)
  int64_t ld;
  int m;
  int n;
  int steps;
  const int* init_pos;
  int* chosen;
  SkSlot* slots;      // 2 x G
  double* slotdata;   // 2 x G x m
  unsigned long long* counter;      // monotone arrival counter (never reset)
  unsigned long long counter_base;  // its value when this launch starts
  int cache_cols;
  int spw;  // register kernel: shared-memory-resident columns per warp (0 = registers only)
  int spw_g;       // register kernel: of those, the last spw_g per warp live in gcols (L2-resident)
  double* gcols;   // [CTA][warp][spw_g][slot k][lane]
  int fixed_reducer;  // register kernel: CTA 0 always reduces the slots (no arrival atomic)
  int cl;             // register kernel: cluster size (> 1: two-level exchange, see SkClu)
  int per;            // register kernel: columns per CTA (column id -> CTA)
};

RQ_DEV unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
RQ_DEV void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// (key, pos) better than (k2, p2)?  Invalid candidates carry key < 0.
RQ_DEV void sk_take_better(double& key, double& tail, int& pos, int& col, int& who, double k2, double t2, int p2,
                           int c2, int w2) {
  if (c2 >= 0 && (col < 0 || piv_better(k2, p2, key, pos))) {
    key = k2;
    tail = t2;
    pos = p2;
    col = c2;
    who = w2;
  }
}

__global__ void __launch_bounds__(SK_THREADS, 1) sketch_cpqr_kernel(const SketchArgs p) {
  extern __shared__ double sm[];
  const int G = gridDim.x;
  const int per = (p.n + G - 1) / G;
  const int c0 = blockIdx.x * per;
  const int c1 = min(p.n, c0 + per);
  const int ncols = max(0, c1 - c0);
  const int m = p.m;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = threadIdx.x / SK_GROUP, gl = threadIdx.x % SK_GROUP;

  double* u = sm;                                       // m
  double* cache = u + m;                                // cache_cols x m
  const int ncache = min(ncols, p.cache_cols);
  int* pos = reinterpret_cast<int*>(cache + (int64_t)p.cache_cols * m);
  int* active = pos + per;
  SweepSlot* red = reinterpret_cast<SweepSlot*>(active + per + 2);
  int* wbuf = reinterpret_cast<int*>(red + SK_WARPS + 2);

  auto colptr = [&](int lc) -> double* {
    return lc < ncache ? cache + (int64_t)lc * m : p.ywork + (int64_t)(c0 + lc) * p.ld;
  };
  for (int lc = warp; lc < ncache; lc += SK_WARPS)
    for (int i = lane; i < m; i += 32) cache[(int64_t)lc * m + i] = p.y[(int64_t)(c0 + lc) * p.ld + i];
  for (int lc = threadIdx.x; lc < ncols; lc += SK_THREADS) {
    pos[lc] = p.init_pos ? p.init_pos[c0 + lc] : c0 + lc;
    active[lc] = 1;
  }
  __syncthreads();

  bool have_refl = false;
  int rj = -1;
  const int rounds = (ncols + SK_GROUPS - 1) / SK_GROUPS;
  for (int j = 0; j < p.steps; j++) {
    const int par = j & 1;
    dbg_stamp(j, 0);
    // -------- phase A: apply the pending reflector, score the candidates --------
    double bk = -1.0, bt = 0.0;
    int bp = INT_MAX, bc = -1, bw = 0;
    for (int r = 0; r < rounds; r++) {
      const int lc = r * SK_GROUPS + grp;
      const bool live = lc < ncols && active[lc];
      double* col = live ? colptr(lc) : u;  // dummy pointer for idle groups
      double d = 0.0;
      if (have_refl && live) {
        double d0 = 0.0, d1 = 0.0;
        int i = rj + gl;
        for (; i + SK_GROUP < m; i += 2 * SK_GROUP) {
          d0 += u[i] * col[i];
          d1 += u[i + SK_GROUP] * col[i + SK_GROUP];
        }
        if (i < m) d0 += u[i] * col[i];
        d = d0 + d1;
      }
      d += __shfl_xor_sync(0xffffffffu, d, 4);
      d += __shfl_xor_sync(0xffffffffu, d, 2);
      d += __shfl_xor_sync(0xffffffffu, d, 1);
      d *= 2.0;
      double t = 0.0;
      if (live) {
        if (have_refl) {
          for (int i = rj + gl; i < m; i += SK_GROUP) {
            const double v = col[i] - d * u[i];
            col[i] = v;
            if (i > j) t += v * v;
          }
        } else {
          for (int i = j + 1 + gl; i < m; i += SK_GROUP) t += col[i] * col[i];
        }
      }
      t += __shfl_xor_sync(0xffffffffu, t, 4);
      t += __shfl_xor_sync(0xffffffffu, t, 2);
      t += __shfl_xor_sync(0xffffffffu, t, 1);
      if (live) {
        const double xj = col[j];
        const double key = xj * xj + t;
        sk_take_better(bk, bt, bp, bc, bw, key, t, pos[lc], c0 + lc, 0);
      }
    }
    // group leaders (lanes 0, 8, 16, 24) -> warp best
#pragma unroll
    for (int o = 8; o < 32; o <<= 1) {
      const double k2 = __shfl_xor_sync(0xffffffffu, bk, o);
      const double t2 = __shfl_xor_sync(0xffffffffu, bt, o);
      const int p2 = __shfl_xor_sync(0xffffffffu, bp, o);
      const int c2 = __shfl_xor_sync(0xffffffffu, bc, o);
      sk_take_better(bk, bt, bp, bc, bw, k2, t2, p2, c2, 0);
    }
    dbg_stamp(j, 1);
    if (lane == 0) red[warp] = SweepSlot{bk, bt, bp, bc};
    __syncthreads();
    dbg_stamp(j, 2);
    if (warp == 0) {
      SweepSlot b = red[lane];  // SK_WARPS == 32
      int who = 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double k2 = __shfl_xor_sync(0xffffffffu, b.key, o);
        const double t2 = __shfl_xor_sync(0xffffffffu, b.tail, o);
        const int p2 = __shfl_xor_sync(0xffffffffu, b.pos, o);
        const int c2 = __shfl_xor_sync(0xffffffffu, b.col, o);
        sk_take_better(b.key, b.tail, b.pos, b.col, who, k2, t2, p2, c2, 0);
      }
      if (lane == 0) red[SK_WARPS] = b;
    }
    __syncthreads();
    // -------- publish the CTA candidate (column first, then the stamped slot) --------
    const SweepSlot mine = red[SK_WARPS];
    double* sd = p.slotdata + ((int64_t)par * G + blockIdx.x) * m;
    if (mine.col >= 0) {
      const double* src = colptr(mine.col - c0);
      for (int i = j + threadIdx.x; i < m; i += SK_THREADS) sd[i] = src[i];
    }
    SkSlot* slot = p.slots + (int64_t)par * G;
    if (threadIdx.x == 0) {
      SkSlot* me = slot + blockIdx.x;
      me->key = mine.col >= 0 ? mine.key : -1.0;
      me->tail = mine.tail;
      me->pos = mine.pos;
      me->col = mine.col;
    }
    // -------- grid barrier: one arrival + one poller per CTA (monotone counter) --------
    __syncthreads();
    dbg_stamp(j, 3);
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(p.counter, 1ull);
      const unsigned long long target = p.counter_base + (unsigned long long)(j + 1) * G;
      while (ld_acquire_u64(p.counter) < target) {
      }
    }
    __syncthreads();
    // -------- every CTA reads the G candidates (one batch of loads) and picks the winner --------
    dbg_stamp(j, 4);
    if (warp == 0) {
      double k = -1.0, t = 0.0;
      int ps = INT_MAX, cl = -1, who = -1;
      constexpr int kMaxK = (kSMs + 31) / 32;
      double kk_key[kMaxK], kk_tail[kMaxK];
      int kk_pos[kMaxK], kk_col[kMaxK];
#pragma unroll
      for (int kk = 0; kk < kMaxK; kk++) {
        const int c = kk * 32 + lane;
        if (c < G) {
          kk_key[kk] = __ldcg(&slot[c].key);
          kk_tail[kk] = __ldcg(&slot[c].tail);
          kk_pos[kk] = __ldcg(&slot[c].pos);
          kk_col[kk] = __ldcg(&slot[c].col);
        } else {
          kk_key[kk] = -1.0;
          kk_col[kk] = -1;
        }
      }
#pragma unroll
      for (int kk = 0; kk < kMaxK; kk++)
        if (kk_key[kk] >= 0.0) sk_take_better(k, t, ps, cl, who, kk_key[kk], kk_tail[kk], kk_pos[kk], kk_col[kk],
                                              kk * 32 + lane);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double k2 = __shfl_xor_sync(0xffffffffu, k, o);
        const double t2 = __shfl_xor_sync(0xffffffffu, t, o);
        const int p2 = __shfl_xor_sync(0xffffffffu, ps, o);
        const int c2 = __shfl_xor_sync(0xffffffffu, cl, o);
        const int w2 = __shfl_xor_sync(0xffffffffu, who, o);
        sk_take_better(k, t, ps, cl, who, k2, t2, p2, c2, w2);
      }
      if (lane == 0) {
        red[SK_WARPS + 1] = SweepSlot{k, t, ps, cl};
        wbuf[0] = who;
      }
    }
    __syncthreads();
    dbg_stamp(j, 5);
    const SweepSlot win = red[SK_WARPS + 1];
    const int wcta = wbuf[0];
    const double* x = p.slotdata + ((int64_t)par * G + wcta) * m;
    const bool refl = (m - j >= 2) && (win.key != 0.0);
    if (refl) {
      const double xj = __ldcg(&x[j]);
      const double nrm = sqrt(win.key);
      const double beta = (xj >= 0.0) ? -nrm : nrm;
      const double h = beta - xj;
      const double inv = 1.0 / sqrt(h * h + win.tail);
      for (int i = j + threadIdx.x; i < m; i += SK_THREADS) u[i] = (i == j) ? h * inv : -__ldcg(&x[i]) * inv;
    }
    for (int lc = threadIdx.x; lc < ncols; lc += SK_THREADS) {
      if (c0 + lc == win.col) {
        pos[lc] = j;
        active[lc] = 0;
      } else if (pos[lc] == j) {
        pos[lc] = win.pos;
      }
    }
    dbg_stamp(j, 6);
    if (blockIdx.x == 0 && threadIdx.x == 0) p.chosen[j] = win.col;
    have_refl = refl;
    rj = j;
    __syncthreads();
    dbg_stamp(j, 7);
  }
}

// ---------------------------------------------------------------------------
// Register-resident sketch CPQR (n' <= G * 16 * CPW columns, m <= 32 * RPL rows).
// 512 threads; warp w of CTA g owns columns g*16*CPW + w*CPW + q (q < CPW),
// lane l holds rows l, l+32, ... of each in registers.
// ---------------------------------------------------------------------------
struct alignas(16) SkSlot2 {
  double key;
  double tail;
  double xj;
  int pos;
  int col;
};

// Winner record published by the last CTA to arrive in each step.
struct alignas(16) SkWin {
  double key;
  double tail;
  double xj;
  int pos;
  int col;
  int cta;
  int pad;
  unsigned long long flag;  // launch-unique step stamp, written last (release)
};

// Per-step state shared by the step templates below.
struct SkKey {
  unsigned hi, lo;  // bits of the non-negative key (monotone as integers)
  int pos;
  int col;          // global column id, -1 = none
};

struct SkShared {
  SkKey wk[16];
  SkKey win;
  double wtail, wxj;
  int wsel[2];
  unsigned long long wbits[16][2];  // last arriver: tail / x_j bits of each warp's best slot
  int wcta[16];
};

// Apply the pending reflector u (rows >= 32*K0 may be non-zero; u is exactly 0
// above the reflector row and below m) to every column the warp owns.
template <int K0, int RPL, int CPW>
RQ_DEV void sk_apply(double (&x)[CPW][RPL], const bool (&act)[CPW], const double* u, int lane) {
  double uk[RPL];
#pragma unroll
  for (int k = K0; k < RPL; k++) uk[k] = u[lane + 32 * k];
  double d[CPW];
#pragma unroll
  for (int q = 0; q < CPW; q++) {
    double acc = 0.0;
#pragma unroll
    for (int k = K0; k < RPL; k++) acc = fma(uk[k], x[q][k], acc);
    d[q] = acc;
  }
  warp_sum_all<CPW, 0, CPW>(d, lane);
#pragma unroll
  for (int q = 0; q < CPW; q++) {
    const double dd = act[q] ? 2.0 * d[q] : 0.0;
#pragma unroll
    for (int k = K0; k < RPL; k++) x[q][k] -= dd * uk[k];
  }
}

// One shared-memory-resident column (same arithmetic as sk_apply).
template <int K0, int RPL>
RQ_DEV void sk_apply1(double (&y)[RPL], const double* u, int lane) {
  double d = 0.0;
#pragma unroll
  for (int k = K0; k < RPL; k++) d = fma(u[lane + 32 * k], y[k], d);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
  d *= 2.0;
#pragma unroll
  for (int k = K0; k < RPL; k++) y[k] -= d * u[lane + 32 * k];
}

// Two shared-memory columns at once (same arithmetic per column as sk_apply1): their
// reductions interleave, halving the latency-bound chain of the shared-memory tier.
template <int K0, int RPL>
RQ_DEV void sk_apply2(double (&y0)[RPL], double (&y1)[RPL], const double* u, int lane) {
  double dd[2] = {0.0, 0.0};
#pragma unroll
  for (int k = K0; k < RPL; k++) {
    const double uk = u[lane + 32 * k];
    dd[0] = fma(uk, y0[k], dd[0]);
    dd[1] = fma(uk, y1[k], dd[1]);
  }
  warp_sum_all<2, 0, 2>(dd, lane);
  const double d0 = 2.0 * dd[0], d1 = 2.0 * dd[1];
#pragma unroll
  for (int k = K0; k < RPL; k++) {
    const double uk = u[lane + 32 * k];
    y0[k] -= d0 * uk;
    y1[k] -= d1 * uk;
  }
}

// Columns beyond the register capacity live in shared memory, [column][slot k][lane].
// Two-level exchange (cluster launch, p.cl = CS > 1): each CTA pushes its candidate record
// (6 words: key, pos|col, tail, x_j, CTA, pad) into its cluster leader's table through
// st.async; the leader (cluster rank 0) reduces its CS records, publishes the cluster's best as
// an LL slot, polls the slots of all G/CS leaders (one L2 round trip, no arrival atomic), and
// pushes the winner record back to the members of its cluster.  Every leader computes the same
// winner from the same slots.
struct SkClu {
  unsigned long long keys[2][16][6];  // leader: member records, by step parity
  unsigned long long win[2][6];       // every CTA: winner record from its leader
  unsigned long long kbar[2];         // leader: member records of step j complete on kbar[j & 1]
  unsigned long long wbar[2];         // winner record of step j complete on wbar[j & 1]
};

struct SkSmem {
  double* xs;
  int* spos;
  int* sact;
  int spw;      // columns per warp beyond the registers (shared memory, then global)
  int cbase_s;  // global id of this warp's first shared-memory column
  SkClu* cl;    // two-level exchange state (p.cl > 1)
  int spw_s;    // of spw: in shared memory ([warp][spw_s][slot k][lane])
  double* xg;   // this warp's spw - spw_s global-memory columns ([s][slot k][lane])
};

// Column s (0 <= s < spw) of a warp's non-register tier, lane 0's slot 0.
template <int RPL>
RQ_DEV double* sk_tier_col(const SkSmem& sm, int warp, int s) {
  return s < sm.spw_s ? sm.xs + (int64_t)(warp * sm.spw_s + s) * RPL * 32 : sm.xg + (int64_t)(s - sm.spw_s) * RPL * 32;
}

// Steps j in [32*KJ, jend): row j lives in register slot KJ (lane j & 31), so
// every row mask below is a compile-time slot range plus one lane predicate.
template <int KJ, int RPL, int CPW, int WARPS, bool SMEM>
RQ_DEV void sk_block(const SketchArgs& p, SkSlot2* slots, SkWin* wins, unsigned long long stamp_base,
                     double (&x)[CPW][RPL], int (&pos)[CPW], bool (&act)[CPW], bool& have_refl, double* u,
                     SkShared& sh, int cbase, int jend, const SkSmem& sm) {
  constexpr int KL = KJ > 0 ? KJ - 1 : 0;  // lowest slot the pending reflector can touch
  constexpr int NT = WARPS * 32;
  const int G = gridDim.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = p.m;
  const int CS = p.cl;
  unsigned crank = 0, cid = 0;
  if (CS > 1) {
    asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    asm("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
  }
  for (int j = 32 * KJ; j < jend; j++) {
    const int par = j & 1;
    const int jl = j & 31;
    dbg_stamp(j, 0);
    if (CS > 1 && threadIdx.x == 0) {
      mbar_expect_tx(&sm.cl->wbar[par], 6 * 8);
      if (crank == 0) mbar_expect_tx(&sm.cl->kbar[par], (unsigned)CS * 6 * 8);
    }
    // -------- A: apply the pending reflector (row j-1), score rows >= j --------
    if (have_refl) {
      if (KJ > 0 && jl == 0) sk_apply<(KJ > 0 ? KJ - 1 : 0), RPL, CPW>(x, act, u, lane);
      else sk_apply<KJ, RPL, CPW>(x, act, u, lane);
    }
    double t[CPW];
    const bool at_or_below = lane >= jl;
#pragma unroll
    for (int q = 0; q < CPW; q++) {
      const double xv = at_or_below ? x[q][KJ] : 0.0;
      double acc = xv * xv;
#pragma unroll
      for (int k = KJ + 1; k < RPL; k++) acc = fma(x[q][k], x[q][k], acc);
      t[q] = acc;
    }
    warp_sum_all<CPW, 0, CPW>(t, lane);
    double bkey = -1.0;
    int bpos = INT_MAX, bq = -1;
#pragma unroll
    for (int q = 0; q < CPW; q++) {
      if (act[q] && (bq < 0 || piv_better(t[q], pos[q], bkey, bpos))) {
        bkey = t[q];
        bpos = pos[q];
        bq = q;
      }
    }
    int bcol = bq >= 0 ? cbase + bq : -1;
    if constexpr (SMEM) {
      // pairs of shared-memory columns, then pairs of global-memory columns (an odd last one of
      // each range is paired with itself, result unused); the same body for both address spaces
      auto pair_step = [&](double* col0, double* col1, int s2, bool has1) {
        const int sc0 = warp * sm.spw + s2;
        const int sc1 = has1 ? sc0 + 1 : sc0;
        const bool a0 = sm.sact[sc0] != 0, a1 = has1 && sm.sact[sc1] != 0;  // warp-uniform
        if (!a0 && !a1) return;
        double y0[RPL], y1[RPL];
#pragma unroll
        for (int k = KL; k < RPL; k++) {
          y0[k] = col0[k * 32];
          y1[k] = col1[k * 32];
        }
        if (have_refl) {
          if (KJ > 0 && jl == 0) sk_apply2<KL, RPL>(y0, y1, u, lane);
          else sk_apply2<KJ, RPL>(y0, y1, u, lane);
        }
        const double yv0 = at_or_below ? y0[KJ] : 0.0, yv1 = at_or_below ? y1[KJ] : 0.0;
        double tt[2] = {yv0 * yv0, yv1 * yv1};
#pragma unroll
        for (int k = KJ + 1; k < RPL; k++) {
          tt[0] = fma(y0[k], y0[k], tt[0]);
          tt[1] = fma(y1[k], y1[k], tt[1]);
        }
        warp_sum_all<2, 0, 2>(tt, lane);
        const double t0 = tt[0], t1 = tt[1];
        if (a0) {
#pragma unroll
          for (int k = KL; k < RPL; k++) col0[k * 32] = y0[k];
          const int ps = sm.spos[sc0];
          if (bcol < 0 || piv_better(t0, ps, bkey, bpos)) {
            bkey = t0;
            bpos = ps;
            bcol = sm.cbase_s + s2;
          }
        }
        if (a1) {
#pragma unroll
          for (int k = KL; k < RPL; k++) col1[k * 32] = y1[k];
          const int ps = sm.spos[sc1];
          if (bcol < 0 || piv_better(t1, ps, bkey, bpos)) {
            bkey = t1;
            bpos = ps;
            bcol = sm.cbase_s + s2 + 1;
          }
        }
      };
      for (int s2 = 0; s2 < sm.spw_s; s2 += 2) {
        const bool has1 = s2 + 1 < sm.spw_s;
        double* col0 = sm.xs + (int64_t)(warp * sm.spw_s + s2) * RPL * 32 + lane;
        pair_step(col0, has1 ? col0 + RPL * 32 : col0, s2, has1);
      }
      for (int s2 = sm.spw_s; s2 < sm.spw; s2 += 2) {
        const bool has1 = s2 + 1 < sm.spw;
        double* col0 = sm.xg + (int64_t)(s2 - sm.spw_s) * RPL * 32 + lane;
        pair_step(col0, has1 ? col0 + RPL * 32 : col0, s2, has1);
      }
    }
    if (lane == 0) {
      const unsigned long long kb = __double_as_longlong(bkey < 0.0 ? 0.0 : bkey);
      sh.wk[warp] = SkKey{(unsigned)(kb >> 32), (unsigned)kb, bpos, bcol};
    }
    dbg_stamp(j, 1);
    __syncthreads();
    dbg_stamp(j, 2);
    // -------- B: the CTA's best warp publishes its key, x_j, tail and column (LL words) --------
    // Every 8-byte word carries the step stamp in its low half: a reader that sees the stamp
    // in every word it needs has current data, so no fences sit on the exchange path.
    const unsigned stamp = (unsigned)(stamp_base + (unsigned long long)j + 1ull);
    unsigned long long* slw = reinterpret_cast<unsigned long long*>(slots) + ((int64_t)par * G) * 8;
    unsigned long long* colw = reinterpret_cast<unsigned long long*>(p.slotdata);
    const int64_t cstride = 2 * (int64_t)(m + 2);
    {
      const SkKey r = lane < WARPS ? sh.wk[lane] : SkKey{0u, 0u, INT_MAX, -1};
      const int wl = warp_argmax(r.hi, r.lo, r.pos, r.col >= 0);  // warp-uniform, same in every warp
      if (wl < 0) {
        if (warp == 0 && lane == 0) {
          if (CS > 1) {
            const uint32_t dst = cluster_map(smem_u32(&sm.cl->keys[par][crank][0]), 0u);
            const uint32_t mb = cluster_map(smem_u32(&sm.cl->kbar[par]), 0u);
            st_async_u64(dst, 0ull, mb);
            st_async_u64(dst + 8, ((unsigned long long)0xffffffffu << 32) | (unsigned)INT_MAX, mb);
            st_async_u64(dst + 16, 0ull, mb);
            st_async_u64(dst + 24, 0ull, mb);
            st_async_u64(dst + 32, 0ull, mb);
            st_async_u64(dst + 40, 0ull, mb);
          } else {
            unsigned long long* me = slw + (int64_t)blockIdx.x * 8;
            st_ll2(me, ll_word(0u, stamp), ll_word(0u, stamp));
            st_ll2(me + 2, ll_word((unsigned)INT_MAX, stamp), ll_word(0xffffffffu, stamp));
            st_ll2(me + 4, ll_word(0u, stamp), ll_word(0u, stamp));
            st_ll2(me + 6, ll_word(0u, stamp), ll_word(0u, stamp));
          }
        }
      } else if (wl == warp) {
        const SkKey b = sh.wk[warp];
        unsigned long long* cb = colw + ((int64_t)par * G + blockIdx.x) * cstride;
        auto publish = [&](const double (&xc)[RPL]) {
          const double xj = __shfl_sync(0xffffffffu, xc[KJ], jl);
          const double xv = lane > jl ? xc[KJ] : 0.0;
          double tl = xv * xv;
#pragma unroll
          for (int k = KJ + 1; k < RPL; k++) tl = fma(xc[k], xc[k], tl);
#pragma unroll
          for (int k = KJ; k < RPL; k++) {
            const int i = lane + 32 * k;
            if (i >= j && i < m) {
              const unsigned long long bits = __double_as_longlong(xc[k]);
              st_ll2(cb + 2 * i, ll_word((unsigned)(bits >> 32), stamp), ll_word((unsigned)bits, stamp));
            }
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) tl += __shfl_xor_sync(0xffffffffu, tl, o);
          if (lane == 0) {
            const unsigned long long tb = __double_as_longlong(tl), xb = __double_as_longlong(xj);
            if (CS > 1) {
              // (the column's LL words above are read only once the winner is known)
              const uint32_t dst = cluster_map(smem_u32(&sm.cl->keys[par][crank][0]), 0u);
              const uint32_t mb = cluster_map(smem_u32(&sm.cl->kbar[par]), 0u);
              st_async_u64(dst, ((unsigned long long)b.hi << 32) | b.lo, mb);
              st_async_u64(dst + 8, ((unsigned long long)(unsigned)b.col << 32) | (unsigned)b.pos, mb);
              st_async_u64(dst + 16, tb, mb);
              st_async_u64(dst + 24, xb, mb);
              st_async_u64(dst + 32, (unsigned long long)blockIdx.x, mb);
              st_async_u64(dst + 40, 0ull, mb);
            } else {
              unsigned long long* me = slw + (int64_t)blockIdx.x * 8;
              st_ll2(me, ll_word(b.hi, stamp), ll_word(b.lo, stamp));
              st_ll2(me + 2, ll_word((unsigned)b.pos, stamp), ll_word((unsigned)b.col, stamp));
              st_ll2(me + 4, ll_word((unsigned)(tb >> 32), stamp), ll_word((unsigned)tb, stamp));
              st_ll2(me + 6, ll_word((unsigned)(xb >> 32), stamp), ll_word((unsigned)xb, stamp));
            }
          }
        };
        bool done = false;
        if constexpr (SMEM) {
          if (b.col >= sm.cbase_s && b.col < sm.cbase_s + sm.spw) {
            const double* col = sk_tier_col<RPL>(sm, warp, b.col - sm.cbase_s) + lane;
            double y[RPL];
#pragma unroll
            for (int k = 0; k < RPL; k++) y[k] = k >= KJ ? col[k * 32] : 0.0;
            publish(y);
            done = true;
          }
        }
        if (!done) {
          const int bqw = b.col - cbase;
#pragma unroll
          for (int q = 0; q < CPW; q++)
            if (q == bqw) publish(x[q]);
        }
      }
    }
    __syncthreads();
    dbg_stamp(j, 3);
    // -------- C: arrive (relaxed); the last CTA reduces every slot and publishes the winner --------
    unsigned long long* wrw = reinterpret_cast<unsigned long long*>(wins) + par * 10;
    if (CS > 1) {
      const int L = G / CS;  // leaders (G is a multiple of CS)
      if (crank == 0) {
        // (1) the cluster's best of its CS member records -> LL slot `cid` (same 8-word format as
        //     the single-level slots; the winning CTA follows from the column id: col / p.per)
        if (warp == 0) {
          mbar_wait_cluster(&sm.cl->kbar[par], (unsigned)(j >> 1) & 1u);
          unsigned khi = 0u, klo = 0u;
          int kpos = INT_MAX, kcol = -1;
          unsigned long long ktb = 0ull, kxb = 0ull;
          if (lane < CS) {
            const unsigned long long* r = sm.cl->keys[par][lane];
            khi = (unsigned)(r[0] >> 32);
            klo = (unsigned)r[0];
            kpos = (int)(unsigned)r[1];
            kcol = (int)(unsigned)(r[1] >> 32);
            ktb = r[2];
            kxb = r[3];
          }
          const int bl = warp_argmax(khi, klo, kpos, kcol >= 0);
          if (lane == (bl < 0 ? 0 : bl)) {
            unsigned long long* me = slw + (int64_t)cid * 8;
            const int cc = bl < 0 ? -1 : kcol;
            st_ll2(me, ll_word(bl < 0 ? 0u : khi, stamp), ll_word(bl < 0 ? 0u : klo, stamp));
            st_ll2(me + 2, ll_word((unsigned)(bl < 0 ? INT_MAX : kpos), stamp), ll_word((unsigned)cc, stamp));
            st_ll2(me + 4, ll_word((unsigned)(ktb >> 32), stamp), ll_word((unsigned)ktb, stamp));
            st_ll2(me + 6, ll_word((unsigned)(kxb >> 32), stamp), ll_word((unsigned)kxb, stamp));
          }
        }
        // (2) every leader reads all L slots (one per thread) and resolves the same winner
        unsigned khi = 0u, klo = 0u;
        int kpos = INT_MAX, kcol = -1;
        unsigned long long ktb = 0ull, kxb = 0ull;
        if ((int)threadIdx.x < L) {
          const unsigned long long* sp = slw + (int64_t)threadIdx.x * 8;
          unsigned long long a0, a1, a2, a3, a4, a5, a6, a7;
          do {
            ld_ll2(sp, a0, a1);
            ld_ll2(sp + 2, a2, a3);
            ld_ll2(sp + 4, a4, a5);
            ld_ll2(sp + 6, a6, a7);
          } while ((unsigned)a0 != stamp || (unsigned)a1 != stamp || (unsigned)a2 != stamp || (unsigned)a3 != stamp ||
                   (unsigned)a4 != stamp || (unsigned)a5 != stamp || (unsigned)a6 != stamp || (unsigned)a7 != stamp);
          khi = (unsigned)(a0 >> 32);
          klo = (unsigned)(a1 >> 32);
          kpos = (int)(a2 >> 32);
          kcol = (int)(a3 >> 32);
          ktb = (a4 & 0xffffffff00000000ull) | (a5 >> 32);
          kxb = (a6 & 0xffffffff00000000ull) | (a7 >> 32);
        }
        if (warp * 32 < L) {
          const int wl = warp_argmax(khi, klo, kpos, kcol >= 0);
          if (lane == (wl < 0 ? 0 : wl)) {
            sh.wk[warp] = SkKey{khi, klo, kpos, wl < 0 ? -1 : kcol};
            sh.wbits[warp][0] = ktb;
            sh.wbits[warp][1] = kxb;
          }
        }
        __syncthreads();
        // (3) push the winner record to every member of this cluster
        if (warp == 0) {
          const int nw = (L + 31) / 32;
          const SkKey r = lane < nw ? sh.wk[lane] : SkKey{0u, 0u, INT_MAX, -1};
          const int gl = warp_argmax(r.hi, r.lo, r.pos, r.col >= 0);
          const int src = gl < 0 ? 0 : gl;
          const unsigned whi = __shfl_sync(0xffffffffu, r.hi, src), wlo = __shfl_sync(0xffffffffu, r.lo, src);
          const int wps = __shfl_sync(0xffffffffu, r.pos, src), wcl = __shfl_sync(0xffffffffu, r.col, src);
          if (lane < CS) {
            const unsigned long long tb = sh.wbits[src][0], xb = sh.wbits[src][1];
            const int col = gl < 0 ? -1 : wcl;
            const int cta = col >= 0 ? col / p.per : 0;
            const uint32_t dst = cluster_map(smem_u32(&sm.cl->win[par][0]), (unsigned)lane);
            const uint32_t mb = cluster_map(smem_u32(&sm.cl->wbar[par]), (unsigned)lane);
            st_async_u64(dst, ((unsigned long long)whi << 32) | wlo, mb);
            st_async_u64(dst + 8, ((unsigned long long)(unsigned)col << 32) | (unsigned)wps, mb);
            st_async_u64(dst + 16, tb, mb);
            st_async_u64(dst + 24, xb, mb);
            st_async_u64(dst + 32, (unsigned long long)cta, mb);
            st_async_u64(dst + 40, 0ull, mb);
          }
        }
      }
      if (warp == 0) {
        mbar_wait_cluster(&sm.cl->wbar[par], (unsigned)(j >> 1) & 1u);
        if (lane == 0) {
          const unsigned long long* r = sm.cl->win[par];
          sh.win = SkKey{(unsigned)(r[0] >> 32), (unsigned)r[0], (int)(unsigned)r[1], (int)(unsigned)(r[1] >> 32)};
          sh.wtail = __longlong_as_double((long long)r[2]);
          sh.wxj = __longlong_as_double((long long)r[3]);
          sh.wsel[1] = (int)r[4];
        }
      }
    } else {
    bool reducer;
    if (p.fixed_reducer) {
      // a fixed CTA polls every slot's stamps directly: one L2 round trip fewer than
      // arrive-then-read (1: CTA 0; 2: the last CTA, which holds the fewest columns)
      reducer = blockIdx.x == (p.fixed_reducer == 2 ? gridDim.x - 1 : 0);
    } else {
      if (threadIdx.x == 0) {
        unsigned long long old;
        asm volatile("atom.relaxed.gpu.global.add.u64 %0, [%1], 1;" : "=l"(old) : "l"(p.counter) : "memory");
        sh.wsel[0] = (old + 1 == p.counter_base + (unsigned long long)(j + 1) * G) ? 1 : 0;
      }
      __syncthreads();
      reducer = sh.wsel[0] != 0;
    }
    if (reducer) {
      // one slot per thread (G <= NT): spin until its four words carry this step's stamp
      unsigned khi = 0u, klo = 0u;
      int kpos = INT_MAX, kcol = -1;
      unsigned long long ktb = 0ull, kxb = 0ull;
      if ((int)threadIdx.x < G) {
        const unsigned long long* sp = slw + (int64_t)threadIdx.x * 8;
        unsigned long long a0, a1, a2, a3, a4, a5, a6, a7;
        do {
          ld_ll2(sp, a0, a1);
          ld_ll2(sp + 2, a2, a3);
          ld_ll2(sp + 4, a4, a5);
          ld_ll2(sp + 6, a6, a7);
        } while ((unsigned)a0 != stamp || (unsigned)a1 != stamp || (unsigned)a2 != stamp || (unsigned)a3 != stamp ||
                 (unsigned)a4 != stamp || (unsigned)a5 != stamp || (unsigned)a6 != stamp || (unsigned)a7 != stamp);
        khi = (unsigned)(a0 >> 32);
        klo = (unsigned)(a1 >> 32);
        kpos = (int)(a2 >> 32);
        kcol = (int)(a3 >> 32);
        ktb = (a4 & 0xffffffff00000000ull) | (a5 >> 32);
        kxb = (a6 & 0xffffffff00000000ull) | (a7 >> 32);
      }
      const int wl = warp_argmax(khi, klo, kpos, kcol >= 0);
      if (lane == (wl < 0 ? 0 : wl)) {
        sh.wk[warp] = SkKey{khi, klo, kpos, wl < 0 ? -1 : kcol};
        sh.wbits[warp][0] = ktb;
        sh.wbits[warp][1] = kxb;
        sh.wcta[warp] = (int)threadIdx.x;
      }
      __syncthreads();
      if (warp == 0) {
        const SkKey r = lane < WARPS ? sh.wk[lane] : SkKey{0u, 0u, INT_MAX, -1};
        const int gl = warp_argmax(r.hi, r.lo, r.pos, r.col >= 0);
        if (lane == gl) {
          const unsigned long long tb = sh.wbits[gl][0], xb = sh.wbits[gl][1];
          const int cta = sh.wcta[gl];
          st_ll2(wrw, ll_word(r.hi, stamp), ll_word(r.lo, stamp));
          st_ll2(wrw + 2, ll_word((unsigned)r.pos, stamp), ll_word((unsigned)r.col, stamp));
          st_ll2(wrw + 4, ll_word((unsigned)cta, stamp), ll_word(0u, stamp));
          st_ll2(wrw + 6, ll_word((unsigned)(tb >> 32), stamp), ll_word((unsigned)tb, stamp));
          st_ll2(wrw + 8, ll_word((unsigned)(xb >> 32), stamp), ll_word((unsigned)xb, stamp));
          sh.win = r;
          sh.wtail = __longlong_as_double((long long)tb);
          sh.wxj = __longlong_as_double((long long)xb);
          sh.wsel[1] = cta;
        }
      }
    } else if (warp == 0) {
      // lanes 0..4 poll one word pair each of the winner record
      unsigned long long a = 0ull, b = 0ull;
      bool ok = lane >= 5;
      do {
        if (!ok) {
          ld_ll2(wrw + 2 * lane, a, b);
          ok = (unsigned)a == stamp && (unsigned)b == stamp;
        }
      } while (!__all_sync(0xffffffffu, ok));
      const unsigned h0 = (unsigned)(__shfl_sync(0xffffffffu, a, 0) >> 32);
      const unsigned l0 = (unsigned)(__shfl_sync(0xffffffffu, b, 0) >> 32);
      const int ps = (int)(__shfl_sync(0xffffffffu, a, 1) >> 32);
      const int cl = (int)(__shfl_sync(0xffffffffu, b, 1) >> 32);
      const int ct = (int)(__shfl_sync(0xffffffffu, a, 2) >> 32);
      const unsigned long long t3a = __shfl_sync(0xffffffffu, a, 3), t3b = __shfl_sync(0xffffffffu, b, 3);
      const unsigned long long t4a = __shfl_sync(0xffffffffu, a, 4), t4b = __shfl_sync(0xffffffffu, b, 4);
      if (lane == 0) {
        sh.win = SkKey{h0, l0, ps, cl};
        sh.wsel[1] = ct;
        sh.wtail = __longlong_as_double((long long)((t3a & 0xffffffff00000000ull) | (t3b >> 32)));
        sh.wxj = __longlong_as_double((long long)((t4a & 0xffffffff00000000ull) | (t4b >> 32)));
      }
    }
    }  // single-level exchange
    __syncthreads();
    dbg_stamp(j, 4);
    // -------- E: reflector from the winning column (LL words in L2); u = 0 outside [j, m) --------
    const SkKey win = sh.win;
    const int wcta = sh.wsel[1];
    const double wkey = __longlong_as_double(((long long)win.hi << 32) | (long long)win.lo);
    const bool refl = (m - j >= 2) && (wkey != 0.0);
    if (refl) {
      const unsigned long long* cb = colw + ((int64_t)par * G + wcta) * cstride;
      const double wxj = sh.wxj;
      const double nrm = sqrt(wkey);
      const double beta = (wxj >= 0.0) ? -nrm : nrm;
      const double h = beta - wxj;
      const double inv = 1.0 / sqrt(h * h + sh.wtail);
      for (int i = 32 * KJ + threadIdx.x; i < 32 * RPL; i += NT) {
        double val = 0.0;
        if (i > j && i < m) {
          unsigned long long c0, c1;
          do {
            ld_ll2(cb + 2 * i, c0, c1);
          } while ((unsigned)c0 != stamp || (unsigned)c1 != stamp);
          val = -__longlong_as_double((long long)((c0 & 0xffffffff00000000ull) | (c1 >> 32))) * inv;
        } else if (i == j) {
          val = h * inv;
        }
        u[i] = val;
      }
    }
#pragma unroll
    for (int q = 0; q < CPW; q++) {
      if (cbase + q == win.col) {
        pos[q] = j;
        act[q] = false;
      } else if (act[q] && pos[q] == j) {
        pos[q] = win.pos;
      }
    }
    if constexpr (SMEM) {
      if (lane < sm.spw) {
        const int sc = warp * sm.spw + lane;
        if (sm.cbase_s + lane == win.col) {
          sm.spos[sc] = j;
          sm.sact[sc] = 0;
        } else if (sm.sact[sc] && sm.spos[sc] == j) {
          sm.spos[sc] = win.pos;
        }
      }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) p.chosen[j] = win.col;
    have_refl = refl;
    __syncthreads();
    dbg_stamp(j, 5);
  }
}

template <int KJ, int RPL, int CPW, int WARPS, bool SMEM>
RQ_DEV void sk_dispatch(int kj, const SketchArgs& p, SkSlot2* slots, SkWin* wins, unsigned long long stamp_base,
                        double (&x)[CPW][RPL], int (&pos)[CPW], bool (&act)[CPW], bool& have_refl, double* u,
                        SkShared& sh, int cbase, int jend, const SkSmem& sm) {
  if constexpr (KJ < RPL) {
    if (kj == KJ)
      sk_block<KJ, RPL, CPW, WARPS, SMEM>(p, slots, wins, stamp_base, x, pos, act, have_refl, u, sh, cbase, jend, sm);
    else
      sk_dispatch<KJ + 1, RPL, CPW, WARPS, SMEM>(kj, p, slots, wins, stamp_base, x, pos, act, have_refl, u, sh,
                                                 cbase, jend, sm);
  }
}

// Register-resident sketch CPQR.  CTA g owns columns [g*PER, (g+1)*PER): WARPS*CPW in registers
// (warp w: g*PER + w*CPW + q) then, with SMEM, WARPS*spw in shared memory (warp w: after the
// register block, w*spw + s).
template <int RPL, int CPW, int WARPS, bool SMEM>
__global__ void __launch_bounds__(WARPS * 32, 1) sketch_reg_kernel(const SketchArgs p, SkSlot2* slots, SkWin* wins,
                                                                   unsigned long long stamp_base) {
  __shared__ double u[32 * RPL];
  __shared__ SkShared sh;
  extern __shared__ double sk_dyn[];
  constexpr int kMaxSpw = kSkMaxSpw;
  __shared__ int spos_s[SMEM ? WARPS * kMaxSpw : 1];
  __shared__ int sact_s[SMEM ? WARPS * kMaxSpw : 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int spw = SMEM ? p.spw : 0;
  const int per = WARPS * CPW + WARPS * spw;
  const int cbase = blockIdx.x * per + warp * CPW;
  __shared__ SkClu clu;
  const int spw_g = SMEM ? p.spw_g : 0;
  SkSmem sm{sk_dyn, spos_s, sact_s, spw, (int)blockIdx.x * per + WARPS * CPW + warp * spw, &clu, spw - spw_g,
            spw_g > 0 ? p.gcols + ((int64_t)blockIdx.x * WARPS + warp) * spw_g * RPL * 32 : nullptr};
  if (p.cl > 1) {
    if (threadIdx.x == 0) {
      mbar_init(&clu.kbar[0], 1);
      mbar_init(&clu.kbar[1], 1);
      mbar_init(&clu.wbar[0], 1);
      mbar_init(&clu.wbar[1], 1);
      mbar_init_fence();
    }
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  double x[CPW][RPL];
  int pos[CPW];
  bool act[CPW];
#pragma unroll
  for (int q = 0; q < CPW; q++) {
    const int c = cbase + q;
    act[q] = c < p.n;
    pos[q] = act[q] ? (p.init_pos ? p.init_pos[c] : c) : INT_MAX;
#pragma unroll
    for (int k = 0; k < RPL; k++) {
      const int i = lane + 32 * k;
      x[q][k] = (act[q] && i < p.m) ? p.y[(int64_t)c * p.ld + i] : 0.0;
    }
  }
  if constexpr (SMEM) {
    for (int s2 = 0; s2 < spw; s2++) {
      const int sc = warp * spw + s2;
      const int c = sm.cbase_s + s2;
      const bool a = c < p.n;
      double* col = sk_tier_col<RPL>(sm, warp, s2) + lane;
#pragma unroll
      for (int k = 0; k < RPL; k++) {
        const int i = lane + 32 * k;
        col[k * 32] = (a && i < p.m) ? p.y[(int64_t)c * p.ld + i] : 0.0;
      }
      if (lane == 0) {
        sact_s[sc] = a ? 1 : 0;
        spos_s[sc] = a ? (p.init_pos ? p.init_pos[c] : c) : INT_MAX;
      }
    }
    __syncthreads();
  }
  bool have_refl = false;
  for (int kj = 0; 32 * kj < p.steps; kj++) {
    const int jend = min(p.steps, 32 * kj + 32);
    sk_dispatch<0, RPL, CPW, WARPS, SMEM>(kj, p, slots, wins, stamp_base, x, pos, act, have_refl, u, sh, cbase, jend,
                                          sm);
  }
  if (p.cl > 1)  // no CTA leaves while a cluster peer may still push into its shared memory
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int RPL, int CPW, int WARPS, bool SMEM = false>
static int launch_sketch_reg(const SketchArgs& a, int G, SkSlot2* slots, SkWin* wins, unsigned long long stamp_base,
                             cudaStream_t st, int64_t* launches) {
  void* args[] = {(void*)&a, (void*)&slots, (void*)&wins, (void*)&stamp_base};
  auto kern = sketch_reg_kernel<RPL, CPW, WARPS, SMEM>;
  const size_t dyn = SMEM ? (size_t)WARPS * (a.spw - a.spw_g) * RPL * 32 * sizeof(double) : 0;
  if (SMEM) {
    static bool attr = false;
    if (!attr) {
      RQ_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      attr = true;
    }
  }
  // two-level exchange over clusters of CS CTAs when the rounded-up grid is co-resident
  // (RQ_SK_CLUSTER=4).  Correct (same pivots) but measured slower: 9.10 vs 5.21 us/step at
  // n' = 10k (35 leaders each polling all 35 slots contend like the flat all-gather did), so off
  static const int env_cl = [] {
    const char* e = getenv("RQ_SK_CLUSTER");
    return e ? atoi(e) : 0;
  }();
  SketchArgs ac = a;
  ac.cl = 0;
  ac.per = a.spw * WARPS + CPW * WARPS;
  for (int CS = env_cl; CS >= 2; CS /= 2) {
    const int Gc = (G + CS - 1) / CS * CS;
    if (Gc > kSMs) continue;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(Gc);
    cfg.blockDim = dim3(WARPS * 32);
    cfg.dynamicSmemBytes = dyn;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nclu = 0;
    if (cudaOccupancyMaxActiveClusters(&nclu, kern, &cfg) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (nclu * CS < Gc) continue;  // every CTA must be resident: they wait on one another
    cfg.numAttrs = 2;
    ac.cl = CS;
    RQ_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, ac, slots, wins, stamp_base));
    if (launches) (*launches)++;
    return RQ_OK;
  }
  RQ_CUDA_TRY(cudaLaunchCooperativeKernel((void*)kern, dim3(G), dim3(WARPS * 32), args, dyn, st));
  if (launches) (*launches)++;
  return RQ_OK;
}

// (warps, columns per warp) options in order of preference; registers: CPW*RPL doubles.
// Beyond their capacity (RPL = 9, i.e. b+p <= 288): 12 warps x 6 register columns plus up to
// 7 shared-memory columns per warp (<= 200 KB), 156 columns per CTA.
template <int RPL>
static int dispatch_sketch_reg(SketchArgs a, int n, SkSlot2* slots, SkWin* wins, unsigned long long stamp_base,
                               cudaStream_t st, int64_t* launches, int* grid, int gmax) {
  struct Opt {
    int warps, cpw;
  };
  // (8, 8) and (8, 9): n' ~ 8.5k..10.6k on 139..148 CTAs instead of 107..125 with (8, 10)
  const Opt opts[] = {{16, 1}, {16, 2}, {16, 3}, {8, 6}, {8, 8}, {8, 9}, {8, 10}};
  a.spw = 0;
  for (const Opt& o : opts) {
    if (RPL * o.cpw > (o.warps == 16 ? 30 : 92)) continue;  // register budget
    const int G = (n + o.warps * o.cpw - 1) / (o.warps * o.cpw);
    if (G > gmax) continue;
    *grid = G;
    if (o.warps == 16 && o.cpw == 1) return launch_sketch_reg<RPL, 1, 16>(a, G, slots, wins, stamp_base, st, launches);
    if (o.warps == 16 && o.cpw == 2) return launch_sketch_reg<RPL, 2, 16>(a, G, slots, wins, stamp_base, st, launches);
    if (o.warps == 16 && o.cpw == 3) return launch_sketch_reg<RPL, 3, 16>(a, G, slots, wins, stamp_base, st, launches);
    if (o.cpw == 6) return launch_sketch_reg<RPL, 6, 8>(a, G, slots, wins, stamp_base, st, launches);
    if constexpr (RPL == 9) {
      if (o.cpw == 8) return launch_sketch_reg<RPL, 8, 8>(a, G, slots, wins, stamp_base, st, launches);
      if (o.cpw == 9) return launch_sketch_reg<RPL, 9, 8>(a, G, slots, wins, stamp_base, st, launches);
    }
    if (o.cpw == 8 || o.cpw == 9) continue;
    return launch_sketch_reg<RPL, 10, 8>(a, G, slots, wins, stamp_base, st, launches);
  }
  if constexpr (RPL == 9) {
    constexpr int W = 12, C = 6;
    const int per_needed = (n + gmax - 1) / gmax;
    const int spw = std::max(1, (per_needed - W * C + W - 1) / W);
    if (spw <= 7 && (size_t)W * spw * RPL * 32 * 8 <= 200 * 1024) {
      a.spw = spw;
      a.spw_g = 0;
      const int per = W * C + W * spw;
      const int G = (n + per - 1) / per;
      *grid = G;
      return launch_sketch_reg<RPL, C, W, true>(a, G, slots, wins, stamp_base, st, launches);
    }
    if (RPL == 9 && spw <= kSkMaxSpw && a.gcols) {
      // beyond 156 columns per CTA: the last spw - 7 columns of each warp live in global memory
      // (L2-resident, streamed through registers every step; sketch_glob_bytes sized gcols)
      a.spw = spw;
      a.spw_g = spw - 7;
      const int per = W * C + W * spw;
      const int G = (n + per - 1) / per;
      *grid = G;
      return launch_sketch_reg<RPL, C, W, true>(a, G, slots, wins, stamp_base, st, launches);
    }
  }
  return -1;  // does not fit: caller falls back
}

size_t sketch_ll_column_bytes(int m) { return 2 * (size_t)kSMs * 2 * ((size_t)m + 2) * 8; }
// True when sketch_cpqr_launch(m, n) runs a register / shared-memory tier, which only reads Y
// (the L2-streaming fallback overwrites it).  Mirrors dispatch_sketch_reg's choice.
bool sketch_cpqr_preserves_input(int m, int n, int gmax) {
  if (gmax <= 0 || gmax > kSMs) gmax = kSMs;
  if (m > 288) return false;
  const int rpl = m <= 96 ? 3 : (m <= 160 ? 5 : 9);
  const int opts[][2] = {{16, 1}, {16, 2}, {16, 3}, {8, 6}, {8, 8}, {8, 9}, {8, 10}};
  for (const auto& o : opts) {
    if (rpl * o[1] > (o[0] == 16 ? 30 : 92)) continue;
    if ((o[1] == 8 || o[1] == 9) && rpl != 9) continue;
    if ((n + o[0] * o[1] - 1) / (o[0] * o[1]) <= gmax) return true;
  }
  if (rpl == 9) {
    const int W = 12, C = 6;
    const int per_needed = (n + gmax - 1) / gmax;
    const int spw = std::max(1, (per_needed - W * C + W - 1) / W);
    if (spw <= kSkMaxSpw) return true;  // shared memory, then the global tier
  }
  return false;
}

// Global-memory tier of the register sketch CPQR for n columns (0 when shared memory suffices).
size_t sketch_glob_bytes(int m, int n) {
  if (m <= 160 || m > 288) return 0;
  const int W = 12, C = 6;
  const int per_needed = (n + kSkMinGrid - 1) / kSkMinGrid;  // the most columns per CTA a launch uses
  const int spw = std::max(1, (per_needed - W * C + W - 1) / W);
  if (spw <= 7 || spw > kSkMaxSpw) return 0;
  return (size_t)kSMs * W * (spw - 7) * 9 * 32 * sizeof(double);
}

size_t sketch_ll_bytes(int m) { return ((2 * (size_t)kSMs * 64 + 255) & ~size_t(255)) + 256 + sketch_ll_column_bytes(m); }
static size_t sketch_base_bytes(int m) {
  return ((2 * (size_t)kSMs * 64 + 255) & ~size_t(255)) + 256 + sketch_ll_column_bytes(m);
}
size_t sketch_workspace_bytes(int m, int n) { return sketch_base_bytes(m) + sketch_glob_bytes(m, n); }

static size_t sketch_fixed_smem(int m, int per) {
  return (size_t)m * 8 + (size_t)per * 8 + 16 + (SK_WARPS + 2) * sizeof(SweepSlot) + 64;
}

int sketch_cpqr_launch(const double* y, int64_t ld, int m, int n, int steps, const int* init_pos, int* chosen,
                       SweepWork& w, unsigned long long* counter, unsigned long long& counter_base, cudaStream_t st,
                       int64_t* launches, int gmax) {
  if (steps <= 0) return RQ_OK;
  if (gmax <= 0 || gmax > kSMs) gmax = kSMs;
  if (gmax < kSkMinGrid) gmax = kSkMinGrid;
  if (m <= 288) {
    SketchArgs a{};
    a.y = y;
    a.ywork = const_cast<double*>(y);
    a.ld = ld;
    a.m = m;
    a.n = n;
    a.steps = steps;
    a.init_pos = init_pos;
    a.chosen = chosen;
    // slots + LL columns: in the caller's scratch, or in the context's placed block (w.ll)
    char* llb = w.ll ? reinterpret_cast<char*>(w.ll) : reinterpret_cast<char*>(w.scratch);
    SkSlot2* slots = reinterpret_cast<SkSlot2*>(llb);  // [2][G] slots of 8 LL words
    const size_t slot_bytes = ((2 * (size_t)kSMs * 64 + 255) & ~size_t(255));
    // dedicated, zero-initialised winner records (2 x 10 LL words) next to the counter
    SkWin* wins = reinterpret_cast<SkWin*>(reinterpret_cast<char*>(counter) + 64);
    a.slotdata = reinterpret_cast<double*>(llb + slot_bytes + 256);  // LL columns
    a.counter = counter;
    a.counter_base = counter_base;
    const size_t need = w.ll ? 0 : slot_bytes + 256 + sketch_ll_column_bytes(m);
    const size_t gbytes = sketch_glob_bytes(m, n);
    a.gcols = (gbytes > 0 && w.scratch_bytes >= need + gbytes)
                  ? reinterpret_cast<double*>(reinterpret_cast<char*>(w.scratch) + need)
                  : nullptr;
    if (w.scratch_bytes >= need) {
      // step stamps are unique across launches: derived from the monotone counter base
      const unsigned long long stamp_base = counter_base;
      static const int env_fr = [] {
        // CTA 0 reduces every step (1; 0 = the last arriver, 2 = the last CTA).  With the
        // reduce-scatter column sums, 1 is slower in isolation (4.96 -> 5.62 us/step at n' = 10k)
        // but faster inside the factorization, where the CTAs of one launch start staggered
        // behind the preceding kernels: n = 5k 56.2 -> 54.9 ms, 10k 142.3 -> 139.5, 20k 569.0 -> 560.8
        const char* e = getenv("RQ_SK_FIXED_REDUCER");
        return e ? atoi(e) : 1;
      }();
      a.fixed_reducer = env_fr;
      int rc, G = 0;
      if (m <= 96) rc = dispatch_sketch_reg<3>(a, n, slots, wins, stamp_base, st, launches, &G, gmax);
      else if (m <= 160) rc = dispatch_sketch_reg<5>(a, n, slots, wins, stamp_base, st, launches, &G, gmax);
      else rc = dispatch_sketch_reg<9>(a, n, slots, wins, stamp_base, st, launches, &G, gmax);
      if (rc >= 0) {
        counter_base += (unsigned long long)steps * G;  // every CTA arrives once per step
        return rc;
      }
    }
  }
  int G = (n + 15) / 16;  // >= 16 columns per CTA
  if (G > gmax) G = gmax;
  if (G < 1) G = 1;
  const int per = (n + G - 1) / G;
  const size_t kMax = 220 * 1024;
  const size_t fixed = sketch_fixed_smem(m, per);
  int cache_cols = (int)std::min<size_t>((size_t)per, (kMax - fixed) / ((size_t)m * 8));
  const size_t smem = ((fixed + (size_t)cache_cols * m * 8) + 15) & ~size_t(15);
  const size_t need = 2 * (size_t)G * sizeof(SkSlot) + 256 + 2 * (size_t)G * m * 8;
  if (w.scratch_bytes < need) return set_error(RQ_EINTERNAL, "sketch workspace too small");
  SketchArgs a;
  a.y = y;
  a.ywork = const_cast<double*>(y);
  a.ld = ld;
  a.m = m;
  a.n = n;
  a.steps = steps;
  a.init_pos = init_pos;
  a.chosen = chosen;
  a.slots = reinterpret_cast<SkSlot*>(w.scratch);
  a.slotdata = reinterpret_cast<double*>(reinterpret_cast<char*>(w.scratch) +
                                         ((2 * (size_t)G * sizeof(SkSlot) + 255) & ~size_t(255)));
  a.counter = counter;
  a.counter_base = counter_base;
  counter_base += (unsigned long long)steps * G;
  a.cache_cols = cache_cols;
  static bool attr = false;
  if (!attr) {
    RQ_CUDA_TRY(cudaFuncSetAttribute(sketch_cpqr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMax));
    attr = true;
  }
  void* args[] = {(void*)&a};
  RQ_CUDA_TRY(cudaLaunchCooperativeKernel((void*)sketch_cpqr_kernel, dim3(G), dim3(SK_THREADS), args, smem, st));
  if (launches) (*launches)++;
  return RQ_OK;
}

// ---------------------------------------------------------------------------
size_t sweep_workspace_bytes(int64_t m, int total_cols, int grid) {
  (void)total_cols;
  size_t b = 2 * (size_t)grid * sizeof(SweepSlot) + 256;
  b += 2 * (size_t)grid * m * sizeof(double) + 256;
  b += (size_t)grid * m * sizeof(double) + 256;  // u fallback
  return b;
}

int sweep_debug_timing(int on, unsigned long long* host, int count) {
  RQ_CUDA_TRY(cudaMemcpyToSymbol(g_sweep_dbg_on, &on, sizeof(int)));
  if (host) RQ_CUDA_TRY(cudaMemcpyFromSymbol(host, g_sweep_dbg, sizeof(unsigned long long) * std::min(count, 512)));
  return RQ_OK;
}

int sweep_grid_size(int total_cols) {
  int g = (total_cols + 3) / 4;  // at least 4 columns per CTA
  if (g > kSMs) g = kSMs;
  if (g < 1) g = 1;
  return g;
}

static int sweep_launch_cluster(const SweepCall& c, int CS, size_t smem, cudaStream_t st, int64_t* launches) {
  SweepArgs a{};
  a.a = c.a;
  a.lda = c.lda;
  a.m = c.m;
  a.n = c.n;
  a.n_acc = c.n_acc;
  a.steps = c.steps;
  a.pivot = c.pivot;
  a.init_pos = c.init_pos;
  a.v = c.v;
  a.ldv = c.ldv;
  a.col_at_pos = c.col_at_pos;
  a.r_out = c.r_out;
  a.ldr = c.ldr;
  static bool attr = false;
  if (!attr) {
    RQ_CUDA_TRY(cudaFuncSetAttribute(sweep_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    RQ_CUDA_TRY(cudaFuncSetAttribute(sweep_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CS);
  cfg.blockDim = dim3(SC_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  RQ_CUDA_TRY(cudaLaunchKernelEx(&cfg, sweep_cluster_kernel, a));
  if (launches) (*launches)++;
  return RQ_OK;
}

int sweep_launch(const SweepCall& c, SweepWork& w, cudaStream_t st, int64_t* launches) {
  if (c.steps <= 0) return RQ_OK;
  const int total = c.n + c.n_acc;
  // register-resident cluster path: one warp per column, rows in registers
  if (c.n_acc == 0 && c.n <= 256 && c.m <= 512) {
    SweepArgs a{};
    a.a = c.a;
    a.lda = c.lda;
    a.m = c.m;
    a.n = c.n;
    a.steps = c.steps;
    a.pivot = c.pivot;
    a.init_pos = c.init_pos;
    a.v = c.v;
    a.ldv = c.ldv;
    a.col_at_pos = c.col_at_pos;
    a.r_out = c.r_out;
    a.ldr = c.ldr;
    const int CS = std::max(1, (c.n + 15) / 16);
    if (c.m <= 64) return launch_reg<2>(a, CS, st, launches);
    if (c.m <= 128) return launch_reg<4>(a, CS, st, launches);
    if (c.m <= 256) return launch_reg<8>(a, CS, st, launches);
    return launch_reg<16>(a, CS, st, launches);
  }
  // cluster path when the whole matrix fits in one 16-CTA cluster's shared memory
  if (c.m <= 4096) {
    for (int CS : {4, 8, 16}) {
      const int per = (total + CS - 1) / CS;
      if (per > 16 && CS < 16) continue;  // prefer 16 CTAs unless the problem is tiny
      const size_t smem = cluster_smem(c.m, per);
      if (smem <= 220 * 1024) return sweep_launch_cluster(c, CS, smem, st, launches);
    }
  }
  const int G = c.grid > 0 ? c.grid : sweep_grid_size(total);
  const int per = (total + G - 1) / G;
  const size_t kMaxSmem = 220 * 1024;
  size_t fixed = (size_t)per * sizeof(int) + per + 16 + (SW_WARPS + 4) * sizeof(SweepSlot) + 64;
  int u_in_smem = (fixed + (size_t)c.m * 8 <= kMaxSmem) ? 1 : 0;
  size_t avail = kMaxSmem - fixed - (u_in_smem ? (size_t)c.m * 8 : 0);
  int cache_cols = (int)std::min<size_t>((size_t)per, avail / ((size_t)c.m * 8));
  size_t smem = fixed + (u_in_smem ? (size_t)c.m * 8 : 0) + (size_t)cache_cols * c.m * 8;
  smem = (smem + 15) & ~size_t(15);

  SweepArgs a;
  a.a = c.a;
  a.lda = c.lda;
  a.m = c.m;
  a.n = c.n;
  a.n_acc = c.n_acc;
  a.steps = c.steps;
  a.pivot = c.pivot;
  a.init_pos = c.init_pos;
  a.v = c.v;
  a.ldv = c.ldv;
  a.col_at_pos = c.col_at_pos;
  a.r_out = c.r_out;
  a.ldr = c.ldr;
  char* ws = reinterpret_cast<char*>(w.scratch);
  a.slots = reinterpret_cast<SweepSlot*>(ws);
  ws += ((2 * (size_t)G * sizeof(SweepSlot) + 255) / 256) * 256;
  a.slotdata = reinterpret_cast<double*>(ws);
  ws += ((2 * (size_t)G * c.m * sizeof(double) + 255) / 256) * 256;
  a.ubuf_global = reinterpret_cast<double*>(ws);
  a.bar = w.next_barrier();
  a.cache_cols = cache_cols;
  a.u_in_smem = u_in_smem;
  if (w.scratch_bytes < sweep_workspace_bytes(c.m, total, G))
    return set_error(RQ_EINTERNAL, "sweep workspace too small");

  static size_t smem_set = 0;
  if (smem > smem_set) {
    RQ_CUDA_TRY(cudaFuncSetAttribute(sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem));
    smem_set = kMaxSmem;
  }
  void* args[] = {(void*)&a};
  RQ_CUDA_TRY(cudaLaunchCooperativeKernel((void*)sweep_kernel, dim3(G), dim3(SW_THREADS), args, smem, st));
  if (launches) (*launches)++;
  return RQ_OK;
}

}  // namespace rq
