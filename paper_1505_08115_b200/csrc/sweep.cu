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
    cluster_barrier();
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
    const SweepSlot win = red[SC_WARPS + 1];
    const unsigned wrank = (unsigned)reinterpret_cast<int*>(&red[SC_WARPS])[2];
    double* xs = xin + (int64_t)par * m;
    if (rank == wrank) {
      // the owner pushes the winning column (rows j..m-1) to every CTA
      const double* src = cols + (int64_t)(win.col - c0) * m;
      for (int dstr = warp; dstr < (int)CS; dstr += SC_WARPS)
        for (int64_t i = j + lane; i < m; i += 32) dsmem_st_f64(xs + i, (unsigned)dstr, src[i]);
    }
    cluster_barrier();
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
    if (lane == 0) red[warp] = SweepSlot{bk, bt, bp, bc};
    __syncthreads();
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
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(p.counter, 1ull);
      const unsigned long long target = p.counter_base + (unsigned long long)(j + 1) * G;
      while (ld_acquire_u64(p.counter) < target) {
      }
    }
    __syncthreads();
    // -------- every CTA reads the G candidates (one batch of loads) and picks the winner --------
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
    if (blockIdx.x == 0 && threadIdx.x == 0) p.chosen[j] = win.col;
    have_refl = refl;
    rj = j;
    __syncthreads();
  }
}

static size_t sketch_fixed_smem(int m, int per) {
  return (size_t)m * 8 + (size_t)per * 8 + 16 + (SK_WARPS + 2) * sizeof(SweepSlot) + 64;
}

int sketch_cpqr_launch(const double* y, int64_t ld, int m, int n, int steps, const int* init_pos, int* chosen,
                       SweepWork& w, unsigned long long* counter, unsigned long long& counter_base, cudaStream_t st,
                       int64_t* launches) {
  if (steps <= 0) return RQ_OK;
  int G = (n + 15) / 16;  // >= 16 columns per CTA
  if (G > kSMs) G = kSMs;
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
