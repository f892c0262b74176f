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

int sweep_launch(const SweepCall& c, SweepWork& w, cudaStream_t st, int64_t* launches) {
  if (c.steps <= 0) return RQ_OK;
  const int total = c.n + c.n_acc;
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
