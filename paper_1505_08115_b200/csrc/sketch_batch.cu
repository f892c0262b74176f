// Batched sketch CPQR: select_pivot_permutation (pivoting.py:114-129), i.e. the first `steps`
// pivots of householder_sweep(pivot=True) (_kernels_numba.py:13-61) on Y^T, with the same greedy
// pivot sequence but ONE grid-wide exchange per *batch* of pivots instead of one per pivot.
//
// The greedy rule picks, at step j, the column of largest trailing norm (rows j..m-1), lowest
// position on ties.  A trailing norm never grows under later reflections (they are orthogonal on
// rows >= j and a row is dropped per step), so at a batch start every CTA ("worker") sends its
// two best columns -- the candidates -- together with an upper bound U on all its other columns
// to one "solver" CTA.  The solver runs the greedy steps on the candidates alone: step 0 of a batch is
// always exact (the global best is some worker's best), and a later step is accepted while its
// winner's current norm exceeds every bound (with a 1e-10 relative margin for rounding), which
// proves that no column outside the candidate set could have won.  Each accepted pivot's
// reflector is published at once; the workers apply the stream of reflectors to their columns
// (registers, then shared memory) while the solver is already at the next step.  When a step
// cannot be proven, the batch ends and the workers send new candidates.
//
// Per-column arithmetic (lane l holds rows l, l+32, ...; per-lane fma chains, fixed butterfly)
// is one device function used by workers and solver alike, so a candidate's copy in the solver
// and the original in its worker stay bitwise equal.
//
// Exchange: LL words (32-bit payload + 32-bit stamp per 8-byte word, sk_common.cuh); stamps are
// launch-unique event numbers, so no fences or flags sit on the path.  Worker -> solver: one
// candidate slot per worker (key, position, column id, bound, the column).  Solver -> workers:
// one event slot per step of the batch (type, step, column id, swap position, the reflector).
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "common.cuh"
#include "sk_common.cuh"
#include "sweep.cuh"

namespace rq {
namespace {

constexpr int SB_TMAX = 32;  // pivots per batch at most (event slots)
constexpr int kSbSolverCpw = 3;  // candidates per solver warp
constexpr unsigned EV_REFL = 1u, EV_PIVOT = 2u, EV_END = 3u, EV_DONE = 4u;

struct SbArgs {
  const double* y;  // m x n (col-major, ld): read only
  int64_t ld;
  int m, n, steps;
  const int* init_pos;
  int* chosen;
  unsigned long long* cand;  // [2 * workers][2 * (3 + 32 RPL)] LL words (two candidate slots per worker)
  unsigned long long* ev;    // [SB_TMAX + 1][2 * (2 + 32 RPL)] LL words
  unsigned stamp_base;
  int per;  // columns per worker
  int spw;  // shared-memory columns per warp (workers)
  int dbg;  // RQ_SB_DBG: the solver prints its batch / cycle counts
};

template <int RPL, int WARPS>
struct SbShared {
  double u[2][32 * RPL];
  unsigned hdr[2][4];  // type, step, column, swap position
  // worker: entry 2w + r = warp w's r-th best column
  unsigned wk_hi[2 * WARPS], wk_lo[2 * WARPS];
  int wk_pos[2 * WARPS], wk_col[2 * WARPS];
  double w2[WARPS];
  double redmax[WARPS];  // solver: each warp's share of the batch's bound
};

RQ_DEV void sb_poll(const unsigned long long* p, unsigned stamp, unsigned long long& a, unsigned long long& b) {
  unsigned spins = 0;
  for (;;) {
    ld_ll2(p, a, b);
    if ((unsigned)a == stamp && (unsigned)b == stamp) return;
    if (++spins > (1u << 25)) __trap();  // a lost peer: fail the launch instead of hanging the GPU
  }
}
RQ_DEV double sb_double(unsigned long long a, unsigned long long b) {
  return __longlong_as_double((long long)((a & 0xffffffff00000000ull) | (b >> 32)));
}
RQ_DEV void sb_put_double(unsigned long long* p, double v, unsigned stamp) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
  st_ll2(p, ll_word((unsigned)(bits >> 32), stamp), ll_word((unsigned)bits, stamp));
}
RQ_DEV double sb_key(unsigned hi, unsigned lo) {
  return __longlong_as_double((long long)(((unsigned long long)hi << 32) | lo));
}
RQ_DEV double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// H = I - 2 u u^T on every register column of the warp (u = 0 outside the reflector's rows).
template <int RPL, int CPW>
RQ_DEV void sb_apply(double (&x)[CPW][RPL], const double (&uk)[RPL], int lane) {
  double d[CPW];
#pragma unroll
  for (int q = 0; q < CPW; q++) {
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < RPL; k++) acc = fma(uk[k], x[q][k], acc);
    d[q] = acc;
  }
  warp_sum_all<CPW, 0, CPW>(d, lane);
#pragma unroll
  for (int q = 0; q < CPW; q++) {
    const double dd = -2.0 * d[q];
#pragma unroll
    for (int k = 0; k < RPL; k++) x[q][k] = fma(dd, uk[k], x[q][k]);
  }
}

// Two shared-memory columns (same arithmetic per column).
template <int RPL>
RQ_DEV void sb_apply2(double (&y0)[RPL], double (&y1)[RPL], const double (&uk)[RPL], int lane) {
  double dd[2] = {0.0, 0.0};
#pragma unroll
  for (int k = 0; k < RPL; k++) {
    dd[0] = fma(uk[k], y0[k], dd[0]);
    dd[1] = fma(uk[k], y1[k], dd[1]);
  }
  warp_sum_all<2, 0, 2>(dd, lane);
  const double d0 = -2.0 * dd[0], d1 = -2.0 * dd[1];
#pragma unroll
  for (int k = 0; k < RPL; k++) {
    y0[k] = fma(d0, uk[k], y0[k]);
    y1[k] = fma(d1, uk[k], y1[k]);
  }
}

// Trailing norms^2 (rows >= j) of the warp's register columns.
template <int RPL, int CPW>
RQ_DEV void sb_keys(const double (&x)[CPW][RPL], int j, int lane, double (&t)[CPW]) {
#pragma unroll
  for (int q = 0; q < CPW; q++) {
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < RPL; k++) {
      const double xv = (lane + 32 * k >= j) ? x[q][k] : 0.0;
      acc = fma(xv, xv, acc);
    }
    t[q] = acc;
  }
  warp_sum_all<CPW, 0, CPW>(t, lane);
}
template <int RPL>
RQ_DEV double sb_key1(const double (&y)[RPL], int j, int lane) {
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < RPL; k++) {
    const double xv = (lane + 32 * k >= j) ? y[k] : 0.0;
    acc = fma(xv, xv, acc);
  }
  return warp_sum(acc);
}

// ---------------------------------------------------------------------------
// Worker: owns columns [c0, c1); local column lc lives in warp lc % WARPS, slot lc / WARPS
// (slots < CPW in registers, the rest in shared memory [warp][s][k][lane]).  Per batch it sends
// its two best columns (candidate slots 2g, 2g + 1) and the bound on all the others.
// ---------------------------------------------------------------------------
struct SbTop {  // a warp's two best columns and the largest key of the rest
  double k1 = -1.0, k2 = -1.0, k3 = -1.0;
  int p1 = INT_MAX, p2 = INT_MAX, s1 = -1, s2 = -1;
  RQ_DEV void offer(double k, int ps, int slot) {
    if (s1 < 0 || piv_better(k, ps, k1, p1)) {
      k3 = fmax(k3, k2);
      k2 = k1, p2 = p1, s2 = s1;
      k1 = k, p1 = ps, s1 = slot;
    } else if (s2 < 0 || piv_better(k, ps, k2, p2)) {
      k3 = fmax(k3, k2);
      k2 = k, p2 = ps, s2 = slot;
    } else {
      k3 = fmax(k3, k);
    }
  }
};

template <int RPL, int CPW, int WARPS>
RQ_DEV void sb_worker(const SbArgs& p, SbShared<RPL, WARPS>& sh, double* xs_all, int* spos_all, int* sact_all) {
  constexpr int NT = WARPS * 32, NR = 32 * RPL, SLOTW = 2 * (3 + NR);
  static_assert(2 * WARPS <= 32, "the CTA's top two are resolved by one warp");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wk = (int)blockIdx.x - 1;
  const int c0 = wk * p.per, c1 = min(p.n, c0 + p.per);
  const int spw = p.spw;
  double* xs = xs_all + (int64_t)warp * spw * NR + lane;
  int* spos = spos_all + warp * spw;
  int* sact = sact_all + warp * spw;

  double x[CPW][RPL];
  int pos[CPW];
  bool act[CPW];
#pragma unroll
  for (int q = 0; q < CPW; q++) {
    const int c = c0 + q * WARPS + warp;
    act[q] = c < c1;
    pos[q] = act[q] ? (p.init_pos ? p.init_pos[c] : c) : INT_MAX;
#pragma unroll
    for (int k = 0; k < RPL; k++) {
      const int i = lane + 32 * k;
      x[q][k] = (act[q] && i < p.m) ? p.y[(int64_t)c * p.ld + i] : 0.0;
    }
  }
  for (int s = 0; s < spw; s++) {
    const int c = c0 + (CPW + s) * WARPS + warp;
    const bool a = c < c1;
#pragma unroll
    for (int k = 0; k < RPL; k++) {
      const int i = lane + 32 * k;
      xs[(int64_t)s * NR + k * 32] = (a && i < p.m) ? p.y[(int64_t)c * p.ld + i] : 0.0;
    }
    if (lane == 0) {
      sact[s] = a ? 1 : 0;
      spos[s] = a ? (p.init_pos ? p.init_pos[c] : c) : INT_MAX;
    }
  }
  __syncwarp();

  unsigned long long* myslots = p.cand + (int64_t)wk * 2 * SLOTW;
  unsigned e = 0;
  int j = 0;
  for (;;) {
    // ---- candidates at step j: the CTA's two best (key, position) and the bound on the rest ----
    SbTop top;
    {
      double t[CPW];
      sb_keys<RPL, CPW>(x, j, lane, t);
#pragma unroll
      for (int q = 0; q < CPW; q++)
        if (act[q]) top.offer(t[q], pos[q], q);
    }
    for (int s = 0; s < spw; s += 2) {
      const bool has1 = s + 1 < spw;
      const bool a0 = sact[s] != 0, a1 = has1 && sact[s + 1] != 0;  // warp-uniform
      if (!a0 && !a1) continue;
      const double* col0 = xs + (int64_t)s * NR;
      const double* col1 = has1 ? col0 + NR : col0;
      double tt[2] = {0.0, 0.0};
#pragma unroll
      for (int k = 0; k < RPL; k++) {
        const bool in = lane + 32 * k >= j;
        const double v0 = in ? col0[k * 32] : 0.0, v1 = in ? col1[k * 32] : 0.0;
        tt[0] = fma(v0, v0, tt[0]);
        tt[1] = fma(v1, v1, tt[1]);
      }
      warp_sum_all<2, 0, 2>(tt, lane);
      if (a0) top.offer(tt[0], spos[s], CPW + s);
      if (a1) top.offer(tt[1], spos[s + 1], CPW + s + 1);
    }
    if (lane == 0) {
      const unsigned long long b1 = (unsigned long long)__double_as_longlong(top.s1 < 0 ? 0.0 : top.k1);
      const unsigned long long b2 = (unsigned long long)__double_as_longlong(top.s2 < 0 ? 0.0 : top.k2);
      sh.wk_hi[2 * warp] = (unsigned)(b1 >> 32);
      sh.wk_lo[2 * warp] = (unsigned)b1;
      sh.wk_pos[2 * warp] = top.p1;
      sh.wk_col[2 * warp] = top.s1 < 0 ? -1 : c0 + top.s1 * WARPS + warp;
      sh.wk_hi[2 * warp + 1] = (unsigned)(b2 >> 32);
      sh.wk_lo[2 * warp + 1] = (unsigned)b2;
      sh.wk_pos[2 * warp + 1] = top.p2;
      sh.wk_col[2 * warp + 1] = top.s2 < 0 ? -1 : c0 + top.s2 * WARPS + warp;
      sh.w2[warp] = top.k3;
    }
    __syncthreads();
    const unsigned cstamp = p.stamp_base + e + 1u;
    {
      // every warp resolves the CTA's best two entries (entry 2w + r = warp w's r-th best)
      const bool lv = lane < 2 * WARPS;
      const unsigned rhi = lv ? sh.wk_hi[lane] : 0u, rlo = lv ? sh.wk_lo[lane] : 0u;
      const int rpos = lv ? sh.wk_pos[lane] : INT_MAX, rcol = lv ? sh.wk_col[lane] : -1;
      const int l1 = warp_argmax(rhi, rlo, rpos, rcol >= 0);
      const int l2 = warp_argmax(rhi, rlo, rpos, rcol >= 0 && lane != l1);
      double uv = lane < WARPS ? sh.w2[lane] : -1.0;
      if (lv && rcol >= 0 && lane != l1 && lane != l2) uv = fmax(uv, sb_key(rhi, rlo));
      uv = warp_max(uv);
#pragma unroll
      for (int r = 0; r < 2; r++) {
        const int le = r == 0 ? l1 : l2;
        unsigned long long* slot = myslots + r * SLOTW;
        if (le < 0) {
          if (warp == 0 && lane == 0) {
            st_ll2(slot, ll_word(0u, cstamp), ll_word(0u, cstamp));
            st_ll2(slot + 2, ll_word((unsigned)INT_MAX, cstamp), ll_word(0xffffffffu, cstamp));
            sb_put_double(slot + 4, r == 0 ? uv : -1.0, cstamp);
          }
        } else if (warp == (le >> 1)) {
          const int bslot = (le & 1) ? top.s2 : top.s1;
          auto publish = [&](const double (&xc)[RPL]) {
#pragma unroll
            for (int k = 0; k < RPL; k++) sb_put_double(slot + 2 * (3 + lane + 32 * k), xc[k], cstamp);
          };
          if (bslot >= CPW) {
            double y[RPL];
#pragma unroll
            for (int k = 0; k < RPL; k++) y[k] = xs[(int64_t)(bslot - CPW) * NR + k * 32];
            publish(y);
          } else {
#pragma unroll
            for (int q = 0; q < CPW; q++)
              if (q == bslot) publish(x[q]);
          }
          if (lane == 0) {
            st_ll2(slot, ll_word(sh.wk_hi[le], cstamp), ll_word(sh.wk_lo[le], cstamp));
            st_ll2(slot + 2, ll_word((unsigned)sh.wk_pos[le], cstamp), ll_word((unsigned)sh.wk_col[le], cstamp));
            sb_put_double(slot + 4, r == 0 ? uv : -1.0, cstamp);
          }
        }
      }
    }
    // ---- the batch's events: reflectors as the solver accepts them ----
    bool done = false;
    for (int idx = 0;; idx++) {
      const unsigned es = p.stamp_base + e + 1u;
      const unsigned long long* slot = p.ev + (int64_t)idx * (2 * (2 + NR));
      const int b = (int)(e & 1u);
      // two lanes wait for the header; the reflector's rows are fetched once it is there
      if (threadIdx.x < 2) {
        unsigned long long a0, a1;
        sb_poll(slot + 2 * threadIdx.x, es, a0, a1);
        sh.hdr[b][2 * threadIdx.x] = (unsigned)(a0 >> 32);
        sh.hdr[b][2 * threadIdx.x + 1] = (unsigned)(a1 >> 32);
      }
      __syncthreads();
      const unsigned type = sh.hdr[b][0];
      const int ecol = (int)sh.hdr[b][2], epos = (int)sh.hdr[b][3];
      if (type == EV_REFL) {
        for (int w = threadIdx.x; w < NR; w += NT) {
          unsigned long long a0, a1;
          sb_poll(slot + 2 * (2 + w), es, a0, a1);
          sh.u[b][w] = sb_double(a0, a1);
        }
        __syncthreads();
      }
      e++;
      if (type == EV_END) break;
      if (type == EV_DONE) {
        done = true;
        break;
      }
      // the pivot of step j: its column leaves, the column that sat at position j takes its place
#pragma unroll
      for (int q = 0; q < CPW; q++) {
        if (c0 + q * WARPS + warp == ecol) {
          pos[q] = j;
          act[q] = false;
        } else if (act[q] && pos[q] == j) {
          pos[q] = epos;
        }
      }
      if (lane < spw) {
        if (c0 + (CPW + lane) * WARPS + warp == ecol) {
          spos[lane] = j;
          sact[lane] = 0;
        } else if (sact[lane] && spos[lane] == j) {
          spos[lane] = epos;
        }
      }
      __syncwarp();
      if (type == EV_REFL) {
        double uk[RPL];
#pragma unroll
        for (int k = 0; k < RPL; k++) uk[k] = sh.u[b][lane + 32 * k];
        sb_apply<RPL, CPW>(x, uk, lane);
        for (int s = 0; s < spw; s += 2) {
          const bool has1 = s + 1 < spw;
          const bool a0 = sact[s] != 0, a1 = has1 && sact[s + 1] != 0;
          if (!a0 && !a1) continue;
          double* col0 = xs + (int64_t)s * NR;
          double* col1 = has1 ? col0 + NR : col0;
          double y0[RPL], y1[RPL];
#pragma unroll
          for (int k = 0; k < RPL; k++) {
            y0[k] = col0[k * 32];
            y1[k] = col1[k * 32];
          }
          sb_apply2<RPL>(y0, y1, uk, lane);
          if (a0) {
#pragma unroll
            for (int k = 0; k < RPL; k++) col0[k * 32] = y0[k];
          }
          if (a1) {
#pragma unroll
            for (int k = 0; k < RPL; k++) col1[k * 32] = y1[k];
          }
        }
      }
      j++;
    }
    if (done) break;
  }
}

// ---------------------------------------------------------------------------
// Solver (CTA 0).  Candidate slot s belongs to warp s % WARPS; each warp keeps the SC best of
// its group as the exact set (registers), every other candidate and every worker's bound enter
// the batch's bound.  One block barrier per step: before it every warp stages its best column
// with the reflector scalars it would have; after it every warp knows the winner, builds the
// reflector in registers, publishes its share of the event and applies it.
// ---------------------------------------------------------------------------
template <int WARPS, int NR>
struct SbStage {
  unsigned hi[WARPS], lo[WARPS];
  int pos[WARPS], col[WARPS];
  double inv[WARPS], hinv[WARPS];
  double colv[WARPS][NR];
};

template <int RPL, int SC, int WARPS>
RQ_DEV void sb_solver(const SbArgs& p, SbShared<RPL, WARPS>& sh, SbStage<WARPS, 32 * RPL>* stage) {
  constexpr int NR = 32 * RPL, SLOTW = 2 * (3 + NR);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NS = 2 * ((int)gridDim.x - 1);  // candidate slots
  const int tid = threadIdx.x;
  double x[SC][RPL];
  int pos[SC], col[SC];
  bool act[SC];
  unsigned e = 0;
  int j = 0;
  long long cyc_hdr = 0, cyc_load = 0, cyc_steps = 0;
  int nbatch = 0;
  while (j < p.steps) {
    nbatch++;
    const long long tc0 = clock64();
    // ---- this warp's group of candidate headers: slots warp + WARPS * i, i = lane, lane + 32 ----
    const unsigned cstamp = p.stamp_base + e + 1u;
    unsigned khi[2] = {0u, 0u}, klo[2] = {0u, 0u};
    int kpos[2] = {INT_MAX, INT_MAX}, kcol[2] = {-1, -1};
    double bound = -1.0;
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int s = warp + WARPS * (lane + 32 * h);
      if (s < NS) {
        const unsigned long long* sp = p.cand + (int64_t)s * SLOTW;
        unsigned long long a0, a1, a2, a3, a4, a5;
        for (unsigned spins = 0;; spins++) {
          ld_ll2(sp, a0, a1);
          ld_ll2(sp + 2, a2, a3);
          ld_ll2(sp + 4, a4, a5);
          if ((unsigned)a0 == cstamp && (unsigned)a1 == cstamp && (unsigned)a2 == cstamp && (unsigned)a3 == cstamp &&
              (unsigned)a4 == cstamp && (unsigned)a5 == cstamp)
            break;
          if (spins > (1u << 25)) __trap();
        }
        khi[h] = (unsigned)(a0 >> 32);
        klo[h] = (unsigned)(a1 >> 32);
        kpos[h] = (int)(a2 >> 32);
        kcol[h] = (int)(a3 >> 32);
        bound = fmax(bound, sb_double(a4, a5));
      }
    }
    const long long tc1 = clock64();
    // ---- the SC best of the group become the exact set ----
    bool taken[2] = {false, false};
    int sel_slot[SC];
#pragma unroll
    for (int r = 0; r < SC; r++) {
      const bool v0 = kcol[0] >= 0 && !taken[0], v1 = kcol[1] >= 0 && !taken[1];
      const bool use1 = v1 && (!v0 || piv_better(sb_key(khi[1], klo[1]), kpos[1], sb_key(khi[0], klo[0]), kpos[0]));
      const unsigned shi = use1 ? khi[1] : khi[0], slo = use1 ? klo[1] : klo[0];
      const int spos = use1 ? kpos[1] : kpos[0], scol = use1 ? kcol[1] : kcol[0];
      const int wl = warp_argmax(shi, slo, spos, v0 || v1);
      act[r] = wl >= 0;
      const int src = wl < 0 ? 0 : wl;
      if (lane == wl) {
        if (use1) taken[1] = true;
        else taken[0] = true;
      }
      sel_slot[r] = __shfl_sync(0xffffffffu, warp + WARPS * (lane + (use1 ? 32 : 0)), src);
      pos[r] = act[r] ? __shfl_sync(0xffffffffu, spos, src) : INT_MAX;
      col[r] = act[r] ? __shfl_sync(0xffffffffu, scol, src) : -1;
    }
#pragma unroll
    for (int h = 0; h < 2; h++)
      if (kcol[h] >= 0 && !taken[h]) bound = fmax(bound, sb_key(khi[h], klo[h]));
    bound = warp_max(bound);
    if (lane == 0) sh.redmax[warp] = bound;  // (read after the first step's barrier)
#pragma unroll
    for (int r = 0; r < SC; r++) {
      if (act[r]) {
        const unsigned long long* sp = p.cand + (int64_t)sel_slot[r] * SLOTW + 6;
        unsigned long long ra[RPL], rb[RPL];
        for (unsigned spins = 0;; spins++) {
          bool okk = true;
#pragma unroll
          for (int k = 0; k < RPL; k++) ld_ll2(sp + 2 * (lane + 32 * k), ra[k], rb[k]);
#pragma unroll
          for (int k = 0; k < RPL; k++) okk = okk && (unsigned)ra[k] == cstamp && (unsigned)rb[k] == cstamp;
          if (okk) break;
          if (spins > (1u << 25)) __trap();
        }
#pragma unroll
        for (int k = 0; k < RPL; k++) x[r][k] = sb_double(ra[k], rb[k]);
      } else {
#pragma unroll
        for (int k = 0; k < RPL; k++) x[r][k] = 0.0;
      }
    }
    const long long tc2 = clock64();
    cyc_hdr += tc1 - tc0;
    cyc_load += tc2 - tc1;
    // ---- greedy steps while provable ----
    double thr = -1.0;
    for (int tt = 0;; tt++) {
      const int kj = j >> 5, jl = j & 31;
      // keys (rows >= j) and tails (rows > j) of the exact set, one butterfly for both
      double t[2 * SC];
#pragma unroll
      for (int r = 0; r < SC; r++) {
        double a = 0.0, b = 0.0;
#pragma unroll
        for (int k = 0; k < RPL; k++) {
          const int i = lane + 32 * k;
          const double v = (i >= j) ? x[r][k] : 0.0, w = (i > j) ? x[r][k] : 0.0;
          a = fma(v, v, a);
          b = fma(w, w, b);
        }
        t[2 * r] = a;
        t[2 * r + 1] = b;
      }
      warp_sum_all<2 * SC, 0, 2 * SC>(t, lane);
      double bkey = -1.0, btail = 0.0;
      int bpos = INT_MAX, br = -1;
#pragma unroll
      for (int r = 0; r < SC; r++) {
        if (act[r] && (br < 0 || piv_better(t[2 * r], pos[r], bkey, bpos))) {
          bkey = t[2 * r];
          btail = t[2 * r + 1];
          bpos = pos[r];
          br = r;
        }
      }
      // stage this warp's best column with the reflector it would give (as sweep.cu's kernels)
      const int par = tt & 1;
      SbStage<WARPS, NR>& sg = stage[par];
      {
        double sel = 0.0;
        int bcol = -1;
#pragma unroll
        for (int r = 0; r < SC; r++) {
          if (r == br) {
            bcol = col[r];
#pragma unroll
            for (int k = 0; k < RPL; k++) {
              sg.colv[warp][lane + 32 * k] = x[r][k];
              if (k == kj) sel = x[r][k];
            }
          }
        }
        const double xj = __shfl_sync(0xffffffffu, sel, jl);
        const bool refl = br >= 0 && (p.m - j >= 2) && (bkey != 0.0);
        const double nrm = sqrt(fmax(bkey, 0.0));
        const double beta = (xj >= 0.0) ? -nrm : nrm;
        const double h = beta - xj;
        const double inv = refl ? 1.0 / sqrt(h * h + btail) : 0.0;
        if (lane == 0) {
          const unsigned long long kb = (unsigned long long)__double_as_longlong(br < 0 ? 0.0 : bkey);
          sg.hi[warp] = (unsigned)(kb >> 32);
          sg.lo[warp] = (unsigned)kb;
          sg.pos[warp] = bpos;
          sg.col[warp] = bcol;
          sg.inv[warp] = inv;
          sg.hinv[warp] = h * inv;
        }
      }
      __syncthreads();
      if (tt == 0) {
        double umax = -1.0;
#pragma unroll
        for (int w = 0; w < WARPS; w++) umax = fmax(umax, sh.redmax[w]);
        thr = umax < 0.0 ? -1.0 : umax * (1.0 + 1e-10);
      }
      const bool lv = lane < WARPS;
      const unsigned rhi = lv ? sg.hi[lane] : 0u, rlo = lv ? sg.lo[lane] : 0u;
      const int rpos = lv ? sg.pos[lane] : INT_MAX, rcol = lv ? sg.col[lane] : -1;
      const int wl = warp_argmax(rhi, rlo, rpos, rcol >= 0);
      if (wl < 0 && tt == 0) __trap();  // more steps than columns (the launcher excludes it)
      const int src = wl < 0 ? 0 : wl;
      const double wkey = sb_key(__shfl_sync(0xffffffffu, rhi, src), __shfl_sync(0xffffffffu, rlo, src));
      const int wpos = __shfl_sync(0xffffffffu, rpos, src);
      const int wcol = __shfl_sync(0xffffffffu, rcol, src);
      const bool ok = wl >= 0 && (tt == 0 || (tt < SB_TMAX && wkey > thr));
      const unsigned es = p.stamp_base + e + 1u;
      unsigned long long* slot = p.ev + (int64_t)tt * (2 * (2 + NR));
      if (!ok) {
        if (tid == 0) {
          st_ll2(slot, ll_word(EV_END, es), ll_word((unsigned)j, es));
          st_ll2(slot + 2, ll_word(0u, es), ll_word(0u, es));
        }
        e++;
        break;
      }
      const bool last = j == p.steps - 1;
      const double inv = sg.inv[src], hinv = sg.hinv[src];
      const unsigned type = last ? EV_DONE : (inv != 0.0 ? EV_REFL : EV_PIVOT);
      double uk[RPL];
      {
        double cvv[RPL];
#pragma unroll
        for (int k = 0; k < RPL; k++) cvv[k] = sg.colv[src][lane + 32 * k];  // (all loads first: no branches)
        const double ninv = type == EV_REFL ? -inv : 0.0, hv = type == EV_REFL ? hinv : 0.0;
#pragma unroll
        for (int k = 0; k < RPL; k++) {
          const int i = lane + 32 * k;
          const double v = cvv[k] * ninv;
          uk[k] = (i == j) ? hv : ((i > j && i < p.m) ? v : 0.0);
        }
      }
      // publish: warp w stores the reflector's row slots k = w, w + WARPS, ...; warp 0 the header
      if (type == EV_REFL) {
#pragma unroll
        for (int k = 0; k < RPL; k++)
          if (k % WARPS == warp) sb_put_double(slot + 2 * (2 + lane + 32 * k), uk[k], es);
      }
      if (tid == 0) {
        st_ll2(slot, ll_word(type, es), ll_word((unsigned)j, es));
        st_ll2(slot + 2, ll_word((unsigned)wcol, es), ll_word((unsigned)wpos, es));
        p.chosen[j] = wcol;
      }
      e++;
      if (last) {
        j++;
        break;
      }
#pragma unroll
      for (int r = 0; r < SC; r++) {
        if (warp == wl && r == br) act[r] = false;
        else if (act[r] && pos[r] == j) pos[r] = wpos;
      }
      if (type == EV_REFL) sb_apply<RPL, SC>(x, uk, lane);
      j++;
    }
    cyc_steps += clock64() - tc2;
  }
  if (p.dbg && tid == 0)
    printf("sketch_batch: n=%d steps=%d batches=%d events=%u cycles: headers %lld load %lld steps %lld\n", p.n, p.steps,
           nbatch, e, cyc_hdr, cyc_load, cyc_steps);
}

template <int RPL, int CPW, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) sketch_batch_kernel(const SbArgs p) {
  __shared__ SbShared<RPL, WARPS> sh;
  extern __shared__ double sb_dyn[];
  if (blockIdx.x == 0) {
    sb_solver<RPL, kSbSolverCpw, WARPS>(p, sh, reinterpret_cast<SbStage<WARPS, 32 * RPL>*>(sb_dyn));
  } else {
    double* xs = sb_dyn;
    int* spos = reinterpret_cast<int*>(sb_dyn + (int64_t)WARPS * p.spw * 32 * RPL);
    int* sact = spos + WARPS * p.spw;
    sb_worker<RPL, CPW, WARPS>(p, sh, xs, spos, sact);
  }
}

constexpr int kSbWarps = 8;
constexpr int sb_cpw(int rpl) { return rpl >= 9 ? 9 : 10; }  // register columns per warp (255-register budget)
constexpr size_t kSbMaxDyn = 190 * 1024;

template <int RPL>
int sb_launch(SbArgs a, int G, cudaStream_t st, int64_t* launches) {
  auto kern = sketch_batch_kernel<RPL, sb_cpw(RPL), kSbWarps>;
  const size_t dyn = std::max((size_t)kSbWarps * a.spw * (32 * RPL * sizeof(double) + 2 * sizeof(int)),
                              2 * sizeof(SbStage<kSbWarps, 32 * RPL>));  // workers' columns / the solver's stage
  static bool attr = false;
  if (!attr) {
    RQ_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSbMaxDyn));
    attr = true;
  }
  void* args[] = {(void*)&a};
  RQ_CUDA_TRY(cudaLaunchCooperativeKernel((void*)kern, dim3(G), dim3(kSbWarps * 32), args, dyn, st));
  if (launches) (*launches)++;
  return RQ_OK;
}

int sb_rpl(int m) { return m <= 96 ? 3 : (m <= 160 ? 5 : 9); }

// Workers and shared-memory columns per warp for n columns on at most gmax CTAs; false = does not fit.
bool sb_plan(int m, int n, int gmax, int* G, int* per, int* spw) {
  if (m > 288 || n < 1) return false;
  if (gmax <= 0 || gmax > kSMs) gmax = kSMs;
  const int rpl = sb_rpl(m);
  int nw = std::min(gmax - 1, (n + 3) / 4);
  if (nw < 1) nw = 1;
  const int pr = (n + nw - 1) / nw;
  const int cpw = (pr + kSbWarps - 1) / kSbWarps;
  const int sp = std::max(0, cpw - sb_cpw(rpl));
  if ((size_t)kSbWarps * sp * (32 * rpl * sizeof(double) + 2 * sizeof(int)) > kSbMaxDyn) return false;
  *G = (n + pr - 1) / pr + 1;
  *per = pr;
  *spw = sp;
  return true;
}

}  // namespace

size_t sketch_batch_workspace_bytes() {
  return (size_t)2 * kSMs * 2 * (3 + 288) * 8 + (size_t)(SB_TMAX + 1) * 2 * (2 + 288) * 8 + 256;
}

bool sketch_batch_fits(int m, int n, int steps, int gmax) {
  int G, per, spw;
  return steps >= 1 && steps <= n && steps < m && sb_plan(m, n, gmax, &G, &per, &spw);
}

// chosen[0..steps) = the greedy CPQR pivots of y (m x n), y untouched.  ws: zero-initialised at
// allocation, sketch_batch_workspace_bytes(), private to the context; stamp_base advances by the
// events a launch can use.  Returns -1 when the shape does not fit (caller falls back).
int sketch_batch_launch(const double* y, int64_t ld, int m, int n, int steps, const int* init_pos, int* chosen,
                        void* ws, unsigned long long& stamp_base, cudaStream_t st, int64_t* launches, int gmax) {
  int G, per, spw;
  if (!(steps >= 1 && steps <= n && steps < m) || !sb_plan(m, n, gmax, &G, &per, &spw)) return -1;
  SbArgs a{};
  a.y = y;
  a.ld = ld;
  a.m = m;
  a.n = n;
  a.steps = steps;
  a.init_pos = init_pos;
  a.chosen = chosen;
  a.cand = reinterpret_cast<unsigned long long*>(ws);
  a.ev = a.cand + (size_t)2 * kSMs * 2 * (3 + 288);
  a.stamp_base = (unsigned)stamp_base;
  a.per = per;
  a.spw = spw;
  static const int env_dbg = getenv("RQ_SB_DBG") ? atoi(getenv("RQ_SB_DBG")) : 0;
  a.dbg = env_dbg;
  stamp_base += 2ull * (unsigned long long)steps + 2ull;
  const int rpl = sb_rpl(m);
  if (rpl == 3) return sb_launch<3>(a, G, st, launches);
  if (rpl == 5) return sb_launch<5>(a, G, st, launches);
  return sb_launch<9>(a, G, st, launches);
}

}  // namespace rq
