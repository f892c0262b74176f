// K11: one-sided Jacobi SVD of the w x w panel triangle (block_rrqr's panel_svd,
// blocked.py:222-236 -> svd_full, svd.py:68-91 -> jacobi_sweeps,
// _kernels_numba.py:64-104).
//
// The reference sweeps the pairs (p, q), p < q, in cyclic row order; each
// rotation touches only columns p and q.  Rotation (p, q) therefore depends on
// exactly (p, q-1) and (p-1, q), and all rotations with p + q = t form a
// "wave" of disjoint column pairs.  Executing the waves t = 1 .. 2w-3 in order
// applies, to every column, the same rotations in the same order as the
// sequential sweep -- so the singular vectors come out with the reference's
// orientation -- with ~2w synchronisations per sweep instead of w^2/2 steps.
// The per-pair skip rules, tau/t/c/s formulas, the sq[] bookkeeping, the
// 1e-14 tolerance, the 60-sweep limit (-> ConvergenceError), the stable
// descending sort and the zero-singular-value completion (_fill_orthonormal)
// follow the reference.
//
// svd_full first takes an unpivoted QR of its (here upper-triangular) input;
// on a triangle each reflector is +-e_j, i.e. W = D R' with D_jj = -1 for
// j < w-1, R'_jj != 0 (exactly), and U' = D u_small.
#include <cstdlib>

#include "common.cuh"
#include "misc.cuh"

namespace rq {

constexpr int JC_THREADS = 1024;

RQ_DEV int dsmem_i32_jc(const int* local, unsigned rank) {
  int v;
  asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(cluster_map(smem_u32(local), rank)));
  return v;
}
constexpr int JC_GROUP = 16;  // threads per rotation pair
constexpr int JC_PAIRS = JC_THREADS / JC_GROUP;

struct JacobiArgs {
  const double* r;  // w x w upper triangle (ldr)
  int64_t ldr;
  int w;
  double* wbuf;     // w x w working matrix (global fallback, ldw)
  int64_t ldw;
  double* vbuf;     // w x w accumulated rotations (ldv)
  int64_t ldv;
  double* d;        // w singular values (non-increasing)
  double* u;        // w x w left vectors U' (ldu)
  int64_t ldu;
  double* vt;       // w x w right vectors V~ (ldvt), columns in d order
  int64_t ldvt;
  int* status;      // sweeps used, or -1 (no convergence)
  int use_smem;
  double rel_tol;
  int max_sweeps;
};

RQ_DEV double group_sum16(double v) {
  v += __shfl_xor_sync(0xffffffffu, v, 8);
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v;
}

__global__ void __launch_bounds__(JC_THREADS, 1) jacobi_wave_kernel(const JacobiArgs p) {
  extern __shared__ double sm[];
  const int w = p.w;
  double* sq = sm;                               // w
  double* W = p.use_smem ? sm + w : p.wbuf;      // column-major, ld = ldW
  const int64_t ldW = p.use_smem ? w : p.ldw;
  double* V = p.vbuf;
  __shared__ int rot_any;
  __shared__ int cand_s;
  __shared__ int rank_tmp[512];

  // W = D R' (see header); V = I
  for (int64_t idx = threadIdx.x; idx < (int64_t)w * w; idx += JC_THREADS) {
    const int c = (int)(idx / w), i = (int)(idx % w);
    double x = (i <= c) ? p.r[(int64_t)c * p.ldr + i] : 0.0;
    const double rii = p.r[(int64_t)i * p.ldr + i];
    if (i < w - 1 && rii != 0.0) x = -x;
    W[(int64_t)c * ldW + i] = x;
    V[(int64_t)c * p.ldv + i] = (i == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int grp = threadIdx.x / JC_GROUP, gl = threadIdx.x % JC_GROUP;
  int sweeps_used = -1;
  for (int sweep = 0; sweep < p.max_sweeps; sweep++) {
    for (int c = threadIdx.x; c < w; c += JC_THREADS) {
      double acc = 0.0;
      for (int i = 0; i < w; i++) acc += W[(int64_t)c * ldW + i] * W[(int64_t)c * ldW + i];
      sq[c] = acc;
    }
    if (threadIdx.x == 0) rot_any = 0;
    __syncthreads();
    for (int t = 1; t <= 2 * w - 3; t++) {
      const int plo = t - (w - 1) > 0 ? t - (w - 1) : 0;
      const int phi = (t - 1) / 2;  // p < q = t - p
      const int npairs = phi - plo + 1;
      // uniform trip count: every lane reaches the group shuffles
      for (int base = 0; base < npairs; base += JC_PAIRS) {
        const int pp = plo + base + grp;
        const bool live = (base + grp) < npairs;
        const int q = t - pp;
        const double app = live ? sq[pp] : 0.0, aqq = live ? sq[q] : 0.0;
        const bool go = live && app != 0.0 && aqq != 0.0;
        double* cp = W + (int64_t)(go ? pp : 0) * ldW;
        double* cq = W + (int64_t)(go ? q : 0) * ldW;
        double apq = 0.0;
        if (go)
          for (int i = gl; i < w; i += JC_GROUP) apq += cp[i] * cq[i];
        apq = group_sum16(apq);
        if (!go || fabs(apq) <= p.rel_tol * sqrt(app * aqq)) continue;  // group-uniform from here on
        const double tau = (aqq - app) / (2.0 * apq);
        const double tt = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
        const double c_ = 1.0 / sqrt(1.0 + tt * tt);
        const double s_ = tt * c_;
        for (int i = gl; i < w; i += JC_GROUP) {
          const double ap = cp[i];
          cp[i] = c_ * ap - s_ * cq[i];
          cq[i] = s_ * ap + c_ * cq[i];
        }
        double* vp = V + (int64_t)pp * p.ldv;
        double* vq = V + (int64_t)q * p.ldv;
        for (int i = gl; i < w; i += JC_GROUP) {
          const double x = vp[i];
          vp[i] = c_ * x - s_ * vq[i];
          vq[i] = s_ * x + c_ * vq[i];
        }
        if (gl == 0) {
          sq[pp] = app - tt * apq;
          sq[q] = aqq + tt * apq;
          rot_any = 1;
        }
      }
      __syncthreads();
    }
    if (!rot_any) {
      sweeps_used = sweep + 1;
      break;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *p.status = sweeps_used;
  if (sweeps_used < 0) return;
  // norms, stable descending order (argsort(-norms, kind="stable"))
  for (int c = threadIdx.x; c < w; c += JC_THREADS) {
    double acc = 0.0;
    for (int i = 0; i < w; i++) acc += W[(int64_t)c * ldW + i] * W[(int64_t)c * ldW + i];
    sq[c] = sqrt(acc);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < w; c += JC_THREADS) {
    int rk = 0;
    for (int c2 = 0; c2 < w; c2++) rk += (sq[c2] > sq[c]) || (sq[c2] == sq[c] && c2 < c);
    rank_tmp[rk] = c;  // order[rk] = c
  }
  __syncthreads();
  for (int j = threadIdx.x; j < w; j += JC_THREADS) p.d[j] = sq[rank_tmp[j]];
  for (int64_t idx = threadIdx.x; idx < (int64_t)w * w; idx += JC_THREADS) {
    const int j = (int)(idx / w), i = (int)(idx % w);
    const int col = rank_tmp[j];
    const double dj = sq[col];
    const double us = dj > 0.0 ? W[(int64_t)col * ldW + i] / dj : 0.0;
    const double rii = p.r[(int64_t)i * p.ldr + i];
    p.u[(int64_t)j * p.ldu + i] = (i < w - 1 && rii != 0.0) ? -us : us;  // U' = D u_small
    p.vt[(int64_t)j * p.ldvt + i] = V[(int64_t)col * p.ldv + i];
  }
  __syncthreads();
  // zero singular values: orthonormal completion as _fill_orthonormal (svd.py:57-65)
  for (int j = 0; j < w; j++) {
    if (p.d[j] > 0.0) continue;  // d is final here; sq is reused as scratch below
    // resid = I - U U^T (current U, including the zero column j); cand = argmax column norm
    double* U = p.u;
    for (int c = threadIdx.x; c < w; c += JC_THREADS) {
      double nrm = 0.0;
      for (int i = 0; i < w; i++) {
        double ri = (i == c) ? 1.0 : 0.0;
        for (int k = 0; k < w; k++) ri -= U[(int64_t)k * p.ldu + i] * U[(int64_t)k * p.ldu + c];
        nrm += ri * ri;
      }
      sq[c] = nrm;  // sq is free after the sort bookkeeping (d already written)
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int cand = 0;
      for (int c = 1; c < w; c++)
        if (sq[c] > sq[cand]) cand = c;
      cand_s = cand;
    }
    __syncthreads();
    const int cand = cand_s;
    // x = resid[:, cand]; x -= U (U^T x); u_j = x / ||x||  (single thread: w <= 512, rare path)
    if (threadIdx.x == 0) {
      double* x = W;  // scratch
      for (int i = 0; i < w; i++) {
        double ri = (i == cand) ? 1.0 : 0.0;
        for (int k = 0; k < w; k++) ri -= U[(int64_t)k * p.ldu + i] * U[(int64_t)k * p.ldu + cand];
        x[i] = ri;
      }
      for (int k = 0; k < w; k++) {
        double dot = 0.0;
        for (int i = 0; i < w; i++) dot += U[(int64_t)k * p.ldu + i] * x[i];
        for (int i = 0; i < w; i++) x[i] -= U[(int64_t)k * p.ldu + i] * dot;
      }
      double nx = 0.0;
      for (int i = 0; i < w; i++) nx += x[i] * x[i];
      nx = sqrt(nx);
      for (int i = 0; i < w; i++) U[(int64_t)j * p.ldu + i] = x[i] / nx;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Two-CTA cluster variant (w <= 128): CTA 0 keeps W in shared memory and runs the
// waves exactly as above; the rotations (c, s) of each wave stream to CTA 1 through
// an st.async ring (mbarrier complete_tx), and CTA 1 applies them, wave by wave in
// the same order, to V in its own shared memory.  V never touches global memory on
// the critical path and CTA 0 never waits for it (except for ring slots, 8 waves deep).
// Skipped pairs stream the exact identity (c, s) = (1, 0).
// ---------------------------------------------------------------------------
constexpr int J2_RING = 8;
constexpr int J2_PAIRS = 64;  // w <= 128: at most 64 disjoint pairs per wave
constexpr double J2_STOP = 2.0, J2_CONT = 1.0;

RQ_DEV void st_async_v2(uint32_t remote_addr, double a, double b, uint32_t remote_mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(remote_addr),
               "l"(__double_as_longlong(a)), "l"(__double_as_longlong(b)), "r"(remote_mbar)
               : "memory");
}
RQ_DEV void mbar_arrive_remote(uint32_t remote_mbar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_mbar) : "memory");
}

__global__ void __launch_bounds__(JC_THREADS, 1) jacobi_pair_kernel(const JacobiArgs p) {
  extern __shared__ double sm[];  // CTA 0: sq[w] then W (w x w); CTA 1: V (w x w)
  __shared__ __align__(16) double ring[J2_RING][J2_PAIRS + 1][2];  // CTA 1: [0] = {flag, -}, [1 + k] = {c, s}
  __shared__ __align__(8) unsigned long long full[J2_RING];        // CTA 1: message landed
  __shared__ __align__(8) unsigned long long empty[J2_RING];       // CTA 0: slot consumed
  __shared__ int rot_any;
  __shared__ int cand_s;
  __shared__ int rank_tmp[512];
  __shared__ int status_s;
  unsigned crank;
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  const int w = p.w;
  const int waves = 2 * w - 3;
  if (threadIdx.x == 0) {
    for (int k = 0; k < J2_RING; k++) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], 1);
    }
    mbar_init_fence();
  }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  const int grp = threadIdx.x / JC_GROUP, gl = threadIdx.x % JC_GROUP;
  if (crank == 0) {
    double* sq = sm;
    double* W = sm + w;
    const int64_t ldW = w;
    for (int64_t idx = threadIdx.x; idx < (int64_t)w * w; idx += JC_THREADS) {
      const int c = (int)(idx / w), i = (int)(idx % w);
      double x = (i <= c) ? p.r[(int64_t)c * p.ldr + i] : 0.0;
      const double rii = p.r[(int64_t)i * p.ldr + i];
      if (i < w - 1 && rii != 0.0) x = -x;
      W[(int64_t)c * ldW + i] = x;
    }
    __syncthreads();
    int sweeps_used = -1;
    long long g = 0;  // messages sent
    const uint32_t ring_r = cluster_map(smem_u32(&ring[0][0][0]), 1u);
    const uint32_t full_r = cluster_map(smem_u32(&full[0]), 1u);
    for (int sweep = 0; sweep < p.max_sweeps; sweep++) {
      for (int c = threadIdx.x; c < w; c += JC_THREADS) {
        double acc = 0.0;
        for (int i = 0; i < w; i++) acc += W[(int64_t)c * ldW + i] * W[(int64_t)c * ldW + i];
        sq[c] = acc;
      }
      if (threadIdx.x == 0) rot_any = 0;
      __syncthreads();
      for (int t = 1; t <= waves; t++, g++) {
        const int slot = (int)(g % J2_RING);
        const uint32_t slot_r = ring_r + (uint32_t)(slot * (J2_PAIRS + 1) * 16);
        const uint32_t mb_r = full_r + (uint32_t)(slot * 8);
        const int plo = t - (w - 1) > 0 ? t - (w - 1) : 0;
        const int phi = (t - 1) / 2;
        const int npairs = phi - plo + 1;
        const bool live = grp < npairs;
        if (g >= J2_RING && (threadIdx.x == 0 || (live && gl == 0)))
          mbar_wait_cluster(&empty[slot], (unsigned)((g / J2_RING) - 1) & 1u);
        const int pp = plo + grp;
        const int q = t - pp;
        const double app = live ? sq[pp] : 0.0, aqq = live ? sq[q] : 0.0;
        const bool go = live && app != 0.0 && aqq != 0.0;
        double* cp = W + (int64_t)(go ? pp : 0) * ldW;
        double* cq = W + (int64_t)(go ? q : 0) * ldW;
        double apq = 0.0;
        if (go)
          for (int i = gl; i < w; i += JC_GROUP) apq += cp[i] * cq[i];
        apq = group_sum16(apq);
        double c_ = 1.0, s_ = 0.0;
        const bool rot = go && !(fabs(apq) <= p.rel_tol * sqrt(app * aqq));
        double tt = 0.0;
        if (rot) {
          const double tau = (aqq - app) / (2.0 * apq);
          tt = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
          c_ = 1.0 / sqrt(1.0 + tt * tt);
          s_ = tt * c_;
          for (int i = gl; i < w; i += JC_GROUP) {
            const double ap = cp[i];
            cp[i] = c_ * ap - s_ * cq[i];
            cq[i] = s_ * ap + c_ * cq[i];
          }
        }
        if (live && gl == 0) {
          st_async_v2(slot_r + (uint32_t)((1 + grp) * 16), c_, s_, mb_r);
          if (rot) {
            sq[pp] = app - tt * apq;
            sq[q] = aqq + tt * apq;
            rot_any = 1;
          }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          const bool last = (t == waves) && (!rot_any || sweep == p.max_sweeps - 1);
          st_async_v2(slot_r, last ? J2_STOP : J2_CONT, 0.0, mb_r);
        }
      }
      if (!rot_any) {
        sweeps_used = sweep + 1;
        break;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      *p.status = sweeps_used;
      status_s = sweeps_used;
    }
    if (sweeps_used >= 0) {
      for (int c = threadIdx.x; c < w; c += JC_THREADS) {
        double acc = 0.0;
        for (int i = 0; i < w; i++) acc += W[(int64_t)c * ldW + i] * W[(int64_t)c * ldW + i];
        sq[c] = sqrt(acc);
      }
      __syncthreads();
      for (int c = threadIdx.x; c < w; c += JC_THREADS) {
        int rk = 0;
        for (int c2 = 0; c2 < w; c2++) rk += (sq[c2] > sq[c]) || (sq[c2] == sq[c] && c2 < c);
        rank_tmp[rk] = c;
      }
      __syncthreads();
      for (int j = threadIdx.x; j < w; j += JC_THREADS) p.d[j] = sq[rank_tmp[j]];
      for (int64_t idx = threadIdx.x; idx < (int64_t)w * w; idx += JC_THREADS) {
        const int j = (int)(idx / w), i = (int)(idx % w);
        const int col = rank_tmp[j];
        const double dj = sq[col];
        const double us = dj > 0.0 ? W[(int64_t)col * ldW + i] / dj : 0.0;
        const double rii = p.r[(int64_t)i * p.ldr + i];
        p.u[(int64_t)j * p.ldu + i] = (i < w - 1 && rii != 0.0) ? -us : us;
      }
      __syncthreads();
      for (int j = 0; j < w; j++) {
        if (p.d[j] > 0.0) continue;
        double* U = p.u;
        for (int c = threadIdx.x; c < w; c += JC_THREADS) {
          double nrm = 0.0;
          for (int i = 0; i < w; i++) {
            double ri = (i == c) ? 1.0 : 0.0;
            for (int k = 0; k < w; k++) ri -= U[(int64_t)k * p.ldu + i] * U[(int64_t)k * p.ldu + c];
            nrm += ri * ri;
          }
          sq[c] = nrm;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          int cand = 0;
          for (int c = 1; c < w; c++)
            if (sq[c] > sq[cand]) cand = c;
          cand_s = cand;
        }
        __syncthreads();
        const int cand = cand_s;
        if (threadIdx.x == 0) {
          double* x = W;
          for (int i = 0; i < w; i++) {
            double ri = (i == cand) ? 1.0 : 0.0;
            for (int k = 0; k < w; k++) ri -= U[(int64_t)k * p.ldu + i] * U[(int64_t)k * p.ldu + cand];
            x[i] = ri;
          }
          for (int k = 0; k < w; k++) {
            double dot = 0.0;
            for (int i = 0; i < w; i++) dot += U[(int64_t)k * p.ldu + i] * x[i];
            for (int i = 0; i < w; i++) x[i] -= U[(int64_t)k * p.ldu + i] * dot;
          }
          double nx = 0.0;
          for (int i = 0; i < w; i++) nx += x[i] * x[i];
          nx = sqrt(nx);
          for (int i = 0; i < w; i++) U[(int64_t)j * p.ldu + i] = x[i] / nx;
        }
        __syncthreads();
      }
    }
  } else {
    double* V = sm;
    const int64_t ldV = w;
    for (int64_t idx = threadIdx.x; idx < (int64_t)w * w; idx += JC_THREADS) {
      const int c = (int)(idx / w), i = (int)(idx % w);
      V[(int64_t)c * ldV + i] = (i == c) ? 1.0 : 0.0;
    }
    __syncthreads();
    const uint32_t empty_r = cluster_map(smem_u32(&empty[0]), 0u);
    long long g = 0;
    bool stop = waves <= 0;  // w <= 1: no rotations, nothing streams
    while (!stop) {
      for (int t = 1; t <= waves && !stop; t++, g++) {
        const int slot = (int)(g % J2_RING);
        const int plo = t - (w - 1) > 0 ? t - (w - 1) : 0;
        const int phi = (t - 1) / 2;
        const int npairs = phi - plo + 1;
        if (threadIdx.x == 0) mbar_expect_tx(&full[slot], (unsigned)(npairs + 1) * 16u);
        mbar_wait_cluster(&full[slot], (unsigned)(g / J2_RING) & 1u);
        if (grp < npairs) {
          const double c_ = ring[slot][1 + grp][0], s_ = ring[slot][1 + grp][1];
          if (!(c_ == 1.0 && s_ == 0.0)) {
            const int pp = plo + grp, q = t - pp;
            double* vp = V + (int64_t)pp * ldV;
            double* vq = V + (int64_t)q * ldV;
            for (int i = gl; i < w; i += JC_GROUP) {
              const double x = vp[i];
              vp[i] = c_ * x - s_ * vq[i];
              vq[i] = s_ * x + c_ * vq[i];
            }
          }
        }
        stop = ring[slot][0][0] == J2_STOP;
        __syncthreads();
        if (threadIdx.x == 0) mbar_arrive_remote(empty_r + (uint32_t)(slot * 8));
      }
    }
  }
  // CTA 1 writes V~ in the order CTA 0 sorted the singular values
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (crank == 1) {
    const int st = dsmem_i32_jc(&status_s, 0u);
    if (st >= 0) {
      const double* V = sm;
      for (int64_t idx = threadIdx.x; idx < (int64_t)w * w; idx += JC_THREADS) {
        const int j = (int)(idx / w), i = (int)(idx % w);
        const int col = dsmem_i32_jc(&rank_tmp[j], 0u);
        p.vt[(int64_t)j * p.ldvt + i] = V[(int64_t)col * w + i];
      }
    }
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

int jacobi_svd(const double* r, int64_t ldr, int w, double* wbuf, int64_t ldw, double* vbuf, int64_t ldv, double* d,
               double* u, int64_t ldu, double* vt, int64_t ldvt, int* status, cudaStream_t st, int64_t* launches) {
  if (w <= 0) return RQ_OK;
  if (w > 512) return set_error(RQ_EUNSUPPORTED, "panel SVD wider than 512");
  JacobiArgs a;
  a.r = r;
  a.ldr = ldr;
  a.w = w;
  a.wbuf = wbuf;
  a.ldw = ldw;
  a.vbuf = vbuf;
  a.ldv = ldv;
  a.d = d;
  a.u = u;
  a.ldu = ldu;
  a.vt = vt;
  a.ldvt = ldvt;
  a.status = status;
  a.rel_tol = 1e-14;   // svd.py:25
  a.max_sweeps = 60;   // svd.py:26
  const size_t smem_full = ((size_t)w + (size_t)w * w) * sizeof(double);
  a.use_smem = smem_full <= 200 * 1024 ? 1 : 0;
  const size_t smem = a.use_smem ? smem_full : (size_t)w * sizeof(double);
  static bool attr = false;
  if (!attr) {
    RQ_CUDA_TRY(cudaFuncSetAttribute(jacobi_wave_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  static const int env_j2 = [] {
    const char* e = getenv("RQ_JACOBI_PAIR");
    return e ? atoi(e) : 1;
  }();
  if (w <= 2 * J2_PAIRS && env_j2) {
    const size_t smem2 = ((size_t)w + (size_t)w * w) * sizeof(double);
    static bool attr2 = false;
    if (!attr2) {
      RQ_CUDA_TRY(cudaFuncSetAttribute(jacobi_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      attr2 = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2);
    cfg.blockDim = dim3(JC_THREADS);
    cfg.dynamicSmemBytes = smem2;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    RQ_CUDA_TRY(cudaLaunchKernelEx(&cfg, jacobi_pair_kernel, a));
    if (launches) (*launches)++;
    return RQ_OK;
  }
  jacobi_wave_kernel<<<1, JC_THREADS, smem, st>>>(a);
  RQ_CUDA_TRY(cudaGetLastError());
  if (launches) (*launches)++;
  return RQ_OK;
}

}  // namespace rq
