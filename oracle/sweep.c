/*
 * oracle/sweep.c -- TEST INFRASTRUCTURE ONLY (the CPU checker and the CPU
 * baseline).  Never linked into, or called by, the product path.
 *
 * Plain-C restatement of the reference's two inner kernels, following the
 * loop order of the numba twins so that summation order (and therefore
 * rounding) matches the reference's default backend:
 *
 *   oracle_householder_sweep  <- /root/reference/pkg/src/randqr/_kernels_numba.py:13-61
 *                                (contract: _kernels_numpy.py:11-22)
 *   oracle_jacobi_sweeps      <- /root/reference/pkg/src/randqr/_kernels_numba.py:64-104
 *                                (contract: _kernels_numpy.py:49-57; the numba
 *                                 twin is compiled with fastmath, so only the
 *                                 plain-C association is reproducible here)
 *
 * Matrices are column-major with an explicit leading dimension.
 */
#include <math.h>
#include <stdint.h>

#define AT(p, ld, i, j) ((p)[(int64_t)(j) * (ld) + (i)])

void oracle_householder_sweep(double *a, int64_t m, int64_t n, int64_t lda,
                              double *v, int64_t ldv, int64_t *perm,
                              int64_t steps, int pivot) {
  for (int64_t j = 0; j < steps; j++) {
    if (pivot) {
      /* norms recomputed from scratch; strict '>' keeps the lowest index */
      int64_t best = j;
      double best_sq = 0.0;
      for (int64_t c = j; c < n; c++) {
        const double *col = &AT(a, lda, 0, c);
        double sq = 0.0;
        for (int64_t i = j; i < m; i++) sq += col[i] * col[i];
        if (sq > best_sq) {
          best_sq = sq;
          best = c;
        }
      }
      if (best != j) {
        double *cj = &AT(a, lda, 0, j), *cb = &AT(a, lda, 0, best);
        for (int64_t i = 0; i < m; i++) {
          double t = cj[i];
          cj[i] = cb[i];
          cb[i] = t;
        }
        int64_t pt = perm[j];
        perm[j] = perm[best];
        perm[best] = pt;
      }
    }
    if (m - j < 2) continue; /* length-1 sub-column: no reflector */
    double *x = &AT(a, lda, 0, j);
    double normsq = 0.0;
    for (int64_t i = j; i < m; i++) normsq += x[i] * x[i];
    if (normsq == 0.0) continue; /* identity reflector, v stays zero */
    double norm = sqrt(normsq);
    double beta = x[j] >= 0.0 ? -norm : norm; /* sign(0) := +1 */
    double *u = &AT(v, ldv, 0, j);
    double usq = 0.0;
    for (int64_t i = j; i < m; i++) {
      double ui = (i == j) ? beta - x[i] : -x[i];
      u[i] = ui;
      usq += ui * ui;
    }
    double uinv = 1.0 / sqrt(usq);
    for (int64_t i = j; i < m; i++) u[i] *= uinv;
    for (int64_t c = j + 1; c < n; c++) {
      double *col = &AT(a, lda, 0, c);
      double s = 0.0;
      for (int64_t i = j; i < m; i++) s += u[i] * col[i];
      s *= 2.0;
      for (int64_t i = j; i < m; i++) col[i] -= s * u[i];
    }
    x[j] = beta;
    for (int64_t i = j + 1; i < m; i++) x[i] = 0.0;
  }
}

int oracle_jacobi_sweeps(double *a, int64_t m, int64_t n, int64_t lda,
                         double *v, int64_t ldv, double rel_tol,
                         int max_sweeps, int accumulate, double *sq) {
  int64_t vrows = accumulate ? n : 0;
  for (int sweep = 0; sweep < max_sweeps; sweep++) {
    for (int64_t c = 0; c < n; c++) {
      const double *col = &AT(a, lda, 0, c);
      double acc = 0.0;
      for (int64_t i = 0; i < m; i++) acc += col[i] * col[i];
      sq[c] = acc;
    }
    int rotated = 0;
    for (int64_t p = 0; p < n - 1; p++) {
      for (int64_t q = p + 1; q < n; q++) {
        double app = sq[p], aqq = sq[q];
        if (app == 0.0 || aqq == 0.0) continue;
        double *cp = &AT(a, lda, 0, p), *cq = &AT(a, lda, 0, q);
        double apq = 0.0;
        for (int64_t i = 0; i < m; i++) apq += cp[i] * cq[i];
        if (fabs(apq) <= rel_tol * sqrt(app * aqq)) continue;
        double tau = (aqq - app) / (2.0 * apq);
        double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
        double c_ = 1.0 / sqrt(1.0 + t * t);
        double s_ = t * c_;
        for (int64_t i = 0; i < m; i++) {
          double ap = cp[i];
          cp[i] = c_ * ap - s_ * cq[i];
          cq[i] = s_ * ap + c_ * cq[i];
        }
        if (accumulate) {
          double *vp = &AT(v, ldv, 0, p), *vq = &AT(v, ldv, 0, q);
          for (int64_t i = 0; i < vrows; i++) {
            double x = vp[i];
            vp[i] = c_ * x - s_ * vq[i];
            vq[i] = s_ * x + c_ * vq[i];
          }
        }
        sq[p] = app - t * apq;
        sq[q] = aqq + t * apq;
        rotated = 1;
      }
    }
    if (!rotated) return sweep + 1;
  }
  return -1;
}
