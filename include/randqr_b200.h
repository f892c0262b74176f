/*
 * randqr_b200.h -- C ABI of librandqr_b200.so, the B200 (sm_100a) drop-in for
 * the HQRRP hot path of the reference package `randqr`
 * (/root/reference/pkg/src/randqr).
 *
 * Every entry point takes plain pointers and sizes.  Matrices are column-major
 * (Fortran order, as the reference's working copies: blocked.py:161) with an
 * explicit leading dimension; "d" pointers are device memory, "h" pointers are
 * host memory.  All work is enqueued on the context's CUDA stream.
 *
 * Return codes map 1:1 onto the reference's exceptions (errors.py:4-13):
 *   RQ_EDIM   -> DimensionError     (blocked.py:152-161, householder.py:177-178)
 *   RQ_EVALUE -> ValueError         (pivoting.py:97-98, :122-123, householder.py:177-178)
 *   RQ_ECONV  -> ConvergenceError   (svd.py:52-53)
 * rq_last_error() returns the message of the last failing call on this thread.
 */
#ifndef RANDQR_B200_H
#define RANDQR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  RQ_OK = 0,
  RQ_EDIM = 1,
  RQ_EVALUE = 2,
  RQ_ECONV = 3,
  RQ_ECUDA = 4,
  RQ_EINTERNAL = 5,
  RQ_EUNSUPPORTED = 6
};

enum { RQ_PIVOT_PERMUTATION = 0, RQ_PIVOT_REFLECTORS = 1 };

/* RQ_SKETCH_FRESH draws a new Omega per panel from the caller's stream, exactly
 * as build_sketch does (pivoting.py:100-101); RQ_SKETCH_DOWNDATE draws G once
 * and downdates Y = G A per panel (HQRRP); its pivots differ legitimately. */
enum { RQ_SKETCH_FRESH = 0, RQ_SKETCH_DOWNDATE = 1 };

typedef struct rq_ctx rq_ctx;
/* The compact factors of one factorization, detached from its context
 * (Factorization's q_transforms / p_transforms, blocked.py:122-149). */
typedef struct rq_factors rq_factors;

/* Mirrors BlockConfig (blocked.py:42-50) + SketchConfig (pivoting.py:28-51). */
typedef struct rq_config {
  int32_t block;       /* b  = BlockConfig.block                                  */
  int32_t oversample;  /* p  = SketchConfig.oversample                            */
  int32_t power;       /* q  = SketchConfig.power                                 */
  int32_t stabilize;   /* -1: None (on iff q >= 2), 0: off, 1: on                 */
  int32_t pivot_kind;  /* RQ_PIVOT_PERMUTATION | RQ_PIVOT_REFLECTORS              */
  int32_t rrqr;        /* 1: block_rrqr semantics (blocked.py:239-279)            */
  int32_t sketch_mode; /* RQ_SKETCH_FRESH | RQ_SKETCH_DOWNDATE                     */
  int32_t flags;       /* RQ_FLAG_* (0: defaults)                                  */
} rq_config;

/* rq_config.flags: RQ_FLAG_NO_LOOKAHEAD runs the downdated-sketch driver without
 * look-ahead (each panel's trailing update completes before the next panel's sketch
 * CPQR); results are identical, only the schedule differs. */
#define RQ_FLAG_NO_LOOKAHEAD 1
/* rq_config.flags: RQ_FLAG_TF32_UPDATE runs the trailing-update GEMMs (the dominant flops) at fp32
 * accuracy on the tcgen05 tensor cores (3xTF32, fp32 accumulation) instead of FP64 DMMA; panels,
 * sketches and pivot selection stay fp64.  The fp32 path of BASELINE cfg 3 (accuracy ~1e-6). */
#define RQ_FLAG_TF32_UPDATE 2

/* Called after each completed panel (the reference's `inspect` hook,
 * blocked.py:184-185, :215-216); the callee may call rq_snapshot(). */
typedef void (*rq_panel_cb)(int32_t panel, void* user);

const char* rq_version(void);
const char* rq_last_error(void);

/* Context: owns workspace, the stored compact factors of the last
 * factorization, and the stream (NULL = legacy default stream). */
int rq_ctx_create(rq_ctx** out, int32_t device, void* stream);
int rq_ctx_destroy(rq_ctx* ctx);
int rq_ctx_set_stream(rq_ctx* ctx, void* stream);
int rq_ctx_set_inspect(rq_ctx* ctx, rq_panel_cb cb, void* user);
/* Cap the grid of this context's GEMMs (rq_gemm, rq_gemm_f32, rq_panel_apply; 0 = whole GPU): a
 * context whose GEMMs run beside a 16-CTA cluster kernel of another stream leaves it its SMs. */
int rq_ctx_set_gemm_cap(rq_ctx* ctx, int32_t max_ctas);

/* block_qr / block_rrqr (blocked.py:175-219 / :239-279) on device memory.
 * dA (m x n, lda >= m) is overwritten with R (exact zeros below the diagonal).
 * *counter is the RngState counter (rng.py:21-26) and is advanced exactly as
 * the reference advances it.  dperm (n int64, may be NULL) receives the
 * composite permutation (A[:, perm] = A P) when pivots are permutations.
 * The Q and P factors stay in the context (see rq_form_q / rq_form_p). */
int rq_factorize(rq_ctx* ctx, const rq_config* cfg, int64_t m, int64_t n, double* dA,
                 int64_t lda, uint64_t seed, uint64_t* counter, int64_t* dperm);

/* Same, end to end from host buffers (copies in and out on the ctx stream,
 * synchronises before returning).  hR may alias hA. */
int rq_factorize_host(rq_ctx* ctx, const rq_config* cfg, int64_t m, int64_t n, const double* hA,
                      int64_t lda, uint64_t seed, uint64_t* counter, double* hR, int64_t ldr,
                      int64_t* hperm);

/* Factorization.expand_q(cols) (blocked.py:134-141): dQ is m x cols, cols in [n, m]. */
int rq_form_q(rq_ctx* ctx, int64_t cols, double* dQ, int64_t ldq);
/* Factorization.expand_p() (blocked.py:143-149): dP is n x n. */
int rq_form_p(rq_ctx* ctx, double* dP, int64_t ldp);

/* Ownership of a factorization's factors (blocked.py:122-149: each Factorization owns its
 * transforms).  rq_factors_detach moves the context's stored factors -- and the device
 * workspace they live in -- into a new rq_factors; the context's next factorization then
 * reserves fresh workspace, so the detached factors stay valid until rq_factors_destroy.
 * rq_factors_form_q / _form_p are rq_form_q / rq_form_p on detached factors (enqueued on
 * ctx's stream; ctx must be on the device the factors live on). */
int rq_factors_detach(rq_ctx* ctx, rq_factors** out);
int rq_factors_destroy(rq_factors* f);
int rq_factors_form_q(rq_ctx* ctx, const rq_factors* f, int64_t cols, double* dQ, int64_t ldq);
int rq_factors_form_p(rq_ctx* ctx, const rq_factors* f, double* dP, int64_t ldp);

/* Per-panel transforms (Factorization.q_transforms / p_transforms, blocked.py:77-119), for
 * detached factors f or, with f = NULL, the context's stored factorization.
 * rq_factors_info: which = 0 lists the left factors (offset s_i, reflector count), which = 1 the
 * orthogonal right factors of reflector pivots (offset, width n - s_i; 0 entries for
 * permutation pivots, whose per-panel orders follow from the composite permutation);
 * *count receives the number of factors, the first min(count, cap) are written.
 * rq_apply_q: X (m x cols) <- U_first ... U_{first+count-1} X (trans = 0) or its transpose
 * applied (trans = 1), U_i = (I - V T V^T) diag(Q2, I) on rows s_i.. (QTransform.left_multiply).
 * rq_apply_p: X (rows x n) <- X P_first ... P_{first+count-1} (RightTransform.right_multiply;
 * reflector pivots only). */
int rq_factors_info(rq_ctx* ctx, const rq_factors* f, int32_t which, int32_t cap, int64_t* offsets,
                    int32_t* widths, int32_t* count);
int rq_apply_q(rq_ctx* ctx, const rq_factors* f, int32_t first, int32_t count, int32_t trans, int64_t cols,
               double* dX, int64_t ldx);
int rq_apply_p(rq_ctx* ctx, const rq_factors* f, int32_t first, int32_t count, int64_t rows, double* dX,
               int64_t ldx);

/* Working matrix after the current panel, in the reference's column order
 * (the matrix `inspect` receives).  Host destination, m x n, ldh >= m. */
int rq_snapshot(rq_ctx* ctx, double* hW, int64_t ldh);
/* Test hook for the HQRRP downdate (RQ_SKETCH_DOWNDATE, inside the inspect callback): the
 * downdated sketch of the trailing block, (b+p) x (n - s) into hY (ldh >= b+p), and the
 * composite permutation so far (n entries, A[:, perm] = A P) into hperm; reference order. */
int rq_snapshot_sketch(rq_ctx* ctx, double* hY, int64_t ldh, int64_t* hperm);

/* Kernel-plugin level (backend.get_kernels(), backend.py:42-47):
 * householder_sweep(a, v, perm, steps, pivot) (_kernels_numpy.py:11-22) on
 * device memory.  dV (m x steps) must be zero and dperm (n) the identity on
 * entry, as in the reference contract. */
int rq_householder_sweep(rq_ctx* ctx, double* dA, int64_t m, int64_t n, int64_t lda, double* dV,
                         int64_t ldv, int64_t* dperm, int64_t steps, int32_t pivot);

/* gaussian_matrix(rows, cols, RngState(seed, counter)) (rng.py:54-68) into
 * device memory; the caller advances its counter by rows*cols. */
int rq_gaussian_matrix(rq_ctx* ctx, int64_t rows, int64_t cols, uint64_t seed, uint64_t counter,
                       double* dOut, int64_t ld);

/* Plain splitmix64 words (rng.py:29-39) for the bitwise integer-stream pin. */
int rq_splitmix_words(rq_ctx* ctx, uint64_t seed, uint64_t first, int64_t count, uint64_t* dOut);

/* Unpivoted blocked Householder QR in place (qr_unpivoted, householder.py:152-161;
 * reflector convention householder.py:55-69), in blocks of `block` columns; m >= n.
 * dA becomes R; the factors are kept in the context for rq_form_q (Q) -- the
 * device-side haar_orthonormal of matrices.py:34-41 is built on it. */
int rq_qr_unpivoted(rq_ctx* ctx, int64_t m, int64_t n, double* dA, int64_t lda, int32_t block);

/* Frobenius truncation errors at scale (metrics.truncation_errors, metrics.py:37-52, without
 * dense expansion): A P = Q R gives ||A - Q(:,1:k) R(1:k,:) P^T||_F = ||R(k:, k:)||_F, so for the
 * n x n upper-triangular block dR this writes dE2[k] = ||R(k:, k:)||_F^2, k = 0..n (n+1 values). */
int rq_trailing_frobenius(rq_ctx* ctx, const double* dR, int64_t n, int64_t ldr, double* dE2);
/* Spectral truncation errors (metrics.truncation_errors, metrics.py:37-52; core.spectral_norm is the
 * largest singular value, core.py:39-46): hOut[i] = ||R(k:, k:)||_2 for k = hks[i] (host arrays),
 * via the Jacobi SVD kernel when n - k <= 512 (hHow[i] = 0), else power iteration on R22^T R22 to a
 * relative change below 1e-13 (hHow[i] = 1); hHow[i] = 2 for k = n.  Synchronous. */
int rq_trailing_spectral(rq_ctx* ctx, const double* dR, int64_t n, int64_t ldr, const int64_t* hks, int32_t nks,
                         double* hOut, int32_t* hHow);

/* ---- Panel-step API: one HQRRP panel at a time on caller-owned device buffers.
 * Used by a driver that owns the column distribution (paper_1505_08115_b200/dist.py,
 * 1-D block-cyclic columns over ranks).  The pieces are those of
 * block_qr's panel loop (blocked.py:175-219): pivot selection (pivoting.py:114-129),
 * qr_tall_pivoted (householder.py:183-198) and the trailing update
 * (householder.py:105-114).  Buffers: column-major, even leading dimensions,
 * 16-byte aligned bases. */

/* C (M x N) = alpha op(A) B + beta C, op(A) = A^T (A is K x M, a_mmajor = 0) or A
 * (A is M x K, a_mmajor = 1); B is K x N.  Views start at element (r0, c0) of
 * buffers with rows x cols extents (FP64 DMMA GEMM). */
/* Panel step (multi-GPU downdated sketch): X = R^{-1} for the k x k upper-triangular R
 * (k <= 512), on the context's stream. */
int rq_trinv_upper(rq_ctx* ctx, const double* dR, int64_t ldr, int32_t k, double* dX, int64_t ldx);

/* fp32 GEMM on the tcgen05 tensor cores (3xTF32 split products, FP32 accumulation in TMEM, TMA
 * staging; the fp32 path's sketch, trailing update and Q formation): the same operands and views
 * as rq_gemm with fp32 buffers, ld % 4 == 0 and 16-byte aligned bases. */
int rq_gemm_f32(rq_ctx* ctx, int32_t a_mmajor, int64_t M, int64_t N, int64_t K, const float* dA, int64_t lda,
                int64_t a_rows, int64_t a_cols, int64_t a_r0, int64_t a_c0, const float* dB, int64_t ldb,
                int64_t b_rows, int64_t b_cols, int64_t b_r0, int64_t b_c0, float* dC, int64_t ldc, double alpha,
                double beta);

int rq_gemm(rq_ctx* ctx, int32_t a_mmajor, int64_t M, int64_t N, int64_t K, const double* dA, int64_t lda,
            int64_t a_rows, int64_t a_cols, int64_t a_r0, int64_t a_c0, const double* dB, int64_t ldb, int64_t b_rows,
            int64_t b_cols, int64_t b_r0, int64_t b_c0, double* dC, int64_t ldc, double alpha, double beta);

/* select_pivot_permutation on a sketch Y (m x n, destroyed): the steps columns a
 * column-pivoted QR of Y picks, in order (dChosen, column indices of Y).  dInitPos
 * (n, or null = 0..n-1) is each column's logical position: ties go to the lower one. */
int rq_sketch_select(rq_ctx* ctx, double* dY, int64_t ldy, int32_t m, int32_t n, int32_t steps,
                     const int32_t* dInitPos, int32_t* dChosen);

/* qr_tall_pivoted of the panel dP (mp x b, mp >= b): unpivoted leaf QR, then a
 * column-pivoted QR of the b x b R'.  On return dP holds R (b x b upper, columns in
 * P-hat order; zero below), dV the panel reflectors (mp x b, unit u with
 * H = I - 2uu^T), dT their compact-WY T (b x b), dQ2 the b x b orthogonal factor of
 * the second stage and dPhat[t] the panel column now at position t. */
int rq_panel_factor(rq_ctx* ctx, double* dP, int64_t ldp, int64_t mp, int32_t b, double* dV, int64_t ldv, double* dT,
                    int64_t ldt, double* dQ2, int64_t ldq2, int32_t* dPhat);

/* Trailing update of an mp x n2 block at (r0, c0) of dA (a_rows x a_cols buffer):
 * A2 <- (I - V T V^T)^T A2, then its top b rows <- Q2^T (top b rows); dQ2 may be null. */
int rq_panel_apply(rq_ctx* ctx, const double* dV, int64_t ldv, const double* dT, int64_t ldt, const double* dQ2,
                   int64_t ldq2, int64_t mp, int32_t b, double* dA, int64_t lda, int64_t a_rows, int64_t a_cols,
                   int64_t r0, int64_t c0, int64_t n2);

/* Test hook: the FP64 DMMA GEMM used by every dense step,
 *   C (M x N) = alpha * op(A) * B + beta * C,  op(A) = A^T (A is K x M, a_mmajor = 0)
 *   or A (A is M x K, a_mmajor = 1); B is K x N.  Views start at element
 *   (a_r0, a_c0) / (b_r0, b_c0) of buffers with a_rows x a_cols / b_rows x b_cols
 *   extents.  Leading dimensions must be even, buffers 16 B aligned. */
int rq_test_gemm(rq_ctx* ctx, int32_t a_mmajor, int64_t M, int64_t N, int64_t K, const double* dA, int64_t lda,
                 int64_t a_rows, int64_t a_cols, int64_t a_r0, int64_t a_c0, const double* dB, int64_t ldb,
                 int64_t b_rows, int64_t b_cols, int64_t b_r0, int64_t b_c0, double* dC, int64_t ldc, double alpha,
                 double beta);

/* Test hooks for the serial kernels (microbenchmarks and parity tests):
 * sketch CPQR pivot selection on dY (m x n, destroyed) -> dChosen[steps];
 * panel leaf QR of dA (mm x w, w <= 32) -> R in place, dV (mm x w), dT (w x w). */
int rq_test_sketch_cpqr(rq_ctx* ctx, double* dY, int64_t ld, int32_t m, int32_t n, int32_t steps, int32_t* dChosen);
int rq_test_leaf_qr(rq_ctx* ctx, double* dA, int64_t lda, int64_t mm, int32_t w, double* dV, int64_t ldv,
                    double* dT, int64_t ldt);
/* Test hook: A (mm x nr) <- A - V T^T (V^T A) for one leaf's w <= 16 reflectors V (mm x w) and
 * T (w x w): cluster != 0 runs the 16-CTA cluster kernel (space-sliced look-ahead), 0 the
 * whole-GPU cooperative kernel. */
int rq_test_wy_update(rq_ctx* ctx, int32_t cluster, double* dA, int64_t lda, int64_t mm, int32_t nr, const double* dV,
                      int64_t ldv, const double* dT, int64_t ldt, int32_t w);

/* Test hook: per-phase clock64 stamps of the cluster sweep (first 64 steps, 8 per step). */
int rq_test_debug_timing(int32_t on, uint64_t* host, int32_t count);

/* Number of kernel launches this context has issued (instrumentation). */
int64_t rq_launch_count(rq_ctx* ctx);

/* Instrumentation: with profiling on, CUDA events bracket every launch of a
 * kernel class (0 trailing-update GEMMs, 1 other GEMMs, 2 sketch CPQR, 3 panel leaves, 4 other,
 * 5 b x b CPQR, 6 sketch GEMMs, 7 panel WY GEMMs, 8 T factors, 9-12 below); rq_profile_read sums their device time (ms) and
 * GEMM flops since the last rq_set_profiling call. */
int rq_set_profiling(rq_ctx* ctx, int32_t on);
int rq_profile_read(rq_ctx* ctx, int32_t category, double* ms, double* flops, int64_t* count);
/* Bandwidth classes (9 column moves, 10 copy2d, 11 Gaussian fills, 12 GEMM split-K reductions):
 * algorithmic HBM bytes moved since the last rq_set_profiling (pair with rq_profile_read's ms). */
int rq_profile_bytes(rq_ctx* ctx, int32_t category, double* bytes);

#ifdef __cplusplus
}
#endif

#endif /* RANDQR_B200_H */
