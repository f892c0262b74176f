// extern "C" entry points of librandqr_b200.so (declared in include/randqr_b200.h).
#include <algorithm>
#include <new>

#include "driver.cuh"
#include "gemm_tf32.cuh"
#include "misc.cuh"
#include "panel.cuh"

namespace rq {
const char* last_error();
void clear_error();
}  // namespace rq

using rq::Ctx;

#define CTX_CHECK(ctx)                                                    \
  do {                                                                    \
    if (!(ctx)) return rq::set_error(RQ_EVALUE, "null rq_ctx");           \
    cudaError_t _e = cudaSetDevice((ctx)->c.device);                      \
    if (_e != cudaSuccess)                                                \
      return rq::set_error(RQ_ECUDA, "cudaSetDevice: %s", cudaGetErrorString(_e)); \
  } while (0)

extern "C" {
#pragma GCC visibility push(default)

const char* rq_version(void) { return "randqr_b200 0.1.0 (sm_100a)"; }
const char* rq_last_error(void) { return rq::last_error(); }

int rq_ctx_create(rq_ctx** out, int32_t device, void* stream) {
  if (!out) return rq::set_error(RQ_EVALUE, "null output pointer");
  *out = nullptr;
  RQ_CUDA_TRY(cudaSetDevice(device));
  rq_ctx* c = new (std::nothrow) rq_ctx;
  if (!c) return rq::set_error(RQ_EINTERNAL, "out of host memory");
  c->c.device = device;
  c->c.stream = (cudaStream_t)stream;
  c->c.nbarriers = 1 << 16;
  cudaError_t e = cudaMalloc(&c->c.barriers, sizeof(unsigned) * c->c.nbarriers);
  if (e == cudaSuccess) e = cudaMemset(c->c.barriers, 0, sizeof(unsigned) * c->c.nbarriers);
  if (e != cudaSuccess) {
    delete c;
    return rq::set_error(RQ_ECUDA, "barrier ring: %s", cudaGetErrorString(e));
  }
  *out = c;
  return RQ_OK;
}

int rq_ctx_destroy(rq_ctx* ctx) {
  if (!ctx) return RQ_OK;
  cudaSetDevice(ctx->c.device);
  if (ctx->c.stream) cudaStreamSynchronize(ctx->c.stream);
  else cudaDeviceSynchronize();
  delete ctx;
  return RQ_OK;
}

int rq_ctx_set_stream(rq_ctx* ctx, void* stream) {
  CTX_CHECK(ctx);
  ctx->c.stream = (cudaStream_t)stream;
  return RQ_OK;
}

int rq_ctx_set_gemm_cap(rq_ctx* ctx, int32_t max_ctas) {
  CTX_CHECK(ctx);
  if (max_ctas < 0) return rq::set_error(RQ_EVALUE, "max_ctas < 0");
  ctx->c.gemm_cap = max_ctas;
  return RQ_OK;
}

int rq_ctx_set_inspect(rq_ctx* ctx, rq_panel_cb cb, void* user) {
  CTX_CHECK(ctx);
  ctx->c.inspect_cb = cb;
  ctx->c.inspect_user = user;
  return RQ_OK;
}

// Validation in the reference's order (blocked.py:152-161, pivoting.py:97-98).
// On a sketch-width error the counter is advanced by the draws of the panels
// the reference completes before raising, so RngState matches afterwards.
static int validate(const rq_config* cfg, int64_t m, int64_t n, uint64_t* counter) {
  if (!cfg) return rq::set_error(RQ_EVALUE, "null config");
  if (m < n) return rq::set_error(RQ_EDIM, "blocked QR needs rows >= cols, got %lldx%lld", (long long)m, (long long)n);
  if (cfg->block < 1 || cfg->block > n)
    return rq::set_error(RQ_EDIM, "block size must lie in [1, %lld], got %d", (long long)n, cfg->block);
  if (cfg->oversample < 0 || cfg->power < 0) return rq::set_error(RQ_EVALUE, "oversample and power must be >= 0");
  const int b = cfg->block, wdt = cfg->block + cfg->oversample;
  uint64_t drawn = 0;
  for (int64_t s = 0; n - s > b; s += b) {
    const int64_t np = n - s;
    if (wdt > np) {
      // fresh: the panels before this one drew their Omegas (pivoting.py:100-101); downdate:
      // G (m x (b+p)) is drawn before the panel loop (the oracle's block_qr_downdate, and
      // dist.factorize_local), so the error comes after those m(b+p) draws
      if (counter) *counter += cfg->sketch_mode == RQ_SKETCH_FRESH ? drawn : (uint64_t)m * (uint64_t)wdt;
      return rq::set_error(RQ_EVALUE, "sketch width %d exceeds the %lld columns being pivoted", wdt, (long long)np);
    }
    drawn += (uint64_t)(m - s) * (uint64_t)wdt;
  }
  return RQ_OK;
}

int rq_factorize(rq_ctx* ctx, const rq_config* cfg, int64_t m, int64_t n, double* dA, int64_t lda, uint64_t seed,
                 uint64_t* counter, int64_t* dperm) {
  CTX_CHECK(ctx);
  rq::clear_error();
  if (!counter) return rq::set_error(RQ_EVALUE, "null counter");
  RQ_TRY(validate(cfg, m, n, counter));
  if (lda < m || (lda & 1) || ((uintptr_t)dA & 15))
    return rq::set_error(RQ_EVALUE, "dA must be 16-byte aligned with an even lda >= m");
  if (cfg->rrqr) {
    if (cfg->sketch_mode != RQ_SKETCH_FRESH)
      return rq::set_error(RQ_EUNSUPPORTED, "block_rrqr uses fresh sketches (reference semantics)");
    return ctx->c.factorize_rrqr(*cfg, m, n, dA, lda, seed, counter);
  }
  if (cfg->pivot_kind == RQ_PIVOT_REFLECTORS && cfg->sketch_mode == RQ_SKETCH_DOWNDATE)
    return rq::set_error(RQ_EUNSUPPORTED, "the downdated sketch applies to permutation pivots");
  if (cfg->sketch_mode == RQ_SKETCH_DOWNDATE && cfg->power != 0)
    return rq::set_error(RQ_EUNSUPPORTED, "downdate sketch with power iterations");
  ctx->c.tf32_update = (cfg->flags & RQ_FLAG_TF32_UPDATE) != 0;
  const int rc = ctx->c.factorize_perm(*cfg, m, n, dA, lda, seed, counter, dperm);
  ctx->c.tf32_update = false;
  return rc;
}

int rq_factorize_host(rq_ctx* ctx, const rq_config* cfg, int64_t m, int64_t n, const double* hA, int64_t lda,
                      uint64_t seed, uint64_t* counter, double* hR, int64_t ldr, int64_t* hperm) {
  CTX_CHECK(ctx);
  rq::clear_error();
  if (!counter) return rq::set_error(RQ_EVALUE, "null counter");
  if (!hA) return rq::set_error(RQ_EVALUE, "null hA");
  if (lda < m) return rq::set_error(RQ_EVALUE, "lda (%lld) < m (%lld)", (long long)lda, (long long)m);
  if (hR && ldr < m) return rq::set_error(RQ_EVALUE, "ldr (%lld) < m (%lld)", (long long)ldr, (long long)m);
  RQ_TRY(validate(cfg, m, n, counter));
  Ctx& c = ctx->c;
  const int64_t ldd = rq::even(m);
  // device copy of A (and the permutation) in a context-owned, grow-only buffer: no per-call
  // allocation (a freed-and-remapped 800 MB pool block cost tens of ms, erratically)
  const size_t abytes = ((size_t)ldd * n * 8 + 255) & ~size_t(255);
  RQ_CUDA_TRY(cudaStreamSynchronize(c.stream));  // the buffer may still feed an earlier call's copies
  RQ_TRY(c.harena.reserve(abytes + (size_t)n * 8));
  double* dA = static_cast<double*>(c.harena.base);
  int64_t* dp = reinterpret_cast<int64_t*>(static_cast<char*>(c.harena.base) + abytes);
  int rc = RQ_OK;
  cudaError_t e = cudaSuccess;
  // HQRRP's downdated sketch needs Y = G A before anything else: A arrives in column chunks on
  // its own stream and every chunk's Y columns are formed while the next chunk is on the wire,
  // so only the last chunk's product is exposed (RQ_H2D_CHUNKS: chunk count, 0/1 = one copy;
  // default 8 from 64 MB up).
  static const int env_chunks = getenv("RQ_H2D_CHUNKS") ? atoi(getenv("RQ_H2D_CHUNKS")) : -1;
  int chunks = env_chunks >= 0 ? env_chunks : ((size_t)m * n * 8 >= ((size_t)64 << 20) ? 8 : 1);
  const bool chunked = chunks > 1 && !cfg->rrqr && cfg->pivot_kind == RQ_PIVOT_PERMUTATION &&
                       cfg->sketch_mode == RQ_SKETCH_DOWNDATE && cfg->power == 0 && n > cfg->block &&
                       !c.inspect_cb;
  if (chunked) {
    chunks = (int)std::min<int64_t>(chunks, n);
    if (!c.h2d_stream && cudaStreamCreateWithFlags(&c.h2d_stream, cudaStreamNonBlocking) != cudaSuccess)
      rc = rq::set_error(RQ_ECUDA, "h2d stream");
    while (rc == RQ_OK && (int)c.h2d_ev.size() < chunks) {
      cudaEvent_t ev;
      if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) rc = rq::set_error(RQ_ECUDA, "event");
      else c.h2d_ev.push_back(ev);
    }
    if (rc == RQ_OK) rc = c.presketch_begin(*cfg, m, n, seed, *counter);
    const int64_t per = (n + chunks - 1) / chunks;
    for (int k = 0; rc == RQ_OK && k < chunks; k++) {
      const int64_t c0 = (int64_t)k * per, c1 = std::min<int64_t>(n, c0 + per);
      if (c1 <= c0) break;
      e = cudaMemcpy2DAsync(dA + c0 * ldd, ldd * 8, hA + c0 * lda, lda * 8, m * 8, c1 - c0, cudaMemcpyHostToDevice,
                            c.h2d_stream);
      if (e == cudaSuccess) e = cudaEventRecord(c.h2d_ev[k], c.h2d_stream);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(c.stream, c.h2d_ev[k], 0);
      if (e != cudaSuccess) rc = rq::set_error(RQ_ECUDA, "H2D chunk: %s", cudaGetErrorString(e));
      if (rc == RQ_OK) rc = c.presketch_cols(*cfg, m, n, dA, ldd, c0, c1);
    }
    c.presketched = rc == RQ_OK;
  } else {
    e = cudaMemcpy2DAsync(dA, ldd * 8, hA, lda * 8, m * 8, n, cudaMemcpyHostToDevice, c.stream);
    if (e != cudaSuccess) rc = rq::set_error(RQ_ECUDA, "H2D: %s", cudaGetErrorString(e));
  }
  // R streams back panel by panel on the context's copy stream (created on its device) while
  // later panels compute
  if (rc == RQ_OK && hR && !c.copy_stream) {
    if (cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c.copy_ev, cudaEventDisableTiming) != cudaSuccess)
      rc = rq::set_error(RQ_ECUDA, "copy stream");
  }
  int64_t copied = 0;   // columns [0, copied) queued
  bool streamed = false;
  cudaError_t cb_err = cudaSuccess;  // first failure inside the callback
  if (rc == RQ_OK && hR) {
    c.on_cols_final = [&](int64_t s, int64_t w) {
      if (s != copied || cb_err != cudaSuccess) return;  // keep the watermark contiguous
      cudaError_t x = cudaEventRecord(c.copy_ev, c.stream);
      if (x == cudaSuccess) x = cudaStreamWaitEvent(c.copy_stream, c.copy_ev, 0);
      if (x == cudaSuccess)
        x = cudaMemcpy2DAsync(hR + s * ldr, ldr * 8, dA + s * ldd, ldd * 8, m * 8, w, cudaMemcpyDeviceToHost,
                              c.copy_stream);
      if (x != cudaSuccess) {
        cb_err = x;
        return;
      }
      streamed = true;
      copied = s + w;
    };
  }
  if (rc == RQ_OK) rc = rq_factorize(ctx, cfg, m, n, dA, ldd, seed, counter, dp);
  c.on_cols_final = nullptr;
  c.presketched = false;
  if (rc == RQ_OK && cb_err != cudaSuccess) rc = rq::set_error(RQ_ECUDA, "D2H (streamed R): %s", cudaGetErrorString(cb_err));
  if (rc == RQ_OK && hR && copied < n) {
    e = cudaMemcpy2DAsync(hR + copied * ldr, ldr * 8, dA + copied * ldd, ldd * 8, m * 8, n - copied,
                          cudaMemcpyDeviceToHost, c.stream);
    if (e != cudaSuccess) rc = rq::set_error(RQ_ECUDA, "D2H: %s", cudaGetErrorString(e));
  }
  if (rc == RQ_OK && hperm) {
    e = cudaMemcpyAsync(hperm, dp, n * 8, cudaMemcpyDeviceToHost, c.stream);
    if (e != cudaSuccess) rc = rq::set_error(RQ_ECUDA, "D2H perm: %s", cudaGetErrorString(e));
  }
  if (streamed) {  // the buffer is reused by the next call on the main stream: after the copies
    e = cudaEventRecord(c.copy_ev, c.copy_stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c.stream, c.copy_ev, 0);
    if (rc == RQ_OK && e != cudaSuccess) rc = rq::set_error(RQ_ECUDA, "copy join: %s", cudaGetErrorString(e));
  }
  e = cudaStreamSynchronize(c.stream);
  if (rc == RQ_OK && e != cudaSuccess) rc = rq::set_error(RQ_ECUDA, "sync: %s", cudaGetErrorString(e));
  if (streamed) {
    e = cudaStreamSynchronize(c.copy_stream);
    if (rc == RQ_OK && e != cudaSuccess) rc = rq::set_error(RQ_ECUDA, "copy sync: %s", cudaGetErrorString(e));
  }
  return rc;
}

static int form_q_checked(Ctx& c, const rq::FactorSet& F, int64_t cols, double* dQ, int64_t ldq) {
  if (!F.have) return rq::set_error(RQ_EVALUE, "no factorization stored in this context");
  if (F.device != c.device) return rq::set_error(RQ_EVALUE, "the factors live on device %d, the context on %d",
                                                 F.device, c.device);
  if (cols < F.fn || cols > F.fm)
    return rq::set_error(RQ_EDIM, "cols must lie in [%lld, %lld]", (long long)F.fn, (long long)F.fm);
  if (ldq < F.fm || (ldq & 1) || ((uintptr_t)dQ & 15))
    return rq::set_error(RQ_EVALUE, "dQ must be 16-byte aligned with an even ldq >= m");
  return c.form_q(F, cols, dQ, ldq);
}

static int form_p_checked(Ctx& c, const rq::FactorSet& F, double* dP, int64_t ldp) {
  if (!F.have) return rq::set_error(RQ_EVALUE, "no factorization stored in this context");
  if (F.device != c.device) return rq::set_error(RQ_EVALUE, "the factors live on device %d, the context on %d",
                                                 F.device, c.device);
  if (ldp < F.fn) return rq::set_error(RQ_EVALUE, "ldp < n");
  return c.form_p(F, dP, ldp);
}

int rq_form_q(rq_ctx* ctx, int64_t cols, double* dQ, int64_t ldq) {
  CTX_CHECK(ctx);
  rq::clear_error();
  return form_q_checked(ctx->c, ctx->c.view(), cols, dQ, ldq);
}

int rq_form_p(rq_ctx* ctx, double* dP, int64_t ldp) {
  CTX_CHECK(ctx);
  rq::clear_error();
  return form_p_checked(ctx->c, ctx->c.view(), dP, ldp);
}

static const rq::FactorSet* pick(Ctx& c, const rq_factors* f, rq::FactorSet& tmp) {
  if (f) return &f->f;
  tmp = c.view();
  return &tmp;
}

int rq_factors_info(rq_ctx* ctx, const rq_factors* f, int32_t which, int32_t cap, int64_t* offsets, int32_t* widths,
                    int32_t* count) {
  CTX_CHECK(ctx);
  rq::clear_error();
  rq::FactorSet tmp;
  const rq::FactorSet* F = pick(ctx->c, f, tmp);
  if (!F->have) return rq::set_error(RQ_EVALUE, "no factorization stored in this context");
  if (!count) return rq::set_error(RQ_EVALUE, "null count");
  if (which == 0) {
    *count = (int32_t)F->factors.size();
    for (int32_t i = 0; i < *count && i < cap; i++) {
      if (offsets) offsets[i] = F->factors[i].s;
      if (widths) widths[i] = F->factors[i].k;
    }
  } else {
    *count = F->p_is_perm ? 0 : (int32_t)F->rfactors.size();
    for (int32_t i = 0; i < *count && i < cap; i++) {
      if (offsets) offsets[i] = F->rfactors[i].s;
      if (widths) widths[i] = (int32_t)F->rfactors[i].np;
    }
  }
  return RQ_OK;
}

int rq_apply_q(rq_ctx* ctx, const rq_factors* f, int32_t first, int32_t count, int32_t trans, int64_t cols,
               double* dX, int64_t ldx) {
  CTX_CHECK(ctx);
  rq::clear_error();
  rq::FactorSet tmp;
  const rq::FactorSet* F = pick(ctx->c, f, tmp);
  if (!F->have) return rq::set_error(RQ_EVALUE, "no factorization stored in this context");
  if (F->device != ctx->c.device) return rq::set_error(RQ_EVALUE, "factors and context on different devices");
  if (cols < 0) return rq::set_error(RQ_EDIM, "cols < 0");
  if (ldx < F->fm || (ldx & 1) || ((uintptr_t)dX & 15))
    return rq::set_error(RQ_EVALUE, "dX must be 16-byte aligned with an even ldx >= m");
  return ctx->c.apply_q(*F, first, count, trans != 0, false, cols, dX, ldx);
}

int rq_apply_p(rq_ctx* ctx, const rq_factors* f, int32_t first, int32_t count, int64_t rows, double* dX,
               int64_t ldx) {
  CTX_CHECK(ctx);
  rq::clear_error();
  rq::FactorSet tmp;
  const rq::FactorSet* F = pick(ctx->c, f, tmp);
  if (!F->have) return rq::set_error(RQ_EVALUE, "no factorization stored in this context");
  if (F->device != ctx->c.device) return rq::set_error(RQ_EVALUE, "factors and context on different devices");
  if (rows < 0) return rq::set_error(RQ_EDIM, "rows < 0");
  if (ldx < rows || (ldx & 1) || ((uintptr_t)dX & 15))
    return rq::set_error(RQ_EVALUE, "dX must be 16-byte aligned with an even ldx >= rows");
  return ctx->c.apply_p(*F, first, count, rows, dX, ldx);
}

int rq_factors_detach(rq_ctx* ctx, rq_factors** out) {
  CTX_CHECK(ctx);
  rq::clear_error();
  if (!out) return rq::set_error(RQ_EVALUE, "null output pointer");
  *out = nullptr;
  rq_factors* f = new (std::nothrow) rq_factors;
  if (!f) return rq::set_error(RQ_EINTERNAL, "out of host memory");
  int rc = ctx->c.detach(&f->f);
  if (rc != RQ_OK) {
    delete f;
    return rc;
  }
  *out = f;
  return RQ_OK;
}

int rq_factors_destroy(rq_factors* f) {
  if (!f) return RQ_OK;
  cudaSetDevice(f->f.device);
  f->f.arena.release();
  delete f;
  return RQ_OK;
}

int rq_factors_form_q(rq_ctx* ctx, const rq_factors* f, int64_t cols, double* dQ, int64_t ldq) {
  CTX_CHECK(ctx);
  rq::clear_error();
  if (!f) return rq::set_error(RQ_EVALUE, "null rq_factors");
  return form_q_checked(ctx->c, f->f, cols, dQ, ldq);
}

int rq_factors_form_p(rq_ctx* ctx, const rq_factors* f, double* dP, int64_t ldp) {
  CTX_CHECK(ctx);
  rq::clear_error();
  if (!f) return rq::set_error(RQ_EVALUE, "null rq_factors");
  return form_p_checked(ctx->c, f->f, dP, ldp);
}

int rq_snapshot(rq_ctx* ctx, double* hW, int64_t ldh) {
  CTX_CHECK(ctx);
  return ctx->c.snapshot(hW, ldh);
}

int rq_snapshot_sketch(rq_ctx* ctx, double* hY, int64_t ldh, int64_t* hperm) {
  CTX_CHECK(ctx);
  return ctx->c.snapshot_sketch(hY, ldh, hperm);
}

int rq_householder_sweep(rq_ctx* ctx, double* dA, int64_t m, int64_t n, int64_t lda, double* dV, int64_t ldv,
                         int64_t* dperm, int64_t steps, int32_t pivot) {
  CTX_CHECK(ctx);
  rq::clear_error();
  if (m < 0 || n < 0 || steps < 0 || steps > n || (steps > 0 && dV == nullptr))
    return rq::set_error(RQ_EDIM, "householder_sweep: bad shape m=%lld n=%lld steps=%lld", (long long)m,
                         (long long)n, (long long)steps);
  if (steps == 0 || m == 0) return RQ_OK;
  Ctx& c = ctx->c;
  const int G = rq::sweep_grid_size((int)n);
  const size_t ws = rq::sweep_workspace_bytes(m, (int)n, G);
  const int64_t ldr = rq::even(m);
  const size_t need = ws + 1024 + (size_t)ldr * n * 8 + (size_t)n * 4 * 3 + (size_t)n * 8 + 4096;
  RQ_TRY(c.qarena.reserve(need));
  char* base = (char*)c.qarena.base;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  c.sweep_ws = base;
  c.sweep_ws_bytes = ws;
  size_t off = al(ws);
  double* rtmp = (double*)(base + off);
  off += al((size_t)ldr * n * 8);
  int* cap = (int*)(base + off);
  off += al((size_t)n * 4);
  int* io = (int*)(base + off);
  off += al((size_t)n * 4);
  int64_t* ost = (int64_t*)(base + off);
  rq::SweepCall sc;
  sc.a = dA;
  sc.lda = lda;
  sc.m = m;
  sc.n = (int)n;
  sc.steps = (int)steps;
  sc.pivot = pivot ? 1 : 0;
  sc.v = dV;
  sc.ldv = ldv;
  sc.col_at_pos = cap;
  sc.r_out = pivot ? rtmp : nullptr;
  sc.ldr = ldr;
  RQ_TRY(c.sweep(sc));
  if (pivot) {
    RQ_TRY(rq::copy2d(rtmp, ldr, dA, lda, m, n, 0, c.stream, &c.launches));
    if (dperm) {
      RQ_TRY(rq::iota(io, (int)n, nullptr, 0, c.stream, &c.launches));
      rq::MoveCall mv{dA, lda, 0, 0, 0, cap, io, nullptr, (int)n, rtmp, ldr, dperm, ost};
      RQ_TRY(rq::move_columns(mv, c.stream, &c.launches));
    }
  }
  return RQ_OK;
}

int rq_gaussian_matrix(rq_ctx* ctx, int64_t rows, int64_t cols, uint64_t seed, uint64_t counter, double* dOut,
                       int64_t ld) {
  CTX_CHECK(ctx);
  if (rows < 1 || cols < 1)
    return rq::set_error(RQ_EDIM, "matrix dimensions must be positive, got %lldx%lld", (long long)rows,
                         (long long)cols);
  return rq::gaussian_fill(dOut, rows, cols, ld, seed, counter, ctx->c.stream, &ctx->c.launches);
}

int rq_splitmix_words(rq_ctx* ctx, uint64_t seed, uint64_t first, int64_t count, uint64_t* dOut) {
  CTX_CHECK(ctx);
  return rq::splitmix_words(dOut, seed, first, count, ctx->c.stream, &ctx->c.launches);
}

int rq_test_gemm(rq_ctx* ctx, int32_t a_mmajor, int64_t M, int64_t N, int64_t K, const double* dA, int64_t lda,
                 int64_t a_rows, int64_t a_cols, int64_t a_r0, int64_t a_c0, const double* dB, int64_t ldb,
                 int64_t b_rows, int64_t b_cols, int64_t b_r0, int64_t b_c0, double* dC, int64_t ldc, double alpha,
                 double beta) {
  CTX_CHECK(ctx);
  rq::clear_error();
  Ctx& c = ctx->c;
  const size_t kb = (size_t)rq::kSMs * 256 * 256 * 8;
  RQ_TRY(c.qarena.reserve(kb));
  c.kwork = (double*)c.qarena.base;
  c.kwork_bytes = kb;
  rq::GemmOperand A{dA, a_rows, a_cols, lda, a_r0, a_c0};
  rq::GemmOperand B{dB, b_rows, b_cols, ldb, b_r0, b_c0};
  return c.gemm(M, N, K, A, a_mmajor != 0, B, dC, ldc, alpha, beta);
}

int rq_qr_unpivoted(rq_ctx* ctx, int64_t m, int64_t n, double* dA, int64_t lda, int32_t block) {
  CTX_CHECK(ctx);
  rq::clear_error();
  if (m < n) return rq::set_error(RQ_EDIM, "qr_unpivoted needs rows >= cols, got %lldx%lld", (long long)m, (long long)n);
  if (n < 1 || block < 1) return rq::set_error(RQ_EDIM, "bad shape n=%lld block=%d", (long long)n, block);
  if (lda < m || (lda & 1) || ((uintptr_t)dA & 15))
    return rq::set_error(RQ_EVALUE, "dA must be 16-byte aligned with an even lda >= m");
  return ctx->c.factorize_unpivoted(m, n, dA, lda, std::min<int64_t>(block, n));
}

// Frobenius truncation errors from R (metrics.truncation_errors at scale): for an
// upper-triangular R (n x n block at dR), e2[k] = ||R[k:, k:]||_F^2, k = 0..n (e2[n] = 0).
int rq_trailing_frobenius(rq_ctx* ctx, const double* dR, int64_t n, int64_t ldr, double* dE2) {
  CTX_CHECK(ctx);
  rq::clear_error();
  if (n < 0 || ldr < n) return rq::set_error(RQ_EDIM, "trailing_frobenius: bad shape");
  return rq::trailing_frobenius(dR, n, ldr, dE2, ctx->c.stream, &ctx->c.launches);
}

int rq_trailing_spectral(rq_ctx* ctx, const double* dR, int64_t n, int64_t ldr, const int64_t* hks, int32_t nks,
                         double* hOut, int32_t* hHow) {
  CTX_CHECK(ctx);
  rq::clear_error();
  if (n < 0 || ldr < n || (ldr & 1) || ((uintptr_t)dR & 15)) return rq::set_error(RQ_EDIM, "trailing_spectral: bad shape");
  if (nks < 0 || (nks > 0 && (!hks || !hOut || !hHow))) return rq::set_error(RQ_EVALUE, "trailing_spectral: null");
  return ctx->c.trailing_spectral(dR, n, ldr, reinterpret_cast<const int64_t*>(hks), nks, hOut, hHow);
}

// ---------------------------------------------------------------------------
// Panel-step API (multi-GPU driver, dist.py)
// ---------------------------------------------------------------------------
static bool al16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

int rq_gemm_f32(rq_ctx* ctx, int32_t a_mmajor, int64_t M, int64_t N, int64_t K, const float* dA, int64_t lda,
                int64_t a_rows, int64_t a_cols, int64_t a_r0, int64_t a_c0, const float* dB, int64_t ldb,
                int64_t b_rows, int64_t b_cols, int64_t b_r0, int64_t b_c0, float* dC, int64_t ldc, double alpha,
                double beta) {
  CTX_CHECK(ctx);
  rq::clear_error();
  if (M < 0 || N < 0 || K < 0) return rq::set_error(RQ_EDIM, "gemm_f32: negative extent");
  if ((lda & 3) || (ldb & 3) || !al16(dA) || !al16(dB))
    return rq::set_error(RQ_EVALUE, "gemm_f32: operands need ld %% 4 == 0 and 16-byte aligned bases");
  if (M == 0 || N == 0) return RQ_OK;
  rq::GemmProblemF32 p;
  p.M = M;
  p.N = N;
  p.K = K;
  p.A = rq::GemmOperandF32{dA, a_rows, a_cols, lda, a_r0, a_c0};
  p.a_mmajor = a_mmajor != 0;
  p.B = rq::GemmOperandF32{dB, b_rows, b_cols, ldb, b_r0, b_c0};
  p.C = dC;
  p.ldc = ldc;
  p.alpha = alpha;
  p.beta = beta;
  p.max_ctas = ctx->c.gemm_cap;
  // split-K slabs: up to 16 partial M x N products, from the context's step-API arena
  const size_t kb = std::min<size_t>((size_t)16 * M * N * sizeof(float), (size_t)1 << 30);
  if (K >= 4096 && rq::ceil_div(M, 128) * rq::ceil_div(N, 128) < 4 * rq::kSMs) {
    RQ_TRY(ctx->c.sarena.reserve(kb));
    p.work = static_cast<float*>(ctx->c.sarena.base);
    p.work_bytes = kb;
  }
  return rq::gemm_tf32x3(p, ctx->c.stream, &ctx->c.launches);
}

int rq_gemm(rq_ctx* ctx, int32_t a_mmajor, int64_t M, int64_t N, int64_t K, const double* dA, int64_t lda,
            int64_t a_rows, int64_t a_cols, int64_t a_r0, int64_t a_c0, const double* dB, int64_t ldb, int64_t b_rows,
            int64_t b_cols, int64_t b_r0, int64_t b_c0, double* dC, int64_t ldc, double alpha, double beta) {
  CTX_CHECK(ctx);
  rq::clear_error();
  if (M < 0 || N < 0 || K < 0) return rq::set_error(RQ_EDIM, "gemm: negative extent");
  if ((lda & 1) || (ldb & 1) || !al16(dA) || !al16(dB))
    return rq::set_error(RQ_EVALUE, "gemm: operands need even leading dimensions and 16-byte aligned bases");
  if (M == 0 || N == 0) return RQ_OK;
  Ctx& c = ctx->c;
  const size_t kb = (size_t)rq::kSMs * 256 * 256 * 8;
  RQ_TRY(c.sarena.reserve(kb));
  c.kwork = (double*)c.sarena.base;
  c.kwork_bytes = kb;
  rq::GemmOperand A{dA, a_rows, a_cols, lda, a_r0, a_c0};
  rq::GemmOperand B{dB, b_rows, b_cols, ldb, b_r0, b_c0};
  return c.gemm(M, N, K, A, a_mmajor != 0, B, dC, ldc, alpha, beta);
}

int rq_trinv_upper(rq_ctx* ctx, const double* dR, int64_t ldr, int32_t k, double* dX, int64_t ldx) {
  CTX_CHECK(ctx);
  rq::clear_error();
  if (k < 0) return rq::set_error(RQ_EDIM, "trinv: negative order");
  Ctx& c = ctx->c;
  return rq::trinv_upper(dR, ldr, k, dX, ldx, c.stream, &c.launches);
}

int rq_sketch_select(rq_ctx* ctx, double* dY, int64_t ldy, int32_t m, int32_t n, int32_t steps,
                     const int32_t* dInitPos, int32_t* dChosen) {
  CTX_CHECK(ctx);
  rq::clear_error();
  if (m <= 0 || n <= 0 || steps < 0 || steps > n || steps > m || ldy < m)
    return rq::set_error(RQ_EDIM, "sketch_select: bad shape m=%d n=%d steps=%d", m, n, steps);
  return ctx->c.step_sketch_select(dY, ldy, m, n, steps, dInitPos, dChosen);
}

int rq_panel_factor(rq_ctx* ctx, double* dP, int64_t ldp, int64_t mp, int32_t b, double* dV, int64_t ldv, double* dT,
                    int64_t ldt, double* dQ2, int64_t ldq2, int32_t* dPhat) {
  CTX_CHECK(ctx);
  rq::clear_error();
  if (b <= 0 || b > 512 || mp < b || ldp < mp || ldv < mp || ldt < b || ldq2 < b)
    return rq::set_error(RQ_EDIM, "panel_factor: bad shape mp=%lld b=%d", (long long)mp, b);
  if ((ldp & 1) || (ldv & 1) || (ldt & 1) || (ldq2 & 1) || !al16(dP) || !al16(dV) || !al16(dT) || !al16(dQ2))
    return rq::set_error(RQ_EVALUE, "panel_factor: buffers need even leading dimensions and 16-byte alignment");
  return ctx->c.step_panel_factor(dP, ldp, mp, b, dV, ldv, dT, ldt, dQ2, ldq2, dPhat);
}

int rq_panel_apply(rq_ctx* ctx, const double* dV, int64_t ldv, const double* dT, int64_t ldt, const double* dQ2,
                   int64_t ldq2, int64_t mp, int32_t b, double* dA, int64_t lda, int64_t a_rows, int64_t a_cols,
                   int64_t r0, int64_t c0, int64_t n2) {
  CTX_CHECK(ctx);
  rq::clear_error();
  if (b <= 0 || b > 512 || mp < b || n2 < 0 || r0 < 0 || c0 < 0 || r0 + mp > a_rows || c0 + n2 > a_cols ||
      lda < a_rows)
    return rq::set_error(RQ_EDIM, "panel_apply: bad shape");
  if ((ldv & 1) || (ldt & 1) || (ldq2 & 1) || (lda & 1) || !al16(dV) || !al16(dT) || !al16(dA) ||
      (dQ2 && !al16(dQ2)))
    return rq::set_error(RQ_EVALUE, "panel_apply: buffers need even leading dimensions and 16-byte alignment");
  return ctx->c.step_panel_apply(dV, ldv, dT, ldt, dQ2, ldq2, mp, b, dA, lda, a_rows, a_cols, r0, c0, n2);
}

int rq_test_sketch_cpqr(rq_ctx* ctx, double* dY, int64_t ld, int32_t m, int32_t n, int32_t steps, int32_t* dChosen) {
  CTX_CHECK(ctx);
  rq::clear_error();
  Ctx& c = ctx->c;
  const size_t ws = std::max(rq::sweep_workspace_bytes(m, n, rq::kSMs), rq::sketch_workspace_bytes(m, n)) + 4096;
  RQ_TRY(c.qarena.reserve(ws));
  c.sweep_ws = c.qarena.base;
  c.sweep_ws_bytes = ws;
  return c.sketch_select(dY, ld, m, n, steps, nullptr, dChosen);
}

int rq_test_leaf_qr(rq_ctx* ctx, double* dA, int64_t lda, int64_t mm, int32_t w, double* dV, int64_t ldv,
                    double* dT, int64_t ldt) {
  CTX_CHECK(ctx);
  rq::clear_error();
  rq::LeafCall lc;
  lc.a = dA;
  lc.lda = lda;
  lc.mm = mm;
  lc.w = w;
  lc.v = dV;
  lc.ldv = ldv;
  lc.tl = dT;
  lc.ldt = ldt;
  return rq::leaf_qr(lc, ctx->c.stream, &ctx->c.launches);
}

int rq_test_wy_update(rq_ctx* ctx, int32_t cluster, double* dA, int64_t lda, int64_t mm, int32_t nr, const double* dV,
                      int64_t ldv, const double* dT, int64_t ldt, int32_t w) {
  CTX_CHECK(ctx);
  rq::clear_error();
  Ctx& c = ctx->c;
  if (cluster)
    return rq::wy_cluster(dA, lda, mm, nr, 0, 0, mm, nr, dV, ldv, mm, w, 0, 0, dT, ldt, w, c.stream, &c.launches);
  if (!rq::wy_update_fits(mm, nr, w)) return rq::set_error(RQ_EUNSUPPORTED, "wy_update does not fit");
  const size_t kb = (size_t)rq::kSMs * 16 * 256 * 8 + 16 * 256 * 8;
  RQ_TRY(c.qarena.reserve(kb));
  RQ_CUDA_TRY(cudaMemsetAsync(c.barriers, 0, sizeof(unsigned) * 64, c.stream));
  return rq::wy_update(dA, lda, mm, nr, dV, ldv, dT, ldt, w, (double*)c.qarena.base, kb, c.barriers, c.stream,
                       &c.launches);
}

int rq_test_debug_timing(int32_t on, uint64_t* host, int32_t count) {
  // on: 1 = cluster/sketch sweeps, 2 = panel leaf
  if (on == 2 || (on == 0 && count < 0)) return rq::leaf_debug_timing(on == 2, (unsigned long long*)host, -count);
  RQ_TRY(rq::leaf_debug_timing(0, nullptr, 0));
  return rq::sweep_debug_timing(on, (unsigned long long*)host, count);
}

int64_t rq_launch_count(rq_ctx* ctx) { return ctx ? ctx->c.launches : 0; }

int rq_set_profiling(rq_ctx* ctx, int32_t on) {
  CTX_CHECK(ctx);
  ctx->c.prof = on != 0;
  ctx->c.prof_recs.clear();
  ctx->c.ev_next = 0;
  if (ctx->c.prof_dev_bytes) RQ_CUDA_TRY(cudaMemset(ctx->c.prof_dev_bytes, 0, 8));
  return RQ_OK;
}

int rq_profile_bytes(rq_ctx* ctx, int32_t category, double* bytes) {
  CTX_CHECK(ctx);
  if (!bytes) return rq::set_error(RQ_EVALUE, "null bytes");
  RQ_CUDA_TRY(cudaStreamSynchronize(ctx->c.stream));
  double b = 0.0;
  for (const auto& r : ctx->c.prof_recs)
    if (r.cat == category) b += r.bytes;
  if (category == rq::PROF_MOVES && ctx->c.prof_dev_bytes) {
    unsigned long long v = 0;
    RQ_CUDA_TRY(cudaMemcpy(&v, ctx->c.prof_dev_bytes, 8, cudaMemcpyDeviceToHost));
    b += (double)v;
  }
  *bytes = b;
  return RQ_OK;
}

int rq_profile_read(rq_ctx* ctx, int32_t category, double* ms, double* flops, int64_t* count) {
  CTX_CHECK(ctx);
  RQ_CUDA_TRY(cudaStreamSynchronize(ctx->c.stream));
  double t = 0.0, f = 0.0;
  int64_t k = 0;
  for (const auto& r : ctx->c.prof_recs) {
    if (r.cat != category) continue;
    float e = 0.f;
    RQ_CUDA_TRY(cudaEventElapsedTime(&e, r.e0, r.e1));
    t += e;
    f += r.flops;
    k++;
  }
  if (ms) *ms = t;
  if (flops) *flops = f;
  if (count) *count = k;
  return RQ_OK;
}

#pragma GCC visibility pop
}  // extern "C"
