// Panel loop of block_qr (HQRRP, Fig. 4) on one B200, enqueue-only: every
// per-panel decision (pivots, moves, P-hat, T) stays on the device; the host
// only walks panel offsets.  C ABI in capi.cu.
//
// Per non-final panel (blocked.py:204-217, restated):
//   1  Omega = next m'(b+p) normals of the caller's stream      (rng.py:54-68)
//   2  Y^T = Omega^T A[s:, s:]                  DMMA GEMM        (pivoting.py:100-101)
//   3  b-step CPQR of Y^T -> chosen columns     cooperative sweep (pivoting.py:114-129)
//   4  plan + move chosen columns into the panel (full height)   (blocked.py:205)
//   5  unpivoted panel QR, leaf by leaf (cluster kernel) + WY GEMMs (householder.py:193)
//   6  b x b CPQR of R' with Q2^T accumulated                     (householder.py:194)
//   7  R, rows-above permuted by P-hat                            (blocked.py:208-209)
//   8  T = (I/2 + striu(V^T V))^{-1}                              (householder.py:197)
//   9  tail <- Q2^T (tail - V T^T V^T tail)                       (blocked.py:210-211)
// The final block (n - s <= b) is one pivoted sweep at full height (blocked.py:195-203).
#include <algorithm>
#include <chrono>
#include <cstring>
#include <vector>

#include "driver.cuh"
#include "gemm_f64.cuh"
#include "gemm_tf32.cuh"
#include "misc.cuh"
#include "panel.cuh"

namespace rq {

// ---------------------------------------------------------------------------
// Device arena
// ---------------------------------------------------------------------------
int Arena::reserve(size_t bytes) {
  if (bytes <= cap) return RQ_OK;
  if (base) cudaFree(base);
  base = nullptr;
  cap = 0;
  RQ_CUDA_TRY(cudaMalloc(&base, bytes));
  cap = bytes;
  // fresh memory may hold another context's data (same address after a free): the sketch
  // CPQR's stamped exchange words must never match a live stamp, so start from zeros
  RQ_CUDA_TRY(cudaMemset(base, 0, bytes));
  return RQ_OK;
}
void Arena::release() {
  if (base) cudaFree(base);
  base = nullptr;
  cap = 0;
}

struct Carver {
  char* p;
  size_t off = 0;
  explicit Carver(void* b) : p((char*)b) {}
  template <class T>
  T* take(size_t count) {
    size_t bytes = ((count * sizeof(T)) + 255) & ~size_t(255);
    T* r = reinterpret_cast<T*>(p ? p + off : nullptr);
    off += bytes;
    return r;
  }
};


// ---------------------------------------------------------------------------
// Layout of scratch + stored factors for one factorization
// ---------------------------------------------------------------------------


static size_t factor_bytes(int64_t m, int64_t n, int b, bool refl = true) {
  size_t t = 0;
  for (int64_t s = 0; s < n; s += b) {
    const int64_t mp = m - s, np = n - s;
    const int w = (int)std::min<int64_t>(b, np);
    const int steps = (int)std::min<int64_t>(mp, w);
    const int64_t ldv = even(mp + 1), ldt = even(b);
    t += (((size_t)ldv * (np <= b ? steps : b) * 8 + 255) & ~size_t(255));
    t += (((size_t)ldt * b * 8 + 255) & ~size_t(255)) * 2;  // T, Q2
    if (refl) {                                              // V_S, T_S, P-hat, V~ (rrqr)
      t += (((size_t)even(np) * b * 8 + 255) & ~size_t(255));
      t += (((size_t)ldt * b * 8 + 255) & ~size_t(255)) * 2;
      t += (((size_t)std::max<int64_t>(np, b) * 4 + 255) & ~size_t(255));
    }
    (void)steps;
  }
  return t;
}

static Layout plan_layout(void* base, int64_t m, int64_t n, int b, int p, int power) {
  Layout L;
  Carver c(base);
  const int wdt = b + p;
  L.ldo = even(m + 1);
  L.ldy = even(wdt);
  const int64_t ldb = even(b);
  L.omega = c.take<double>((size_t)L.ldo * wdt);
  L.yt = c.take<double>((size_t)std::max<int64_t>(L.ldy * n, even(n) * wdt));  // Y^T, or Y scratch
  L.w1 = c.take<double>((size_t)ldb * n);
  L.w2 = c.take<double>((size_t)ldb * n);
  L.ttop = c.take<double>((size_t)ldb * n);
  L.gram = c.take<double>((size_t)ldb * b);
  L.tleaf = c.take<double>(32 * 32);
  L.rinv = c.take<double>((size_t)ldb * b);
  L.zbuf = c.take<double>((size_t)even(m) * b);
  L.z2buf = c.take<double>((size_t)even(m) * b);
  L.vst = c.take<double>((size_t)ldb * n);
  L.ov = c.take<double>((size_t)even(std::max(m, n) + 1) * wdt);
  L.ot = c.take<double>((size_t)even(wdt) * wdt);
  L.oe = c.take<double>((size_t)even(std::max(m, n) + 1) * wdt);
  L.wside = c.take<double>((size_t)ldb * n);
  L.gram2 = c.take<double>((size_t)ldb * b);
  L.kwork2_bytes = std::max<size_t>((size_t)kSMs * (b + 1) * b * 8, (size_t)8 * (b + 1) * n * 8);
  L.kwork2 = c.take<double>(L.kwork2_bytes / 8);
  L.jw = c.take<double>((size_t)ldb * b);
  L.jv = c.take<double>((size_t)ldb * b);
  L.jd = c.take<double>((size_t)ldb);
  L.jstat = c.take<int>((size_t)n / std::max(b, 1) + 2);
  L.g1 = c.take<double>((size_t)even(wdt) * b);
  L.ybuf = c.take<double>((size_t)std::max<int64_t>(even(n) * wdt, (int64_t)L.ldy * n));
  // split-K slabs: up to 16 splits of the (b+p+1) x n sketch, or 148 of the b x b Gram
  L.kwork_bytes = std::max<size_t>((size_t)kSMs * (b + 1) * b * 8, (size_t)16 * (wdt + 1) * n * 8);
  L.kwork = c.take<double>(L.kwork_bytes / 8);
  L.lds_small = ldb;
  L.small = c.take<double>((size_t)ldb * 2 * b);
  L.rfin = c.take<double>((size_t)ldb * b);
  L.stage = c.take<double>((size_t)even(m) * 2 * b + (size_t)even(m) * b);
  L.chosen = c.take<int>(n);
  L.lorderA = c.take<int>(n);
  L.lorderB = c.take<int>(n);
  L.rankA = c.take<int>(n);
  L.rankB = c.take<int>(n);
  L.newloc = c.take<int>(n);
  L.src = c.take<int>(2 * (size_t)std::max<int64_t>(b, n));
  L.dst = c.take<int>(2 * (size_t)std::max<int64_t>(b, n));
  L.nmoves = c.take<int>(4);
  L.cap = c.take<int>(n);
  L.iota_b = c.take<int>(std::max<int64_t>(b, n));
  L.flag = c.take<unsigned char>(n);
  L.orig = c.take<int64_t>(n);
  L.ostage = c.take<int64_t>(std::max<int64_t>(2 * b, n));
  L.cap2 = c.take<int>(std::max<int64_t>(b, n));
  L.stage2 = c.take<double>((size_t)even(m) * 2 * b + (size_t)even(m) * b);
  L.ostage2 = c.take<int64_t>(std::max<int64_t>(2 * b, n));
  L.sweep_ws2_bytes = sweep_workspace_bytes(b, 2 * b, sweep_grid_size(2 * b));
  L.sweep_ws2 = c.take<char>(L.sweep_ws2_bytes);
  // sweep workspace: largest of (sketch: wdt rows x n cols), (small: b rows x 2b), (final: m rows x b)
  size_t sw = 0;
  sw = std::max(sw, sweep_workspace_bytes(wdt, (int)n, sweep_grid_size((int)n)));
  sw = std::max(sw, sweep_workspace_bytes(b, 2 * b, sweep_grid_size(2 * b)));
  sw = std::max(sw, sweep_workspace_bytes(m, b, sweep_grid_size(b)));
  sw = std::max(sw, sketch_workspace_bytes(wdt, (int)n));
  L.sweep_ws_bytes = sw;
  L.sweep_ws = c.take<char>(sw);
  L.fstore = c.take<double>(factor_bytes(m, n, b) / 8 + 64);
  L.total = c.off;
  return L;
}

// ---------------------------------------------------------------------------
// GEMM shorthands (column-major views)
// ---------------------------------------------------------------------------
static GemmOperand op(const double* base, int64_t rows, int64_t cols, int64_t ld, int64_t r0 = 0, int64_t c0 = 0) {
  GemmOperand o;
  o.base = base;
  o.rows = rows;
  o.cols = cols;
  o.ld = ld;
  o.r0 = r0;
  o.c0 = c0;
  return o;
}

struct CatGuard {
  int& c;
  int saved;
  CatGuard(int& c_, int v) : c(c_), saved(c_) { c = v; }
  ~CatGuard() { c = saved; }
};

cudaEvent_t Ctx::prof_event() {
  if (ev_next == ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    ev_pool.push_back(e);
  }
  return ev_pool[ev_next++];
}
void Ctx::prof_begin(cudaEvent_t* e0) {
  *e0 = nullptr;
  if (!prof) return;
  *e0 = prof_event();
  cudaEventRecord(*e0, stream);
}
void Ctx::prof_end(cudaEvent_t e0, double flops, double bytes) {
  if (!prof || !e0) return;
  cudaEvent_t e1 = prof_event();
  cudaEventRecord(e1, stream);
  prof_recs.push_back(ProfRec{cat, e0, e1, flops, bytes});
}

// Bandwidth-bound helpers with per-class timing and algorithmic bytes when profiling is on.
int Ctx::copy2d_p(const double* S, int64_t lds, double* D, int64_t ldd, int64_t rows, int64_t cols, int upper_only,
                  cudaStream_t st, int64_t* l) {
  if (!prof) return copy2d(S, lds, D, ldd, rows, cols, upper_only, st, l);
  double elems = 0.0;
  if (!upper_only) elems = (double)rows * (double)cols;
  else
    for (int64_t j = 0; j < cols; j++) elems += (double)std::min<int64_t>(j + 1, rows);
  CatGuard g(cat, PROF_COPY);
  cudaEvent_t e0;
  prof_begin(&e0);
  const int rc = copy2d(S, lds, D, ldd, rows, cols, upper_only, st, l);
  prof_end(e0, 0.0, 16.0 * elems);
  return rc;
}

int Ctx::move_columns_p(MoveCall c, cudaStream_t st, int64_t* l) {
  if (!prof) return move_columns(c, st, l);
  if (!prof_dev_bytes) {
    if (cudaMalloc(&prof_dev_bytes, 8) != cudaSuccess) return set_error(RQ_ECUDA, "profiling counter");
    cudaMemset(prof_dev_bytes, 0, 8);
  }
  c.bytes = prof_dev_bytes;
  CatGuard g(cat, PROF_MOVES);
  cudaEvent_t e0;
  prof_begin(&e0);
  const int rc = move_columns(c, st, l);
  prof_end(e0, 0.0, 0.0);  // bytes: the device counter (read by rq_profile_bytes)
  return rc;
}

int Ctx::gaussian_fill_p(double* out, int64_t rows, int64_t cols, int64_t ld, uint64_t seed, uint64_t counter,
                         cudaStream_t st, int64_t* l) {
  if (!prof) return gaussian_fill(out, rows, cols, ld, seed, counter, st, l);
  CatGuard g(cat, PROF_RNG);
  cudaEvent_t e0;
  prof_begin(&e0);
  const int rc = gaussian_fill(out, rows, cols, ld, seed, counter, st, l);
  prof_end(e0, 0.0, 8.0 * (double)rows * (double)cols);
  return rc;
}

int Ctx::gemm(int64_t M, int64_t N, int64_t K, const GemmOperand& A, bool a_mmajor, const GemmOperand& B,
              double* C, int64_t ldc, double alpha, double beta) {
  cudaEvent_t e0;
  const int saved = cat;
  if (cat != PROF_TRAIL && cat != PROF_SKETCH_GEMM && cat != PROF_PANEL_GEMM && cat != PROF_TFACTOR)
    cat = PROF_GEMM_OTHER;
  prof_begin(&e0);
  if (prof) {
    gemm_mid = prof_event();
    gemm_splitk = 1;
  }
  int rc = gemm_raw(M, N, K, A, a_mmajor, B, C, ldc, alpha, beta);
  if (prof && e0 && gemm_splitk > 1) {
    // the GEMM up to its split-K reduce, then the reduce (slabs read, C read-modify-written)
    prof_recs.push_back(ProfRec{cat, e0, gemm_mid, 2.0 * (double)M * (double)N * (double)K, 0.0});
    cat = PROF_SPLITK;
    const double mn = (double)M * (double)N;
    prof_end(gemm_mid, 0.0, 8.0 * mn * (gemm_splitk + 1 + (beta != 0.0 ? 1 : 0)));
  } else {
    prof_end(e0, 2.0 * (double)M * (double)N * (double)K);
  }
  gemm_mid = nullptr;
  cat = saved;
  return rc;
}

int Ctx::gemm_raw(int64_t M, int64_t N, int64_t K, const GemmOperand& A, bool a_mmajor, const GemmOperand& B,
                  double* C, int64_t ldc, double alpha, double beta) {
  GemmProblem p;
  p.M = M;
  p.N = N;
  p.K = K;
  p.A = A;
  p.a_mmajor = a_mmajor;
  p.B = B;
  p.C = C;
  p.ldc = ldc;
  p.alpha = alpha;
  p.beta = beta;
  p.splitk = 0;  // automatic
  p.work = kwork;
  p.work_bytes = kwork ? kwork_bytes : 0;
  p.max_ctas = gemm_max_ctas > 0 ? gemm_max_ctas : gemm_cap;
  p.pdl = gemm_pdl;
  p.mid_event = gemm_mid;
  p.splitk_used = gemm_mid ? &gemm_splitk : nullptr;
  if (tf32_update && cat == PROF_TRAIL) return gemm_tf32x3_f64(p, stream, &launches);
  RQ_TRY(sched_for(stream, &p.sched, &p.sched_base));
  return gemm_f64(p, stream, &launches);
}

int Ctx::sched_for(cudaStream_t st, unsigned long long** ctr, unsigned long long** base) {
  // measured at n = 10k / 20k: 155.2 / 637.5 ms with it vs 155.0 / 635.7 without (the producer's
  // atomic fetch per unit), so off by default; RQ_GEMM_DYN=1 turns it on
  static const int env_dyn = [] {
    const char* e = getenv("RQ_GEMM_DYN");
    return e ? atoi(e) : 0;
  }();
  *ctr = nullptr;
  *base = nullptr;
  if (!env_dyn) return RQ_OK;
  if (!gsched) {
    RQ_CUDA_TRY(cudaMalloc(&gsched, 3 * sizeof(unsigned long long)));
    RQ_CUDA_TRY(cudaMemset(gsched, 0, 3 * sizeof(unsigned long long)));
  }
  const int k = (side && st == side) ? 1 : (hip && st == hip) ? 2 : 0;
  *ctr = gsched + k;
  *base = &gsched_base[k];
  return RQ_OK;
}

void Ctx::phase(int id) {
  if (!phases_on) return;
  cudaEvent_t e;
  if (cudaEventCreate(&e) != cudaSuccess) return;
  cudaEventRecord(e, stream);
  phase_ev.emplace_back(id, e);
  phase_host.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch())
                           .count());
}

void Ctx::side_phase(int id) {
  if (!phases_on || !side) return;
  cudaEvent_t e;
  if (cudaEventCreate(&e) != cudaSuccess) return;
  cudaEventRecord(e, side);
  side_ev.emplace_back(id, e);
}

void Ctx::phase_report() {
  if (!phases_on || phase_ev.empty()) return;
  static const char* names[] = {"start", "panel_qr", "cpqr||W,T", "wait_T", "W2,top", "downdate",
                                "sketch_cpqr", "moves,NNc", "final", "fresh_sketch", "trail+dd", "small_q",
                                "R,moves"};
  double acc[16] = {0};
  cudaEventSynchronize(phase_ev.back().second);
  for (size_t k = 1; k < phase_ev.size(); k++) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, phase_ev[k - 1].second, phase_ev[k].second);
    acc[phase_ev[k].first] += ms;
  }
  float tot = 0.f;
  cudaEventElapsedTime(&tot, phase_ev.front().second, phase_ev.back().second);
  static const bool seq = getenv("RQ_PHASES") && atoi(getenv("RQ_PHASES")) >= 2;
  if (seq) {  // the raw sequence (id:ms since the previous event), for per-panel analysis
    fprintf(stderr, "[rq phase-seq]");
    for (size_t k = 1; k < phase_ev.size(); k++) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, phase_ev[k - 1].second, phase_ev[k].second);
      fprintf(stderr, " %d:%.4f", phase_ev[k].first, ms);
    }
    fprintf(stderr, "\n[rq phase-host]");  // host enqueue time between the same phase calls
    for (size_t k = 1; k < phase_host.size(); k++)
      fprintf(stderr, " %d:%.4f", phase_ev[k].first, phase_host[k] - phase_host[k - 1]);
    fprintf(stderr, "\n");
  }
  fprintf(stderr, "[rq phases] total %.2f ms:", tot);
  for (int i = 1; i < 13; i++)
    if (acc[i] > 0) fprintf(stderr, " %s=%.2f", names[i], acc[i]);
  fprintf(stderr, "\n");
  for (auto& pe : phase_ev) cudaEventDestroy(pe.second);
  phase_ev.clear();
  phase_host.clear();
  if (!side_ev.empty()) {
    // side stream: id 0 = CPQR done (start of W), 1 = capped W part, 2 = rest of W, 3 = T
    double sacc[4] = {0};
    cudaEventSynchronize(side_ev.back().second);
    for (size_t k = 1; k < side_ev.size(); k++) {
      if (side_ev[k].first == 0) continue;
      float ms = 0.f;
      cudaEventElapsedTime(&ms, side_ev[k - 1].second, side_ev[k].second);
      sacc[side_ev[k].first] += ms;
    }
    fprintf(stderr, "[rq side] W capped=%.2f W rest=%.2f T=%.2f\n", sacc[1], sacc[2], sacc[3]);
    for (auto& pe : side_ev) cudaEventDestroy(pe.second);
    side_ev.clear();
  }
}

// Pending look-ahead tiles [la.next, upto): beside a leaf kernel (programmatic dependent launch,
// grid capped to the SMs outside the leaf's 16-CTA cluster) or, at the end, on the whole GPU.
int Ctx::la_chunk(int64_t upto, bool beside_leaf) {
  if (!la.on) return RQ_OK;
  upto = std::min(upto, la.tiles);
  if (upto > la.next) {
    GemmProblem p = la.g;
    p.tile_begin = la.next;
    p.tile_end = upto;
    p.work = nullptr;  // no split-K inside a tile range
    p.work_bytes = 0;
    p.splitk = 1;
    static const int env_pdl = [] {
      const char* e = getenv("RQ_LA_PDL");
      return e ? atoi(e) : 1;
    }();
    p.max_ctas = beside_leaf ? kSMs - 16 : 0;
    p.pdl = beside_leaf && env_pdl != 0;
    RQ_TRY(sched_for(stream, &p.sched, &p.sched_base));
    CatGuard g(cat, PROF_TRAIL);
    // (in a profiled step the events between the leaf and its chunk serialise them: the per-class
    //  breakdown is taken from a separate step, never from the timed ones)
    cudaEvent_t e0;
    prof_begin(&e0);
    const int rc = tf32_update ? gemm_tf32x3_f64(p, stream, &launches) : gemm_f64(p, stream, &launches);
    prof_end(e0, 2.0 * (double)p.M * (double)p.N * (double)p.K * (double)(upto - la.next) / (double)la.tiles);
    RQ_TRY(rc);
    la.next = upto;
  }
  if (la.next >= la.tiles) la.on = false;
  return RQ_OK;
}

int Ctx::ensure_side() {
  if (side) return RQ_OK;
  int lo = 0, hi = 0;
  RQ_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  RQ_CUDA_TRY(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, lo));
  RQ_CUDA_TRY(cudaStreamCreateWithPriority(&hip, cudaStreamNonBlocking, hi));
  RQ_CUDA_TRY(cudaStreamCreateWithPriority(&hip2, cudaStreamNonBlocking, hi));
  RQ_CUDA_TRY(cudaEventCreateWithFlags(&ev_q2, cudaEventDisableTiming));
  RQ_CUDA_TRY(cudaEventCreateWithFlags(&ev_gram, cudaEventDisableTiming));
  RQ_CUDA_TRY(cudaEventCreateWithFlags(&ev_t, cudaEventDisableTiming));
  RQ_CUDA_TRY(cudaEventCreateWithFlags(&ev_v, cudaEventDisableTiming));
  RQ_CUDA_TRY(cudaEventCreateWithFlags(&ev_side, cudaEventDisableTiming));
  RQ_CUDA_TRY(cudaEventCreateWithFlags(&ev_hi, cudaEventDisableTiming));
  RQ_CUDA_TRY(cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking));
  RQ_CUDA_TRY(cudaEventCreateWithFlags(&ev_w2, cudaEventDisableTiming));
  RQ_CUDA_TRY(cudaEventCreateWithFlags(&ev_l0, cudaEventDisableTiming));
  RQ_CUDA_TRY(cudaEventCreateWithFlags(&ev_aux, cudaEventDisableTiming));
  RQ_CUDA_TRY(cudaEventCreateWithFlags(&ev_g1, cudaEventDisableTiming));
  RQ_CUDA_TRY(cudaEventCreateWithFlags(&ev_hipdone, cudaEventDisableTiming));
  return RQ_OK;
}

int Ctx::sweep(SweepCall c) {
  cudaEvent_t e0;
  const int saved = cat;
  cat = (c.n_acc > 0 || c.r_out) ? PROF_SMALL : PROF_SWEEP;
  prof_begin(&e0);
  int rc = sweep_raw(c);
  prof_end(e0, 0.0);
  cat = saved;
  return rc;
}

int Ctx::sketch_select(const double* yt, int64_t ldy, int m, int n, int steps, const int* init_pos, int* chosen) {
  if (m > 1024) {
    SweepCall sc;
    sc.a = const_cast<double*>(yt);
    sc.lda = ldy;
    sc.m = m;
    sc.n = n;
    sc.steps = steps;
    sc.pivot = 1;
    sc.init_pos = init_pos;
    sc.col_at_pos = chosen;
    return sweep(sc);
  }
  RQ_TRY(place_sketch_words(m, n, steps));
  cudaEvent_t e0;
  const int saved = cat;
  cat = PROF_SWEEP;
  if (sketch_batched(m, n, steps, sketch_gmax)) {
    if (!sb_ws) {
      RQ_CUDA_TRY(cudaMalloc(&sb_ws, sketch_batch_workspace_bytes()));
      RQ_CUDA_TRY(cudaMemsetAsync(sb_ws, 0, sketch_batch_workspace_bytes(), stream));
    }
    prof_begin(&e0);
    const int rc = sketch_batch_launch(yt, ldy, m, n, steps, init_pos, chosen, sb_ws, sb_stamp_base, stream, &launches,
                                       sketch_gmax);
    prof_end(e0, 0.0);
    cat = saved;
    if (rc >= 0) return rc;
  }
  prof_begin(&e0);
  SweepWork w;
  w.scratch = sweep_ws;
  w.scratch_bytes = sweep_ws_bytes;
  w.ll = sk_ll;
  const int rc = sketch_cpqr_launch(yt, ldy, m, n, steps, init_pos, chosen, w, sk_counter, sk_counter_base, stream,
                                    &launches, sketch_gmax);
  prof_end(e0, 0.0);
  cat = saved;
  return rc;
}

// The sketch CPQR's winner record -- one line written by the reducer CTA and polled by every
// other CTA each step -- costs ~0.8 us more per step at some addresses than at others (B200,
// n' = 10k: 4.55 vs 5.4 us per step; e.g. fast at offsets 0, 64 KB, 3 MB of a block and slow at
// 4 KB, 128 KB, 1 MB, 2 MB: the line's L2 slice / die relative to the reducer).  cudaMalloc gives
// no control over that, and the address a 256-byte allocation gets shifts with whatever the
// process allocated before (a context created after PyTorch's stream pool landed on a slow line:
// 136.9 instead of 129.1 ms per n = 10k factorization).  So the context allocates a block once,
// times a short sketch CPQR with the record at 16 offsets of it and keeps the fastest
// (RQ_SK_PLACE_CAL=0: offset 0; 2: print the timings).
int Ctx::place_sketch_words(int m, int n, int steps) {
  static const int env_cal = [] {
    const char* e = getenv("RQ_SK_PLACE_CAL");
    return e ? atoi(e) : 1;
  }();
  constexpr int kCand = 16;
  constexpr size_t kStride = 4096;
  if (!sk_block) {
    // [16 candidate winner records][slots + LL columns (b + p <= 288) + 16 candidate offsets]
    const size_t llb = sketch_ll_bytes(288) + kCand * kStride;
    RQ_CUDA_TRY(cudaMalloc(&sk_block, kCand * kStride + llb));
    RQ_CUDA_TRY(cudaMemsetAsync(sk_block, 0, kCand * kStride + llb, stream));
    sk_counter = reinterpret_cast<unsigned long long*>(sk_block);
    sk_ll = sk_block + kCand * kStride;
  }
  char* blk = sk_block;
  char* ll0 = sk_block + kCand * kStride;
  // (small problems never repay the one-off ~6 ms: calibrate at the first sizeable sketch)
  if (sk_placed || env_cal == 0 || m > 288 || n < 2048 || steps < 32) return RQ_OK;
  sk_placed = true;
  const int cn = 2048, csteps = 32;
  const size_t ws = sketch_workspace_bytes(m, cn) + 4096;
  const int64_t ldc = even(m);
  double* ycal = nullptr;
  void* wcal = nullptr;
  int* ccal = nullptr;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  auto cleanup = [&] {
    if (ycal) cudaFree(ycal);
    if (wcal) cudaFree(wcal);
    if (ccal) cudaFree(ccal);
    if (t0) cudaEventDestroy(t0);
    if (t1) cudaEventDestroy(t1);
  };
  if (cudaMalloc(&ycal, (size_t)ldc * cn * 8) != cudaSuccess || cudaMalloc(&wcal, ws) != cudaSuccess ||
      cudaMalloc(&ccal, 1024) != cudaSuccess || cudaEventCreate(&t0) != cudaSuccess ||
      cudaEventCreate(&t1) != cudaSuccess) {
    cleanup();
    cudaGetLastError();
    return RQ_OK;  // no calibration: offset 0
  }
  cudaMemsetAsync(wcal, 0, ws, stream);
  int rc = gaussian_fill(ycal, m, cn, ldc, 0x5eedULL, 0, stream, nullptr);
  SweepWork w;
  w.scratch = wcal;
  w.scratch_bytes = ws;
  w.ll = ll0;
  float tms[kCand], tll[kCand];
  int best = 0, best_ll = 0;
  auto time_one = [&](unsigned long long* ctr, int ncols) {
    float best_ms = 1e30f;
    for (int rep = 0; rep < 3 && rc == RQ_OK; rep++) {
      // (the arrival counter of RQ_SK_FIXED_REDUCER=0 must equal the host mirror at launch)
      if (cudaMemcpyAsync(ctr, &sk_counter_base, 8, cudaMemcpyHostToDevice, stream) != cudaSuccess ||
          cudaStreamSynchronize(stream) != cudaSuccess) {
        rc = set_error(RQ_ECUDA, "sketch counter");
        break;
      }
      cudaEventRecord(t0, stream);
      rc = sketch_cpqr_launch(ycal, ldc, m, ncols, csteps, nullptr, ccal, w, ctr, sk_counter_base, stream, nullptr, 0);
      cudaEventRecord(t1, stream);
      if (rc == RQ_OK && cudaStreamSynchronize(stream) != cudaSuccess) rc = set_error(RQ_ECUDA, "calibration run");
      float ms = 0.0f;
      if (rc == RQ_OK && rep > 0 && cudaEventElapsedTime(&ms, t0, t1) == cudaSuccess) best_ms = std::min(best_ms, ms);
    }
    return best_ms;
  };
  // two grid sizes (128 and 63 CTAs: the slots span two 4 KB chunks or one), mean of both
  auto time_run = [&](unsigned long long* ctr, float* out) { *out = 0.5f * (time_one(ctr, cn) + time_one(ctr, 1008)); };
  // (1) the winner record's offset, (2) with it, the offset of the slots + LL columns (the reducer
  // polls every CTA's slot each step; 4.39-4.67 us per step at n' = 10k, 3.06-3.62 at n' = 1k)
  for (int i = 0; i < kCand && rc == RQ_OK; i++) {
    time_run(reinterpret_cast<unsigned long long*>(blk + i * kStride), &tms[i]);
    if (tms[i] < tms[best]) best = i;
  }
  for (int i = 0; i < kCand && rc == RQ_OK; i++) {
    w.ll = ll0 + i * kStride;
    time_run(reinterpret_cast<unsigned long long*>(blk + best * kStride), &tll[i]);
    if (tll[i] < tll[best_ll]) best_ll = i;
  }
  if (rc == RQ_OK) {
    sk_ll = ll0 + best_ll * kStride;
    sk_counter = reinterpret_cast<unsigned long long*>(blk + best * kStride);
    // every candidate's arrival counter saw its own launches only: set the chosen one to the
    // host mirror (the stamps keep growing: records and slots written so far stay in the past)
    if (cudaMemcpyAsync(sk_counter, &sk_counter_base, 8, cudaMemcpyHostToDevice, stream) != cudaSuccess ||
        cudaStreamSynchronize(stream) != cudaSuccess)
      rc = set_error(RQ_ECUDA, "sketch counter");
    if (env_cal == 2) {
      fprintf(stderr, "[rq] sketch CPQR winner-record placement (us/step at 4 KB offsets):");
      for (int i = 0; i < kCand; i++) fprintf(stderr, " %.2f", tms[i] * 1e3f / csteps);
      fprintf(stderr, " -> offset %d KB; slots + LL columns:", best * 4);
      for (int i = 0; i < kCand; i++) fprintf(stderr, " %.2f", tll[i] * 1e3f / csteps);
      fprintf(stderr, " -> offset %d KB\n", best_ll * 4);
    }
  }
  cleanup();
  return rc;
}

// RQ_SK_BATCH=1: the batched sketch CPQR (sketch_batch.cu) where the shape fits.  Same pivots as
// the per-step kernel; measured at parity with it (n' = 10k: 4.9 vs 4.5 us/step, 20k: 7.8 vs 7.8,
// its solver step costs as much as the exchanges it saves), so it stays opt-in.
bool Ctx::sketch_batched(int m, int n, int steps, int gmax) const {
  static const int env_sb = [] {
    const char* e = getenv("RQ_SK_BATCH");
    return e ? atoi(e) : 0;
  }();
  return env_sb != 0 && m <= 288 && sketch_batch_fits(m, n, steps, gmax);
}

int Ctx::sweep_raw(SweepCall c) {
  SweepWork w;
  w.scratch = sweep_ws;
  w.scratch_bytes = sweep_ws_bytes;
  w.barriers = barriers;
  w.nbarriers = nbarriers;
  w.next = next_barrier;
  int rc = sweep_launch(c, w, stream, &launches);
  next_barrier = w.next;
  if (w.wrapped) {
    // ring wrapped: re-zero (stream-ordered after every launch that used it)
    RQ_CUDA_TRY(cudaMemsetAsync(barriers, 0, sizeof(unsigned) * nbarriers, stream));
    launches++;
  }
  return rc;
}

// ---------------------------------------------------------------------------
// Panel QR of A[s:, s:s+b] (m' x b): leaf kernels + WY updates of the rest.
// ---------------------------------------------------------------------------
int Ctx::panel_qr(double* A, int64_t lda, int64_t m, int64_t n, int64_t s, int64_t mp, int b, double* V, int64_t ldv,
                  int vpad, double* tleaf, double* w1, double* w2, double* T, int64_t ldt, bool* t_done) {
  if (t_done) *t_done = false;
  CatGuard guard(cat, PROF_PANEL_GEMM);
  int wl_max = leaf_reg_width_for(mp);
  if (wl_max == 0) wl_max = leaf_width_for(mp);
  if (wl_max == 0) {
    // A panel taller than one 16-CTA cluster holds (m' > 65536 rows): the grid-wide Householder
    // sweep, unpivoted (householder_sweep(pivot=False), _kernels_numba.py:13-61), on the whole
    // panel; columns stream through L2 each step.  Same reflector convention as the leaves.
    RQ_TRY(la_flush());
    SweepCall sc;
    sc.a = A + s + s * lda;
    sc.lda = lda;
    sc.m = mp;
    sc.n = b;
    sc.steps = (int)std::min<int64_t>(mp, b);
    sc.pivot = 0;
    sc.v = V + vpad;
    sc.ldv = ldv;
    return sweep(sc);
  }
  const int wl = std::min(wl_max, 32);
  // look-ahead: spread the pending tiles over the leaves in whole waves of the capped grid
  const int nleaves = (b + wl - 1) / wl;
  const int64_t la_wave = kSMs - 16;
  const int64_t la_t0 = la.next, la_waves = la.on ? ceil_div(la.tiles - la.next, la_wave) : 0;
  // Space-sliced look-ahead: when the pending trailing update outlasts this panel's leaves and
  // WY updates, run ALL of it as one 132-CTA launch beside the first leaf and keep the rest of
  // the panel (leaves + wy_cluster updates) on the first leaf's 16 SMs on the `aux` stream;
  // otherwise (time-sliced) the chunks run beside each leaf and the WY updates take the GPU.
  // RQ_LA_SPACE: 0 time-sliced, 1 space-sliced, 2 (default) by the estimate below.
  static const int env_space = [] {
    const char* e = getenv("RQ_LA_SPACE");
    return e ? atoi(e) : 2;
  }();
  bool space = false, t_on_aux = false;
  if (la.on && env_space != 0 && nleaves > 1) {
    // (the tcgen05 3xTF32 update of the fp32 mode runs ~2x the in-situ DMMA rate)
    const double nn_rate = tf32_update ? 48e12 : 24e12;
    const double nn_s = 2.0 * (double)la.g.M * (double)la.g.N * (double)la.g.K *
                        ((double)(la.tiles - la.next) / (double)la.tiles) / nn_rate;
    double rest_cols = 0.0;
    for (int k0 = wl; k0 < b; k0 += wl) rest_cols += (double)(b - k0);
    // leaves ~3.6 us per column plus the cluster WY updates at a nominal 110 GB/s per SM (they
    // measure ~20: this optimistic estimate picked the better schedule at n = 10k and 20k:
    // 148.6 / 586.7 ms, against 148.8 / 619.1 with the measured rate)
    const double leaf_s = (double)b * 3.6e-6 + 3.0 * ((double)mp / 16.0) * 8.0 * rest_cols / 110e9 +
                          (double)nleaves * 8e-6;
    space = env_space == 1 || nn_s > 1.15 * leaf_s;
    // and the panel's T on the same 16 SMs when the trailing update still outlasts that too
    const double t_s = 2.0 * (double)mp * (double)b * (double)b / (16.0 * 0.15e12) + 60e-6;
    t_on_aux = space && nn_s > 1.5 * (leaf_s + t_s);
  }
  cudaStream_t saved_stream = stream;
  for (int k0 = 0; k0 < b; k0 += wl) {
    const int w = std::min(wl, b - k0);
    const int64_t mm = mp - k0;
    LeafCall lc;
    lc.a = A + (s + k0) + (s + k0) * lda;
    lc.lda = lda;
    lc.mm = mm;
    lc.w = w;
    lc.v = V + vpad + k0 + (int64_t)k0 * ldv;
    lc.ldv = ldv;
    lc.tl = tleaf;
    lc.ldt = 32;
    {
      cudaEvent_t e0;
      const int saved = cat;
      cat = PROF_LEAF;
      prof_begin(&e0);
      const int rc = leaf_qr(lc, stream, &launches);
      prof_end(e0, 0.0);
      cat = saved;
      RQ_TRY(rc);
    }
    if (space && k0 == 0) {
      RQ_TRY(ensure_side());
      RQ_CUDA_TRY(cudaEventRecord(ev_l0, stream));  // completes with the first leaf
      RQ_TRY(la_chunk(la.tiles, true));               // all of it, beside the first leaf
      RQ_CUDA_TRY(cudaStreamWaitEvent(aux, ev_l0, 0));
      stream = aux;
    } else if (la.on && !space) {
      const int64_t leaf = k0 / wl + 1;
      RQ_TRY(la_chunk(la_t0 + ceil_div(la_waves * leaf, (int64_t)nleaves) * la_wave, true));
    }
    const int64_t nrest = b - k0 - w;
    if (nrest <= 0) break;
    // A_rest -= V_l T_l^T (V_l^T A_rest)
    if (space) {
      cudaEvent_t e0;
      prof_begin(&e0);
      const int rc = wy_cluster(A, lda, m, n, s + k0, s + k0 + w, mm, (int)nrest, V, ldv, mp + vpad, b, vpad + k0, k0,
                                tleaf, 32, w, stream, &launches);
      prof_end(e0, 4.0 * (double)mm * w * nrest);
      RQ_TRY(rc);
    } else if (wy_update_fits(mm, (int)nrest, w)) {
      cudaEvent_t e0;
      prof_begin(&e0);
      SweepWork sw;
      sw.barriers = barriers;
      sw.nbarriers = nbarriers;
      sw.next = next_barrier;
      unsigned int* bar = sw.next_barrier();
      next_barrier = sw.next;
      int rc = wy_update(A + (s + k0) + (s + k0 + w) * lda, lda, mm, (int)nrest, V + vpad + k0 + (int64_t)k0 * ldv, ldv,
                         tleaf, 32, w, kwork, kwork_bytes, bar, stream, &launches);
      if (sw.wrapped) {
        RQ_CUDA_TRY(cudaMemsetAsync(barriers, 0, sizeof(unsigned) * nbarriers, stream));
        launches++;
      }
      prof_end(e0, 4.0 * (double)mm * w * nrest);
      RQ_TRY(rc);
    } else {
      const int64_t ldw = even(w);
      RQ_TRY(gemm(w, nrest, mm, op(V, mp + vpad, b, ldv, vpad + k0, k0), false, op(A, m, n, lda, s + k0, s + k0 + w),
                  w1, ldw, 1.0, 0.0));
      RQ_TRY(gemm(w, nrest, w, op(tleaf, 32, 32, 32), false, op(w1, w, nrest, ldw), w2, ldw, 1.0, 0.0));
      RQ_TRY(gemm(mm, nrest, w, op(V, mp + vpad, b, ldv, vpad + k0, k0), true, op(w2, w, nrest, ldw),
                  A + (s + k0) + (s + k0 + w) * lda, lda, -1.0, 1.0));
    }
  }
  if (space && t_on_aux && T && t_done) {
    // the panel's T on the same 16 SMs, while the trailing update still holds the others (it
    // outlasts the leaves here); the main stream's split-K slabs and Gram scratch are idle now
    static const int env_taux = [] {
      const char* e = getenv("RQ_T_AUX");
      return e ? atoi(e) : 1;
    }();
    if (env_taux) {
      gemm_max_ctas = 16;
      const int rc = tfactor(V, mp, b, ldv, vpad, T, ldt, gram_aux);
      gemm_max_ctas = 0;
      RQ_TRY(rc);
      *t_done = true;
    }
  }
  if (space && aux_g1 && t_on_aux) {  // the downdate's G1' too (form_g1), on the same 16 SMs
    gemm_max_ctas = 16;
    const int rc = aux_g1();
    gemm_max_ctas = 0;
    RQ_TRY(rc);
    g1_done = true;
  }
  if (space) {  // the main stream continues once the panel is factored (its chunk is in order)
    stream = saved_stream;
    RQ_CUDA_TRY(cudaEventRecord(ev_aux, aux));
    RQ_CUDA_TRY(cudaStreamWaitEvent(stream, ev_aux, 0));
  }
  return RQ_OK;
}

// Q2 = H'_0 ... H'_{k-1} = I - V2 T2 V2^T (k x k), dense, from the b x b CPQR reflectors.
int Ctx::small_q(const double* V2, int64_t ldv2, int k, double* Q2, int64_t ldq, Layout& L) {
  CatGuard guard(cat, PROF_TFACTOR);
  static const int env_q = [] {
    const char* e = getenv("RQ_SMALLQ_GEMM");  // 1: the compact-WY path below
    return e ? atoi(e) : 0;
  }();
  if (env_q == 0 && k <= 256) {
    cudaEvent_t e0;
    prof_begin(&e0);
    const int rc = q_from_reflectors(V2, ldv2, k, k, Q2, ldq, stream, &launches);
    prof_end(e0, 2.0 * k * (double)k * k);
    return rc;
  }
  double* T2s = L.ttop;  // k x k scratch (free until the trailing update)
  const int64_t ldk = even(k);
  RQ_TRY(tfactor(V2, k, k, ldv2, 0, T2s, ldk, L.gram));
  RQ_TRY(fill_eye(Q2, ldq, k, k, 0, stream, &launches));
  // W = V2^T I ; W2 = T2 W ; Q2 -= V2 W2
  RQ_TRY(gemm(k, k, k, op(V2, k, k, ldv2), false, op(Q2, k, k, ldq), L.w1, ldk, 1.0, 0.0));
  RQ_TRY(gemm(k, k, k, op(T2s, k, k, ldk), true, op(L.w1, k, k, ldk), L.w2, ldk, 1.0, 0.0));
  RQ_TRY(gemm(k, k, k, op(V2, k, k, ldv2), true, op(L.w2, k, k, ldk), Q2, ldq, -1.0, 1.0));
  return RQ_OK;
}

// T (k x k) of the reflectors V (rows x k): Gram by DMMA GEMM, then back substitution.
int Ctx::tfactor(const double* V, int64_t rows, int k, int64_t ldv, int vpad, double* T, int64_t ldt, double* gram) {
  CatGuard guard(cat, PROF_TFACTOR);
  cudaEvent_t e0;
  prof_begin(&e0);
  const int64_t ldg = even(k);
  RQ_TRY(gemm(k, k, rows, op(V, rows + vpad, k, ldv, vpad), false, op(V, rows + vpad, k, ldv, vpad), gram, ldg, 1.0,
              0.0));
  const int rc = tfactor_from_gram(gram, ldg, k, T, ldt, stream, &launches);
  prof_end(e0, 0.0);
  return rc;
}

// A[:, s:s+np] <- A[:, s:s+np] (I - V_S T_S V_S^T) on `rows` rows (apply_wy_right,
// householder.py:117-124, at full height as blocked.py:205/261 do).
int Ctx::apply_right_wy(double* A, int64_t lda, int64_t rows, int64_t ncols_total, int64_t s, int64_t np, int k,
                        const double* VS, int64_t ldvs, const double* TS, int64_t ldts, double* vst, double* z,
                        double* z2, int64_t ldz) {
  const int64_t ldk = even(k);
  RQ_TRY(transpose(VS, ldvs, vst, ldk, np, k, stream, &launches));
  RQ_TRY(gemm(rows, k, np, op(A, rows, ncols_total, lda, 0, s), true, op(VS, np, k, ldvs), z, ldz, 1.0, 0.0));
  RQ_TRY(gemm(rows, k, k, op(z, rows, k, ldz), true, op(TS, k, k, ldts), z2, ldz, 1.0, 0.0));
  return gemm(rows, np, k, op(z2, rows, k, ldz), true, op(vst, k, np, ldk), A + s * lda, lda, -1.0, 1.0);
}

// ---------------------------------------------------------------------------
// block_qr with permutation pivots, fresh sketches (reference semantics)
// ---------------------------------------------------------------------------
int Ctx::factorize_perm(const rq_config& cfg, int64_t m, int64_t n, double* A, int64_t lda, uint64_t seed,
                        uint64_t* counter, int64_t* dperm) {
  const int b = cfg.block, p = cfg.oversample, wdt = b + p;
  size_t need = plan_layout(nullptr, m, n, b, p, cfg.power).total;
  RQ_TRY(arena.reserve(need));
  Layout L = plan_layout(arena.base, m, n, b, p, cfg.power);
  kwork = L.kwork;
  kwork_bytes = L.kwork_bytes;
  sweep_ws = L.sweep_ws;
  sweep_ws_bytes = L.sweep_ws_bytes;
  cur_A = A;
  cur_lda = lda;
  cur_m = m;
  cur_n = n;
  cur_orig = L.orig;
  cur_yt = cfg.sketch_mode == RQ_SKETCH_DOWNDATE ? L.yt : nullptr;
  cur_ldy = L.ldy;
  cur_wdt = wdt;

  have_factors = false;  // a failed run leaves nothing readable
  factors.clear();
  rfactors.clear();
  const bool refl_piv = cfg.pivot_kind == RQ_PIVOT_REFLECTORS;
  p_is_perm = !refl_piv;
  factors_perm = L.orig;
  fm = m;
  fn = n;
  fb = b;

  RQ_TRY(iota(L.lorderA, (int)n, L.orig, n, stream, &launches));
  RQ_TRY(iota(L.rankA, (int)n, nullptr, 0, stream, &launches));
  RQ_TRY(iota(L.iota_b, (int)std::max<int64_t>(b, n), nullptr, 0, stream, &launches));
  int* lorder = L.lorderA;
  int* lorder_n = L.lorderB;
  int* rank = L.rankA;
  int* rank_n = L.rankB;
  Carver fc(L.fstore);
  double* tleaf = L.tleaf;

  const bool downdate = cfg.sketch_mode == RQ_SKETCH_DOWNDATE;
  // look-ahead (downdated sketches, permutation pivots): the next panel's sketch CPQR and column
  // moves run as soon as the top b rows (R12) are final, the next panel's columns are updated
  // first, and the rest of A2 -= V W2 runs in chunks beside the next panel's leaf kernels.
  static const int env_la = [] {
    const char* e = getenv("RQ_LOOKAHEAD");
    return e ? atoi(e) : 1;
  }();
  const bool la_mode = downdate && !refl_piv && !inspect_cb && env_la != 0 && !(cfg.flags & RQ_FLAG_NO_LOOKAHEAD);
  la.on = false;
  static const bool env_phases = getenv("RQ_PHASES") && atoi(getenv("RQ_PHASES")) != 0;
  phases_on = env_phases && !prof;
  phase(0);
  if (downdate && n > b) {
    // HQRRP: G = Omega^T drawn once (m(b+p) normals), Y = G A; downdated per panel
    // (rq_factorize_host forms both while A's column chunks arrive: presketch_begin / _cols)
    if (!presketched) {
      RQ_TRY(gaussian_fill_p(L.omega, m, wdt, L.ldo, seed, *counter, stream, &launches));
      RQ_TRY(gemm(wdt, n, m, op(L.omega, m, wdt, L.ldo), false, op(A, m, n, lda, 0, 0), L.yt, L.ldy, 1.0, 0.0));
    }
    *counter += (uint64_t)m * (uint64_t)wdt;
  }
  presketched = false;
  int panel = 0;
  for (int64_t s = 0; s < n; s += b) {
    panel++;
    const int64_t mp = m - s, np = n - s;
    cur_s = s;
    cur_lorder = lorder;
    cur_np = np;
    if (np <= b) {
      // ---------------- final block: CPQR at full height ----------------
      const int w = (int)np;
      const int steps = (int)std::min<int64_t>(mp, w);
      // bring the remaining columns into reference order
      MoveCall mv{A, lda, s, 0, m, lorder, L.iota_b, nullptr, w, L.stage, even(m), L.orig, L.ostage};
      RQ_TRY(move_columns_p(mv, stream, &launches));
      const int64_t ldv = even(mp + 1);
      const int vpad = (int)(s & 1);
      double* Vf = fc.take<double>((size_t)ldv * steps);
      double* Tf = fc.take<double>((size_t)even(b) * b);
      RQ_CUDA_TRY(cudaMemsetAsync(Vf, 0, (size_t)ldv * steps * 8, stream));
      launches++;
      SweepCall sc;
      sc.a = A + s + s * lda;
      sc.lda = lda;
      sc.m = mp;
      sc.n = w;
      sc.steps = steps;
      sc.pivot = 1;
      sc.v = Vf + vpad;
      sc.ldv = ldv;
      sc.col_at_pos = L.cap;
      sc.r_out = L.stage;
      sc.ldr = even(mp);
      RQ_TRY(sweep(sc));
      RQ_TRY(copy2d_p(L.stage, even(mp), A + s + s * lda, lda, mp, w, 0, stream, &launches));
      // rows above and labels follow the final block's permutation
      MoveCall mv2{A, lda, s, 0, s, L.cap, L.iota_b, nullptr, w, L.stage, even(m), L.orig, L.ostage};
      RQ_TRY(move_columns_p(mv2, stream, &launches));
      RQ_TRY(tfactor(Vf, mp, steps, ldv, vpad, Tf, even(b), L.gram));
      factors.push_back(PanelFactors{s, steps, Vf, ldv, vpad, Tf, even(b), nullptr, 0});
      if (refl_piv) {
        int* phat = fc.take<int>((size_t)w);
        RQ_CUDA_TRY(cudaMemcpyAsync(phat, L.cap, (size_t)w * sizeof(int), cudaMemcpyDeviceToDevice, stream));
        rfactors.push_back(RightFactors{s, np, 0, nullptr, 0, nullptr, 0, phat, w, nullptr, 0, 0});
      }
      RQ_TRY(iota(lorder, (int)np, nullptr, 0, stream, &launches));
      if (on_cols_final) on_cols_final(s, np);
      if (inspect_cb) {
        cur_lorder = nullptr;
        RQ_CUDA_TRY(cudaStreamSynchronize(stream));
        inspect_cb(panel, inspect_user);
      }
      break;
    }
    if (refl_piv) {
      // ---------------- reflector pivots (select_pivot_reflectors, pivoting.py:132-146) ----------------
      RQ_TRY(reflector_pivot(cfg, A, lda, m, n, s, L, &fc, seed, counter));
      rfactors.back().nphat = b;
    } else if (!(la_mode && panel > 1)) {  // (look-ahead: selected and moved at the end of the last panel)
    // ---------------- 1-2: sketch Y^T = Omega^T X (fresh) or the downdated Y (HQRRP) ----------------
    double* ycur = L.yt;
    if (!downdate) {
      RQ_TRY(gaussian_fill_p(L.omega + (s & 1), mp, wdt, L.ldo, seed, *counter, stream, &launches));
      *counter += (uint64_t)mp * (uint64_t)wdt;
      RQ_TRY(sketch(cfg, A, lda, m, n, s, mp, np, L));
    } else {
      ycur = L.yt + s * L.ldy;
      // the CPQR overwrites its input: work on a copy of the trailing sketch columns
      RQ_TRY(copy2d_p(ycur, L.ldy, L.ybuf, L.ldy, wdt, np, 0, stream, &launches));
    }
    // ---------------- 3: b-step CPQR of Y^T ----------------
    RQ_TRY(sketch_select(downdate ? L.ybuf : L.yt, L.ldy, wdt, (int)np, b, rank, L.cap));
    // ---------------- 4: move the chosen columns into the panel ----------------
    PlanCall pc{L.cap, b, lorder, (int)np, L.flag, L.newloc, L.src, L.dst, L.nmoves, lorder_n, rank_n};
    RQ_TRY(plan_moves(pc, stream, &launches));
    MoveCall mv{A, lda, s, 0, m, L.src, L.dst, L.nmoves, 2 * b, L.stage, even(m), L.orig, L.ostage};
    RQ_TRY(move_columns_p(mv, stream, &launches));
    if (downdate) {  // the sketch columns follow their matrix columns
      MoveCall my{L.yt, L.ldy, s, 0, wdt, L.src, L.dst, L.nmoves, 2 * b, L.stage, L.ldy, nullptr, nullptr};
      RQ_TRY(move_columns_p(my, stream, &launches));
    }
    }  // permutation pivots
    phase(la_mode ? 7 : 9);
    // ---------------- 5: unpivoted panel QR ----------------
    const int64_t ldv = even(mp + 1), ldt = even(b);
    const int vpad = (int)(s & 1);
    double* V = fc.take<double>((size_t)ldv * b);
    double* T = fc.take<double>((size_t)ldt * b);
    double* Q2 = fc.take<double>((size_t)ldt * b);
    // V is lower trapezoidal: the leaves write rows >= their diagonal only
    RQ_CUDA_TRY(cudaMemsetAsync(V, 0, (size_t)ldv * b * sizeof(double), stream));
    launches++;
    // (look-ahead: L.w2 holds the previous panel's W2 until its last chunk ran; ttop is free)
    gram_aux = L.gram;
    bool t_done = false;
    g1_done = false;
    if (downdate && !refl_piv && np > b) {  // G1' from R'11 and the selected sketch columns (form_g1)
      aux_g1 = [this, A, lda, s, b, wdt, n, &L]() { return form_g1(A, lda, s, b, wdt, n, L); };
    }
    RQ_TRY(panel_qr(A, lda, m, n, s, mp, b, V, ldv, vpad, tleaf, L.w1, la_mode ? L.ttop : L.w2, T, ldt, &t_done));
    // G1' not formed on aux: with the overlap below it runs on the high-priority stream once the
    // b x b CPQR is done (beside the rest of W); otherwise here
    static const int env_hip = [] {
      const char* e = getenv("RQ_HIP_TAIL");
      return e ? atoi(e) : 1;
    }();
    const bool hip_tail = env_hip != 0 && overlap_on && np - b > 0;
    // and the panel's T there too (instead of after W on the side stream): RQ_T_HIP=1; measured
    // slower (n = 10k 146.7 -> 148.7 ms: its Gram GEMM competes with the rest of W), so off
    static const int env_thip = [] {
      const char* e = getenv("RQ_T_HIP");
      return e ? atoi(e) : 0;
    }();
    const bool t_on_hip = hip_tail && env_thip != 0 && !t_done;
    if (aux_g1 && (g1_done || !hip_tail)) {
      if (!g1_done) RQ_TRY(aux_g1());
      aux_g1 = nullptr;
    }
    RQ_TRY(la_flush());
    phase(1);
    const int64_t n2 = np - b;
    // ---- overlap: the b x b CPQR below runs on its 16-SM cluster from a highest-priority
    //      stream (so it is dispatched first), while W = V^T A2 (half the trailing update)
    //      and T run on the remaining SMs from a side stream ----
    static const int env_overlap = [] {
      const char* e = getenv("RQ_OVERLAP");
      return e ? atoi(e) : 1;
    }();
    const bool overlap = overlap_on && env_overlap != 0 && n2 > 0;
    // RQ_W2_SIDE=1: W2 = T^T W on the side stream after T, the top rows from (V_top T^T) W on the
    // main stream; measured even with the default (n = 10k 146.5 vs 146.5 ms, 20k 576 vs 575)
    static const int env_w2s = [] {
      const char* e = getenv("RQ_W2_SIDE");
      return e ? atoi(e) : 0;
    }();
    w2_side = overlap && la_mode && env_w2s != 0 && !(t_on_hip && hip_tail);
    // RQ_CPQR_OFF=1: the b x b CPQR and its follow-ups (Q2, R, rows-above moves) leave the critical
    // path -- the tail waits for W and T only, and the next panel's sketch CPQR (capped at
    // kSkMinGrid CTAs) runs beside the CPQR's 16-SM cluster; the downdate uses R'12, so it needs
    // neither Q2 nor P-hat (form_g1)
    static const int env_off = [] {
      const char* e = getenv("RQ_CPQR_OFF");
      return e ? atoi(e) : 1;
    }();
    // Only where the CPQR outlasts W = V^T A2 (the late panels): the capped sketch grid costs
    // ~25 % per step at n' ~ 10k, and early panels hide the CPQR behind W anyway.
    // (threshold re-tuned with T on the aux stream: 20 -> 30 TF/s, n = 10k 131.3 -> 130.8 ms)
    static const double env_off_tf = getenv("RQ_CPQR_OFF_TF") ? atof(getenv("RQ_CPQR_OFF_TF")) : 30.0;
    const double w_s = 2.0 * b * (double)mp * (double)n2 / (env_off_tf * 1e12);
    const double cpqr_s = b * 2.2e-6;
    cpqr_off = la_mode && overlap && env_off != 0 && b <= 256 && !w2_side && !t_on_hip &&
               (env_off == 2 || w_s < cpqr_s) && hip2 != nullptr;
    // ---------------- 6: b x b CPQR of R' (reflectors V2), then Q2 = I - V2 T2 V2^T ----------------
    double* S = L.small;
    double* V2 = L.small + (int64_t)b * L.lds_small;
    RQ_TRY(copy2d_p(A + s + s * lda, lda, S, L.lds_small, b, b, 1, stream, &launches));
    RQ_CUDA_TRY(cudaMemsetAsync(V2, 0, (size_t)L.lds_small * b * sizeof(double), stream));
    launches++;
    SweepCall ss;
    ss.a = S;
    ss.lda = L.lds_small;
    ss.m = b;
    ss.n = b;
    ss.steps = b;
    ss.pivot = 1;
    ss.v = V2;
    ss.ldv = L.lds_small;
    ss.col_at_pos = L.cap;
    ss.r_out = L.rfin;
    ss.ldr = L.lds_small;
    bool t_early = false;
    if (overlap) {
      // env_overlap 1: CPQR then the W GEMM in one stream, the GEMM a programmatic dependent launch
      //   (it starts once every CPQR CTA is resident, so the cluster never waits behind it), with a
      //   CPQR-done event between them for small_q; 3: the same without that event;
      // 4: CPQR on a highest-priority stream, W on a lowest-priority one.
      RQ_TRY(ensure_side());
      if (phases_on) {  // fork time (main stream), the reference for the side-stream parts
        cudaEvent_t e;
        if (cudaEventCreate(&e) == cudaSuccess) {
          cudaEventRecord(e, stream);
          side_ev.emplace_back(0, e);
        }
      }
      RQ_CUDA_TRY(cudaEventRecord(ev_v, stream));
      const bool pdl = env_overlap != 4 && !cpqr_off;  // off-chain: the CPQR on hip2, W on side
      cudaStream_t cpqr_stream = cpqr_off ? hip2 : pdl ? side : hip;
      RQ_CUDA_TRY(cudaStreamWaitEvent(cpqr_stream, ev_v, 0));
      if (!pdl) RQ_CUDA_TRY(cudaStreamWaitEvent(side, ev_v, 0));
      cudaStream_t main_stream = stream;
      stream = cpqr_stream;
      void* sws = sweep_ws;
      const size_t swb = sweep_ws_bytes;
      if (cpqr_off) {  // its own workspace and pivot buffer: the next sketch CPQR runs beside it
        sweep_ws = L.sweep_ws2;
        sweep_ws_bytes = L.sweep_ws2_bytes;
        ss.col_at_pos = L.cap2;
      }
      int rc = sweep(ss);
      sweep_ws = sws;
      sweep_ws_bytes = swb;
      const bool hi_event = env_overlap != 3;
      if (rc == RQ_OK && hi_event)
        rc = cudaEventRecord(ev_hi, cpqr_stream) == cudaSuccess ? RQ_OK : set_error(RQ_ECUDA, "event");
      double* kw = kwork;
      const size_t kwb = kwork_bytes;
      // off-chain panels: the main stream idles until W and T are there, so T (Gram + triangular
      // inverse, independent of W) runs beside W on the aux stream with the main stream's split-K
      // slabs and Gram scratch instead of behind W on the side stream (RQ_T_OFF_AUX=0: behind W)
      static const int env_toff = [] {
        const char* e = getenv("RQ_T_OFF_AUX");
        return e ? atoi(e) : 1;
      }();
      if (rc == RQ_OK && cpqr_off && !t_done && env_toff != 0 && !t_on_hip) {
        if (cudaStreamWaitEvent(aux, ev_v, 0) != cudaSuccess) rc = set_error(RQ_ECUDA, "wait");
        stream = aux;
        if (rc == RQ_OK) rc = tfactor(V, mp, b, ldv, vpad, T, ldt, L.gram);
        if (rc == RQ_OK && cudaEventRecord(ev_t, aux) != cudaSuccess) rc = set_error(RQ_ECUDA, "event");
        t_done = true;
        t_early = rc == RQ_OK;
      }
      if (rc == RQ_OK) {
        stream = side;
        kwork = L.kwork2;
        kwork_bytes = L.kwork2_bytes;
        gemm_max_ctas = kSMs - 16;
        gemm_pdl = pdl;
        {
          // the CPQR holds 16 SMs for ~b * 2.7 us: the first n_a columns of W run capped beside
          // it, the rest (launched once those finish) on the whole GPU
          CatGuard g(cat, PROF_TRAIL);
          // measured b x b CPQR step (2.26 us at b = 256) and capped DMMA rate; RQ_CPQR_US /
          // RQ_CAPPED_TF override them (tuning)
          static const double env_us = getenv("RQ_CPQR_US") ? atof(getenv("RQ_CPQR_US")) : 2.7;
          static const double env_tf = getenv("RQ_CAPPED_TF") ? atof(getenv("RQ_CAPPED_TF")) : 30.0;
          const double cpqr_s = (double)b * env_us * 1e-6, rate = env_tf * 1e12;
          int64_t n_a = (int64_t)(cpqr_s * rate / (2.0 * b * (double)mp));
          n_a = std::max<int64_t>(128, (n_a + 127) / 128 * 128);
          if (n_a >= n2 - 256) n_a = n2;
          // RQ_TN_SPLIT=0: one launch on the whole grid (with dynamic scheduling its CTAs that do not
          // fit beside the CPQR start when it ends and take fewer units); measured slower
          // (157.2 vs 155.0 ms at n = 10k), so the capped part + remainder split stays the default
          static const int env_split = [] {
            const char* e = getenv("RQ_TN_SPLIT");
            return e ? atoi(e) : 1;
          }();
          if (env_split == 0) {
            n_a = n2;
            gemm_max_ctas = 0;
          }
          rc = gemm(b, n_a, mp, op(V, mp + vpad, b, ldv, vpad), false, op(A, m, n, lda, s, s + b), L.wside, even(b),
                    1.0, 0.0);
          gemm_pdl = false;
          gemm_max_ctas = 0;
          side_phase(1);
          // the panel's T: its Gram GEMM here (whole GPU, short), its latency-bound triangular
          // inverse on the second high-priority stream beside the rest of W (RQ_TINV_HIP=1;
          // measured neutral to slightly slower: n = 10k 143.8 vs 144.6 ms, so off)
          static const int env_th = [] {
            const char* e = getenv("RQ_TINV_HIP");
            return e ? atoi(e) : 0;
          }();
          tinv_par = rc == RQ_OK && env_th != 0 && hip2 != nullptr && !t_done && !(t_on_hip && hip_tail) &&
                     n_a < n2;
          if (tinv_par) {
            CatGuard gt(cat, PROF_TFACTOR);
            const int64_t ldg2 = even(b);
            rc = gemm(b, b, mp, op(V, mp + vpad, b, ldv, vpad), false, op(V, mp + vpad, b, ldv, vpad), L.gram2, ldg2,
                      1.0, 0.0);
            if (rc == RQ_OK) rc = cudaEventRecord(ev_gram, side) == cudaSuccess ? RQ_OK : set_error(RQ_ECUDA, "ev");
            if (rc == RQ_OK) rc = cudaStreamWaitEvent(hip2, ev_gram, 0) == cudaSuccess ? RQ_OK : set_error(RQ_ECUDA, "w");
            if (rc == RQ_OK) rc = tfactor_from_gram(L.gram2, ldg2, b, T, even(b), hip2, &launches);
            if (rc == RQ_OK) rc = cudaEventRecord(ev_t, hip2) == cudaSuccess ? RQ_OK : set_error(RQ_ECUDA, "ev");
          }
          if (rc == RQ_OK && n_a < n2)
            rc = gemm(b, n2 - n_a, mp, op(V, mp + vpad, b, ldv, vpad), false, op(A, m, n, lda, s, s + b + n_a),
                      L.wside + n_a * even(b), even(b), 1.0, 0.0);
        }
        gemm_pdl = false;
        side_phase(2);
        if (rc == RQ_OK && !t_done && !(t_on_hip && hip_tail) && !tinv_par)
          rc = tfactor(V, mp, b, ldv, vpad, T, even(b), L.gram2);
        if (rc == RQ_OK && tinv_par)  // T done on hip2: the side stream's completion includes it
          rc = cudaStreamWaitEvent(side, ev_t, 0) == cudaSuccess ? RQ_OK : set_error(RQ_ECUDA, "w");
        side_phase(3);
        if (rc == RQ_OK) rc = cudaEventRecord(ev_side, side) == cudaSuccess ? RQ_OK : set_error(RQ_ECUDA, "event");
        // look-ahead: W2 = T^T W (needed only by the trailing update of the rows below the top,
        // after the next panel's CPQR) stays on the side stream, off the tail's critical path
        if (rc == RQ_OK && w2_side) {
          CatGuard g(cat, PROF_TRAIL);
          rc = gemm(b, n2, b, op(T, b, b, ldt), false, op(L.wside, b, n2, even(b)), L.w2, even(b), 1.0, 0.0);
          if (rc == RQ_OK) rc = cudaEventRecord(ev_w2, side) == cudaSuccess ? RQ_OK : set_error(RQ_ECUDA, "event");
        }
      }
      gemm_max_ctas = 0;
      gemm_pdl = false;
      kwork = kw;
      kwork_bytes = kwb;
      stream = main_stream;
      RQ_TRY(rc);
      if (!cpqr_off) RQ_CUDA_TRY(cudaStreamWaitEvent(stream, hi_event ? ev_hi : ev_side, 0));
    } else {
      RQ_TRY(sweep(ss));
    }
    phase(2);
    if (cpqr_off) {
      // hip (highest priority): G1' first -- it reads R'11, which the R copy below overwrites --
      // then, once the CPQR (hip2) is done, Q2, R and the rows above (its own stage buffers)
      cudaStream_t main_stream = stream;
      double* kw = kwork;
      const size_t kwb = kwork_bytes;
      RQ_CUDA_TRY(cudaStreamWaitEvent(hip, ev_v, 0));
      stream = hip;
      kwork = nullptr;  // no split-K slabs: the main stream's GEMMs own kwork
      kwork_bytes = 0;
      int rc = RQ_OK;
      if (aux_g1) {
        rc = aux_g1();
        aux_g1 = nullptr;
      }
      if (rc == RQ_OK && cudaEventRecord(ev_g1, hip) != cudaSuccess) rc = set_error(RQ_ECUDA, "event");
      if (rc == RQ_OK && cudaStreamWaitEvent(hip, ev_hi, 0) != cudaSuccess) rc = set_error(RQ_ECUDA, "wait");
      if (rc == RQ_OK) rc = small_q(V2, L.lds_small, b, Q2, ldt, L);
      if (rc == RQ_OK) rc = copy2d_p(L.rfin, L.lds_small, A + s + s * lda, lda, b, b, 0, stream, &launches);
      if (rc == RQ_OK) {
        MoveCall mv2{A, lda, s, 0, s, L.cap2, L.iota_b, nullptr, b, L.stage2, even(m), L.orig, L.ostage2};
        rc = move_columns_p(mv2, stream, &launches);
      }
      if (rc == RQ_OK && on_cols_final) on_cols_final(s, b);
      if (rc == RQ_OK && cudaEventRecord(ev_hipdone, hip) != cudaSuccess) rc = set_error(RQ_ECUDA, "event");
      stream = main_stream;
      kwork = kw;
      kwork_bytes = kwb;
      RQ_TRY(rc);
      phase(12);
      RQ_CUDA_TRY(cudaStreamWaitEvent(stream, ev_g1, 0));    // G1' (the downdate)
      RQ_CUDA_TRY(cudaStreamWaitEvent(stream, ev_side, 0));  // W and T
      if (t_early) RQ_CUDA_TRY(cudaStreamWaitEvent(stream, ev_t, 0));  // (T from the aux stream)
      phase(3);
      RQ_TRY(lookahead_tail(cfg, A, lda, m, n, s, mp, b, n2, V, ldv, vpad, T, ldt, Q2, L, L.wside, lorder, lorder_n,
                            rank, rank_n));
      cpqr_off = false;
      factors.push_back(PanelFactors{s, b, V, ldv, vpad, T, ldt, Q2, ldt});
      phase(7);
      continue;
    }
    // the small post-CPQR work (G1', Q2, R, the rows above) on the highest-priority stream: its
    // CTAs take the SMs the CPQR frees before the queued CTAs of the rest of W
    cudaStream_t tail_saved = stream;
    const bool on_hip = overlap && hip_tail;
    (void)on_hip;
    if (on_hip) {
      RQ_CUDA_TRY(cudaEventRecord(ev_v, stream));
      RQ_CUDA_TRY(cudaStreamWaitEvent(hip, ev_v, 0));
      stream = hip;
    }
    // Q2 (small_q) and G1' (form_g1) are independent: Q2 on a second high-priority stream
    const bool q2_par = on_hip && aux_g1 && hip2 != nullptr;
    if (q2_par) {
      RQ_CUDA_TRY(cudaEventRecord(ev_v, hip));
      RQ_CUDA_TRY(cudaStreamWaitEvent(hip2, ev_v, 0));
      stream = hip2;
      RQ_TRY(small_q(V2, L.lds_small, b, Q2, ldt, L));
      RQ_CUDA_TRY(cudaEventRecord(ev_q2, hip2));
      stream = hip;
    }
    if (aux_g1) {
      RQ_TRY(aux_g1());  // (before R overwrites R'11 in A)
      aux_g1 = nullptr;
    }
    if (on_hip && t_on_hip) RQ_TRY(tfactor(V, mp, b, ldv, vpad, T, ldt, L.gram));
    if (q2_par) RQ_CUDA_TRY(cudaStreamWaitEvent(stream, ev_q2, 0));
    else RQ_TRY(small_q(V2, L.lds_small, b, Q2, ldt, L));
    phase(11);
    if (refl_piv)
      RQ_CUDA_TRY(cudaMemcpyAsync(rfactors.back().phat, L.cap, (size_t)b * sizeof(int), cudaMemcpyDeviceToDevice,
                                  stream));
    // ---------------- 7: R and the rows above follow P-hat ----------------
    RQ_TRY(copy2d_p(L.rfin, L.lds_small, A + s + s * lda, lda, b, b, 0, stream, &launches));
    MoveCall mv2{A, lda, s, 0, s, L.cap, L.iota_b, nullptr, b, L.stage, even(m), L.orig, L.ostage};
    RQ_TRY(move_columns_p(mv2, stream, &launches));
    if (on_cols_final) on_cols_final(s, b);  // later steps only touch columns >= s + b
    // (the sketch's panel columns are not needed after form_g1: no P-hat on them)
    if (on_hip) {
      RQ_CUDA_TRY(cudaEventRecord(ev_hi, hip));
      stream = tail_saved;
      RQ_CUDA_TRY(cudaStreamWaitEvent(stream, ev_hi, 0));
    }
    phase(12);
    // ---------------- 8: T of the panel reflectors (on the side stream when overlapped) ----------------
    if (overlap) RQ_CUDA_TRY(cudaStreamWaitEvent(stream, ev_side, 0));
    else if (!t_done) RQ_TRY(tfactor(V, mp, b, ldv, vpad, T, ldt, L.gram));
    phase(3);
    // ---------------- 9: trailing update ----------------
    if (la_mode && n2 > 0) {
      RQ_TRY(lookahead_tail(cfg, A, lda, m, n, s, mp, b, n2, V, ldv, vpad, T, ldt, Q2, L,
                            overlap ? L.wside : nullptr, lorder, lorder_n, rank, rank_n));
      factors.push_back(PanelFactors{s, b, V, ldv, vpad, T, ldt, Q2, ldt});
      phase(7);
      continue;  // lorder/rank were swapped for the next panel inside
    }
    if (n2 > 0) RQ_TRY(trailing_update(A, lda, m, n, s, mp, b, n2, V, ldv, vpad, T, ldt, Q2, L,
                                       overlap ? L.wside : nullptr));
    if (downdate && n2 > 0) {
      // Y2 <- Y2 - G1' R'12 (form_g1 ran after the panel QR; R'12 = the top rows before Q2^T,
      // which trailing_update left in L.ttop): the sketch of the new trailing block
      const int64_t ldg = even(wdt);
      RQ_TRY(gemm(wdt, n2, b, op(L.g1, wdt, b, ldg), true, op(L.ttop, b, n2, even(b)), L.yt + (s + b) * L.ldy,
                  L.ldy, -1.0, 1.0));
    }
    factors.push_back(PanelFactors{s, b, V, ldv, vpad, T, ldt, Q2, ldt});
    phase(10);
    if (!refl_piv) {
      std::swap(lorder, lorder_n);
      std::swap(rank, rank_n);
    } else {
      RQ_TRY(iota(lorder, (int)(np - b), nullptr, 0, stream, &launches));  // columns stay in place
    }
    if (inspect_cb) {
      cur_s = s + b;
      cur_lorder = lorder;
      cur_np = np - b;
      RQ_CUDA_TRY(cudaStreamSynchronize(stream));
      inspect_cb(panel, inspect_user);
    }
  }
  cur_lorder = nullptr;
  cur_yt = nullptr;
  if (dperm) {
    RQ_CUDA_TRY(cudaMemcpyAsync(dperm, L.orig, n * sizeof(int64_t), cudaMemcpyDeviceToDevice, stream));
    launches++;
  }
  phase(8);
  phase_report();
  have_factors = true;
  return RQ_OK;
}

// The downdated sketch's G and Y = G A ahead of factorize_perm (same arena layout), so that the
// host entry can form Y chunk by chunk while the rest of A is still on its way to the device.
int Ctx::presketch_begin(const rq_config& cfg, int64_t m, int64_t n, uint64_t seed, uint64_t counter) {
  const int b = cfg.block, p = cfg.oversample, wdt = b + p;
  RQ_TRY(arena.reserve(plan_layout(nullptr, m, n, b, p, cfg.power).total));
  Layout L = plan_layout(arena.base, m, n, b, p, cfg.power);
  return gaussian_fill_p(L.omega, m, wdt, L.ldo, seed, counter, stream, &launches);
}

int Ctx::presketch_cols(const rq_config& cfg, int64_t m, int64_t n, const double* A, int64_t lda, int64_t c0,
                        int64_t c1) {
  const int b = cfg.block, p = cfg.oversample, wdt = b + p;
  Layout L = plan_layout(arena.base, m, n, b, p, cfg.power);
  kwork = L.kwork;
  kwork_bytes = L.kwork_bytes;
  return gemm(wdt, c1 - c0, m, op(L.omega, m, wdt, L.ldo), false, op(A, m, n, lda, 0, c0), L.yt + c0 * L.ldy, L.ldy,
              1.0, 0.0);
}

// ---------------------------------------------------------------------------
// Unpivoted blocked Householder QR (qr_unpivoted, householder.py:152-161, in
// blocks of b): the panel kernels + T + trailing update, no sketch, no pivots.
// Used by the device-side test-matrix generator (haar_orthonormal,
// matrices.py:34-41).  R overwrites A; the factors are stored for form_q.
// ---------------------------------------------------------------------------
int Ctx::factorize_unpivoted(int64_t m, int64_t n, double* A, int64_t lda, int b) {
  size_t need = plan_layout(nullptr, m, n, b, 0, 0).total;
  RQ_TRY(arena.reserve(need));
  Layout L = plan_layout(arena.base, m, n, b, 0, 0);
  kwork = L.kwork;
  kwork_bytes = L.kwork_bytes;
  sweep_ws = L.sweep_ws;
  sweep_ws_bytes = L.sweep_ws_bytes;
  have_factors = false;  // a failed run leaves nothing readable
  factors.clear();
  rfactors.clear();
  p_is_perm = true;
  factors_perm = L.orig;
  fm = m;
  fn = n;
  fb = b;
  RQ_TRY(iota(nullptr, 0, L.orig, n, stream, &launches));
  Carver fc(L.fstore);
  for (int64_t s = 0; s < n; s += b) {
    const int w = (int)std::min<int64_t>(b, n - s);
    const int64_t mp = m - s;
    const int64_t ldv = even(mp + 1), ldt = even(b);
    const int vpad = (int)(s & 1);
    double* V = fc.take<double>((size_t)ldv * w);  // as factor_bytes sizes the final panel
    double* T = fc.take<double>((size_t)ldt * b);
    RQ_CUDA_TRY(cudaMemsetAsync(V, 0, (size_t)ldv * w * sizeof(double), stream));
    launches++;
    RQ_TRY(panel_qr(A, lda, m, n, s, mp, w, V, ldv, vpad, L.tleaf, L.w1, L.w2, nullptr, 0, nullptr));
    RQ_TRY(tfactor(V, mp, w, ldv, vpad, T, ldt, L.gram));
    const int64_t n2 = n - s - w;
    if (n2 > 0) RQ_TRY(trailing_update(A, lda, m, n, s, mp, w, n2, V, ldv, vpad, T, ldt, nullptr, L));
    factors.push_back(PanelFactors{s, w, V, ldv, vpad, T, ldt, nullptr, 0});
  }
  have_factors = true;
  return RQ_OK;
}

// Y^T ((b+p) x n') of the trailing block X = A[s:, s:]: (X^T X)^q X^T Omega,
// built from TN/NN DMMA GEMMs (pivoting.py:87-111, unstabilised powers).
int Ctx::sketch(const rq_config& cfg, double* A, int64_t lda, int64_t m, int64_t n, int64_t s, int64_t mp, int64_t np,
                Layout& L, bool want_y) {
  CatGuard guard(cat, PROF_SKETCH_GEMM);
  const int wdt = cfg.block + cfg.oversample;
  const bool stab = cfg.stabilize < 0 ? cfg.power >= 2 : cfg.stabilize != 0;
  const GemmOperand X = op(A, m, n, lda, s, s);
  const int pad = (int)(s & 1);
  const GemmOperand Om = op(L.omega, mp + pad, wdt, L.ldo, pad);
  if (stab) {
    // build_sketch with re-orthonormalisation after every application (pivoting.py:102-110)
    double* Y = L.ybuf;  // np x wdt
    const int64_t ldY = even(np);
    RQ_TRY(gemm(np, wdt, mp, X, false, Om, Y, ldY, 1.0, 0.0));
    RQ_TRY(orth(Y, np, wdt, ldY, L));
    for (int it = 0; it < cfg.power; it++) {
      RQ_TRY(gemm(mp, wdt, np, op(A, m, n, lda, s, s), true, op(Y, np, wdt, ldY), L.omega + pad, L.ldo, 1.0, 0.0));
      RQ_TRY(orth(L.omega + pad, mp, wdt, L.ldo, L));
      RQ_TRY(gemm(np, wdt, mp, X, false, Om, Y, ldY, 1.0, 0.0));
      RQ_TRY(orth(Y, np, wdt, ldY, L));
    }
    if (want_y) return RQ_OK;
    return transpose(Y, ldY, L.yt, L.ldy, np, wdt, stream, &launches);
  }
  if (cfg.power == 0) {
    if (want_y) return gemm(np, wdt, mp, X, false, Om, L.ybuf, even(np), 1.0, 0.0);  // Y = X^T Omega
    return gemm(wdt, np, mp, Om, false, X, L.yt, L.ldy, 1.0, 0.0);                   // Y^T = Omega^T X
  }
  // Y = X^T Omega (np x wdt) in w1-sized scratch; Z = X Y (mp x wdt) in omega
  double* Y = want_y ? L.yt : L.ybuf;  // np x wdt intermediate (the output goes to ybuf when want_y)
  const int64_t ldY = even(np);
  RQ_TRY(gemm(np, wdt, mp, X, false, Om, Y, ldY, 1.0, 0.0));
  for (int it = 0; it < cfg.power; it++) {
    // Z = X Y, stored with the same row padding as Omega
    RQ_TRY(gemm(mp, wdt, np, op(A, m, n, lda, s, s), true, op(Y, np, wdt, ldY), L.omega + pad, L.ldo, 1.0, 0.0));
    if (it + 1 < cfg.power) RQ_TRY(gemm(np, wdt, mp, X, false, Om, Y, ldY, 1.0, 0.0));
  }
  if (want_y) return gemm(np, wdt, mp, X, false, Om, L.ybuf, even(np), 1.0, 0.0);  // Y = X^T Z
  // Y^T = Z^T X
  return gemm(wdt, np, mp, Om, false, X, L.yt, L.ldy, 1.0, 0.0);
}

// G1' = Y1 R'11^{-1} for the downdate, from the panel's leaf R' (before the b x b CPQR) and the
// sketch columns of the panel as selected (before P-hat): the downdate
//   Y2 <- Y2 - G1 R12 = Y2 - Y1 R11^{-1} R12 = Y2 - (Y1 P^T)(Q2^T R'11)^{-1}... = Y2 - G1' R'12
// (R11 = Q2^T R'11 P-hat, R12 = Q2^T R'12, Y1 = Y1' P-hat) needs neither Q2 nor P-hat, so G1'
// is formed while the panel's trailing update still runs, and R'12 (the top rows before Q2^T)
// is the copy the Q2^T product reads anyway.
int Ctx::form_g1(double* A, int64_t lda, int64_t s, int b, int wdt, int64_t n, Layout& L) {
  const int64_t ldb2 = even(b), ldg = even(wdt);
  RQ_TRY(trinv_upper(A + s + s * lda, lda, b, L.rinv, ldb2, stream, &launches));
  return gemm(wdt, b, b, op(L.yt, wdt, n, L.ldy, 0, s), true, op(L.rinv, b, b, ldb2), L.g1, ldg, 1.0, 0.0);
}

// Off-chain CPQR (cpqr_off): join the hip stream (Q2, R, rows-above moves of the panel at s) and
// apply Q2^T to the top rows R'12 (kept in L.ttop): R12 = Q2^T R'12.
int Ctx::finish_top(double* A, int64_t lda, int64_t s, int b, int64_t n2, const double* Q2, int64_t ldt, Layout& L) {
  const int64_t ldw = even(b);
  RQ_CUDA_TRY(cudaStreamWaitEvent(stream, ev_hipdone, 0));
  CatGuard guard(cat, PROF_TRAIL);
  return gemm(b, n2, b, op(Q2, b, b, ldt), false, op(L.ttop, b, n2, ldw), A + s + (s + b) * lda, lda, 1.0, 0.0);
}

// Look-ahead tail of a non-final panel at s (downdated sketches, permutation pivots):
//   W2 = T^T W;  top b rows: R12 = Q2^T (A2_top - V_top W2)  (final);
//   Y2 <- Y2 - G1 R12 (the next panel's sketch);
//   if the next panel is not the final block: its b-step CPQR, plan and column moves (A at full
//   height, Y, and W2's columns, whose rows below the top are not applied yet), then
//   A2 -= V W2 on the next panel's b columns, and the rest left pending (la) for panel_qr to
//   issue beside the next panel's leaves;  otherwise A2 -= V W2 now.
// lorder/rank are swapped to the next panel's (as the end of the panel loop does).
int Ctx::lookahead_tail(const rq_config& cfg, double* A, int64_t lda, int64_t m, int64_t n, int64_t s, int64_t mp,
                        int b, int64_t n2, const double* V, int64_t ldv, int vpad, const double* T, int64_t ldt,
                        const double* Q2, Layout& L, const double* Wpre, int*& lorder, int*& lorder_n, int*& rank,
                        int*& rank_n) {
  const int wdt = b + cfg.oversample;
  const int64_t ldw = even(b);
  const GemmOperand Vop = op(V, mp + vpad, b, ldv, vpad);
  const GemmOperand Vlow = op(V, mp + vpad, b, ldv, vpad + b);  // rows b.. of V
  {
    CatGuard guard(cat, PROF_TRAIL);
    const double* W = Wpre ? Wpre : L.w1;
    if (!Wpre) RQ_TRY(gemm(b, n2, mp, Vop, false, op(A, m, n, lda, s, s + b), L.w1, ldw, 1.0, 0.0));
    if (w2_side) {
      // top b rows: A2_top -= (V_top T^T) W while the side stream forms W2 = T^T W
      RQ_TRY(transpose(T, ldt, L.jw, ldw, b, b, stream, &launches));
      RQ_TRY(gemm(b, b, b, Vop, true, op(L.jw, b, b, ldw), L.jv, ldw, 1.0, 0.0));
      RQ_TRY(gemm(b, n2, b, op(L.jv, b, b, ldw), true, op(W, b, n2, ldw), A + s + (s + b) * lda, lda, -1.0, 1.0));
    } else {
      RQ_TRY(gemm(b, n2, b, op(T, b, b, ldt), false, op(W, b, n2, ldw), L.w2, ldw, 1.0, 0.0));
      // top b rows: A2_top -= V_top W2, then Q2^T
      RQ_TRY(gemm(b, n2, b, Vop, true, op(L.w2, b, n2, ldw), A + s + (s + b) * lda, lda, -1.0, 1.0));
    }
    RQ_TRY(copy2d_p(A + s + (s + b) * lda, lda, L.ttop, ldw, b, n2, 0, stream, &launches));
    if (!cpqr_off)
      RQ_TRY(gemm(b, n2, b, op(Q2, b, b, ldt), false, op(L.ttop, b, n2, ldw), A + s + (s + b) * lda, lda, 1.0, 0.0));
  }
  phase(4);
  std::swap(lorder, lorder_n);
  std::swap(rank, rank_n);
  const int64_t np2 = n - s - b;  // the next panel's columns
  const bool next_full = np2 > b;
  if (!next_full) {
    if (cpqr_off) RQ_TRY(finish_top(A, lda, s, b, n2, Q2, ldt, L));
    CatGuard guard(cat, PROF_TRAIL);
    if (w2_side) RQ_CUDA_TRY(cudaStreamWaitEvent(stream, ev_w2, 0));
    return gemm(mp - b, n2, b, Vlow, true, op(L.w2, b, n2, ldw), A + (s + b) + (s + b) * lda, lda, -1.0, 1.0);
  }
  // Y2 <- Y2 - G1' R'12 (form_g1; R'12 = the top rows before Q2^T, kept in L.ttop)
  const int64_t ldg = even(wdt);
  RQ_TRY(gemm(wdt, n2, b, op(L.g1, wdt, b, ldg), true, op(L.ttop, b, n2, ldw), L.yt + (s + b) * L.ldy, L.ldy, -1.0,
              1.0));
  phase(5);
  // the next panel's pivots (b-step CPQR of a copy of its sketch) and moves
  const int64_t s2 = s + b;
  sketch_gmax = cpqr_off ? kSkMinGrid : 0;  // leave the b x b CPQR's cluster its 16 SMs
  int rc;
  if (sketch_batched(wdt, (int)np2, b, sketch_gmax) ||
      sketch_cpqr_preserves_input(wdt, (int)np2, sketch_gmax)) {  // (these kernels only read Y)
    rc = sketch_select(L.yt + s2 * L.ldy, L.ldy, wdt, (int)np2, b, rank, L.cap);
  } else {
    rc = copy2d_p(L.yt + s2 * L.ldy, L.ldy, L.ybuf, L.ldy, wdt, np2, 0, stream, &launches);
    if (rc == RQ_OK) rc = sketch_select(L.ybuf, L.ldy, wdt, (int)np2, b, rank, L.cap);
  }
  sketch_gmax = 0;
  RQ_TRY(rc);
  phase(6);
  if (cpqr_off) RQ_TRY(finish_top(A, lda, s, b, n2, Q2, ldt, L));  // before the moves touch the top rows
  PlanCall pc{L.cap, b, lorder, (int)np2, L.flag, L.newloc, L.src, L.dst, L.nmoves, lorder_n, rank_n};
  RQ_TRY(plan_moves(pc, stream, &launches));
  MoveCall mv{A, lda, s2, 0, m, L.src, L.dst, L.nmoves, 2 * b, L.stage, even(m), L.orig, L.ostage};
  RQ_TRY(move_columns_p(mv, stream, &launches));
  MoveCall my{L.yt, L.ldy, s2, 0, wdt, L.src, L.dst, L.nmoves, 2 * b, L.stage, L.ldy, nullptr, nullptr};
  RQ_TRY(move_columns_p(my, stream, &launches));
  if (w2_side) RQ_CUDA_TRY(cudaStreamWaitEvent(stream, ev_w2, 0));
  MoveCall mw{L.w2, ldw, 0, 0, b, L.src, L.dst, L.nmoves, 2 * b, L.stage, even(m), nullptr, nullptr};
  RQ_TRY(move_columns_p(mw, stream, &launches));
  // the next panel's columns first; the rest pending
  {
    CatGuard guard(cat, PROF_TRAIL);
    RQ_TRY(gemm(mp - b, b, b, Vlow, true, op(L.w2, b, n2, ldw), A + s2 + s2 * lda, lda, -1.0, 1.0));
  }
  GemmProblem& g = la.g;
  g = GemmProblem();
  g.M = mp - b;
  g.N = n2 - b;
  g.K = b;
  g.A = Vlow;
  g.a_mmajor = true;
  g.B = op(L.w2, b, n2, ldw, 0, b);
  g.C = A + s2 + (s2 + b) * lda;
  g.ldc = lda;
  g.alpha = -1.0;
  g.beta = 1.0;
  la.tiles = g.N > 0 ? (tf32_update ? gemm_tf32x3_tiles(g.M, g.N, g.a_mmajor, g.A.r0) : gemm_f64_tiles(g)) : 0;
  la.next = 0;
  la.on = la.tiles > 0;
  return RQ_OK;
}

int Ctx::trailing_update(double* A, int64_t lda, int64_t m, int64_t n, int64_t s, int64_t mp, int b, int64_t n2,
                         const double* V, int64_t ldv, int vpad, const double* T, int64_t ldt, const double* Q2,
                         Layout& L, const double* Wpre) {
  const int64_t ldw = even(b);
  const GemmOperand Vop = op(V, mp + vpad, b, ldv, vpad);
  CatGuard guard(cat, PROF_TRAIL);
  // W = V^T A2   (b x n2, K = m'), unless the side stream already formed it
  const double* W = Wpre ? Wpre : L.w1;
  if (!Wpre) RQ_TRY(gemm(b, n2, mp, Vop, false, op(A, m, n, lda, s, s + b), L.w1, ldw, 1.0, 0.0));
  // W2 = T^T W
  RQ_TRY(gemm(b, n2, b, op(T, b, b, ldt), false, op(W, b, n2, ldw), L.w2, ldw, 1.0, 0.0));
  // A2 -= V W2
  RQ_TRY(gemm(mp, n2, b, Vop, true, op(L.w2, b, n2, ldw), A + s + (s + b) * lda, lda, -1.0, 1.0));
  if (Q2) {
    // top b rows <- Q2^T top   (TN with A = Q2)
    RQ_TRY(copy2d_p(A + s + (s + b) * lda, lda, L.ttop, ldw, b, n2, 0, stream, &launches));
    RQ_TRY(gemm(b, n2, b, op(Q2, b, b, ldt), false, op(L.ttop, b, n2, ldw), A + s + (s + b) * lda, lda, 1.0, 0.0));
  }
  return RQ_OK;
}

// _orth (pivoting.py:80-84): src (rows x cols) <- the first cols columns of Q
// from its unpivoted Householder QR (panel kernels + DMMA GEMMs).
int Ctx::orth(double* src, int64_t rows, int cols, int64_t ld, Layout& L) {
  const int64_t lde = even(rows);
  double* E = L.oe;
  double* Vo = L.ov;
  const int64_t ldc = even(cols);
  RQ_TRY(copy2d_p(src, ld, E, lde, rows, cols, 0, stream, &launches));
  RQ_CUDA_TRY(cudaMemsetAsync(Vo, 0, (size_t)lde * cols * sizeof(double), stream));
  launches++;
  RQ_TRY(panel_qr(E, lde, rows, cols, 0, rows, cols, Vo, lde, 0, L.tleaf, L.w1, L.w2));
  RQ_TRY(tfactor(Vo, rows, cols, lde, 0, L.ot, ldc, L.gram));
  RQ_TRY(fill_eye(E, lde, rows, cols, 0, stream, &launches));
  RQ_TRY(gemm(cols, cols, rows, op(Vo, rows, cols, lde), false, op(E, rows, cols, lde), L.w1, ldc, 1.0, 0.0));
  RQ_TRY(gemm(cols, cols, cols, op(L.ot, cols, cols, ldc), true, op(L.w1, cols, cols, ldc), L.w2, ldc, 1.0, 0.0));
  RQ_TRY(gemm(rows, cols, cols, op(Vo, rows, cols, lde), true, op(L.w2, cols, cols, ldc), E, lde, -1.0, 1.0));
  return copy2d_p(E, lde, src, ld, rows, cols, 0, stream, &launches);
}

// Reflector pivot of the panel at s: sketch Y, its first b unpivoted reflectors,
// A[:, s:] <- A[:, s:] S at full height.  Records the right factor.
int Ctx::reflector_pivot(const rq_config& cfg, double* A, int64_t lda, int64_t m, int64_t n, int64_t s, Layout& L,
                         void* fc_ptr, uint64_t seed, uint64_t* counter) {
  Carver& fc = *reinterpret_cast<Carver*>(fc_ptr);
  const int b = cfg.block, wdt = cfg.block + cfg.oversample;
  const int64_t mp = m - s, np = n - s;
  RQ_TRY(gaussian_fill_p(L.omega + (s & 1), mp, wdt, L.ldo, seed, *counter, stream, &launches));
  *counter += (uint64_t)mp * (uint64_t)wdt;
  RQ_TRY(sketch(cfg, A, lda, m, n, s, mp, np, L, true));  // Y (np x wdt) in ybuf
  const int64_t ldvs = even(np), ldt = even(b);
  double* VS = fc.take<double>((size_t)ldvs * b);
  double* TS = fc.take<double>((size_t)ldt * b);
  int* phat = fc.take<int>((size_t)std::max<int64_t>(np, b));
  RQ_CUDA_TRY(cudaMemsetAsync(VS, 0, (size_t)ldvs * b * sizeof(double), stream));
  launches++;
  RQ_TRY(panel_qr(L.ybuf, even(np), np, wdt, 0, np, b, VS, ldvs, 0, L.tleaf, L.w1, L.w2));
  RQ_TRY(tfactor(VS, np, b, ldvs, 0, TS, ldt, L.gram));
  RQ_TRY(apply_right_wy(A, lda, m, n, s, np, b, VS, ldvs, TS, ldt, L.vst, L.zbuf, L.z2buf, even(m)));
  rfactors.push_back(RightFactors{s, np, b, VS, ldvs, TS, ldt, phat, 0, nullptr, 0, 0});
  return RQ_OK;
}

// ---------------------------------------------------------------------------
// block_rrqr (blocked.py:239-279): reflector pivots, panel SVD (unpivoted QR +
// wave-parallel cyclic Jacobi), diag(d) blocks, V~ on the rows above,
// tail <- U'^T Q~^T tail.
// ---------------------------------------------------------------------------
int Ctx::factorize_rrqr(const rq_config& cfg0, int64_t m, int64_t n, double* A, int64_t lda, uint64_t seed,
                        uint64_t* counter) {
  rq_config cfg = cfg0;
  cfg.pivot_kind = RQ_PIVOT_REFLECTORS;  // blocked.py:251
  const int b = cfg.block, p = cfg.oversample;
  size_t need = plan_layout(nullptr, m, n, b, p, cfg.power).total;
  RQ_TRY(arena.reserve(need));
  Layout L = plan_layout(arena.base, m, n, b, p, cfg.power);
  kwork = L.kwork;
  kwork_bytes = L.kwork_bytes;
  sweep_ws = L.sweep_ws;
  sweep_ws_bytes = L.sweep_ws_bytes;
  cur_A = A;
  cur_lda = lda;
  cur_m = m;
  cur_n = n;
  have_factors = false;  // a failed run leaves nothing readable
  factors.clear();
  rfactors.clear();
  p_is_perm = false;
  fm = m;
  fn = n;
  fb = b;
  Carver fc(L.fstore);
  int panel = 0;
  for (int64_t s = 0; s < n; s += b) {
    const int w = (int)std::min<int64_t>(b, n - s);
    const bool final = n - s <= b;
    const int64_t mp = m - s, np = n - s;
    cur_s = s;
    cur_lorder = nullptr;
    if (!final) RQ_TRY(reflector_pivot(cfg, A, lda, m, n, s, L, &fc, seed, counter));
    // panel_svd: unpivoted QR of the m' x w panel, then the SVD of its w x w triangle
    const int64_t ldv = even(mp + 1), ldt = even(b);
    const int vpad = (int)(s & 1);
    double* V = fc.take<double>((size_t)ldv * w);
    double* T = fc.take<double>((size_t)ldt * b);
    double* U = fc.take<double>((size_t)ldt * b);
    double* Vt = fc.take<double>((size_t)ldt * b);
    RQ_CUDA_TRY(cudaMemsetAsync(V, 0, (size_t)ldv * w * sizeof(double), stream));
    launches++;
    RQ_TRY(panel_qr(A, lda, m, n, s, mp, w, V, ldv, vpad, L.tleaf, L.w1, L.w2, nullptr, 0, nullptr));
    {
      cudaEvent_t e0;
      const int saved = cat;
      cat = PROF_SMALL;
      prof_begin(&e0);
      const int rc = jacobi_svd(A + s + s * lda, lda, w, L.jw, ldt, L.jv, ldt, L.jd, U, ldt, Vt, ldt, L.jstat + panel,
                                stream, &launches);
      prof_end(e0, 0.0);
      cat = saved;
      RQ_TRY(rc);
    }
    // rows above: A[:s, s:s+w] <- A[:s, s:s+w] V~   (blocked.py:265)
    if (s > 0) {
      RQ_TRY(copy2d_p(A + s * lda, lda, L.stage, even(m), s, w, 0, stream, &launches));
      RQ_TRY(gemm(s, w, w, op(L.stage, s, w, even(m)), true, op(Vt, w, w, ldt), A + s * lda, lda, 1.0, 0.0));
    }
    RQ_TRY(tfactor(V, mp, w, ldv, vpad, T, ldt, L.gram));
    RQ_TRY(set_diag_block(A + s + s * lda, lda, mp, w, L.jd, stream, &launches));  // blocked.py:266-268
    if (!final) RQ_TRY(trailing_update(A, lda, m, n, s, mp, w, np - w, V, ldv, vpad, T, ldt, U, L));
    factors.push_back(PanelFactors{s, w, V, ldv, vpad, T, ldt, U, ldt});
    rfactors.push_back(RightFactors{s, np, 0, nullptr, 0, nullptr, 0, nullptr, 0, Vt, ldt, w});
    panel++;
    if (inspect_cb) {
      RQ_CUDA_TRY(cudaStreamSynchronize(stream));
      inspect_cb(panel, inspect_user);
    }
  }
  cur_lorder = nullptr;
  // ConvergenceError after 60 sweeps (svd.py:52-53)
  std::vector<int> st((size_t)panel);
  RQ_CUDA_TRY(cudaMemcpyAsync(st.data(), L.jstat, (size_t)panel * sizeof(int), cudaMemcpyDeviceToHost, stream));
  RQ_CUDA_TRY(cudaStreamSynchronize(stream));
  for (int i = 0; i < panel; i++)
    if (st[i] < 0) return set_error(RQ_ECONV, "Jacobi SVD did not converge in 60 sweeps (panel %d)", i + 1);
  have_factors = true;
  return RQ_OK;
}

// ---------------------------------------------------------------------------
// Q = U_1 ... U_L applied to eye(m, cols) (blocked.py:134-141), backwards, on
// the trailing block X = Q[s:, s:] only (columns < s are untouched unit vectors).
// ---------------------------------------------------------------------------
FactorSet Ctx::view() const {
  FactorSet F;
  F.factors = factors;
  F.rfactors = rfactors;
  F.p_is_perm = p_is_perm;
  F.perm = factors_perm;
  F.fm = fm;
  F.fn = fn;
  F.fb = fb;
  F.have = have_factors;
  F.device = device;
  return F;
}

// The stored factors live in `arena`: hand the arena over with them.  The next
// factorization on this context reserves a fresh arena.
int Ctx::detach(FactorSet* out) {
  if (!have_factors) return set_error(RQ_EVALUE, "no factorization stored in this context");
  RQ_CUDA_TRY(cudaStreamSynchronize(stream));
  *out = view();
  out->arena = arena;
  arena = Arena{};
  have_factors = false;  // a failed run leaves nothing readable
  factors.clear();
  rfactors.clear();
  factors_perm = nullptr;
  have_factors = false;
  cur_A = nullptr;
  return RQ_OK;
}

int Ctx::form_q(const FactorSet& F, int64_t cols, double* Q, int64_t ldq) {
  if (!F.have) return set_error(RQ_EVALUE, "no factorization stored in this context");
  RQ_TRY(fill_eye(Q, ldq, F.fm, cols, 0, stream, &launches));
  return apply_q(F, 0, (int)F.factors.size(), false, true, cols, Q, ldq);
}

// X (m x cols) <- U_first ... U_last X  (trans: U_last^T ... U_first^T X), U_i = (I - V T V^T) diag(Q2, I)
// on rows s_i.. (QTransform.left_multiply, blocked.py:90-99).  eye: X is the identity on entry, so
// U_i only touches the block X[s_i:, s_i:] (columns < s_i are untouched unit vectors).
int Ctx::apply_q(const FactorSet& F, int first, int count, bool trans, bool eye, int64_t cols, double* Q,
                 int64_t ldq) {
  if (!F.have) return set_error(RQ_EVALUE, "no factorization stored in this context");
  const int nf = (int)F.factors.size();
  if (first < 0 || count < 0 || first + count > nf)
    return set_error(RQ_EVALUE, "panel range [%d, %d) outside the %d stored panels", first, first + count, nf);
  if (count == 0 || cols == 0) return RQ_OK;
  const int64_t m = F.fm;
  const int b = F.fb;
  const int64_t ldw = even(std::max(b, 2));
  size_t need = (size_t)3 * ldw * cols * 8 + (size_t)kSMs * b * b * 8 + 1024;
  RQ_TRY(qarena.reserve(need));
  Carver c(qarena.base);
  double* w1 = c.take<double>((size_t)ldw * cols);
  double* w2 = c.take<double>((size_t)ldw * cols);
  double* tt = c.take<double>((size_t)ldw * cols);
  double* save_kw = kwork;
  size_t save_kb = kwork_bytes;
  kwork = c.take<double>((size_t)kSMs * b * b);
  kwork_bytes = (size_t)kSMs * b * b * 8;
  int rc = RQ_OK;
  for (int it = 0; it < count && rc == RQ_OK; it++) {
    const PanelFactors& f = F.factors[trans ? first + it : first + count - 1 - it];
    const int64_t s = f.s, mp = m - s;
    const int64_t c0 = eye ? s : 0, nc = cols - c0;
    if (nc <= 0) continue;
    double* X = Q + s + c0 * ldq;
    const GemmOperand Vop = op(f.v, mp + f.vpad, f.k, f.ldv, f.vpad);
    auto small = [&]() {  // X[0:k] <- Q2 X[0:k]  (trans: Q2^T)
      int r = copy2d_p(X, ldq, tt, ldw, f.k, nc, 0, stream, &launches);
      if (r == RQ_OK)
        r = gemm(f.k, nc, f.k, op(f.q2, f.k, f.k, f.ldq2), !trans, op(tt, f.k, nc, ldw), X, ldq, 1.0, 0.0);
      return r;
    };
    if (f.q2 && !trans) rc = small();
    if (rc != RQ_OK) break;
    // X <- X - V T (V^T X)   (trans: T^T)
    rc = gemm(f.k, nc, mp, Vop, false, op(Q, m, cols, ldq, s, c0), w1, ldw, 1.0, 0.0);
    if (rc == RQ_OK)
      rc = gemm(f.k, nc, f.k, op(f.t, f.k, f.k, f.ldt), !trans, op(w1, f.k, nc, ldw), w2, ldw, 1.0, 0.0);
    if (rc == RQ_OK) rc = gemm(mp, nc, f.k, Vop, true, op(w2, f.k, nc, ldw), X, ldq, -1.0, 1.0);
    if (rc == RQ_OK && f.q2 && trans) rc = small();
  }
  kwork = save_kw;
  kwork_bytes = save_kb;
  return rc;
}

int Ctx::form_p(const FactorSet& F, double* P, int64_t ldp) {
  if (!F.have) return set_error(RQ_EVALUE, "no factorization stored in this context");
  if (F.p_is_perm) return perm_to_dense(F.perm, F.fn, P, ldp, stream, &launches);
  // P = prod_i (S_i, P-hat_i) applied to I in order (Factorization.expand_p, blocked.py:143-149)
  RQ_TRY(fill_eye(P, ldp, F.fn, F.fn, 0, stream, &launches));
  return apply_p(F, 0, (int)F.rfactors.size(), F.fn, P, ldp);
}

// X (rows x n) <- X P_first ... P_last for orthogonal (reflector-pivot) right factors
// (RightTransform.right_multiply, blocked.py:108-119): S_i = I - V_S T_S V_S^T, then P-hat_i, then
// the panel SVD's V~ (DenseOrtho, blocked.py:53-63).
int Ctx::apply_p(const FactorSet& F, int first, int count, int64_t rows, double* P, int64_t ldp) {
  if (!F.have) return set_error(RQ_EVALUE, "no factorization stored in this context");
  if (F.p_is_perm) return set_error(RQ_EUNSUPPORTED, "permutation pivots: apply the permutation instead");
  const int nf = (int)F.rfactors.size();
  if (first < 0 || count < 0 || first + count > nf)
    return set_error(RQ_EVALUE, "panel range [%d, %d) outside the %d stored right factors", first, first + count, nf);
  if (count == 0 || rows == 0) return RQ_OK;
  const int64_t n = F.fn;
  const int b = F.fb;
  const int64_t ldz = even(rows), ldk = even(b);
  const size_t need = (size_t)3 * ldz * b * 8 + (size_t)ldk * n * 8 + (size_t)ldz * b * 8 + (size_t)n * 4 * 2 + 8192;
  RQ_TRY(qarena.reserve(need));
  Carver c(qarena.base);
  double* z = c.take<double>((size_t)ldz * b);
  double* z2 = c.take<double>((size_t)ldz * b);
  double* vst = c.take<double>((size_t)ldk * n);
  double* stage = c.take<double>((size_t)ldz * std::max<int64_t>(b, 1) * 2);
  int* io = c.take<int>((size_t)n);
  RQ_TRY(iota(io, (int)n, nullptr, 0, stream, &launches));
  for (int i = first; i < first + count; i++) {
    const RightFactors& f = F.rfactors[i];
    if (f.k > 0)
      RQ_TRY(apply_right_wy(P, ldp, rows, n, f.s, f.np, f.k, f.vs, f.ldvs, f.ts, f.ldts, vst, z, z2, ldz));
    if (f.nphat > 0) {
      MoveCall mv{P, ldp, f.s, 0, rows, f.phat, io, nullptr, f.nphat, stage, ldz, nullptr, nullptr};
      RQ_TRY(move_columns_p(mv, stream, &launches));
    }
    if (f.dense) {  // DenseOrtho (blocked.py:53-63): P[:, s:s+w] <- P[:, s:s+w] V~
      RQ_TRY(copy2d_p(P + f.s * ldp, ldp, z, ldz, rows, f.wd, 0, stream, &launches));
      RQ_TRY(gemm(rows, f.wd, f.wd, op(z, rows, f.wd, ldz), true, op(f.dense, f.wd, f.wd, f.ldd), P + f.s * ldp,
                  ldp, 1.0, 0.0));
    }
  }
  return RQ_OK;
}

// Spectral truncation errors ||R(k:, k:)||_2 (metrics.truncation_errors' spectral half,
// metrics.py:37-52, via A P = Q R).  Blocks up to 512 wide: largest singular value from the
// Jacobi SVD kernel (the reference's core.spectral_norm is its Jacobi svd_values, core.py:39-46);
// wider: power iteration on R22^T R22 (DMMA GEMMs), stopped at a relative change below 1e-13 or
// after 2000 iterations.  how[i] = 0 exact (Jacobi), 1 power iteration, 2 empty block.
int Ctx::trailing_spectral(const double* R, int64_t n, int64_t ldr, const int64_t* ks, int nks, double* out,
                           int32_t* how) {
  const int64_t wmax = 512;
  const int64_t ldw = wmax;
  const int64_t ldx = even(n) + 2;
  const size_t need = (size_t)4 * ldw * wmax * 8 + (size_t)wmax * 8 + 64 + (size_t)ldx * 2 * 8 * 2 + 4096 * 8 +
                      (size_t)kSMs * 8 * 8 * 64;
  RQ_TRY(qarena.reserve(need));
  Carver c(qarena.base);
  double* wb = c.take<double>((size_t)ldw * wmax);
  double* vb = c.take<double>((size_t)ldw * wmax);
  double* ub = c.take<double>((size_t)ldw * wmax);
  double* vt = c.take<double>((size_t)ldw * wmax);
  double* d = c.take<double>((size_t)wmax);
  int* status = c.take<int>(16);
  double* x = c.take<double>((size_t)ldx * 2);
  double* y = c.take<double>((size_t)ldx * 2);
  double* norms = c.take<double>(4096);
  double* save_kw = kwork;
  const size_t save_kb = kwork_bytes;
  kwork = nullptr;
  kwork_bytes = 0;
  int rc = RQ_OK;
  for (int i = 0; i < nks && rc == RQ_OK; i++) {
    const int64_t k = ks[i];
    if (k < 0 || k > n) {
      rc = set_error(RQ_EVALUE, "ranks must lie in [0, %lld]", (long long)n);
      break;
    }
    const int64_t w = n - k;
    const double* Rk = R + k + k * ldr;
    if (w == 0) {
      out[i] = 0.0;
      how[i] = 2;
      continue;
    }
    if (w <= wmax) {
      rc = jacobi_svd(Rk, ldr, (int)w, wb, ldw, vb, ldw, d, ub, ldw, vt, ldw, status, stream, &launches);
      if (rc != RQ_OK) break;
      int st = 0;
      double d0 = 0.0;
      if (cudaMemcpyAsync(&st, status, sizeof(int), cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
          cudaMemcpyAsync(&d0, d, 8, cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
          cudaStreamSynchronize(stream) != cudaSuccess) {
        rc = set_error(RQ_ECUDA, "spectral: readback");
        break;
      }
      if (st < 0) {
        rc = set_error(RQ_ECONV, "Jacobi SVD did not converge in 60 sweeps");
        break;
      }
      out[i] = d0;
      how[i] = 0;
      continue;
    }
    // power iteration: x <- R22^T (R22 x) / ||.||, start from the all-ones vector (deterministic)
    std::vector<double> ones((size_t)ldx * 2, 0.0);
    for (int64_t r = 0; r < w; r++) ones[r] = 1.0;
    if (cudaMemcpyAsync(x, ones.data(), (size_t)ldx * 2 * 8, cudaMemcpyHostToDevice, stream) != cudaSuccess ||
        cudaStreamSynchronize(stream) != cudaSuccess) {
      rc = set_error(RQ_ECUDA, "spectral: upload");
      break;
    }
    const GemmOperand Rop = op(R, n, n, ldr, k, k);  // R22 (w x w), NN / TN views
    double prev = -1.0, est = 0.0;
    const int batch = 20, max_it = 2000;
    for (int it = 0; it < max_it && rc == RQ_OK; it += batch) {
      for (int t = 0; t < batch && rc == RQ_OK; t++) {
        rc = gemm(w, 2, w, Rop, true, op(x, ldx, 2, ldx), y, ldx, 1.0, 0.0);            // y = R22 x
        if (rc == RQ_OK) rc = gemm(w, 2, w, Rop, false, op(y, ldx, 2, ldx), x, ldx, 1.0, 0.0);  // x = R22^T y
        if (rc == RQ_OK) rc = normalize_col(x, w, norms, t, stream, &launches);
      }
      if (rc != RQ_OK) break;
      std::vector<double> hn(batch);
      if (cudaMemcpyAsync(hn.data(), norms, batch * 8, cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
          cudaStreamSynchronize(stream) != cudaSuccess) {
        rc = set_error(RQ_ECUDA, "spectral: readback");
        break;
      }
      est = std::sqrt(hn[batch - 1]);  // ||R22^T R22 x|| -> sigma_max^2 for unit x
      const double before = std::sqrt(hn[batch - 2]);
      if (std::fabs(est - before) <= 1e-13 * est || (prev >= 0.0 && std::fabs(est - prev) <= 1e-13 * est)) break;
      prev = est;
    }
    out[i] = est;
    how[i] = 1;
  }
  kwork = save_kw;
  kwork_bytes = save_kb;
  return rc;
}

int Ctx::snapshot(double* hW, int64_t ldh) {
  if (!cur_A) return set_error(RQ_EVALUE, "no factorization in progress");
  RQ_CUDA_TRY(cudaStreamSynchronize(stream));
  const int64_t m = cur_m, n = cur_n, s = cur_lorder ? cur_s : n;
  RQ_CUDA_TRY(cudaMemcpy2D(hW, ldh * 8, cur_A, cur_lda * 8, m * 8, s, cudaMemcpyDeviceToHost));
  if (cur_lorder && s < n) {
    std::vector<int> lo((size_t)(n - s));
    RQ_CUDA_TRY(cudaMemcpy(lo.data(), cur_lorder, (n - s) * sizeof(int), cudaMemcpyDeviceToHost));
    for (int64_t r = 0; r < n - s; r++)
      RQ_CUDA_TRY(cudaMemcpy(hW + (s + r) * ldh, cur_A + (s + lo[r]) * cur_lda, m * 8, cudaMemcpyDeviceToHost));
  }
  return RQ_OK;
}

// The downdated sketch of the current trailing block (Y2 = G2 A22' in exact arithmetic, SURVEY
// section 8 "Two sketch modes") and the composite permutation so far, both in the reference's
// column order: hY is wdt x (n - s) (ldh >= wdt), hperm has n entries.  Test hook for the
// downdate identity; valid inside the inspect callback of a downdated-sketch run.
int Ctx::snapshot_sketch(double* hY, int64_t ldh, int64_t* hperm) {
  if (!cur_A || !cur_yt) return set_error(RQ_EVALUE, "no downdated-sketch factorization in progress");
  if (ldh < cur_wdt) return set_error(RQ_EVALUE, "ldh < sketch width %d", cur_wdt);
  RQ_CUDA_TRY(cudaStreamSynchronize(stream));
  const int64_t n = cur_n, s = cur_lorder ? cur_s : n;
  std::vector<int> lo((size_t)(n - s));
  for (int64_t r = 0; r < n - s; r++) lo[r] = (int)r;
  if (cur_lorder && s < n)
    RQ_CUDA_TRY(cudaMemcpy(lo.data(), cur_lorder, (n - s) * sizeof(int), cudaMemcpyDeviceToHost));
  std::vector<int64_t> orig((size_t)n);
  RQ_CUDA_TRY(cudaMemcpy(orig.data(), cur_orig, n * sizeof(int64_t), cudaMemcpyDeviceToHost));
  for (int64_t r = 0; r < n - s; r++)
    if (hY)
      RQ_CUDA_TRY(cudaMemcpy(hY + r * ldh, cur_yt + (s + lo[r]) * cur_ldy, (size_t)cur_wdt * 8,
                             cudaMemcpyDeviceToHost));
  if (hperm) {
    for (int64_t j = 0; j < s; j++) hperm[j] = orig[j];
    for (int64_t r = 0; r < n - s; r++) hperm[s + r] = orig[s + lo[r]];
  }
  return RQ_OK;
}

// ---------------------------------------------------------------------------
// Panel-step API: the pieces of factorize_perm (steps 3, 5-9) on caller-owned
// buffers, for a driver that distributes the columns itself (dist.py, SURVEY
// section 8(e)).  Scratch comes from `sarena`.
// ---------------------------------------------------------------------------
namespace {
struct StepScratch {
  double *w1, *w2, *ttop, *gram, *tleaf, *small, *rfin, *kwork, *vpad;
  size_t kwork_bytes;
  void* sweep_ws;
  size_t sweep_ws_bytes;
  size_t total;
};

StepScratch plan_step(void* base, int64_t ncols, int b, int64_t mp = 0) {
  StepScratch S;
  Carver c(base);
  const int64_t ldb = even(b);
  const int64_t nc = std::max<int64_t>(ncols, b);
  S.w1 = c.take<double>((size_t)ldb * nc);
  S.w2 = c.take<double>((size_t)ldb * nc);
  S.ttop = c.take<double>((size_t)ldb * nc);
  S.gram = c.take<double>((size_t)ldb * b);
  S.tleaf = c.take<double>(32 * 32);
  S.small = c.take<double>((size_t)ldb * 2 * b);
  S.rfin = c.take<double>((size_t)ldb * b);
  S.kwork_bytes = std::max<size_t>((size_t)kSMs * (b + 1) * b * 8, (size_t)16 * (b + 1) * nc * 8);
  S.kwork = c.take<double>(S.kwork_bytes / 8);
  S.sweep_ws_bytes = sweep_workspace_bytes(b, 2 * b, sweep_grid_size(2 * b));
  S.sweep_ws = c.take<char>(S.sweep_ws_bytes);
  S.vpad = c.take<double>((size_t)even(mp + 1) * b);  // V at a one-row offset (operand parity)
  S.total = c.off;
  return S;
}
}  // namespace

int Ctx::step_sketch_select(double* Y, int64_t ldy, int m, int n, int steps, const int* init_pos, int* chosen) {
  const size_t ws = std::max(sweep_workspace_bytes(m, n, kSMs), sketch_workspace_bytes(m, n)) + 4096;
  RQ_TRY(sarena.reserve(ws));
  sweep_ws = sarena.base;
  sweep_ws_bytes = ws;
  return sketch_select(Y, ldy, m, n, steps, init_pos, chosen);
}

int Ctx::step_panel_factor(double* P, int64_t ldp, int64_t mp, int b, double* V, int64_t ldv, double* T, int64_t ldt,
                           double* Q2, int64_t ldq2, int* phat) {
  RQ_TRY(sarena.reserve(plan_step(nullptr, b, b).total));
  StepScratch S = plan_step(sarena.base, b, b);
  kwork = S.kwork;
  kwork_bytes = S.kwork_bytes;
  sweep_ws = S.sweep_ws;
  sweep_ws_bytes = S.sweep_ws_bytes;
  const int64_t lds = even(b);
  // 5: unpivoted panel QR (V lower trapezoidal: leaves write rows >= their diagonal)
  RQ_CUDA_TRY(cudaMemsetAsync(V, 0, (size_t)ldv * b * sizeof(double), stream));
  launches++;
  RQ_TRY(panel_qr(P, ldp, mp, b, 0, mp, b, V, ldv, 0, S.tleaf, S.w1, S.w2));
  // 6: b x b CPQR of R' (reflectors V2), Q2 = I - V2 T2 V2^T
  double* Sm = S.small;
  double* V2 = S.small + (int64_t)b * lds;
  RQ_TRY(copy2d_p(P, ldp, Sm, lds, b, b, 1, stream, &launches));
  RQ_CUDA_TRY(cudaMemsetAsync(V2, 0, (size_t)lds * b * sizeof(double), stream));
  launches++;
  SweepCall ss;
  ss.a = Sm;
  ss.lda = lds;
  ss.m = b;
  ss.n = b;
  ss.steps = b;
  ss.pivot = 1;
  ss.v = V2;
  ss.ldv = lds;
  ss.col_at_pos = phat;
  ss.r_out = S.rfin;
  ss.ldr = lds;
  RQ_TRY(sweep(ss));
  Layout L{};
  L.ttop = S.ttop;
  L.gram = S.gram;
  L.w1 = S.w1;
  L.w2 = S.w2;
  RQ_TRY(small_q(V2, lds, b, Q2, ldq2, L));
  // 7: R of the panel (columns in P-hat order)
  RQ_TRY(copy2d_p(S.rfin, lds, P, ldp, b, b, 0, stream, &launches));
  // 8: T of the panel reflectors
  return tfactor(V, mp, b, ldv, 0, T, ldt, S.gram);
}

int Ctx::step_panel_apply(const double* V, int64_t ldv, const double* T, int64_t ldt, const double* Q2, int64_t ldq2,
                          int64_t mp, int b, double* A, int64_t lda, int64_t a_rows, int64_t a_cols, int64_t r0,
                          int64_t c0, int64_t n2) {
  if (n2 <= 0 || mp <= 0) return RQ_OK;
  const bool odd = (r0 & 1) != 0;
  RQ_TRY(sarena.reserve(plan_step(nullptr, n2, b, odd ? mp : 0).total));
  StepScratch S = plan_step(sarena.base, n2, b, odd ? mp : 0);
  kwork = S.kwork;
  kwork_bytes = S.kwork_bytes;
  const int64_t ldw = even(b);
  // the GEMM's K origins of V and A2 must share parity (16-byte TMA coordinates):
  // for an odd r0, V is staged one row down, as factorize_perm's vpad does
  GemmOperand Vop = op(V, mp, b, ldv, 0);
  if (odd) {
    const int64_t ldp = even(mp + 1);
    RQ_TRY(copy2d_p(V, ldv, S.vpad + 1, ldp, mp, b, 0, stream, &launches));
    Vop = op(S.vpad, mp + 1, b, ldp, 1);
  }
  CatGuard guard(cat, PROF_TRAIL);
  double* A2 = A + r0 + c0 * lda;
  RQ_TRY(gemm(b, n2, mp, Vop, false, op(A, a_rows, a_cols, lda, r0, c0), S.w1, ldw, 1.0, 0.0));
  RQ_TRY(gemm(b, n2, b, op(T, b, b, ldt), false, op(S.w1, b, n2, ldw), S.w2, ldw, 1.0, 0.0));
  RQ_TRY(gemm(mp, n2, b, Vop, true, op(S.w2, b, n2, ldw), A2, lda, -1.0, 1.0));
  if (Q2) {
    RQ_TRY(copy2d_p(A2, lda, S.ttop, ldw, b, n2, 0, stream, &launches));
    RQ_TRY(gemm(b, n2, b, op(Q2, b, b, ldq2), false, op(S.ttop, b, n2, ldw), A2, lda, 1.0, 0.0));
  }
  return RQ_OK;
}

Ctx::~Ctx() {
  if (sk_block) cudaFree(sk_block);
  if (sb_ws) cudaFree(sb_ws);
  if (gsched) cudaFree(gsched);
  for (auto e : ev_pool) cudaEventDestroy(e);
  arena.release();
  qarena.release();
  sarena.release();
  harena.release();
  if (side) cudaStreamDestroy(side);
  if (hip) cudaStreamDestroy(hip);
  if (copy_stream) cudaStreamDestroy(copy_stream);
  if (ev_g1) cudaEventDestroy(ev_g1);
  if (ev_hipdone) cudaEventDestroy(ev_hipdone);
  if (copy_ev) cudaEventDestroy(copy_ev);
  if (h2d_stream) cudaStreamDestroy(h2d_stream);
  for (cudaEvent_t e : h2d_ev) cudaEventDestroy(e);
  if (ev_v) cudaEventDestroy(ev_v);
  if (ev_side) cudaEventDestroy(ev_side);
  if (ev_hi) cudaEventDestroy(ev_hi);
  if (aux) cudaStreamDestroy(aux);
  if (ev_l0) cudaEventDestroy(ev_l0);
  if (ev_aux) cudaEventDestroy(ev_aux);
  if (ev_w2) cudaEventDestroy(ev_w2);
  if (hip2) cudaStreamDestroy(hip2);
  if (ev_q2) cudaEventDestroy(ev_q2);
  if (ev_gram) cudaEventDestroy(ev_gram);
  if (ev_t) cudaEventDestroy(ev_t);
  if (barriers) cudaFree(barriers);
}

}  // namespace rq
