// Host-side driver state (see driver.cu) behind the opaque rq_ctx.
#pragma once
#include <functional>
#include <vector>

#include "common.cuh"
#include "gemm_f64.cuh"
#include "misc.cuh"
#include "sweep.cuh"

namespace rq {

static inline int64_t even(int64_t x) { return (x + 1) & ~int64_t(1); }

struct Arena {
  void* base = nullptr;
  size_t cap = 0;
  int reserve(size_t bytes);
  void release();
};

struct Layout {
  // scratch
  double *omega, *yt, *w1, *w2, *gram, *tleaf, *ybuf, *kwork, *small, *rfin, *stage, *ttop, *rinv, *g1;
  double *zbuf, *z2buf, *vst;  // reflector pivots: A V_S, (A V_S) T_S, V_S^T
  double *ov, *ot, *oe;         // _orth scratch: reflectors, T, Q
  double *wside, *gram2, *kwork2;  // side stream: W = V^T A2, Gram, split-K slabs
  size_t kwork2_bytes;
  double *jw, *jv, *jd;         // panel SVD scratch
  int* jstat;                   // per-panel Jacobi sweep counts
  int64_t ldo, ldy, lds_small;
  int *chosen, *lorderA, *lorderB, *rankA, *rankB, *newloc, *src, *dst, *nmoves, *cap, *iota_b;
  unsigned char* flag;
  int64_t *orig, *ostage;
  // the b x b CPQR's own buffers when it runs beside the next panel's sketch CPQR (cpqr_off)
  int* cap2;
  double* stage2;
  int64_t* ostage2;
  void* sweep_ws2;
  size_t sweep_ws2_bytes;
  void* sweep_ws;
  size_t sweep_ws_bytes;
  size_t kwork_bytes;
  // stored factors
  double* fstore;
  size_t total;
};

// Compact factors of one panel: U = (I - V T V^T) diag(Q2, I) on rows s..m-1.
struct PanelFactors {
  int64_t s;
  int k;  // reflector count
  double* v;  // buffer base; row r of the reflectors is v[vpad + r]
  int64_t ldv;
  int vpad;   // 1 when s is odd: keeps TMA coordinates 16-byte aligned
  double* t;
  int64_t ldt;
  double* q2;   // k x k Q2 of the b x b CPQR (null for the final block)
  int64_t ldq2;
};

// Kernel classes timed with CUDA events when profiling is on (rq_set_profiling).
enum ProfCat {
  PROF_TRAIL = 0,       // trailing-update GEMMs
  PROF_GEMM_OTHER = 1,  // sketch, Gram, intra-panel GEMMs
  PROF_SWEEP = 2,       // sketch CPQR (pivot selection)
  PROF_LEAF = 3,        // panel leaf QR
  PROF_OTHER = 4,
  PROF_SMALL = 5,       // b x b CPQR of R' and the final block
  PROF_SKETCH_GEMM = 6, // Y = Omega^T X (+ power iterations)
  PROF_PANEL_GEMM = 7,  // WY updates between panel leaves
  PROF_TFACTOR = 8,     // Gram V^T V + T back substitution, small Q2
  PROF_MOVES = 9,       // column moves (gather + scatter at full height)
  PROF_COPY = 10,       // copy2d
  PROF_RNG = 11,        // Gaussian fills
  PROF_SPLITK = 12,     // split-K reductions of the GEMMs
  PROF_NCAT = 13
};

struct ProfRec {
  int cat;
  cudaEvent_t e0, e1;
  double flops;
  double bytes = 0.0;  // algorithmic HBM bytes (bandwidth classes)
};

// Right factor of one panel with reflector pivots: S = I - V_S T_S V_S^T on
// columns s.., followed by the panel's inner permutation P-hat.
struct RightFactors {
  int64_t s, np;
  int k;
  double* vs;  // np x k
  int64_t ldvs;
  double* ts;  // k x k
  int64_t ldts;
  int* phat;   // k (or np for the final block)
  int nphat;
  double* dense;  // w x w right factor V~ of the panel SVD (block_rrqr), or null
  int64_t ldd;
  int wd;
};

// A factorization's compact factors, detached from the context that computed them
// (rq_factors_detach): the set owns the device workspace they live in, so later
// factorizations on the context allocate fresh workspace and never overwrite them.
struct FactorSet {
  Arena arena;
  std::vector<PanelFactors> factors;
  std::vector<RightFactors> rfactors;
  bool p_is_perm = true;
  int64_t* perm = nullptr;
  int64_t fm = 0, fn = 0;
  int fb = 0;
  bool have = false;
  int device = 0;
};

struct Ctx {
  int device = 0;
  // profiling
  bool prof = false;
  int cat = PROF_OTHER;
  std::vector<ProfRec> prof_recs;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_next = 0;
  cudaEvent_t prof_event();
  void prof_begin(cudaEvent_t* e0);
  void prof_end(cudaEvent_t e0, double flops, double bytes = 0.0);
  unsigned long long* prof_dev_bytes = nullptr;  // device counter: bytes of the column moves
  int copy2d_p(const double* S, int64_t lds, double* D, int64_t ldd, int64_t rows, int64_t cols, int upper_only,
               cudaStream_t st, int64_t* l);
  int move_columns_p(MoveCall c, cudaStream_t st, int64_t* l);
  int gaussian_fill_p(double* out, int64_t rows, int64_t cols, int64_t ld, uint64_t seed, uint64_t counter,
                      cudaStream_t st, int64_t* l);
  cudaStream_t stream = nullptr;
  rq_panel_cb inspect_cb = nullptr;
  void* inspect_user = nullptr;
  int64_t launches = 0;
  Arena arena, qarena, sarena;  // factorization, Q/P formation + test hooks, panel-step API
  Arena harena;                 // rq_factorize_host: device copy of A and the permutation
  cudaStream_t copy_stream = nullptr;  // rq_factorize_host: R streams to the host on this stream
  cudaEvent_t copy_ev = nullptr;
  cudaStream_t h2d_stream = nullptr;   // rq_factorize_host: A arrives in column chunks on this stream
  std::vector<cudaEvent_t> h2d_ev;     // one per chunk
  bool presketched = false;            // the next factorize_perm finds G drawn and Y = G A formed (presketch_*)
  int presketch_begin(const rq_config& cfg, int64_t m, int64_t n, uint64_t seed, uint64_t counter);
  int presketch_cols(const rq_config& cfg, int64_t m, int64_t n, const double* A, int64_t lda, int64_t c0,
                     int64_t c1);
  unsigned int* barriers = nullptr;
  int nbarriers = 0;
  int next_barrier = 0;
  // overlap (factorize_perm): the b x b CPQR on a highest-priority stream `hip`,
  // W = V^T A2 and T on a lowest-priority stream `side`
  cudaStream_t side = nullptr, hip = nullptr;
  cudaEvent_t ev_v = nullptr, ev_side = nullptr, ev_hi = nullptr;
  // space-sliced look-ahead (panel_qr): the panel's later leaves and cluster WY updates on `aux`
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_l0 = nullptr, ev_aux = nullptr;
  cudaEvent_t ev_w2 = nullptr;  // look-ahead: W2 = T^T W formed on the side stream
  cudaStream_t hip2 = nullptr;  // second highest-priority stream (Q2 beside G1')
  cudaEvent_t ev_q2 = nullptr, ev_gram = nullptr, ev_t = nullptr;
  bool tinv_par = false;  // the panel's T inverse on hip2 beside the rest of W
  bool w2_side = false;
  bool overlap_on = true;
  // called (host side, enqueue order) when columns [s, s + w) of R are final: no later step
  // writes them (rq_factorize_host streams them to the host while later panels compute)
  std::function<void(int64_t, int64_t)> on_cols_final;
  int gemm_max_ctas = 0;
  bool tf32_update = false;  // RQ_FLAG_TF32_UPDATE: trailing-update GEMMs on the tcgen05 3xTF32 kernel
  int gemm_cap = 0;  // rq_ctx_set_gemm_cap: default grid cap of this context's GEMMs (0 = none)
  bool gemm_pdl = false;
  cudaEvent_t gemm_mid = nullptr;  // profiling: split-K reduce boundary of the current GEMM
  int gemm_splitk = 1;
  // dynamic GEMM unit scheduling: one monotone device counter per stream (main, side, hip) and
  // its host mirror (GEMMs on one stream never overlap each other, so a counter is never shared)
  unsigned long long* gsched = nullptr;
  unsigned long long gsched_base[3] = {0, 0, 0};
  int sched_for(cudaStream_t st, unsigned long long** ctr, unsigned long long** base);
  int ensure_side();
  // look-ahead (factorize_perm, downdated sketches): the previous panel's A2 -= V W2 on the
  // columns after the current panel, issued in tile-range chunks, each launched right behind one
  // of the current panel's leaf kernels (programmatic serialization: it runs on the SMs the
  // leaf's cluster leaves free)
  struct LaPending {
    bool on = false;
    GemmProblem g;  // the whole GEMM; chunks set tile_begin/tile_end
    int64_t tiles = 0, next = 0;
  } la;
  int la_chunk(int64_t upto, bool beside_leaf);
  // RQ_PHASES=1: CUDA events at phase boundaries of factorize_perm on the main stream (never
  // between a leaf and its look-ahead chunk); per-phase totals printed to stderr per call
  bool phases_on = false;
  std::vector<std::pair<int, cudaEvent_t>> phase_ev;
  std::vector<double> phase_host;  // host clock (ms) at each phase() call
  std::vector<std::pair<int, cudaEvent_t>> side_ev;  // side stream: W GEMM parts and T
  void phase(int id);
  void side_phase(int id);
  void phase_report();
  int la_flush() { return la.on ? la_chunk(la.tiles, false) : RQ_OK; }
  // scratch views used by helpers
  double* kwork = nullptr;
  size_t kwork_bytes = 0;
  void* sweep_ws = nullptr;
  size_t sweep_ws_bytes = 0;
  // stored factorization
  std::vector<PanelFactors> factors;
  std::vector<RightFactors> rfactors;  // reflector pivots (P is orthogonal, not a permutation)
  bool p_is_perm = true;
  int64_t* factors_perm = nullptr;
  int64_t fm = 0, fn = 0;
  int fb = 0;
  bool have_factors = false;
  // in-progress view for rq_snapshot
  double* cur_A = nullptr;
  int64_t cur_lda = 0, cur_m = 0, cur_n = 0, cur_s = 0, cur_np = 0;
  int* cur_lorder = nullptr;
  int64_t* cur_orig = nullptr;
  double* cur_yt = nullptr;  // downdated sketch (rq_snapshot_sketch): wdt x n, physical column slots
  int64_t cur_ldy = 0;
  int cur_wdt = 0;

  ~Ctx();
  int gemm(int64_t M, int64_t N, int64_t K, const GemmOperand& A, bool a_mmajor, const GemmOperand& B, double* C,
           int64_t ldc, double alpha, double beta);
  int gemm_raw(int64_t M, int64_t N, int64_t K, const GemmOperand& A, bool a_mmajor, const GemmOperand& B, double* C,
               int64_t ldc, double alpha, double beta);
  int sweep(SweepCall c);
  int sweep_raw(SweepCall c);
  // off-chain b x b CPQR (look-ahead, RQ_CPQR_OFF): panel i's CPQR, Q2, R and rows-above moves run
  // on the 16-SM cluster / hip stream beside panel i+1's sketch CPQR, which is capped at
  // kSkMinGrid CTAs; the main stream joins them (ev_hipdone) before it moves panel i+1's columns
  bool cpqr_off = false;
  int sketch_gmax = 0;
  cudaEvent_t ev_g1 = nullptr, ev_hipdone = nullptr;
  int finish_top(double* A, int64_t lda, int64_t s, int b, int64_t n2, const double* Q2, int64_t ldt, Layout& L);
  unsigned long long* sk_counter = nullptr;  // device: monotone arrival counter of the sketch CPQR + its winner records
  unsigned long long sk_counter_base = 0;    // host mirror of its value
  char* sk_block = nullptr;  // the allocation sk_counter points into (place_sketch_words)
  bool sk_placed = false;    // its offset was calibrated
  char* sk_ll = nullptr;     // the sketch CPQR's slots + LL columns (inside sk_block, offset calibrated)
  int place_sketch_words(int m, int n, int steps);
  void* sb_ws = nullptr;                     // device: exchange words of the batched sketch CPQR (sketch_batch.cu)
  unsigned long long sb_stamp_base = 0;      // its monotone event stamps
  bool sketch_batched(int m, int n, int steps, int gmax) const;  // sketch_select takes the batched kernel
  int sketch_select(const double* yt, int64_t ldy, int m, int n, int steps, const int* init_pos, int* chosen);
  int panel_qr(double* A, int64_t lda, int64_t m, int64_t n, int64_t s, int64_t mp, int b, double* V, int64_t ldv,
               int vpad, double* tleaf, double* w1, double* w2, double* T = nullptr, int64_t ldt = 0,
               bool* t_done = nullptr);
  double* gram_aux = nullptr;  // Gram scratch for the panel's T computed on the aux stream
  std::function<int()> aux_g1;  // form_g1 of the current panel (run on aux in space mode)
  bool g1_done = false;
  int form_g1(double* A, int64_t lda, int64_t s, int b, int wdt, int64_t n, Layout& L);
  int tfactor(const double* V, int64_t rows, int k, int64_t ldv, int vpad, double* T, int64_t ldt, double* gram);
  int sketch(const rq_config& cfg, double* A, int64_t lda, int64_t m, int64_t n, int64_t s, int64_t mp, int64_t np,
             Layout& L, bool want_y = false);
  int apply_right_wy(double* A, int64_t lda, int64_t rows, int64_t ncols_total, int64_t s, int64_t np, int k,
                     const double* VS, int64_t ldvs, const double* TS, int64_t ldts, double* vst, double* z,
                     double* z2, int64_t ldz);
  int trailing_update(double* A, int64_t lda, int64_t m, int64_t n, int64_t s, int64_t mp, int b, int64_t n2,
                      const double* V, int64_t ldv, int vpad, const double* T, int64_t ldt, const double* Q2,
                      Layout& L, const double* Wpre = nullptr);
  int lookahead_tail(const rq_config& cfg, double* A, int64_t lda, int64_t m, int64_t n, int64_t s, int64_t mp, int b,
                     int64_t n2, const double* V, int64_t ldv, int vpad, const double* T, int64_t ldt, const double* Q2,
                     Layout& L, const double* Wpre, int*& lorder, int*& lorder_n, int*& rank, int*& rank_n);
  int factorize_perm(const rq_config& cfg, int64_t m, int64_t n, double* A, int64_t lda, uint64_t seed,
                     uint64_t* counter, int64_t* dperm);
  int small_q(const double* V2, int64_t ldv2, int k, double* Q2, int64_t ldq, Layout& L);
  int factorize_rrqr(const rq_config& cfg, int64_t m, int64_t n, double* A, int64_t lda, uint64_t seed,
                     uint64_t* counter);
  int orth(double* src, int64_t rows, int cols, int64_t ld, Layout& L);
  int reflector_pivot(const rq_config& cfg, double* A, int64_t lda, int64_t m, int64_t n, int64_t s, Layout& L,
                      void* fc_ptr, uint64_t seed, uint64_t* counter);
  FactorSet view() const;     // the stored factorization (no workspace ownership)
  int detach(FactorSet* out);  // move the stored factorization and its workspace out
  int form_q(const FactorSet& F, int64_t cols, double* Q, int64_t ldq);
  int factorize_unpivoted(int64_t m, int64_t n, double* A, int64_t lda, int b);
  // Panel-step API for drivers that own the column distribution (multi-GPU, dist.py)
  int step_sketch_select(double* Y, int64_t ldy, int m, int n, int steps, const int* init_pos, int* chosen);
  int step_panel_factor(double* P, int64_t ldp, int64_t mp, int b, double* V, int64_t ldv, double* T, int64_t ldt,
                        double* Q2, int64_t ldq2, int* phat);
  int step_panel_apply(const double* V, int64_t ldv, const double* T, int64_t ldt, const double* Q2, int64_t ldq2,
                       int64_t mp, int b, double* A, int64_t lda, int64_t a_rows, int64_t a_cols, int64_t r0,
                       int64_t c0, int64_t n2);
  int form_p(const FactorSet& F, double* P, int64_t ldp);
  int apply_q(const FactorSet& F, int first, int count, bool trans, bool eye, int64_t cols, double* X, int64_t ldx);
  int apply_p(const FactorSet& F, int first, int count, int64_t rows, double* X, int64_t ldx);
  int snapshot(double* hW, int64_t ldh);
  int trailing_spectral(const double* R, int64_t n, int64_t ldr, const int64_t* ks, int nks, double* out,
                        int32_t* how);
  int snapshot_sketch(double* hY, int64_t ldh, int64_t* hperm);
};

}  // namespace rq

struct rq_ctx {
  rq::Ctx c;
};

struct rq_factors {
  rq::FactorSet f;
};
