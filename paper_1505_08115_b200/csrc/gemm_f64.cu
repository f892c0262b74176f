// FP64 DMMA GEMM with a TMA/mbarrier producer-consumer pipeline (see gemm_f64.cuh).
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "gemm_f64.cuh"

namespace rq {

// ---------------------------------------------------------------------------
// PTX wrappers: mbarrier + TMA
// ---------------------------------------------------------------------------

RQ_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
RQ_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
RQ_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
RQ_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}
RQ_DEV void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
RQ_DEV void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

RQ_DEV void dmma_16x8x4(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// ---------------------------------------------------------------------------
// Kernel
// ---------------------------------------------------------------------------
constexpr int BK = 16;  // 16 doubles = one 128 B swizzle row

struct KArgs {
  int64_t M, N, K;
  int a_c0, a_c1;  // TMA coordinate origins of the A view (dim0, dim1)
  int b_c0, b_c1;
  double* C;
  int64_t ldc;
  double alpha, beta;
  int tiles_m, tiles_n, splitk, kchunks_per_split;
  int64_t kchunks;
  double* work;  // split-K slabs (ld = M)
  int k_lo;      // 1: element k = 0 is padding (odd K origin shifted to even)
  int m_lo;      // 1: output row 0 is padding (odd M origin shifted to even)
  int u0, u1;    // unit range of this launch (a tile-range chunk of a larger GEMM, or all units)
  unsigned long long* sched;       // non-null: units handed out by an atomic counter (dynamic)
  unsigned long long sched_base;   // the counter's value when this launch starts
};

template <int BM, int BN, int WARPS_M, int WARPS_N, bool A_MMAJOR, int STAGES>
struct GemmCfg {
  static constexpr int kConsumerWarps = WARPS_M * WARPS_N;
  static constexpr int kThreads = kConsumerWarps * 32;  // thread 0 doubles as the TMA producer
  static constexpr int WTM = BM / WARPS_M;
  static constexpr int WTN = BN / WARPS_N;
  static constexpr int MT = WTM / 16;
  static constexpr int NT = WTN / 8;
  static constexpr int A_LDM = BM + 4;  // padded M-major row: 4 k-rows of a half-warp hit 4 distinct 32 B bank groups
  static constexpr int A_BYTES = A_MMAJOR ? BK * A_LDM * 8 : BM * BK * 8;
  static constexpr int A_BYTES_AL = (A_BYTES + 1023) / 1024 * 1024;
  static constexpr int B_BYTES = BN * BK * 8;
  static constexpr int STAGE_BYTES = A_BYTES_AL + B_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 2 * STAGES * 8 + 8 * 4 /*unit ring*/;
  static_assert(WTM % 16 == 0 && WTN % 8 == 0, "warp tile");
  static_assert(B_BYTES % 1024 == 0, "swizzle-128B stage alignment");
};

// MMA row/column index g -> shared-memory row, so that the 16 lanes of a
// half-warp (g = 0..3 x 4 k) hit 8 distinct 16-byte chunks of the 128B-swizzled
// K-major tile (rows 0,2,4,6 then 1,3,5,7).  Undone in the epilogue.
RQ_DEV int perm8(int g) { return ((g & 3) << 1) | (g >> 2); }

// element (r, k) of a K-major 16-wide tile written by TMA with SWIZZLE_128B
RQ_DEV double ld_kmajor(const char* tile, int r, int k) {
  const int off = r * 128 + ((((k >> 1) ^ (r & 7))) << 4) + ((k & 1) << 3);
  return *reinterpret_cast<const double*>(tile + off);
}

// Walks this CTA's (unit, k-chunk) sequence.  Units are assigned round-robin (static) or, with
// a.sched, taken from an atomic counter as the producer reaches them (dynamic: CTAs that start
// late, e.g. behind a concurrent kernel, simply take fewer units).  In dynamic mode the producer
// publishes each unit it starts in a shared-memory ring (entry -1: no more units) that the
// consumer warps read after the unit's first stage is full.  Every unit has >= 1 k-chunk.
struct ChunkCursor {
  int u;
  int64_t kc, kc_end;
  bool valid;
  int seq;
  RQ_DEV void unit_range(const KArgs& a) {
    const int split = u % a.splitk;
    kc = (int64_t)split * a.kchunks_per_split;
    kc_end = kc + a.kchunks_per_split;
    if (kc_end > a.kchunks) kc_end = a.kchunks;
  }
  RQ_DEV void begin_unit(const KArgs& a, int units, int* ring) {
    valid = u < units;
    if (a.sched) ring[seq & 7] = valid ? u : -1;
    seq++;
    if (valid) unit_range(a);
  }
  RQ_DEV int fetch(const KArgs& a) {
    const unsigned long long t = atomicAdd(a.sched, 1ull) - a.sched_base;
    return a.u0 + (int)min(t, (unsigned long long)0x3fffffff);
  }
  RQ_DEV void start(const KArgs& a, int units, int* ring) {
    seq = 0;
    u = a.sched ? fetch(a) : a.u0 + (int)blockIdx.x;
    begin_unit(a, units, ring);
  }
  RQ_DEV void next(const KArgs& a, int units, int* ring) {
    kc++;
    if (kc < kc_end) return;
    u = a.sched ? fetch(a) : u + (int)gridDim.x;
    begin_unit(a, units, ring);
  }
};

template <int BM, int BN, int WARPS_M, int WARPS_N, bool A_MMAJOR, int STAGES>
RQ_DEV void issue_stage(const CUtensorMap* tmA, const CUtensorMap* tmB, const KArgs& a, unsigned char* smem,
                        uint64_t* full, int stage, const ChunkCursor& c) {
  using Cfg = GemmCfg<BM, BN, WARPS_M, WARPS_N, A_MMAJOR, STAGES>;
  const int t = c.u / a.splitk;
  const int tm = t % a.tiles_m;
  const int tn = t / a.tiles_m;
  unsigned char* sA = smem + stage * Cfg::STAGE_BYTES;
  unsigned char* sB = sA + Cfg::A_BYTES_AL;
  mbar_expect_tx(&full[stage], Cfg::A_BYTES + Cfg::B_BYTES);
  const int k = (int)(c.kc * BK);
  if (A_MMAJOR)
    tma_load_2d(sA, tmA, &full[stage], a.a_c0 + tm * BM, a.a_c1 + k);
  else
    tma_load_2d(sA, tmA, &full[stage], a.a_c0 + k, a.a_c1 + tm * BM);
  tma_load_2d(sB, tmB, &full[stage], a.b_c0 + k, a.b_c1 + tn * BN);
}

template <int BM, int BN, int WARPS_M, int WARPS_N, bool A_MMAJOR, int STAGES>
__global__ void __launch_bounds__(GemmCfg<BM, BN, WARPS_M, WARPS_N, A_MMAJOR, STAGES>::kThreads,
                                  (GemmCfg<BM, BN, WARPS_M, WARPS_N, A_MMAJOR, STAGES>::kThreads <= 128) ? 2 : 1)
    gemm_f64_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const KArgs args) {
  using Cfg = GemmCfg<BM, BN, WARPS_M, WARPS_N, A_MMAJOR, STAGES>;
  extern __shared__ unsigned char smem_raw[];
  // 1024-byte alignment by offsetting the __shared__ array itself (not through uintptr_t),
  // so fragment loads stay LDS instead of generic LD with 64-bit address arithmetic
  const uint32_t mis = (uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u;
  unsigned char* smem = smem_raw + ((1024u - mis) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  int* ring = reinterpret_cast<int*>(empty + STAGES);
  const bool dyn = args.sched != nullptr;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int units = args.u1;  // units [u0, u1) of tiles_m * tiles_n * splitk

  // producer cursor (thread 0 only) runs STAGES chunks ahead of the consumers
  ChunkCursor prod;
  int pstage = 0;
  uint32_t pphase = 0;
  bool pterm = false;  // dynamic: the "no more units" stage was signalled
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    prod.start(args, units, ring);
    for (int s = 0; s < STAGES; s++) {
      if (prod.valid) {
        issue_stage<BM, BN, WARPS_M, WARPS_N, A_MMAJOR, STAGES>(&tmA, &tmB, args, smem, full, pstage, prod);
        prod.next(args, units, ring);
      } else if (dyn && !pterm) {
        mbar_arrive(&full[pstage]);  // empty stage: the consumers read ring entry -1 and stop
        pterm = true;
      } else {
        break;
      }
      if (++pstage == STAGES) {
        pstage = 0;
        pphase ^= 1;
      }
    }
  }
  __syncthreads();

  const int wm = warp % WARPS_M;
  const int wn = warp / WARPS_M;
  const int g = lane >> 2;
  const int tq = lane & 3;
  const int pg = perm8(g);
  int stage = 0;
  uint32_t phase = 0;

  int cseq = 0;
  for (int u = args.u0 + blockIdx.x;; u += gridDim.x) {
    if (dyn) {
      mbar_wait(&full[stage], phase);  // the unit's first stage (or the terminal signal)
      u = ring[cseq & 7];
      cseq++;
      if (u < 0) break;
    } else if (u >= units) {
      break;
    }
    const int split = u % args.splitk;
    const int t = u / args.splitk;
    const int tm = t % args.tiles_m;
    const int tn = t / args.tiles_m;
    const int64_t kc_begin = (int64_t)split * args.kchunks_per_split;
    int64_t kc_end = kc_begin + args.kchunks_per_split;
    if (kc_end > args.kchunks) kc_end = args.kchunks;

    double acc[Cfg::MT][Cfg::NT][4];
#pragma unroll
    for (int i = 0; i < Cfg::MT; i++)
#pragma unroll
      for (int j = 0; j < Cfg::NT; j++)
#pragma unroll
        for (int e = 0; e < 4; e++) acc[i][j][e] = 0.0;
    if (args.splitk == 1 && args.beta != 0.0) {
      // pull this warp's C sub-tile (WTM x WTN) towards L2 while the mainloop runs
      const int64_t pm0 = (int64_t)tm * BM + wm * Cfg::WTM;
      const int64_t pn0 = (int64_t)tn * BN + wn * Cfg::WTN;
      constexpr int kLinesPerCol = (Cfg::WTM * 8 + 127) / 128;
      for (int q = lane; q < Cfg::WTN * kLinesPerCol; q += 32) {
        const int64_t n = pn0 + q / kLinesPerCol;
        const int64_t m = pm0 + (q % kLinesPerCol) * 16;
        if (n < args.N && m < args.M && m >= 0)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(args.C + n * args.ldc + m));
      }
    }

    for (int64_t kc = kc_begin; kc < kc_end; kc++) {
      mbar_wait(&full[stage], phase);
      const unsigned char* sA = smem + stage * Cfg::STAGE_BYTES;
      const unsigned char* sB = sA + Cfg::A_BYTES_AL;
      const int64_t kvalid = args.K - kc * BK;  // >= 16 except on the K tail
      const int klo = (kc == 0) ? args.k_lo : 0;  // leading padding element
      if (kvalid >= BK && klo == 0) {
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
          double af[Cfg::MT][2], bf[Cfg::NT];
#pragma unroll
          for (int i = 0; i < Cfg::MT; i++) {
            if (A_MMAJOR) {
              const int r = wm * Cfg::WTM + i * 16 + g;
              const double* a = reinterpret_cast<const double*>(sA);
              af[i][0] = a[(kk + tq) * Cfg::A_LDM + r];
              af[i][1] = a[(kk + tq) * Cfg::A_LDM + r + 8];
            } else {
              const int r = wm * Cfg::WTM + i * 16 + pg;
              af[i][0] = ld_kmajor((const char*)sA, r, kk + tq);
              af[i][1] = ld_kmajor((const char*)sA, r + 8, kk + tq);
            }
          }
#pragma unroll
          for (int j = 0; j < Cfg::NT; j++)
            bf[j] = ld_kmajor((const char*)sB, wn * Cfg::WTN + j * 8 + pg, kk + tq);
#pragma unroll
          for (int i = 0; i < Cfg::MT; i++)
#pragma unroll
            for (int j = 0; j < Cfg::NT; j++) dmma_16x8x4(acc[i][j], af[i][0], af[i][1], bf[j]);
        }
      } else {
        // K tail: mask k >= K (the TMA box may have read real, unrelated data)
        for (int kk = 0; kk < BK; kk += 4) {
          const bool ok = (kk + tq) < kvalid && (kk + tq) >= klo;
          double af[Cfg::MT][2], bf[Cfg::NT];
#pragma unroll
          for (int i = 0; i < Cfg::MT; i++) {
            if (A_MMAJOR) {
              const int r = wm * Cfg::WTM + i * 16 + g;
              const double* a = reinterpret_cast<const double*>(sA);
              af[i][0] = ok ? a[(kk + tq) * Cfg::A_LDM + r] : 0.0;
              af[i][1] = ok ? a[(kk + tq) * Cfg::A_LDM + r + 8] : 0.0;
            } else {
              const int r = wm * Cfg::WTM + i * 16 + pg;
              af[i][0] = ok ? ld_kmajor((const char*)sA, r, kk + tq) : 0.0;
              af[i][1] = ok ? ld_kmajor((const char*)sA, r + 8, kk + tq) : 0.0;
            }
          }
#pragma unroll
          for (int j = 0; j < Cfg::NT; j++)
            bf[j] = ok ? ld_kmajor((const char*)sB, wn * Cfg::WTN + j * 8 + pg, kk + tq) : 0.0;
#pragma unroll
          for (int i = 0; i < Cfg::MT; i++)
#pragma unroll
            for (int j = 0; j < Cfg::NT; j++) dmma_16x8x4(acc[i][j], af[i][0], af[i][1], bf[j]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      // producer: refill this stage with the chunk STAGES ahead once every warp released it
      if (threadIdx.x == 0 && (prod.valid || (dyn && !pterm))) {
        mbar_wait(&empty[pstage], pphase ^ 1);
        if (prod.valid) {
          issue_stage<BM, BN, WARPS_M, WARPS_N, A_MMAJOR, STAGES>(&tmA, &tmB, args, smem, full, pstage, prod);
          prod.next(args, units, ring);
        } else {
          mbar_arrive(&full[pstage]);
          pterm = true;
        }
        if (++pstage == STAGES) {
          pstage = 0;
          pphase ^= 1;
        }
      }
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }

    // ------------------------------ epilogue ------------------------------
    const int64_t m_base = (int64_t)tm * BM + wm * Cfg::WTM;
    const int64_t n_base = (int64_t)tn * BN + wn * Cfg::WTN;
    if (args.splitk > 1) {
      double* W = args.work + (int64_t)split * args.M * args.N;
#pragma unroll
      for (int i = 0; i < Cfg::MT; i++)
#pragma unroll
        for (int j = 0; j < Cfg::NT; j++)
#pragma unroll
          for (int e = 0; e < 4; e++) {
            const int64_t m = m_base + i * 16 + (A_MMAJOR ? g : pg) + ((e & 2) ? 8 : 0);
            const int64_t n = n_base + j * 8 + perm8(2 * tq + (e & 1));
            if (m < args.M && n < args.N) W[n * args.M + m] = acc[i][j][e];
          }
    } else {
      // one m16 row block at a time: issue its (NT x 4) C loads together, then store
#pragma unroll
      for (int i = 0; i < Cfg::MT; i++) {
        double cv[Cfg::NT][4];
        bool okv[Cfg::NT][4];
#pragma unroll
        for (int j = 0; j < Cfg::NT; j++)
#pragma unroll
          for (int e = 0; e < 4; e++) {
            const int64_t m = m_base + i * 16 + (A_MMAJOR ? g : pg) + ((e & 2) ? 8 : 0);
            const int64_t n = n_base + j * 8 + perm8(2 * tq + (e & 1));
            okv[j][e] = m < args.M && n < args.N && m >= args.m_lo;
            cv[j][e] = (okv[j][e] && args.beta != 0.0) ? __ldcg(args.C + n * args.ldc + m) : 0.0;
          }
#pragma unroll
        for (int j = 0; j < Cfg::NT; j++)
#pragma unroll
          for (int e = 0; e < 4; e++) {
            if (!okv[j][e]) continue;
            const int64_t m = m_base + i * 16 + (A_MMAJOR ? g : pg) + ((e & 2) ? 8 : 0);
            const int64_t n = n_base + j * 8 + perm8(2 * tq + (e & 1));
            double v = args.alpha * acc[i][j][e];
            if (args.beta != 0.0) v = fma(args.beta, cv[j][e], v);
            args.C[n * args.ldc + m] = v;
          }
      }
    }
  }
}

// Deterministic split-K reduction: C = alpha * sum_s W_s + beta * C (fixed s order).
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const double* __restrict__ work, int splitk, int64_t M,
                                                            int64_t N, double* C, int64_t ldc, double alpha,
                                                            double beta, int m_lo) {
  // 2-D grid (row blocks x columns): no 64-bit division per element, every slab load of a thread
  // issued before the (fixed-order) sum
  const int64_t total = M * N;
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M || m < m_lo) return;
  for (int64_t n = blockIdx.y; n < N; n += gridDim.y) {
    const double* w = work + n * M + m;
    double part[8];
    double s = 0.0;
    int k = 0;
    for (; k + 8 <= splitk; k += 8) {
#pragma unroll
      for (int q = 0; q < 8; q++) part[q] = __ldcs(w + (int64_t)(k + q) * total);
#pragma unroll
      for (int q = 0; q < 8; q++) s += part[q];
    }
    for (; k < splitk; k++) s += __ldcs(w + (int64_t)k * total);
    double* c = C + n * ldc + m;
    double v = alpha * s;
    if (beta != 0.0) v = fma(beta, *c, v);
    *c = v;
  }
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static int get_encoder() {
  static std::once_flag once;
  static int rc = RQ_OK;
  std::call_once(once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || fn == nullptr || q != cudaDriverEntryPointSuccess)
      rc = set_error(RQ_ECUDA, "cuTensorMapEncodeTiled unavailable");
    else
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return rc;
}

static int make_map(CUtensorMap* map, const GemmOperand& op, uint32_t box0, uint32_t box1, bool swizzle) {
  if (((uintptr_t)op.base & 15) != 0 || (op.ld & 1) != 0)
    return set_error(RQ_EINTERNAL, "TMA operand misaligned (base %p, ld %lld)", op.base, (long long)op.ld);
  cuuint64_t dims[2] = {(cuuint64_t)op.rows, (cuuint64_t)op.cols};
  cuuint64_t strides[1] = {(cuuint64_t)op.ld * 8};
  cuuint32_t box[2] = {box0, box1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(op.base), dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(RQ_ECUDA, "cuTensorMapEncodeTiled failed (%d): dims %llu x %llu ld %lld box %u x %u", (int)r,
                     (unsigned long long)op.rows, (unsigned long long)op.cols, (long long)op.ld, box0, box1);
  return RQ_OK;
}

int make_tensor_map_f64(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld, int box0,
                        int box1, bool swizzle) {
  RQ_TRY(get_encoder());
  GemmOperand o{base, rows, cols, ld, 0, 0};
  return make_map(map, o, (uint32_t)box0, (uint32_t)box1, swizzle);
}

static int num_sms() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = kSMs;
  }
  return sms;
}

template <int BM, int BN, int WARPS_M, int WARPS_N, bool A_MMAJOR, int STAGES>
static int launch_cfg(const GemmProblem& p, cudaStream_t stream, int64_t* launches) {
  using Cfg = GemmCfg<BM, BN, WARPS_M, WARPS_N, A_MMAJOR, STAGES>;
  auto kern = gemm_f64_kernel<BM, BN, WARPS_M, WARPS_N, A_MMAJOR, STAGES>;
  static bool attr_set = false;
  if (!attr_set) {
    RQ_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
    attr_set = true;
  }
  CUtensorMap ma, mb;
  if (A_MMAJOR)
    RQ_TRY(make_map(&ma, p.A, Cfg::A_LDM, BK, false));
  else
    RQ_TRY(make_map(&ma, p.A, BK, BM, true));
  RQ_TRY(make_map(&mb, p.B, BK, BN, true));

  KArgs a;
  // TMA faults on an odd fp64 coordinate along the contiguous dimension: shift
  // odd K origins (both operands, same parity) and odd M-major M origins down
  // by one element and mask the padding element.
  const int kshift = (int)(p.B.r0 & 1);
  if (!A_MMAJOR && (int)(p.A.r0 & 1) != kshift)
    return set_error(RQ_EINTERNAL, "gemm: K origins of A (%lld) and B (%lld) differ in parity", (long long)p.A.r0,
                     (long long)p.B.r0);
  const int mshift = A_MMAJOR ? (int)(p.A.r0 & 1) : 0;
  a.M = p.M + mshift;
  a.N = p.N;
  a.K = p.K + kshift;
  a.k_lo = kshift;
  a.m_lo = mshift;
  a.a_c0 = (int)p.A.r0 - (A_MMAJOR ? mshift : kshift);
  a.a_c1 = (int)p.A.c0 - (A_MMAJOR ? kshift : 0);
  a.b_c0 = (int)p.B.r0 - kshift;
  a.b_c1 = (int)p.B.c0;
  a.C = p.C - mshift;
  a.ldc = p.ldc;
  a.alpha = p.alpha;
  a.beta = p.beta;
  a.tiles_m = (int)ceil_div(a.M, BM);
  a.tiles_n = (int)ceil_div(a.N, BN);
  a.kchunks = ceil_div(a.K, BK);
  a.splitk = p.splitk > 1 ? p.splitk : 1;
  a.kchunks_per_split = (int)ceil_div(a.kchunks, a.splitk);
  a.splitk = (int)ceil_div(a.kchunks, a.kchunks_per_split);  // no empty splits
  a.work = p.work;
  const int64_t all_units = (int64_t)a.tiles_m * a.tiles_n * a.splitk;
  a.u0 = 0;
  a.u1 = (int)all_units;
  if (p.tile_end > 0) {  // a tile-range chunk (no split-K)
    if (a.splitk != 1) return set_error(RQ_EINTERNAL, "gemm: tile ranges need splitk == 1");
    a.u0 = (int)std::min<int64_t>(p.tile_begin, all_units);
    a.u1 = (int)std::min<int64_t>(p.tile_end, all_units);
    if (a.u1 <= a.u0) return RQ_OK;
  }
  const int64_t units = a.u1 - a.u0;
  a.sched = p.sched;
  a.sched_base = p.sched ? *p.sched_base : 0;
  static int per_sm = 0;
  if (per_sm == 0) {
    RQ_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Cfg::kThreads, Cfg::SMEM));
    if (per_sm < 1) per_sm = 1;
  }
  const int sm_cap = p.max_ctas > 0 ? std::min(num_sms(), p.max_ctas) : num_sms();
  const int64_t slots = (int64_t)sm_cap * per_sm;
  const int grid = (int)(units < slots ? units : slots);
  if (p.pdl) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(Cfg::kThreads);
    lc.dynamicSmemBytes = Cfg::SMEM;
    lc.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    cudaLaunchKernelEx(&lc, kern, ma, mb, a);
  } else {
    kern<<<grid, Cfg::kThreads, Cfg::SMEM, stream>>>(ma, mb, a);
  }
  {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      cudaFuncAttributes fa;
      cudaFuncGetAttributes(&fa, kern);
      return set_error(RQ_ECUDA, "gemm<%d,%d,%d> launch: %s (regs %d, maxThreads %d, static smem %zu, dyn %d, maxdyn %d, grid %d)",
                       BM, BN, (int)A_MMAJOR, cudaGetErrorString(e), fa.numRegs, fa.maxThreadsPerBlock,
                       fa.sharedSizeBytes, Cfg::SMEM, fa.maxDynamicSharedSizeBytes, grid);
    }
  }
  if (launches) (*launches)++;
  if (p.sched) *p.sched_base += (unsigned long long)units + (unsigned long long)grid;  // one failing fetch per CTA
  if (p.splitk_used) *p.splitk_used = a.splitk > 1 ? a.splitk : 1;
  if (a.splitk > 1) {
    if (p.mid_event) cudaEventRecord(p.mid_event, stream);
    const dim3 rgrid((unsigned)ceil_div(a.M, 256), (unsigned)std::min<int64_t>(a.N, 65535));
    splitk_reduce_kernel<<<rgrid, 256, 0, stream>>>(p.work, a.splitk, a.M, a.N, a.C, p.ldc, p.alpha, p.beta,
                                                    a.m_lo);
    RQ_CUDA_TRY(cudaGetLastError());
    if (launches) (*launches)++;
  }
  return RQ_OK;
}

size_t gemm_splitk_workspace(int64_t M, int64_t N, int splitk) {
  return splitk > 1 ? (size_t)splitk * M * N * sizeof(double) : 0;
}

// Split-K factor that best fills the machine (wave efficiency), deterministic
// reduction afterwards; only when K is long enough to amortise it.
static int choose_splitk(const GemmProblem& p, int BM, int BN) {
  if (p.splitk > 0) return p.splitk;
  if (!p.work) return 1;
  const int sms = p.max_ctas > 0 ? std::min(num_sms(), p.max_ctas) : num_sms();
  const int mshift = p.a_mmajor ? (int)(p.A.r0 & 1) : 0, kshift = (int)(p.B.r0 & 1);
  const int64_t tiles = ceil_div(p.M + mshift, BM) * ceil_div(p.N, BN);
  const int64_t kch = ceil_div(p.K + kshift, 16);
  auto eff = [&](int64_t units) {
    const int64_t waves = ceil_div(units, sms);
    return (double)units / (double)(waves * sms);
  };
  int best = 1;
  double best_eff = eff(tiles);
  if (best_eff >= 0.9 || tiles >= 8 * sms) return 1;
  for (int s = 2; s <= 32; s++) {
    if (kch / s < 8) break;
    if (gemm_splitk_workspace(p.M + 1, p.N, s) > p.work_bytes) break;
    const double e = eff(tiles * s) * (1.0 - 0.01 * s);  // mild penalty for the reduction traffic
    if (e > best_eff + 0.03) {
      best = s;
      best_eff = e;
    }
  }
  return best;
}

template <int BM, int BN, int WARPS_M, int WARPS_N, bool A_MMAJOR, int STAGES>
static int launch_auto(GemmProblem p, cudaStream_t stream, int64_t* launches) {
  // Long-K products whose tile count is a little over a whole number of waves (W = V^T A2 at
  // n2 > 9.4k: 2 x 79 tiles on 148 SMs): whole waves of unsplit tiles first, then the remaining
  // tile columns alone with split-K -- the last wave costs 1/s of a tile instead of a whole one,
  // and only the remainder's slabs go through the reduction.  RQ_GEMM_WAVES=0 restores the
  // single launch with one split factor for all tiles.
  static const int env_waves = [] {
    const char* e = getenv("RQ_GEMM_WAVES");
    return e ? atoi(e) : 1;
  }();
  if (env_waves != 0 && p.splitk == 0 && p.work && p.tile_end == 0 && !p.sched) {
    using Cfg = GemmCfg<BM, BN, WARPS_M, WARPS_N, A_MMAJOR, STAGES>;
    const int sms = p.max_ctas > 0 ? std::min(num_sms(), p.max_ctas) : num_sms();
    const int64_t slots = (int64_t)sms * (Cfg::kThreads <= 128 ? 2 : 1);
    const int mshift = A_MMAJOR ? (int)(p.A.r0 & 1) : 0, kshift = (int)(p.B.r0 & 1);
    const int64_t tiles_m = ceil_div(p.M + mshift, BM), tiles_n = ceil_div(p.N, BN);
    const int64_t tiles = tiles_m * tiles_n, kch = ceil_div(p.K + kshift, BK);
    const int64_t whole_cols = (tiles / slots) * slots / tiles_m;  // tile columns in whole waves
    const double eff = (double)tiles / (double)(ceil_div(tiles, slots) * slots);
    if (tiles > slots && tiles < 8 * slots && eff < 0.93 && kch >= 128 && whole_cols > 0 && whole_cols < tiles_n) {
      GemmProblem p1 = p;
      p1.N = whole_cols * BN;
      p1.splitk = 1;
      p1.mid_event = nullptr;
      p1.splitk_used = nullptr;
      RQ_TRY((launch_cfg<BM, BN, WARPS_M, WARPS_N, A_MMAJOR, STAGES>(p1, stream, launches)));
      GemmProblem p2 = p;
      p2.N = p.N - p1.N;
      p2.B.c0 += p1.N;
      p2.C += p1.N * p.ldc;
      p2.splitk = choose_splitk(p2, BM, BN);
      return launch_cfg<BM, BN, WARPS_M, WARPS_N, A_MMAJOR, STAGES>(p2, stream, launches);
    }
  }
  p.splitk = choose_splitk(p, BM, BN);
  return launch_cfg<BM, BN, WARPS_M, WARPS_N, A_MMAJOR, STAGES>(p, stream, launches);
}

// Output tiles of the configuration gemm_f64 picks for p (for tile-range chunks).
int64_t gemm_f64_tiles(const GemmProblem& p) {
  int bm = 128, bn = 128;
  const bool m144 = (p.M > 128 && p.M <= 144) || (p.M > 256 && p.M <= 288);
  const char* e = getenv("RQ_GEMM_BIG");
  if (e && atoi(e) == 1 && p.M >= 128 && p.N >= 128 && (p.a_mmajor || !m144)) {
    bn = 64;
  } else if (p.a_mmajor) {
    if (p.M >= 128 && p.N >= 128) bn = 128;
    else if (p.N < 128) bn = 32;
    else bm = 64;
  } else {
    if (m144 && p.N >= 128) bm = 144;
    else if (p.M >= 128 && p.N >= 128) bn = 128;
    else if (p.N < 128) bn = 32;
    else bm = 64;
  }
  const int mshift = p.a_mmajor ? (int)(p.A.r0 & 1) : 0;
  return ceil_div(p.M + mshift, bm) * ceil_div(p.N, bn);
}

int gemm_f64(const GemmProblem& p, cudaStream_t stream, int64_t* launches) {
  if (p.M <= 0 || p.N <= 0) return RQ_OK;
  if (p.K <= 0) {
    // C = beta * C
    if (p.beta == 1.0) return RQ_OK;
    return set_error(RQ_EINTERNAL, "gemm_f64: K == 0 with beta != 1 not supported");
  }
  RQ_TRY(get_encoder());
  if (p.splitk > 1 && p.work == nullptr) return set_error(RQ_EINTERNAL, "gemm_f64: split-K without workspace");
  // Tile selection: skinny outputs use narrower tiles so the grid fills 148 SMs;
  // M in (128, 144] or (256, 288] (the b+p sketch rows) uses 144-row tiles.
  const bool m144 = (p.M > 128 && p.M <= 144) || (p.M > 256 && p.M <= 288);
  static int big = -1;  // RQ_GEMM_BIG=1: 128x64 tiles, 2 CTAs/SM, for large outputs (tuning switch)
  if (big < 0) {
    const char* e = getenv("RQ_GEMM_BIG");
    big = e ? atoi(e) : 0;
  }
  if (big == 1 && p.M >= 128 && p.N >= 128) {
    if (p.a_mmajor) return launch_auto<128, 64, 2, 2, true, 4>(p, stream, launches);
    if (!m144) return launch_auto<128, 64, 2, 2, false, 4>(p, stream, launches);
  }
  if (p.a_mmajor) {
    if (p.M >= 128 && p.N >= 128) return launch_auto<128, 128, 2, 4, true, 4>(p, stream, launches);
    if (p.N < 128) return launch_auto<128, 32, 4, 2, true, 6>(p, stream, launches);
    return launch_auto<64, 128, 2, 4, true, 5>(p, stream, launches);
  } else {
    if (m144 && p.N >= 128) return launch_auto<144, 128, 3, 4, false, 4>(p, stream, launches);
    if (p.M >= 128 && p.N >= 128) return launch_auto<128, 128, 2, 4, false, 4>(p, stream, launches);
    if (p.N < 128) return launch_auto<128, 32, 4, 2, false, 6>(p, stream, launches);
    return launch_auto<64, 128, 2, 4, false, 5>(p, stream, launches);
  }
}

}  // namespace rq
