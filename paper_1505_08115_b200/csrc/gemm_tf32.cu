// FP32 GEMM on the 5th-generation tensor cores for sm_100a: 3xTF32 split products on
// tcgen05.mma (kind::tf32), operands staged by TMA, the accumulator in TMEM.
//
//   C[M x N] = alpha * op(A) * B + beta * C        (fp32, column-major)
//     op(A) = A^T, A stored K x M (a_mmajor = false, "TN")  /  op(A) = A, A stored M x K ("NN")
//     B stored K x N (K contiguous)
//
// TF32 keeps 10 mantissa bits, so one TF32 product cannot meet the fp32 path's 1e-5 bar.  Every
// operand x is split as hi = tf32(x) and lo = tf32(x - hi) (round to nearest; both exact in TF32,
// |x - hi - lo| <= 2^-23 |x|), and each k-block issues
// A_hi B_hi + A_hi B_lo + A_lo B_hi into one FP32 TMEM accumulator (the lo x lo term is below
// fp32 rounding).  Persistent CTAs (<= one per SM, optionally capped) walk their 128 x 128 output
// tiles as one stream of (tile, k-block) steps, BK = 32; roles per CTA:
//   warp 0      TMA producer: raw fp32 tiles of A and B into a 2-deep ring (mbarrier complete_tx)
//   warps 2-9   converters: raw -> hi / lo tiles in the canonical K-major SWIZZLE_128B layout
//               (an M-major A is transposed here), zeroing k outside the view; then the epilogue
//   warp 1      TMEM allocation and the single-thread tcgen05.mma issue, tcgen05.commit frees a
//               converted stage / signals the epilogue
// Accumulation: each k-block's 12 MMAs go to one of two TMEM accumulators (k-block parity); the
// converter warps drain it with tcgen05.ld 32x32b (warp w reads TMEM lanes 32 (w % 4) ..) into fp32
// registers while the tensor core fills the other.  Epilogue: alpha / beta, coalesced column
// stores (lanes = consecutive rows).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "gemm_tf32.cuh"

namespace rq {

namespace {

constexpr int TBM = 128, TBN = 128;
constexpr int kRawTile = 16384;           // one raw operand tile: 128 rows x 128 B (TMA box)
constexpr int kRawStages = 3, kConvStages = 2;
constexpr int kThreads = 320;             // warps 0 (TMA), 1 (MMA), 2-9 (convert + drain + epilogue)
constexpr int kConvThreads = 256;
constexpr int kHalf = TBN / 2;            // accumulator columns per converter thread

// Per input type: k-block depth (one 128-byte TMA row of the raw operand), and the converted
// tf32 tiles' K-major swizzle (rows of BK tf32: 128 B -> SWIZZLE_128B, 64 B -> SWIZZLE_64B).
template <typename T>
struct TfCfg;
template <>
struct TfCfg<float> {
  static constexpr int BK = 32, ROWB = 128, LAYOUT = 2, SBO = 1024;
};
template <>
struct TfCfg<double> {
  static constexpr int BK = 16, ROWB = 64, LAYOUT = 4, SBO = 512;
};
template <typename T>
constexpr int conv_tile() { return TBM * TfCfg<T>::BK * 4; }
template <typename T>
constexpr int smem_bytes() { return kRawStages * 2 * kRawTile + kConvStages * 4 * conv_tile<T>() + 1024 + 256; }
static_assert(smem_bytes<float>() <= 232448 && smem_bytes<double>() <= 232448, "shared memory per CTA");

struct TArgs {
  int M, N, Kv;        // output extent (M includes m_lo padding rows), valid k range [k_lo, Kv)
  int k_lo, m_lo;
  int a_c0, a_c1, b_c0, b_c1;
  void* C;             // fp32 or fp64 (the input type)
  int64_t ldc;
  float alpha, beta;
  int tiles_m, tiles;
  int kblocks;  // k-blocks per unit (a split's range; the last split's tail reads zeros)
  int splits;   // units = tiles * splits; > 1: partial sums into work slabs, then a reduce
  float* work;  // splits x (M x N), ld = M
  int u0;       // first unit (a tile-range chunk of a larger GEMM: tiles u0 .. u0 + tiles - 1)
  int four;     // 1: also A_lo B_lo (4 products; tuning / accuracy probe)
};

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(b)), "r"(n));
}
__device__ __forceinline__ void bar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
          s_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          s_u32(dst)),
      "l"(m), "r"(s_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// K-major swizzled shared-memory matrix descriptor (sm100, version 1): SWIZZLE_128B (layout type 2,
// 128-byte rows, 8-row atoms 1024 B apart) or SWIZZLE_64B (type 4, 64-byte rows, atoms 512 B apart)
template <int LAYOUT, int SBO>
__device__ __forceinline__ uint64_t sw_desc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(SBO >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)LAYOUT << 61);
}
// kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = 128
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TBN >> 3) << 17) |
                            ((uint32_t)(TBM >> 4) << 24);

__device__ __forceinline__ void umma_tf32(uint32_t tmem, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
      "l"(da), "l"(db), "r"(kIdesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s_u32(bar))
               : "memory");
}

// byte offset of tf32 element (row r, k) in a 128-row K-major swizzled tile: 16-byte chunk c of
// row r sits at chunk c ^ (r & 7) (128-byte rows) or c ^ ((r >> 1) & 3) (64-byte rows)
template <int ROWB>
__device__ __forceinline__ int sw_off(int r, int k) {
  if constexpr (ROWB == 128)
    return (r >> 3) * 1024 + (r & 7) * 128 + ((((k >> 2) ^ (r & 7))) << 4) + ((k & 3) << 2);
  else
    return (r >> 3) * 512 + (r & 7) * 64 + ((((k >> 2) ^ ((r >> 1) & 3))) << 4) + ((k & 3) << 2);
}

// hi = x rounded to TF32 (nearest, ties away), lo = (x - hi) rounded to TF32: both exactly
// representable, so the tensor core's TF32 read loses nothing; |x - hi - lo| <= 2^-23 |x|
__device__ __forceinline__ void split_tf32(double xd, float& hi, float& lo) {
  const float x = (float)xd;  // fp32-level accuracy: the fp64 input rounded once
  uint32_t h, l;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  const float r = x - __uint_as_float(h);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(r));
  hi = __uint_as_float(h);
  lo = __uint_as_float(l);
}
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  uint32_t h, l;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  const float r = x - __uint_as_float(h);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(r));
  hi = __uint_as_float(h);
  lo = __uint_as_float(l);
}

template <typename T, bool A_MMAJOR>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, const TArgs a) {
  using Cfg = TfCfg<T>;
  constexpr int BK = Cfg::BK;
  constexpr int kConv = conv_tile<T>();
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* raw = sm;                                   // [stage][A, B] 16 KB each
  unsigned char* conv = sm + kRawStages * 2 * kRawTile;      // [stage][Ahi, Alo, Bhi, Blo]
  uint64_t* bars = (uint64_t*)(conv + kConvStages * 4 * kConv);
  uint64_t* raw_full = bars;        // [kRawStages]
  uint64_t* raw_empty = bars + 4;   // [kRawStages]
  uint64_t* conv_full = bars + 8;   // [2]
  uint64_t* conv_empty = bars + 10;
  uint64_t* acc_full = bars + 12;   // [2]: a k-block's products landed in TMEM accumulator (g & 1)
  uint64_t* acc_empty = bars + 14;  // [2]: the converter warps drained it into registers
  uint32_t* tmem_slot = (uint32_t*)(bars + 16);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // persistent: this CTA's units blockIdx.x, blockIdx.x + gridDim.x, ... (unit = tile x split);
  // one stream of (unit, k-block) steps g = j * kblocks + kb through every pipeline
  const int units = a.tiles * a.splits;  // (relative to u0)
  const int my_units = units > (int)blockIdx.x ? (units - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  const int G = my_units * a.kblocks;
  auto unit_of = [&](int g) { return a.u0 + (int)blockIdx.x + (g / a.kblocks) * (int)gridDim.x; };
  auto tile_of = [&](int g) { return unit_of(g) / a.splits; };
  auto kb_of = [&](int g) { return (unit_of(g) % a.splits) * a.kblocks + g % a.kblocks; };  // global k-block

  if (threadIdx.x == 0) {
    for (int s = 0; s < kRawStages; s++) {
      bar_init(&raw_full[s], 1);
      bar_init(&raw_empty[s], kConvThreads);
    }
    for (int s = 0; s < 2; s++) {
      bar_init(&conv_full[s], kConvThreads);
      bar_init(&conv_empty[s], 1);
      bar_init(&acc_full[s], 1);
      bar_init(&acc_empty[s], kConvThreads);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&ma) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mb) : "memory");
  }
  if (warp == 1) {  // 256 TMEM columns: two 128 x 128 fp32 accumulators (step parity)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(s_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      for (int g = 0; g < G; g++) {
        const int t = tile_of(g), kb = kb_of(g);
        const int tm = t % a.tiles_m, tn = t / a.tiles_m;
        const int s = g % kRawStages;
        bar_wait(&raw_empty[s], ((g / kRawStages) & 1) ^ 1);
        bar_expect_tx(&raw_full[s], 2 * kRawTile);
        unsigned char* ra = raw + (s * 2) * kRawTile;
        unsigned char* rb = raw + (s * 2 + 1) * kRawTile;
        if (A_MMAJOR)
          tma2d(ra, &ma, &raw_full[s], a.a_c0 + tm * TBM, a.a_c1 + kb * BK);
        else
          tma2d(ra, &ma, &raw_full[s], a.a_c0 + kb * BK, a.a_c1 + tm * TBM);
        tma2d(rb, &mb, &raw_full[s], a.b_c0 + kb * BK, a.b_c1 + tn * TBN);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread) ----------------
    // Each step accumulates into its own (parity) TMEM accumulator, which the converter warps
    // add into fp32 registers: the tensor core's accumulation then spans 32 k only (its long
    // in-TMEM sums measured ~6x less accurate than an fp32 SGEMM, tools/gemm_acc.py).
    if (lane == 0) {
      for (int g = 0; g < G; g++) {
        const int s = g & 1;
        bar_wait(&conv_full[s], (g >> 1) & 1);
        bar_wait(&acc_empty[s], ((g >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t base = s_u32(conv + (s * 4) * kConv);
        const uint32_t ahi = base, alo = base + kConv, bhi = base + 2 * kConv, blo = base + 3 * kConv;
        const uint32_t acc = tmem + (uint32_t)(s * TBN);
        constexpr int L = Cfg::LAYOUT, SB = Cfg::SBO;
#pragma unroll
        for (int kk = 0; kk < BK / 8; kk++) {  // 8 tf32 (32 B) per MMA along K
          const uint32_t o = kk * 32;
          umma_tf32(acc, sw_desc<L, SB>(ahi + o), sw_desc<L, SB>(bhi + o), kk != 0);
          umma_tf32(acc, sw_desc<L, SB>(ahi + o), sw_desc<L, SB>(blo + o), 1u);
          umma_tf32(acc, sw_desc<L, SB>(alo + o), sw_desc<L, SB>(bhi + o), 1u);
          if (a.four) umma_tf32(acc, sw_desc<L, SB>(alo + o), sw_desc<L, SB>(blo + o), 1u);
        }
        umma_commit(&conv_empty[s]);  // the stage's smem is free once these MMAs completed
        umma_commit(&acc_full[s]);
      }
    }
  } else {
    // ---------------- converters, drains and epilogues ----------------
    const int c = threadIdx.x - 64;
    const int q = warp & 3;            // TMEM lanes 32q .. 32q + 31 = output rows of this thread's warp
    const int h0 = ((warp - 2) >> 2) * kHalf;  // this thread's accumulator columns h0 .. h0 + 63
    float accr[kHalf];
#pragma unroll
    for (int j = 0; j < kHalf; j++) accr[j] = 0.0f;
    // add step gd's TMEM accumulator (parity gd & 1) into accr and release it
    auto drain = [&](int gd) {
      const int s = gd & 1;
      bar_wait(&acc_full[s], (gd >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int cb = 0; cb < kHalf / 32; cb++) {
        uint32_t r[32];
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(s * TBN + h0 + cb * 32);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
            "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
              "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
              "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; j++) accr[cb * 32 + j] += __uint_as_float(r[j]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      bar_arrive(&acc_empty[s]);
    };
    // registers -> C, or the unit's split-K slab (fp32, ld = M), for unit u (the tensor core
    // already works on the next unit)
    auto epilogue = [&](int u) {
      const int t = u / a.splits, sp = u % a.splits;
      const int tm = t % a.tiles_m, tn = t / a.tiles_m;
      const int m = tm * TBM + q * 32 + lane;
      const int nv = min(kHalf, a.N - tn * TBN - h0);
      if (a.splits > 1) {
        if (m < a.M) {
          float* w = a.work + (int64_t)sp * a.M * a.N + (int64_t)(tn * TBN + h0) * a.M + m;
#pragma unroll
          for (int j = 0; j < kHalf; j++)
            if (j < nv) __stcg(w + (int64_t)j * a.M, accr[j]);
        }
      } else if (m >= a.m_lo && m < a.M) {
        T* cbase = static_cast<T*>(a.C) + (int64_t)(tn * TBN + h0) * a.ldc + m;
#pragma unroll
        for (int gq = 0; gq < kHalf / 8; gq++) {
          // 8 independent loads of C first (the stores below could alias them), then 8 stores
          T cv[8];
          if (a.beta != 0.0f) {
#pragma unroll
            for (int j = 0; j < 8; j++)
              cv[j] = (gq * 8 + j < nv) ? __ldcs(cbase + (int64_t)(gq * 8 + j) * a.ldc) : T(0);
          }
#pragma unroll
          for (int j = 0; j < 8; j++) {
            if (gq * 8 + j < nv) {
              T v = (T)a.alpha * (T)accr[gq * 8 + j];
              if (a.beta != 0.0f) v = fma((T)a.beta, cv[j], v);
              __stcs(cbase + (int64_t)(gq * 8 + j) * a.ldc, v);
            }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < kHalf; j++) accr[j] = 0.0f;
    };
    for (int g = 0; g < G; g++) {
      const int s = g & 1, rs = g % kRawStages;
      const uint32_t ph = (g >> 1) & 1;
      bar_wait(&raw_full[rs], (g / kRawStages) & 1);
      bar_wait(&conv_empty[s], ph ^ 1);
      const unsigned char* ra = raw + (rs * 2) * kRawTile;
      const unsigned char* rb = raw + (rs * 2 + 1) * kRawTile;
      unsigned char* ahi = conv + (s * 4) * kConv;
      unsigned char* alo = ahi + kConv;
      unsigned char* bhi = ahi + 2 * kConv;
      unsigned char* blo = ahi + 3 * kConv;
      const int kbase = kb_of(g) * BK;
      // K-major raw tiles (B, and A when it is K-major) were written by TMA with SWIZZLE_128B:
      // 16-byte vector v holds row r = v / 8, chunk (v % 8) ^ (r % 8) of the 128-byte row
#pragma unroll
      for (int t = 0; t < 1024 / kConvThreads; t++) {
        const int v = c + kConvThreads * t;  // 16-byte vector index 0..1023
        const int r = v >> 3;
        const int ch = (v & 7) ^ (r & 7);
        if constexpr (sizeof(T) == 4) {
          const int k0 = ch << 2;
#pragma unroll
          for (int opnd = 0; opnd < (A_MMAJOR ? 1 : 2); opnd++) {
            const unsigned char* src = opnd == 0 ? rb : ra;
            unsigned char* dh = opnd == 0 ? bhi : ahi;
            unsigned char* dl = opnd == 0 ? blo : alo;
            const float4 x = *reinterpret_cast<const float4*>(src + v * 16);
            const float xs[4] = {x.x, x.y, x.z, x.w};
            float h[4], l[4];
#pragma unroll
            for (int e = 0; e < 4; e++) {
              const int kg = kbase + k0 + e;
              split_tf32((kg >= a.k_lo && kg < a.Kv) ? xs[e] : 0.0f, h[e], l[e]);
            }
            *reinterpret_cast<float4*>(dh + v * 16) = make_float4(h[0], h[1], h[2], h[3]);
            *reinterpret_cast<float4*>(dl + v * 16) = make_float4(l[0], l[1], l[2], l[3]);
          }
        } else {
          const int k0 = ch << 1;  // two doubles -> two tf32 of a 64-byte converted row
          const int off = sw_off<Cfg::ROWB>(r, k0);
#pragma unroll
          for (int opnd = 0; opnd < (A_MMAJOR ? 1 : 2); opnd++) {
            const unsigned char* src = opnd == 0 ? rb : ra;
            unsigned char* dh = opnd == 0 ? bhi : ahi;
            unsigned char* dl = opnd == 0 ? blo : alo;
            const double2 x = *reinterpret_cast<const double2*>(src + v * 16);
            float h0, l0, h1, l1;
            const int kg = kbase + k0;
            split_tf32((kg >= a.k_lo && kg < a.Kv) ? x.x : 0.0, h0, l0);
            split_tf32((kg + 1 >= a.k_lo && kg + 1 < a.Kv) ? x.y : 0.0, h1, l1);
            *reinterpret_cast<float2*>(dh + off) = make_float2(h0, h1);
            *reinterpret_cast<float2*>(dl + off) = make_float2(l0, l1);
          }
        }
      }
      if (A_MMAJOR) {
        // raw A: BK k-rows of 128 contiguous m (no swizzle) -> K-major swizzled hi / lo.  Each
        // thread builds one 16-byte target chunk (row r, k = 4 kc .. 4 kc + 3): lanes take
        // consecutive rows, so the reads are consecutive words and the 16-byte stores of a
        // quarter-warp land in distinct swizzled chunks
#pragma unroll
        for (int t = 0; t < (TBM * BK / 4) / kConvThreads; t++) {
          const int v = c + kConvThreads * t;
          const int r = v & (TBM - 1), kc = v >> 7;
          const T* src = reinterpret_cast<const T*>(ra) + (kc * 4) * TBM + r;
          float h[4], l[4];
#pragma unroll
          for (int e = 0; e < 4; e++) {
            const int kg = kbase + kc * 4 + e;
            split_tf32((kg >= a.k_lo && kg < a.Kv) ? src[e * TBM] : T(0), h[e], l[e]);
          }
          const int off = sw_off<Cfg::ROWB>(r, kc * 4);
          *reinterpret_cast<float4*>(ahi + off) = make_float4(h[0], h[1], h[2], h[3]);
          *reinterpret_cast<float4*>(alo + off) = make_float4(l[0], l[1], l[2], l[3]);
        }
      }
      // generic-proxy smem writes -> the tensor core's async proxy
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bar_arrive(&raw_empty[rs]);
      bar_arrive(&conv_full[s]);
      if (g > 0) {  // (the tensor core works on step g meanwhile)
        drain(g - 1);
        if ((g - 1) % a.kblocks == a.kblocks - 1) epilogue(unit_of(g - 1));
      }
    }
    if (G > 0) {
      drain(G - 1);
      epilogue(unit_of(G - 1));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
  }
}

// Deterministic split-K reduction: C = alpha * sum_s work_s + beta * C (fixed s order).
template <typename T>
__global__ void splitk_reduce_tf_kernel(const float* __restrict__ work, int splits, int M, int N, T* C, int64_t ldc,
                                        float alpha, float beta, int m_lo) {
  const int64_t total = (int64_t)M * N;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(idx % M), n = (int)(idx / M);
    if (m < m_lo) continue;
    float s = 0.0f;
    for (int k = 0; k < splits; k++) s += __ldcg(work + k * total + idx);
    T* c = C + (int64_t)n * ldc + m;
    T v = (T)alpha * (T)s;
    if (beta != 0.0f) v = fma((T)beta, *c, v);
    *c = v;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 g_enc32 = nullptr;

int encoder() {
  static std::once_flag once;
  static int rc = RQ_OK;
  std::call_once(once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || fn == nullptr || q != cudaDriverEntryPointSuccess)
      rc = set_error(RQ_ECUDA, "cuTensorMapEncodeTiled unavailable");
    else
      g_enc32 = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return rc;
}

// Input-type-independent description of one product (pointers of the input type).
struct TfProblem {
  int64_t M, N, K;
  const void* a_base;
  int64_t a_rows, a_cols, a_ld, a_r0, a_c0;
  bool a_mmajor;
  const void* b_base;
  int64_t b_rows, b_cols, b_ld, b_r0, b_c0;
  void* C;
  int64_t ldc;
  double alpha, beta;
  int max_ctas;
  float* work;
  size_t work_bytes;
  int64_t tile_begin, tile_end;  // tile_end > 0: only output tiles [tile_begin, tile_end), no split-K
  bool pdl;
};

template <typename T>
int map_t(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld, uint32_t box0, uint32_t box1,
          bool swizzle) {
  constexpr int per16 = 16 / (int)sizeof(T);
  if (((uintptr_t)base & 15) != 0 || (ld % per16) != 0)
    return set_error(RQ_EVALUE, "tf32 GEMM operand needs a 16-byte aligned base and 16-byte strides (ld %lld)",
                     (long long)ld);
  cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(T)};
  cuuint32_t box[2] = {box0, box1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_enc32(map, sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                       const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(RQ_ECUDA, "cuTensorMapEncodeTiled (tf32 GEMM) failed (%d): %llu x %llu ld %lld", (int)r,
                     (unsigned long long)rows, (unsigned long long)cols, (long long)ld);
  return RQ_OK;
}

int num_sms32() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = kSMs;
  }
  return sms;
}

template <typename T, bool A_MMAJOR>
int launch(const TfProblem& p, cudaStream_t st, int64_t* launches) {
  using Cfg = TfCfg<T>;
  constexpr int BK = Cfg::BK;
  constexpr int per16 = 16 / (int)sizeof(T);
  auto kern = gemm_tf32x3_kernel<T, A_MMAJOR>;
  static bool attr = false;
  if (!attr) {
    RQ_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<T>()));
    attr = true;
  }
  // TMA origins along a contiguous dimension are rounded down to 16 bytes; the converters zero
  // the padding k's, the epilogue skips the padding rows.
  const int kshift = (int)(p.b_r0 % per16);
  if (!A_MMAJOR && (int)(p.a_r0 % per16) != kshift)
    return set_error(RQ_EINTERNAL, "tf32 gemm: K origins of A (%lld) and B (%lld) differ modulo 16 bytes",
                     (long long)p.a_r0, (long long)p.b_r0);
  const int ashift = A_MMAJOR ? (int)(p.a_r0 % per16) : 0;  // M-major A: pad rows of the output
  CUtensorMap ma, mb;
  if (A_MMAJOR)
    RQ_TRY(map_t<T>(&ma, p.a_base, p.a_rows, p.a_cols, p.a_ld, TBM, BK, false));
  else
    RQ_TRY(map_t<T>(&ma, p.a_base, p.a_rows, p.a_cols, p.a_ld, BK, TBM, true));
  RQ_TRY(map_t<T>(&mb, p.b_base, p.b_rows, p.b_cols, p.b_ld, BK, TBN, true));
  TArgs a;
  a.M = (int)(p.M + ashift);
  a.N = (int)p.N;
  a.k_lo = kshift;
  a.Kv = (int)(p.K + kshift);
  a.m_lo = ashift;
  if (A_MMAJOR) {
    a.a_c0 = (int)(p.a_r0 - ashift);
    a.a_c1 = (int)(p.a_c0 - kshift);  // the k coordinate is the outer dimension: shifted with B's k
  } else {
    a.a_c0 = (int)(p.a_r0 - kshift);
    a.a_c1 = (int)p.a_c0;
  }
  a.b_c0 = (int)(p.b_r0 - kshift);
  a.b_c1 = (int)p.b_c0;
  a.C = static_cast<T*>(p.C) - ashift;
  a.ldc = p.ldc;
  a.alpha = (float)p.alpha;
  a.beta = (float)p.beta;
  a.tiles_m = (int)ceil_div(a.M, TBM);
  const int tiles_n = (int)ceil_div(a.N, TBN);
  const int kb_total = (int)ceil_div(a.Kv, BK);
  static const int env_four = getenv("RQ_TF32X4") ? atoi(getenv("RQ_TF32X4")) : 0;
  a.four = env_four;
  int64_t tiles = (int64_t)a.tiles_m * tiles_n;
  if (tiles > 0x7fffffff) return set_error(RQ_EUNSUPPORTED, "tf32 gemm: too many tiles");
  a.u0 = 0;
  if (p.tile_end > 0) {  // a tile-range chunk of a larger product
    const int64_t t1 = std::min<int64_t>(p.tile_end, tiles);
    a.u0 = (int)std::min<int64_t>(p.tile_begin, t1);
    tiles = t1 - a.u0;
    if (tiles <= 0) return RQ_OK;
  }
  a.tiles = (int)tiles;
  const int sms = num_sms32();
  const int cap = p.max_ctas > 0 ? std::min(p.max_ctas, sms) : sms;  // persistent: <= one CTA per SM
  // split-K when the tiles fill the grid poorly (wave efficiency), K is long enough and the
  // context's workspace holds the slabs
  auto eff = [&](int64_t u) { return (double)u / (double)(ceil_div(u, cap) * cap); };
  int splits = 1;
  double best = eff(tiles);
  if (p.work && p.tile_end <= 0 && best < 0.9 && tiles < 4 * cap) {
    for (int sp = 2; sp <= 16; sp++) {
      if (kb_total / sp < 4) break;
      if ((size_t)sp * a.M * a.N * sizeof(float) > p.work_bytes) break;
      const double e = eff(tiles * sp) * (1.0 - 0.02 * sp);
      if (e > best + 0.03) {
        best = e;
        splits = sp;
      }
    }
  }
  a.splits = splits;
  a.kblocks = (int)ceil_div(kb_total, splits);
  a.work = p.work;
  const int grid = (int)std::min<int64_t>(tiles * splits, cap);
  if (p.pdl) {
    // programmatic dependent launch behind the previous kernel of the stream (the look-ahead's
    // chunks beside a leaf cluster): reads none of that kernel's outputs
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(kThreads);
    lc.dynamicSmemBytes = smem_bytes<T>();
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    RQ_CUDA_TRY(cudaLaunchKernelEx(&lc, kern, ma, mb, a));
  } else {
    kern<<<grid, kThreads, smem_bytes<T>(), st>>>(ma, mb, a);
    RQ_CUDA_TRY(cudaGetLastError());
  }
  if (launches) (*launches)++;
  if (splits > 1) {
    const int64_t total = (int64_t)a.M * a.N;
    const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 4 * sms);
    splitk_reduce_tf_kernel<T><<<blocks, 256, 0, st>>>(a.work, splits, a.M, a.N, static_cast<T*>(a.C), a.ldc,
                                                        a.alpha, a.beta, a.m_lo);
    RQ_CUDA_TRY(cudaGetLastError());
    if (launches) (*launches)++;
  }
  return RQ_OK;
}

}  // namespace

int gemm_tf32x3(const GemmProblemF32& p, cudaStream_t st, int64_t* launches) {
  if (p.M <= 0 || p.N <= 0) return RQ_OK;
  if (p.K <= 0) {
    if (p.beta == 1.0) return RQ_OK;
    return set_error(RQ_EINTERNAL, "fp32 gemm: K == 0 with beta != 1 not supported");
  }
  RQ_TRY(encoder());
  TfProblem q{p.M, p.N, p.K, p.A.base, p.A.rows, p.A.cols, p.A.ld, p.A.r0, p.A.c0, p.a_mmajor, p.B.base, p.B.rows,
              p.B.cols, p.B.ld, p.B.r0, p.B.c0, p.C, p.ldc, p.alpha, p.beta, p.max_ctas, p.work, p.work_bytes, 0, 0,
              false};
  return p.a_mmajor ? launch<float, true>(q, st, launches) : launch<float, false>(q, st, launches);
}

int gemm_tf32x3_f64(const GemmProblem& p, cudaStream_t st, int64_t* launches) {
  if (p.M <= 0 || p.N <= 0) return RQ_OK;
  if (p.K <= 0) {
    if (p.beta == 1.0) return RQ_OK;
    return set_error(RQ_EINTERNAL, "tf32 gemm (fp64 operands): K == 0 with beta != 1 not supported");
  }
  RQ_TRY(encoder());
  TfProblem q{p.M, p.N, p.K, p.A.base, p.A.rows, p.A.cols, p.A.ld, p.A.r0, p.A.c0, p.a_mmajor, p.B.base, p.B.rows,
              p.B.cols, p.B.ld, p.B.r0, p.B.c0, p.C, p.ldc, p.alpha, p.beta, p.max_ctas,
              reinterpret_cast<float*>(p.work), p.work ? p.work_bytes : 0, p.tile_begin, p.tile_end, p.pdl};
  return p.a_mmajor ? launch<double, true>(q, st, launches) : launch<double, false>(q, st, launches);
}

int64_t gemm_tf32x3_tiles(int64_t M, int64_t N, bool a_mmajor, int64_t a_r0) {
  const int64_t ashift = a_mmajor ? (a_r0 & 1) : 0;
  return ceil_div(M + ashift, TBM) * ceil_div(N, TBN);
}

}  // namespace rq
