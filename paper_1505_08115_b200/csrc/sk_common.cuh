// Device helpers shared by the sketch CPQR kernels (sweep.cu, sketch_batch.cu).
#pragma once
#include "common.cuh"

namespace rq {

// Winner among 32 lanes: max key, then min position.  Returns the lane, or -1.
RQ_DEV int warp_argmax(unsigned hi, unsigned lo, int pos, bool valid) {
  const unsigned all = 0xffffffffu;
  const unsigned h = __reduce_max_sync(all, valid ? hi : 0u);
  const bool c1 = valid && hi == h;
  const unsigned l = __reduce_max_sync(all, c1 ? lo : 0u);
  const bool c2 = c1 && lo == l;
  const int pm = (int)__reduce_min_sync(all, c2 ? (unsigned)pos : 0xffffffffu);
  const unsigned ball = __ballot_sync(all, c2 && pos == pm);
  return ball ? __ffs(ball) - 1 : -1;
}

// LL words: 32-bit payload (high half) + 32-bit step stamp (low half), stored and loaded
// as 16-byte pairs; each 8-byte word is single-copy atomic, so a stamp match is a data match.
RQ_DEV unsigned long long ll_word(unsigned data, unsigned stamp) {
  return ((unsigned long long)data << 32) | stamp;
}
RQ_DEV void st_ll2(unsigned long long* p, unsigned long long a, unsigned long long b) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
RQ_DEV void ld_ll2(const unsigned long long* p, unsigned long long& a, unsigned long long& b) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

// Warp sums of P values at once (P a power of two <= 16): a reduce-scatter butterfly (each
// round a lane sends the half of its values its xor-partner keeps, so P - 1 shuffles instead of
// 5 P over the first log2 P rounds, one value per round after that), then every lane reads each
// total from the lane that owns it.  Every lane ends with the same bits of every sum.
template <int P, int OFF, int N>
RQ_DEV void warp_sum_pow2(double (&v)[N], int lane) {
  constexpr int LOGP = P >= 16 ? 4 : P >= 8 ? 3 : P >= 4 ? 2 : P >= 2 ? 1 : 0;
  double w[P];
#pragma unroll
  for (int i = 0; i < P; i++) w[i] = v[OFF + i];
#pragma unroll
  for (int r = 0; r < 5; r++) {
    const int o = 16 >> r;
    const int c = P >> r;  // values still held (0 or 1: the plain butterfly)
    if (c >= 2) {
      const int h = c / 2;
      const bool hi = (lane & o) != 0;
#pragma unroll
      for (int i = 0; i < h; i++) {
        const double send = hi ? w[i] : w[i + h];
        const double keep = hi ? w[i + h] : w[i];
        w[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    } else {
      w[0] += __shfl_xor_sync(0xffffffffu, w[0], o);
    }
  }
  if constexpr (P == 1) {
    v[OFF] = w[0];
  } else {
#pragma unroll
    for (int q = 0; q < P; q++) {
      int src = 0;
#pragma unroll
      for (int r = 0; r < LOGP; r++) src |= ((q >> (LOGP - 1 - r)) & 1) << (4 - r);
      v[OFF + q] = __shfl_sync(0xffffffffu, w[0], src);
    }
  }
}

// Warp sums of v[OFF..OFF+C), split into power-of-two groups (C = 9: 8 + 1).
template <int C, int OFF, int N>
RQ_DEV void warp_sum_all(double (&v)[N], int lane) {
  if constexpr (C > 0) {
    constexpr int P = C >= 16 ? 16 : C >= 8 ? 8 : C >= 4 ? 4 : C >= 2 ? 2 : 1;
    warp_sum_pow2<P, OFF, N>(v, lane);
    warp_sum_all<C - P, OFF + P, N>(v, lane);
  }
}

}  // namespace rq
