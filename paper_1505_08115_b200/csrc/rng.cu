// K1: counter-based Gaussian stream (splitmix64 + Box-Muller cosine branch).
// Restates rng.py:15-68 of the reference: draw k of seed s uses words 2k and
// 2k+1, word i = mix(s + (i+1) * gamma); u1 = ((r1 >> 11) + 1) 2^-53 in (0, 1],
// u2 = (r2 >> 11) 2^-53 in [0, 1); z = sqrt(-2 ln u1) cos(2 pi u2).
// The integer stream is bit-exact; the normals agree with numpy to ~1 ulp
// (numpy's SIMD log/cos vs CUDA's libdevice).
#include "common.cuh"

namespace rq {

RQ_DEV uint64_t splitmix_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
RQ_DEV uint64_t splitmix_word(uint64_t seed, uint64_t idx) {
  return splitmix_mix(seed + (idx + 1ull) * 0x9E3779B97F4A7C15ull);
}
RQ_DEV double normal_draw(uint64_t seed, uint64_t k) {
  const uint64_t r1 = splitmix_word(seed, 2ull * k);
  const uint64_t r2 = splitmix_word(seed, 2ull * k + 1ull);
  const double u1 = ((double)(r1 >> 11) + 1.0) * 0x1.0p-53;
  const double u2 = (double)(r2 >> 11) * 0x1.0p-53;
  // numpy evaluates 2.0 * np.pi * u2 as (2*pi) * u2
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

// Column-major rows x cols fill; element (i, c) is draw counter + c*rows + i.
__global__ void gaussian_fill_kernel(double* __restrict__ out, int64_t rows, int64_t cols, int64_t ld,
                                     uint64_t seed, uint64_t counter) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = idx / rows, i = idx - c * rows;
    out[c * ld + i] = normal_draw(seed, counter + (uint64_t)idx);
  }
}

__global__ void splitmix_words_kernel(uint64_t* out, uint64_t seed, uint64_t first, int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = splitmix_word(seed, first + (uint64_t)i);
}

int gaussian_fill(double* out, int64_t rows, int64_t cols, int64_t ld, uint64_t seed, uint64_t counter,
                  cudaStream_t st, int64_t* launches) {
  if (rows <= 0 || cols <= 0) return RQ_OK;
  const int64_t total = rows * cols;
  int blocks = (int)ceil_div(total, 256);
  if (blocks > 16 * kSMs) blocks = 16 * kSMs;
  gaussian_fill_kernel<<<blocks, 256, 0, st>>>(out, rows, cols, ld, seed, counter);
  RQ_CUDA_TRY(cudaGetLastError());
  if (launches) (*launches)++;
  return RQ_OK;
}

int splitmix_words(uint64_t* out, uint64_t seed, uint64_t first, int64_t count, cudaStream_t st,
                   int64_t* launches) {
  if (count <= 0) return RQ_OK;
  int blocks = (int)ceil_div(count, 256);
  if (blocks > 4 * kSMs) blocks = 4 * kSMs;
  splitmix_words_kernel<<<blocks, 256, 0, st>>>(out, seed, first, count);
  RQ_CUDA_TRY(cudaGetLastError());
  if (launches) (*launches)++;
  return RQ_OK;
}

}  // namespace rq
