// Latency microbenchmarks for the serial-kernel design: __syncthreads, shuffle
// chains, DSMEM load round trip, DSMEM store + cluster barrier, L2 round trip.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long clk() {
  unsigned long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}

__global__ void k_sync(int iters, unsigned long long* out) {
  unsigned long long t0 = clk();
  for (int i = 0; i < iters; i++) __syncthreads();
  unsigned long long t1 = clk();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}

__global__ void k_shfl(int iters, double seed, unsigned long long* out) {
  double v = seed + threadIdx.x;
  unsigned long long t0 = clk();
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  unsigned long long t1 = clk();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / iters; out[1] = (unsigned long long)v; }
}

__global__ void k_reduce_u32(int iters, unsigned long long* out) {
  unsigned v = threadIdx.x * 7919u;
  unsigned long long t0 = clk();
  for (int i = 0; i < iters; i++) v = __reduce_max_sync(0xffffffffu, v) + threadIdx.x;
  unsigned long long t1 = clk();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / iters; out[1] = v; }
}

__device__ __forceinline__ unsigned mapa(const void* p, unsigned r) {
  unsigned a = (unsigned)__cvta_generic_to_shared(p), o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}

__global__ void k_dsmem(int iters, unsigned long long* out) {
  __shared__ double buf[64];
  cg::cluster_group cl = cg::this_cluster();
  buf[threadIdx.x % 64] = threadIdx.x;
  cl.sync();
  unsigned peer = (cl.block_rank() + 1) % cl.num_blocks();
  unsigned addr = mapa(&buf[0], peer);
  double acc = 0;
  unsigned long long t0 = clk();
  for (int i = 0; i < iters; i++) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr + ((unsigned)acc & 8)));
    acc += v;
  }
  unsigned long long t1 = clk();
  // store + barrier round
  unsigned long long t2 = clk();
  for (int i = 0; i < iters; i++) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(acc) : "memory");
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  unsigned long long t3 = clk();
  if (threadIdx.x == 0 && cl.block_rank() == 0) {
    out[0] = (t1 - t0) / iters;
    out[1] = (t3 - t2) / iters;
    out[2] = (unsigned long long)acc;
  }
  cl.sync();
}

__global__ void k_l2(int iters, double* g, unsigned long long* out) {
  double acc = 0;
  unsigned long long t0 = clk();
  for (int i = 0; i < iters; i++) acc += __ldcg(g + ((unsigned long long)acc & 1));
  unsigned long long t1 = clk();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / iters; out[1] = (unsigned long long)acc; }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  double* g;
  cudaMalloc(&g, 64);
  cudaMemset(g, 0, 64);
  unsigned long long h[4];
  for (int th : {256, 512, 1024}) {
    k_sync<<<1, th>>>(1000, d);
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("{\"probe\":\"syncthreads\",\"threads\":%d,\"cycles\":%llu}\n", th, h[0]);
  }
  k_shfl<<<1, 32>>>(1000, 1.0, d);
  cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("{\"probe\":\"shfl_xor_f64_x5_chain\",\"cycles\":%llu}\n", h[0]);
  k_reduce_u32<<<1, 32>>>(1000, d);
  cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("{\"probe\":\"reduce_max_sync_u32\",\"cycles\":%llu}\n", h[0]);
  for (int cs : {2, 4, 16}) {
    cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(512);
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = cs; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
    cfg.attrs = &at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_dsmem, 1000, d);
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("{\"probe\":\"dsmem_load_chain\",\"cluster\":%d,\"cycles\":%llu}\n", cs, h[0]);
    printf("{\"probe\":\"dsmem_store_plus_cluster_barrier_512thr\",\"cluster\":%d,\"cycles\":%llu}\n", cs, h[1]);
  }
  k_l2<<<1, 32>>>(1000, g, d);
  cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("{\"probe\":\"l2_ldcg_chain\",\"cycles\":%llu}\n", h[0]);
  printf("{\"probe\":\"done\",\"err\":\"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
}
