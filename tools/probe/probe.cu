// Microbenchmarks that fix the design constants on B200 (sm_100a):
// DFMA vs DMMA throughput, grid-barrier and cluster-barrier latency.
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void dfma_peak(double* out, int iters) {
  double a[16];
  for (int i = 0; i < 16; i++) a[i] = threadIdx.x * 1e-9 + i;
  double x = 1.0000001, y = 0.9999999;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) a[i] = fma(a[i], x, y);
  }
  double s = 0;
  for (int i = 0; i < 16; i++) s += a[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void dmma_peak(double* out, int iters) {
  double c[8][4];
  for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) c[i][j] = 0;
  double a0 = threadIdx.x * 1e-3, a1 = 1.0, b0 = 0.5;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b0));
  }
  double s = 0;
  for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) s += c[i][j];
  if (s == 12345.0) out[0] = s;
}

__global__ void grid_bar(unsigned* ctr, int iters, double* out) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; i++) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = 1;
}

// hand-rolled barrier: one atomic per CTA, generation counter
__device__ __forceinline__ void my_grid_barrier(unsigned* bar, unsigned nblocks, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    gen++;
    unsigned target = gen * nblocks;
    __threadfence();
    atomicAdd(bar, 1u);
    while (true) {
      unsigned v;
      asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(bar));
      if (v >= target) break;
    }
  }
  __syncthreads();
}
__global__ void grid_bar2(unsigned* bar, int iters, double* out) {
  unsigned gen = 0;
  for (int i = 0; i < iters; i++) my_grid_barrier(bar, gridDim.x, gen);
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = 1;
}

__global__ void cluster_bar(int iters, double* out) {
  cg::cluster_group cl = cg::this_cluster();
  for (int i = 0; i < iters; i++) cl.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = 1;
}

int main() {
  double* out; cudaMalloc(&out, 1024);
  unsigned* ctr; cudaMalloc(&ctr, 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float ms;
  for (int warps : {4, 8, 16, 32}) {
    int iters = 4000;
    dfma_peak<<<sms * 2, warps * 32>>>(out, 10);
    cudaEventRecord(e0);
    dfma_peak<<<sms * 2, warps * 32>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * iters * (double)sms * 2 * warps * 32;
    printf("{\"probe\":\"dfma\",\"warps_per_cta\":%d,\"tflops\":%.2f}\n", warps, fl / ms / 1e9);
  }
  for (int warps : {4, 8, 16}) {
    int iters = 2000;
    dmma_peak<<<sms * 2, warps * 32>>>(out, 10);
    cudaEventRecord(e0);
    dmma_peak<<<sms * 2, warps * 32>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * 8 * 4 * 8.0 * iters * (double)sms * 2 * warps;
    printf("{\"probe\":\"dmma_m16n8k4\",\"warps_per_cta\":%d,\"tflops\":%.2f}\n", warps, fl / ms / 1e9);
  }
  for (int nb : {16, 32, 64, 148}) {
    int iters = 2000;
    void* args[] = {&ctr, &iters, &out};
    cudaLaunchCooperativeKernel((void*)grid_bar, nb, 256, args, 0, 0);
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((void*)grid_bar, nb, 256, args, 0, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"probe\":\"cg_grid_sync\",\"ctas\":%d,\"us_per_barrier\":%.3f}\n", nb, ms * 1e3 / iters);
    cudaMemset(ctr, 0, 4);
    cudaLaunchCooperativeKernel((void*)grid_bar2, nb, 256, args, 0, 0);
    cudaDeviceSynchronize();
    cudaMemset(ctr, 0, 4);
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((void*)grid_bar2, nb, 256, args, 0, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"probe\":\"atomic_grid_barrier\",\"ctas\":%d,\"us_per_barrier\":%.3f}\n", nb, ms * 1e3 / iters);
  }
  for (int cs : {2, 4, 8, 16}) {
    int iters = 20000;
    cudaFuncSetAttribute(cluster_bar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs); cfg.blockDim = dim3(256);
    cudaLaunchAttribute attr; attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = cs; attr.val.clusterDim.y = 1; attr.val.clusterDim.z = 1;
    cfg.attrs = &attr; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, cluster_bar, iters, out);
    cudaEventRecord(e0);
    cudaError_t err = cudaLaunchKernelEx(&cfg, cluster_bar, iters, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"probe\":\"cluster_sync\",\"cluster\":%d,\"us_per_barrier\":%.4f,\"err\":\"%s\"}\n", cs, ms * 1e3 / iters, cudaGetErrorString(err));
  }
  // launch latency
  {
    int iters = 1000;
    cudaEventRecord(e0);
    for (int i = 0; i < iters; i++) dfma_peak<<<1, 32>>>(out, 1);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"probe\":\"empty_launch_stream\",\"us_per_launch\":%.3f}\n", ms * 1e3 / iters);
  }
  printf("{\"probe\":\"done\",\"err\":\"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
