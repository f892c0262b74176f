// Probe: cooperative launch combined with thread-block clusters; max active clusters.
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__global__ void __launch_bounds__(256, 1) k_coop_cluster(int* out) {
  __shared__ double pad[20000];  // ~160 KB: one CTA per SM
  pad[threadIdx.x] = threadIdx.x;
  cg::grid_group g = cg::this_grid();
  g.sync();
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    out[blockIdx.x] = (int)smid + (int)pad[1] * 0;
  }
}

int main() {
  int* d;
  cudaMalloc(&d, 4096 * sizeof(int));
  cudaFuncSetAttribute(k_coop_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 0;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(cs);
    int nclusters = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&nclusters, (void*)k_coop_cluster, &cfg);
    cfg.numAttrs = 2;
    cfg.gridDim = dim3(cs * (nclusters > 0 ? nclusters : 1));
    cudaError_t e2 = cudaLaunchKernelEx(&cfg, k_coop_cluster, d);
    cudaError_t e3 = cudaDeviceSynchronize();
    printf("{\"probe\":\"coop_cluster\",\"cluster\":%d,\"max_active_clusters\":%d,\"occ_err\":\"%s\",\"launch\":\"%s\",\"sync\":\"%s\"}\n",
           cs, nclusters, cudaGetErrorString(e), cudaGetErrorString(e2), cudaGetErrorString(e3));
    cudaGetLastError();
  }
  return 0;
}
