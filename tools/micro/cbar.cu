// barrier.cluster latency (cluster of N CTAs x 512 threads).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cl(int iters, unsigned long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  unsigned long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}
__global__ void k_cta(int iters, unsigned long long* out) {
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  unsigned long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[1] = (t1 - t0) / iters;
}

int main() {
  unsigned long long* o;
  cudaMallocManaged(&o, 64);
  int iters = 1000;
  for (int n : {2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(n);
    cfg.blockDim = dim3(512);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = n;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (n > 8) cudaFuncSetAttribute(k_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_cl, iters, o);
    cudaError_t e2 = cudaDeviceSynchronize();
    std::printf("cluster %2d: %llu cycles per barrier (%s %s)\n", n, o[0], cudaGetErrorString(e), cudaGetErrorString(e2));
  }
  k_cta<<<1, 512>>>(iters, o);
  cudaDeviceSynchronize();
  std::printf("__syncthreads 512: %llu cycles\n", o[1]);
  return 0;
}
