// Grid-barrier cost vs participating CTAs (cooperative launch of 148 x 512).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void k_cg(int iters, unsigned long long* out) {
  cg::grid_group g = cg::this_grid();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) g.sync();
  unsigned long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}

__global__ void k_custom(int iters, int nPart, unsigned* ctr, unsigned long long* out) {
  if ((int)blockIdx.x >= nPart) return;
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(ctr, 1u);
      const unsigned target = (unsigned)nPart * (unsigned)(i + 1);
      while (ld_acquire(ctr) < target) {
      }
    }
    __syncthreads();
  }
  unsigned long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[1] = (t1 - t0) / iters;
}

int main() {
  unsigned long long* o;
  unsigned* c;
  cudaMallocManaged(&o, 64);
  cudaMalloc(&c, 4);
  int iters = 1000;
  void* a1[] = {&iters, &o};
  cudaLaunchCooperativeKernel((void*)k_cg, 148, 512, a1, 0, 0);
  cudaDeviceSynchronize();
  std::printf("cg grid.sync over 148 CTAs: %llu cycles\n", o[0]);
  for (int n : {148, 74, 37, 16, 8}) {
    cudaMemset(c, 0, 4);
    void* a2[] = {&iters, &n, &c, &o};
    cudaLaunchCooperativeKernel((void*)k_custom, 148, 512, a2, 0, 0);
    cudaDeviceSynchronize();
    std::printf("custom barrier over %3d CTAs: %llu cycles\n", n, o[1]);
  }
  return 0;
}
